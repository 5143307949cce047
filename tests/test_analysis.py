"""The bench harness mirror (analysis.cpp:137-223): CSV schema and formatting
(CPU) and compare_methods on the GPU."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix


def test_to_csv_schema_and_precision():
    rows = [R.BenchRow("d", "cg", "", 0, 0.1, 1e-6, 3, 0.0012345678901234, 1.0),
            R.BenchRow("d", "fcg_twolevel", "km(k=5)", 5, 0.1, 1e-6, 2, 0.5, 2.5)]
    lines = R.to_csv(rows).splitlines()
    assert lines[0] == "dataset,method,clustering,f_c,beta,tol,iterations,wall_time_s,speedup"
    assert lines[1] == "d,cg,,0,0.1,1e-06,3,0.00123456789012,1"  # ostream precision(12)
    assert lines[2] == "d,fcg_twolevel,km(k=5),5,0.1,1e-06,2,0.5,2.5"


def test_clustering_description():
    def spec(kind, **kw):
        return R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[R.LevelSpec(clustering=R.ClusteringChoice(kind=kind, **kw))])
    assert R.clustering_description(spec(R.KMEANS, target_size=9), 9) == "km(k=9)"
    assert R.clustering_description(spec(R.LEADER_TARGET, target_size=9), 8) == "lf(fc=8)"
    assert R.clustering_description(spec(R.LEADER_TOLERANCE, tolerance=0.5), 7) == "lf(tol=0.5,fc=7)"
    assert R.clustering_description(R.MethodSpec(kind=R.CG), 0) == ""


def test_compare_methods_validation():
    with pytest.raises(ValueError):
        R.compare_methods(None, "d", [], [1e-6], [R.MethodSpec()])


@pytest.mark.gpu
def test_compare_methods_gpu(gpu):
    x = random_matrix(200, 80, 5, 0.3)
    m = R.DeviceMatrix(x, R.default_context())
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=10),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    methods = [R.MethodSpec(kind=R.CG), R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]),
               R.MethodSpec(kind=R.FGMRES_TWOLEVEL, levels=[lv])]
    rows = R.compare_methods(m, "rnd", [1e-2, 1.0], [1e-6], methods, n_repeats=2)
    assert len(rows) == 6
    assert [r.method for r in rows[:3]] == ["cg", "fcg_twolevel", "fgmres_twolevel"]
    for r in rows:
        assert r.iterations > 0 and r.wall_time_s > 0.0
        if r.method == "cg":
            assert r.speedup == 1.0 and r.f_c == 0
        else:
            assert r.clustering == "km(k=10)" and r.f_c == 10 and r.speedup > 0.0
    b = R.generate_rhs(m, 42).b
    sol = R.solve_system(m, 1e-2, b, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]))
    assert rows[1].iterations == sol.report.iterations
