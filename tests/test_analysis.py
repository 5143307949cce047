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


@pytest.mark.gpu
@pytest.mark.parametrize("dataset,kind,param", [("lpsc105", "lf_target", 134), ("lpsc105", "lf_target", 56),
                                                 ("cnae", "lf_tol", 0.5)])
def test_compare_methods_rows_next_to_reference(gpu, ref, dataset, kind, param):
    """The GPU's compare_methods rows against the reference's own (oracle/_ref: the
    same loop, analysis.cpp:137-211, on the reference's PreparedMethod, same rhs):
    identical method / clustering / f_c columns; iteration columns within +-2 for
    the solves of up to 100 iterations.  CNAE's plain and Jacobi CG (656 / 241
    iterations on an 856-dimensional beta = 1e-6 system) follow the summation order
    (DESIGN.md §5): CG is held to its measured envelope, Jacobi CG to the rows
    existing side by side."""
    import json
    import os

    import oracle
    from helpers import golden_matrix, load_golden
    x = golden_matrix(load_golden(dataset))
    m = R.DeviceMatrix(x)
    ck = R.LEADER_TARGET if kind == "lf_target" else R.LEADER_TOLERANCE
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=ck, target_size=param if kind == "lf_target" else 0,
                                                   tolerance=param if kind == "lf_tol" else 1.0))
    olv = [dict(clustering_kind=oracle.CLUSTER_LEADER_TARGET if kind == "lf_target" else
                oracle.CLUSTER_LEADER_TOLERANCE, target_size=param if kind == "lf_target" else 0,
                tolerance=param if kind == "lf_tol" else 1.0)]
    names = ["cg", "jacobi_cg", "fcg_twolevel", "fgmres_twolevel"]
    gspecs = [R.MethodSpec(kind=R.method_from_string(n), levels=[lv] if "level" in n else []) for n in names]
    rows = R.compare_methods(m, dataset, [1e-6], [1e-6], gspecs, n_repeats=1)
    om = ref.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
    rrows = oracle.compare_methods(ref, om, dataset, [1e-6], [1e-6], [(n, olv if "level" in n else []) for n in names])
    env = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "envelope.json")))
    for g, r in zip(rows, rrows):
        assert (g.method, g.clustering, g.f_c) == (r["method"], r["clustering"], r["f_c"]), (g, r)
        if dataset == "cnae" and g.method == "cg":
            lo, hi = env["cnae"]["cg_iterations_range"]
            assert lo - 2 <= g.iterations <= hi + 2, (g.iterations, r["iterations"])
        elif r["iterations"] > 100:
            assert g.iterations > 0
        else:
            assert abs(g.iterations - r["iterations"]) <= 2, (g.method, g.iterations, r["iterations"])
