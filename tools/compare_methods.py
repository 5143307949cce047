"""compare_methods / to_csv (analysis.cpp:137-223) on the GPU: CSV rows in the
reference's schema for a BASELINE config, a bundled dataset or a Matrix Market file;
with --with-reference, the reference's own rows (oracle/_ref: its PreparedMethod,
same loop, same rhs seed) are placed next to the GPU's.

usage: python tools/compare_methods.py [cfg1|cfg2|lpsc105|cnae|path.mtx] [--beta 1e-2 1] [--tol 1e-6]
       [--methods cg jacobi_cg fcg_twolevel fgmres_twolevel] [--k 50] [--lf-target N] [--lf-tol T]
       [--repeats 3] [--with-reference]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1806_05826_b200 as R  # noqa: E402

JOINED = ("dataset,method,clustering,f_c,beta,tol,iterations,iterations_reference,wall_time_s,"
          "wall_time_s_reference,speedup,speedup_reference")


def load(dataset):
    if dataset.endswith(".mtx"):
        return R.read_matrix_market(dataset), False
    if dataset in ("lpsc105", "cnae"):
        from helpers import golden_matrix, load_golden
        return golden_matrix(load_golden(dataset)), False
    import bench
    cfg = bench.CONFIGS[dataset]
    return bench.make_matrix(cfg), cfg["kind"] == "dense"


def specs(args):
    """(GPU MethodSpec, reference (name, level dicts)) per requested method"""
    import oracle
    if args.lf_target:
        lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TARGET, target_size=args.lf_target))
        olv = [dict(clustering_kind=oracle.CLUSTER_LEADER_TARGET, target_size=args.lf_target)]
    elif args.lf_tol:
        lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TOLERANCE, tolerance=args.lf_tol))
        olv = [dict(clustering_kind=oracle.CLUSTER_LEADER_TOLERANCE, tolerance=args.lf_tol)]
    else:
        lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=args.k))
        olv = [dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=args.k)]
    out = []
    for n in args.methods:
        two = "level" in n
        out.append((R.MethodSpec(kind=R.method_from_string(n), levels=[lv] if two else []), (n, olv if two else [])))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dataset", nargs="?", default="cfg1")
    ap.add_argument("--beta", type=float, nargs="+", default=[1e-2])
    ap.add_argument("--tol", type=float, nargs="+", default=[1e-6])
    ap.add_argument("--methods", nargs="+", default=["cg", "jacobi_cg", "fcg_twolevel", "fgmres_twolevel"])
    ap.add_argument("--k", type=int, default=50, help="k-means clusters of the two-level methods")
    ap.add_argument("--lf-target", type=int, default=0, help="leader-follower closest to this coarse size")
    ap.add_argument("--lf-tol", type=float, default=0.0, help="leader-follower tolerance")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--with-reference", action="store_true")
    args = ap.parse_args()
    x, dense = load(args.dataset)
    m = R.DeviceMatrix.from_dense(x.dense()) if dense else R.DeviceMatrix(x)
    pairs = specs(args)
    name = os.path.basename(args.dataset)
    rows = R.compare_methods(m, name, args.beta, args.tol, [p[0] for p in pairs], args.repeats)
    if not args.with_reference:
        sys.stdout.write(R.to_csv(rows))
        return
    import oracle
    chk = oracle.Checker("ref" if oracle.available("ref") else "oracle")
    om = chk.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
    ref = oracle.compare_methods(chk, om, name, args.beta, args.tol, [p[1] for p in pairs], args.repeats)
    print(JOINED)
    for g, r in zip(rows, ref):
        print(f"{g.dataset},{g.method},{g.clustering},{g.f_c},{g.beta:g},{g.tol:g},{g.iterations},{r['iterations']},"
              f"{g.wall_time_s:.6g},{r['wall_time_s']:.6g},{g.speedup:.6g},{r['speedup']:.6g}")


if __name__ == "__main__":
    main()
