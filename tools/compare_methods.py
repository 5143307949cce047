"""compare_methods / to_csv (analysis.cpp:137-223) on the GPU: CSV rows in the
reference's schema for a BASELINE config or a Matrix Market file.

usage: python tools/compare_methods.py [cfg1|cfg2|path.mtx] [--beta 1e-2 1] [--tol 1e-6]
       [--methods cg fcg_twolevel fgmres_twolevel] [--k 50] [--repeats 3]
(The reference's own CPU rows come from `bench.py --impl reference`.)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_05826_b200 as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dataset", nargs="?", default="cfg1")
    ap.add_argument("--beta", type=float, nargs="+", default=[1e-2])
    ap.add_argument("--tol", type=float, nargs="+", default=[1e-6])
    ap.add_argument("--methods", nargs="+", default=["cg", "jacobi_cg", "fcg_twolevel", "fgmres_twolevel"])
    ap.add_argument("--k", type=int, default=50, help="k-means clusters of the two-level methods")
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()
    if args.dataset.endswith(".mtx"):
        x = R.read_matrix_market(args.dataset)
        m = R.DeviceMatrix(x)
    else:
        import bench
        cfg = bench.CONFIGS[args.dataset]
        x = bench.make_matrix(cfg)
        m = R.DeviceMatrix.from_dense(x.dense()) if cfg["kind"] == "dense" else R.DeviceMatrix(x)
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=args.k),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    methods = [R.MethodSpec(kind=R.method_from_string(n), levels=[lv] if "level" in n else [])
               for n in args.methods]
    rows = R.compare_methods(m, os.path.basename(args.dataset), args.beta, args.tol, methods, args.repeats)
    sys.stdout.write(R.to_csv(rows))


if __name__ == "__main__":
    main()
