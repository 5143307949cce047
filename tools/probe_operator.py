"""Probe: XᵀX operator timing (cold / warm L2) + parity vs the oracle.
usage: python tools/probe_operator.py [cfg2|cfg5shard]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1806_05826_b200 as R
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
t0 = time.time()
dense = None
if name == "cfg2":
    x = bench.make_matrix(bench.CONFIGS["cfg2"])
elif name == "cfg4shard":  # cfg4 per-GPU shard at 8 GPUs: 500k of its 4M rows, fp32 storage
    dense = bench.cfg4_shard_matrix()
    import types
    x = types.SimpleNamespace(n_samples=dense.shape[0], n_features=dense.shape[1])
else:  # cfg5 per-GPU shard at 4 GPUs: 4M of its 16M rows
    x = R.synth_sparse_zipf(4_000_000, 500_000, 64.0, 1.05, False, 0, row_streams=True)
t1 = time.time()
m = R.DeviceMatrix.from_dense(dense) if dense is not None else R.DeviceMatrix(x)
t2 = time.time()
print(f"{name}: N={x.n_samples} F={x.n_features} nnz={m.nnz} gen {t1-t0:.1f}s upload {t2-t1:.1f}s", flush=True)
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.CG))
fb = (bench.dense_algorithmic_bytes(*dense.shape, 4) if dense is not None
      else bench.algorithmic_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern))
for flush in (True, False):
    t, k1, k2 = pm.time_operator(0, 20, flush)
    print(f"{'cold' if flush else 'warm'}: {t*1e3:.1f} us/apply (K1 {k1*1e3:.1f}, K2 {k2*1e3:.1f}) -> {fb/(t*1e6):.0f} GB/s "
          f"= {fb/(t*1e6)/6549.1:.3f} of 6549", flush=True)
if name == "cfg2":
    import oracle
    o = oracle.Checker("oracle")
    om = o.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices)
    w = np.random.default_rng(0).standard_normal(x.n_features)
    got, want = m.ridge_apply(1.0, w), o.ridge_apply(om, 1.0, w)
    print("parity rel", np.linalg.norm(got - want) / np.linalg.norm(want))
    t_got, t_want = m.spmv(w), o.spmv(om, w)
    print("K1 bit-exact vs oracle:", bool(np.array_equal(t_got, t_want)),
          "max abs diff", float(np.max(np.abs(t_got - t_want))))
if name == "cfg4shard":
    u = np.random.default_rng(1).standard_normal(dense.shape[0])
    got = m.spmv_transpose(u)
    want = dense.astype(np.float64).T @ u
    print("X^T u vs numpy: rel", np.linalg.norm(got - want) / np.linalg.norm(want))
elif name != "cfg2":
    print("hybrid hot features:", m.hybrid_hot_features(), flush=True)
    u = np.random.default_rng(1).standard_normal(x.n_samples)
    got = m.spmv_transpose(u)
    rows = np.repeat(np.arange(x.n_samples), np.diff(x.row_offsets.astype(np.int64)))
    want = np.bincount(x.column_indices.astype(np.int64), weights=u[rows], minlength=x.n_features)
    print("X^T u vs numpy: rel", np.linalg.norm(got - want) / np.linalg.norm(want))
