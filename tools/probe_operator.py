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
elif name == "cfg3":  # cfg 3 operator: N=1M x F=100k, ~50 nnz/row, |N(0,1)|, Zipf(1.1); 16-RHS block
    x = R.synth_sparse_zipf(1_000_000, 100_000, 50.0, 1.1, True, 0, row_streams=True)
elif name == "cfg4shard":  # cfg4 per-GPU shard at 8 GPUs: 500k of its 4M rows, fp32 storage
    dense = bench.cfg4_shard_matrix()
    import types
    x = types.SimpleNamespace(n_samples=dense.shape[0], n_features=dense.shape[1])
elif name == "cfg5full":  # cfg5 on one GPU: all 16M rows
    x = R.synth_sparse_zipf(16_000_000, 500_000, 64.0, 1.05, False, 0, row_streams=True)
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
if name == "cfg3":
    import torch
    K = 16
    vb = torch.randn(x.n_features, K, dtype=torch.float64, device="cuda")
    ob = torch.empty_like(vb)
    lib = m.lib
    def blk():
        R.ridgemg._lib.check(lib.rmg_ridge_apply_block(m.h, 1.0, vb.data_ptr(), ob.data_ptr(), K, 1))
    for _ in range(3):
        blk()
    flushbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(10):
        flushbuf.random_(0, 255)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blk()
        ts.append(time.perf_counter() - t0)
    tb = sorted(ts)[len(ts) // 2]
    bb = 2 * m.nnz * 12 + 4 * (x.n_samples + 1) + 4 * (x.n_features + 1) + K * 8 * (x.n_features + 2 * x.n_samples + 2 * x.n_features)
    print(f"block k={K}: {tb*1e6:.1f} us/apply (host-timed, synced) -> {bb/tb/1e9:.0f} GB/s = {bb/tb/1e9/6549.1:.3f}; "
          f"per RHS {tb*1e6/K:.1f} us vs single apply {t*1e3:.1f} us")
    col = m.ridge_apply(1.0, vb[:, 3].cpu().numpy())
    print("block column vs single apply rel", np.linalg.norm(ob[:, 3].cpu().numpy() - col) / np.linalg.norm(col))
if name == "cfg4shard":
    u = np.random.default_rng(1).standard_normal(dense.shape[0])
    got = m.spmv_transpose(u)
    want = dense.astype(np.float64).T @ u
    print("X^T u vs numpy: rel", np.linalg.norm(got - want) / np.linalg.norm(want))
elif name not in ("cfg2", "cfg3", "cfg5full"):
    print("hybrid hot features:", m.hybrid_hot_features(), flush=True)
    u = np.random.default_rng(1).standard_normal(x.n_samples)
    got = m.spmv_transpose(u)
    rows = np.repeat(np.arange(x.n_samples), np.diff(x.row_offsets.astype(np.int64)))
    want = np.bincount(x.column_indices.astype(np.int64), weights=u[rows], minlength=x.n_features)
    print("X^T u vs numpy: rel", np.linalg.norm(got - want) / np.linalg.norm(want))
