"""Probe: the cfg 3 block operator (k = 16) alone: time per apply (host-timed, synced,
L2 flushed, median of 10) and each column against the single-vector operator.
usage: [RMG_BLOCK_K1V2=0|1|2] python tools/probe_block.py [n_applies_only]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1806_05826_b200 as R

only = len(sys.argv) > 1
t0 = time.time()
x = R.synth_sparse_zipf(1_000_000, 100_000, 50.0, 1.1, True, 0, row_streams=True)
t1 = time.time()
m = R.DeviceMatrix(x)
t2 = time.time()
K = 16
vb = torch.randn(x.n_features, K, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
ob = torch.empty_like(vb)
lib = m.lib


def blk():
    R.ridgemg._lib.check(lib.rmg_ridge_apply_block(m.h, 1.0, vb.data_ptr(), ob.data_ptr(), K, 1))


if only:
    for _ in range(int(sys.argv[1])):
        blk()
    sys.exit(0)
for _ in range(3):
    blk()
flushbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flushbuf.random_(0, 255)
    torch.cuda.synchronize()
    t = time.perf_counter()
    blk()
    ts.append(time.perf_counter() - t)
tb = sorted(ts)[len(ts) // 2]
bb = 2 * m.nnz * 12 + 4 * (x.n_samples + 1) + 4 * (x.n_features + 1) + K * 8 * (x.n_features + 2 * x.n_samples + 2 * x.n_features)
print(f"mode K1V2={os.environ.get('RMG_BLOCK_K1V2', 'default')} gen {t1-t0:.1f}s upload {t2-t1:.1f}s block k={K}: "
      f"{tb*1e6:.1f} us/apply -> {bb/tb/1e9:.0f} GB/s", flush=True)
worst = 0.0
for q in (0, 3, 7, 8, 15):
    col = m.ridge_apply(1.0, vb[:, q].cpu().numpy())
    worst = max(worst, float(np.linalg.norm(ob[:, q].cpu().numpy() - col) / np.linalg.norm(col)))
print("block columns vs single applies: worst rel", worst, flush=True)
