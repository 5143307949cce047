"""Probe: dense X with 16 right-hand sides on cfg 4's per-GPU shard
(500 k x 1024, fp32 storage): the DMMA SYRK (G = X^T X), the block apply (DMMA GEMM) and
the one-sweep X^T B (k_xtb_dmma), each timed with CUDA events and checked against torch.
usage: python tools/probe_dense_multi.py [rows]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1806_05826_b200 as R

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
a = bench.cfg4_shard_matrix(n=rows)
ctx = R.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
m = R.DeviceMatrix.from_dense(a, ctx)
K, F = 16, a.shape[1]
vb = torch.randn(F, K, dtype=torch.float64, device="cuda")
ob = torch.empty_like(vb)
lib = m.lib


def blk():
    R.ridgemg._lib.check(lib.rmg_ridge_apply_block(m.h, 1e-4, vb.data_ptr(), ob.data_ptr(), K, 1))


torch.cuda.synchronize()
t0 = time.perf_counter()
blk()
torch.cuda.synchronize()
t_syrk = time.perf_counter() - t0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(50):
    blk()
e1.record(stream)
torch.cuda.synchronize()
xd = torch.from_numpy(a).cuda()
want = torch.zeros(F, K, dtype=torch.float64, device="cuda")
for r in range(0, rows, 1 << 18):
    xb = xd[r:r + (1 << 18)].double()
    want += xb.T @ (xb @ vb)
want += 1e-4 * vb
flops = 2.0 * rows * F * F / 2  # the upper triangle
print(f"rows {rows}: SYRK + first apply {t_syrk*1e3:.1f} ms ({flops / t_syrk / 1e12:.1f} TFLOP/s of the triangle), "
      f"block apply {e0.elapsed_time(e1) / 50 * 1e3:.1f} us, rel vs torch {float(torch.linalg.norm(ob - want) / torch.linalg.norm(want)):.2e}",
      flush=True)
# X^T B through a batched jacobi_cg solve's rhs: time the solve_batch with max_iters = 1
pm = R.PreparedMethod(m, 1e-4, R.MethodSpec(kind=R.JACOBI_CG, solver=R.SolverConfig(1e-6, 1)))
bcm = torch.randn(K, rows, dtype=torch.float64, device="cuda")
wcm = torch.empty(K, F, dtype=torch.float64, device="cuda")
reps = (R.ridgemg._lib.SolveReportC * K)()
for _ in range(2):
    lib.rmg_method_solve_batch(pm.h, bcm.data_ptr(), wcm.data_ptr(), K, reps, 1)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(5):
    lib.rmg_method_solve_batch(pm.h, bcm.data_ptr(), wcm.data_ptr(), K, reps, 1)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
gb = a.nbytes / 1e9
print(f"one-iteration batch (X^T B sweep + 1 PCG iteration): {ms:.3f} ms; X is {gb:.2f} GB -> >= {gb / (ms * 1e-3) / 1e3:.2f} TB/s "
      f"if the sweep were all of it", flush=True)
