"""Probe: BASELINE cfg 3's batched pcg_vcycle solve (16 right-hand sides, one beta),
with a cudaProfilerStart/Stop window around exactly one timed batch so that
`ncu --profile-from-start off` lists only its launches.  Also prints the
per-level sizes and (optional, `cg`) the plain / Jacobi CG iteration counts per beta.

usage: python tools/probe_cfg3_batch.py [beta] [cg]
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
      --log-file gpurun_out/cfg3_batch.csv python tools/probe_cfg3_batch.py 1
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1806_05826_b200 as R

beta = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = bench.CONFIGS["cfg3"]
t0 = time.time()
ctx = R.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x, ctx)
spec = R.MethodSpec(kind=R.PCG_VCYCLE if "mult" in sys.argv[2:] else R.PCG_VCYCLE_ADDITIVE, levels=bench.level_specs(cfg), solver=R.SolverConfig(cfg["tol"], 1000))
pm = R.PreparedMethod(m, beta, spec)
print(f"setup {time.time() - t0:.1f} s", flush=True)
for k in range(pm.n_levels):
    print("level", k, pm.level(k) if k else {"n_features": x.n_features, "nnz": m.nnz}, flush=True)
nb = cfg["n_rhs"]
bcm = torch.stack([torch.from_numpy(R.rng_normals(42 + k, x.n_samples)) for k in range(nb)], 0).cuda().contiguous()
wcm = torch.empty(nb, x.n_features, dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    if rep == 2:
        torch.cuda.profiler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    R.ridgemg._lib.check(pm.lib.rmg_method_solve_batch(pm.h, bcm.data_ptr(), wcm.data_ptr(), nb, None, 1))
    e1.record(stream)
    torch.cuda.synchronize()
    if rep == 2:
        torch.cuda.profiler.stop()
    print(f"batch {rep}: {e0.elapsed_time(e1):.2f} ms ({e0.elapsed_time(e1) / nb:.3f} ms per rhs)", flush=True)
if "cg" in sys.argv[2:]:
    b = torch.from_numpy(R.rng_normals(42, x.n_samples)).cuda()
    w = torch.empty(x.n_features, dtype=torch.float64, device="cuda")
    for kind, name in ((R.JACOBI_CG, "jacobi_cg"), (R.CG, "cg")):
        for bt in cfg["betas"][::-1]:
            pc = R.PreparedMethod(m, bt, R.MethodSpec(kind=kind, solver=R.SolverConfig(1e-6, 400000)))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = pc.solve_device(b.data_ptr(), w.data_ptr())
            e1.record(stream)
            torch.cuda.synchronize()
            print(f"{name} beta {bt:g}: {rep.iterations} iterations, converged {rep.converged}, "
                  f"{e0.elapsed_time(e1):.1f} ms, |w| {float(torch.linalg.norm(w)):.12e}", flush=True)
            pc.close()
