"""Probe: cfg 3 batched solve, device buffers vs pinned host buffers, with and without
a beta change before each call (graph rebuild), wall-clock per call.
usage: python tools/probe_e2e.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1806_05826_b200 as R

cfg = bench.CONFIGS["cfg3"]
ctx = R.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x, ctx)
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.PCG_VCYCLE, levels=bench.level_specs(cfg),
                                           solver=R.SolverConfig(1e-6, 1000)))
nb = 16
bcm = torch.stack([torch.from_numpy(R.rng_normals(42 + k, x.n_samples)) for k in range(nb)], 0).cuda().contiguous()
wcm = torch.empty(nb, x.n_features, dtype=torch.float64, device="cuda")
hb = bcm.cpu().pin_memory()
hw = torch.empty(nb, x.n_features, dtype=torch.float64).pin_memory()
betas = cfg["betas"]


def run(dev, change):
    out = []
    for i in range(6):
        if change:
            pm.set_beta(betas[i % len(betas)])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if dev:
            pm.solve_batch_device(bcm.data_ptr(), wcm.data_ptr(), nb, True)
            torch.cuda.synchronize()
        else:
            pm.solve_batch_device(hb.data_ptr(), hw.data_ptr(), nb, False)
        out.append((time.perf_counter() - t0) * 1e3)
    return out


for dev in (True, False):
    for change in (False, True):
        ms = run(dev, change)
        print(f"device={dev} beta_change={change}: " + " ".join(f"{v:.1f}" for v in ms), flush=True)
