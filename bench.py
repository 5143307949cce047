#!/usr/bin/env python
"""Benchmark of the ridgemg_b200 solve path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]

Default workload: BASELINE configs[2] = cfg 3, the largest single-GPU config: a
regularisation sweep (5 betas) over one fixed 4-level hierarchy with 16
right-hand sides solved as a batched block operator.  One step = one beta's
batch of 16 solves to relative residual 1e-6, X, the hierarchy and B already
resident in HBM (rhs = X^T b formation included); value = device ms per
right-hand side.  `e2e` = the same batched call from pinned host buffers.
Multi-GPU (torchrun): the (beta, batch) units are dealt round-robin to the
ranks, max-over-ranks device time.  `--config cfg2 | cfg4 | cfg1 | cfg5` run the
other BASELINE configs (cfg 2: the reference's own multilevel FCG, bit-exact
labels; `--shard`: the row-sharded operator over NCCL).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref: the unmodified reference sources) with all
host threads on the same config, its input built by the reference's own
CounterRng (oracle/synth.hpp; SHA-256 in `config`), never by this repo's library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG time-to-1e-6 rel. residual per solve; XᵀX-operator HBM GB/s vs roofline"

CONFIGS = {
    "cfg2": dict(
        workload="cfg2: sparse binary CSR N=100000 x F=20000, nnz/row max(1,Poisson(40)), Zipf(1.1) columns; "
                 "3-level hierarchy k-means(unit-normalised columns, seed 0) 2000/200, inner FCG tol 1e-6; "
                 "beta=1; outer FCG(m=20) to rel. residual 1e-6",
        kind="zipf", n=100000, f=20000, mean=40.0, zipf=1.1, abs_values=False, seed=0, beta=1.0,
        ks=[2000, 200], normalize=True, method="fcg_multilevel", tol=1e-6, max_iters=1000, golden="cfg2_full"),
    "cfg4": dict(
        workload="cfg4: dense tall-skinny N=4,000,000 x F=1024, fp32 storage / fp64 arithmetic, X = U diag(i^-1.5) "
                 "V^T + 1e-3 N(0,1), U and V orthonormal (CholeskyQR / QR of seeded Gaussians); 3-level hierarchy k-means(unit-normalised columns, seed 0) 128/16 (setup on "
                 "the device, DESIGN.md §4.9), inner FCG tol 1e-6; beta=1e-4; outer FCG(m=20) to rel. residual 1e-6",
        kind="lowrank", n=4_000_000, f=1024, seed=0, beta=1e-4, ks=[128, 16], normalize=True,
        method="fcg_multilevel", tol=1e-6, max_iters=1000, golden="cfg4_none", ref_rows=50_000),
    "cfg3": dict(
        workload="cfg3: sparse CSR N=1,000,000 x F=100,000, nnz/row max(1,Poisson(50)), Zipf(1.1) columns, "
                 "values |N(0,1)| fp64 (generator oracle/synth.hpp = the product's, one CounterRng stream per row, "
                 "seed 0); regularisation sweep beta in {1e-3,1e-2,1e-1,1,10} over one fixed 4-level hierarchy "
                 "10000/1000/100 (sketched k-means on unit-normalised columns, DESIGN.md §4.10); 16 right-hand "
                 "sides b_k = normals(42+k) solved as one batched block operator per beta; rel. residual 1e-6",
        kind="zipf", n=1_000_000, f=100_000, mean=50.0, zipf=1.1, abs_values=True, seed=0, beta=1.0,
        ks=[10_000, 1_000, 100], normalize=True, method="pcg_vcycle_additive", additive_levels=[1], tol=1e-6,
        max_iters=1000, golden="cfg3_none", betas=[1e-3, 1e-2, 1e-1, 1.0, 10.0], n_rhs=16, sketch=32, ref_method="jacobi_cg",
        ref_fixture="cfg3_ref.json"),
    "cfg5": dict(
        workload="cfg5: binary CSR N=16,000,000 x F=500,000 (1.02e9 nonzeros), nnz/row max(1,Poisson(64)), Zipf(1.05) "
                 "columns, on ONE GPU; 4-level hierarchy 50000/5000/500 by sketched k-means (d=32, unit-normalised "
                 "columns, DESIGN.md §4.10); beta=0.5; solver pcg_vcycle_additive (levels 0-1 additive, DESIGN.md §4.15) to "
                 "rel. residual 1e-6",
        kind="zipf", n=16_000_000, f=500_000, mean=64.0, zipf=1.05, abs_values=False, seed=0, beta=0.5,
        ks=[50_000, 5_000, 500], normalize=True, method="pcg_vcycle_additive", additive_levels=[1], tol=1e-6,
        max_iters=1000,
        golden="cfg5_none", betas=[0.5], n_rhs=1, sketch=32, ref_method="jacobi_cg"),
    "cfg1": dict(
        workload="cfg1: dense clustered N=2000 x F=500 fp64 (row-major dense path); 2-level k-means 50; beta=1e-2; "
                 "FCG(m=20) to rel. residual 1e-6",
        kind="dense", n=2000, f=500, groups=50, noise=0.1, seed=0, beta=1e-2, ks=[50], normalize=False,
        method="fcg_twolevel", tol=1e-6, max_iters=1000, golden="cfg1"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class DenseX:
    """A dense synthetic X (cfg 4): shape plus the row-major array (fp32 storage)."""

    def __init__(self, a):
        self.a = a
        self.n_samples, self.n_features = a.shape

    def dense(self):
        return self.a

    def row_sample(self, rows):
        """CSR of the first `rows` samples (fp32 values widened exactly): the
        bounded CPU-baseline workload (the reference's CSR of all 4M rows is 65 GB)."""
        import paper_1806_05826_b200 as R
        return R.from_dense(self.a[:rows].astype(np.float64))


def make_matrix(cfg):
    import paper_1806_05826_b200 as R
    if cfg.get("sketch"):  # large: one RNG stream per row (threaded generator)
        return R.synth_sparse_zipf(cfg["n"], cfg["f"], cfg["mean"], cfg["zipf"], cfg["abs_values"], cfg["seed"],
                                   row_streams=True)
    if cfg["kind"] == "lowrank":
        return DenseX(cfg4_shard_matrix(n=cfg["n"], f=cfg["f"], seed=cfg["seed"]))
    if cfg["kind"] == "zipf":
        return R.synth_sparse_zipf(cfg["n"], cfg["f"], cfg["mean"], cfg["zipf"], cfg["abs_values"], cfg["seed"])
    return R.synth_dense_clustered(cfg["n"], cfg["f"], cfg["groups"], cfg["noise"], cfg["seed"])


class CheckerCsr:
    """A CSR exported from a CPU checker (FeatureMatrix-like: the reference arm's input)."""

    def __init__(self, n, f, rp, ci, v):
        self.n_samples, self.n_features = n, f
        self.row_offsets, self.column_indices, self.values = rp, ci, v

    def value_array(self):
        return self.values


def make_reference_matrix(cfg):
    """The reference arm's input, built by the checker's own generator (oracle/synth.hpp on
    the reference's CounterRng) -- never by the product library."""
    if cfg["kind"] == "lowrank":
        return DenseX(cfg4_shard_matrix(n=cfg["n"], f=cfg["f"], seed=cfg["seed"]))
    import oracle
    chk = oracle.Checker("ref" if oracle.available("ref") else "oracle")
    if cfg["kind"] == "zipf":
        m = chk.synth_sparse_zipf(cfg["n"], cfg["f"], cfg["mean"], cfg["zipf"], cfg["abs_values"], cfg["seed"],
                                  row_streams=bool(cfg.get("sketch")))
    else:
        m = chk.synth_dense_clustered(cfg["n"], cfg["f"], cfg["groups"], cfg["noise"], cfg["seed"])
    rp, ci, v = m.export()
    return CheckerCsr(cfg["n"], cfg["f"], rp, ci, v)


def level_specs(cfg, labels=None):
    import paper_1806_05826_b200 as R
    specs = []
    for i, k in enumerate(cfg["ks"]):
        last = i == len(cfg["ks"]) - 1
        if labels is not None:
            cl = R.ClusteringChoice(kind=R.IMPORTED, labels=labels[i], n_clusters=k)
        elif cfg.get("sketch"):
            cl = R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=0, kmeans_max_iters=100,
                                    normalize_columns=cfg["normalize"], sketch_dim=cfg["sketch"])
        else:
            cl = R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0, kmeans_max_iters=100,
                                    normalize_columns=cfg["normalize"])
        sv = R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG, tol=1e-6, max_iters=500)
        add = cfg["method"] == "pcg_vcycle_additive" and i in cfg.get("additive_levels", [])
        specs.append(R.LevelSpec(clustering=cl, solver=sv, additive=add))
    return specs


def algorithmic_bytes(n, f, nnz, pattern):
    """one operator application, S = 2 sweeps (X, then X^T):
    indices (4 B) + values (0 or 8 B) per nonzero per sweep, int32 row pointers
    of both sweeps, and the compulsory vector traffic 8(F + 2N + 2F)."""
    s_val = 0 if pattern else 8
    return 2 * nnz * (4 + s_val) + 4 * (n + 1) + 4 * (f + 1) + 8 * (f + 2 * n + 2 * f)


class ClockSampler:
    """SM clock and throttle reasons of the timed region: one sample after every timed step
    (the step's device work has just finished -- clock and throttle state outlive it by far
    more than the microseconds in between), taken with in-process NVML (nvidia_ml_py), or a
    one-shot nvidia-smi query when NVML is not importable.

    Why not a free-running `nvidia-smi -lms 50` (round 1): a query that lands INSIDE a step
    stalls the GPU for ~15 ms on this platform -- the same 5 steps of cfg 3 timed 29.6 ms each
    with no query inside them and 30.5-34.6 ms with 1-4 (`-lms 50 / 200`, or NVML from a
    thread every 50 / 150 ms); between steps it costs nothing that is timed.
    BENCH_NO_NVML=1 (one-shot nvidia-smi between steps) and BENCH_NO_STEP_SAMPLES=1 (one
    sample after the region) stay as diagnostics.  The occasional 40-60 ms step seen with
    them (profiles/r2_bench_clock_sampler_modes.log) was not the sampler: the loop graph's
    capture + instantiate inside the solve after a set_beta took 4-23 ms instead of 0.3 ms
    in one solve out of three to ten; set_beta now rebuilds that graph itself
    (profiles/r2_bench_graph_rebuild.log: 60 steps, none above 31.6 ms)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.lines, self.handle, self.nv = device, [], None, None

    def __enter__(self):
        try:
            if os.environ.get("BENCH_NO_NVML"):
                raise RuntimeError("disabled")
            import pynvml as nv
            nv.nvmlInit()
            # NVML orders devices by PCI bus id; honour CUDA_VISIBLE_DEVICES when it is a plain index list
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = self.device
            if vis and all(p.strip().isdigit() for p in vis.split(",")):
                idx = int(vis.split(",")[self.device])
            self.handle = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv = nv
        except Exception:
            self.nv = None
        return self

    def sample(self):
        """Call right after a timed step has completed (never inside one)."""
        if os.environ.get("BENCH_NO_STEP_SAMPLES") and not self._final:
            return
        try:
            if self.nv is not None:
                nv, h = self.nv, self.handle

                def bit(new, old):
                    return getattr(nv, new, None) or getattr(nv, old)

                bits = [bit("nvmlClocksEventReasonHwSlowdown", "nvmlClocksThrottleReasonHwSlowdown"),
                        bit("nvmlClocksEventReasonHwThermalSlowdown", "nvmlClocksThrottleReasonHwThermalSlowdown"),
                        bit("nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksThrottleReasonSwThermalSlowdown"),
                        bit("nvmlClocksEventReasonSwPowerCap", "nvmlClocksThrottleReasonSwPowerCap")]
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.lines.append(", ".join([str(sm), str(mx)] + ["Active" if mask & b else "Not Active" for b in bits]))
            else:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i",
                                      str(self.device)], capture_output=True, text=True, timeout=10).stdout
                self.lines += [ln.strip() for ln in out.splitlines() if ln.strip()]
        except Exception:
            pass

    _final = False

    def __exit__(self, *exc):
        if not self.lines:
            self._final = True
            self.sample()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_golden_labels(cfg):
    path = os.path.join(ROOT, "tests", "golden", cfg["golden"] + ".npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    if "labels0" not in g.files:
        return None
    return [g[f"labels{i}"].astype(np.int64) for i in range(len(cfg["ks"]))]


# ---------------------------------------------------------------- reference arm / CPU baseline
def reference_solve_sample(cfg, x, labels, threads, sample_iters, rhs_seed=42):
    """The reference's own PreparedMethod-equivalent solve (oracle/_ref: the
    unmodified reference sources) capped at `sample_iters` outer iterations;
    returns (seconds per outer iteration, kind, iterations run)."""
    import oracle
    kind = "reference" if oracle.available("ref") else "port"
    chk = oracle.Checker("ref" if kind == "reference" else "oracle")
    chk.set_num_threads(threads)
    m = chk.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
    levels = []
    for i, k in enumerate(cfg["ks"]):
        last = i == len(cfg["ks"]) - 1
        levels.append(dict(labels=labels[i], n_clusters=k,
                           coarse_kind=oracle.COARSE_DIRECT if last else oracle.COARSE_INNER_FCG,
                           coarse_tol=1e-6, coarse_max_iters=500))
    b = chk.normals(rhs_seed, x.n_samples)
    s = chk.solve(m, cfg["beta"], b, cfg["method"], levels=levels, tol=cfg["tol"], max_iters=sample_iters)
    return s.wall_time_s / max(1, s.iterations), kind, s.iterations


def lowrank_sample_labels(cfg):
    """cfg 4's CPU sample imports round-robin clusters of the configured sizes: the
    reference's per-iteration cost on dense X does not depend on which features
    share a cluster (its k-means on 1024 x 50k would dominate the sample)."""
    labels, f = [], cfg["f"]
    for k in cfg["ks"]:
        labels.append(np.arange(f, dtype=np.int64) % k)
        f = k
    return labels


def csr_sha(rp, ci, v):
    """SHA-256 of a CSR as the checkers export it (uint64 offsets / indices, fp64 values)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp, np.uint64).tobytes())
    h.update(np.ascontiguousarray(ci, np.uint64).tobytes())
    h.update(np.ascontiguousarray(v, np.float64).tobytes())
    return h.hexdigest()


def sweep_config(cfg, nnz, sha):
    """The config keys both arms print for a beta-sweep workload (same_config)."""
    nb = cfg["n_rhs"]
    return {"workload": cfg["workload"], "n_samples": cfg["n"], "n_features": cfg["f"], "nnz": int(nnz),
            "x_sha256": sha, "betas": cfg["betas"], "n_rhs": nb, "rhs_seeds": f"42..{42 + nb - 1}",
            "tol": cfg["tol"], "levels": [cfg["f"]] + list(cfg["ks"]),
            "l2": "inputs larger than L2 (X >= 600 MB; no flush needed)"}


def ref_fixture(cfg):
    path = os.path.join(ROOT, "tests", "golden", cfg.get("ref_fixture", "none"))
    try:
        return json.load(open(path))
    except Exception:
        return {}


def ref_method_text(cfg):
    return (f"reference {cfg['ref_method']} (krylov.cpp:94-157 + JacobiPreconditioner :41-47): the reference's "
            f"fastest method on this system -- its fcg_multilevel needs > 1000 outer iterations here and its k-means "
            f"cannot build the hierarchy (DESIGN.md §4.10, §6)")


def run_reference_sweep(args, cfg):
    """The reference arm of a beta-sweep config (cfg 3): the reference's own
    sources (oracle/_ref) on all host threads, input built by the reference's
    own CounterRng (oracle/synth.hpp, SHA-256 printed), every step one COMPLETE
    solve -- b = normals(42 + step mod 16), beta = betas[step mod 5], the
    reference timer (krylov.cpp:651-668, setup and rhs formation untimed)."""
    import oracle
    world = dist_setup()[0]
    t0 = time.time()
    kind = "reference" if oracle.available("ref") else "port"
    chk = oracle.Checker("ref" if kind == "reference" else "oracle")
    threads = os.cpu_count() or 1
    chk.set_num_threads(threads)
    m = chk.synth_sparse_zipf(cfg["n"], cfg["f"], cfg["mean"], cfg["zipf"], cfg["abs_values"], cfg["seed"],
                              row_streams=True)
    sha = csr_sha(*m.export())
    t_gen = time.time() - t0
    per, its = [], []
    nb, betas = cfg["n_rhs"], cfg["betas"]
    for step in range(args.warmup + args.steps):
        beta = betas[step % len(betas)]
        b = chk.normals(42 + step % nb, cfg["n"])
        s = chk.solve(m, beta, b, cfg["ref_method"], tol=cfg["tol"], max_iters=400_000)
        if step >= args.warmup:
            per.append(s.wall_time_s * 1e3)
            its.append(int(s.iterations))
    value = statistics.mean(per)
    sample = (f"complete {cfg['ref_method']} solves, one per step (beta = betas[step mod 5], b = normals(42 + step "
              f"mod 16)), reference timer, {threads} host threads; no extrapolation")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": sweep_config(cfg, m.nnz, sha),
        "algorithm": ref_method_text(cfg), "execution": f"host threads x{threads}",
        "iterations": its,
        "same_algorithm": {"method": cfg["ref_method"], "reference_ms_per_solve": value},
        "cpu_baseline": {"value": value, "unit": "ms/solve", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "ms/solve", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_generation_s": t_gen, "wall_s": time.time() - t0}), flush=True)


def run_reference_arm(args, cfg):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    if cfg.get("sketch"):  # cfg 3 / 5: complete solves of the reference's fastest method
        run_reference_sweep(args, cfg)
        return
    x = make_reference_matrix(cfg)
    scale, iters_fixed = 1.0, None
    if cfg["kind"] == "lowrank":  # bounded sample: the first ref_rows samples, solved to tolerance
        scale = x.n_samples / cfg["ref_rows"]
        x = x.row_sample(cfg["ref_rows"])
        labels = lowrank_sample_labels(cfg)
    else:
        labels = load_golden_labels(cfg)
    if labels is None:
        import oracle
        o = oracle.Checker("oracle")
        o.set_num_threads(os.cpu_count() or 1)
        m = o.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
        labels, cur = [], m
        for k in cfg["ks"]:
            lab, _, _ = o.kmeans(cur, k, 100, 0, normalize=cfg["normalize"])
            labels.append(lab)
            cur = o.coarsen(cur, lab, k)
    threads = os.cpu_count() or 1
    full_iters = None
    g = os.path.join(ROOT, "tests", "golden", cfg["golden"] + ".npz")
    if os.path.exists(g):
        gz = np.load(g)
        key = "ml_iterations" if "ml_iterations" in gz.files else "fcg_iterations"
        if key in gz.files:
            full_iters = int(gz[key])
    per_iter = []
    t0 = time.time()
    sample_iters = args.ref_sample_iters if cfg["kind"] != "lowrank" else cfg["max_iters"]
    for step in range(args.warmup + args.steps):
        sec, kind, ran = reference_solve_sample(cfg, x, labels, threads, sample_iters, 42 + step)
        if step >= args.warmup:
            per_iter.append(sec)
    iters = full_iters or ran
    value = statistics.mean(per_iter) * iters * scale * 1e3
    sample = (f"{sample_iters} outer FCG iterations per step (setup untimed, the reference's own "
              f"krylov.cpp timer), extrapolated x {iters} iterations")
    if cfg["kind"] == "lowrank":
        sample = (f"the first {cfg['ref_rows']} of {int(scale * cfg['ref_rows'])} samples as CSR, solved to "
                  f"tolerance ({iters} iterations, reference timer), x {scale:.0f} rows (cost linear in N); "
                  f"round-robin labels of the same cluster counts")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "ms/solve", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "ms/solve", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0}), flush=True)


# ---------------------------------------------------------------- B200 arm
def dense_algorithmic_bytes(n, f, elem_bytes, sweeps=1):
    """SURVEY.md §8(d), dense: B = S·N·F·s_val + 8(F + 2N + 2F); the dense path
    is one fused sweep (S = 1)."""
    return sweeps * n * f * elem_bytes + 8 * (f + 2 * n + 2 * f)


def cfg4_shard_matrix(n=500_000, f=1024, seed=0, n_total=4_000_000, row0=0):
    """BASELINE cfg 4 (fp32 storage): X = U diag(i^-1.5) V^T + 1e-3 N(0,1) with U the
    n_total x 1024 orthonormal factor of a seeded Gaussian and V = Q of a seeded
    1024^2 Gaussian; returns rows [row0, row0 + n) (n = 500 k: one GPU's shard at 8
    GPUs; n = n_total: the whole matrix).  U by CholeskyQR over all n_total rows: G = A^T A
    summed over row chunks, U = A L^-T (a 4 M x 1024 Gaussian has condition number
    ~1.03, so one pass is orthonormal to ~1e-15).  Seeded torch generators on the GPU
    (one per 64 k-row chunk, so every chunk is reproducible); returned as host float32."""
    import torch
    step = 65536
    dev = "cuda"

    def gen(tag, r):
        return torch.Generator(device=dev).manual_seed((seed * 1_000_003 + tag) * 100_003 + r // step)

    def a_chunk(r):
        return torch.randn(min(step, n_total - r), f, generator=gen(1, r), device=dev, dtype=torch.float64)

    v, _ = torch.linalg.qr(torch.randn(f, f, generator=gen(0, 0), device=dev, dtype=torch.float64))
    sig = torch.arange(1, f + 1, device=dev, dtype=torch.float64) ** -1.5
    w = sig[:, None] * v.T  # diag(sigma) V^T
    g = torch.zeros(f, f, device=dev, dtype=torch.float64)
    for r in range(0, n_total, step):
        a = a_chunk(r)
        g += a.T @ a
    lower = torch.linalg.cholesky(g)  # G = L L^T, A = U L^T
    out = torch.empty(n, f, dtype=torch.float32, device="cpu")
    for c in range(row0 // step * step, row0 + n, step):  # whole chunks, sliced to the row range
        ce = min(n_total, c + step)
        u = torch.linalg.solve_triangular(lower, a_chunk(c).T, upper=False).T
        noise = torch.randn(ce - c, f, generator=gen(2, c), device=dev, dtype=torch.float64)
        lo, hi = max(c, row0), min(ce, row0 + n)
        out[lo - row0:hi - row0] = (u @ w + 1e-3 * noise)[lo - c:hi - c].to(torch.float32).cpu()
    return out.numpy()


def dense_operator_roofline(peak):
    """The dense path's operator on cfg 4's per-GPU shard at 8
    GPUs: one fused sweep over 2 GB of fp32 X per apply, L2 flushed before each."""
    import paper_1806_05826_b200 as R
    t0 = time.time()
    a = cfg4_shard_matrix()
    m = R.DeviceMatrix.from_dense(a)
    pm = R.PreparedMethod(m, 1e-4, R.MethodSpec(kind=R.CG))
    setup = time.time() - t0
    cold = pm.time_operator(0, 10, True)
    warm = pm.time_operator(0, 10, False)
    fb = dense_algorithmic_bytes(a.shape[0], a.shape[1], 4)
    out = {"workload": "cfg4 per-GPU shard at 8 GPUs: N=500,000 x F=1024 dense, fp32 storage / fp64 arithmetic, "
                       "X = U diag(i^-1.5) V^T + 1e-3 N(0,1), beta=1e-4",
           "bound": "hbm", "kernel": "k_dense_ata (fused X^T X single sweep) + k_dense_finish",
           "algorithmic_bytes_per_apply": fb, "ms_per_apply": cold[0], "achieved": fb / (cold[0] * 1e6),
           "peak": peak, "unit": "GB/s", "frac": fb / (cold[0] * 1e6) / peak, "warm_ms": warm[0],
           "setup_s": setup, "frac_of_nominal_8000": fb / (cold[0] * 1e6) / 8000.0,
           "note": "peak is the measured copy bandwidth (read + write); this sweep only reads, which can exceed it"}
    del pm, m, a
    return out


def cfg4_full_summary(peak):
    """BASELINE cfg 4 at full scale on this GPU (4M x 1024 fp32 = 16.4 GB): the
    dense fused operator's roofline (L2 flushed is moot at 16 GB) and the
    multilevel solve (hierarchy built on the device), device-timed
    with CUDA events on the library's stream.  `bench.py --config cfg4` is the
    full bench line for this config (profiles/r1_bench_cfg4.json)."""
    import torch
    import paper_1806_05826_b200 as R
    cfg = CONFIGS["cfg4"]
    t0 = time.time()
    a = cfg4_shard_matrix(n=cfg["n"], f=cfg["f"], seed=cfg["seed"])
    stream = torch.cuda.current_stream()
    ctx = R.Context(torch.cuda.current_device())
    ctx.set_stream(stream.cuda_stream)  # the events below bracket the library's own launches
    m = R.DeviceMatrix.from_dense(a, ctx)
    del a
    pm = R.PreparedMethod(m, cfg["beta"], R.MethodSpec(kind=R.method_from_string(cfg["method"]),
                                                        levels=level_specs(cfg),
                                                        solver=R.SolverConfig(cfg["tol"], cfg["max_iters"])))
    setup = time.time() - t0
    op = pm.time_operator(0, 10, False)
    fb = dense_algorithmic_bytes(cfg["n"], cfg["f"], 4)
    b = torch.from_numpy(R.rng_normals(42, cfg["n"])).cuda()
    w = torch.empty(cfg["f"], dtype=torch.float64, device="cuda")
    ms, its = [], []
    for s in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        rep = pm.solve_device(b.data_ptr(), w.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        if s > 0:
            ms.append(e0.elapsed_time(e1))
            its.append(rep.iterations)
    out = {"workload": cfg["workload"], "setup_s": setup, "ms_per_solve": statistics.mean(ms), "iterations": its,
           "operator": {"bound": "hbm", "kernel": "k_dense_ata (fused X^T X single sweep) + k_dense_finish",
                        "algorithmic_bytes_per_apply": fb, "ms_per_apply": op[0], "achieved": fb / (op[0] * 1e6),
                        "peak": peak, "unit": "GB/s", "frac": fb / (op[0] * 1e6) / peak,
                        "frac_of_nominal_8000": fb / (op[0] * 1e6) / 8000.0,
                        "note": "back-to-back applies (16.4 GB: no L2 reuse); peak is the measured copy bandwidth "
                                "(read + write), which a read-only sweep can exceed"}}
    pm.close()
    m.close()
    ctx.close()
    return out


def shard_operator_roofline(peak):
    """The metric's HBM-bound operator figure: BASELINE cfg 5 (16M x 500k binary,
    Poisson(64) nnz/row, Zipf(1.05)) is row-sharded; one GPU's shard at 4 GPUs
    (4M rows) is generated (per-row RNG streams, threaded) and the fine-level
    operator timed with L2 flushed before every apply (cfg 2's 34 MB operator is
    L2-resident; this one streams 2 GB of indices per apply)."""
    import paper_1806_05826_b200 as R
    t0 = time.time()
    x = R.synth_sparse_zipf(4_000_000, 500_000, 64.0, 1.05, False, 0, row_streams=True)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, R.MethodSpec(kind=R.CG))
    setup = time.time() - t0
    cold = pm.time_operator(0, 10, True)
    warm = pm.time_operator(0, 10, False)
    fb = algorithmic_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern)
    out = {"workload": "cfg5 per-GPU shard at 4 GPUs: N=4,000,000 x F=500,000 binary CSR, nnz/row "
                       "max(1,Poisson(64)), Zipf(1.05) columns (per-row seeded streams), beta=0.5",
           "nnz": m.nnz, "bound": "hbm", "kernel": "K1 (X v, SELL-32) + K2 (X^T pass, segmented)",
           "algorithmic_bytes_per_apply": fb, "ms_per_apply": cold[0], "achieved": fb / (cold[0] * 1e6),
           "peak": peak, "unit": "GB/s", "frac": fb / (cold[0] * 1e6) / peak, "cold_k1_ms": cold[1],
           "cold_k2_ms": cold[2], "warm_ms": warm[0], "setup_s": setup}
    del pm, m, x
    return out


def run_b200(args, cfg):
    import torch
    import paper_1806_05826_b200 as R

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    ctx = R.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    t_setup = time.time()
    x = make_matrix(cfg)
    comm = None
    if args.shard:  # row-sharded fine operator: NCCL all-reduce of the F-vector per X^T pass
        obj = [R.Comm.new_unique_id() if rank == 0 else None]
        if pg:
            pg.broadcast_object_list(obj, src=0)
        comm = R.Comm(ctx, world, rank, obj[0])
    if cfg["kind"] in ("dense", "lowrank"):  # dense inputs: fused single-sweep dense path
        m = R.DeviceMatrix.from_dense(x.dense(), ctx, comm=comm)
    else:
        m = R.DeviceMatrix(x, ctx, comm=comm)
    labels = None
    if world > 1:  # rank 0 clusters once; the other ranks import its labels
        obj = [None]
        if rank == 0:
            pm0 = R.PreparedMethod(m, cfg["beta"], R.MethodSpec(kind=R.method_from_string(cfg["method"]),
                                                                levels=level_specs(cfg),
                                                                solver=R.SolverConfig(cfg["tol"], cfg["max_iters"])))
            obj = [[pm0.labels(i) for i in range(len(cfg["ks"]))]]
            pm0.close()
        pg.broadcast_object_list(obj, src=0)
        labels = obj[0]
    spec = R.MethodSpec(kind=R.method_from_string(cfg["method"]), levels=level_specs(cfg, labels),
                        solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
    pm = R.PreparedMethod(m, cfg["beta"], spec)
    setup_s = time.time() - t_setup
    if labels is None:
        labels = [pm.labels(i) for i in range(len(cfg["ks"]))]

    dev = torch.device("cuda", local)
    nsteps = args.warmup + args.steps
    rseed = 0 if args.shard else rank * 10007  # sharded: every rank solves the same system
    bs = [torch.from_numpy(R.rng_normals(42 + rseed + s, x.n_samples)).to(dev) for s in range(nsteps)]
    w = torch.empty(x.n_features, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    reports = []
    for s in range(args.warmup):
        flush.random_(0, 255)
        reports.append(pm.solve_device(bs[s].data_ptr(), w.data_ptr()))
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    timed = []
    with ClockSampler(local) as clocks:
        for s in range(args.steps):
            flush.random_(0, 255)  # L2 flush, outside the step's events
            ev[s][0].record(stream)
            timed.append(pm.solve_device(bs[args.warmup + s].data_ptr(), w.data_ptr()))
            ev[s][1].record(stream)
            torch.cuda.synchronize()
            clocks.sample()  # between steps: never inside one
        torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if pg:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
    solves = args.steps * (1 if args.shard else world)
    value = total_ms / solves  # whole-job ms per solve (replicas: aggregate throughput)
    ms_per_step = total_ms / args.steps

    # in-situ operator profile over the same kind of steps (events around every
    # K1 / K2 launch of every level), run right after the timed region
    pm.set_profiling(True)
    prof_reports = []
    for s in range(min(args.steps, 3)):
        flush.random_(0, 255)
        prof_reports.append(pm.solve_device(bs[args.warmup + s].data_ptr(), w.data_ptr()))
    torch.cuda.synchronize()
    prof = []
    for lv in range(pm.n_levels):
        napp, k1, k2 = pm.profile(lv)
        info = pm.level(lv) if lv > 0 else {"n_features": x.n_features, "nnz": m.nnz}
        prof.append(dict(level=lv, applications=napp, ms_k1=k1, ms_k2=k2, n_features=info["n_features"],
                         nnz=info["nnz"]))
    pm.set_profiling(False)
    dom = max(prof, key=lambda p: p["ms_k1"] + p["ms_k2"])
    latency = None
    peak, peak_kind = peaks()
    ms_launch = (dom["ms_k1"] + dom["ms_k2"]) / max(1, dom["applications"])
    if dom["level"] > 0 and dom["ms_k2"] < 0.01 * max(dom["ms_k1"], 1e-9):
        # persistent inner solver (dense_level.cu): one launch = one inner FCG solve;
        # per inner iteration it must read A_k (n^2 fp64, from SMEM) and the
        # low-rank preconditioner Q (n x n_{k+1}, from L2) once, plus <= 48
        # n-vectors of Krylov state
        nk = dom["n_features"]
        nnext = prof[dom["level"] + 1]["n_features"] if dom["level"] + 1 < len(prof) else nk
        inner_mean = float(np.mean([np.mean(r.inner_iterations) for r in prof_reports if len(r.inner_iterations)]))
        # DRAM bytes the launch must move: A_k (n^2 fp64, then SMEM-resident), Q (n x n_next) and
        # the level's vectors once; everything else is SMEM / L2 traffic.  The kernel is
        # latency bound (two grid-wide exchanges per inner iteration), so `frac` is small by
        # construction and `latency` carries the figures that matter.
        bytes_per_launch = 8 * (nk * nk + nk * nnext + 48 * nk)
        kernel_name = (f"k_dense_krylov2: persistent level-{dom['level']} inner FCG (n={nk}, "
                       f"{inner_mean:.1f} iterations/launch), in-situ events; latency bound: two grid-wide "
                       f"exchanges per inner iteration (DESIGN.md §4.4, profiles/r1b_dense2.md)")
        latency = {"us_per_inner_iteration": None, "inner_iterations_per_launch": inner_mean,
                   "barrier_share_ncu": "5.5 of 10.0 us per inner iteration (profiles/r1b_dense2.md)",
                   "dram_bytes_per_launch_ncu": 35.3e6}
    elif m.is_dense():  # dense levels: one fused sweep (fine: its storage; device-built coarse levels: fp64)
        esz = x.dense().itemsize if dom["level"] == 0 else 8
        bytes_per_launch = dense_algorithmic_bytes(x.n_samples, dom["n_features"], esz)
        kernel_name = f"level-{dom['level']} dense operator (k_dense_ata fused X^T X sweep + finish), in-situ events"
    else:
        pattern = m.is_pattern if dom["level"] == 0 else False
        bytes_per_launch = algorithmic_bytes(x.n_samples, dom["n_features"], dom["nnz"], pattern)
        kernel_name = f"level-{dom['level']} operator (K1 X v + K2 X^T pass), in-situ events"
    achieved = bytes_per_launch / (ms_launch * 1e-3) / 1e9 if ms_launch > 0 else 0.0
    if latency is not None and inner_mean > 0:
        latency["us_per_inner_iteration"] = ms_launch * 1e3 / inner_mean
    prof_total = sum(p["ms_k1"] + p["ms_k2"] for p in prof)
    prof_step_ms = sum(r.wall_time_s for r in prof_reports) * 1e3

    # cold / warm fine-operator timing (dedicated loop, L2 flushed or not)
    cold = pm.time_operator(0, 20, True)
    warm = pm.time_operator(0, 20, False)
    if m.is_dense():
        fine_bytes = dense_algorithmic_bytes(x.n_samples, x.n_features, x.dense().itemsize)
        op_kernel = "k_dense_ata (fused X^T X single sweep, 1D TMA tiles) + k_dense_finish"
    else:
        fine_bytes = algorithmic_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern)
        op_kernel = "K1 (X v, SELL-32) + K2 (X^T pass, segmented)"

    # e2e: host buffers through the C ABI (H2D of b, D2H of w inside each step)
    pinned_b = [torch.from_numpy(R.rng_normals(42 + rseed + s, x.n_samples)).pin_memory()
                for s in range(args.steps)]
    pinned_w = torch.empty(x.n_features, dtype=torch.float64).pin_memory()
    e2e_ms = []
    for s in range(args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        R.ridgemg._lib.check(pm.lib.rmg_method_solve(pm.h, R.ridgemg._ptr(pinned_b[s].numpy()),
                                                     R.ridgemg._ptr(pinned_w.numpy()), None, 0))
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_total = sum(e2e_ms)
    if pg:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = e2e_total / solves

    # extension: the same systems through pcg_vcycle -- plain PCG with a
    # symmetric Jacobi-smoothed V-cycle over the same hierarchy (BASELINE cfg 1's
    # "1 pre-, 1 post-sweep"); not the reference's algorithm, so not the headline
    vcycle = None
    if rank == 0:
        try:
            pv = R.PreparedMethod(m, cfg["beta"], R.MethodSpec(kind=R.PCG_VCYCLE, levels=level_specs(cfg, labels),
                                                                solver=R.SolverConfig(cfg["tol"], cfg["max_iters"])))
            wv = torch.empty_like(w)
            pv.solve_device(bs[0].data_ptr(), wv.data_ptr())
            vms, vits = [], []
            for s in range(args.steps):
                flush.random_(0, 255)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rep = pv.solve_device(bs[args.warmup + s].data_ptr(), wv.data_ptr())
                e1.record(stream)
                torch.cuda.synchronize()
                vms.append(e0.elapsed_time(e1))
                vits.append(rep.iterations)
            pm.solve_device(bs[args.warmup + args.steps - 1].data_ptr(), w.data_ptr())
            torch.cuda.synchronize()
            vcycle = {"method": "pcg_vcycle (extension: PCG + symmetric V-cycle, damped-Jacobi pre/post smoothing)",
                      "ms_per_solve": statistics.mean(vms), "iterations": vits,
                      "rel_diff_w_vs_headline_method": float(torch.linalg.norm(wv - w) / torch.linalg.norm(w))}
            pv.close()
        except Exception as e:  # reported, never fatal
            vcycle = {"failed": str(e)}

    # extension: dense X with 16 right-hand sides -- the operator as a dense
    # contraction on the FP64 tensor cores (G = X^T X by a DMMA SYRK once, then DMMA GEMMs)
    dense_multi = None
    if rank == 0 and world == 1 and m.is_dense():
        try:
            K = 16
            vb = torch.randn(x.n_features, K, dtype=torch.float64, device=dev)
            ob = torch.empty_like(vb)

            def blk():
                R.ridgemg._lib.check(m.lib.rmg_ridge_apply_block(m.h, cfg["beta"], vb.data_ptr(), ob.data_ptr(), K, 1))

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            blk()  # the first call forms G
            torch.cuda.synchronize()
            syrk_s = time.perf_counter() - t0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(20):
                blk()
            e1.record(stream)
            torch.cuda.synchronize()
            col = torch.empty(x.n_features, dtype=torch.float64, device=dev)
            R.ridgemg._lib.check(m.lib.rmg_ridge_apply(m.h, cfg["beta"], vb[:, 3].contiguous().data_ptr(), col.data_ptr(), 1))
            torch.cuda.synchronize()
            pb = R.PreparedMethod(m, cfg["beta"], R.MethodSpec(kind=R.PCG_VCYCLE, levels=level_specs(cfg, labels),
                                                                solver=R.SolverConfig(cfg["tol"], cfg["max_iters"])))
            bcm = torch.stack([torch.from_numpy(R.rng_normals(42 + q, x.n_samples)) for q in range(K)], 0).to(dev).contiguous()
            wcm = torch.empty(K, x.n_features, dtype=torch.float64, device=dev)
            reps = (R.ridgemg._lib.SolveReportC * K)()
            ms = []
            for _ in range(3):
                e0b, e1b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0b.record(stream)
                R.ridgemg._lib.check(pb.lib.rmg_method_solve_batch(pb.h, bcm.data_ptr(), wcm.data_ptr(), K, reps, 1))
                e1b.record(stream)
                torch.cuda.synchronize()
                ms.append(e0b.elapsed_time(e1b))
            dense_multi = {
                "what": "dense X, 16 right-hand sides: G = X^T X by a DMMA SYRK once (beta-free, reused by a beta "
                        "sweep), block apply and the batched pcg_vcycle as DMMA GEMMs (DESIGN.md §4.16)",
                "syrk_first_apply_s": syrk_s,
                "block_apply_ms": e0.elapsed_time(e1) / 20,
                "block_column_vs_single_apply_rel": float(torch.linalg.norm(ob[:, 3] - col) / torch.linalg.norm(col)),
                "batched_pcg_vcycle_ms_per_rhs": min(ms) / K,
                "batched_pcg_vcycle_ms_per_batch": ms,
                "iterations": [int(r.iterations) for r in reps],
                "includes": "rhs = X^T B inside every batch: one DMMA sweep of X for the 16 columns (k_xtb_dmma)",
            }
            pb.close()
        except Exception as e:  # reported, never fatal
            dense_multi = {"failed": str(e)}

    # CPU baseline: the reference on this host, rank 0 at N=1 only, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            iters = statistics.mean(r.iterations for r in timed)
            if cfg["kind"] == "lowrank":  # reference CSR of all rows would be 65 GB: a row sample, scaled
                rows = cfg["ref_rows"]
                sec, kind, ran = reference_solve_sample(cfg, x.row_sample(rows), lowrank_sample_labels(cfg), 1,
                                                        cfg["max_iters"])
                cpu = {"value": sec * ran * (x.n_samples / rows) * 1e3, "unit": "ms/solve", "cores": 1,
                       "kind": kind,
                       "sample": f"the first {rows} samples as CSR solved to tolerance ({ran} iterations, reference "
                                 f"timer), x {x.n_samples / rows:.0f} (cost linear in N); round-robin labels"}
            else:
                sec, kind, ran = reference_solve_sample(cfg, x, labels, 1, args.ref_sample_iters)
                cpu = {"value": sec * iters * 1e3, "unit": "ms/solve", "cores": 1, "kind": kind,
                       "sample": f"{ran} outer FCG iterations of the same solve (reference timer, setup untimed), "
                                 f"x {iters:.1f} iterations/solve"}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "ms/solve", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    large_op = dense_op = cfg4_full = None
    if rank == 0 and not args.no_large_operator:
        try:
            large_op = shard_operator_roofline(peak)
        except Exception as e:  # reported, never fatal
            large_op = {"failed": str(e)}
        try:
            dense_op = dense_operator_roofline(peak)
        except Exception as e:
            dense_op = {"failed": str(e)}
        if args.config != "cfg4":
            try:
                cfg4_full = cfg4_full_summary(peak)
            except Exception as e:
                cfg4_full = {"failed": str(e)}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        its = [r.iterations for r in timed]
        inner = [float(np.mean(r.inner_iterations)) if len(r.inner_iterations) else 0.0 for r in timed]
        line = {
            "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong" if args.shard else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded CounterRng generator with BASELINE cfg shapes (DESIGN.md §6)",
            "config": {"workload": cfg["workload"], "n_samples": x.n_samples, "n_features": x.n_features,
                       "nnz": m.nnz, "levels": [x.n_features] + list(cfg["ks"]), "beta": cfg["beta"],
                       "tol": cfg["tol"], "method": cfg["method"],
                       "l2": "flushed (256 MiB write) before every timed step, outside its events",
                       "parallelism": (f"row-sharded x{world} (NCCL all-reduce of the F-vector)" if args.shard
                                       else f"replicas x{world}" if world > 1 else "single GPU")},
            "iterations": its, "inner_iterations_mean": inner, "converged": all(r.converged for r in timed),
            "setup_s": setup_s,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name,
                         "algorithmic_bytes_per_launch": bytes_per_launch, "ms_per_launch": ms_launch,
                         "peak_kind": peak_kind,
                         # MEASURED_PEAKS' HBM figure is a copy (read + write): a read-only sweep such as
                         # the dense operator can run slightly above it
                         **({"peak_note": "the peak is a copy kernel's read + write rate; this read-only sweep "
                                          "exceeds it"} if achieved > peak else {}),
                         "share_of_step": (dom['ms_k1'] + dom['ms_k2']) / (prof_step_ms or 1.0),
                         "latency": latency},
            "operator_profile": prof,
            # the metric's second half: X^T X operator, fine level, L2 flushed before every apply
            "operator_roofline": {"bound": "hbm", "kernel": op_kernel,
                                  "algorithmic_bytes_per_apply": fine_bytes, "ms_per_apply": cold[0],
                                  "achieved": fine_bytes / (cold[0] * 1e6), "peak": peak, "unit": "GB/s",
                                  "frac": fine_bytes / (cold[0] * 1e6) / peak, "warm_ms": warm[0],
                                  "warm_gbs": fine_bytes / (warm[0] * 1e6), "cold_k1_ms": cold[1],
                                  "cold_k2_ms": cold[2], "in_situ_ms_per_apply":
                                      (prof[0]["ms_k1"] + prof[0]["ms_k2"]) / max(1, prof[0]["applications"])},
            "operator_roofline_cfg5_shard": large_op,
            "dense_multi_rhs": dense_multi,
            "operator_roofline_cfg4_shard": dense_op,
            "cfg4_full_scale": cfg4_full,
            "pcg_vcycle": vcycle,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "ms/solve", "h2d_bytes_per_step": x.n_samples * 8,
                    "d2h_bytes_per_step": x.n_features * 8},
            "gpu_launches": int(sum(r.kernel_launches for r in timed)),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def timed_batches(pm, stream, bcm, wcm, nb, betas, schedule, cur, clocks=None):
    """Batched solves (one rmg_method_solve_batch per step), beta changed between steps
    outside the events; returns per-step device ms and the reports."""
    import torch
    ms, reps = [], []
    for bi in schedule:
        beta = betas[bi]
        if cur[0] != beta:
            pm.set_beta(beta)
            cur[0] = beta
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tw = time.perf_counter()
        rs = pm.solve_batch_device(bcm.data_ptr(), wcm.data_ptr(), nb, True)
        tw = time.perf_counter() - tw
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if os.environ.get("RMG_BENCH_TRACE"):
            print(f"[trace] step event {ms[-1]:.2f} ms, call wall {1e3 * tw:.2f} ms, solver wall "
                  f"{1e3 * max(r.wall_time_s for r in rs):.2f} ms", file=sys.stderr, flush=True)
        reps.append(rs)
        if clocks is not None:
            clocks.sample()  # between steps: never inside one
    return ms, reps


def block_bytes(n, f, nnz, pattern, k):
    """SURVEY.md §8(d) for k right-hand sides: the index / value streams of both sweeps
    once, the vector term (v, beta v, t written + read, out) k times."""
    s_val = 0 if pattern else 8
    return 2 * nnz * (4 + s_val) + 4 * (n + 1) + 4 * (f + 1) + 8 * (f + 2 * n + 2 * f) * k


def sweep_algorithm_text(cfg, lock):
    if cfg["method"] == "pcg_vcycle_additive":
        add = sorted({0} | set(cfg.get("additive_levels", [])))
        first_mult = max(add) + 1
        return (f"pcg_vcycle_additive: PCG (krylov.cpp:94-157) preconditioned by the config's 4-level hierarchy with "
                f"level(s) {add} entered additively, z_k = D_k^-1 r_k + P_k M_(k+1)(P_k^T r_k), and the symmetric "
                f"damped-Jacobi V-cycle on levels {first_mult}-3 (dense G_k where smaller than the level's sweeps; "
                f"coarsest level direct; DESIGN.md §4.11, §4.14, §4.15), {lock}")
    return (f"{cfg['method']}: PCG (krylov.cpp:94-157) preconditioned by a symmetric V-cycle over the "
            f"config's 4-level hierarchy (damped-Jacobi pre/post smoothing; dense G_k for levels 1-2, "
            f"DESIGN.md §4.11, §4.14), {lock}")


def run_sweep(args, cfg):
    """BASELINE cfg 3: a beta sweep over one fixed hierarchy with 16 right-hand sides
    solved as a batched block operator.  A step = one beta's batch (one
    rmg_method_solve_batch of the 16 columns), betas in sweep order (set_beta between
    steps, outside the events: it rebuilds only the beta-dependent coarse factors and the
    batched loop's CUDA graph, whose nodes carry beta and those buffers).
    value = device ms per right-hand side.  N > 1 ranks: the (beta, batch) steps are
    independent units, dealt round-robin to the ranks (no collective on the data
    path); value = max-over-ranks time / all solves."""
    import torch
    import paper_1806_05826_b200 as R
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    ctx = R.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    trace = (lambda *a: print("[trace]", *a, file=sys.stderr, flush=True)) if os.environ.get("RMG_BENCH_TRACE") else (
        lambda *a: None)
    t0 = time.time()
    x = make_matrix(cfg)
    sha = csr_sha(x.row_offsets, x.column_indices, x.value_array()) if rank == 0 else None
    m = R.DeviceMatrix(x, ctx)
    betas, nb = cfg["betas"], cfg["n_rhs"]
    spec = R.MethodSpec(kind=R.method_from_string(cfg["method"]), levels=level_specs(cfg),
                        solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
    pm = R.PreparedMethod(m, betas[0], spec)
    cur = [betas[0]]
    setup_s = time.time() - t0
    trace("setup", setup_s)
    dev = torch.device("cuda", local)
    bcm = torch.stack([torch.from_numpy(R.rng_normals(42 + k, x.n_samples)) for k in range(nb)], 0).to(dev)
    bcm = bcm.contiguous()  # column-major n x nb block (column k = b_k)
    wcm = torch.empty(nb, x.n_features, dtype=torch.float64, device=dev)
    sched = lambda i: (i * world + rank) % len(betas)  # noqa: E731  round-robin units over ranks
    timed_batches(pm, stream, bcm, wcm, nb, betas, [sched(i) for i in range(args.warmup)], cur)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ms, reps = timed_batches(pm, stream, bcm, wcm, nb, betas,
                                 [sched(args.warmup + i) for i in range(args.steps)], cur, clocks)
    total = sum(ms)
    if pg:
        pg.barrier()
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total = float(t.item())
    value = total / (args.steps * nb * world)
    trace("timed", value)

    # e2e: the same batched call with host buffers (pinned B in, W out, copies inside)
    hb = bcm.cpu().pin_memory()
    hw = torch.empty(nb, x.n_features, dtype=torch.float64).pin_memory()
    pm.solve_batch_device(hb.data_ptr(), hw.data_ptr(), nb, False)  # untimed: first-use staging
    e2e = []
    for i in range(args.steps):
        beta = betas[sched(args.warmup + i)]
        if cur[0] != beta:
            pm.set_beta(beta)
            cur[0] = beta
        torch.cuda.synchronize()
        tt = time.perf_counter()
        pm.solve_batch_device(hb.data_ptr(), hw.data_ptr(), nb, False)
        e2e.append((time.perf_counter() - tt) * 1e3)
    e2e_total = sum(e2e)
    if pg:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = e2e_total / (args.steps * nb * world)
    trace("e2e", e2e_value)
    if rank != 0:
        pm.close()
        m.close()
        pg.barrier()
        pg.destroy_process_group()
        return

    # the dominant kernel: the fine-level block operator; pcg_vcycle applies it 3 times per lock-step
    # PCG iteration (one outside, two inside the V-cycle), pcg_vcycle_additive once
    peak, peak_kind = peaks()
    vb = torch.randn(x.n_features, nb, dtype=torch.float64, device=dev)
    ob = torch.empty_like(vb)
    tb = []
    for i in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        R.ridgemg._lib.check(m.lib.rmg_ridge_apply_block(m.h, 1.0, vb.data_ptr(), ob.data_ptr(), nb, 1))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            tb.append(e0.elapsed_time(e1))
    t_block = statistics.mean(tb)
    bb = block_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern, nb)
    max_its = [max(r.iterations for r in rs) for rs in reps]
    fine_applies = sum(3 * it + 2 for it in max_its) if cfg["method"] == "pcg_vcycle" else sum(it + 1 for it in max_its)
    cold = pm.time_operator(0, 10, True)
    fb = algorithmic_bytes(x.n_samples, x.n_features, m.nnz, m.is_pattern)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config, {}).get(
            "dram_bytes_per_launch")
    except Exception:
        traffic = None

    # same algorithm as the reference arm: the reference's fastest method, batched here
    fx = ref_fixture(cfg)
    same = None
    try:
        pj = R.PreparedMethod(m, betas[0], R.MethodSpec(kind=R.method_from_string(cfg["ref_method"]),
                                                        solver=R.SolverConfig(cfg["tol"], 400_000)))
        jc = [betas[0]]
        timed_batches(pj, stream, bcm, wcm, nb, betas, [0], jc)
        jms, jreps = timed_batches(pj, stream, bcm, wcm, nb, betas, list(range(len(betas))), jc)
        wj = wcm.clone()
        ref_its = fx.get(f"{cfg['ref_method']}/threads1/tol{cfg['tol']:g}", {})
        same = {"method": cfg["ref_method"],
                "gpu": f"batched block operator, {nb} columns in lock step" if nb > 1 else "single-RHS operator",
                "gpu_ms_per_solve": statistics.mean(jms) / nb,
                "gpu_ms_per_solve_by_beta": {f"{b:g}": t / nb for b, t in zip(betas, jms)},
                "gpu_iterations_b42_by_beta": {f"{b:g}": rs[0].iterations for b, rs in zip(betas, jreps)},
                "reference_iterations_b42_by_beta": {k: v["iterations"] for k, v in ref_its.items()},
                "reference_fixture": "tests/golden/cfg3_ref.json (oracle/_ref, threads = 1)"}
        pj.close()
        del wj
    except Exception as e:  # reported, never fatal
        same = {"failed": str(e)}

    # CPU baseline: the reference (oracle/_ref) on ONE host thread, complete solves
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            kind = "reference" if oracle.available("ref") else "port"
            chk = oracle.Checker("ref" if kind == "reference" else "oracle")
            chk.set_num_threads(1)
            om = chk.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
            bsel = [betas[-1], betas[len(betas) // 2]]
            secs = [chk.solve(om, bt, chk.normals(42, x.n_samples), cfg["ref_method"], tol=cfg["tol"],
                              max_iters=400_000).wall_time_s for bt in bsel]
            cpu = {"value": statistics.mean(secs) * 1e3, "unit": "ms/solve", "cores": 1, "kind": kind,
                   "sample": f"complete {cfg['ref_method']} solves at beta {[f'{b:g}' for b in bsel]} (b = "
                             f"normals(42)), the reference's own timer, 1 host thread; no extrapolation"}
            del om
        except Exception as e:
            cpu = {"value": None, "unit": "ms/solve", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    its = [[r.iterations for r in rs] for rs in reps]
    if nb > 1:
        roof = {"bound": "hbm", "kernel": f"level-0 block operator X^T (X V) + beta V, k = {nb} (k_spmm_k1v3 + "
                                          "k_xt_block + k_xt_hotblk + k_hot_fold + k_block_finish + k_vperm_block; "
                                          "profiles/r2_block_operator_v3.md), CUDA events on the library stream",
                "bound_note": "HBM is the reported roofline (SURVEY §8(d) bytes); the kernels themselves sit at 75 % of "
                              "the shared-memory / L1 data pipe (hot passes) and 0.87 of the random 128-byte gather "
                              "ceiling (cold pass): profiles/r2_block_operator_v3.md",
                "achieved": bb / (t_block * 1e6), "peak": peak, "unit": "GB/s", "frac": bb / (t_block * 1e6) / peak,
                "traffic": traffic, "algorithmic_bytes_per_launch": bb, "ms_per_launch": t_block,
                "peak_kind": peak_kind, "share_of_step": fine_applies * t_block / total}
    else:  # one right-hand side: the solve runs the single-RHS operator (K1 + K2), not the block one
        roof = {"bound": "hbm", "kernel": "level-0 operator X^T (X v) + beta v, one RHS (K1 SELL-32 + K2 X^T "
                                          "pass), L2 flushed, CUDA events on the library stream",
                "achieved": fb / (cold[0] * 1e6), "peak": peak, "unit": "GB/s", "frac": fb / (cold[0] * 1e6) / peak,
                "traffic": traffic, "algorithmic_bytes_per_launch": fb, "ms_per_launch": cold[0],
                "peak_kind": peak_kind, "share_of_step": fine_applies * cold[0] / total}
    lock = f"{nb} columns in lock step over the block operator" if nb > 1 else "one right-hand side"
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / args.steps, "step_ms": [round(t, 3) for t in ms],
        "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded CounterRng generator with BASELINE cfg shapes (DESIGN.md §6)",
        "config": sweep_config(cfg, m.nnz, sha),
        "algorithm": sweep_algorithm_text(cfg, lock),
        "execution": (f"{world} GPUs, independent (beta, batch) units round-robin" if world > 1 else "single GPU"),
        "iterations_per_step": its, "converged": all(r.converged for rs in reps for r in rs),
        "betas_per_step": [betas[sched(args.warmup + i)] for i in range(args.steps)],
        "setup_s": setup_s,
        "roofline": roof,
        "operator_roofline": {"bound": "hbm", "kernel": "K1 (X v, SELL-32) + K2 (X^T pass), one RHS, L2 flushed",
                              "algorithmic_bytes_per_apply": fb, "ms_per_apply": cold[0],
                              "achieved": fb / (cold[0] * 1e6), "peak": peak, "unit": "GB/s",
                              "frac": fb / (cold[0] * 1e6) / peak},
        "same_algorithm": same,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "ms/solve", "h2d_bytes_per_step": x.n_samples * 8 * nb,
                "d2h_bytes_per_step": x.n_features * 8 * nb,
                "ms_per_step": [round(v, 2) for v in e2e],
                "note": f"one batched call of {nb} right-hand side(s) per step from pinned host memory"},
        "gpu_launches": int(sum(sum(r.kernel_launches for r in rs) for rs in reps)),
        "clocks": clocks.summary()}), flush=True)
    pm.close()
    m.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def run_sharded(args, cfg):
    """`--shard` on a sparse sweep config (cfg 3 / cfg 5): X row-sharded over the ranks
    with per-rank input -- each rank generates and holds only its rows
    (synth_sparse_zipf_row_range, rmg_matrix_create_csr_rows) -- and the hierarchy
    set up sharded (sketch S, coarse Grams, Jacobi diagonals all-reduced over NCCL,
    X_k = X P coarsened row-locally).  A step = one single-RHS solve (beta and b
    cycling through the sweep); every X^T pass all-reduces the F-vector.  Strong
    scaling: the total work per step is fixed; value = max-over-ranks ms per solve."""
    import torch
    import paper_1806_05826_b200 as R
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    ctx = R.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    obj = [R.Comm.new_unique_id() if rank == 0 else None]
    if pg:
        pg.broadcast_object_list(obj, src=0)
    comm = R.Comm(ctx, world, rank, obj[0])
    t0 = time.time()
    n = cfg["n"]
    r0, r1 = rank * n // world, (rank + 1) * n // world
    xl = R.synth_sparse_zipf_row_range(n, cfg["f"], cfg["mean"], cfg["zipf"], cfg["abs_values"], cfg["seed"], r0, r1)
    m = R.DeviceMatrix.from_rows(xl, n, r0, comm, ctx)
    nnz_local = m.nnz
    del xl
    betas, nb = cfg["betas"], cfg["n_rhs"]
    spec = R.MethodSpec(kind=R.method_from_string(cfg["method"]), levels=level_specs(cfg),
                        solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
    pm = R.PreparedMethod(m, betas[0], spec)
    cur = betas[0]
    setup_s = time.time() - t0
    dev = torch.device("cuda", local)
    bs = [torch.from_numpy(R.rng_normals(42 + k, n)).to(dev) for k in range(min(nb, 4))]
    w = torch.empty(cfg["f"], dtype=torch.float64, device=dev)
    units = [(b_i, k) for b_i in range(len(betas)) for k in range(len(bs))]

    def step(i):
        nonlocal cur
        bi, k = units[i % len(units)]
        if cur != betas[bi]:
            pm.set_beta(betas[bi])
            cur = betas[bi]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = pm.solve_device(bs[k].data_ptr(), w.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), rep

    for i in range(args.warmup):
        step(i)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        res = []
        for i in range(args.steps):
            res.append(step(args.warmup + i))
            clocks.sample()  # between steps: never inside one
    total = sum(r[0] for r in res)
    if pg:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total = float(t.item())
        z = torch.tensor([float(nnz_local)], dtype=torch.float64, device=dev)
        pg.all_reduce(z)
        nnz_total = int(z.item())
    else:
        nnz_total = nnz_local
    value = total / args.steps
    cold = pm.time_operator(0, 10, True)  # this rank's shard, no collective inside the loop
    if rank == 0:
        peak, peak_kind = peaks()
        fb = algorithmic_bytes(r1 - r0, cfg["f"], nnz_local, m.is_pattern)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded CounterRng generator with BASELINE cfg shapes, generated per rank",
            "config": {"workload": cfg["workload"], "n_samples": n, "n_features": cfg["f"], "nnz": nnz_total,
                       "levels": [cfg["f"]] + list(cfg["ks"]), "betas": betas, "tol": cfg["tol"],
                       "parallelism": f"row-sharded x{world} (per-rank input; NCCL all-reduce of the F-vector)"},
            "algorithm": f"{cfg['method']} over the sharded hierarchy (DESIGN.md §7)",
            "iterations": [r[1].iterations for r in res], "converged": all(r[1].converged for r in res),
            "setup_s": setup_s,
            "roofline": {"bound": "hbm", "kernel": "rank-0 shard operator K1 + K2 (cold L2), no collective",
                         "algorithmic_bytes_per_launch": fb, "ms_per_launch": cold[0],
                         "achieved": fb / (cold[0] * 1e6), "peak": peak, "unit": "GB/s",
                         "frac": fb / (cold[0] * 1e6) / peak, "traffic": None, "peak_kind": peak_kind},
            "e2e": None, "gpu_launches": int(sum(r[1].kernel_launches for r in res)),
            "clocks": clocks.summary()}), flush=True)
    pm.close()
    m.close()
    comm.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def run_sharded_dense(args, cfg):
    """`--shard` on cfg 4: the dense X row-sharded with per-rank input -- each rank
    generates only its rows (cfg4_shard_matrix(row0=...)) and uploads them with
    rmg_matrix_create_dense_rows; no host CSR anywhere.  The hierarchy is set up
    sharded on the device: sketched k-means (S = sum_i G_i^T X_i and the column
    norms all-reduced; exact k-means needs every row of a column on one device),
    X_k = X_i P per rank, coarse Grams all-reduced.  A step = one solve; strong
    scaling (total work fixed), value = max-over-ranks ms per solve."""
    import torch
    import paper_1806_05826_b200 as R
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    ctx = R.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    obj = [R.Comm.new_unique_id() if rank == 0 else None]
    if pg:
        pg.broadcast_object_list(obj, src=0)
    comm = R.Comm(ctx, world, rank, obj[0])
    n, f = cfg["n"], cfg["f"]
    r0, r1 = rank * n // world, (rank + 1) * n // world
    t0 = time.time()
    xl = cfg4_shard_matrix(n=r1 - r0, f=f, seed=cfg["seed"], n_total=n, row0=r0)
    gen_s = time.time() - t0
    t0 = time.time()
    m = R.DeviceMatrix.from_dense_rows(xl, n, r0, comm, ctx)
    del xl
    scfg = dict(cfg, sketch=32)
    spec = R.MethodSpec(kind=R.method_from_string(cfg["method"]), levels=level_specs(scfg),
                        solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
    pm = R.PreparedMethod(m, cfg["beta"], spec)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    dev = torch.device("cuda", local)
    b = torch.from_numpy(R.rng_normals(42, n)).to(dev)
    w = torch.empty(f, dtype=torch.float64, device=dev)

    def step():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = pm.solve_device(b.data_ptr(), w.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), rep

    for _ in range(args.warmup):
        step()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        res = []
        for _ in range(args.steps):
            res.append(step())
            clocks.sample()  # between steps: never inside one
    total = sum(r[0] for r in res)
    if pg:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total = float(t.item())
    value = total / args.steps
    cold = pm.time_operator(0, 10, True)
    if rank == 0:
        peak, peak_kind = peaks()
        fb = dense_algorithmic_bytes(r1 - r0, f, 4)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "ms/solve", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: cfg 4's seeded low-rank generator, rows generated per rank",
            "config": {"workload": cfg["workload"].replace("k-means(", "sketched k-means(d=32, "),
                       "n_samples": n, "n_features": f, "levels": [f] + list(cfg["ks"]), "beta": cfg["beta"],
                       "tol": cfg["tol"],
                       "parallelism": f"row-sharded x{world} (per-rank dense input; NCCL all-reduce of the F-vector)"},
            "algorithm": f"{cfg['method']} over a sharded sketched-k-means hierarchy (DESIGN.md §7)",
            "iterations": [r[1].iterations for r in res], "converged": all(r[1].converged for r in res),
            "generate_s": gen_s, "setup_s": setup_s,
            "roofline": {"bound": "hbm", "kernel": "rank-0 shard fused dense operator (cold L2), no collective",
                         "algorithmic_bytes_per_launch": fb, "ms_per_launch": cold[0],
                         "achieved": fb / (cold[0] * 1e6), "peak": peak, "unit": "GB/s",
                         "frac": fb / (cold[0] * 1e6) / peak, "traffic": None, "peak_kind": peak_kind,
                         "note": "peak is the measured COPY figure (read + write); a read-only sweep runs above it"},
            "e2e": None, "gpu_launches": int(sum(r[1].kernel_launches for r in res)),
            "clocks": clocks.summary()}), flush=True)
    pm.close()
    m.close()
    comm.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def main():
    # stdout carries exactly one JSON line: keep NCCL's banner off it unless asked for
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-sample-iters", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large-operator", action="store_true",
                    help="skip the cfg5-shard operator roofline (about 20 s of setup)")
    ap.add_argument("--shard", action="store_true", help="row-shard X across ranks (strong scaling)")
    ap.add_argument("--method", default=None, help="override the config's solver (e.g. pcg_vcycle)")
    ap.add_argument("--additive-levels", default=None,
                    help="pcg_vcycle_additive: comma-separated levels >= 1 entered additively too (rmg_level_spec.additive)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.method:
        cfg["method"] = args.method
    if args.additive_levels is not None:
        cfg["additive_levels"] = [int(t) for t in args.additive_levels.split(",") if t]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    elif args.config in ("cfg3", "cfg5") and args.shard:
        run_sharded(args, cfg)
    elif args.config == "cfg4" and args.shard:
        run_sharded_dense(args, cfg)
    elif args.config in ("cfg3", "cfg5"):
        run_sweep(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
