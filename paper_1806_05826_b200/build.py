"""Build libridgemg_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1806_05826_b200.build [--force]

Device code: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
Host code: no FMA contraction (-ffp-contract=off) so the host-side setup
(clustering, coarsening) keeps the reference's floating-point order.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libridgemg_b200.so")
SOURCES = ["kernels.cu", "dense_level.cu", "dense_setup.cu", "fgmres.cu", "kmeans_gpu.cu", "dense_gram.cu", "spmm_tma.cu", "runtime.cu", "capi.cu", "host_setup.cpp", "ingest.cpp"]
HEADERS = ["kernels.cuh", "dense_level.cuh", "dense_setup.hpp", "fgmres.cuh", "kmeans_gpu.hpp", "dense_gram.cuh", "spmm_tma.cuh", "runtime.cuh", "host_setup.hpp", "ingest.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    """NCCL matching the one torch loads (same SONAME -> one NCCL per process)."""
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (2.28.x)
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ridgemg_b200.h"),
                                                                  os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", CSRC, "-I",
              os.path.join(ROOT, "include"), "-I", nccl_inc]
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", *common, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-O3", "--expt-relaxed-constexpr"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out)
        if verbose and out:
            print(out)
    link = [NVCC, *ARCH, "-shared", *objs, "-o", LIB + ".tmp", "-lcudart",
            "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-L" + nccl_lib, "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + nccl_lib, "-L/usr/lib/x86_64-linux-gnu", "-l:libstdc++.so.6", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(link) + "\n" + r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
