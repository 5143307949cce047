"""The C++ mirror (include/ridgemg_b200.hpp) compiles against the C ABI and
behaves like the reference interface."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1806_05826_b200")


@pytest.fixture(scope="module")
def example(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "example_solve")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "example_solve.cpp"), "-L", PKG, "-l:libridgemg_b200.so",
           "-Wl,-rpath," + PKG, "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_cpp_client_cpu_only(example):
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present: covered by the gpu variant")
    r = subprocess.run([example, "--cpu-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok:" in r.stdout


@pytest.mark.gpu
def test_cpp_client_solves(example):
    r = subprocess.run([example], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("converged=1") == 5
