"""CPU-side checks of the product boundary (no GPU needed):
the C-ABI library loads, exports every function include/ridgemg_b200.h
declares, and its host-only entry points (RNG, synthetic generators,
generate_rhs's b) match the oracle / the pinned goldens.  Device entry points
must fail loudly without a GPU (no CPU fallback)."""
import ctypes as C
import hashlib
import os
import re

import numpy as np
import pytest

import paper_1806_05826_b200 as R
from paper_1806_05826_b200 import _lib
from helpers import load_golden

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ridgemg_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rmg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding covers the whole header
    assert set(names) <= set(_lib.exported_symbols())


def test_built_for_sm100a():
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_rng_matches_oracle(orc):
    for seed in (0, 42, 0x5EED, 2 ** 63 + 5):
        assert np.array_equal(R.rng_normals(seed, 777), orc.normals(seed, 777))


def _sha(x):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x.row_offsets, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.column_indices, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.value_array(), np.float64).tobytes())
    return h.hexdigest()


def test_synthetic_generators_pinned():
    assert _sha(R.synth_dense_clustered(2000, 500, 50, 0.1, 0)) == str(load_golden("cfg1")["sha256"])
    x = R.synth_sparse_zipf(10000, 2000, 40.0, 1.1, False, 0)
    assert _sha(x) == str(load_golden("cfg2_small")["sha256"])
    # canonical CSR: strictly increasing columns per row, every row non-empty
    rp = x.row_offsets.astype(np.int64)
    assert np.all(np.diff(rp) >= 1)
    ci = x.column_indices.astype(np.int64)
    for r in range(0, 10000, 997):
        row = ci[rp[r]:rp[r + 1]]
        assert np.all(np.diff(row) > 0)
    xv = R.synth_sparse_zipf(1000, 300, 20.0, 1.05, True, 3)
    assert xv.values is not None and np.all(xv.values >= 0.0)


def test_generate_rhs_host_part(orc):
    # b is produced on the host (glibc libm); rhs needs the device
    x = R.synth_sparse_zipf(500, 80, 10.0, 1.1, False, 1)
    assert np.array_equal(R.rng_normals(42, 500), orc.generate_rhs(orc.matrix(500, 80, x.row_offsets,
                                                                               x.column_indices), 42)[0])


def test_csr_from_triplets_matches_reference(ref):
    rng = np.random.default_rng(5)
    rows = rng.integers(0, 7, 40)
    cols = rng.integers(0, 9, 40)
    vals = rng.standard_normal(40)
    ours = R.csr_from_triplets(7, 9, rows, cols, vals)
    theirs = ref.from_triplets(7, 9, rows, cols, vals)
    rp, ci, v = theirs.export()
    assert np.array_equal(ours.row_offsets, rp) and np.array_equal(ours.column_indices, ci)
    # duplicates are summed in std::sort order there (unstable, sparse.cpp:42-46): rounding-level only
    assert np.allclose(ours.values, v, rtol=1e-15, atol=1e-15)
    uniq = np.unique(rows * 9 + cols, return_index=True)[1]
    ours = R.csr_from_triplets(7, 9, rows[uniq], cols[uniq], vals[uniq])
    rp, ci, v = ref.from_triplets(7, 9, rows[uniq], cols[uniq], vals[uniq]).export()
    assert np.array_equal(ours.values, v) and np.array_equal(ours.column_indices, ci)
    with pytest.raises(ValueError):
        R.csr_from_triplets(2, 2, [0, 5], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        R.csr_from_triplets(2, 2, [0], [0], [np.inf])


@pytest.mark.parametrize("name", ["lpsc105", "cnae"])
def test_matrix_market_reader_matches_reference(name):
    path = f"/root/reference/proj/data/{name}.mtx"
    if not os.path.exists(path):
        pytest.skip("reference data not on this machine")
    g = load_golden(name)
    x = R.read_matrix_market(path)
    assert np.array_equal(x.row_offsets, g["x_row_offsets"].astype(np.uint64))
    assert np.array_equal(x.column_indices, g["x_column_indices"].astype(np.uint64))
    assert np.array_equal(x.values, g["x_values"])


def test_device_entry_points_fail_loudly_without_gpu():
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is present")
    with pytest.raises(R.RmgCudaError):
        R.Context(0)


def test_null_arguments_are_invalid():
    lib = _lib.load()
    assert lib.rmg_context_create(0, None) == _lib.RMG_ERR_INVALID_ARGUMENT
    assert b"must not be NULL" in lib.rmg_last_error()
    assert lib.rmg_rng_normals(1, 5, None) == _lib.RMG_ERR_INVALID_ARGUMENT
    major, minor = C.c_int32(), C.c_int32()
    assert lib.rmg_version(C.byref(major), C.byref(minor)) == 0


def _msha(m):
    rp, ci, v = m.export()
    h = hashlib.sha256()
    h.update(rp.tobytes())
    h.update(ci.tobytes())
    h.update(v.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_checker_generators_match_product(kind, request):
    """The reference arm builds its inputs with the checkers' own generator
    (oracle/synth.hpp on the reference's CounterRng): same bytes as the product's."""
    chk = request.getfixturevalue("orc" if kind == "oracle" else "ref")
    assert _msha(chk.synth_dense_clustered(2000, 500, 50, 0.1, 0)) == str(load_golden("cfg1")["sha256"])
    assert _msha(chk.synth_sparse_zipf(10000, 2000, 40.0, 1.1, False, 0)) == str(load_golden("cfg2_small")["sha256"])
    for args in ((3000, 700, 25.0, 1.05, True, 3), (2000, 50, 60.0, 1.1, False, 9)):
        for rows in (False, True):
            assert _msha(chk.synth_sparse_zipf(*args, row_streams=rows)) == _sha(
                R.synth_sparse_zipf(*args, row_streams=rows)), (args, rows)


@pytest.mark.parametrize("values", [True, False])
def test_csr_cache_roundtrip_and_sha(tmp_path, values):
    """The binary CSR cache (ingest.cpp): SHA-256 of the exported arrays equals
    hashlib's, a save/load round trip is exact, a corrupted file is refused."""
    x = R.synth_sparse_zipf(3000, 400, 15.0, 1.1, values, 7)
    assert R.csr_sha256(x) == _sha(x)
    path = str(tmp_path / "x.csr")
    assert R.save_csr(x, path) == _sha(x)
    y, sha = R.load_csr(path)
    assert sha == _sha(x) and _sha(y) == _sha(x)
    assert (y.values is None) == (not values)
    raw = bytearray(open(path, "rb").read())
    if values:
        raw[-9] ^= 0x40  # flip a bit in the last value
    else:  # a pattern's stored values are 1.0 by definition: corrupt a column index instead
        raw[-8 * x.nnz - 16] ^= 0x01
    open(path, "wb").write(bytes(raw))
    with pytest.raises((RuntimeError, ValueError)):  # digest mismatch (or an invalid CSR)
        R.load_csr(path)


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n", "unsupported field"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "entry count mismatch"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix array pattern general\n2 2\n", "pattern field"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n", "square"),
])
def test_matrix_market_errors_like_reference(tmp_path, ref, text, msg):
    """Malformed files are refused with the reference's error (matrix_market.cpp)."""
    path = str(tmp_path / "bad.mtx")
    open(path, "w").write(text)
    with pytest.raises(RuntimeError) as ours:
        R.read_matrix_market(path)
    assert msg in str(ours.value)
    with pytest.raises(Exception) as theirs:
        ref.read_matrix_market(path)
    assert msg in str(theirs.value)


def test_matrix_market_symmetric_and_array(tmp_path, ref):
    """symmetric coordinate / array files: mirrored entries, zeros of arrays dropped."""
    cases = ["%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2.0\n3 1 -1.5\n2 2 4\n",
             "%%MatrixMarket matrix array real general\n2 3\n1\n0\n2.5\n0\n0\n-3\n",
             "%%MatrixMarket matrix array integer symmetric\n3 3\n1\n2\n0\n4\n5\n6\n"]
    for i, text in enumerate(cases):
        path = str(tmp_path / f"m{i}.mtx")
        open(path, "w").write(text)
        x = R.read_matrix_market(path)
        rp, ci, v = ref.read_matrix_market(path).export()
        assert np.array_equal(x.row_offsets, rp) and np.array_equal(x.column_indices, ci)
        assert np.array_equal(x.value_array(), v)
