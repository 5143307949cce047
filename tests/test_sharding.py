"""Row sharding of the X^T X operator.

CPU (gloo, world size 2): the product's nnz-balanced partition
(rmg_shard_rows) + per-rank partial X_i^T (X_i v) + all-reduce of the
F-vector reproduce the full operator, and a replicated-vector CG driven by
that composition takes the oracle's iteration count.  The per-rank local
product is computed with the CPU oracle here (no GPU in this container);
on the GPU the same composition is the library's NCCL path (test below,
single rank - gpurun provides one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1806_05826_b200 as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_csr(x, r0, r1):
    rp = x.row_offsets.astype(np.int64)
    lo, hi = rp[r0], rp[r1]
    return (rp[r0:r1 + 1] - lo).astype(np.uint64), x.column_indices[lo:hi], x.value_array()[lo:hi]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        orc = oracle.Checker("oracle")
        x = R.synth_sparse_zipf(6000, 700, 25.0, 1.1, True, 5)
        bounds = R.shard_rows(x.row_offsets, world).astype(np.int64)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rp, ci, vals = _local_csr(x, r0, r1)
        local = orc.matrix(r1 - r0, x.n_features, rp, ci, vals)
        beta = 0.3

        def apply(v):
            part = orc.spmv_transpose(local, orc.spmv(local, v))
            t = torch.from_numpy(part.copy())
            dist.all_reduce(t)
            return t.numpy() + beta * v

        full = orc.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
        v = np.random.default_rng(1).standard_normal(x.n_features)
        err = np.linalg.norm(apply(v) - orc.ridge_apply(full, beta, v)) / np.linalg.norm(orc.ridge_apply(full, beta, v))
        # replicated-vector CG on the sharded operator (krylov.cpp:94-157)
        b = orc.normals(42, x.n_samples)
        rhs_part = torch.from_numpy(orc.spmv_transpose(local, b[r0:r1].copy()))
        dist.all_reduce(rhs_part)
        rhs = rhs_part.numpy()
        xs = np.zeros_like(rhs)
        r = rhs.copy()
        p = r.copy()
        rz = r @ r
        nb = np.sqrt(rhs @ rhs)
        its = 0
        for its in range(1, 500):
            ap = apply(p)
            alpha = rz / (p @ ap)
            xs += alpha * p
            r -= alpha * ap
            if np.sqrt(r @ r) / nb <= 1e-8:
                break
            rz2 = r @ r
            p = r + (rz2 / rz) * p
            rz = rz2
        ref = orc.solve(full, beta, b, "cg", tol=1e-8, max_iters=500)
        q.put((rank, err, its, ref.iterations, np.linalg.norm(xs - ref.w) / np.linalg.norm(ref.w),
               (r0, r1), int(x.row_offsets[r1]) - int(x.row_offsets[r0])))
        dist.destroy_process_group()
    except Exception as e:  # report, never hang the parent
        q.put((rank, repr(e)))


def test_partition_properties():
    x = R.synth_sparse_zipf(5000, 300, 30.0, 1.1, False, 2)
    rp = x.row_offsets.astype(np.int64)
    for world in (1, 2, 3, 8):
        b = R.shard_rows(x.row_offsets, world).astype(np.int64)
        assert b[0] == 0 and b[-1] == x.n_samples and np.all(np.diff(b) >= 0)
        loads = rp[b[1:]] - rp[b[:-1]]
        assert loads.sum() == x.nnz
        assert loads.max() - x.nnz / world <= np.diff(rp).max() + 1  # balanced to within one row


def test_sharded_operator_and_cg_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for item in res:
        assert len(item) == 7, item
        rank, err, its, ref_its, werr, rng, load = item
        assert err <= 1e-13
        assert abs(its - ref_its) <= 2
        assert werr <= 1e-8
    # the two ranks own complementary row blocks
    r = sorted((it[5] for it in res))
    assert r[0][0] == 0 and r[0][1] == r[1][0]


@pytest.mark.gpu
def test_sharded_matrix_single_rank_nccl(gpu):
    """The library's NCCL path (all-reduce + epilogue pass) on one rank equals the
    unsharded operator and solve."""
    x = R.synth_sparse_zipf(20000, 2000, 30.0, 1.1, True, 9)
    uid = R.Comm.new_unique_id()
    comm = R.Comm(gpu, 1, 0, uid)
    ms = R.DeviceMatrix(x, gpu, comm=comm)
    mu = R.DeviceMatrix(x, gpu)
    assert ms.row_range == (0, x.n_samples)
    v = np.random.default_rng(3).standard_normal(x.n_features)
    a, b = ms.ridge_apply(0.5, v), mu.ridge_apply(0.5, v)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)
    u = np.random.default_rng(4).standard_normal(x.n_samples)
    assert np.linalg.norm(ms.spmv(v) - mu.spmv(v)) <= 1e-13 * np.linalg.norm(mu.spmv(v))
    assert np.linalg.norm(ms.spmv_transpose(u) - mu.spmv_transpose(u)) <= 1e-13 * np.linalg.norm(mu.spmv_transpose(u))
    bb = R.rng_normals(42, x.n_samples)
    spec = R.MethodSpec(kind=R.FCG_TWOLEVEL,
                        levels=[R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=100))],
                        solver=R.SolverConfig(1e-10, 500))
    s1, s2 = R.solve_system(ms, 0.5, bb, spec), R.solve_system(mu, 0.5, bb, spec)
    assert s1.report.converged and abs(s1.report.iterations - s2.report.iterations) <= 1
    assert np.linalg.norm(s1.w - s2.w) <= 1e-9 * np.linalg.norm(s2.w)
    ms.close()
    comm.close()


@pytest.mark.gpu
def test_dense_sharded_single_rank_nccl(gpu):
    """Dense X row-sharded over NCCL (cfg 4's layout) on one rank equals the
    unsharded dense operator and solve."""
    a = np.random.default_rng(8).standard_normal((5000, 300)).astype(np.float32)
    uid = R.Comm.new_unique_id()
    comm = R.Comm(gpu, 1, 0, uid)
    ms = R.DeviceMatrix.from_dense(a, gpu, comm=comm)
    mu = R.DeviceMatrix.from_dense(a, gpu)
    assert ms.is_dense() and ms.row_range == (0, 5000)
    v = np.random.default_rng(3).standard_normal(300)
    u = np.random.default_rng(4).standard_normal(5000)
    for got, want in ((ms.ridge_apply(0.5, v), mu.ridge_apply(0.5, v)), (ms.spmv(v), mu.spmv(v)),
                      (ms.spmv_transpose(u), mu.spmv_transpose(u)), (ms.gram_diagonal(0.5), mu.gram_diagonal(0.5))):
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    bb = R.rng_normals(42, 5000)
    spec = R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-10, 2000))
    s1, s2 = R.solve_system(ms, 1e-2, bb, spec), R.solve_system(mu, 1e-2, bb, spec)
    assert s1.report.converged and abs(s1.report.iterations - s2.report.iterations) <= 1
    assert np.linalg.norm(s1.w - s2.w) <= 1e-9 * np.linalg.norm(s2.w)
    ms.close()
    comm.close()


@pytest.mark.gpu
def test_sharded_pcg_vcycle_single_rank_nccl(gpu):
    """pcg_vcycle on the row-sharded operator: the fine-level
    applications go through the all-reduce path, the coarse levels are replicated;
    equal to the unsharded solve."""
    x = R.synth_sparse_zipf(8000, 900, 25.0, 1.1, True, 5)
    uid = R.Comm.new_unique_id()
    comm = R.Comm(gpu, 1, 0, uid)
    ms = R.DeviceMatrix(x, gpu, comm=comm)
    mu = R.DeviceMatrix(x, gpu)
    levels = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=90),
                          solver=R.CoarseSolveChoice(kind=R.INNER_FCG)),
              R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=12))]
    spec = R.MethodSpec(kind=R.PCG_VCYCLE, levels=levels, solver=R.SolverConfig(1e-10, 2000))
    bb = R.rng_normals(7, x.n_samples)
    s1, s2 = R.solve_system(ms, 0.5, bb, spec), R.solve_system(mu, 0.5, bb, spec)
    assert s1.report.converged and abs(s1.report.iterations - s2.report.iterations) <= 1
    assert np.linalg.norm(s1.w - s2.w) <= 1e-9 * np.linalg.norm(s2.w)
    ms.close()
    comm.close()
