"""The row-sharded product path with two ranks on ONE GPU.

NCCL refuses two ranks on one device, so the ranks talk through the library's
host-staged communicator (rmg_comm_create_host): every all-reduce of the
operator, the Gram / Jacobi / sketch setup sums is staged through pinned host
memory and summed by a gloo all-reduce.  Each rank holds only its own rows
(rmg_matrix_create_csr_rows, generated per rank with
synth_sparse_zipf_row_range), and the whole hierarchy setup is sharded: the
kmeans_sketch sketch S = sum_i G_i^T X_i is all-reduced, X_k = X_i P is
coarsened row-locally, the coarse Grams and Jacobi diagonals are all-reduced.
Results are held to the CPU oracle on the full matrix and to the same solves
on one unsharded device."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, F, MEAN, ZIPF, SEED = 6000, 700, 25.0, 1.1, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def _levels(R, kind, ks, labels=None, tol=1e-6):
    out = []
    for i, k in enumerate(ks):
        if labels is not None:
            cl = R.ClusteringChoice(kind=R.IMPORTED, labels=labels[i], n_clusters=k)
        elif kind == "sketch":
            cl = R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=0, normalize_columns=True,
                                    sketch_dim=16)
        else:
            cl = R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0)
        out.append(R.LevelSpec(clustering=cl, solver=R.CoarseSolveChoice(
            kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG, tol=tol, max_iters=500)))
    return out


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        import oracle
        import paper_1806_05826_b200 as R

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        R.load()
        ctx = R.Context(0)

        def allreduce(buf):
            dist.all_reduce(torch.from_numpy(buf))  # in place on the staged vector

        comm = R.Comm.host_staged(ctx, world, rank, allreduce)
        r0, r1 = rank * N // world, (rank + 1) * N // world
        xl = R.synth_sparse_zipf_row_range(N, F, MEAN, ZIPF, True, SEED, r0, r1)
        m = R.DeviceMatrix.from_rows(xl, N, r0, comm, ctx)
        full = R.synth_sparse_zipf(N, F, MEAN, ZIPF, True, SEED, row_streams=True)
        mf = R.DeviceMatrix(full, ctx)  # the same system on one unsharded device
        orc = oracle.Checker("oracle")
        om = orc.matrix(N, F, full.row_offsets, full.column_indices, full.value_array())
        res = {"rows": (m.row_range, (r0, r1)), "n": m.n_samples}
        v = np.random.default_rng(1).standard_normal(F)
        res["apply"] = _rel(m.ridge_apply(0.3, v), orc.ridge_apply(om, 0.3, v))
        res["spmv"] = _rel(m.spmv(v), orc.spmv(om, v))
        res["diag"] = _rel(m.gram_diagonal(0.3), orc.gram_diagonal(om, 0.3))
        b = R.rng_normals(42, N)
        ref12 = orc.solve(om, 0.3, b, "cg", tol=1e-12, max_iters=20000)
        for method in ("cg", "jacobi_cg"):
            pm = R.PreparedMethod(m, 0.3, R.MethodSpec(kind=R.method_from_string(method),
                                                       solver=R.SolverConfig(1e-10, 20000)))
            w, rep = pm.solve(b)
            pf = R.PreparedMethod(mf, 0.3, R.MethodSpec(kind=R.method_from_string(method),
                                                        solver=R.SolverConfig(1e-10, 20000)))
            wf, repf = pf.solve(b)
            res[method] = (rep.converged, rep.iterations, repf.iterations, _rel(w, ref12.w))
            pm.close()
            pf.close()
        # pcg_vcycle over a sharded sketch hierarchy (labels identical on every rank)
        pv = R.PreparedMethod(m, 0.3, R.MethodSpec(kind=R.PCG_VCYCLE, levels=_levels(R, "sketch", [80, 12]),
                                                   solver=R.SolverConfig(1e-10, 2000)))
        w, rep = pv.solve(b)
        labels = [pv.labels(0), pv.labels(1)]
        res["vcycle"] = (rep.converged, rep.iterations, _rel(w, ref12.w))
        res["labels"] = [lab.tolist() for lab in labels]
        pv.close()
        # pcg_vcycle_additive with levels 0-1 additive (bench cfg 5's solver), sharded vs one device
        lv = _levels(R, None, [80, 12], labels)
        lv[1].additive = True
        spec = R.MethodSpec(kind=R.PCG_VCYCLE_ADDITIVE, levels=lv, solver=R.SolverConfig(1e-10, 2000))
        pa, pf = R.PreparedMethod(m, 0.3, spec), R.PreparedMethod(mf, 0.3, spec)
        wa, repa = pa.solve(b)
        wf, repf = pf.solve(b)
        res["additive"] = (repa.converged, repa.iterations, repf.iterations, _rel(wa, ref12.w))
        pa.close()
        pf.close()
        # the reference's multilevel FCG over the same (imported) labels, sharded vs one device
        spec = R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=_levels(R, None, [80, 12], labels, tol=1e-10),
                            solver=R.SolverConfig(1e-10, 1000))
        ps, pf = R.PreparedMethod(m, 0.3, spec), R.PreparedMethod(mf, 0.3, spec)
        ws, reps = ps.solve(b)
        wf, repf = pf.solve(b)
        res["fcg_ml"] = (reps.converged, reps.iterations, repf.iterations, _rel(ws, wf), _rel(ws, ref12.w))
        ps.close()
        pf.close()
        # exact k-means needs every row of a column on one device: refused
        try:
            R.PreparedMethod(m, 0.3, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=_levels(R, "kmeans", [40])))
            res["kmeans_refused"] = False
        except ValueError:
            res["kmeans_refused"] = True
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))


def test_two_ranks_one_gpu_host_staged():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in out[r], out[r].get("error")
    for r in range(2):
        res = out[r]
        assert tuple(res["rows"][0]) == tuple(res["rows"][1]) and res["n"] == N
        assert res["apply"] <= 1e-13 and res["spmv"] <= 1e-14 and res["diag"] <= 1e-14, res
        for method in ("cg", "jacobi_cg"):
            cv, its, its_full, err = res[method]
            assert cv and err <= 1e-8, (method, res[method])
            assert abs(its - its_full) <= max(2, its_full // 20), (method, its, its_full)
        cv, its, err = res["vcycle"]
        assert cv and err <= 1e-8, res["vcycle"]
        cv, its, its_full, err = res["additive"]
        assert cv and abs(its - its_full) <= 2 and err <= 1e-8, res["additive"]
        cv, its, its_full, d_full, err = res["fcg_ml"]
        assert cv and abs(its - its_full) <= 2 and d_full <= 1e-8 and err <= 1e-8, res["fcg_ml"]
        assert res["kmeans_refused"]
    assert out[0]["labels"] == out[1]["labels"]  # every rank built the same hierarchy
    print({k: v for k, v in out[0].items() if k != "labels"})
