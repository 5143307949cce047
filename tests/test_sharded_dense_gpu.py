"""Per-rank DENSE input with sharded device setup (rmg_matrix_create_dense_rows),
two ranks on ONE GPU through the host-staged communicator.

Each rank uploads only its own rows of a dense X (cfg 4's shape class: tall, a
few hundred features); no CSR is built anywhere.  kmeans_sketch runs on
S = sum_i G_i^T X_i (all-reduced, then scaled by the all-reduced column norms),
X_k = X_i P is formed per rank on the device, the coarse Grams are all-reduced.
Held to the CPU oracle on the full matrix and to the same solves on one
unsharded device."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, F = 5000, 240


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def _dense(seed=3):
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((N, 12))
    x = u @ rng.standard_normal((12, F)) + 0.3 * rng.standard_normal((N, F))
    x[rng.random((N, F)) < 0.05] = 0.0  # exact zeros: the oracle's CSR drops them
    return x


def _levels(R, ks, labels=None, tol=1e-10):
    out = []
    for i, k in enumerate(ks):
        if labels is not None:
            cl = R.ClusteringChoice(kind=R.IMPORTED, labels=labels[i], n_clusters=k)
        else:
            cl = R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=0, normalize_columns=True,
                                    sketch_dim=16)
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
            dist.all_reduce(torch.from_numpy(buf))

        comm = R.Comm.host_staged(ctx, world, rank, allreduce)
        x = _dense()
        r0, r1 = rank * N // world, (rank + 1) * N // world
        m = R.DeviceMatrix.from_dense_rows(x[r0:r1], N, r0, comm, ctx)
        mf = R.DeviceMatrix.from_dense(x, ctx)
        nzr, nzc = np.nonzero(x)
        rp = np.zeros(N + 1, np.int64)
        np.add.at(rp, nzr + 1, 1)
        orc = oracle.Checker("oracle")
        om = orc.matrix(N, F, np.cumsum(rp), nzc, x[nzr, nzc])
        res = {"rows": m.row_range, "want_rows": (r0, r1), "n": m.n_samples}
        v = np.random.default_rng(1).standard_normal(F)
        res["apply"] = _rel(m.ridge_apply(0.3, v), orc.ridge_apply(om, 0.3, v))
        res["diag"] = _rel(m.gram_diagonal(0.3), orc.gram_diagonal(om, 0.3))
        b = R.rng_normals(42, N)
        ref12 = orc.solve(om, 0.3, b, "cg", tol=1e-12, max_iters=20000)
        for method in ("cg", "jacobi_cg"):
            spec = R.MethodSpec(kind=R.method_from_string(method), solver=R.SolverConfig(1e-10, 20000))
            pm, pf = R.PreparedMethod(m, 0.3, spec), R.PreparedMethod(mf, 0.3, spec)
            (w, rep), (wf, repf) = pm.solve(b), pf.solve(b)
            res[method] = (rep.converged, rep.iterations, repf.iterations, _rel(w, ref12.w))
            pm.close()
            pf.close()
        pv = R.PreparedMethod(m, 0.3, R.MethodSpec(kind=R.PCG_VCYCLE, levels=_levels(R, [40, 8]),
                                                   solver=R.SolverConfig(1e-10, 2000)))
        w, rep = pv.solve(b)
        labels = [pv.labels(0), pv.labels(1)]
        res["vcycle"] = (rep.converged, rep.iterations, _rel(w, ref12.w))
        res["labels"] = [lab.tolist() for lab in labels]
        pv.close()
        # the sketch labels on one unsharded device (same S up to rounding of the sums)
        pu = R.PreparedMethod(mf, 0.3, R.MethodSpec(kind=R.PCG_VCYCLE, levels=_levels(R, [40, 8]),
                                                    solver=R.SolverConfig(1e-10, 2000)))
        res["labels_agree"] = float(np.mean(pu.labels(0) == labels[0]))
        pu.close()
        # the reference's multilevel FCG over the same imported labels, sharded vs one device
        spec = R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=_levels(R, [40, 8], labels),
                            solver=R.SolverConfig(1e-10, 1000))
        ps, pf = R.PreparedMethod(m, 0.3, spec), R.PreparedMethod(mf, 0.3, spec)
        (ws, reps), (wf, repf) = ps.solve(b), pf.solve(b)
        res["fcg_ml"] = (reps.converged, reps.iterations, repf.iterations, _rel(ws, wf), _rel(ws, ref12.w))
        ps.close()
        pf.close()
        try:
            R.PreparedMethod(m, 0.3, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[R.LevelSpec(
                clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=20, seed=0))]))
            res["kmeans_refused"] = False
        except ValueError:
            res["kmeans_refused"] = True
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        import traceback
        q.put((rank, {"error": repr(e) + traceback.format_exc()}))


def test_two_ranks_dense_rows_one_gpu():
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
        assert tuple(res["rows"]) == tuple(res["want_rows"]) and res["n"] == N, res
        assert res["apply"] <= 1e-13 and res["diag"] <= 1e-14, res
        for method in ("cg", "jacobi_cg"):
            cv, its, its_full, err = res[method]
            assert cv and err <= 1e-8, (method, res[method])
            assert abs(its - its_full) <= max(2, its_full // 20), (method, its, its_full)
        cv, its, err = res["vcycle"]
        assert cv and err <= 1e-8, res["vcycle"]
        assert res["labels_agree"] >= 0.9, res["labels_agree"]
        cv, its, its_full, d_full, err = res["fcg_ml"]
        assert cv and abs(its - its_full) <= 2 and d_full <= 1e-8 and err <= 1e-8, res["fcg_ml"]
        assert res["kmeans_refused"]
    assert out[0]["labels"] == out[1]["labels"]
    print({k: v for k, v in out[0].items() if k != "labels"})
