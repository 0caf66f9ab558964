"""Multi-rank host logic of the element-partitioned solve, on CPU with gloo.

Two processes (world_size 2) each own a contiguous element slab.  With the CPU
oracle doing the per-rank block arithmetic, the test checks that the slab plan,
the halo exchange (torch.distributed isend/irecv) and the allreduce-based
classical Gram-Schmidt GMRES reproduce the single-process answer for the same
partition (reference partition_keep_mask semantics, precond.py:26-45).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.distributed import HaloExchange, SlabPlan
from paper_1701_07181_b200.meshes import partition_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(cfg, P):
    wl = W.make_workload(cfg, norm_iters=20)
    prob = O.problem_from_workload(wl)
    b = partition_bounds(wl.pattern.T, P)
    part = np.repeat(np.arange(P), np.diff(b))
    return wl, prob, part


def _local_ops(wl, plan, s, nb):
    """Per-rank operator (extended pattern + dummy ghost rows) and partitioned factor."""
    Tl, ng = plan.T_local, plan.n_ghost
    ip = np.concatenate([plan.ext_indptr, plan.ext_indptr[-1] + 1 + np.arange(ng)])
    ix = np.concatenate([plan.ext_indices, Tl + np.arange(ng)])
    J = np.concatenate([wl.J[plan.row_block_src], np.zeros((ng, nb, nb))])
    M = np.concatenate([wl.M[plan.lo:plan.hi], np.broadcast_to(np.eye(nb), (ng, nb, nb))])
    dg = np.concatenate([plan.ext_diag, plan.ext_indptr[-1] + np.arange(ng)])
    op = O.Problem(ip, ix, dg, [J] * s, M, wl.a_inv, wl.dt)
    fprob = O.Problem(plan.loc_indptr, plan.loc_indices, plan.loc_diag,
                      [np.ascontiguousarray(wl.J[plan.loc_block_src])] * s,
                      np.ascontiguousarray(wl.M[plan.lo:plan.hi]), wl.a_inv, wl.dt)
    fac = O.stage_uncoupled_factorize(fprob, wl.shifts)
    return op, fac


def _dist_matvec(op, halo, plan, s, nb, x):
    Tl, ng = plan.T_local, plan.n_ghost
    ghost = torch.zeros(s * max(ng, 1) * nb, dtype=torch.float64)
    halo.exchange(x, ghost)
    xe = np.concatenate([x.numpy().reshape(s, Tl, nb), ghost.numpy()[: s * ng * nb].reshape(s, ng, nb)], axis=1)
    ye = op.matvec(xe.reshape(-1)).reshape(s, Tl + ng, nb)
    return torch.from_numpy(np.ascontiguousarray(ye[:, :Tl]).reshape(-1))


def _cgs_gmres(mv, pre, b, rtol, restart, maxit=200):
    """Left-preconditioned restarted GMRES with CGS + DGKS and allreduced dots
    (the reduction pattern of the native irk_gmres)."""
    def dot_all(vs, w):
        h = torch.stack([torch.dot(v, w) for v in vs] + [torch.dot(w, w)])
        dist.all_reduce(h)
        return h

    def norm(v):
        t = torch.dot(v, v).reshape(1)
        dist.all_reduce(t)
        return float(t.sqrt())

    x = torch.zeros_like(b)
    r = pre(b)
    bnorm = beta = norm(r)
    tol = rtol * bnorm
    total = 0
    while total < maxit:
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        g = np.zeros(restart + 1)
        g[0] = beta
        cs, sn = np.zeros(restart), np.zeros(restart)
        done = 0
        res = beta
        for j in range(restart):
            w = pre(mv(V[j]))
            h = dot_all(V, w)
            hj, nb0 = h[:-1], float(h[-1].sqrt())
            w = w - sum(c * v for c, v in zip(hj, V))
            nw = norm(w)
            if nw < 0.7071 * nb0:
                h2 = dot_all(V, w)[:-1]
                w = w - sum(c * v for c, v in zip(h2, V))
                hj = hj + h2
                nw = norm(w)
            H[: j + 1, j] = hj.numpy()
            H[j + 1, j] = nw
            V.append(w / nw)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            done = j + 1
            res = abs(g[j + 1])
            if res <= tol:
                break
        y = np.linalg.solve(np.triu(H[:done, :done]), g[:done])
        x = x + sum(float(c) * v for c, v in zip(y, V[:done]))
        if res <= tol:
            return x, total
        r = pre(b - mv(x))
        beta = norm(r)
    return x, total


def _worker(rank, world, port, cfgd, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = W.SolveConfig(**cfgd)
        wl, prob, part = _problem(cfg, world)
        s, nb, T = cfg.s, cfg.nb, wl.pattern.T
        p = wl.pattern
        plan = SlabPlan.build(p.indptr, p.indices, p.diag_pos, world, rank)
        halo = HaloExchange(plan, s, nb, "cpu")
        op, fac = _local_ops(wl, plan, s, nb)
        lo, hi = plan.lo, plan.hi
        loc = lambda v: np.ascontiguousarray(v.reshape(s, T, nb)[:, lo:hi]).reshape(-1)  # noqa: E731
        rng = np.random.default_rng(11)
        w = rng.standard_normal(s * T * nb)
        # (1) halo-exchanged matvec == rows of the global matvec
        y = _dist_matvec(op, halo, plan, s, nb, torch.from_numpy(loc(w))).numpy()
        err_mv = np.linalg.norm(y - loc(prob.matvec(w))) / np.linalg.norm(loc(prob.matvec(w)))
        # (1b) overlapped matvec: interior rows computed while the exchange is posted (ghosts
        # still zero), boundary rows after finish() -- equals the synchronous one
        Tl, ng = plan.T_local, plan.n_ghost
        xw = torch.from_numpy(loc(w))
        ghost = torch.zeros(s * max(ng, 1) * nb, dtype=torch.float64)
        works = halo.start(xw)
        r0, r1 = plan.interior
        xe = np.concatenate([xw.numpy().reshape(s, Tl, nb), ghost.numpy()[: s * ng * nb].reshape(s, ng, nb)], axis=1)
        y_int = op.matvec(xe.reshape(-1)).reshape(s, Tl + ng, nb)[:, r0:r1]
        halo.finish(works, ghost)
        xe = np.concatenate([xw.numpy().reshape(s, Tl, nb), ghost.numpy()[: s * ng * nb].reshape(s, ng, nb)], axis=1)
        y_all = op.matvec(xe.reshape(-1)).reshape(s, Tl + ng, nb)[:, :Tl].copy()
        y_ovl = y_all.copy()
        y_ovl[:, r0:r1] = y_int
        err_mv = max(err_mv, float(np.abs(y_ovl.reshape(-1) - y).max() / np.abs(y).max()))
        # (2) local partitioned ILU apply == global apply with the partition keep mask
        gfac = O.stage_uncoupled_factorize(prob, wl.shifts, partition_of=part)
        err_ap = np.linalg.norm(fac.apply(loc(w)) - loc(gfac.apply(w))) / np.linalg.norm(loc(gfac.apply(w)))
        # (3) distributed GMRES == single-process partitioned solve
        mv = lambda v: _dist_matvec(op, halo, plan, s, nb, v)  # noqa: E731
        pre = lambda v: torch.from_numpy(fac.apply(v.numpy()))  # noqa: E731
        xd, it = _cgs_gmres(mv, pre, torch.from_numpy(loc(wl.rhs)), cfg.rtol, cfg.restart)
        xo, so = O.gmres(prob.matvec, gfac.apply, wl.rhs, O.GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
        err_x = np.linalg.norm(xd.numpy() - loc(xo)) / np.linalg.norm(loc(xo))
        np.save(f"{out_path}.{rank}.npy", np.array([err_mv, err_ap, err_x, it, so.iterations,
                                                    plan.n_ghost, sum(len(v) for v in plan.send.values())]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mesh,N,nb", [("tet3d", 4, 6), ("tri2d", 8, 8)])
def test_partitioned_solve_two_ranks(tmp_path, mesh, N, nb):
    cfg = W.CONFIGS[2].scaled(mesh=mesh, N=N, nb=nb)
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), dict(cfg.__dict__), out), nprocs=2, join=True)
    for r in range(2):
        err_mv, err_ap, err_x, it, it_ref, ng, nsend = np.load(f"{out}.{r}.npy")
        assert ng > 0 and nsend > 0
        assert err_mv < 1e-12, err_mv
        assert err_ap < 1e-12, err_ap
        assert abs(it - it_ref) <= 1
        assert err_x < 1e-8, err_x


def test_slab_plan_consistency():
    """Send lists of one rank are exactly the ghost lists of its peers."""
    cfg = W.CONFIGS[2].scaled(N=4, nb=4)
    p = W.Pattern.from_table(W.mesh_table(cfg.mesh, cfg.N))
    P = 4
    plans = [SlabPlan.build(p.indptr, p.indices, p.diag_pos, P, r) for r in range(P)]
    for r, pl in enumerate(plans):
        for q, idx in pl.recv.items():
            sent = plans[q].lo + plans[q].send[r]
            np.testing.assert_array_equal(pl.ghosts[idx], sent)
        # extended pattern rows are sorted and contain the diagonal
        for i in range(pl.T_local):
            row = pl.ext_indices[pl.ext_indptr[i]:pl.ext_indptr[i + 1]]
            assert np.all(np.diff(row) > 0) and row[pl.ext_diag[i] - pl.ext_indptr[i]] == i
        r0, r1 = pl.interior
        assert r1 > r0
