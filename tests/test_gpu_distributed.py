"""Element-partitioned solve through the native multi-GPU layer (csrc/comm.cu),
two ranks in two processes on ONE GPU.

The transport is the host-staged one (``Comm.host``: the library hands the
packed halo send buffer and the GMRES allreduce buffers to a gloo exchange on
the host), so no kernel of one rank ever waits on the other rank's kernels;
everything else is the production path: ``irk_halo`` pack kernel and ghost
buffer, ``irk_dist_op`` (interior/boundary rows), the fused Arnoldi product in
halo mode, and ``irk_gmres`` with ``irk_comm_allreduce`` -- no Python operator
callbacks.  NCCL itself needs one GPU per rank (not available to this build).

Each rank's rows must match the single-process oracle with the reference's
partition map (meshing.py:81-90, precond.py:26-45): operator and fused product
within 1e-12, GMRES iterations within +-1 and x within 1e-10 at equal counts.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfgd, out):
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.distributed import DistributedStageSolver, SlabPlan
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.meshes import partition_bounds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = W.SolveConfig(**cfgd)
        P = world
        full = W.make_workload(cfg.scaled(extra={"parts": P}), norm_iters=20)
        prob = O.problem_from_workload(full)
        T, s, nb = full.pattern.T, cfg.s, cfg.nb
        b = partition_bounds(T, P)
        part = np.repeat(np.arange(P), np.diff(b))
        gfac = O.make_preconditioner(prob, "uncoupled", full.shifts, partition_of=part)
        pat, J, M, rhs = W.make_slab_workload(cfg, P, rank)
        plan = SlabPlan.build(pat.indptr, pat.indices, pat.diag_pos, P, rank)
        lo, hi = plan.lo, plan.hi
        loc = lambda v: np.ascontiguousarray(v.reshape(s, T, nb)[:, lo:hi]).reshape(-1)  # noqa: E731
        assert np.array_equal(rhs, loc(full.rhs))
        sol = DistributedStageSolver(plan, J, M, full.a_inv, full.dt, "uncoupled", full.shifts,
                                     GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart), transport="host")
        w = np.random.default_rng(5).standard_normal(s * T * nb)
        wd = torch.from_numpy(loc(w)).cuda()
        y = sol.matvec(wd).cpu().numpy()
        yref = loc(prob.matvec(w))
        err_mv = np.linalg.norm(y - yref) / np.linalg.norm(yref)
        sol.factorize()
        a = sol.fac.apply(wd).cpu().numpy()
        aref = loc(gfac.apply(w))
        err_ap = np.linalg.norm(a - aref) / np.linalg.norm(aref)
        x_p, fused = sol.product(wd)
        pref = loc(gfac.apply(prob.matvec(w)))
        err_pr = np.linalg.norm(x_p.cpu().numpy() - pref) / np.linalg.norm(pref)
        x, st = sol.solve(torch.from_numpy(rhs).cuda())
        xo, so = O.gmres(prob.matvec, gfac.apply, full.rhs, O.GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
        err_x = np.linalg.norm(x.cpu().numpy() - loc(xo)) / np.linalg.norm(loc(xo))
        np.save(f"{out}.{rank}.npy", np.array([err_mv, err_ap, err_pr, err_x, st.iterations, so.iterations,
                                               float(fused), float(st.converged), plan.n_ghost]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("mesh,N,nb,ordering", [("tet3d", 4, 50, "color"), ("tri2d", 8, 40, "color"),
                                                ("tet3d", 4, 10, "natural")])
def test_two_ranks_native_layer_vs_oracle(tmp_path, mesh, N, nb, ordering):
    import torch.multiprocessing as mp

    from paper_1701_07181_b200 import workloads as W
    cfg = W.CONFIGS[2].scaled(mesh=mesh, N=N, nb=nb, ordering=ordering)
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), dict(cfg.__dict__), out), nprocs=2, join=True)
    for r in range(2):
        err_mv, err_ap, err_pr, err_x, it, it_ref, fused, conv, ng = np.load(f"{out}.{r}.npy")
        assert ng > 0
        assert err_mv < 1e-12, err_mv
        assert err_ap < 1e-12, err_ap
        assert err_pr < 1e-12, err_pr
        # colour-major slabs: 2-level local schedules, the halo-mode fused product runs
        if ordering == "color":
            assert bool(fused)
        assert conv and abs(it - it_ref) <= 1, (it, it_ref)
        if it == it_ref:
            assert err_x < 1e-10, err_x


def test_nccl_comm_single_rank():
    """The NCCL transport inside libirkb200 (dlopen of the process's libnccl.so.2):
    unique id, communicator of one rank, in-place allreduce on the stream, and a
    DistributedStageSolver driven by it (P=1: no halo peers) equal to StageSolver."""
    import ctypes

    import torch

    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.distributed import Comm, DistributedStageSolver, SlabPlan
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    assert L.lib().irk_comm_nccl_available() == 1
    buf = (ctypes.c_ubyte * 128)()
    L.check(L.lib().irk_comm_nccl_unique_id(buf, 128), "unique id")
    h = ctypes.c_void_p()
    L.check(L.lib().irk_comm_create_nccl(L.ctx(), buf, 1, 0, ctypes.byref(h)), "create")
    comm = Comm(h.value, 1, 0)
    v = torch.arange(7, dtype=torch.float64, device="cuda")
    fn, user = comm.native_allreduce
    L.check(L.lib().irk_comm_allreduce(user, v.data_ptr(), 7, L.stream_ptr()), "allreduce")
    assert torch.equal(v, torch.arange(7, dtype=torch.float64, device="cuda"))
    cfg = W.CONFIGS[2].scaled(N=4, nb=10, ordering="color")
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    plan = SlabPlan.build(p.indptr, p.indices, p.diag_pos, 1, 0)
    gc = GmresConfig(rel_tol=1e-8, restart=40)
    ds = DistributedStageSolver(plan, wl.J, wl.M, wl.a_inv, wl.dt, "uncoupled", wl.shifts, gc, transport=comm)
    ds.factorize()
    rhs = torch.from_numpy(wl.rhs).cuda()
    x, st = ds.solve(rhs)
    ss = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                     kind="uncoupled", shifts=wl.shifts, gmres_cfg=gc)
    ss.factorize()
    x2, st2 = ss.solve(rhs)
    assert st.iterations == st2.iterations and st.converged
    assert torch.equal(x, x2)
    _, fused = ds.product(torch.randn(ds.n_local, dtype=torch.float64, device="cuda"))
    assert fused
