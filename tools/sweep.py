#!/usr/bin/env python
"""BASELINE configs 3 and 4 (and config 2 kernels) on one B200, one JSON line each.

  python tools/sweep.py config3 [--nb 24 40 50 100] [--s 1 2 3 4]
  python tools/sweep.py config4 [--dtn 10 100 1000]
  python tools/sweep.py config2kernels

config3: BSR matvec and plain block-ILU(0) apply of J itself (one factor, s
right-hand sides, every factor block read once: irk_factor_apply_rhs) on the
config-1 mesh (T = 32768, colour numbering), nb in {24, 40, 50, 100}, s in
{1..4}.  GB/s = algorithmic bytes / CUDA-event time, algorithmic bytes as
SURVEY 8d: matvec nnzb*Bk + 2 s v + idx; apply "J + 2 s v" = nnzb*Bk + 2 s v
(the factor has the storage of J: L, U off-diagonal blocks and T D^-1 blocks).

config4: DIRK33 (3 sequential stage Newton solves, ILU(0) of M - dt g J,
GMRES(40)) vs RADAU23 transformed coupled GMRES(40), equal order 3, on the
config-1 mesh/blocks (nb = 40), linear problem M du/dt = J u, dt*||J||_2 in
{10, 100, 1000}, rtol 1e-8.  Time per step in steady state (the frozen-J
factors are cached, as for any fixed-dt integration of a linear problem) and
the first step including the factorisations.

config2kernels: the config-2 operator (32^3 cubes -> 196608 Kuhn tets, nb=50,
s=3) on ONE GPU: fused stage matvec, shifted uncoupled factorisation and apply.

Inputs are HBM-resident (J >= 0.6 GB >> L2); timings are CUDA events after warm-up.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def peak():
    try:
        return float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps):
    import torch
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def emit(d):
    print(json.dumps(d), flush=True)


def config3(args):
    import torch
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.precond import ilu0_factorize
    pk = peak()
    base = W.CONFIGS[1].scaled(ordering="color")
    table = W.mesh_table(base.mesh, base.N, "natural")
    from paper_1701_07181_b200.meshes import slab_color_permutation
    for nb in args.nb:
        t0 = time.perf_counter()
        pat = W.Pattern.from_table(table)
        J = W.jacobian_blocks(pat, nb, base.seed, base.jstd)
        M = np.zeros((pat.T, nb, nb))
        rhs = np.zeros(pat.T * nb)
        _, pat, J, _, _ = W.relabel(table, J, M, rhs, 1, slab_color_permutation(table, 1))
        del M, rhs
        dp = DevicePattern(pat.indptr, pat.indices, pat.diag_pos)
        Jd = BlockSparseMatrix(dp, DeviceBlocks.from_host(J))
        gen_s = time.perf_counter() - t0
        T, nnzb = pat.T, pat.nnzb
        del J
        t0 = time.perf_counter()
        fac = ilu0_factorize(Jd)
        torch.cuda.synchronize()
        t_create = time.perf_counter() - t0
        tf = timed(lambda: fac.refactor(Jd), 3)
        Bk, v = 8 * nb * nb, 8 * T * nb
        for s in args.s:
            Y = torch.randn(s * T * nb, dtype=torch.float64, device="cuda")
            X = torch.empty_like(Y)
            op = Jd.rhs_op(s)
            from paper_1701_07181_b200 import _lib as L
            lib = L.lib()
            st = L.stream_ptr()

            def mv():
                L.check(lib.irk_stage_op_apply(op.handle, Y.data_ptr(), X.data_ptr(), st))

            def ap():
                fac.apply_rhs_device(Y, X, s)

            t_mv = timed(mv, 20)
            t_ap = timed(ap, 20)
            b_mv = nnzb * Bk + 2 * s * v + 4 * (nnzb + T + 1)
            b_ap = nnzb * Bk + 2 * s * v + 4 * (nnzb + T + 1)
            emit({"config": 3, "T": T, "nb": nb, "s": s, "matvec_ms": 1e3 * t_mv,
                  "matvec_GBps": b_mv / t_mv / 1e9, "matvec_frac": b_mv / t_mv / 1e9 / pk,
                  "apply_ms": 1e3 * t_ap, "apply_GBps": b_ap / t_ap / 1e9,
                  "apply_frac": b_ap / t_ap / 1e9 / pk, "refactor_ms": 1e3 * tf,
                  "create_ms": 1e3 * t_create,
                  "levels": list(fac.levels()), "implicit_l": fac.implicit_l,
                  "bytes_matvec": b_mv, "bytes_apply": b_ap, "peak_GBps": pk, "gen_s": gen_s})
        del fac, Jd
        torch.cuda.empty_cache()


def config4(args):
    import torch
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.stepper import (LinearProblem, PrecondSpec, StepCache, dirk_step,
                                               irk_step_transformed)
    from paper_1701_07181_b200.tableau import builtin_tableau
    sys.path.insert(0, REPO)
    from bench import jnorm_device
    cfg = W.CONFIGS[1].scaled(ordering="color")
    wl = W.make_workload(cfg, jnorm=1.0)
    p = wl.pattern
    jn = args.jnorm or jnorm_device(p, wl.J)
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    u0 = torch.from_numpy(np.random.default_rng(11).standard_normal(prob.n)).cuda()
    gcfg = GmresConfig(rel_tol=1e-8, restart=40)
    for dtn in args.dtn:
        dt = dtn / jn
        for scheme in ("DIRK33", "RADAU23"):
            tab = builtin_tableau(scheme)
            cache = StepCache()

            def step(u, k):
                if tab.kind == "dirk":
                    return dirk_step(prob, tab, u, k * dt, dt, gmres_cfg=gcfg, cache=cache)
                return irk_step_transformed(prob, tab, u, k * dt, dt, PrecondSpec(kind="coupled"),
                                            gmres_cfg=gcfg, cache=cache)

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                r = step(u0, 0)
            except Exception as e:   # NewtonError / GMRES non-convergence: report it
                emit({"config": 4, "scheme": scheme, "dt_norm": dtn, "error": str(e)[:200]})
                continue
            torch.cuda.synchronize()
            first = time.perf_counter() - t0
            u = r.u_next
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            newton = gm = 0
            eq = 0.0
            for k in range(1, 1 + args.steps):
                r = step(u, k)
                u = r.u_next
                newton += r.newton_iterations
                gm += sum(st.iterations for st in r.gmres_stats)
                eq += r.equivalent_mults_avg
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.steps
            emit({"config": 4, "scheme": scheme, "precond": "ilu0" if tab.kind == "dirk" else "coupled",
                  "dt_norm": dtn, "dt": dt, "T": p.T, "nb": cfg.nb, "ms_per_step": ms,
                  "first_step_ms_with_factor": 1e3 * first, "steps": args.steps,
                  "newton_per_step": newton / args.steps, "gmres_per_step": gm / args.steps,
                  "equivalent_mults_per_step": eq / args.steps,
                  "u_norm": float(torch.linalg.vector_norm(u))})


def config2kernels(args):
    import torch
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    from bench import bytes_apply_uncoupled_shared, bytes_matvec
    cfg = W.CONFIGS[2].scaled(ordering="color")
    t0 = time.perf_counter()
    wl = W.make_workload(cfg, jnorm=1.0)
    gen = time.perf_counter() - t0
    p = wl.pattern
    jn = args.jnorm or 2.5
    dt = cfg.dt_norm / jn
    solver = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, dt,
                         kind="uncoupled", shifts=wl.shifts,
                         gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    rhs = torch.from_numpy(wl.rhs).cuda()
    del wl
    s, T, nb = cfg.s, cfg.T, cfg.nb
    w = torch.randn(s * T * nb, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    t_fac = timed(lambda: solver.factorize(), 2)
    t_mv = timed(lambda: solver.op.apply_device(w, y), 10)
    t_ap = timed(lambda: solver.fac.apply_device(w, y), 10)
    x = torch.empty_like(rhs)
    solver.solve(rhs, x=x)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    solver.factorize()
    _, st = solver.solve(rhs, x=x)
    b.record()
    torch.cuda.synchronize()
    pk = peak()
    t_up = int(np.count_nonzero(p.indptr[1:] - 1 > p.diag_pos))
    bm = bytes_matvec(T, 4, nb, s)
    ba = bytes_apply_uncoupled_shared(T, 4, nb, s, solver.fac.implicit_l, t_up)
    emit({"config": 2, "gpus": 1, "T": T, "nb": nb, "s": s, "dt_norm_assumed_jnorm": jn,
          "matvec_ms": 1e3 * t_mv, "matvec_GBps": bm / t_mv / 1e9, "matvec_frac": bm / t_mv / 1e9 / pk,
          "apply_ms": 1e3 * t_ap, "apply_GBps": ba / t_ap / 1e9, "apply_frac": ba / t_ap / 1e9 / pk,
          "factor_ms": 1e3 * t_fac, "stage_solve_ms": a.elapsed_time(b),
          "stage_solves_per_s": 1e3 / a.elapsed_time(b), "gmres_iterations": st.iterations,
          "converged": st.converged, "levels": list(solver.fac.levels()),
          "device_mem_used_GB": (lambda f: (f[1] - f[0]) / 1e9)(torch.cuda.mem_get_info()), "gen_s": gen})


def config0(args):
    """BASELINE config 0 (16x16 quads -> 512 triangles, nb=24, RADAU23, coupled block
    ILU(0), GMRES(30), dt*||J||=20): stage-solves/s (L2-resident plumbing case)."""
    import torch
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    cfg = W.CONFIGS[0]
    wl = W.make_workload(cfg)
    p = wl.pattern
    solver = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                         kind="coupled", gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    rhs = torch.from_numpy(wl.rhs).cuda()
    x = torch.empty_like(rhs)

    def step():
        solver.factorize()
        return solver.solve(rhs, x=x)[1]

    for _ in range(3):
        st = step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        st = step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    t_ap = timed(lambda: solver.fac.apply_device(rhs, x), 50)
    t_mv = timed(lambda: solver.op.apply_device(rhs, x), 50)
    t_fac = timed(lambda: solver.factorize(), 10)
    emit({"config": 0, "T": p.T, "nb": cfg.nb, "s": cfg.s, "precond": "coupled", "ms_per_stage_solve": ms,
          "stage_solves_per_s": 1e3 / ms, "gmres_iterations": st.iterations, "apply_us": 1e6 * t_ap,
          "matvec_us": 1e6 * t_mv, "factor_us": 1e6 * t_fac})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["config0", "config3", "config4", "config2kernels"])
    ap.add_argument("--nb", type=int, nargs="+", default=[24, 40, 50, 100])
    ap.add_argument("--s", type=int, nargs="+", default=[1, 2, 3, 4])
    ap.add_argument("--dtn", type=float, nargs="+", default=[10.0, 100.0, 1000.0])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--jnorm", type=float, default=None)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    {"config0": config0, "config3": config3, "config4": config4, "config2kernels": config2kernels}[a.what](a)


if __name__ == "__main__":
    main()
