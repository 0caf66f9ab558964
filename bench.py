#!/usr/bin/env python
"""Benchmark of the irk-b200 hot path (driver contract: one JSON line on rank 0).

Metric (BASELINE.json): IRK stage-solves/s; also BSR-matvec and ILU-apply GB/s
against the measured B200 HBM peak.  A *step* = one stage-solve = build the
shifted stage-uncoupled block ILU(0) of B = A^-1 (x) M - dt blkdiag(J) and run
GMRES(40) to rtol 1e-8, all on device-resident inputs (BASELINE config 1:
periodic 128x128 quad grid -> T=32768 triangles, nb=40, Radau IIA s=3,
dt*||J||_2 = 100).  Synthetic seeded inputs (no dataset exists); J entries
N(0, (1/nb)^2) (SURVEY 8d reading).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N>1 (torchrun): each rank runs its own replica of the workload (the single
config-1 system does not need partitioning; the partitioned solve lives in
paper_1701_07181_b200.distributed), timed with a barrier and the max over
ranks.  --impl reference times the CPU oracle (C restatement of the
reference kernels + its GMRES) on the host cores.
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

MEASURED = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE config (default: 1 at N=1, the 3D config 2 partitioned at N>1)")
    ap.add_argument("--N", type=int, default=None, help="override mesh cells per side")
    ap.add_argument("--ordering", default="color", choices=["natural", "color"],
                    help="element numbering (color: colour-major, the mesh-colouring level schedule)")
    ap.add_argument("--no-alt", action="store_true", help="skip the other-ordering measurement")
    ap.add_argument("--cpu-N", type=int, default=None,
                    help="CPU arms on a reduced mesh (cells per side; default: the full workload)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="timed steps only (for ncu)")
    ap.add_argument("--jnorm", type=float, default=None,
                    help="use this ||J||_2 instead of the power iteration (profiling runs)")
    ap.add_argument("--partitioned", action="store_true",
                    help="element-partitioned solve even at N=1 (always used for N>1)")
    ap.add_argument("--no-single", action="store_true",
                    help="N>1: skip rank 0's single-GPU solve of the same system")
    args = ap.parse_args()
    if args.config is None:
        args.config = 2 if (dist_env()[0] > 1 or args.partitioned) else 1
    return args


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def hbm_peak():
    try:
        with open(MEASURED) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes (Bk = 8 nb^2, v = 8 T nb, int32 indices)
# ---------------------------------------------------------------------------

def bytes_matvec(T, r, nb, s):
    nnzb = T * (r + 1)
    Bk, v = 8 * nb * nb, 8 * T * nb
    return nnzb * Bk + T * Bk + 2 * s * v + 4 * (nnzb + T + 1)


def bytes_apply_uncoupled_shared(T, r, nb, s, implicit_l=False, t_up=None):
    """Stored L: L and D^-1 per stage, U = -dt J upper read once for all stages.
    Implicit L: the stage-shared J is read once for the lower and once for the
    upper blocks; D^-1 of rows with upper blocks is read twice (w = D^-1 z in
    the forward sweep, x in the backward one) and their w is written and
    gathered back (t_up = number of such rows)."""
    Bk, v = 8 * nb * nb, 8 * T * nb
    up = T * r // 2
    if not implicit_l:
        return up * Bk + s * (up + T) * Bk + 2 * s * v
    t_up = T if t_up is None else t_up
    return 2 * up * Bk + s * (T + t_up) * Bk + 2 * s * v + 2 * s * 8 * t_up * nb


def factor_flops(T, r, nb, s):
    """Uncoupled simplified ILU(0) flops: s*T*nb^3*(2 + 2r)."""
    return s * T * nb ** 3 * (2 + 2 * r)


def fp64_peak():
    """Measured FP64 tensor-core (DMMA) peak: tools/dmma_peak.cu run on a B200 of
    this pool (profiles/r2_fp64_peak.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "r2_fp64_peak.json")) as fh:
            d = json.load(fh)
        d["source"] = "profiles/r2_fp64_peak.json (tools/dmma_peak.cu, measured)"
        return d
    except Exception:
        return None


def make_config(args):
    from paper_1701_07181_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    kw = {"ordering": args.ordering}
    if args.N:
        kw["N"] = args.N
    return cfg.scaled(**kw)


def jnorm_device(pattern, J, iters=60, seed=7):
    """||J||_2 by power iteration on J^T J with the library's BSR matvec."""
    import torch
    from paper_1701_07181_b200.blocks import BlockSparseMatrix, DeviceBlocks
    p = pattern
    rows = np.repeat(np.arange(p.T), np.diff(p.indptr))
    # transposed pattern is the same (symmetric adjacency); block (i,j) of J^T = J_ji^T
    order = np.lexsort((rows, p.indices))          # sort by (col, row)
    JT = np.ascontiguousarray(J[order].transpose(0, 2, 1))
    from paper_1701_07181_b200.blocks import DevicePattern
    dp = DevicePattern(p.indptr, p.indices, p.diag_pos)
    A = BlockSparseMatrix(dp, DeviceBlocks.from_host(J))
    At = BlockSparseMatrix(dp, DeviceBlocks.from_host(JT))
    g = torch.Generator(device="cpu").manual_seed(seed)
    v = torch.randn(p.T * J.shape[1], generator=g, dtype=torch.float64).cuda()
    v /= torch.linalg.vector_norm(v)
    lam = 0.0
    for _ in range(iters):
        w = At.matvec(A.matvec(v))
        lam = float(torch.linalg.vector_norm(w))
        v = w / lam
    return float(np.sqrt(lam))


def jnorm_host(pattern, J, iters=60, seed=7):
    """||J||_2 on the host: the same power iteration on J^T J as jnorm_device
    (same start vector, same iteration count) with the oracle's C BSR matvec."""
    import torch
    import oracle as O
    p = pattern
    rows = np.repeat(np.arange(p.T), np.diff(p.indptr))
    order = np.lexsort((rows, p.indices))
    JT = np.ascontiguousarray(J[order].transpose(0, 2, 1))
    g = torch.Generator(device="cpu").manual_seed(seed)
    v = torch.randn(p.T * J.shape[1], generator=g, dtype=torch.float64).numpy()
    v = v / np.linalg.norm(v)
    lam = 0.0
    for _ in range(iters):
        w = O.bsr_matvec(p.indptr, p.indices, JT, O.bsr_matvec(p.indptr, p.indices, J, v))
        lam = float(np.linalg.norm(w))
        v = w / lam
    return float(np.sqrt(lam))


def cpu_workload(args):
    """The config's workload on the host (same generator, seeds and numbering as
    the GPU arm; ||J||_2 by the same power iteration) for the CPU arms."""
    from paper_1701_07181_b200 import workloads as W
    cfg = make_config(args)
    scfg = cfg.scaled(N=args.cpu_N) if args.cpu_N else cfg
    wl = W.make_workload(scfg, jnorm=1.0)
    jn = args.jnorm if args.jnorm else jnorm_host(wl.pattern, wl.J)
    wl.jnorm, wl.dt = jn, scfg.dt_norm / jn
    return cfg, scfg, wl


def cpu_sample(args, reps=1, prebuilt=None):
    """CPU oracle (C restatement of the reference kernels, OpenMP, + its numpy
    MGS GMRES) on one full stage-solve of the SAME workload (no extrapolation):
    about 10 s of host work at config 1.  ``prebuilt`` = (cfg, wl) reuses the GPU
    arm's host arrays and dt."""
    import oracle as O
    if prebuilt is not None:
        cfg, wl = prebuilt
        scfg = cfg
    else:
        cfg, scfg, wl = cpu_workload(args)
    prob = O.problem_from_workload(wl)
    times = []
    iters = None
    for _ in range(reps):
        t0 = time.perf_counter()
        fac = O.make_preconditioner(prob, scfg.precond, wl.shifts, workers=scfg.s)
        x, st = O.gmres(prob.matvec, fac.apply, wl.rhs,
                        O.GmresConfig(rel_tol=scfg.rtol, restart=scfg.restart))
        times.append(time.perf_counter() - t0)
        iters = st.iterations
    t = min(times)
    scale = wl.pattern.T / cfg.T
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    return {
        "value": scale / t, "unit": "stage-solves/s", "cores": threads, "kind": "port",
        "sample": (f"oracle/irk_oracle.c (C restatement of the reference numba kernels, OpenMP "
                   f"rows + {scfg.s} stage threads) + numpy MGS GMRES: one complete stage-solve "
                   f"(factor + GMRES to rtol) of the config-{args.config} workload itself "
                   f"(T={wl.pattern.T}), {t:.2f} s, {iters} GMRES iterations"
                   + ("" if scale == 1.0 else f"; rate scaled by T_sample/T = {scale:.4f}")),
        "reference_numba_1core": REFERENCE_NUMBA,
    }


def _ref_numba():
    """The unmodified reference (irksolve, numba backend, one core: its kernels
    hold the GIL) timed on the same config-1 stage-solve in the BUILD container
    (tools/ref_numba_rate.py; /root/reference does not exist on the GPU box)."""
    try:
        with open(os.path.join(REPO, "profiles", "r2_reference_numba_1core.json")) as fh:
            d = json.load(fh)
        return {"value": d["stage_solves_per_s_at_T"], "unit": "stage-solves/s", "cores": 1,
                "seconds_per_stage_solve": d["total_s"], "iterations": d["iterations"],
                "where": "build container, 8-core x86_64 (not this box); tools/ref_numba_rate.py",
                "source": "profiles/r2_reference_numba_1core.json"}
    except Exception:
        return None


REFERENCE_NUMBA = _ref_numba()


def run_reference(args):
    """The reference arm: the reference's algorithm on the host cores (the C
    oracle port -- the reference is Python/numba, nothing to compile), every
    step one COMPLETE stage-solve of the same full-size workload (factor + GMRES
    to rtol; ~10 s on 16 threads at config 1).  Warm-up capped at one step so the
    whole run stays within a few minutes."""
    world, rank, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    import oracle as O
    t_setup = time.perf_counter()
    cfg, scfg, wl = cpu_workload(args)
    prob = O.problem_from_workload(wl)
    t_setup = time.perf_counter() - t_setup

    def step():
        fac = O.make_preconditioner(prob, scfg.precond, wl.shifts, workers=scfg.s)
        return O.gmres(prob.matvec, fac.apply, wl.rhs, O.GmresConfig(rel_tol=scfg.rtol, restart=scfg.restart))

    warm = min(args.warmup, 1)
    for _ in range(warm):
        step()
    t0 = time.perf_counter()
    conv = True
    for _ in range(args.steps):
        _, st = step()
        conv &= bool(st.converged)
    t = time.perf_counter() - t0
    scale = wl.pattern.T / cfg.T
    value = args.steps * scale / t
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    line = {
        "impl": "reference", "metric": "IRK stage-solves/sec", "value": value,
        "unit": "stage-solves/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": warm,
        "ms_per_step": 1e3 * t / args.steps / scale, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args),
        "cpu_baseline": {"value": value, "unit": "stage-solves/s", "cores": threads,
                         "kind": "port",
                         "sample": (f"each step: one complete stage-solve of the config-{args.config} "
                                    f"workload (T={wl.pattern.T}) with the C oracle (OpenMP, "
                                    f"{threads} threads) + MGS GMRES, {st.iterations} iterations, "
                                    f"converged={conv}; warm-up capped at {warm}"
                                    + ("" if scale == 1.0 else f"; rate scaled by {scale:.4f}")),
                         "reference_numba_1core": REFERENCE_NUMBA},
        "e2e": {"value": value, "unit": "stage-solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "consistency": {"timed_s": t, "setup_s": t_setup,
                        "steps_x_ms_per_step_s": args.steps * 1e-3 * (1e3 * t / args.steps / scale)},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def config_dict(cfg, args):
    mesh = (f"periodic {cfg.N}x{cfg.N} quads -> {cfg.T} triangles" if cfg.mesh == "tri2d" else
            f"periodic {cfg.N}^3 cubes -> {cfg.T} Kuhn tetrahedra")
    return {
        "workload": (f"cfg{args.config}: {mesh}, "
                     f"nb={cfg.nb}, {cfg.scheme} (s={cfg.s}), {cfg.precond} block ILU(0) "
                     f"({cfg.ordering} numbering), GMRES({cfg.restart}) rtol {cfg.rtol}, "
                     f"dt*||J||2={cfg.dt_norm}, J std 1/nb"),
        "T": cfg.T, "nb": cfg.nb, "s": cfg.s, "precond": cfg.precond, "restart": cfg.restart,
        "rtol": cfg.rtol, "ordering": cfg.ordering,
        "l2": "inputs larger than L2 (J alone is %.2f GB > 126 MB)" % (cfg.T * 4 * 8 * cfg.nb ** 2 / 1e9),
        "parallelism": "single GPU",
    }


def run_b200(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.blocks import DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    from paper_1701_07181_b200.tableau import builtin_tableau, derive

    cfg = make_config(args)
    s = cfg.s
    wl = W.make_workload(cfg, jnorm=1.0)     # host arrays; dt comes from the GPU norm below
    pat, J, M, rhs_h = wl.pattern, wl.J, wl.M, wl.rhs
    der = derive(builtin_tableau(cfg.scheme))
    log(f'workload generated T={pat.T}')
    jnorm = args.jnorm if args.jnorm else jnorm_device(pat, J)
    log(f'jnorm {jnorm:.4f}')
    dt = cfg.dt_norm / jnorm
    dpat = DevicePattern(pat.indptr, pat.indices, pat.diag_pos)
    gcfg = GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart, max_iters=cfg.max_iters)
    solver = StageSolver(dpat, J, M, der.a_inv, dt, kind=cfg.precond, shifts=der.shifts,
                         gmres_cfg=gcfg)
    log('solver ready')
    rhs = torch.from_numpy(rhs_h).cuda()
    x = torch.empty_like(rhs)
    stream = torch.cuda.current_stream()

    def step():
        solver.factorize()
        _, st = solver.solve(rhs, x=x)
        return st

    b_norm = float(np.linalg.norm(rhs_h))
    for _ in range(max(args.warmup, 0)):
        st = step()
        log(f'warmup step: {st.iterations} iterations')
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    launches0 = L.lib().irk_launch_count()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.profile:
        torch.cuda.profiler.start()    # ncu --profile-from-start off: the timed steps only
    ev0.record(stream)
    iters, stats = [], []
    for _ in range(args.steps):
        st = step()
        iters.append(st.iterations)
        stats.append(st)
    ev1.record(stream)
    torch.cuda.synchronize()
    if args.profile:
        torch.cuda.profiler.stop()
    launches = L.lib().irk_launch_count() - launches0
    log('timed region done')
    # every timed stage-solve must have converged (GmresStats are host scalars read
    # after each solve's single end-of-loop sync; no extra sync inside the region)
    assert all(st_.converged for st_ in stats), [st_.iterations for st_ in stats]
    true_res = [st_.final_true_residual / b_norm for st_ in stats]
    clocks = clk.stop()
    t_local = ev0.elapsed_time(ev1) / 1e3
    t = t_local
    if dist:
        tt = torch.tensor([t_local], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt)
        dist.barrier()
    value = world * args.steps / t
    if args.profile:
        if rank == 0:
            print(json.dumps({"metric": "IRK stage-solves/sec", "value": value, "profile": True}))
        return

    # ---- component timings (outside the timed region) -------------------
    T, r, nb = cfg.T, 3 if cfg.mesh == "tri2d" else 4, cfg.nb
    w = torch.randn(s * T * nb, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3 / reps

    t_mv = timed(lambda: solver.op.apply_device(w, y), 20)
    log('components timed')
    t_ap = timed(lambda: solver.fac.apply_device(w, y), 10)
    # the Arnoldi product P^-1 (B v) as irk_gmres runs it (stage matvec fused into the
    # forward sweep when the factor qualifies, krylov.cu / apply.cu k_unc_fused_fwd)
    import ctypes
    from paper_1701_07181_b200 import _lib as L
    fused_flag = ctypes.c_int(0)

    def product():
        L.check(L.lib().irk_op_factor_apply(solver.op._op.handle, solver.fac.handle, w.data_ptr(),
                                            y.data_ptr(), ctypes.byref(fused_flag), L.stream_ptr()),
                "irk_op_factor_apply")
    def timed_each(fn, reps):
        # one synchronised event pair per call: irk_gmres waits on the host after every
        # Arnoldi step, so back-to-back calls (PDL-chained across calls) are not its regime
        fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b) / 1e3
        return tot / reps
    t_fu = timed_each(product, 10) if solver.fac is not None else None
    t_fu_b2b = timed(product, 10) if solver.fac is not None else None
    t_fac = timed(lambda: solver.factorize(), 3)
    t_sol = timed(lambda: solver.solve(rhs, x=x), 3)
    peak, peak_src = hbm_peak()
    bm = bytes_matvec(T, r, nb, s)
    implicit_l = bool(getattr(solver.fac, "implicit_l", False))
    t_up = int(np.count_nonzero(pat.indptr[1:] - 1 > pat.diag_pos))   # rows with an upper block
    ba = (bytes_apply_uncoupled_shared(T, r, nb, s, implicit_l, t_up)
          if cfg.precond.startswith("uncoupled") else None)
    ms_step = 1e3 * t / args.steps
    it_mean = float(np.mean(iters))
    # operator applications per stage-solve: 1 (P^-1 b) + iters (+ restarts) applies,
    # iters + 1 (true residual) matvecs
    share_ap = (it_mean + 1) * t_ap / (t / args.steps)
    share_mv = (it_mean + 1) * t_mv / (t / args.steps)
    bf = (bm + ba - (T * r // 2) * 8 * nb * nb - 2 * s * 8 * T * nb) if (ba is not None and implicit_l) else None
    if bf is not None and fused_flag.value:
        # per stage-solve: `iters` fused products, one plain apply (P^-1 b), one matvec (true residual)
        share_ap = t_ap / (t / args.steps)
        share_mv = t_mv / (t / args.steps)
        share_fu = it_mean * t_fu / (t / args.steps)
    else:
        share_fu = 0.0
    if share_fu > max(share_ap, share_mv):
        dom = {"name": "arnoldi_product P^-1 (B v) (matvec fused into the forward sweep + backward sweep)",
               "bytes": bf, "t": t_fu, "share": share_fu, "key": "arnoldi_product"}
    elif ba is not None and share_ap >= share_mv:
        dom = {"name": "ilu0_apply (fwd+bwd sweeps, all stages)", "bytes": ba, "t": t_ap, "share": share_ap,
               "key": "ilu0_apply"}
    else:
        dom = {"name": "stage_matvec (fused)", "bytes": bm, "t": t_mv, "share": share_mv, "key": "stage_matvec"}
    achieved = dom["bytes"] / dom["t"] / 1e9
    traffic = None
    traffic_src = None
    try:   # DRAM bytes per launch from the latest committed ncu capture (profiles/rNN_traffic.json)
        import glob
        cands = sorted(glob.glob(os.path.join(REPO, "profiles", "r*_traffic.json")))
        with open(cands[-1]) as fh:
            tj = json.load(fh)
        traffic = tj[dom["key"]]
        traffic_src = "profiles/" + os.path.basename(cands[-1])
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": dom["name"],
                "algorithmic_bytes_per_launch": dom["bytes"], "avg_launch_ms": 1e3 * dom["t"],
                "share_of_step": dom["share"], "peak_source": peak_src, "traffic_source": traffic_src,
                # DRAM bytes (ncu, profiles/) over the event-timed launch: wasted re-reads show here
                "traffic_GBps": (traffic / dom["t"] / 1e9) if traffic else None}
    components = {
        "matvec_ms": 1e3 * t_mv, "matvec_GBps": bm / t_mv / 1e9, "matvec_frac": bm / t_mv / 1e9 / peak,
        "apply_ms": 1e3 * t_ap,
        "apply_GBps": (ba / t_ap / 1e9) if ba else None,
        "apply_frac": (ba / t_ap / 1e9 / peak) if ba else None,
        "arnoldi_product_ms": (1e3 * t_fu) if t_fu else None,
        "arnoldi_product_fused": bool(fused_flag.value),
        "arnoldi_product_back_to_back_ms": (1e3 * t_fu_b2b) if t_fu_b2b else None,
        "arnoldi_product_GBps": (bf / t_fu / 1e9) if (bf and t_fu and fused_flag.value) else None,
        "arnoldi_product_frac": (bf / t_fu / 1e9 / peak) if (bf and t_fu and fused_flag.value) else None,
        "factor_ms": 1e3 * t_fac, "gmres_ms": 1e3 * t_sol, "gmres_iterations": iters[-1],
        "gmres_ms_per_iteration": 1e3 * t_sol / max(iters[-1], 1),
        "levels_fwd_bwd": list(solver.fac.levels()) if solver.fac is not None else None,
        "jnorm2": jnorm, "dt": dt,
        "all_timed_steps_converged": True,
        "final_true_residual_rel": true_res[-1],
        "max_true_residual_rel": max(true_res),
    }
    # the reference-level drop-in (install_stepper): the reference's glue builds a fresh
    # factor and calls gmres with its wrappers lambda v: op.matvec(v, counter) /
    # lambda v: fac.apply(v, counter) on a host rhs (stepper.py:164-170); krylov.gmres
    # recognises them and runs the native loop (fused product), charging the counters
    from paper_1701_07181_b200 import krylov as K
    from paper_1701_07181_b200.blocks import OpCounter
    from paper_1701_07181_b200.precond import stage_uncoupled_factorize
    ctr = OpCounter()
    op_ = solver.op

    def dropin_step():
        fac_ = stage_uncoupled_factorize(op_, der.shifts, ctr)
        x_, st_ = K.gmres(lambda v: op_.matvec(v, ctr), lambda v: fac_.apply(v, ctr), rhs_h, gcfg)
        return st_
    if cfg.precond == "uncoupled":
        dropin_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            st_d = dropin_step()
        torch.cuda.synchronize()
        components["dropin_reference_glue_ms"] = 1e3 * (time.perf_counter() - t0) / 3
        components["dropin_reference_glue_iterations"] = st_d.iterations
        components["dropin_note"] = ("reference stepper glue through install_stepper: new factor + gmres with "
                                     "the reference's lambda wrappers on a host rhs (H2D rhs, D2H x), native loop")
    fp64 = fp64_peak()
    if fp64:
        flops_factor = factor_flops(T, r, nb, s)
        components["factor_tflops"] = flops_factor / t_fac / 1e12
        components["factor_frac_of_fp64_tc_peak"] = flops_factor / t_fac / 1e12 / fp64["fp64_dmma_tflops"]
        components["fp64_tc_peak_tflops"] = fp64["fp64_dmma_tflops"]
        components["fp64_peak_source"] = fp64["source"]

    # ---- end to end through host buffers (pinned), C-ABI upload path ------
    e2e = None
    if not args.no_e2e:
        Jp = torch.from_numpy(J).pin_memory()
        Mp = torch.from_numpy(M).pin_memory()
        rp = torch.from_numpy(rhs_h).pin_memory()
        xp = torch.empty_like(rp).pin_memory()
        jb = solver.op.jacobians[0].blocks
        mb = solver.op.mass.device

        def e2e_step():
            jb.upload(Jp.numpy())
            mb.upload(Mp.numpy())
            rhs.copy_(rp, non_blocking=True)
            solver.factorize()
            solver.solve(rhs, x=x)
            xp.copy_(x, non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        ne = max(1, min(args.steps, 3))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        te_serial = time.perf_counter() - t0

        # Double-buffered: a second device copy of the system (its own J, M, factor and
        # vectors); step k+1's inputs go H2D on a copy stream while step k factorises and
        # solves, so the PCIe transfer (the bound) runs back to back.  Every step still
        # uploads its own J, M, rhs and downloads its own solution inside the timed region.
        solver_b = StageSolver(dpat, J, M, der.a_inv, dt, kind=cfg.precond, shifts=der.shifts,
                               gmres_cfg=gcfg)
        rhs_b, x_b = torch.empty_like(rhs), torch.empty_like(x)
        sets = [(solver, rhs, x), (solver_b, rhs_b, x_b)]
        xps = [xp, torch.empty_like(rp).pin_memory()]
        cstream = torch.cuda.Stream()
        up_done = [torch.cuda.Event(), torch.cuda.Event()]
        comp_done = [torch.cuda.Event(), torch.cuda.Event()]
        for e in comp_done:
            e.record(stream)

        def upload(k):
            sv, r, _ = sets[k % 2]
            with torch.cuda.stream(cstream):
                cstream.wait_event(comp_done[k % 2])   # the set's previous solve is finished
                sv.op.jacobians[0].blocks.upload(Jp.numpy())
                sv.op.mass.device.upload(Mp.numpy())
                r.copy_(rp, non_blocking=True)
                up_done[k % 2].record(cstream)

        def compute(k):
            sv, r, xx = sets[k % 2]
            stream.wait_event(up_done[k % 2])
            sv.factorize()
            sv.solve(r, x=xx)
            xps[k % 2].copy_(xx, non_blocking=True)
            comp_done[k % 2].record(stream)

        solver_b.factorize()
        torch.cuda.synchronize()
        npipe = max(3, min(2 * args.steps, 20))   # pipeline fill amortised over <= 20 systems (~0.8 s)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        upload(0)
        for k in range(npipe):
            if k + 1 < npipe:
                upload(k + 1)
            compute(k)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        ok = bool(torch.equal(x, x_b)) and bool(torch.equal(xps[0], xps[1]))
        if dist:
            tt = torch.tensor([te, te_serial], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te, te_serial = float(tt[0]), float(tt[1])
        e2e = {"value": world * npipe / te, "unit": "stage-solves/s",
               "h2d_bytes_per_step": int(J.nbytes + M.nbytes + rhs_h.nbytes),
               "d2h_bytes_per_step": int(rhs_h.nbytes),
               "serial_value": world * ne / te_serial,
               "double_buffered_results_identical": ok,
               "note": "pinned host J, M, rhs -> irk_blocks_upload / H2D, factorise + GMRES, "
                       "solution D2H, every step; double-buffered (two device copies of the system, "
                       "step k+1's H2D on a copy stream during step k's solve); serial_value: one "
                       "device copy, upload -> solve -> download in turn"}
        del solver_b, sets
    log('e2e done')
    alt = None
    if not args.no_alt:
        # the same system under the other element numbering (a different ILU(0))
        other = "natural" if cfg.ordering == "color" else "color"
        wl2 = W.make_workload(cfg.scaled(ordering=other), jnorm=1.0)
        p2 = wl2.pattern
        s2 = StageSolver(DevicePattern(p2.indptr, p2.indices, p2.diag_pos), wl2.J, wl2.M,
                         der.a_inv, dt, kind=cfg.precond, shifts=der.shifts, gmres_cfg=gcfg)
        r2 = torch.from_numpy(wl2.rhs).cuda()
        x2 = torch.empty_like(r2)

        def step2():
            s2.factorize()
            return s2.solve(r2, x=x2)[1]

        step2()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        n2 = 3
        for _ in range(n2):
            st2 = step2()
        a1.record(stream)
        torch.cuda.synchronize()
        t2 = a0.elapsed_time(a1) / 1e3 / n2
        alt = {"ordering": other, "stage_solves_per_s": 1.0 / t2, "ms_per_step": 1e3 * t2,
               "gmres_iterations": st2.iterations,
               "apply_ms": 1e3 * timed(lambda: s2.fac.apply_device(w, y), 5),
               "factor_ms": 1e3 * timed(lambda: s2.factorize(), 2),
               "levels_fwd_bwd": list(s2.fac.levels())}
        del s2
        log('other ordering done')
    if rank != 0:
        return
    if not args.no_cpu:
        wl.jnorm, wl.dt = jnorm, dt
        cpu = cpu_sample(args, prebuilt=(cfg, wl))
    else:
        cpu = None
    line = {
        "metric": "IRK stage-solves/sec", "value": value, "unit": "stage-solves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, no dataset; J std 1/nb)",
        "config": config_dict(cfg, args), "gmres_iterations_mean": it_mean,
        "roofline": roofline, "components": components, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches), "clocks": clocks, "other_ordering": alt,
    }
    print(json.dumps(line), flush=True)


def log(msg):
    if os.environ.get("BENCH_QUIET") != "1":
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def estimate_jnorm(cfg):
    """||J||_2 for dt: exact power iteration on the GPU when the global J fits
    comfortably on one rank (config 1), else on a reduced mesh of the same
    generator (16^3 cubes for the 3D workload: the norm of these random block
    matrices is nearly independent of the mesh size -- 2.4485 at 32x32 vs 2.4496
    at 128x128 quads)."""
    from paper_1701_07181_b200 import workloads as W
    c = cfg if cfg.T <= 40000 else cfg.scaled(N=16 if cfg.mesh == "tet3d" else 32)
    wl = W.make_workload(c.scaled(ordering="natural"), jnorm=1.0)
    return jnorm_device(wl.pattern, wl.J), c.T


def fused_bytes_local(plan, fac_levels_ok, s, nb):
    """Algorithmic bytes of one partitioned Arnoldi product P^-1 (B v) on a rank
    (the N=1 formula of DESIGN.md section 3 on the slab): every operator block of
    the slab's rows once (own and ghost columns), M, the kept upper blocks (the
    backward sweep reads U = -dt J), D^-1 once per row and once more for rows with
    a kept upper block, v (+ ghosts) read, x written, w = D^-1 z of those rows
    written and gathered back."""
    Bk = 8 * nb * nb
    Tl, ng = plan.T_local, plan.n_ghost
    rows = np.repeat(np.arange(Tl), np.diff(plan.loc_indptr))
    up = int(np.count_nonzero(plan.loc_indices > rows))
    t_up = int(np.count_nonzero(np.bincount(rows[plan.loc_indices > rows], minlength=Tl)))
    ext_nnzb = int(plan.ext_indptr[-1])
    return (ext_nnzb + up + Tl + s * (Tl + t_up)) * Bk + 8 * nb * s * (2 * Tl + ng + 2 * t_up)


def run_partitioned(args):
    """Element-partitioned solve of ONE global system over all ranks (strong
    scaling): the 3D workload (BASELINE config 2: 32^3 cubes -> 196,608 Kuhn
    tets, nb=50, Radau IIA s=3, shifted uncoupled ILU(0), GMRES(40)) cut into
    contiguous z-slabs (colour-major inside each slab), the native layer of
    libirkb200 on every rank: NCCL halo (irk_halo), the slab's operator rows
    (irk_dist_op, fused Arnoldi product after the exchange), partitioned
    communication-free ILU(0), irk_gmres with NCCL allreduces (no Python in the
    loop).  Rank 0 also solves the same system alone on its GPU first (P=1) and
    reports it as ``single_gpu`` so the per-N values of this workload can be
    compared."""
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200 import workloads as W
    from paper_1701_07181_b200.distributed import DistributedStageSolver, SlabPlan
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.tableau import builtin_tableau, derive
    cfg = make_config(args)
    P = world
    der = derive(builtin_tableau(cfg.scheme))
    gcfg = GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart, max_iters=cfg.max_iters)
    stream = torch.cuda.current_stream()
    if rank == 0:
        jnorm, norm_T = (args.jnorm, None) if args.jnorm else estimate_jnorm(cfg)
    else:
        jnorm, norm_T = 0.0, None
    if dist:
        tj = torch.tensor([jnorm], dtype=torch.float64, device="cuda")
        dist.broadcast(tj, 0)
        jnorm = float(tj)
    dt = cfg.dt_norm / jnorm
    s, nb = cfg.s, cfg.nb

    def build(Pn, r, group_transport):
        pat, J, M, rhs_h = W.make_slab_workload(cfg, Pn, r)
        plan = SlabPlan.build(pat.indptr, pat.indices, pat.diag_pos, Pn, r)
        sol = DistributedStageSolver(plan, J, M, der.a_inv, dt, cfg.precond, der.shifts, gcfg,
                                     transport=group_transport)
        return plan, sol, J, M, rhs_h

    def run_steps(sol, rhs, x, n):
        its, conv = [], True
        for _ in range(n):
            sol.factorize()
            st = sol.solve(rhs, x=x)[1]
            its.append(st.iterations)
            conv &= bool(st.converged)
        return its, conv, st

    # ---- P = 1 on rank 0 (same system, same numbering rule, one GPU) ----------
    single = None
    if world > 1 and rank == 0 and not args.no_single:
        from paper_1701_07181_b200.distributed import Comm
        plan1, sol1, *_rest, rhs1 = build(1, 0, Comm.single())
        r1 = torch.from_numpy(rhs1).cuda()
        x1 = torch.empty_like(r1)
        run_steps(sol1, r1, x1, 2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n1 = max(2, min(args.steps, 5))
        e0.record(stream)
        its1, conv1, _ = run_steps(sol1, r1, x1, n1)
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = e0.elapsed_time(e1) / 1e3
        single = {"value": n1 / t1, "unit": "stage-solves/s", "ms_per_step": 1e3 * t1 / n1,
                  "gmres_iterations": its1[-1], "converged": conv1,
                  "note": "the same global system solved by rank 0 alone (P=1 partition, one GPU), "
                          "measured in this run before the partitioned steps"}
        del sol1, plan1, _rest, r1, x1
        torch.cuda.empty_cache()
        log(f"single-GPU reference: {single['value']:.2f} stage-solves/s")
    if dist:
        dist.barrier()
    plan, sol, J, M, rhs_h = build(P, rank, "auto")
    rhs = torch.from_numpy(rhs_h).cuda()
    x = torch.empty_like(rhs)
    log(f"rank {rank}: slab {plan.lo}..{plan.hi} ghosts {plan.n_ghost}")
    run_steps(sol, rhs, x, max(args.warmup, 0))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    launches0 = L.lib().irk_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters, conv, st = run_steps(sol, rhs, x, args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = L.lib().irk_launch_count() - launches0
    clocks = clk.stop()
    assert conv, iters
    t = ev0.elapsed_time(ev1) / 1e3
    # local components (outside the timed region): the partitioned Arnoldi product
    # (halo exchange + fused sweeps) and the factor
    v = torch.randn(sol.n_local, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    _, fused = sol.product(v, out)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sol.product(v, out)
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b) / 1e3
    t_prod = tot / 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        sol.factorize()
    b.record(stream)
    torch.cuda.synchronize()
    t_fac = a.elapsed_time(b) / 1e3 / 3
    # e2e through the public API: this rank's slab J, M, rhs from pinned host memory, factor,
    # solve, solution back, every step (serial)
    # (the slab solver keeps two device copies of its J rows: the operator's, in extended-pattern
    # order with the ghost columns, and the factor's, local columns only -- both are uploaded)
    Jp = torch.from_numpy(np.ascontiguousarray(J[plan.row_block_src - plan.q0])).pin_memory()
    Jfp = torch.from_numpy(np.ascontiguousarray(J[plan.loc_block_src - plan.q0])).pin_memory()
    rp = torch.from_numpy(rhs_h).pin_memory()
    xp = torch.empty_like(rp).pin_memory()
    jb = sol.op.jacobians[0].blocks
    jfb = sol.fac_op.jacobians[0].blocks
    Mp = torch.from_numpy(np.ascontiguousarray(M)).pin_memory()
    mb = sol.fac_op.mass.device
    mob = sol.mass.device

    def e2e_step():
        jb.upload(Jp.numpy())
        jfb.upload(Jfp.numpy())
        mb.upload(Mp.numpy())
        mob.upload(Mp.numpy())
        rhs.copy_(rp, non_blocking=True)
        sol.factorize()
        sol.solve(rhs, x=x)
        xp.copy_(x, non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    if dist:
        dist.barrier()
    ne = 2
    t0 = time.perf_counter()
    for _ in range(ne):
        e2e_step()
    te = time.perf_counter() - t0
    tt = torch.tensor([t, t_prod, t_fac, te], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t, t_prod_max, t_fac_max, te = (float(v_) for v_ in tt)
    value = args.steps / t
    if rank != 0:
        if dist:
            dist.barrier()
        return
    peak, peak_src = hbm_peak()
    fb = fused_bytes_local(plan, True, s, nb)
    r = 3 if cfg.mesh == "tri2d" else 4
    line = {
        "metric": "IRK stage-solves/sec", "value": value, "unit": "stage-solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, no dataset; J std 1/nb)",
        "config": dict(config_dict(cfg, args), parallelism=f"element-partitioned x{world} (z-slabs; "
                       "native NCCL halo send/recv + allreduce in libirkb200; partitioned block ILU(0))",
                       jnorm_mesh_T=norm_T),
        "gmres_iterations_mean": float(np.mean(iters)),
        "all_timed_steps_converged": True,
        "final_true_residual_rel": st.final_true_residual / float(np.linalg.norm(rhs_h)) if world == 1 else None,
        "single_gpu": single,
        "roofline": {"bound": "hbm", "achieved": fb / t_prod / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": fb / t_prod / 1e9 / peak, "traffic": None,
                     "kernel": "rank-0 partitioned Arnoldi product P^-1 (B v): halo pack + NCCL exchange + "
                               "fused forward sweep (ghost segments) + backward sweep",
                     "algorithmic_bytes_per_launch": fb, "avg_launch_ms": 1e3 * t_prod,
                     "fused": bool(fused), "peak_source": peak_src},
        "components": {"arnoldi_product_ms_rank0": 1e3 * t_prod, "arnoldi_product_ms_max": 1e3 * t_prod_max,
                       "factor_ms_max": 1e3 * t_fac_max, "halo_elements_rank0": int(plan.n_ghost),
                       "halo_bytes_per_exchange_rank0": int(8 * s * nb * plan.n_ghost),
                       "T_local_rank0": int(plan.T_local), "jnorm2": jnorm, "dt": dt},
        "cpu_baseline": None,
        "e2e": {"value": ne / te, "unit": "stage-solves/s",
                "h2d_bytes_per_step": int(Jp.numel() * 8 + Jfp.numel() * 8 + 2 * Mp.numel() * 8 + rp.numel() * 8),
                "d2h_bytes_per_step": int(xp.numel() * 8),
                "note": "per rank: its slab's J, M, rhs from pinned host memory through irk_blocks_upload / "
                        "H2D, factor + GMRES, solution D2H, every step (serial); max over ranks; bytes are "
                        "rank 0's"},
        "gpu_launches": int(launches), "clocks": clocks,
        "note": "cpu_baseline is reported by the N=1 run (config 1)",
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()


def main():
    import faulthandler
    faulthandler.enable()
    if os.environ.get("BENCH_HANG_DUMP"):
        faulthandler.dump_traceback_later(float(os.environ["BENCH_HANG_DUMP"]), exit=True)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1 or args.partitioned:
        run_partitioned(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
