"""Tuning sweep for the ILU(0) sweep kernels (config 1): ring stages x groups.

Reads the IRK_APPLY_NST / IRK_APPLY_G knobs of apply.cu; prints one line
per setting with the apply time and the fraction of the measured HBM peak.
"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1701_07181_b200 import workloads as W  # noqa: E402
from paper_1701_07181_b200.blocks import DevicePattern  # noqa: E402
from paper_1701_07181_b200.krylov import GmresConfig  # noqa: E402
from paper_1701_07181_b200.solver import StageSolver  # noqa: E402
from paper_1701_07181_b200.tableau import builtin_tableau, derive  # noqa: E402


def main():
    cfg = W.CONFIGS[1].scaled(ordering=os.environ.get("ORDERING", "color"))
    wl = W.make_workload(cfg, jnorm=1.0)
    der = derive(builtin_tableau(cfg.scheme))
    dt = cfg.dt_norm / 2.4496432463318416
    dpat = DevicePattern(wl.pattern.indptr, wl.pattern.indices, wl.pattern.diag_pos)
    solver = StageSolver(dpat, wl.J, wl.M, der.a_inv, dt, kind=cfg.precond, shifts=der.shifts,
                         gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    solver.factorize()
    T, nb, s = wl.pattern.T, cfg.nb, cfg.s
    t_up = int(np.count_nonzero(wl.pattern.indptr[1:] - 1 > wl.pattern.diag_pos))
    ba = bench.bytes_apply_uncoupled_shared(T, 3, nb, s, solver.fac.implicit_l, t_up)
    peak = bench.hbm_peak()[0]
    w = torch.randn(s * T * nb, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    ref = None
    nsts = [int(v) for v in os.environ.get("NSTS", "2,3,4,5,6,8").split(",")]
    groups = [int(v) for v in os.environ.get("TUNE_G", "1,2,3,4,5").split(",")]
    for bkb, g in itertools.product(nsts, groups):
        if bkb > 0:
            os.environ["IRK_APPLY_NST"] = str(bkb)
        else:
            os.environ.pop("IRK_APPLY_NST", None)   # 0 = library default
        os.environ["IRK_APPLY_G"] = str(g)
        solver.fac.apply_device(w, y)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        err = float((y - ref).abs().max() / ref.abs().max())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a.record()
        for _ in range(reps):
            solver.fac.apply_device(w, y)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 1e3 / reps
        print(f"nst={bkb:3d} G={g}  apply={1e3 * t:.4f} ms  frac={ba / t / 1e9 / peak:.3f}  err={err:.1e}",
              flush=True)


if __name__ == "__main__":
    main()
