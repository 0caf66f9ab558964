"""Factor (and with TIME_SOLVE=1 also solve) a config, warm then timed; run under
`ncu --metrics gpu__time_duration.sum` to get per-kernel durations.

usage: python tools/time_factor.py [config] [ordering]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_07181_b200 import workloads as W  # noqa: E402
from paper_1701_07181_b200.blocks import DevicePattern  # noqa: E402
from paper_1701_07181_b200.krylov import GmresConfig  # noqa: E402
from paper_1701_07181_b200.solver import StageSolver  # noqa: E402
from paper_1701_07181_b200.tableau import builtin_tableau, derive  # noqa: E402


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    order = sys.argv[2] if len(sys.argv) > 2 else "color"
    cfg = W.CONFIGS[ci].scaled(ordering=order)
    if len(sys.argv) > 3:
        cfg = cfg.scaled(N=int(sys.argv[3]))
    wl = W.make_workload(cfg, jnorm=1.0)
    der = derive(builtin_tableau(cfg.scheme))
    dt = cfg.dt_norm / 2.4496432463318416
    dpat = DevicePattern(wl.pattern.indptr, wl.pattern.indices, wl.pattern.diag_pos)
    solver = StageSolver(dpat, wl.J, wl.M, der.a_inv, dt, kind=cfg.precond, shifts=der.shifts,
                         gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    solver.factorize()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        solver.factorize()
    b.record()
    torch.cuda.synchronize()
    print(f"factorize {a.elapsed_time(b) / 3:.3f} ms", flush=True)
    if os.environ.get("TIME_SOLVE"):
        rhs = torch.from_numpy(wl.rhs).cuda()
        x = torch.empty_like(rhs)
        _, st = solver.solve(rhs, x=x)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            _, st = solver.solve(rhs, x=x)
        b.record()
        torch.cuda.synchronize()
        print(f"solve {a.elapsed_time(b) / 3:.3f} ms iters {st.iterations} reorth {st.reorth_passes} "
              f"applies {st.operator_applies}", flush=True)


if __name__ == "__main__":
    main()
