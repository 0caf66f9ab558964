"""Stress run of the deep (natural-numbering) sweeps with self-validating values: thousands of
back-to-back applies, output buffer dirtied before each, results compared bitwise with the first
apply -- a missed dependency, a stale value or a hang would show here.

    timeout 1200 python tools/stress_deep.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_07181_b200 import workloads as W  # noqa: E402
from paper_1701_07181_b200.blocks import DevicePattern  # noqa: E402
from paper_1701_07181_b200.krylov import GmresConfig  # noqa: E402
from paper_1701_07181_b200.solver import StageSolver  # noqa: E402

CASES = (("RADAU35", "uncoupled", 128, 1500), ("RADAU23", "coupled", 128, 800),
         ("RADAU35", "coupled", 20, 3000), ("RADAU35", "uncoupled", 20, 3000))

for scheme, kind, N, reps in CASES:
    cfg = W.CONFIGS[1].scaled(ordering="natural", scheme=scheme, precond=kind, N=N)
    wl = W.make_workload(cfg, jnorm=2.4496432463318416)
    p = wl.pattern
    s = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt, kind=kind,
                    shifts=wl.shifts, gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    s.factorize()
    w = torch.randn(s.n, dtype=torch.float64, device="cuda")
    y0, y = torch.empty_like(w), torch.empty_like(w)
    s.fac.apply_device(w, y0)
    torch.cuda.synchronize()
    t0, bad = time.time(), 0
    for r in range(reps):
        y.fill_(float(r))
        s.fac.apply_device(w, y)
        if r % 50 == 0:
            torch.cuda.synchronize()
            bad += 0 if torch.equal(y, y0) else 1
    torch.cuda.synchronize()
    bad += 0 if torch.equal(y, y0) else 1
    print(f"{scheme} {kind} N={N}: {reps} applies in {time.time() - t0:.2f} s, mismatches {bad}, "
          f"levels {s.fac.levels()}", flush=True)
    assert bad == 0
    del s
print("stress done")
