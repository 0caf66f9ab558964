"""Small end-to-end workload for compute-sanitizer (racecheck / synccheck /
memcheck / initcheck): every kernel family of the hot path at sizes the
sanitizers finish in minutes.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

* config-0 shape (RADAU23, coupled ILU(0), natural numbering: deep DAG ->
  persistent stage-skewed flag-synchronised sweeps, ld.acquire / st.release);
* config-1 shape, natural numbering (uncoupled persistent sweeps, the
  ticket-ordered producer / flag protocol);
* config-1 shape, colour numbering (level launches, the fused Arnoldi product
  with its mbarrier / bulk-copy rings, tensor-core inverse + Schur);
* config-2 shape (nb=50: padded DMMA tiles, pivoted inverse fallback sizes).
Each runs factor + GMRES and checks convergence.
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_07181_b200 import workloads as W  # noqa: E402
from paper_1701_07181_b200.blocks import DevicePattern  # noqa: E402
from paper_1701_07181_b200.krylov import GmresConfig  # noqa: E402
from paper_1701_07181_b200.solver import StageSolver  # noqa: E402

CASES = [
    ("cfg0 natural coupled", W.CONFIGS[0].scaled(N=8)),
    ("cfg1 natural uncoupled", W.CONFIGS[1].scaled(N=6, ordering="natural")),
    ("cfg1 colour uncoupled", W.CONFIGS[1].scaled(N=6, ordering="color")),
    ("cfg2 colour nb50", W.CONFIGS[2].scaled(N=3, ordering="color")),
]

for name, cfg in CASES:
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    s = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                    kind=cfg.precond, shifts=wl.shifts, gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
    s.factorize()
    x, st = s.solve(torch.from_numpy(wl.rhs).cuda())
    torch.cuda.synchronize()
    levels = s.fac.levels() if s.fac is not None else None
    print(f"{name}: T={p.T} nb={cfg.nb} levels={levels} iterations={st.iterations} converged={st.converged}")
    assert st.converged and np.isfinite(x.cpu().numpy()).all()
print("sanitize workload done")
