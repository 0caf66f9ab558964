#!/bin/bash
# persistent (deep-DAG) sweep knobs at config 1, natural numbering: apply time per setting
python -c "import __graft_entry__ as g; g.build()" || exit 1
for knobs in "" "IRK_APPLY_CTAS=2" "IRK_APPLY_CTAS=3" "IRK_APPLY_CTAS=6" "IRK_APPLY_CTAS=8" "IRK_APPLY_NST=2" "IRK_APPLY_NST=3" "IRK_APPLY_NST=6" "IRK_APPLY_G=1" "IRK_APPLY_G=2" "IRK_APPLY_G=2 IRK_APPLY_CTAS=6" "IRK_APPLY_G=1 IRK_APPLY_CTAS=8" "IRK_PDL=0"; do
  echo -n "[$knobs] "
  env $knobs ORDERING=natural NSTS=0 TUNE_G=0 python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.blocks import DevicePattern
from paper_1701_07181_b200.krylov import GmresConfig
from paper_1701_07181_b200.solver import StageSolver
from paper_1701_07181_b200.tableau import builtin_tableau, derive
cfg = W.CONFIGS[1].scaled(ordering="natural")
wl = W.make_workload(cfg, jnorm=1.0)
der = derive(builtin_tableau(cfg.scheme))
dt = cfg.dt_norm / 2.4496432463318416
dpat = DevicePattern(wl.pattern.indptr, wl.pattern.indices, wl.pattern.diag_pos)
s = StageSolver(dpat, wl.J, wl.M, der.a_inv, dt, kind=cfg.precond, shifts=der.shifts, gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart))
s.factorize()
w = torch.randn(s.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(w)
s.fac.apply_device(w, y); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): s.fac.apply_device(w, y)
b.record(); torch.cuda.synchronize()
print(f"apply {a.elapsed_time(b)/10:.3f} ms")
PY
done
