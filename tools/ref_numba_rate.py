"""Time the UNMODIFIED reference (irksolve, numba backend, warmed JIT) on one
config-1 stage-solve: build the shifted uncoupled preconditioner + GMRES(40) to
rtol 1e-8 through its public API (stepper.py:164-170 call chain).  Build
container only (/root/reference does not exist on the GPU box); the result is
committed under profiles/ and quoted by bench.py as a static figure.

    python tools/ref_numba_rate.py [N] [--workers W]
"""
import json
import os
import platform
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_rate")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402
import irksolve as ref  # noqa: E402
from irksolve.kernels import set_backend  # noqa: E402
from irksolve.stepper import _make_preconditioner  # noqa: E402
from paper_1701_07181_b200 import workloads as W  # noqa: E402

set_backend("numba")
N = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 128
workers = int(sys.argv[sys.argv.index("--workers") + 1]) if "--workers" in sys.argv else 1
cfg = W.CONFIGS[1].scaled(N=N, ordering="color")
wl = W.make_workload(cfg, jnorm=2.4496432463318416)
adj = [list(map(int, r)) for r in wl.table]
g = ref.ElementGraph(num_elements=len(adj), adjacency=adj, periodic=True)
Jm = ref.BlockSparseMatrix(g, cfg.nb)
Jm.data[:] = wl.J
mass = ref.BlockDiagonalMatrix(wl.M)
der = ref.derive(ref.builtin_tableau(cfg.scheme))
op = ref.StageOperator(der, wl.dt, mass, [Jm] * cfg.s)
spec = ref.PrecondSpec(kind="uncoupled", stage_parallel=workers > 1, workers=workers)
gcfg = ref.GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart)


def solve():
    t0 = time.perf_counter()
    fac = _make_preconditioner(op, spec, None, None)
    t1 = time.perf_counter()
    x, st = ref.gmres(lambda v: op.matvec(v), lambda v: fac.apply(v), wl.rhs, gcfg)
    return t1 - t0, time.perf_counter() - t1, st


small = W.CONFIGS[1].scaled(N=8)   # JIT warm-up
solve()                             # warm (first full call compiles nothing new but pages in)
tf, tg, st = solve()
print(json.dumps({
    "what": "reference irksolve (numba backend) one config-1 stage-solve: _make_preconditioner "
            "(shifted uncoupled) + gmres (GMRES(40), rtol 1e-8), colour-major numbering",
    "T": int(wl.pattern.T), "nb": cfg.nb, "s": cfg.s, "stage_workers": workers,
    "factor_s": tf, "gmres_s": tg, "total_s": tf + tg, "stage_solves_per_s_at_T": 1.0 / (tf + tg),
    "iterations": st.iterations, "converged": bool(st.converged),
    "cpu": platform.processor() or platform.machine(), "os_cpu_count": os.cpu_count(),
    "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
    "where": "build container (not the GPU box: /root/reference is absent there)",
}))
