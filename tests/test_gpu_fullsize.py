"""GPU parity at the benchmarked sizes (VERDICT r1 "next round" item 1).

* Config 1 at full size (T=32,768 triangles, nb=40, Radau IIA s=3, shifted
  uncoupled block ILU(0), GMRES(40), rtol 1e-8), colour-major and natural
  numbering: the stage matvec, the preconditioner apply and the fused Arnoldi
  product P^-1 (B v) (the bench's roofline kernel) vs the C oracle within 1e-12
  relative; GMRES iterations within +-1 and x within 1e-10 at equal counts;
  convergence and the true residual asserted.
* Config-2 shape at its real block size (nb=50, s=3, 3D Kuhn tets) on 8^3 cubes
  (T=3,072) against REFERENCE-run goldens at P = 1, 2, 4, 8 (natural numbering,
  partition(graph, P), meshing.py:81-90 / precond.py:26-45) and the slab-colour
  numbering at P=8 (samples of every 61st entry + full norms, made by
  tests/golden/make_golden.py --r2), plus full vectors against the oracle; and
  16^3 cubes (T=24,576) against the oracle at P = 1, 2, 4, 8.

The oracle is the checker only (oracle/, C restatement of numba_backend.py +
numpy GMRES restating krylov.py); every product call goes through
libirkb200.so.
"""

import ctypes

import numpy as np
import pytest

import oracle as O
from paper_1701_07181_b200 import workloads as W
from tests.helpers import load_golden, rel, sha

pytestmark = pytest.mark.gpu
TOL = 1e-12
JNORM_CFG1 = 2.4496432463318416     # ||J||_2 of the config-1 generator (bench.py power iteration)


def _solver(wl, kind, part=None, restart=40, rtol=1e-8):
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    p = wl.pattern
    return StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                       kind=kind, shifts=wl.shifts, partition_of=part,
                       gmres_cfg=GmresConfig(rel_tol=rtol, restart=restart))


def _product(solver, v):
    """irk_op_factor_apply: the Arnoldi product as irk_gmres runs it."""
    import torch
    from paper_1701_07181_b200 import _lib as L
    vd = torch.from_numpy(v).cuda()
    out = torch.empty_like(vd)
    fused = ctypes.c_int(0)
    L.check(L.lib().irk_op_factor_apply(solver.op._op.handle, solver.fac.handle, vd.data_ptr(),
                                        out.data_ptr(), ctypes.byref(fused), L.stream_ptr()),
            "irk_op_factor_apply")
    return out.cpu().numpy(), fused.value


def _part_map(T, P):
    if P == 1:
        return None
    return np.concatenate([np.full(len(c), k) for k, c in enumerate(np.array_split(np.arange(T), P))])


def _check_solve(solver, wl, prob, ofac, restart=40):
    import torch
    x, st = solver.solve(torch.from_numpy(wl.rhs).cuda())
    xo, so = O.gmres(prob.matvec, ofac.apply, wl.rhs, O.GmresConfig(rel_tol=1e-8, restart=restart))
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 1, (st.iterations, so.iterations)
    xh = x.cpu().numpy()
    if st.iterations == so.iterations:
        assert rel(xh, xo) < 1e-10
    # the true residual the bench reports, recomputed on the oracle side
    tr = np.linalg.norm(wl.rhs - prob.matvec(xh)) / np.linalg.norm(wl.rhs)
    assert abs(st.final_true_residual / np.linalg.norm(wl.rhs) - tr) <= 1e-6 * max(tr, 1e-300) + 1e-15
    pb = np.linalg.norm(ofac.apply(wl.rhs))
    assert np.linalg.norm(ofac.apply(wl.rhs - prob.matvec(xh))) <= 2e-8 * pb
    return st, so


@pytest.mark.parametrize("ordering", ["color", "natural"])
def test_config1_full_size_vs_oracle(ordering):
    cfg = W.CONFIGS[1].scaled(ordering=ordering)
    wl = W.make_workload(cfg, jnorm=JNORM_CFG1)
    assert wl.pattern.T == 32768 and cfg.nb == 40 and cfg.s == 3
    solver = _solver(wl, "uncoupled")
    prob = O.problem_from_workload(wl)
    rng = np.random.default_rng(2024)
    w = rng.standard_normal(solver.n)
    mv = prob.matvec(w)
    assert rel(solver.op.matvec(w), mv) < TOL
    solver.factorize()
    ofac = O.make_preconditioner(prob, "uncoupled", wl.shifts, workers=3)
    assert rel(solver.fac.apply(w), ofac.apply(w)) < TOL
    prod, fused = _product(solver, w)
    assert rel(prod, ofac.apply(mv)) < TOL
    if ordering == "color":
        assert fused == 1 and solver.fac.levels() == (2, 2)   # the benchmarked path
    _check_solve(solver, wl, prob, ofac)


CFG2_GOLDEN = [("natural", 1), ("natural", 2), ("natural", 4), ("natural", 8), ("color", 8)]


def _cfg2(N, ordering, P, jnorm=None):
    c = W.CONFIGS[2].scaled(N=N, ordering=ordering, extra={"parts": P} if ordering == "color" else {})
    return c, W.make_workload(c, jnorm=jnorm, norm_iters=30)


@pytest.mark.parametrize("ordering,P", CFG2_GOLDEN)
def test_config2_8cubed_nb50_vs_reference(ordering, P):
    """8^3 cubes, nb=50, s=3 vs the reference's own run at P partitions."""
    g = load_golden(f"cfg2_n8_nb50_{ordering}_p{P}")
    c, wl = _cfg2(8, ordering, P, jnorm=float(g["jnorm"]))
    assert sha(wl.J, wl.M, wl.rhs) == str(g["input_sha"]) and wl.dt == float(g["dt"])
    part = _part_map(wl.pattern.T, P)
    solver = _solver(wl, "uncoupled", part)
    idx = g["idx"]
    w = np.random.default_rng(99).standard_normal(solver.n)
    assert sha(w) == str(g["w_sha"])
    mv = solver.op.matvec(w)
    assert rel(mv[idx], g["matvec"]) < TOL and abs(np.linalg.norm(mv) / g["matvec_norm"] - 1) < TOL
    solver.factorize()
    ap = solver.fac.apply(w)
    assert rel(ap[idx], g["apply"]) < TOL and abs(np.linalg.norm(ap) / g["apply_norm"] - 1) < TOL
    import torch
    x, st = solver.solve(torch.from_numpy(wl.rhs).cuda())
    ref_it = int(g["iterations"])
    assert st.converged and abs(st.iterations - ref_it) <= 1, (st.iterations, ref_it)
    xh = x.cpu().numpy()
    if st.iterations == ref_it:
        assert rel(xh[idx], g["x"]) < 1e-10 and abs(np.linalg.norm(xh) / g["x_norm"] - 1) < 1e-10
    # full vectors against the oracle (pinned to the same reference run in the CPU suite)
    prob = O.problem_from_workload(wl)
    ofac = O.make_preconditioner(prob, "uncoupled", wl.shifts, partition_of=part, workers=3)
    assert rel(ap, ofac.apply(w)) < TOL
    prod, _ = _product(solver, w)
    assert rel(prod, ofac.apply(prob.matvec(w))) < TOL


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_config2_16cubed_nb50_vs_oracle(P):
    """16^3 cubes (T=24,576), nb=50, s=3, partitioned ILU(0) at P = 1, 2, 4, 8:
    operator, apply and fused product vs the oracle; the full solve at P = 1, 8."""
    c, wl = _cfg2(16, "natural", P, jnorm=2.5)
    assert wl.pattern.T == 24576
    part = _part_map(wl.pattern.T, P)
    solver = _solver(wl, "uncoupled", part)
    prob = O.problem_from_workload(wl)
    w = np.random.default_rng(7).standard_normal(solver.n)
    mv = prob.matvec(w)
    assert rel(solver.op.matvec(w), mv) < TOL
    solver.factorize()
    ofac = O.make_preconditioner(prob, "uncoupled", wl.shifts, partition_of=part, workers=3)
    assert rel(solver.fac.apply(w), ofac.apply(w)) < TOL
    prod, _ = _product(solver, w)
    assert rel(prod, ofac.apply(mv)) < TOL
    if P in (1, 8):
        _check_solve(solver, wl, prob, ofac)
