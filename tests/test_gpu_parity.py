"""GPU parity: the CUDA path (through the C ABI) vs the reference golden
vectors and the CPU oracle.

Bars (BASELINE north star): matvec and preconditioner apply within 1e-12
relative; factor blocks within 1e-12; GMRES iteration counts within +-1 and
the stage solution within 1e-10 relative at equal iteration counts; the
singular-pivot decision (element, stage) identical.
"""

import numpy as np
import pytest

import oracle as O
from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.meshes import line_mesh, partition
from paper_1701_07181_b200.tableau import builtin_tableau, derive
from tests.helpers import load_golden, pattern_of, rel, sha

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def ks():
    return load_golden("kernels_small")


@pytest.fixture(scope="module")
def be():
    from paper_1701_07181_b200 import backend
    return backend


def line(T, periodic=True):
    return pattern_of(line_mesh(T, periodic=periodic).adjacency)


# ---------------------------------------------------------------------------
# backend protocol (kernels/numba_backend.py) vs reference golden vectors
# ---------------------------------------------------------------------------

def test_protocol_bsr_matvec(ks, be):
    ip, ix, _ = line(10)
    assert rel(be.bsr_matvec(ip, ix, ks["line_data"], ks["line_x"]), ks["line_matvec"]) < TOL


@pytest.mark.parametrize("tag,keep_key", [("", None), ("4", "line_keep4")])
def test_protocol_ilu0(ks, be, tag, keep_key):
    ip, ix, dp = line(10)
    keep = np.ones(len(ix), bool) if keep_key is None else ks[keep_key]
    data = ks["line_data"].copy()
    f, d, fail = be.ilu0_factor(ip, ix, dp, data, keep, True)
    np.testing.assert_array_equal(data, ks["line_data"])  # inputs never mutated
    assert fail == -1
    assert rel(f, ks[f"line_f{tag}"]) < TOL
    assert rel(d, ks[f"line_dinv{tag}"]) < TOL
    x = be.ilu0_solve(ip, ix, dp, ks[f"line_f{tag}"], ks[f"line_dinv{tag}"], keep, ks["line_x"])
    assert rel(x, ks[f"line_solve{tag}"]) < TOL


def test_protocol_general_triangle(ks, be):
    ip, ix, dp = pattern_of([[1, 2], [0, 2], [0, 1]])
    keep = np.ones(len(ix), bool)
    f, d, fail = be.ilu0_factor(ip, ix, dp, ks["tri_data"], keep, False)
    assert fail == -1
    assert rel(f, ks["tri_f"]) < TOL
    assert rel(d, ks["tri_dinv"]) < TOL
    assert rel(be.ilu0_solve(ip, ix, dp, f, d, keep, ks["tri_y"]), ks["tri_solve"]) < TOL


@pytest.mark.parametrize("which", ["0", "2"])
def test_protocol_singular_pivot(ks, be, which):
    ip, ix, dp = line(4, periodic=False)
    _, _, fail = be.ilu0_factor(ip, ix, dp, ks[f"sing_data{which}"], np.ones(len(ix), bool), True)
    assert fail == int(ks[f"sing_fail{which}"])


@pytest.mark.parametrize("lit", [False, True])
def test_protocol_coupled(ks, be, lit):
    ip, ix, dp = line(8)
    der = derive(builtin_tableau("RADAU35"))
    s, T = 3, 8
    jac = list(ks["cpl_J"])
    stage_data = np.stack([O.build_stage_matrix(der.a_inv[k, k], ks["cpl_M"], jac[k], dp, 0.08)
                           for k in range(s)])
    coupling = np.zeros((s, s, T, 3, 3))
    for k in range(s):
        for l in range(s):
            if k != l:
                coupling[k, l] = der.a_inv[k, l] * ks["cpl_M"]
    keep = np.ones(len(ix), bool)
    f, g, d, fs, fe = be.coupled_factor(ip, ix, dp, stage_data, coupling, keep, lit)
    tag = "lit" if lit else "std"
    assert (fs, fe) == (-1, -1)
    assert rel(f, ks[f"cpl_{tag}_fstage"]) < TOL
    assert rel(g, ks[f"cpl_{tag}_fcoupling"]) < TOL
    assert rel(d, ks[f"cpl_{tag}_dinv"]) < TOL
    x = be.coupled_solve(ip, ix, dp, ks[f"cpl_{tag}_fstage"], ks[f"cpl_{tag}_fcoupling"],
                         ks[f"cpl_{tag}_dinv"], keep, ks["cpl_w"])
    assert rel(x, ks[f"cpl_{tag}_apply"]) < TOL


# ---------------------------------------------------------------------------
# device-resident operator / preconditioners / GMRES vs reference
# ---------------------------------------------------------------------------

class _Der:
    def __init__(self, a_inv):
        self.a_inv = a_inv


def _device_setup(ks, shared=False):
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix
    from paper_1701_07181_b200.stage_system import StageOperator
    g = line_mesh(8, periodic=True)
    der = derive(builtin_tableau("RADAU35"))
    jacs = [BlockSparseMatrix.from_host(g, j) for j in ks["cpl_J"]]
    if shared:
        jacs = [jacs[0]] * 3
    op = StageOperator(der, 0.08, BlockDiagonalMatrix(ks["cpl_M"]), jacs)
    return der, op


def test_stage_operator_distinct_j(ks):
    _, op = _device_setup(ks)
    assert rel(op.matvec(ks["cpl_w"]), ks["cpl_matvec"]) < TOL


def test_stage_operator_counters(ks):
    from paper_1701_07181_b200.blocks import OpCounter
    _, op = _device_setup(ks)
    c = OpCounter()
    op.matvec(np.zeros(op.total_dim), c)
    assert c.jacobian_multiplies == 3 * 24 and c.mass_multiplies == 9 * 8
    with pytest.raises(ValueError):
        op.matvec(np.zeros(op.total_dim + 1))


def test_device_preconditioners(ks):
    from paper_1701_07181_b200 import precond as P
    from paper_1701_07181_b200.blocks import OpCounter
    der, op = _device_setup(ks)
    w = ks["cpl_w"]
    for lit in (False, True):
        fac = P.stage_coupled_factorize(op, literal_update=lit)
        assert rel(fac.apply(w), ks[f"cpl_{'lit' if lit else 'std'}_apply"]) < TOL
    unc = P.stage_uncoupled_factorize(op, der.shifts)
    assert rel(unc.apply(w), ks["unc_apply"]) < TOL
    assert rel(P.stage_uncoupled_factorize(op, None).apply(w), ks["unc0_apply"]) < TOL
    bj = P.stage_uncoupled_factorize(op, der.shifts, partition_of=np.arange(8))
    assert rel(bj.apply(w), ks["bj_apply"]) < TOL
    cp4 = P.stage_coupled_factorize(op, partition_of=np.repeat(np.arange(4), 2))
    assert rel(cp4.apply(w), ks["cpl4_apply"]) < TOL
    # counters (tests/test_precond.py:238-255): s=3, T=8, r=2
    c = OpCounter()
    P.stage_coupled_factorize(op, c)
    assert c.block_factorizations == 24 and c.block_multiplies == 3 * 2 * 8 + 6 * 8
    c = OpCounter()
    unc.apply(np.zeros(op.total_dim), c)
    assert c.block_multiplies == 3 * 3 * 8


def test_device_gmres_vs_reference(ks):
    from paper_1701_07181_b200 import precond as P
    from paper_1701_07181_b200.krylov import GmresConfig, gmres
    der, op = _device_setup(ks)
    for tag, fac in (("cpl", P.stage_coupled_factorize(op)),
                     ("unc", P.stage_uncoupled_factorize(op, der.shifts))):
        x, st = gmres(op.matvec, fac.apply, ks["gm_rhs"], GmresConfig(rel_tol=1e-8))
        ref_it = int(ks[f"gm_{tag}_iters"])
        assert abs(st.iterations - ref_it) <= 1
        if st.iterations == ref_it:
            assert rel(x, ks[f"gm_{tag}_x"]) < 1e-10
        # python-callback path (lambdas, as irksolve.stepper passes them)
        x2, st2 = gmres(lambda v: op.matvec(v), lambda v: fac.apply(v), ks["gm_rhs"],
                        GmresConfig(rel_tol=1e-8))
        assert st2.iterations == st.iterations
        np.testing.assert_array_equal(x2, x)
        xr, str_ = gmres(op.matvec, fac.apply, ks["gm_rhs"], GmresConfig(rel_tol=1e-10, restart=3))
        rst_it = int(ks[f"gm_{tag}_rst_iters"])
        assert abs(str_.iterations - rst_it) <= 1
        # the solution bar (1e-10) whenever the iteration counts agree
        assert rel(xr, ks[f"gm_{tag}_rst_x"]) < (1e-10 if str_.iterations == rst_it else 1e-8)


def test_singular_pivot_error_device():
    from paper_1701_07181_b200 import SingularPivotError
    from paper_1701_07181_b200 import precond as P
    from paper_1701_07181_b200.blocks import BlockSparseMatrix
    from tests.helpers import random_blocks
    g = line_mesh(4)
    data = random_blocks(g.adjacency, 2, seed=8)
    ip, ix, dp = pattern_of(g.adjacency)
    data[dp[0]] = 0.0
    with pytest.raises(SingularPivotError) as exc:
        P.ilu0_factorize(BlockSparseMatrix.from_host(g, data))
    assert exc.value.element == 0 and exc.value.stage is None


# ---------------------------------------------------------------------------
# workload-level: same cases the oracle is pinned on (tests/test_oracle_golden.py)
# ---------------------------------------------------------------------------

from tests.test_oracle_golden import CASES  # noqa: E402


def _solver_for(name):
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.meshes import partition_bounds
    from paper_1701_07181_b200.solver import StageSolver
    cfg, kind, opts = CASES[name]
    g = load_golden(name)
    wl = W.make_workload(cfg)
    assert sha(wl.J, wl.M, wl.rhs) == str(g["input_sha"])
    dt = float(g["dt"])
    part = None
    if opts.get("partitions"):
        b = partition_bounds(wl.pattern.T, opts["partitions"])
        part = np.repeat(np.arange(opts["partitions"]), np.diff(b))
    p = wl.pattern
    solver = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, dt,
                         kind=kind or cfg.precond, shifts=wl.shifts, partition_of=part,
                         gmres_cfg=GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart,
                                               max_iters=opts.get("max_iters", 500)))
    return cfg, g, wl, solver


@pytest.mark.parametrize("name", list(CASES))
def test_workload_parity(name):
    import torch
    cfg, g, wl, solver = _solver_for(name)
    assert rel(solver.op.matvec(g["w"]), g["matvec"]) < TOL
    solver.factorize()
    assert rel(solver.fac.apply(g["w"]), g["apply"]) < TOL
    x, st = solver.solve(torch.from_numpy(wl.rhs).cuda())
    xr = x.cpu().numpy()
    ref_it = int(g["iterations"])
    assert abs(st.iterations - ref_it) <= 1, (st.iterations, ref_it)
    if st.iterations == ref_it:
        assert rel(xr, g["x"]) < 1e-10
    assert st.converged == bool(g["converged"]) or abs(st.iterations - ref_it) <= 1


def test_solve_is_deterministic():
    import torch
    cfg, g, wl, solver = _solver_for("cfg1_n8")
    solver.factorize()
    rhs = torch.from_numpy(wl.rhs).cuda()
    x1, s1 = solver.solve(rhs)
    x2, s2 = solver.solve(rhs)
    assert torch.equal(x1, x2) and s1.residual_history == s2.residual_history


def test_medium_vs_oracle():
    """Config-1 shape on a 32x32 quad mesh (T=2048): matvec, apply and solve
    vs the oracle on identical inputs."""
    import torch
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    cfg = W.CONFIGS[1].scaled(N=32)
    wl = W.make_workload(cfg, norm_iters=30)
    p = wl.pattern
    solver = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv,
                         wl.dt, kind="uncoupled", shifts=wl.shifts,
                         gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
    prob = O.problem_from_workload(wl)
    w = np.random.default_rng(5).standard_normal(prob.s * prob.T * prob.m)
    assert rel(solver.op.matvec(w), prob.matvec(w)) < TOL
    solver.factorize()
    ofac = O.make_preconditioner(prob, "uncoupled", wl.shifts, workers=3)
    assert rel(solver.fac.apply(w), ofac.apply(w)) < TOL
    x, st = solver.solve(torch.from_numpy(wl.rhs).cuda())
    xo, so = O.gmres(prob.matvec, ofac.apply, wl.rhs, O.GmresConfig(rel_tol=1e-8, restart=40))
    assert abs(st.iterations - so.iterations) <= 1
    if st.iterations == so.iterations:
        assert rel(x.cpu().numpy(), xo) < 1e-10


def test_refactor_in_place_matches_fresh():
    """irk_factor_refactor on new values == a freshly created factor."""
    import torch
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    for kind in ("uncoupled", "coupled"):
        cfg = W.CONFIGS[1].scaled(N=8, scheme="RADAU23" if kind == "coupled" else "RADAU35")
        wl = W.make_workload(cfg)
        p = wl.pattern
        dp = DevicePattern(p.indptr, p.indices, p.diag_pos)
        mk = lambda dt: StageSolver(dp, wl.J, wl.M, wl.a_inv, dt, kind=kind, shifts=wl.shifts,  # noqa: E731
                                    gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
        a = mk(wl.dt)
        a.factorize()
        b = mk(0.5 * wl.dt)
        b.factorize()
        a.op = b.op            # same structure, new values (dt halved)
        a.factorize()          # refactor in place
        w = np.random.default_rng(1).standard_normal(a.n)
        np.testing.assert_array_equal(a.fac.apply(w), b.fac.apply(w))


@pytest.mark.parametrize("ordering", ["color", "natural"])
def test_implicit_l_matches_stored_l(ordering, monkeypatch):
    """Implicit L (forward sweep on the stage-shared J with w_j = Dinv_j z_j,
    rows without upper blocks finished in the forward sweep) == stored L:
    the apply agrees to rounding, the exported L blocks too, and the level
    (colour) and persistent (natural) sweep schedules both work."""
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    cfg = W.CONFIGS[1].scaled(N=8, ordering=ordering)
    wl = W.make_workload(cfg)
    p = wl.pattern
    dp = DevicePattern(p.indptr, p.indices, p.diag_pos)

    def build():
        s = StageSolver(dp, wl.J, wl.M, wl.a_inv, wl.dt, kind="uncoupled", shifts=wl.shifts,
                        gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
        s.factorize()
        return s
    imp = build()
    monkeypatch.setenv("IRK_EXPLICIT_L", "1")
    exp = build()
    assert imp.fac.implicit_l and not exp.fac.implicit_l
    w = np.random.default_rng(3).standard_normal(imp.n)
    assert rel(imp.fac.apply(w), exp.fac.apply(w)) < 1e-13
    fi, di, _ = imp.fac.export()
    fe, de, _ = exp.fac.export()
    np.testing.assert_array_equal(di, de)
    assert rel(fi, fe) < 1e-13
    import torch
    r = torch.from_numpy(wl.rhs).cuda()
    xi, si = imp.solve(r)
    xe, se = exp.solve(r)
    assert abs(si.iterations - se.iterations) <= 1 and rel(xi.cpu().numpy(), xe.cpu().numpy()) < 1e-10


@pytest.mark.parametrize("nb", [5, 24, 33, 40, 50, 70])
def test_block_sizes_vs_oracle(nb):
    """Every inverse specialisation (warp-register GJ for nb<=64, CTA fallback
    above) and odd block sizes, through the protocol shims and the device API."""
    from paper_1701_07181_b200 import backend as be
    mesh = W.CONFIGS[1].scaled(N=3, nb=nb)
    wl = W.make_workload(mesh, norm_iters=20)
    p = wl.pattern
    keep = np.ones(p.nnzb, bool)
    mat = O.build_stage_matrix(1.3, wl.M, wl.J, p.diag_pos, wl.dt)
    f, d, fail = be.ilu0_factor(p.indptr, p.indices, p.diag_pos, mat, keep, True)
    fo, do, failo = O.ilu0_factor(p.indptr, p.indices, p.diag_pos, mat, keep, True)
    assert fail == failo == -1
    assert rel(f, fo) < TOL and rel(d, do) < TOL
    y = np.random.default_rng(nb).standard_normal(p.T * nb)
    assert rel(be.ilu0_solve(p.indptr, p.indices, p.diag_pos, fo, do, keep, y),
               O.ilu0_solve(p.indptr, p.indices, p.diag_pos, fo, do, keep, y)) < TOL
    x = np.random.default_rng(nb + 1).standard_normal(p.T * nb)
    assert rel(be.bsr_matvec(p.indptr, p.indices, wl.J, x), O.bsr_matvec(p.indptr, p.indices, wl.J, x)) < TOL


@pytest.mark.parametrize("nb", [24, 40, 50, 100])
@pytest.mark.parametrize("ordering", ["color", "natural"])
def test_config3_multi_rhs_vs_oracle(nb, ordering):
    """BASELINE config 3 kernels: plain ILU(0) of J itself and the BSR matvec,
    one factor / one matrix applied to s = 1..4 right-hand sides in one sweep
    (factor blocks read once).  Each column must match the oracle's ilu0_solve /
    bsr_matvec (numba_backend.py:21-30, 75-91) and the single-RHS device apply."""
    import torch
    from paper_1701_07181_b200.blocks import BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.precond import ilu0_factorize
    cfg = W.CONFIGS[1].scaled(N=6, nb=nb, ordering=ordering)
    wl = W.make_workload(cfg, jnorm=1.0)
    p = wl.pattern
    keep = np.ones(p.nnzb, bool)
    fo, do, fail = O.ilu0_factor(p.indptr, p.indices, p.diag_pos, wl.J, keep, True)
    assert fail == -1
    J = BlockSparseMatrix(DevicePattern(p.indptr, p.indices, p.diag_pos), DeviceBlocks.from_host(wl.J))
    fac = ilu0_factorize(J)
    n = p.T * nb
    rng = np.random.default_rng(nb)
    for nrhs in (1, 2, 3, 4):
        Y = rng.standard_normal((nrhs, n))
        X = fac.apply_rhs(Y)
        Z = J.matvec_rhs(Y)
        for k in range(nrhs):
            xo = O.ilu0_solve(p.indptr, p.indices, p.diag_pos, fo, do, keep, Y[k])
            assert rel(X[k], xo) < TOL
            assert rel(Z[k], O.bsr_matvec(p.indptr, p.indices, wl.J, Y[k])) < TOL
            x1 = fac.apply(torch.from_numpy(Y[k]).cuda()).cpu().numpy()
            assert rel(X[k], x1) < 1e-14


@pytest.mark.parametrize("m", [24, 40, 56, 64])
@pytest.mark.parametrize("boost", [3.0, 30.0])
def test_inverse_paths_vs_oracle(be, m, boost):
    """Pivot-block inverses: strongly diagonal blocks take the tensor-core
    blocked Gauss-Jordan (no row interchange is ever chosen), weakly diagonal
    ones need partial pivoting and are handed to the pivoted warp kernels;
    both must match the reference algorithm (oracle ilu0_factor, LAPACK-style
    partial pivoting) to 1e-12."""
    from paper_1701_07181_b200.meshes import line_mesh
    from tests.helpers import random_blocks
    g = line_mesh(12, periodic=True)
    ip, ix, dp = pattern_of(g.adjacency)
    data = random_blocks(g.adjacency, m, seed=m, diag_boost=boost)
    keep = np.ones(len(ix), bool)
    f, d, fail = be.ilu0_factor(ip, ix, dp, data, keep, True)
    fo, do, failo = O.ilu0_factor(ip, ix, dp, data, keep, True)
    assert fail == failo
    if failo == -1:
        # two correct partial-pivoting inverses differ by ~cond * eps: the 1e-12 bar
        # applies to well-conditioned pivots (boost 30: cond < 12); the weakly
        # diagonal fixture reaches cond ~6e6 at m = 64
        cond = max(np.linalg.cond(fo[q], 1) for q in dp)
        tol = max(TOL, 4e-16 * cond)
        assert rel(d, do) < tol
        assert rel(f, fo) < tol


@pytest.mark.parametrize("scheme", ["RADAU23", "RADAU35"])
@pytest.mark.parametrize("m", [4, 24])
@pytest.mark.parametrize("ordering", ["color", "natural"])
def test_coupled_pipe_vs_oracle(scheme, m, ordering):
    """Coupled preconditioner on the element-task pipelined sweeps (even nb, s = 2, 3):
    device factor + apply (implicit couplings A^-1_kl M_i, shared J) and the protocol
    coupled_solve on imported factors (stored couplings, stored upper blocks), both
    vs the oracle's coupled_factor / coupled_solve (numba_backend.py:94-151)."""
    import torch
    from paper_1701_07181_b200 import backend as be
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.precond import stage_coupled_factorize
    from paper_1701_07181_b200.stage_system import StageOperator
    cfg = W.CONFIGS[1].scaled(N=5, nb=m, scheme=scheme, ordering=ordering)
    wl = W.make_workload(cfg, norm_iters=20)
    p = wl.pattern
    prob = O.problem_from_workload(wl)
    cf = O.stage_coupled_factorize(prob)
    y = np.random.default_rng(m).standard_normal(prob.s * p.T * m)
    xo = cf.apply(y)
    dp = DevicePattern(p.indptr, p.indices, p.diag_pos)
    J = BlockSparseMatrix(dp, DeviceBlocks.from_host(wl.J))
    op = StageOperator(_Der(wl.a_inv), wl.dt, BlockDiagonalMatrix(wl.M), [J] * prob.s)
    fac = stage_coupled_factorize(op)
    x = fac.apply(torch.from_numpy(y).cuda()).cpu().numpy()
    assert rel(x, xo) < TOL
    keep = np.ones(p.nnzb, bool)
    xp = be.coupled_solve(p.indptr, p.indices, p.diag_pos, cf.fstage, cf.fcoupling, cf.dinv, keep, y)
    assert rel(xp, xo) < TOL


@pytest.mark.parametrize("nb", [8, 5])
def test_stage_matvec_row_range_and_list(nb):
    """irk_stage_op_apply_range (pipelined kernel on a contiguous row range, the
    slab interior of the multi-GPU matvec) + irk_stage_op_apply_rows (row list, the
    boundary) reproduce the full fused matvec bitwise."""
    import torch
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.stage_system import StageOperator
    cfg = W.CONFIGS[1].scaled(N=6, nb=nb)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    J = BlockSparseMatrix(DevicePattern(p.indptr, p.indices, p.diag_pos), DeviceBlocks.from_host(wl.J))
    op = StageOperator(_Der(wl.a_inv), wl.dt, BlockDiagonalMatrix(wl.M), [J] * cfg.s)
    w = torch.from_numpy(np.random.default_rng(nb).standard_normal(op.total_dim)).cuda()
    y_full = torch.empty_like(w)
    op.apply_device(w, y_full)
    r0, r1 = 7, p.T - 11
    y = torch.full_like(w, float("nan"))
    op.apply_device_range(w, y, r0, r1)
    rest = torch.tensor(list(range(0, r0)) + list(range(r1, p.T)), dtype=torch.int32, device="cuda")
    op.apply_device_rows(w, y, rest)
    yf, yy = y_full.view(cfg.s, p.T, nb), y.view(cfg.s, p.T, nb)
    assert torch.equal(yy[:, r0:r1], yf[:, r0:r1])
    assert rel(yy.cpu().numpy(), yf.cpu().numpy()) < 1e-15


@pytest.mark.parametrize("s_scheme,nb", [("RADAU23", 40), ("RADAU35", 40), ("RADAU35", 24), ("RADAU23", 100)])
@pytest.mark.parametrize("ordering,nparts", [("color", 1), ("color", 3), ("natural", 1)])
def test_fused_operator_precond_product(s_scheme, nb, ordering, nparts):
    """irk_op_factor_apply (the Arnoldi product P^-1 (B v) with the stage matvec
    fused into the implicit-L forward sweep, krylov.py:88-89) == the separate
    irk_stage_op_apply + irk_factor_apply, within the 1e-12 apply bar; colour
    schedules take the fused kernel (also with cross-partition lower blocks
    dropped; nb = 100 runs the two-group consumer layout), the deep natural schedule
    falls back to the two calls."""
    import ctypes
    import torch
    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    from paper_1701_07181_b200.meshes import partition_bounds
    cfg = W.CONFIGS[1].scaled(N=8, ordering=ordering, scheme=s_scheme, nb=nb)
    s = cfg.s
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    dp = DevicePattern(p.indptr, p.indices, p.diag_pos)
    part = None if nparts == 1 else np.repeat(np.arange(nparts), np.diff(partition_bounds(p.T, nparts)))
    sol = StageSolver(dp, wl.J, wl.M, wl.a_inv, wl.dt, kind="uncoupled", shifts=wl.shifts,
                      partition_of=part, gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
    sol.factorize()
    assert sol.fac.implicit_l
    v = torch.from_numpy(np.random.default_rng(s).standard_normal(sol.n)).cuda()
    y = torch.empty_like(v)
    x_ref = torch.empty_like(v)
    sol.op.apply_device(v, y)
    sol.fac.apply_device(y, x_ref)
    x = torch.full_like(v, float("nan"))
    fused = ctypes.c_int(-1)
    L.check(L.lib().irk_op_factor_apply(sol.op._op.handle, sol.fac.handle, v.data_ptr(), x.data_ptr(),
                                        ctypes.byref(fused), L.stream_ptr()), "irk_op_factor_apply")
    torch.cuda.synchronize()
    assert fused.value == (1 if ordering == "color" else 0)
    assert rel(x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-12


def test_fused_product_dirk_stage_matrix():
    """The DIRK stage (build_stage_matrix + ilu0_factorize + gmres(mat.matvec, fac.apply),
    stepper.py:268-274) takes the fused Arnoldi product with s = 1: same result as the
    StageMatrix matvec followed by the factor apply (<= 1e-12), and the GMRES solve
    through the fused path matches the oracle's iteration count and solution."""
    import ctypes
    import torch
    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig, gmres
    from paper_1701_07181_b200.precond import build_stage_matrix, ilu0_factorize
    cfg = W.CONFIGS[1].scaled(N=8, ordering="color")
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    J = BlockSparseMatrix(DevicePattern(p.indptr, p.indices, p.diag_pos), DeviceBlocks.from_host(wl.J))
    gamma_dt = 0.4358665215 * wl.dt
    mat = build_stage_matrix(1.0, BlockDiagonalMatrix(wl.M), J, gamma_dt)
    fac = ilu0_factorize(mat)
    v = torch.from_numpy(np.random.default_rng(5).standard_normal(mat.n)).cuda()
    y = torch.empty_like(v)
    x_ref = torch.empty_like(v)
    mat.apply_device(v, y)
    fac.apply_device(y, x_ref)
    x = torch.full_like(v, float("nan"))
    fused = ctypes.c_int(-1)
    L.check(L.lib().irk_op_factor_apply(mat._native_op().handle, fac.handle, v.data_ptr(), x.data_ptr(),
                                        ctypes.byref(fused), L.stream_ptr()), "irk_op_factor_apply")
    torch.cuda.synchronize()
    assert fused.value == 1
    assert rel(x.cpu().numpy(), x_ref.cpu().numpy()) < 1e-12
    # GMRES through the fused path vs the oracle on the same stage matrix
    rhs = np.random.default_rng(6).standard_normal(mat.n)
    xg, st = gmres(mat.matvec, fac.apply, rhs, GmresConfig(rel_tol=1e-8, restart=40))
    A = mat.data
    prob_mv = lambda z: O.bsr_matvec(p.indptr, p.indices, A, z)
    ofac, odinv, ofail = O.ilu0_factor(p.indptr, p.indices, p.diag_pos, A, np.ones(len(p.indices), bool), True)
    assert ofail == -1
    oapply = lambda z: O.ilu0_solve(p.indptr, p.indices, p.diag_pos, ofac, odinv, np.ones(len(p.indices), bool), z)
    xo, so = O.gmres(prob_mv, oapply, rhs, O.GmresConfig(rel_tol=1e-8, restart=40))
    assert abs(st.iterations - so.iterations) <= 1
    if st.iterations == so.iterations:
        assert rel(np.asarray(xg), xo) < 1e-10


def test_gmres_allreduce_callback_uses_fused_cgs():
    """With an allreduce callback (the element-partitioned solve; here one rank, so
    the callback is the identity) irk_gmres runs the same 128-bit fused CGS passes,
    allreducing the two dot vectors on the stream between them: the solve is bitwise
    the callback-free one, and the callback sees 2 (nv + 1)-vectors per iteration
    plus the norms."""
    import torch
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig, gmres_device
    from paper_1701_07181_b200.solver import StageSolver
    cfg = W.CONFIGS[1].scaled(N=8, ordering="color")
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    sol = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                      kind="uncoupled", shifts=wl.shifts, gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
    sol.factorize()
    rhs = torch.from_numpy(wl.rhs).cuda()
    gc = GmresConfig(rel_tol=1e-8, restart=40)
    x0, s0 = gmres_device(sol.op.matvec, sol.fac.apply, rhs, gc)
    sizes = []
    x1, s1 = gmres_device(sol.op.matvec, sol.fac.apply, rhs, gc, allreduce=lambda buf: sizes.append(buf.numel()))
    torch.cuda.synchronize()
    assert s0.iterations == s1.iterations and s0.converged and s1.converged
    assert torch.equal(x0, x1)
    assert s0.final_true_residual == s1.final_true_residual
    for j in range(1, s1.iterations + 1):
        assert sizes.count(j + 1) >= 2, (j, sizes)


@pytest.mark.parametrize("nb,count,first", [(100, 7000, 0), (99, 3 * 3389 + 5, 17)])
def test_chunked_upload_roundtrip(nb, count, first):
    """irk_blocks_upload of more than one 256 MiB staging chunk (two staging buffers,
    copies and layout permutes on two streams) then download: bitwise round trip,
    even and odd (padded) block sizes, at an offset inside the array."""
    from paper_1701_07181_b200.blocks import DeviceBlocks
    rng = np.random.default_rng(nb)
    data = rng.standard_normal((count, nb, nb))
    db = DeviceBlocks(nb, count + first)
    db.upload(data, first=first)
    back = db.download(first=first, count=count)
    assert np.array_equal(back, data)


def test_dirk_stage_vs_reference_golden():
    """DIRK33 implicit stage (stepper.py:268-274: build_stage_matrix(1.0, M, J,
    dt*a_ii) + ilu0_factorize + gmres(mat.matvec, fac.apply)) vs the reference-run
    golden dirk_small.npz: matvec / apply within 1e-12, iterations +-1, x within
    1e-10 at equal counts."""
    from paper_1701_07181_b200 import precond as P
    from paper_1701_07181_b200.blocks import (BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks,
                                              DevicePattern)
    from paper_1701_07181_b200.krylov import GmresConfig, gmres
    g = load_golden("dirk_small")
    cfg = W.CONFIGS[1].scaled(N=6, nb=8)
    wl = W.make_workload(cfg)
    assert sha(wl.J, wl.M, wl.rhs) == str(g["input_sha"]) and wl.dt == float(g["dt"])
    p = wl.pattern
    J = BlockSparseMatrix(DevicePattern(p.indptr, p.indices, p.diag_pos), DeviceBlocks.from_host(wl.J))
    mat = P.build_stage_matrix(1.0, BlockDiagonalMatrix(wl.M), J, wl.dt * float(g["aii"]))
    fac = P.ilu0_factorize(mat)
    assert rel(mat.matvec(g["w"]), g["matvec"]) < TOL
    assert rel(fac.apply(g["w"]), g["apply"]) < TOL
    n = mat.n
    # the reference's closures, exactly as dirk_step builds them
    x, st = gmres(lambda v: mat.matvec(v, None), lambda v: fac.apply(v, None), wl.rhs[:n],
                  GmresConfig(rel_tol=1e-8, restart=40))
    ref_it = int(g["iterations"])
    assert abs(st.iterations - ref_it) <= 1 and st.converged
    if st.iterations == ref_it:
        assert rel(x, g["x"]) < 1e-10


@pytest.mark.parametrize("workers", [2, 3, 4, 8])
def test_protocol_shims_concurrent_threads(be, workers):
    """The reference calls ilu0_factor / ilu0_solve from up to s pool threads at
    once (precond.py:228-237, 270-277); ctypes drops the GIL, so the irk_ref_*
    shims run truly concurrently.  Results must be bitwise identical to the
    serial calls for any thread count (per-call streams and workspaces)."""
    from concurrent.futures import ThreadPoolExecutor
    cfg = W.CONFIGS[1].scaled(N=8)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    keep = np.ones(p.nnzb, bool)
    coefs = np.diag(wl.a_inv) + wl.shifts
    stages = []
    for c in list(coefs) * 2:          # 6 stage matrices (two rounds of the 3 stages)
        d = -wl.dt * wl.J
        d[p.diag_pos] += c * wl.M
        stages.append(d)
    ys = [np.random.default_rng(k).standard_normal(p.T * cfg.nb) for k in range(len(stages))]

    def fac(k):
        return be.ilu0_factor(p.indptr, p.indices, p.diag_pos, stages[k], keep, True)

    serial = [fac(k) for k in range(len(stages))]
    sol_serial = [be.ilu0_solve(p.indptr, p.indices, p.diag_pos, serial[k][0], serial[k][1], keep, ys[k])
                  for k in range(len(stages))]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        conc = list(pool.map(fac, range(len(stages))))
        sol = list(pool.map(lambda k: be.ilu0_solve(p.indptr, p.indices, p.diag_pos, conc[k][0],
                                                    conc[k][1], keep, ys[k]), range(len(stages))))
    for k in range(len(stages)):
        assert conc[k][2] == serial[k][2] == -1
        np.testing.assert_array_equal(conc[k][0], serial[k][0])
        np.testing.assert_array_equal(conc[k][1], serial[k][1])
        np.testing.assert_array_equal(sol[k], sol_serial[k])


@pytest.mark.parametrize("m", [24, 40, 50])
@pytest.mark.parametrize("eps,fails", [(1e-12, False), (3e-14, False), (1e-15, True)])
def test_condition_threshold_two_stage_check(be, m, eps, fails):
    """_inv_with_cond (numba_backend.py:33-40): a pivot block fails iff cond_1 = |D|_1 |D^-1|_1 >
    1e14.  The tensor-core inverse clears most blocks with the bound nb |D|_F |D^-1|_F and computes
    the exact 1-norms only when the bound exceeds 1e14: a block with cond_1 = 1/eps just below the
    threshold (the bound is above it: exact path) must pass, one above must fail at the same
    element as the oracle."""
    from paper_1701_07181_b200.meshes import line_mesh
    from tests.helpers import random_blocks
    g = line_mesh(6, periodic=True)
    ip, ix, dp = pattern_of(g.adjacency)
    data = random_blocks(g.adjacency, m, seed=3, diag_boost=30.0)
    keep = np.ones(len(ix), bool)
    keep[:] = ix == np.repeat(np.arange(6), np.diff(ip))      # block Jacobi: pivots are the diagonal blocks
    bad = 3
    d = np.eye(m)
    d[m - 1, m - 1] = eps
    data[dp[bad]] = d
    f, dinv, fail = be.ilu0_factor(ip, ix, dp, data, keep, True)
    fo, do, failo = O.ilu0_factor(ip, ix, dp, data, keep, True)
    assert fail == failo == (bad if fails else -1)
    if not fails:
        np.testing.assert_allclose(dinv[bad], np.diag(1.0 / np.diag(d)), rtol=1e-12)


@pytest.mark.parametrize("scheme", ["RADAU23", "RADAU35"])
def test_deep_sweeps_self_validating_values(scheme):
    """Deep (natural-numbering) schedules run the self-validating-value sweeps (k_unc_deep_sent:
    outputs pre-filled with a NaN sentinel, consumers poll the values they need).  The apply
    matches the oracle to 1e-12, leaves no sentinel / NaN behind, does not touch its input, is
    bitwise repeatable, and the C ABI rejects x aliasing y (the pre-fill would destroy the input)."""
    import torch
    from paper_1701_07181_b200 import _lib as L
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.solver import StageSolver
    cfg = W.CONFIGS[1].scaled(N=8, ordering="natural", scheme=scheme)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    sol = StageSolver(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M, wl.a_inv, wl.dt,
                      kind="uncoupled", shifts=wl.shifts, gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40))
    sol.factorize()
    assert sol.fac.implicit_l and sol.fac.levels()[0] > 16
    y = np.random.default_rng(7).standard_normal(sol.n)
    yd = torch.from_numpy(y).cuda()
    x1 = torch.empty_like(yd)
    x2 = torch.full_like(yd, 3.0)
    sol.fac.apply_device(yd, x1)
    sol.fac.apply_device(yd, x2)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)
    assert torch.equal(yd, torch.from_numpy(y).cuda())
    assert not np.isnan(x1.cpu().numpy()).any()
    prob = O.problem_from_workload(wl)
    ofac = O.make_preconditioner(prob, "uncoupled", wl.shifts)
    assert rel(x1.cpu().numpy(), ofac.apply(y)) < 1e-12
    rc = L.lib().irk_factor_apply(sol.fac.handle, x2.data_ptr(), x2.data_ptr(), L.stream_ptr())
    assert rc not in (L.IRK_OK, L.IRK_ESINGULAR)        # IRK_EINVAL: "x must not alias y"


@pytest.mark.parametrize("m", [24, 40])
@pytest.mark.parametrize("boost", [30.0, 0.5])
def test_deep_factor_optimistic_fallback(be, m, boost):
    """Deep factor schedules (here a 40-element line: 40 levels) run their levels without the
    per-level pivoted-fallback launch and repeat the factorisation the regular way if any pivot
    block needed row interchanges (boost 0.5: weakly diagonal blocks do).  Both cases must match
    the oracle's partial-pivoting factor (numba_backend.py:33-72)."""
    from paper_1701_07181_b200.meshes import line_mesh
    from tests.helpers import random_blocks
    g = line_mesh(40)
    ip, ix, dp = pattern_of(g.adjacency)
    data = random_blocks(g.adjacency, m, seed=11 + m, diag_boost=boost)
    keep = np.ones(len(ix), bool)
    f, d, fail = be.ilu0_factor(ip, ix, dp, data, keep, True)
    fo, do, failo = O.ilu0_factor(ip, ix, dp, data, keep, True)
    assert fail == failo
    if failo == -1:
        cond = max(np.linalg.cond(fo[q], 1) for q in dp)
        tol = max(TOL, 4e-16 * cond * 40)
        assert rel(d, do) < tol
        assert rel(f, fo) < tol


@pytest.mark.parametrize("scheme", ["RADAU23", "RADAU35"])
@pytest.mark.parametrize("m", [6, 24])
def test_coupled_deep_sweeps_self_validating_values(scheme, m):
    """Stage-coupled ILU(0) on a deep schedule (natural numbering, the reference's default
    preconditioner on its own element order): the (stage, element) sweeps with self-validating
    values (k_cpl_deep_sent) match the oracle's coupled_solve (numba_backend.py:128-151) to 1e-12,
    are bitwise repeatable and leave neither the input touched nor a sentinel behind."""
    import torch
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
    from paper_1701_07181_b200.precond import stage_coupled_factorize
    from paper_1701_07181_b200.stage_system import StageOperator
    cfg = W.CONFIGS[1].scaled(N=10, nb=m, scheme=scheme, ordering="natural")
    wl = W.make_workload(cfg, norm_iters=20)
    p = wl.pattern
    prob = O.problem_from_workload(wl)
    cf = O.stage_coupled_factorize(prob)
    y = np.random.default_rng(m).standard_normal(prob.s * p.T * m)
    xo = cf.apply(y)
    dp = DevicePattern(p.indptr, p.indices, p.diag_pos)
    J = BlockSparseMatrix(dp, DeviceBlocks.from_host(wl.J))
    op = StageOperator(_Der(wl.a_inv), wl.dt, BlockDiagonalMatrix(wl.M), [J] * prob.s)
    fac = stage_coupled_factorize(op)
    assert fac.levels()[0] > 16
    yd = torch.from_numpy(y).cuda()
    x1 = fac.apply(yd)
    x2 = fac.apply(yd)
    assert torch.equal(x1, x2) and torch.equal(yd, torch.from_numpy(y).cuda())
    xh = x1.cpu().numpy()
    assert not np.isnan(xh).any()
    assert rel(xh, xo) < TOL
