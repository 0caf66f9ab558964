"""Pin the CPU oracle against golden vectors produced by the reference itself.

The golden files come from tests/golden/make_golden.py, which ran the
reference ``irksolve`` (numba backend) in the build container.  Tolerances
follow the reference's own backend-parity test (tests/test_backends.py:38-84,
atol 1e-12) expressed relatively; GMRES must reproduce iteration counts
exactly (the oracle is the same MGS algorithm).
"""

import numpy as np
import pytest

import oracle as O
from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.tableau import builtin_tableau, derive
from tests.helpers import load_golden, pattern_of, random_blocks, rel, sha

TOL = 1e-12


@pytest.fixture(scope="module")
def ks():
    return load_golden("kernels_small")


def line_pattern(T, periodic=True):
    from paper_1701_07181_b200.meshes import line_mesh
    g = line_mesh(T, periodic=periodic)
    return g.adjacency, pattern_of(g.adjacency)


def test_random_blocks_restatement(ks):
    adj, _ = line_pattern(10)
    np.testing.assert_array_equal(random_blocks(adj, 3, seed=3), ks["line_data"])


def test_bsr_matvec(ks):
    adj, (ip, ix, dp) = line_pattern(10)
    y = O.bsr_matvec(ip, ix, ks["line_data"], ks["line_x"])
    assert rel(y, ks["line_matvec"]) < TOL


@pytest.mark.parametrize("tag,keep_key", [("", None), ("4", "line_keep4")])
def test_ilu0_factor_solve(ks, tag, keep_key):
    adj, (ip, ix, dp) = line_pattern(10)
    keep = np.ones(len(ix), bool) if keep_key is None else ks[keep_key]
    f, d, fail = O.ilu0_factor(ip, ix, dp, ks["line_data"], keep, True)
    assert fail == -1
    assert rel(f, ks[f"line_f{tag}"]) < TOL
    assert rel(d, ks[f"line_dinv{tag}"]) < TOL
    x = O.ilu0_solve(ip, ix, dp, f, d, keep, ks["line_x"])
    assert rel(x, ks[f"line_solve{tag}"]) < TOL


def test_keep_mask_restatement(ks):
    from paper_1701_07181_b200.meshes import line_mesh, partition
    g = partition(line_mesh(10, periodic=True), 4)
    ip, ix, _ = pattern_of(g.adjacency)
    np.testing.assert_array_equal(O.partition_keep_mask(ip, ix, g.partition_of),
                                  ks["line_keep4"])


def test_general_path_triangle(ks):
    adj = [[1, 2], [0, 2], [0, 1]]
    ip, ix, dp = pattern_of(adj)
    keep = np.ones(len(ix), bool)
    f, d, fail = O.ilu0_factor(ip, ix, dp, ks["tri_data"], keep, False)
    assert fail == int(ks["tri_fail"]) == -1
    assert rel(f, ks["tri_f"]) < TOL
    assert rel(d, ks["tri_dinv"]) < TOL
    assert rel(O.ilu0_solve(ip, ix, dp, f, d, keep, ks["tri_y"]), ks["tri_solve"]) < TOL
    # the simplified sweep differs on this graph (tests/test_precond.py:136-151)
    f2, _, _ = O.ilu0_factor(ip, ix, dp, ks["tri_data"], keep, True)
    assert np.abs(f2 - ks["tri_f"]).max() > 1e-3


@pytest.mark.parametrize("which", ["0", "2"])
def test_singular_pivot_index(ks, which):
    adj = line_pattern(4, periodic=False)[0]
    ip, ix, dp = pattern_of(adj)
    _, _, fail = O.ilu0_factor(ip, ix, dp, ks[f"sing_data{which}"], np.ones(len(ix), bool), True)
    assert fail == int(ks[f"sing_fail{which}"]) == int(which)


def _coupled_problem(ks):
    adj, (ip, ix, dp) = line_pattern(8)
    der = derive(builtin_tableau("RADAU35"))
    jac = [np.ascontiguousarray(j) for j in ks["cpl_J"]]
    return O.Problem(ip, ix, dp, jac, ks["cpl_M"], der.a_inv, 0.08), der


def test_stage_matvec_distinct_j(ks):
    prob, _ = _coupled_problem(ks)
    assert rel(prob.matvec(ks["cpl_w"]), ks["cpl_matvec"]) < TOL


@pytest.mark.parametrize("lit", [False, True])
def test_coupled_factor_apply(ks, lit):
    prob, _ = _coupled_problem(ks)
    fac = O.stage_coupled_factorize(prob, literal_update=lit)
    tag = "lit" if lit else "std"
    assert rel(fac.fstage, ks[f"cpl_{tag}_fstage"]) < TOL
    assert rel(fac.fcoupling, ks[f"cpl_{tag}_fcoupling"]) < TOL
    assert rel(fac.dinv, ks[f"cpl_{tag}_dinv"]) < TOL
    assert rel(fac.apply(ks["cpl_w"]), ks[f"cpl_{tag}_apply"]) < TOL


def test_uncoupled_variants(ks):
    prob, der = _coupled_problem(ks)
    fac = O.stage_uncoupled_factorize(prob, der.shifts)
    assert rel(fac.apply(ks["cpl_w"]), ks["unc_apply"]) < TOL
    assert rel(np.stack([f[1] for f in fac.factors]), ks["unc_dinv"]) < TOL
    assert rel(O.stage_uncoupled_factorize(prob, None).apply(ks["cpl_w"]), ks["unc0_apply"]) < TOL
    bj = O.stage_uncoupled_factorize(prob, der.shifts, partition_of=np.arange(8))
    assert rel(bj.apply(ks["cpl_w"]), ks["bj_apply"]) < TOL
    part = np.repeat(np.arange(4), 2)
    cp4 = O.stage_coupled_factorize(prob, partition_of=part)
    assert rel(cp4.apply(ks["cpl_w"]), ks["cpl4_apply"]) < TOL
    # stage-parallel apply is bitwise identical (criterion 11)
    par = O.stage_uncoupled_factorize(prob, der.shifts, workers=3)
    np.testing.assert_array_equal(par.apply(ks["cpl_w"]), fac.apply(ks["cpl_w"]))


def test_gmres_restatement(ks):
    prob, der = _coupled_problem(ks)
    for tag, fac in (("cpl", O.stage_coupled_factorize(prob)),
                     ("unc", O.stage_uncoupled_factorize(prob, der.shifts))):
        x, st = O.gmres(prob.matvec, fac.apply, ks["gm_rhs"], O.GmresConfig(rel_tol=1e-8))
        assert st.iterations == int(ks[f"gm_{tag}_iters"])
        assert rel(x, ks[f"gm_{tag}_x"]) < 1e-10
        np.testing.assert_allclose(st.residual_history, ks[f"gm_{tag}_hist"], rtol=1e-9)
        x, st = O.gmres(prob.matvec, fac.apply, ks["gm_rhs"],
                        O.GmresConfig(rel_tol=1e-10, restart=3))
        assert st.iterations == int(ks[f"gm_{tag}_rst_iters"])
        assert rel(x, ks[f"gm_{tag}_rst_x"]) < 1e-10


@pytest.mark.parametrize("name", ["RADAU23", "RADAU35", "DIRK33"])
def test_tableau_kats(ks, name):
    d = derive(builtin_tableau(name))
    np.testing.assert_allclose(d.a_inv, ks[f"tab_{name}_a_inv"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(d.shifts, ks[f"tab_{name}_shifts"], rtol=0, atol=1e-13)
    if name == "RADAU23":  # tests/test_tableaux.py:94-97
        np.testing.assert_allclose(d.a_inv, [[1.5, 0.5], [-4.5, 2.5]], atol=1e-13)
        np.testing.assert_allclose(d.shifts, [4.5, 0.5], atol=1e-13)


CASES = {
    "cfg0": (W.CONFIGS[0], None, {}),
    "cfg1_n8": (W.CONFIGS[1].scaled(N=8), None, {}),
    "cfg1_n8_color": (W.CONFIGS[1].scaled(N=8, ordering="color"), None, {}),
    "cfg1_n6_coupled": (W.CONFIGS[1].scaled(N=6, scheme="RADAU23"), "coupled", {}),
    "cfg2_n4": (W.CONFIGS[2].scaled(N=4, nb=10), None, {}),
    "cfg2_n3_full": (W.CONFIGS[2].scaled(N=3, nb=6), None, {}),
    "cfg2_n4_p4": (W.CONFIGS[2].scaled(N=4, nb=10), None, {"partitions": 4}),
    "cfg2_n4_color": (W.CONFIGS[2].scaled(N=4, nb=10, ordering="color"), None, {}),
    "cfg1_n8_var": (W.CONFIGS[1].scaled(N=8, jstd="sqrtnb"), None, {"max_iters": 60}),
}


def oracle_case(name):
    cfg, kind, opts = CASES[name]
    g = load_golden(name)
    wl = W.make_workload(cfg)
    assert sha(wl.J, wl.M, wl.rhs) == str(g["input_sha"]), "generator drifted"
    assert abs(wl.dt - float(g["dt"])) <= 1e-14 * wl.dt
    prob = O.problem_from_workload(wl)
    prob.dt = float(g["dt"])
    part = None
    if opts.get("partitions"):
        from paper_1701_07181_b200.meshes import partition_bounds
        b = partition_bounds(wl.pattern.T, opts["partitions"])
        part = np.repeat(np.arange(opts["partitions"]), np.diff(b))
    fac = O.make_preconditioner(prob, kind or cfg.precond, wl.shifts, part)
    return cfg, g, wl, prob, fac, opts


@pytest.mark.parametrize("name", list(CASES))
def test_workload_case(name):
    cfg, g, wl, prob, fac, opts = oracle_case(name)
    assert rel(prob.matvec(g["w"]), g["matvec"]) < TOL
    assert rel(fac.apply(g["w"]), g["apply"]) < TOL
    x, st = O.gmres(prob.matvec, fac.apply, wl.rhs,
                    O.GmresConfig(rel_tol=cfg.rtol, restart=cfg.restart,
                                  max_iters=opts.get("max_iters", 500)))
    assert st.iterations == int(g["iterations"])
    assert st.converged == bool(g["converged"])
    assert rel(x, g["x"]) < 1e-10
    assert st.operator_applies == int(g["operator_applies"])
    if "fdata" in g:
        assert rel(np.stack([f[0] for f in fac.factors]), g["fdata"]) < TOL
        assert rel(np.stack([f[1] for f in fac.factors]), g["dinv"]) < TOL


# ---------------------------------------------------------------------------
# Newton time steps on M du/dt = J u (stepper.py:127-181, 229-287), reference run
# by tests/golden/make_golden.py::stepper_cases
# ---------------------------------------------------------------------------

STEP_CASES = [("r23c", "RADAU23", "coupled"), ("r35u", "RADAU35", "uncoupled"),
              ("dirk", "DIRK33", None)]


def stepper_inputs(gs, dtn):
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=dtn)
    wl = W.make_workload(cfg)
    tag = f"dt{int(dtn)}"
    assert sha(wl.J, wl.M) == str(gs[f"{tag}_sha"])
    assert wl.dt == float(gs[f"{tag}_dt"])
    return wl, tag


@pytest.fixture(scope="module")
def gs():
    return load_golden("stepper_small")


@pytest.mark.parametrize("dtn", [10.0, 100.0])
@pytest.mark.parametrize("name,scheme,kind", STEP_CASES)
def test_oracle_newton_steps(gs, dtn, name, scheme, kind):
    wl, tag = stepper_inputs(gs, dtn)
    p = wl.pattern
    tab = builtin_tableau(scheme)
    cfg = O.GmresConfig(rel_tol=1e-8, restart=40)
    u = gs[f"{tag}_u0"]
    for step in (1, 2):
        if kind is None:
            u, newton, gm = O.dirk_step_linear(p.indptr, p.indices, p.diag_pos, wl.J, wl.M, tab.A,
                                               tab.b, u, wl.dt, cfg)
        else:
            u, newton, gm = O.irk_step_linear(p.indptr, p.indices, p.diag_pos, wl.J, wl.M, tab.A,
                                              tab.b, u, wl.dt, kind, cfg)
        assert newton == int(gs[f"{tag}_{name}_newton{step}"])
        assert gm == list(gs[f"{tag}_{name}_gmres{step}"])
        assert rel(u, gs[f"{tag}_{name}_u{step}"]) < 1e-10


def test_text_format_matches_reference_dump():
    """dump_matrix / read_matrix_blocks (reference blocks.py:193-216): our dump of the
    reference's matrix is byte-identical to the reference's file, and parsing it
    recovers the blocks exactly (repr is the shortest round-trip form)."""
    import os
    import tempfile
    from types import SimpleNamespace
    from paper_1701_07181_b200.blocks import dump_matrix, read_matrix_blocks
    from paper_1701_07181_b200.meshes import line_mesh
    from tests.helpers import GOLDEN
    g = line_mesh(6, periodic=True)
    ip, ix, _ = pattern_of(g.adjacency)
    data = random_blocks(g.adjacency, 3, seed=21)
    data[0, 0, 0] = 1e-300
    data[1, 1, 1] = -0.1
    data[2, 2, 2] = 12345678901234.5
    ref_path = os.path.join(GOLDEN, "matrix_line6.txt")
    back = read_matrix_blocks(ref_path, ip, ix)
    np.testing.assert_array_equal(back, data)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "m.txt")
        dump_matrix(SimpleNamespace(indptr=ip, indices=ix, data=data), out)
        assert open(out).read() == open(ref_path).read()
    with pytest.raises(ValueError):
        read_matrix_blocks(ref_path, ip[:-1], ix)


# ---------------------------------------------------------------------------
# round 2: generated Radau IIA (s = 4, 5), ESDIRK65, partition map, r2 steps
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def gt():
    return load_golden("tableaux_r2")


@pytest.mark.parametrize("name", ["RADAU23", "RADAU35", "RADAU47", "RADAU59", "DIRK33", "ESDIRK65"])
def test_builtin_tableaux_vs_reference(gt, name):
    """Every builtin scheme (tableaux.py:140-155) incl. the generated RADAU47 /
    RADAU59 and ESDIRK65: A, b, c, order and derive() (A^-1, b^T A^-1, shifts;
    tableaux.py:257-275, ESDIRK on A[1:,1:]) equal the reference's."""
    from paper_1701_07181_b200.tableau import builtin_tableau, derive
    tab = builtin_tableau(name)
    d = derive(tab)
    for k, v in (("A", tab.A), ("b", tab.b), ("c", tab.c)):
        np.testing.assert_allclose(v, gt[f"{name}_{k}"], rtol=0, atol=2e-15)
    for k, v in (("a_inv", d.a_inv), ("bT_a_inv", d.bT_a_inv), ("shifts", d.shifts)):
        ref_v = gt[f"{name}_{k}"]
        assert np.max(np.abs(v - ref_v)) <= 1e-13 * max(1.0, np.max(np.abs(ref_v))), k
    assert tab.order == int(gt[f"{name}_order"])
    assert tab.kind == {"fully_implicit": "irk", "dirk": "dirk", "esdirk": "esdirk"}[str(gt[f"{name}_kind"])]


@pytest.mark.parametrize("s", range(1, 10))
def test_generate_radau_iia_vs_reference(gt, s):
    """generate_radau_iia(s) (tableaux.py:246-254) for s = 1..9."""
    from paper_1701_07181_b200.tableau import generate_radau_iia
    tab = generate_radau_iia(s)
    np.testing.assert_allclose(tab.A, gt[f"gen{s}_A"], rtol=0, atol=5e-15)
    np.testing.assert_allclose(tab.c, gt[f"gen{s}_c"], rtol=0, atol=5e-15)
    assert tab.c[-1] == 1.0 and np.allclose(tab.A.sum(axis=1), tab.c, atol=1e-14)
    with pytest.raises(ValueError):
        generate_radau_iia(10)


@pytest.mark.parametrize("T,P", [(50, 4), (7, 3), (10, 10), (3072, 8), (101, 8), (12, 5)])
def test_partition_map_vs_reference(gt, T, P):
    """meshes.partition / partition_bounds and the stepper's LinearProblem.partition_of
    reproduce the reference's partition (meshing.py:81-90) when T % P != 0 (T=50,
    P=4 -> 13/13/12/12)."""
    from paper_1701_07181_b200.meshes import line_mesh, partition, partition_bounds
    from paper_1701_07181_b200.stepper import LinearProblem
    want = gt[f"part_{T}_{P}"]
    np.testing.assert_array_equal(partition(line_mesh(T, periodic=True), P).partition_of, want)
    b = partition_bounds(T, P)
    np.testing.assert_array_equal(np.repeat(np.arange(P), np.diff(b)), want)
    fake = LinearProblem.__new__(LinearProblem)
    fake.pattern = type("P", (), {"T": T})()
    np.testing.assert_array_equal(fake.partition_of(P), want)


R2_STEPS = [("r47u", "RADAU47", "uncoupled"), ("r47c", "RADAU47", "coupled"),
            ("r59u", "RADAU59", "uncoupled"), ("r59c", "RADAU59", "coupled"),
            ("esdirk", "ESDIRK65", None)]


@pytest.mark.parametrize("name,scheme,kind", R2_STEPS)
def test_oracle_newton_steps_r2(name, scheme, kind):
    """The oracle's restated steppers with s = 4 / 5 and the ESDIRK explicit stage
    reproduce the reference's steps (stepper_r2.npz)."""
    g2 = load_golden("stepper_r2")
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=10.0)
    wl = W.make_workload(cfg)
    assert sha(wl.J, wl.M) == str(g2["sha"]) and wl.dt == float(g2["dt"])
    p = wl.pattern
    tab = builtin_tableau(scheme)
    cfgm = O.GmresConfig(rel_tol=1e-8, restart=40)
    u = g2["u0"]
    for step in (1, 2):
        if kind is None:
            u, newton, gm = O.dirk_step_linear(p.indptr, p.indices, p.diag_pos, wl.J, wl.M, tab.A,
                                               tab.b, u, wl.dt, cfgm)
        else:
            u, newton, gm = O.irk_step_linear(p.indptr, p.indices, p.diag_pos, wl.J, wl.M, tab.A,
                                              tab.b, u, wl.dt, kind, cfgm)
        assert newton == int(g2[f"{name}_newton{step}"])
        want = list(g2[f"{name}_gmres{step}"])
        assert len(gm) == len(want) and all(abs(a - b) <= 1 for a, b in zip(gm, want)), (gm, want)
        assert rel(u, g2[f"{name}_u{step}"]) < 1e-10


@pytest.mark.parametrize("ordering,P", [("natural", 1), ("natural", 2), ("natural", 4), ("natural", 8),
                                        ("color", 8)])
def test_oracle_config2_nb50_vs_reference(ordering, P):
    """The oracle pinned at the config-2 block size (nb=50, s=3, 8^3 Kuhn cubes)
    against the reference's own runs at P = 1, 2, 4, 8 (cfg2_n8_nb50_*.npz):
    matvec / apply samples within 1e-12, identical GMRES iteration counts, x
    within 1e-10."""
    g = load_golden(f"cfg2_n8_nb50_{ordering}_p{P}")
    c = W.CONFIGS[2].scaled(N=8, ordering=ordering, extra={"parts": P} if ordering == "color" else {})
    wl = W.make_workload(c, jnorm=float(g["jnorm"]))
    assert sha(wl.J, wl.M, wl.rhs) == str(g["input_sha"]) and wl.dt == float(g["dt"])
    part = None if P == 1 else np.concatenate(
        [np.full(len(ch), k) for k, ch in enumerate(np.array_split(np.arange(wl.pattern.T), P))])
    prob = O.problem_from_workload(wl)
    fac = O.make_preconditioner(prob, "uncoupled", wl.shifts, partition_of=part, workers=3)
    w = np.random.default_rng(99).standard_normal(prob.s * prob.T * prob.m)
    idx = g["idx"]
    assert rel(prob.matvec(w)[idx], g["matvec"]) < 1e-12
    assert rel(fac.apply(w)[idx], g["apply"]) < 1e-12
    x, st = O.gmres(prob.matvec, fac.apply, wl.rhs, O.GmresConfig(rel_tol=1e-8, restart=40))
    assert st.iterations == int(g["iterations"]) and st.converged
    assert rel(x[idx], g["x"]) < 1e-10
