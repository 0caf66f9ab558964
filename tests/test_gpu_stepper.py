"""GPU parity of the device-resident Newton steps against
the reference's own steppers (golden stepper_small.npz, made by running
irk_step_transformed / dirk_step on M du/dt = J u) and the CPU oracle.

Bars: Newton iteration counts equal; GMRES iterations per Newton iteration
within +-1; u_next within 1e-9 relative (Newton stops at |r|_inf <= 1e-8, so
two converged runs agree to about that level); OpCounter totals equal to the
reference's (stepper.py counts, precond.py/stage_system.py increments).
"""

import numpy as np
import pytest

from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.tableau import builtin_tableau
from tests.helpers import load_golden, rel, sha

pytestmark = pytest.mark.gpu

CASES = [("r23c", "RADAU23", "coupled"), ("r35u", "RADAU35", "uncoupled"), ("dirk", "DIRK33", None)]


@pytest.fixture(scope="module")
def gs():
    return load_golden("stepper_small")


@pytest.mark.parametrize("dtn", [10.0, 100.0])
@pytest.mark.parametrize("name,scheme,kind", CASES)
def test_device_steps_vs_reference(gs, dtn, name, scheme, kind):
    from paper_1701_07181_b200.blocks import DevicePattern, OpCounter
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.stepper import (LinearProblem, NewtonConfig, PrecondSpec, StepCache,
                                               dirk_step, irk_step_transformed)
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=dtn)
    wl = W.make_workload(cfg)
    tag = f"dt{int(dtn)}"
    assert sha(wl.J, wl.M) == str(gs[f"{tag}_sha"])
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    tab = builtin_tableau(scheme)
    gcfg = GmresConfig(rel_tol=1e-8, restart=40)
    ctr = OpCounter()
    cache = StepCache()
    u = gs[f"{tag}_u0"]
    for step in (1, 2):
        if kind is None:
            res = dirk_step(prob, tab, u, 0.0, wl.dt, NewtonConfig(), gcfg, ctr, cache=cache)
        else:
            res = irk_step_transformed(prob, tab, u, 0.0, wl.dt, PrecondSpec(kind=kind),
                                       NewtonConfig(), gcfg, ctr, cache=cache)
        u = res.u_next
        assert res.newton_iterations == int(gs[f"{tag}_{name}_newton{step}"])
        gref = list(gs[f"{tag}_{name}_gmres{step}"])
        got = [st.iterations for st in res.gmres_stats]
        assert len(got) == len(gref) and all(abs(a - b) <= 1 for a, b in zip(got, gref)), (got, gref)
        assert rel(u.cpu().numpy(), gs[f"{tag}_{name}_u{step}"]) < 1e-9
    want = gs[f"{tag}_{name}_counter"]
    have = np.array([ctr.block_multiplies, ctr.block_solves, ctr.block_factorizations,
                     ctr.mass_multiplies, ctr.jacobian_multiplies])
    if all(a == b for a, b in zip(got, gref)):
        np.testing.assert_array_equal(have, want)


def test_integrate_reuses_factor_and_matches_steps():
    """integrate() (stepper.py:328-375) == repeated steps with a fresh cache
    (frozen-J reuse changes no result)."""
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.stepper import (LinearProblem, PrecondSpec, integrate,
                                               irk_step_transformed)
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=100.0)
    wl = W.make_workload(cfg)
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    u0 = np.random.default_rng(11).standard_normal(prob.n)
    gcfg = GmresConfig(rel_tol=1e-8, restart=40)
    res = integrate(prob, "RADAU35", 0.0, 3 * wl.dt, wl.dt, PrecondSpec(kind="uncoupled"),
                    gmres_cfg=gcfg, u0=u0)
    u = u0
    for k in range(3):
        u = irk_step_transformed(prob, builtin_tableau("RADAU35"), u, k * wl.dt, wl.dt,
                                 PrecondSpec(kind="uncoupled"), gmres_cfg=gcfg).u_next
    assert len(res.step_results) == 3
    np.testing.assert_array_equal(res.u_final.cpu().numpy(), u.cpu().numpy())


def test_cost_report_counts_match_reference_predictions():
    """studies.cost_report (reference studies.py:261-353) on the GPU objects: every
    measured block-operation count equals the reference's exact prediction and, on
    this uniform-degree mesh, its closed-form (s, r, T) model where one exists."""
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.stepper import LinearProblem
    from paper_1701_07181_b200.studies import cost_report
    cfg = W.CONFIGS[1].scaled(N=4, nb=6)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    for scheme in ("RADAU23", "RADAU35"):
        rows = cost_report(prob, scheme, dt=0.1)
        for row in rows:
            if row.measured is not None:
                assert row.match, row
        # model matches where the reference's model is exact for its implemented algorithm
        by = {row.operation: row for row in rows}
        for name in ("transformed-matvec jacobian products", "coupled-factorize block LU",
                     "uncoupled-apply block products", "dirk-apply block products"):
            assert by[name].model_match, by[name]


def test_partition_study_iterations_grow_with_p():
    """run_partition_study (reference studies.py:204-242): partitioned block ILU(0)
    drops cross-partition blocks, so GMRES iterations do not decrease with P."""
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.stepper import LinearProblem
    from paper_1701_07181_b200.studies import run_partition_study
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=100.0)
    wl = W.make_workload(cfg)
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    u0 = np.random.default_rng(11).standard_normal(prob.n)
    recs = run_partition_study(prob, "RADAU35", wl.dt, [1, 2, 4, 8], num_steps=2,
                               gmres_cfg=GmresConfig(rel_tol=1e-8, restart=40), u0=u0)
    its = [r.gmres_iters_avg for r in recs]
    assert all(r.converged for r in recs)
    assert its[-1] >= its[0], its


def test_stepper_argument_errors_and_newton_failure():
    """stepper.py:140-143, 241-244 (dt > 0, scheme kind) and the NewtonError of the
    shared skeleton (stepper.py:119-120) with an unreachable tolerance."""
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.stepper import (LinearProblem, NewtonConfig, NewtonError, PrecondSpec,
                                               dirk_step, irk_step_transformed)
    cfg = W.CONFIGS[1].scaled(N=4, nb=6)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    u0 = np.random.default_rng(1).standard_normal(prob.n)
    with pytest.raises(ValueError):
        irk_step_transformed(prob, "RADAU23", u0, 0.0, 0.0)
    with pytest.raises(ValueError):
        irk_step_transformed(prob, "DIRK33", u0, 0.0, wl.dt)
    with pytest.raises(ValueError):
        dirk_step(prob, "RADAU23", u0, 0.0, wl.dt)
    with pytest.raises(ValueError):
        PrecondSpec(kind="bogus")
    with pytest.raises(NewtonError) as ei:
        irk_step_transformed(prob, "RADAU23", u0, 0.0, wl.dt, PrecondSpec("coupled"),
                             NewtonConfig(abs_tol_inf=1e-300, max_iters=1))
    assert len(ei.value.residual_history) == 2


R2_CASES = [("r47u", "RADAU47", "uncoupled"), ("r47c", "RADAU47", "coupled"),
            ("r59u", "RADAU59", "uncoupled"), ("r59c", "RADAU59", "coupled"),
            ("esdirk", "ESDIRK65", None)]


@pytest.mark.parametrize("name,scheme,kind", R2_CASES)
def test_device_steps_r2_vs_reference(name, scheme, kind):
    """s = 4 / 5 Radau IIA (generated tableaux, tableaux.py:246-254) through the
    device transformed step -- stage operator, coupled / shifted-uncoupled factor
    and GMRES at s > 3 -- and the ESDIRK65 step whose first stage is explicit (one
    block-diagonal mass solve, stepper.py:253-259), against the reference's steps
    (stepper_r2.npz): Newton counts equal, GMRES +-1, u within 1e-9, counters equal."""
    from paper_1701_07181_b200.blocks import DevicePattern, OpCounter
    from paper_1701_07181_b200.krylov import GmresConfig
    from paper_1701_07181_b200.stepper import (LinearProblem, NewtonConfig, PrecondSpec, StepCache,
                                               dirk_step, irk_step_transformed)
    g2 = load_golden("stepper_r2")
    cfg = W.CONFIGS[1].scaled(N=6, nb=8, dt_norm=10.0)
    wl = W.make_workload(cfg)
    assert sha(wl.J, wl.M) == str(g2["sha"])
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    tab = builtin_tableau(scheme)
    gcfg = GmresConfig(rel_tol=1e-8, restart=40)
    ctr, cache = OpCounter(), StepCache()
    u = g2["u0"]
    exact = True
    for step in (1, 2):
        if kind is None:
            res = dirk_step(prob, tab, u, 0.0, wl.dt, NewtonConfig(), gcfg, ctr, cache=cache)
        else:
            res = irk_step_transformed(prob, tab, u, 0.0, wl.dt, PrecondSpec(kind=kind),
                                       NewtonConfig(), gcfg, ctr, cache=cache)
        u = res.u_next
        assert res.newton_iterations == int(g2[f"{name}_newton{step}"])
        gref = list(g2[f"{name}_gmres{step}"])
        got = [st.iterations for st in res.gmres_stats]
        assert len(got) == len(gref) and all(abs(a - b) <= 1 for a, b in zip(got, gref)), (got, gref)
        exact &= got == gref
        assert rel(u.cpu().numpy(), g2[f"{name}_u{step}"]) < 1e-9
    have = np.array([ctr.block_multiplies, ctr.block_solves, ctr.block_factorizations,
                     ctr.mass_multiplies, ctr.jacobian_multiplies])
    if exact:
        np.testing.assert_array_equal(have, g2[f"{name}_counter"])


def test_mass_solve_vs_lu():
    """BlockDiagonalMatrix.solve (reference blocks.py:172-176, np.linalg.solve per
    block) on the device: the inverse of every mass block applied in one sweep,
    equal to the LU solve within 1e-12; counter += T block solves."""
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, OpCounter
    for nb, T in ((8, 72), (40, 512), (50, 300)):
        M = W.mass_blocks(T, nb, seed=5)
        x = np.random.default_rng(nb).standard_normal(T * nb)
        bd = BlockDiagonalMatrix(M)
        ctr = OpCounter()
        y = bd.solve(x, ctr)
        want = np.linalg.solve(M, x.reshape(T, nb, 1)).reshape(-1)
        assert rel(y, want) < 1e-12
        assert ctr.block_solves == T
        assert rel(bd.matvec(y), x) < 1e-12
        with pytest.raises(ValueError):
            bd.solve(x[:-1])


def test_partitioned_factor_t_not_divisible_by_p():
    """LinearProblem.partition_of for T % P != 0 (T=72, P=5 -> 15/15/14/14/14, the
    reference's np.array_split, meshing.py:81-90): the device partitioned ILU(0)
    apply equals the oracle's with the reference's keep mask (precond.py:26-45)."""
    import oracle as O
    from paper_1701_07181_b200.blocks import DevicePattern
    from paper_1701_07181_b200.precond import stage_uncoupled_factorize
    from paper_1701_07181_b200.stage_system import StageOperator
    from paper_1701_07181_b200.stepper import LinearProblem
    from paper_1701_07181_b200.tableau import derive
    cfg = W.CONFIGS[1].scaled(N=6, nb=8)
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    prob = LinearProblem(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J, wl.M)
    part = prob.partition_of(5)
    ref_part = np.concatenate([np.full(len(c), k) for k, c in enumerate(np.array_split(np.arange(p.T), 5))])
    np.testing.assert_array_equal(part, ref_part)
    np.testing.assert_array_equal(np.bincount(part), [15, 15, 14, 14, 14])
    der = derive(builtin_tableau("RADAU35"))
    op = StageOperator(der, wl.dt, prob.mass(), [prob.jac] * 3)
    fac = stage_uncoupled_factorize(op, der.shifts, partition_of=part)
    w = np.random.default_rng(5).standard_normal(3 * prob.n)
    oprob = O.problem_from_workload(wl)
    ofac = O.make_preconditioner(oprob, "uncoupled", der.shifts, partition_of=ref_part)
    assert rel(fac.apply(w), ofac.apply(w)) < 1e-12


@pytest.mark.parametrize("kind", ["uncoupled", "coupled", "dirk"])
def test_reference_closure_wrappers_run_native(kind):
    """The reference's stepper glue passes ``lambda v: op.matvec(v, counter)`` and
    ``lambda v: fac.apply(v, counter)`` to gmres (stepper.py:164-170, 268-274).
    With install_stepper those wrap this package's device objects; krylov.gmres
    recognises the wrappers and runs the native loop on the objects (fused Arnoldi
    product, no Python per iteration), charging the captured counters exactly as the
    wrappers would have been called.  Checked against the same solve through
    non-recognisable wrappers (Python callbacks every iteration): same iterations,
    x within 1e-10, identical OpCounter totals."""
    from paper_1701_07181_b200 import krylov
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DevicePattern, OpCounter
    from paper_1701_07181_b200.precond import (build_stage_matrix, ilu0_factorize, stage_coupled_factorize,
                                               stage_uncoupled_factorize)
    from paper_1701_07181_b200.stage_system import StageOperator
    from paper_1701_07181_b200.tableau import derive
    cfg = W.CONFIGS[1].scaled(N=8, ordering="color")
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    jac = BlockSparseMatrix.from_host(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J)
    mass = BlockDiagonalMatrix(wl.M)
    gcfg = krylov.GmresConfig(rel_tol=1e-8, restart=40)
    if kind == "dirk":
        tab = builtin_tableau("DIRK33")
        mat = build_stage_matrix(1.0, mass, jac, wl.dt * tab.A[0, 0])
        rhs = wl.rhs[:mat.n]
    else:
        tab = builtin_tableau("RADAU23" if kind == "coupled" else "RADAU35")
        der = derive(tab)
        op = StageOperator(der, wl.dt, mass, [jac] * tab.s)
        rhs = np.random.default_rng(3).standard_normal(op.total_dim)

    def run(recognisable):
        counter = OpCounter()
        if kind == "dirk":
            fac = ilu0_factorize(mat, counter)
            target = mat
        elif kind == "coupled":
            fac = stage_coupled_factorize(op, counter)
            target = op
        else:
            fac = stage_uncoupled_factorize(op, der.shifts, counter)
            target = op
        if recognisable:   # exactly the reference's wrappers
            a_op = lambda v: target.matvec(v, counter)  # noqa: E731
            a_pre = lambda v: fac.apply(v, counter)  # noqa: E731
            assert krylov.closure_call(a_op) is not None and krylov.closure_call(a_pre) is not None
        else:
            def a_op(v):
                y = target.matvec(v, counter)
                return y

            def a_pre(v):
                y = fac.apply(v, counter)
                return y
            assert krylov.closure_call(a_op) is None
        x, st = krylov.gmres(a_op, a_pre, rhs, gcfg)
        return x, st, counter.snapshot(), target, fac

    x1, s1, c1, target, fac = run(True)
    x2, s2, c2, _, _ = run(False)
    assert s1.converged and s1.iterations == s2.iterations
    assert rel(x1, x2) < 1e-10
    # the charged totals are the reference's (krylov.py:37-130: 2 + k + cycles matvecs and
    # applies); the callback loop skips the two calls whose results it already has (B*0 = 0,
    # so P^-1(b - B x0) is P^-1 b; no restart residual after the converged cycle), so it
    # calls each wrapper exactly twice less
    one = OpCounter()
    target._charge(one)
    fac._charge(one)
    one = one.snapshot()
    assert c1 == {k: c2[k] + 2 * one[k] for k in c2}, (c1, c2, one)


@pytest.mark.parametrize("kind", ["uncoupled", "coupled", "dirk"])
def test_factor_structure_pool_reuses_buffers(kind):
    """A collected factor parks its native handle; the next *_factorize call with the same
    structure re-factorises those buffers in place (the reference's steppers build a new
    preconditioner per Newton iteration, stepper.py:86-104).  Same handle, bitwise the same
    apply as the first (freshly allocated) factor; a different keep mask or shift count does
    not match; clear_factor_pool() empties the pool."""
    import gc
    from paper_1701_07181_b200 import precond as P
    from paper_1701_07181_b200.blocks import BlockDiagonalMatrix, BlockSparseMatrix, DevicePattern
    from paper_1701_07181_b200.stage_system import StageOperator
    from paper_1701_07181_b200.tableau import derive
    cfg = W.CONFIGS[1].scaled(N=6, ordering="color")
    wl = W.make_workload(cfg, norm_iters=10)
    p = wl.pattern
    jac = BlockSparseMatrix.from_host(DevicePattern(p.indptr, p.indices, p.diag_pos), wl.J)
    mass = BlockDiagonalMatrix(wl.M)
    tab = builtin_tableau("DIRK33" if kind == "dirk" else ("RADAU23" if kind == "coupled" else "RADAU35"))
    if kind == "dirk":
        mat = P.build_stage_matrix(1.0, mass, jac, wl.dt * tab.A[0, 0])
        make = lambda **kw: P.ilu0_factorize(mat, **kw)  # noqa: E731
        n = mat.n
    else:
        der = derive(tab)
        op = StageOperator(der, wl.dt, mass, [jac] * tab.s)
        n = op.total_dim
        if kind == "coupled":
            make = lambda **kw: P.stage_coupled_factorize(op, **kw)  # noqa: E731
        else:
            make = lambda **kw: P.stage_uncoupled_factorize(op, der.shifts, **kw)  # noqa: E731
    gc.collect()              # factors left by earlier tests park first, then the pool is emptied
    P.clear_factor_pool()
    y = np.random.default_rng(11).standard_normal(n)
    f1 = make()
    h1 = f1.handle
    x1 = f1.apply(y)
    del f1
    gc.collect()
    assert sum(len(v) for v in P._POOL.values()) == 1
    f2 = make()
    assert f2.handle == h1 and not P._POOL
    assert np.array_equal(f2.apply(y), x1)
    part = (np.arange(p.T) >= p.T // 2).astype(np.int64)
    f3 = make(partition_of=part)          # other keep mask: new structure
    assert f3.handle != h1
    del f2, f3
    gc.collect()
    assert len(P._POOL) == 2
    P.clear_factor_pool()
    assert not P._POOL
