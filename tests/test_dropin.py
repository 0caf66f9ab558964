"""The drop-in boundary: names, signatures and installation into the
unmodified reference package (skipped where /root/reference is absent, e.g.
on the GPU box)."""

import inspect
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def irksolve():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    sys.path.insert(0, REF)
    import irksolve as ref
    return ref


def _params(fn):
    return list(inspect.signature(fn).parameters)


def test_backend_protocol_signatures(irksolve):
    from irksolve.kernels import numpy_backend as ref_be

    from paper_1701_07181_b200 import backend
    assert backend.COND_LIMIT == ref_be.COND_LIMIT
    for name in ("bsr_matvec", "ilu0_factor", "ilu0_solve", "coupled_factor", "coupled_solve"):
        assert _params(getattr(backend, name)) == _params(getattr(ref_be, name)), name


def test_stepper_level_signatures(irksolve):
    from paper_1701_07181_b200 import krylov, precond, stage_system
    pairs = [(stage_system.StageOperator.__init__, irksolve.StageOperator.__init__),
             (precond.build_stage_matrix, irksolve.build_stage_matrix),
             (precond.ilu0_factorize, irksolve.ilu0_factorize),
             (precond.stage_coupled_factorize, irksolve.stage_coupled_factorize),
             (precond.stage_uncoupled_factorize, irksolve.stage_uncoupled_factorize),
             (precond.partition_keep_mask, irksolve.partition_keep_mask),
             (krylov.gmres, irksolve.gmres)]
    for mine, ref in pairs:
        ref_p = _params(ref)
        assert _params(mine)[:len(ref_p)] == ref_p, (mine, ref)
    for field in ("rel_tol", "max_iters", "restart", "left_precondition"):
        assert hasattr(krylov.GmresConfig(), field)
    for field in ("iterations", "operator_applies", "residual_history", "converged",
                  "final_true_residual"):
        assert hasattr(krylov.GmresStats(), field)


def test_install_and_restore(irksolve):
    from paper_1701_07181_b200 import backend, dropin, krylov, stage_system
    before = {n: getattr(irksolve.stepper, n) for n in dropin.STEPPER_NAMES}
    restore = dropin.install_stepper(irksolve)
    assert irksolve.stepper.StageOperator is stage_system.StageOperator
    assert irksolve.stepper.gmres is krylov.gmres
    restore()
    assert {n: getattr(irksolve.stepper, n) for n in dropin.STEPPER_NAMES} == before
    prev = irksolve.kernels.get_backend()
    restore = dropin.install_backend(irksolve)
    assert irksolve.kernels.get_backend() is backend
    restore()
    assert irksolve.kernels.get_backend() is prev
