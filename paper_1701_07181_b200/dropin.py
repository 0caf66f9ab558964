"""Install the B200 path into an unmodified reference ``irksolve`` package.

Two drop-in levels:

* ``install_backend(irksolve)`` -- parity mode: the reference's kernel-plugin
  global ``irksolve.kernels._backend`` (kernels/__init__.py:14, 32-36) is set
  to ``paper_1701_07181_b200.backend``; every ``bsr_matvec / ilu0_factor /
  ilu0_solve / coupled_factor / coupled_solve`` call of the reference then runs
  on the GPU through the host-pointer shims of the C ABI.

* ``install_stepper(irksolve)`` -- performance mode: the names that
  ``irksolve.stepper`` binds at import (stepper.py:18-24: ``StageOperator``,
  ``build_stage_matrix``, ``ilu0_factorize``, ``stage_coupled_factorize``,
  ``stage_uncoupled_factorize``, ``gmres``) are replaced by the device-resident
  versions of this package, so ``irk_step_transformed`` / ``dirk_step`` /
  ``integrate`` keep J, M, the factors and the Krylov basis in HBM for a whole
  linear solve.  ``pkg/src`` is not modified.

Both return a callable that restores the previous state.
"""

from __future__ import annotations

STEPPER_NAMES = ("StageOperator", "build_stage_matrix", "ilu0_factorize",
                 "stage_coupled_factorize", "stage_uncoupled_factorize", "gmres")


def install_backend(irksolve):
    from . import backend
    kernels = irksolve.kernels
    previous = kernels._backend
    kernels._backend = backend

    def restore():
        kernels._backend = previous
    return restore


def install_stepper(irksolve):
    from . import krylov, precond, stage_system
    stepper = irksolve.stepper
    mine = {
        "StageOperator": stage_system.StageOperator,
        "build_stage_matrix": precond.build_stage_matrix,
        "ilu0_factorize": precond.ilu0_factorize,
        "stage_coupled_factorize": precond.stage_coupled_factorize,
        "stage_uncoupled_factorize": precond.stage_uncoupled_factorize,
        "gmres": krylov.gmres,
    }
    previous = {name: getattr(stepper, name) for name in STEPPER_NAMES}
    for name, obj in mine.items():
        setattr(stepper, name, obj)

    def restore():
        for name, obj in previous.items():
            setattr(stepper, name, obj)
    return restore
