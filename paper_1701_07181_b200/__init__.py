"""irk-b200: B200-native linear-solve hot path of arXiv 1701.07181.

Transformed Radau IIA stage system B = A^-1 (x) M - dt blkdiag(J_k), block
ILU(0) preconditioners (stage-coupled, shifted stage-uncoupled) and
left-preconditioned GMRES, in hand-written sm_100a CUDA behind the C ABI of
include/irkb200.h.  The Python API mirrors the reference package ``irksolve``
(same names and signatures for the hot-path objects), so reference code can
swap these in.

Importing the package does not touch the GPU; the first device call loads
libirkb200.so and fails loudly if it is missing.
"""

from ._lib import IrkError, SingularPivotError  # noqa: F401

__version__ = "0.1.0"

_LAZY = {
    "OpCounter": "blocks", "BlockSparseMatrix": "blocks", "BlockDiagonalMatrix": "blocks",
    "DevicePattern": "blocks", "DeviceBlocks": "blocks",
    "StageOperator": "stage_system",
    "partition_keep_mask": "precond", "build_stage_matrix": "precond", "BlockIlu0": "precond",
    "ilu0_factorize": "precond", "StageCoupledIlu0": "precond",
    "stage_coupled_factorize": "precond", "StageUncoupledIlu0": "precond",
    "stage_uncoupled_factorize": "precond",
    "GmresConfig": "krylov", "GmresStats": "krylov", "gmres": "krylov",
    "equivalent_multiplications": "krylov",
    "StageSolver": "solver",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
