"""One transformed-system stage-solve, fully native: the hot path as a unit.

A *stage-solve* (BASELINE metric) is: build the preconditioner for
B = A^-1 (x) M - dt blkdiag(J) and run left-preconditioned GMRES to rtol --
what reference ``irk_step_transformed.solve_correction`` does per Newton
iteration (stepper.py:164-170: ``_make_preconditioner`` + ``gmres``).
``StageSolver`` keeps J, M and the factors resident in HBM and drives
``irk_gmres`` with native operator/preconditioner handles (no Python in the
iteration loop).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib as L
from .blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
from .krylov import GmresConfig, GmresStats, gmres_device
from .precond import (partition_keep_mask, stage_coupled_factorize,
                      stage_uncoupled_factorize)
from .stage_system import StageOperator

KINDS = ("coupled", "coupled-literal", "uncoupled", "uncoupled-unshifted", "block-jacobi", "none")


class _Derived:
    def __init__(self, a_inv):
        self.a_inv = np.asarray(a_inv, dtype=np.float64)


class StageSolver:
    """Device-resident stage system + preconditioner + native GMRES.

    Parameters mirror the reference call chain: ``kind`` is a PrecondSpec kind
    (stepper.py:39-59), ``shifts`` the tableau shifts (tableaux.py:274),
    ``partition_of`` the ILU partition map (precond.py:26-45).
    """

    def __init__(self, pattern: DevicePattern, J, M, a_inv, dt: float, kind: str = "uncoupled",
                 shifts=None, partition_of=None, gmres_cfg: GmresConfig | None = None):
        if kind not in KINDS:
            raise ValueError(f"unknown preconditioner kind {kind!r}")
        a_inv = np.asarray(a_inv, dtype=np.float64)
        s = a_inv.shape[0]
        jm = J if isinstance(J, BlockSparseMatrix) else BlockSparseMatrix(
            pattern, J if isinstance(J, DeviceBlocks) else DeviceBlocks.from_host(J))
        mm = M if isinstance(M, BlockDiagonalMatrix) else BlockDiagonalMatrix(M)
        self.op = StageOperator(_Derived(a_inv), dt, mm, [jm] * s)
        self.kind = kind
        self.shifts = np.zeros(s) if shifts is None else np.asarray(shifts, dtype=np.float64)
        self.partition_of = partition_of
        self.cfg = gmres_cfg or GmresConfig(rel_tol=1e-8, restart=40)
        self.fac = None

    @property
    def n(self) -> int:
        return self.op.total_dim

    def factorize(self):
        """(Re)build the preconditioner; an existing factor of the same kind is
        re-factorised in place (no allocation)."""
        k = self.kind
        op = self.op
        if self.fac is not None and k in ("coupled", "coupled-literal"):
            return self.fac.refactor(op)
        if self.fac is not None and k == "uncoupled":
            return self.fac.refactor(op, self.shifts)
        if self.fac is not None and k in ("block-jacobi", "uncoupled-unshifted"):
            return self.fac.refactor(op, self.fac.shifts)
        if k == "none":
            self.fac = None
        elif k in ("coupled", "coupled-literal"):
            self.fac = stage_coupled_factorize(op, partition_of=self.partition_of,
                                               literal_update=k == "coupled-literal")
        elif k == "block-jacobi":
            self.fac = stage_uncoupled_factorize(op, self.shifts, partition_of=np.arange(op.pattern.T))
        elif k == "uncoupled":
            self.fac = stage_uncoupled_factorize(op, self.shifts, partition_of=self.partition_of)
        else:
            self.fac = stage_uncoupled_factorize(op, None, partition_of=self.partition_of)
        return self.fac

    def solve(self, rhs, x=None, allreduce=None) -> tuple:
        """GMRES on a CUDA-tensor rhs with native linops."""
        pre = None if self.fac is None else self.fac.apply
        return gmres_device(self.op.matvec, pre, rhs, self.cfg, allreduce=allreduce, x=x)

    def stage_solve(self, rhs, x=None):
        self.factorize()
        return self.solve(rhs, x=x)


def stage_solve_host(indptr, indices, diag_pos, J, M, a_inv, dt, rhs, kind="uncoupled",
                     shifts=None, partition_of=None, gmres_cfg=None):
    """End-to-end through host buffers: upload pattern, J, M and rhs, factorise,
    solve, return the solution to the host.  Returns (x, stats, timings)."""
    t = L.torch()
    t0 = time.perf_counter()
    pat = DevicePattern(indptr, indices, diag_pos)
    solver = StageSolver(pat, np.asarray(J), np.asarray(M), a_inv, dt, kind, shifts, partition_of,
                         gmres_cfg)
    rd = t.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64)).cuda()
    solver.factorize()
    x, stats = solver.solve(rd)
    xh = x.cpu().numpy()
    return xh, stats, time.perf_counter() - t0
