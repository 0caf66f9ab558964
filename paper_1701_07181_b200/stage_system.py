"""Transformed stage operator B = A^-1 (x) M - dt blkdiag(J_1..J_s) on the GPU.

Drop-in for the reference ``StageOperator`` (stage_system.py:32-78): same
constructor, ``s``/``n``/``total_dim`` and ``matvec(w, counter=None)`` with the
same counter increments (stage_system.py:65-69).  The product runs as ONE fused
kernel (``irk_stage_op_apply``): every Jacobian block is read once and applied
to all s stage vectors, the block-diagonal mass term is read once, and the
s x s A^-1 mixing happens in registers -- instead of the reference's s
Jacobian sweeps plus s^2 mass sweeps.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from .blocks import (BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, OpCounter,
                     empty_like_dev, from_device, make_stage_op, pattern_for, to_device)


def as_device_matrix(J) -> BlockSparseMatrix:
    if isinstance(J, BlockSparseMatrix):
        return J
    return BlockSparseMatrix.from_reference(J)


def as_device_mass(M) -> BlockDiagonalMatrix:
    if isinstance(M, BlockDiagonalMatrix):
        return M
    return BlockDiagonalMatrix.from_reference(M)


def upload_stage_jacobians(jacobians):
    """Device matrices for a list of (reference or device) Jacobians, uploading
    a repeated object only once (shared Jacobian)."""
    seen = {}
    out = []
    for J in jacobians:
        key = id(J)
        if key not in seen:
            seen[key] = as_device_matrix(J)
        out.append(seen[key])
    return out


class StageOperator:
    """B = A^-1 (x) M - dt blkdiag(J_1, ..., J_s), device resident."""

    def __init__(self, derived, dt: float, mass, jacobians):
        a_inv = np.asarray(derived.a_inv, dtype=np.float64)
        if len(jacobians) != a_inv.shape[0]:
            raise ValueError("number of Jacobians must equal the stage count")
        graph = jacobians[0].graph
        m = jacobians[0].m
        for J in jacobians[1:]:
            if J.graph is not graph or J.m != m:
                raise ValueError("all stage Jacobians must share one graph and block size")
        T = len(jacobians[0].indptr) - 1
        if mass.T_elems != T or mass.m != m:
            raise ValueError("mass matrix dimensions do not match the Jacobians")
        self.derived = derived
        self.dt = float(dt)
        self.a_inv = a_inv
        self.host_jacobians = jacobians
        self.jacobians = upload_stage_jacobians(jacobians)
        self.mass = as_device_mass(mass)
        self.pattern = self.jacobians[0].pattern
        self._op = make_stage_op(self.pattern, self.s, [J.blocks for J in self.jacobians],
                                 [J.first for J in self.jacobians], self.mass.device, a_inv,
                                 -self.dt)

    @property
    def s(self) -> int:
        return len(self.jacobians)

    @property
    def n(self) -> int:
        return self.mass.n

    @property
    def total_dim(self) -> int:
        return self.s * self.n

    @property
    def shared_jacobian(self) -> bool:
        return all(J is self.jacobians[0] for J in self.jacobians)

    def apply_device(self, w, y) -> None:
        """y = B w for CUDA tensors (no allocation, no counters)."""
        L.check(L.lib().irk_stage_op_apply(self._op.handle, w.data_ptr(), y.data_ptr(),
                                           L.stream_ptr()), "irk_stage_op_apply")

    def apply_device_range(self, w, y, row_lo: int, row_hi: int) -> None:
        """Rows [row_lo, row_hi) of y = B w (multi-GPU interior rows)."""
        L.check(L.lib().irk_stage_op_apply_range(self._op.handle, w.data_ptr(), y.data_ptr(), int(row_lo),
                                                 int(row_hi), L.stream_ptr()), "irk_stage_op_apply_range")

    def apply_device_rows(self, w, y, rows) -> None:
        """Rows ``rows`` (CUDA int32 tensor) of y = B w (multi-GPU boundary rows)."""
        L.check(L.lib().irk_stage_op_apply_rows(self._op.handle, w.data_ptr(), y.data_ptr(), rows.data_ptr(),
                                                rows.numel(), L.stream_ptr()), "irk_stage_op_apply_rows")

    def matvec(self, w, counter: OpCounter | None = None):
        if tuple(w.shape) != (self.total_dim,):
            raise ValueError(f"expected vector of length {self.total_dim}, got {tuple(w.shape)}")
        wd, was_np = to_device(w)
        y = empty_like_dev(self.total_dim)
        self.apply_device(wd, y)
        if counter is not None:
            self._charge(counter)
        return from_device(y, was_np)

    def _charge(self, counter: OpCounter) -> None:
        """Counter increments of one matvec, exactly as stage_system.py:65-69."""
        jac = sum(J.nnz_blocks for J in self.jacobians)
        T = self.mass.T_elems
        counter.jacobian_multiplies += jac
        counter.mass_multiplies += self.s * self.s * T
        counter.block_multiplies += jac + self.s * self.s * T

    def native_linop(self):
        op = L.Linop()
        L.check(L.lib().irk_linop_stage_op(self._op.handle, op), "irk_linop_stage_op")
        return op, self
