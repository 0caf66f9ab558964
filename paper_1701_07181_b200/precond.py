"""Block ILU(0) preconditioners on the GPU, mirroring reference ``precond.py``.

Same public names, signatures, counters and error behaviour as the reference
(precond.py:16-280): ``partition_keep_mask``, ``build_stage_matrix``,
``ilu0_factorize`` / ``BlockIlu0``, ``stage_coupled_factorize`` /
``StageCoupledIlu0`` and ``stage_uncoupled_factorize`` / ``StageUncoupledIlu0``,
``SingularPivotError(element, stage)``.

Factorisation and apply run in libirkb200 (``irk_factor_*``).  A stage matrix
coef*M - dt*J is never assembled: the factorisation reads J and M directly and
forms coef*M_j - dt*J_jj on the fly, and the upper factor blocks U_ij =
-dt*J_ij are read from J itself (they are identical for all stages when J is
shared), so the uncoupled preconditioner stores only L and D^-1 per stage.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._lib import SingularPivotError
from .blocks import (BlockDiagonalMatrix, BlockSparseMatrix, DevicePattern, OpCounter,
                     empty_like_dev, from_device, make_stage_op, pattern_for, to_device)
from .stage_system import StageOperator, as_device_mass, as_device_matrix

__all__ = ["SingularPivotError", "partition_keep_mask", "build_stage_matrix", "StageMatrix",
           "BlockIlu0", "ilu0_factorize", "StageCoupledIlu0", "stage_coupled_factorize",
           "StageUncoupledIlu0", "stage_uncoupled_factorize", "simplified_condition",
           "clear_factor_pool"]


def partition_keep_mask(mat, partition_of) -> np.ndarray:
    """True for blocks kept in the factorisation pattern (precond.py:26-45)."""
    nnzb = int(mat.indptr[-1])
    keep = np.ones(nnzb, dtype=np.bool_)
    if partition_of is None:
        return keep
    part = np.asarray(partition_of)
    T = len(mat.indptr) - 1
    if part.shape != (T,):
        raise ValueError(f"partition map must have length {T}")
    rows = np.repeat(np.arange(T), np.diff(mat.indptr))
    cols = np.asarray(mat.indices)
    return (rows == cols) | (part[rows] == part[cols])


_SIMPLIFIED: dict = {}


def simplified_condition(pattern) -> bool:
    """No two neighbours of any element are neighbours (meshing.py:43-52),
    vectorised over a pattern (anything with indptr/indices), cached."""
    key = id(pattern)
    hit = _SIMPLIFIED.get(key)
    if hit is not None and hit[0] is pattern:
        return hit[1]
    ip, ix = np.asarray(pattern.indptr), np.asarray(pattern.indices)
    T = len(ip) - 1
    rows = np.repeat(np.arange(T), np.diff(ip))
    off = ix != rows
    nbr_rows, nbr_cols = rows[off], ix[off]
    keys = np.sort(nbr_rows * T + nbr_cols)
    ok = True
    # for each element, test every pair (u, v) of its neighbours
    start = np.searchsorted(nbr_rows, np.arange(T))
    end = np.searchsorted(nbr_rows, np.arange(T), side="right")
    deg = end - start
    for d in np.unique(deg):
        if d < 2:
            continue
        els = np.nonzero(deg == d)[0]
        nb = nbr_cols[start[els][:, None] + np.arange(d)[None, :]]
        for a in range(d):
            for b in range(a + 1, d):
                q = nb[:, a] * T + nb[:, b]
                pos = np.searchsorted(keys, q)
                pos = np.minimum(pos, len(keys) - 1)
                if np.any(keys[pos] == q):
                    ok = False
                    break
            if not ok:
                break
        if not ok:
            break
    _SIMPLIFIED[key] = (pattern, ok)
    return ok


class StageMatrix:
    """coef * M - dt * J on J's pattern, kept implicit on the device
    (reference build_stage_matrix, precond.py:48-54, assembles it)."""

    def __init__(self, coef: float, mass, jac, dt: float):
        self.coef = float(coef)
        self.dt = float(dt)
        self.jac = as_device_matrix(jac)
        self.mass = as_device_mass(mass)
        self.pattern = self.jac.pattern
        self.graph = self.jac.graph
        self.m = self.jac.m
        self.indptr, self.indices, self.diag_pos = self.jac.indptr, self.jac.indices, self.jac.diag_pos
        self._op = None

    @property
    def T_elems(self) -> int:
        return self.pattern.T

    @property
    def n(self) -> int:
        return self.pattern.T * self.m

    @property
    def nnz_blocks(self) -> int:
        return self.pattern.nnzb

    @property
    def data(self) -> np.ndarray:
        out = self.jac.data * (-self.dt)
        out[self.diag_pos] += self.coef * self.mass.blocks
        return out

    def _native_op(self):
        if self._op is None:
            self._op = make_stage_op(self.pattern, 1, [self.jac.blocks], [self.jac.first],
                                     self.mass.device, np.array([[self.coef]]), -self.dt)
        return self._op

    def native_linop(self):
        op = L.Linop()
        L.check(L.lib().irk_linop_stage_op(self._native_op().handle, op), "irk_linop_stage_op")
        return op, self

    def apply_device(self, x, y) -> None:
        L.check(L.lib().irk_stage_op_apply(self._native_op().handle, x.data_ptr(), y.data_ptr(),
                                           L.stream_ptr()), "irk_stage_op_apply")

    def matvec(self, x, counter: OpCounter | None = None):
        if tuple(x.shape) != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {tuple(x.shape)}")
        self._native_op()
        xd, was_np = to_device(x)
        y = empty_like_dev(self.n)
        L.check(L.lib().irk_stage_op_apply(self._op.handle, xd.data_ptr(), y.data_ptr(),
                                           L.stream_ptr()), "irk_stage_op_apply")
        if counter is not None:
            self._charge(counter)
        return from_device(y, was_np)

    def _charge(self, counter: OpCounter) -> None:
        """Counter increments of one matvec (precond.py:57 via BlockSparseMatrix.matvec)."""
        counter.block_multiplies += self.nnz_blocks


def build_stage_matrix(coef: float, mass, jac, dt: float) -> StageMatrix:
    return StageMatrix(coef, mass, jac, dt)


# Structure pool.  The reference's steppers build a NEW preconditioner object in every Newton
# iteration (stepper.py:86-104); creating an ``irk_factor`` allocates its device buffers and
# builds the level schedules on the host (config 1: ~18 ms, more than the 10 ms stage-solve).
# A factor object that is garbage-collected parks its native handle here, keyed by everything
# ``irk_factor_refactor`` requires to stay the same (pattern, kind, stage count, block size, keep
# mask, simplified / store_diag / literal, shared-J structure); the next ``*_factorize`` call with
# the same key takes it and re-factorises in place -- same numerics (bitwise: in-place refactor ==
# fresh factor, tested), no allocation.  At most ``_POOL_PER_KEY`` handles per key and
# ``_POOL_KEYS`` keys are parked (a parked config-1 factor holds 2.5 GB); IRK_FACTOR_POOL=0
# disables it, ``clear_factor_pool()`` frees the parked handles.
import os as _os

_POOL: dict = {}
_POOL_PER_KEY, _POOL_KEYS = 1, 2
_POOL_ON = _os.environ.get("IRK_FACTOR_POOL", "1") != "0"


def clear_factor_pool() -> None:
    """Destroy every parked factor handle (device memory is returned)."""
    while _POOL:
        _, items = _POOL.popitem()
        for h, _keep in items:
            if L._lib is not None:
                L._lib.irk_factor_destroy(h)


def _pool_key(kind, pattern, jblocks, mass, keep_u8, *flags):
    shared = tuple(int(b.handle == jblocks[0].handle) for b in jblocks)
    return (kind, int(pattern.handle), len(jblocks), int(jblocks[0].nb), shared, mass is None,
            keep_u8.tobytes(), *flags)


def _pool_take(key):
    items = _POOL.get(key) if _POOL_ON else None
    if not items:
        return None
    item = items.pop()
    if not items:
        del _POOL[key]
    return item


class _Factor:
    """Owns an ``irk_factor`` handle plus everything it references."""

    _pool_key = None

    def __init__(self, handle, keepalive, s, n_elem, m, keep):
        self.handle = handle
        self.keepalive = keepalive
        self.s = s
        self.T_elems = n_elem
        self.m = m
        self.keep = keep

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and L._lib is not None:
            key = self._pool_key
            if _POOL_ON and key is not None and (key in _POOL or len(_POOL) < _POOL_KEYS) \
                    and len(_POOL.get(key, ())) < _POOL_PER_KEY:
                _POOL.setdefault(key, []).append((h, self.keepalive))
            else:
                L._lib.irk_factor_destroy(h)
            self.handle = None

    def apply_device(self, y, x) -> None:
        L.check(L.lib().irk_factor_apply(self.handle, y.data_ptr(), x.data_ptr(), L.stream_ptr()),
                "irk_factor_apply")

    def _apply(self, y, n_total):
        if tuple(y.shape) != (n_total,):
            raise ValueError(f"expected vector of length {n_total}, got {tuple(y.shape)}")
        yd, was_np = to_device(y)
        x = empty_like_dev(n_total)
        self.apply_device(yd, x)
        return from_device(x, was_np)

    def native_linop(self):
        op = L.Linop()
        L.check(L.lib().irk_linop_factor(self.handle, op), "irk_linop_factor")
        return op, self

    @property
    def implicit_l(self) -> bool:
        """True when L is never stored (forward sweep uses w_j = Dinv_j z_j)."""
        rc = L.lib().irk_factor_implicit_l(self.handle)
        L.check(min(rc, 0), "irk_factor_implicit_l")
        return rc == 1

    def levels(self) -> tuple[int, int]:
        f, b = ctypes.c_int64(), ctypes.c_int64()
        L.check(L.lib().irk_factor_levels(self.handle, ctypes.byref(f), ctypes.byref(b)))
        return f.value, b.value

    def export(self):
        """(fstage (s,nnzb,m,m), dinv (s,T,m,m), fcoupling or None) on the host,
        in the reference's factor layout."""
        nnzb = len(self.keep)
        fs = np.empty((self.s, nnzb, self.m, self.m))
        dv = np.empty((self.s, self.T_elems, self.m, self.m))
        fc = np.empty((self.s, self.s, self.T_elems, self.m, self.m)) if self._coupled else None
        L.check(L.lib().irk_factor_export(self.handle, fs.ctypes.data, dv.ctypes.data,
                                          None if fc is None else fc.ctypes.data, L.stream_ptr()),
                "irk_factor_export")
        return fs, dv, fc

    _coupled = False

    def _refactor(self, jblocks, jfirst, mass, coef, alpha, staged):
        s = len(jblocks)
        jarr = (ctypes.c_void_p * s)(*[b.handle for b in jblocks])
        jf = (ctypes.c_int64 * s)(*[int(v) for v in jfirst])
        carr = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
        fs, fe = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = L.lib().irk_factor_refactor(self.handle, jarr, jf,
                                         None if mass is None else mass.handle, L.ptr(carr),
                                         float(alpha), None, ctypes.byref(fs), ctypes.byref(fe),
                                         L.stream_ptr())
        L.check(rc, "irk_factor_refactor")
        self.keepalive = (self.keepalive[0], jblocks, mass, carr, self.keepalive[4], jarr, jf)
        if rc == L.IRK_ESINGULAR:
            raise SingularPivotError(fe.value, stage=fs.value if staged else None)
        return self


def _call_factor(fn, *args):
    h = ctypes.c_void_p()
    fs, fe = ctypes.c_int64(-1), ctypes.c_int64(-1)
    rc = fn(*args, ctypes.byref(h), ctypes.byref(fs), ctypes.byref(fe), L.stream_ptr())
    L.check(rc, fn.__name__)
    return h.value, rc, fs.value, fe.value


def _stage_sources(jacobians):
    """Device block arrays + first-block offsets for a list of device matrices."""
    return [J.blocks for J in jacobians], [J.first for J in jacobians]


def _uncoupled(cls, pattern, jblocks, jfirst, mass, coefs, alpha, keep, simplified, store_diag,
               staged):
    s = len(jblocks)
    jarr = (ctypes.c_void_p * s)(*[b.handle for b in jblocks])
    jf = (ctypes.c_int64 * s)(*jfirst)
    coef = None if coefs is None else np.ascontiguousarray(coefs, dtype=np.float64)
    keep_u8 = np.ascontiguousarray(keep, dtype=np.uint8)
    key = _pool_key(cls.__name__, pattern, jblocks, mass, keep_u8, bool(simplified), bool(store_diag))
    parked = _pool_take(key)
    if parked is not None:
        # same structure as a collected factor: re-factorise its buffers in place
        fac = cls(parked[0], parked[1], s, pattern.T, jblocks[0].nb, keep_u8.astype(bool))
        fac._pool_key = key
        return fac._refactor(jblocks, jfirst, mass, coef, alpha, staged)
    h, rc, fs, fe = _call_factor(L.lib().irk_factor_uncoupled, pattern.ctx, pattern.handle, s, jarr,
                                 jf, None if mass is None else mass.handle, L.ptr(coef),
                                 float(alpha), keep_u8.ctypes.data, int(simplified),
                                 int(store_diag))
    fac = cls(h, (pattern, jblocks, mass, coef, keep_u8, jarr, jf), s, pattern.T,
              jblocks[0].nb, keep_u8.astype(bool))
    fac._pool_key = key
    if rc == L.IRK_ESINGULAR:
        del fac
        raise SingularPivotError(fe, stage=fs if staged else None)
    return fac


class BlockIlu0(_Factor):
    """Zero-fill block LU factors of one Jacobian-pattern matrix (precond.py:57-87)."""

    @property
    def n(self) -> int:
        return self.T_elems * self.m

    @property
    def num_kept_offdiag(self) -> int:
        return int(self.keep.sum()) - self.T_elems

    def refactor(self, mat) -> "BlockIlu0":
        """Numeric re-factorisation for new values on the same structure, in
        place (no allocation): a StageMatrix (coef M - dt J) or a matrix J."""
        if isinstance(mat, StageMatrix):
            return self._refactor([mat.jac.blocks], [mat.jac.first], mat.mass.device, [mat.coef],
                                  -mat.dt, False)
        dm = as_device_matrix(mat)
        return self._refactor([dm.blocks], [dm.first], None, None, 1.0, False)

    def apply(self, y, counter: OpCounter | None = None):
        x = self._apply(y, self.n)
        if counter is not None:
            self._charge(counter)
        return x

    def _charge(self, counter: OpCounter) -> None:
        """precond.py:84-86"""
        counter.block_multiplies += self.num_kept_offdiag + self.T_elems

    def apply_rhs_device(self, y, x, nrhs: int) -> None:
        """x = P^-1 y for nrhs stage-major columns (nrhs, T, m) in one sweep that
        reads the factor once (BASELINE config 3; same result as nrhs applies)."""
        L.check(L.lib().irk_factor_apply_rhs(self.handle, int(nrhs), y.data_ptr(), x.data_ptr(),
                                             L.stream_ptr()), "irk_factor_apply_rhs")

    def apply_rhs(self, Y, counter: OpCounter | None = None):
        """Apply to the rows of Y (nrhs, n) (numpy or CUDA tensor)."""
        nrhs = int(Y.shape[0])
        if tuple(Y.shape) != (nrhs, self.n):
            raise ValueError(f"expected shape (nrhs, {self.n}), got {tuple(Y.shape)}")
        yd, was_np = to_device(Y.reshape(-1))
        x = empty_like_dev(nrhs * self.n)
        self.apply_rhs_device(yd, x, nrhs)
        if counter is not None:
            counter.block_multiplies += nrhs * (self.num_kept_offdiag + self.T_elems)
        return from_device(x, was_np).reshape(nrhs, self.n)

    @property
    def fdata(self) -> np.ndarray:
        return self.export()[0][0]

    @property
    def dinv(self) -> np.ndarray:
        return self.export()[1][0]


def ilu0_factorize(mat, counter: OpCounter | None = None, partition_of=None,
                   force_general: bool = False, store_diag: bool = False) -> BlockIlu0:
    """Block ILU(0) (precond.py:90-110); simplified sweep whenever the graph allows."""
    if isinstance(mat, StageMatrix):
        pattern, jb, jf = mat.pattern, [mat.jac.blocks], [mat.jac.first]
        mass, coefs, alpha = mat.mass.device, [mat.coef], -mat.dt
    else:
        dm = as_device_matrix(mat)
        pattern, jb, jf = dm.pattern, [dm.blocks], [dm.first]
        mass, coefs, alpha = None, None, 1.0
    simplified = simplified_condition(pattern) and not force_general
    keep = partition_keep_mask(pattern, partition_of)
    fac = _uncoupled(BlockIlu0, pattern, jb, jf, mass, coefs, alpha, keep, simplified,
                     store_diag or not simplified, staged=False)
    if counter is not None:
        counter.block_factorizations += pattern.T
        counter.block_multiplies += 2 * pattern.upper_count(keep)
    return fac


class StageUncoupledIlu0(_Factor):
    """s independent shifted ILU(0) factors (precond.py:203-241), held and
    applied together: one kernel sweep handles all stages of an element."""

    shifts: np.ndarray = None
    workers: int = 1

    @property
    def n(self) -> int:
        return self.T_elems * self.m

    def memory_blocks(self) -> int:
        return self.s * len(self.keep)

    def refactor(self, op: StageOperator, shifts=None) -> "StageUncoupledIlu0":
        """Re-factorise for a new operator with the same structure, in place
        (no device allocation; one Newton iteration's preconditioner)."""
        shifts = self.shifts if shifts is None else np.asarray(shifts, dtype=np.float64)
        jb, jf = _stage_sources(op.jacobians)
        self.shifts = shifts
        return self._refactor(jb, jf, op.mass.device, np.diag(op.a_inv) + shifts, -op.dt, True)

    def apply(self, y, counter: OpCounter | None = None):
        x = self._apply(y, self.s * self.n)
        if counter is not None:
            self._charge(counter)
        return x

    def _charge(self, counter: OpCounter) -> None:
        """precond.py:228-241 (s per-stage applies, precond.py:84-86 each)"""
        kept_off = int(self.keep.sum()) - self.T_elems
        counter.block_multiplies += self.s * (kept_off + self.T_elems)


def stage_uncoupled_factorize(op: StageOperator, shifts=None, counter: OpCounter | None = None,
                              partition_of=None, workers: int = 1,
                              store_diag: bool = False) -> StageUncoupledIlu0:
    """s ILU(0) factors of (A^-1_ii + alpha_i) M - dt J_i (precond.py:244-280).
    ``workers`` is accepted for API parity: all stages always run concurrently
    on the device and results do not depend on it."""
    s = op.s
    a_inv_diag = np.diag(op.a_inv)
    shifts = np.zeros(s) if shifts is None else np.asarray(shifts, dtype=np.float64)
    if shifts.shape != (s,):
        raise ValueError(f"expected {s} shifts, got shape {shifts.shape}")
    keep = partition_keep_mask(op.pattern, partition_of)
    simplified = simplified_condition(op.pattern)
    jb, jf = _stage_sources(op.jacobians)
    coefs = a_inv_diag + shifts
    fac = _uncoupled(StageUncoupledIlu0, op.pattern, jb, jf, op.mass.device, coefs, -op.dt, keep,
                     simplified, store_diag or not simplified, staged=True)
    fac.shifts = shifts
    fac.workers = workers
    if counter is not None:
        counter.block_factorizations += s * op.pattern.T
        counter.block_multiplies += 2 * s * op.pattern.upper_count(keep)
    return fac


class StageCoupledIlu0(_Factor):
    """Stage-coupled block ILU(0) of the transformed operator (precond.py:117-162)."""

    _coupled = True

    @property
    def n_total(self) -> int:
        return self.s * self.T_elems * self.m

    @property
    def num_kept_offdiag_per_stage(self) -> int:
        return int(self.keep.sum()) - self.T_elems

    @property
    def num_coupling_blocks(self) -> int:
        return (self.s * self.s - self.s) * self.T_elems

    def memory_blocks(self) -> int:
        return self.s * len(self.keep) + self.num_coupling_blocks

    def refactor(self, op: StageOperator) -> "StageCoupledIlu0":
        jb, jf = _stage_sources(op.jacobians)
        return self._refactor(jb, jf, op.mass.device, np.ascontiguousarray(op.a_inv), -op.dt, True)

    def apply(self, y, counter: OpCounter | None = None):
        x = self._apply(y, self.n_total)
        if counter is not None:
            self._charge(counter)
        return x

    def _charge(self, counter: OpCounter) -> None:
        """precond.py:158-161"""
        counter.block_multiplies += (self.s * self.num_kept_offdiag_per_stage
                                     + self.num_coupling_blocks + self.s * self.T_elems)


def stage_coupled_factorize(op: StageOperator, counter: OpCounter | None = None,
                            partition_of=None, literal_update: bool = False,
                            store_diag: bool = False) -> StageCoupledIlu0:
    """Stage-coupled ILU(0), Alg. 3 (precond.py:165-200)."""
    s, T = op.s, op.pattern.T
    keep = partition_keep_mask(op.pattern, partition_of)
    keep_u8 = np.ascontiguousarray(keep, dtype=np.uint8)
    jb, jf = _stage_sources(op.jacobians)
    jarr = (ctypes.c_void_p * s)(*[b.handle for b in jb])
    jfa = (ctypes.c_int64 * s)(*jf)
    a_inv = np.ascontiguousarray(op.a_inv, dtype=np.float64)
    key = _pool_key("StageCoupledIlu0", op.pattern, jb, op.mass.device, keep_u8, bool(literal_update),
                    bool(store_diag))
    parked = _pool_take(key)
    if parked is not None:
        fac = StageCoupledIlu0(parked[0], parked[1], s, T, op.jacobians[0].m, keep)
        fac._pool_key = key
        fac._refactor(jb, jf, op.mass.device, a_inv, -op.dt, True)
        if counter is not None:
            counter.block_factorizations += s * T
            counter.block_multiplies += 2 * s * op.pattern.upper_count(keep) + (s * s - s) * T
        return fac
    h, rc, fs, fe = _call_factor(L.lib().irk_factor_coupled, op.pattern.ctx, op.pattern.handle, s,
                                 jarr, jfa, op.mass.device.handle, a_inv.ctypes.data, -op.dt, None,
                                 keep_u8.ctypes.data, int(bool(literal_update)), int(store_diag))
    fac = StageCoupledIlu0(h, (op.pattern, jb, op.mass, a_inv, keep_u8, jarr, jfa), s, T,
                           op.jacobians[0].m, keep)
    fac._pool_key = key
    if rc == L.IRK_ESINGULAR:
        del fac
        raise SingularPivotError(fe, stage=fs)
    if counter is not None:
        counter.block_factorizations += s * T
        counter.block_multiplies += 2 * s * op.pattern.upper_count(keep) + (s * s - s) * T
    return fac
