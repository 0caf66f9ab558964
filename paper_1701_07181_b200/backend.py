"""Kernel-plugin module with the reference backend protocol, on the GPU.

The reference selects its block kernels through a module global
(``irksolve.kernels._backend``, kernels/__init__.py:14,32-36); any module with
``NAME, COND_LIMIT, bsr_matvec, ilu0_factor, ilu0_solve, coupled_factor,
coupled_solve`` (numba_backend.py:10-151) can be installed there.  This module
implements that protocol through the host-pointer shims of libirkb200
(``irk_ref_*``): same arguments (int64 CSR-of-blocks, row-major (.., m, m)
fp64 blocks, bool keep masks), fresh output arrays, inputs never mutated, a
returned fail index instead of an exception.  See INTEGRATION.md.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L

NAME = "b200"
COND_LIMIT = 1e14


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _k(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def bsr_matvec(indptr, indices, data, x):
    indptr, indices, data, x = _i(indptr), _i(indices), _f(data), _f(x)
    T, m = len(indptr) - 1, data.shape[1]
    y = np.empty(T * m)
    L.check(L.lib().irk_ref_bsr_matvec(L.ctx(), T, m, indptr.ctypes.data, indices.ctypes.data,
                                       data.ctypes.data, x.ctypes.data, y.ctypes.data),
            "bsr_matvec")
    return y


def ilu0_factor(indptr, indices, diag_pos, data, keep, simplified):
    indptr, indices, diag_pos, data, keep = _i(indptr), _i(indices), _i(diag_pos), _f(data), _k(keep)
    T, m = len(indptr) - 1, data.shape[1]
    f = np.empty_like(data)
    dinv = np.empty((T, m, m))
    fail = ctypes.c_int64(-1)
    L.check(L.lib().irk_ref_ilu0_factor(L.ctx(), T, m, indptr.ctypes.data, indices.ctypes.data,
                                        diag_pos.ctypes.data, data.ctypes.data, keep.ctypes.data,
                                        int(bool(simplified)), f.ctypes.data, dinv.ctypes.data,
                                        ctypes.byref(fail)), "ilu0_factor")
    return f, dinv, int(fail.value)


def ilu0_solve(indptr, indices, diag_pos, fdata, dinv, keep, y):
    indptr, indices, diag_pos = _i(indptr), _i(indices), _i(diag_pos)
    fdata, dinv, keep, y = _f(fdata), _f(dinv), _k(keep), _f(y)
    T, m = len(indptr) - 1, fdata.shape[1]
    x = np.empty(T * m)
    L.check(L.lib().irk_ref_ilu0_solve(L.ctx(), T, m, indptr.ctypes.data, indices.ctypes.data,
                                       diag_pos.ctypes.data, fdata.ctypes.data, dinv.ctypes.data,
                                       keep.ctypes.data, y.ctypes.data, x.ctypes.data),
            "ilu0_solve")
    return x


def coupled_factor(indptr, indices, diag_pos, stage_data, coupling, keep, literal):
    indptr, indices, diag_pos = _i(indptr), _i(indices), _i(diag_pos)
    stage_data, coupling, keep = _f(stage_data), _f(coupling), _k(keep)
    s, T, m = stage_data.shape[0], len(indptr) - 1, stage_data.shape[2]
    f = np.empty_like(stage_data)
    g = np.empty_like(coupling)
    dinv = np.empty((s, T, m, m))
    fs, fe = ctypes.c_int64(-1), ctypes.c_int64(-1)
    L.check(L.lib().irk_ref_coupled_factor(L.ctx(), s, T, m, indptr.ctypes.data,
                                           indices.ctypes.data, diag_pos.ctypes.data,
                                           stage_data.ctypes.data, coupling.ctypes.data,
                                           keep.ctypes.data, int(bool(literal)), f.ctypes.data,
                                           g.ctypes.data, dinv.ctypes.data, ctypes.byref(fs),
                                           ctypes.byref(fe)), "coupled_factor")
    return f, g, dinv, int(fs.value), int(fe.value)


def coupled_solve(indptr, indices, diag_pos, fstage, fcoupling, dinv, keep, y):
    indptr, indices, diag_pos = _i(indptr), _i(indices), _i(diag_pos)
    fstage, fcoupling, dinv, keep, y = _f(fstage), _f(fcoupling), _f(dinv), _k(keep), _f(y)
    s, T, m = fstage.shape[0], len(indptr) - 1, fstage.shape[2]
    x = np.empty(s * T * m)
    L.check(L.lib().irk_ref_coupled_solve(L.ctx(), s, T, m, indptr.ctypes.data,
                                          indices.ctypes.data, diag_pos.ctypes.data,
                                          fstage.ctypes.data, fcoupling.ctypes.data,
                                          dinv.ctypes.data, keep.ctypes.data, y.ctypes.data,
                                          x.ctypes.data), "coupled_solve")
    return x
