"""ctypes binding of libirkb200.so (the C ABI in include/irkb200.h).

The CUDA library is the only compute path: importing this module on a machine
where the library is missing raises immediately, and every entry point raises
on a CUDA or argument error (there is no CPU fallback).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "csrc", "libirkb200.so")

IRK_OK = 0
IRK_ESINGULAR = 1


class IrkError(RuntimeError):
    """Error reported by libirkb200 (irk_last_error())."""


class SingularPivotError(IrkError):
    """A pivot block was numerically singular during factorization
    (same fields and message as reference precond.py:16-23)."""

    def __init__(self, element: int, stage: int | None = None):
        self.element = element
        self.stage = stage
        where = f"element {element}" if stage is None else f"stage {stage}, element {element}"
        super().__init__(f"numerically singular pivot block at {where}")


c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P = ctypes.POINTER

APPLY_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_vp, c_vp, c_vp)
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_vp, c_i64, c_vp)
XFER_FN = ctypes.CFUNCTYPE(c_int, c_vp, c_vp, c_vp, c_vp)


class Linop(ctypes.Structure):
    _fields_ = [("fn", c_vp), ("user", c_vp)]


class GmresCfg(ctypes.Structure):
    _fields_ = [("rel_tol", c_dbl), ("max_iters", c_int), ("restart", c_int),
                ("reorth_eta", c_dbl)]


class GmresStatsC(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("operator_applies", c_int), ("converged", c_int),
                ("breakdown", c_int), ("reorth_passes", c_int), ("history_len", c_int),
                ("b_norm", c_dbl), ("final_true_residual", c_dbl)]


_SIGS = {
    "irk_version": (c_int, []),
    "irk_last_error": (ctypes.c_char_p, []),
    "irk_launch_count": (c_i64, []),
    "irk_ctx_create": (c_int, [c_int, P(c_vp)]),
    "irk_ctx_destroy": (None, [c_vp]),
    "irk_pattern_create": (c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, P(c_vp)]),
    "irk_pattern_destroy": (None, [c_vp]),
    "irk_blocks_create": (c_int, [c_vp, c_int, c_i64, P(c_vp)]),
    "irk_blocks_destroy": (None, [c_vp]),
    "irk_blocks_upload": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_vp]),
    "irk_blocks_download": (c_int, [c_vp, c_i64, c_i64, c_vp, c_int, c_vp]),
    "irk_stage_op_create": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_dbl, P(c_vp)]),
    "irk_stage_op_destroy": (None, [c_vp]),
    "irk_stage_op_apply": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "irk_stage_op_set_halo": (c_int, [c_vp, c_i64, c_vp, c_i64]),
    "irk_factor_uncoupled": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp,
                                     c_int, c_int, P(c_vp), P(c_i64), P(c_i64), c_vp]),
    "irk_factor_coupled": (c_int, [c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp, c_vp,
                                   c_int, c_int, P(c_vp), P(c_i64), P(c_i64), c_vp]),
    "irk_factor_refactor": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp, P(c_i64), P(c_i64),
                                    c_vp]),
    "irk_factor_destroy": (None, [c_vp]),
    "irk_factor_apply": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "irk_op_factor_apply": (c_int, [c_vp, c_vp, c_vp, c_vp, P(c_int), c_vp]),
    "irk_stage_op_apply_range": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp]),
    "irk_stage_op_apply_rows": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "irk_factor_apply_rhs": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp]),
    "irk_factor_export": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "irk_factor_levels": (c_int, [c_vp, P(c_i64), P(c_i64)]),
    "irk_factor_implicit_l": (c_int, [c_vp]),
    "irk_linop_stage_op": (c_int, [c_vp, P(Linop)]),
    "irk_linop_factor": (c_int, [c_vp, P(Linop)]),
    "irk_gmres": (c_int, [c_vp, c_i64, Linop, Linop, c_vp, c_vp, c_vp, c_vp, P(GmresCfg),
                          P(GmresStatsC), c_vp, c_int, c_vp]),
    "irk_vec_multidot": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "irk_vec_update": (c_int, [c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "irk_comm_nccl_available": (c_int, []),
    "irk_comm_nccl_unique_id": (c_int, [c_vp, c_i64]),
    "irk_comm_create_nccl": (c_int, [c_vp, c_vp, c_int, c_int, P(c_vp)]),
    "irk_comm_create_callback": (c_int, [c_vp, c_int, c_int, c_vp, c_vp, c_vp, P(c_vp)]),
    "irk_comm_destroy": (None, [c_vp]),
    "irk_comm_allreduce": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "irk_halo_create": (c_int, [c_vp, c_int, c_int, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                                P(c_vp)]),
    "irk_halo_destroy": (None, [c_vp]),
    "irk_halo_exchange": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "irk_dist_op_create": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, P(c_vp)]),
    "irk_dist_op_destroy": (None, [c_vp]),
    "irk_dist_op_apply": (c_int, [c_vp, c_vp, c_vp, c_vp]),
    "irk_dist_op_factor_apply": (c_int, [c_vp, c_vp, c_vp, c_vp, P(c_int), c_vp]),
    "irk_linop_dist_op": (c_int, [c_vp, P(Linop)]),
    "irk_ref_bsr_matvec": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "irk_ref_ilu0_factor": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_int,
                                    c_vp, c_vp, P(c_i64)]),
    "irk_ref_ilu0_solve": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "irk_ref_coupled_factor": (c_int, [c_vp, c_int, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_int, c_vp, c_vp, c_vp, P(c_i64), P(c_i64)]),
    "irk_ref_coupled_solve": (c_int, [c_vp, c_int, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.RLock()


def load(path: str = LIB_PATH):
    """Load libirkb200.so (no compute; safe without a GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"libirkb200.so not built ({path}); run __graft_entry__.build() or "
                    "python -m paper_1701_07181_b200.build")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib():
    return _lib if _lib is not None else load()


def last_error() -> str:
    msg = lib().irk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> int:
    if rc < 0:
        raise IrkError(f"{what}: {last_error()} (status {rc})" if what else last_error())
    return rc


# ---------------------------------------------------------------------------
# context + device helpers (torch is only the device-memory / stream provider)
# ---------------------------------------------------------------------------

_ctx = {}


def torch():
    import torch as _t
    return _t


def ctx(device: int | None = None) -> int:
    t = torch()
    if not t.cuda.is_available():
        raise IrkError("no CUDA device: the irk-b200 path runs only on the GPU")
    dev = t.cuda.current_device() if device is None else int(device)
    with _lock:
        if dev not in _ctx:
            h = c_vp()
            check(lib().irk_ctx_create(dev, ctypes.byref(h)), "irk_ctx_create")
            _ctx[dev] = h.value
    return _ctx[dev]


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def ptr(a) -> int | None:
    """Raw pointer of a torch tensor or numpy array (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def f64_host(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64_host(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


class _DevBuf:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, p: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False),
                                         "version": 3, "strides": None}


def wrap_device(p: int, n: int):
    return torch().as_tensor(_DevBuf(p, n), device="cuda")
