"""Left-preconditioned restarted GMRES, drop-in for reference ``krylov.py``.

``gmres(apply_operator, apply_precond, rhs, cfg)`` has the reference's
signature, configuration (``GmresConfig``) and statistics (``GmresStats``)
(krylov.py:10-130).  The solver loop is the native ``irk_gmres`` (C++/CUDA,
fused classical Gram-Schmidt).  Operators are either this package's device
objects (bound ``matvec``/``apply`` methods run natively, with no Python in the
loop) or arbitrary Python callables on CUDA tensors, which the native loop
calls back.  ``rhs`` may be a numpy array (the solution comes back as numpy)
or a CUDA tensor.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .blocks import from_device, to_device


@dataclass
class GmresConfig:
    rel_tol: float = 1e-5
    max_iters: int = 500
    restart: int | None = None  # None = full (unrestarted) GMRES
    left_precondition: bool = True
    reorth_eta: float = 0.7071067811865476  # DGKS re-orthogonalisation threshold

    def __post_init__(self):
        if self.rel_tol <= 0:
            raise ValueError("rel_tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")


@dataclass
class GmresStats:
    iterations: int = 0
    operator_applies: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    final_true_residual: float = np.nan
    reorth_passes: int = 0
    b_norm: float = np.nan


def equivalent_multiplications(stats: GmresStats, s_implicit: int, is_irk: bool) -> int:
    """krylov.py:153-162: iterations x implicit stage count."""
    del is_irk
    return stats.iterations * s_implicit


_SKIP_OPS = {"RESUME", "COPY_FREE_VARS", "CACHE", "PUSH_NULL", "PRECALL", "NOP", "MAKE_CELL", "KW_NAMES"}


def closure_call(fn):
    """Recognise the reference's operator wrappers -- ``lambda v: op.matvec(v,
    counter)`` / ``lambda v: fac.apply(v, counter)`` (stepper.py:168-170, 272-274)
    -- by their bytecode: one positional parameter, a single call of the
    ``matvec`` / ``apply`` method of a captured object with (v) or (v, counter),
    returned as is.  Returns (object, method name, counter) or None."""
    import builtins
    import dis
    import types
    if not isinstance(fn, types.FunctionType) or fn.__code__.co_argcount != 1 or fn.__defaults__:
        return None
    code = fn.__code__
    cells = dict(zip(code.co_freevars, [c.cell_contents for c in (fn.__closure__ or ())]))

    def value(ins):
        if ins.opname == "LOAD_DEREF" and ins.argval in cells:
            return True, cells[ins.argval]
        if ins.opname == "LOAD_GLOBAL":
            g = fn.__globals__
            if ins.argval in g:
                return True, g[ins.argval]
            if hasattr(builtins, ins.argval):
                return True, getattr(builtins, ins.argval)
        return False, None

    try:
        ops = [i for i in dis.get_instructions(fn) if i.opname not in _SKIP_OPS]
    except Exception:  # noqa: BLE001
        return None
    if len(ops) not in (5, 6) or ops[-1].opname != "RETURN_VALUE" or not ops[-2].opname.startswith("CALL"):
        return None
    ok, obj = value(ops[0])
    if not ok or ops[1].opname not in ("LOAD_ATTR", "LOAD_METHOD") or ops[1].argval not in ("matvec", "apply"):
        return None
    if ops[2].opname != "LOAD_FAST" or ops[2].argval != code.co_varnames[0]:
        return None
    counter = None
    if len(ops) == 6:
        ok, counter = value(ops[3])
        if not ok:
            return None
    nargs = ops[-2].arg
    if nargs != len(ops) - 4:
        return None
    from .blocks import OpCounter
    if counter is not None and not isinstance(counter, OpCounter):
        return None
    if not hasattr(obj, "native_linop") or not hasattr(obj, "_charge"):
        return None
    return obj, ops[1].argval, counter


def charge_gmres(op_obj, op_counter, pre_obj, pre_counter, stats: "GmresStats", restart, max_iters):
    """Counter increments the reference's gmres makes through its operator
    wrappers (krylov.py:37-130): P^-1 b and P^-1 (b - B x0) (1 matvec, 2 applies),
    one of each per iteration, one of each per finished cycle (restart residual),
    and the final true residual (1 matvec).  A zero rhs touches nothing."""
    if stats.operator_applies == 0 and stats.iterations == 0 and stats.converged:
        return
    k = stats.iterations
    R = restart or max_iters
    cycles = (k + R - 1) // R if k > 0 else 0
    for obj, ctr, times in ((op_obj, op_counter, 1 + k + cycles + 1), (pre_obj, pre_counter, 2 + k + cycles)):
        if obj is None or ctr is None or times <= 0:
            continue
        from .blocks import OpCounter
        one = OpCounter()
        obj._charge(one)
        for key, v in one.snapshot().items():
            setattr(ctr, key, getattr(ctr, key) + times * v)


def _native(fn):
    """Native linop for a bound method of a device object, else None."""
    owner = getattr(fn, "__self__", None)
    name = getattr(getattr(fn, "__func__", None), "__name__", "")
    if owner is not None and name in ("matvec", "apply") and hasattr(owner, "native_linop"):
        return owner.native_linop()
    if hasattr(fn, "native_linop"):
        return fn.native_linop()
    return None


class _Callback:
    """Python callable exposed to the native loop as an irk_apply_fn."""

    def __init__(self, fn, n):
        self.fn, self.n, self.exc = fn, n, None

        def cb(user, in_p, out_p, stream):
            try:
                xin = L.wrap_device(in_p, self.n)
                out = L.wrap_device(out_p, self.n)
                r = self.fn(xin)
                r, _ = to_device(r)
                out.copy_(r.reshape(-1))
                return 0
            except BaseException as e:  # noqa: BLE001 -- re-raised after the native call
                self.exc = e
                return 1

        self.cfunc = L.APPLY_FN(cb)

    def linop(self):
        op = L.Linop()
        op.fn = ctypes.cast(self.cfunc, ctypes.c_void_p).value
        op.user = None
        return op


def _linop(fn, n, keep):
    if fn is None:
        return L.Linop()
    nat = _native(fn)
    if nat is not None:
        keep.append(nat)
        return nat[0]
    cb = _Callback(fn, n)
    keep.append(cb)
    return cb.linop()


def gmres_device(apply_operator, apply_precond, rhs, cfg: GmresConfig, allreduce=None, x=None,
                 native_allreduce=None):
    """Run the native loop on a CUDA-tensor rhs; returns (x, GmresStats).
    ``allreduce``: Python callable summing a CUDA tensor across ranks in place;
    ``native_allreduce``: (irk_allreduce_fn address, user pointer), e.g.
    ``irk_comm_allreduce`` with an ``irk_comm`` (no Python in the loop)."""
    t = L.torch()
    n = rhs.numel()
    keep: list = []
    op = _linop(apply_operator, n, keep)
    pre = _linop(apply_precond, n, keep)
    if op.fn is None:
        raise ValueError("apply_operator is required")
    if x is None:
        x = t.empty(n, dtype=t.float64, device="cuda")
    restart = cfg.restart or cfg.max_iters
    eta = getattr(cfg, "reorth_eta", 0.7071067811865476)   # reference GmresConfig has none
    ccfg = L.GmresCfg(cfg.rel_tol, cfg.max_iters, min(restart, cfg.max_iters), eta)
    st = L.GmresStatsC()
    hist = np.zeros(cfg.max_iters + 2)
    ar_fn, ar_user = None, None
    if native_allreduce is not None:
        ar_fn, ar_user = native_allreduce
    elif allreduce is not None:
        def _ar(user, buf, count, stream):
            try:
                allreduce(L.wrap_device(buf, count))
                return 0
            except BaseException as e:  # noqa: BLE001
                keep.append(e)
                return 1
        ar_c = L.ALLREDUCE_FN(_ar)
        keep.append(ar_c)
        ar_fn = ctypes.cast(ar_c, ctypes.c_void_p).value
    rc = L.lib().irk_gmres(L.ctx(), n, op, pre, ar_fn, ar_user, rhs.data_ptr(), x.data_ptr(),
                           ctypes.byref(ccfg), ctypes.byref(st), hist.ctypes.data, len(hist),
                           L.stream_ptr())
    for k in keep:
        if isinstance(k, _Callback) and k.exc is not None:
            raise k.exc
        if isinstance(k, BaseException):
            raise k
    L.check(rc, "irk_gmres")
    stats = GmresStats(iterations=st.iterations, operator_applies=st.operator_applies,
                       residual_history=[float(v) for v in hist[:min(st.history_len, len(hist))]],
                       converged=bool(st.converged),
                       final_true_residual=float(st.final_true_residual),
                       reorth_passes=st.reorth_passes, b_norm=float(st.b_norm))
    return x, stats


def gmres(apply_operator, apply_precond, rhs, cfg: GmresConfig | None = None):
    """Left-preconditioned GMRES (krylov.py:37-130); right preconditioning via
    the reference's reduction to a left solve (krylov.py:133-150)."""
    cfg = cfg or GmresConfig()
    rd, was_np = to_device(rhs)
    rd = rd.reshape(-1)
    if not getattr(cfg, "left_precondition", True):
        inner = GmresConfig(rel_tol=cfg.rel_tol, max_iters=cfg.max_iters, restart=cfg.restart,
                            left_precondition=True,
                            reorth_eta=getattr(cfg, "reorth_eta", 0.7071067811865476))
        pre = apply_precond if apply_precond is not None else (lambda v: v)
        u, stats = gmres_device(lambda v: apply_operator(pre(v)), None, rd, inner)
        x, _ = to_device(pre(u))
        r, _ = to_device(apply_operator(x))
        stats.final_true_residual = float(L.torch().linalg.vector_norm(rd - r))
        return from_device(x, was_np), stats
    # the reference's wrappers around this package's device objects (install_stepper):
    # run the native loop on the objects themselves and charge the wrapped counters
    # exactly as the wrappers would have been called
    cop = closure_call(apply_operator)
    cpre = closure_call(apply_precond) if apply_precond is not None else None
    if cop is not None and cop[1] == "matvec" and (apply_precond is None or (cpre is not None and cpre[1] == "apply")):
        x, stats = gmres_device(cop[0].matvec, None if cpre is None else cpre[0].apply, rd, cfg)
        charge_gmres(cop[0], cop[2], None if cpre is None else cpre[0], None if cpre is None else cpre[2],
                     stats, cfg.restart, cfg.max_iters)
        return from_device(x, was_np), stats
    x, stats = gmres_device(apply_operator, apply_precond, rd, cfg)
    return from_device(x, was_np), stats
