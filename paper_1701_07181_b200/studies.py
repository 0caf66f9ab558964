"""Operation-count accounting and solver studies on the GPU path.

``cost_report`` is reference ``studies.py:261-353`` run on this package's
device objects: every operator / preconditioner variant is applied once with
an ``OpCounter`` and the measured block-operation counts are set against the
reference's exact predictions and its closed-form (s, r, T) model -- the
paper's Table 2-4 accounting -- so a user can check that the GPU
path does exactly the work the reference counts.  The untransformed operator
(``UntransformedOperator``) is not on the hot path and is not built here; its
two rows are reported from the reference's formulas with ``measured = None``.

``run_partition_study`` / ``run_precond_study`` mirror ``studies.py:175-242``
on the device ``integrate`` (linear problems, ``stepper.LinearProblem``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .blocks import OpCounter
from .krylov import GmresConfig
from .precond import build_stage_matrix, ilu0_factorize, stage_coupled_factorize, stage_uncoupled_factorize
from .stage_system import StageOperator
from .stepper import NewtonConfig, NewtonError, PrecondSpec, integrate
from .tableau import Tableau, builtin_tableau, derive


@dataclass
class CostRow:
    operation: str
    measured: int | None
    predicted: int          # structurally exact count for the implemented algorithm
    model: int | None       # closed-form cost-model value (None when not modeled)

    @property
    def match(self) -> bool:
        return self.measured == self.predicted

    @property
    def model_match(self) -> bool | None:
        return None if self.model is None or self.measured is None else self.measured == self.model


@dataclass
class StudyRecord:
    scheme: str
    precond: str
    partitions: int | None
    dt: float
    gmres_iters_avg: float
    equivalent_mults_avg: float
    newton_iters_avg: float
    counters: dict
    wall_time: float
    converged: bool = True

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def _uniform_degree(pattern):
    indptr = np.asarray(pattern.indptr)
    T = len(indptr) - 1
    edges = int(indptr[-1]) - T
    if edges % T:
        raise ValueError("cost model requires a uniform-degree mesh")
    return T, edges // T


def cost_report(problem, scheme, dt: float = 0.1) -> list:
    """Measured block-operation counts of one apply / factorisation of every
    operator variant vs exact predictions and the closed-form model
    (reference studies.py:261-353)."""
    tab = scheme if isinstance(scheme, Tableau) else builtin_tableau(scheme)
    der = derive(tab)
    s = tab.s
    pat = problem.pattern
    T, r = _uniform_degree(pat)
    nnzb = pat.nnzb
    upper = pat.upper_count(np.ones(nnzb, bool))
    mass = problem.mass()
    jac = problem.jacobian(0.0, None)
    op = StageOperator(der, dt, mass, [jac] * s)
    rng = np.random.default_rng(12345)
    w = rng.standard_normal(op.total_dim)
    rows = []
    c = OpCounter()
    op.matvec(w, c)
    rows.append(CostRow("transformed-matvec jacobian products", c.jacobian_multiplies, s * nnzb, s * (r + 1) * T))
    rows.append(CostRow("transformed-matvec mass products", c.mass_multiplies, s * s * T, (s * s - s) * T))
    rows.append(CostRow("untransformed-matvec jacobian products", None, s * s * nnzb, s * s * (r + 1) * T))
    rows.append(CostRow("untransformed-matvec mass products", None, s * T, None))
    dirk_mat = build_stage_matrix(1.0, mass, jac, dt)
    c = OpCounter()
    dirk_mat.matvec(w[:dirk_mat.n], c)
    rows.append(CostRow("dirk-matvec block products", c.block_multiplies, nnzb, (r + 1) * T))
    c = OpCounter()
    coupled = stage_coupled_factorize(op, c)
    rows.append(CostRow("coupled-factorize block LU", c.block_factorizations, s * T, s * T))
    rows.append(CostRow("coupled-factorize block products", c.block_multiplies,
                        2 * s * upper + (s * s - s) * T, s * (r + s) * T))
    c = OpCounter()
    coupled.apply(w, c)
    rows.append(CostRow("coupled-apply block products", c.block_multiplies,
                        s * (nnzb - T) + (s * s - s) * T + s * T, s * (r + s) * T))
    c = OpCounter()
    uncoupled = stage_uncoupled_factorize(op, der.shifts, c)
    rows.append(CostRow("uncoupled-factorize block LU", c.block_factorizations, s * T, s * T))
    rows.append(CostRow("uncoupled-factorize block products", c.block_multiplies, 2 * s * upper, s * r * T))
    c = OpCounter()
    uncoupled.apply(w, c)
    rows.append(CostRow("uncoupled-apply block products", c.block_multiplies, s * nnzb, s * (r + 1) * T))
    c = OpCounter()
    dirk_fac = ilu0_factorize(dirk_mat, c)
    rows.append(CostRow("dirk-factorize block LU", c.block_factorizations, T, T))
    rows.append(CostRow("dirk-factorize block products", c.block_multiplies, 2 * upper, r * T))
    c = OpCounter()
    dirk_fac.apply(w[:dirk_mat.n], c)
    rows.append(CostRow("dirk-apply block products", c.block_multiplies, nnzb, (r + 1) * T))
    rows.append(CostRow("memory blocks: stage Jacobians", s * nnzb, s * nnzb, s * (r + 1) * T))
    rows.append(CostRow("memory blocks: coupled preconditioner", coupled.memory_blocks(),
                        s * nnzb + (s * s - s) * T, s * (r + s) * T))
    rows.append(CostRow("memory blocks: uncoupled preconditioner", uncoupled.memory_blocks(),
                        s * nnzb, s * (r + 1) * T))
    rows.append(CostRow("memory blocks: dirk preconditioner", nnzb, nnzb, (r + 1) * T))
    return rows


def _record(res, scheme, precond, partitions, dt, wall, converged=True) -> StudyRecord:
    return StudyRecord(scheme=scheme, precond=precond, partitions=partitions, dt=dt,
                       gmres_iters_avg=res.gmres_iters_avg, equivalent_mults_avg=res.equivalent_mults_avg,
                       newton_iters_avg=res.newton_iters_avg, counters=res.counter.snapshot(),
                       wall_time=wall, converged=converged)


def _failed(scheme, precond, partitions, dt, wall) -> StudyRecord:
    nan = float("nan")
    return StudyRecord(scheme=scheme, precond=precond, partitions=partitions, dt=dt, gmres_iters_avg=nan,
                       equivalent_mults_avg=nan, newton_iters_avg=nan, counters={}, wall_time=wall,
                       converged=False)


def run_precond_study(problem, schemes, dts, preconds, num_steps: int = 5, t0: float = 0.0,
                      newton_cfg: NewtonConfig | None = None, gmres_cfg: GmresConfig | None = None,
                      u0=None) -> list:
    """One record per (scheme, preconditioner kind, dt), fixed step count
    (reference studies.py:175-201)."""
    records = []
    for scheme in schemes:
        name = scheme if isinstance(scheme, str) else scheme.name
        for kind in preconds:
            for dt in dts:
                start = time.perf_counter()
                try:
                    res = integrate(problem, scheme, t0, t0 + num_steps * dt, dt, PrecondSpec(kind=kind),
                                    newton_cfg, gmres_cfg, keep_trajectory=False, u0=u0)
                    records.append(_record(res, name, kind, None, dt, time.perf_counter() - start))
                except NewtonError:
                    records.append(_failed(name, kind, None, dt, time.perf_counter() - start))
    return records


def run_partition_study(problem, scheme, dt: float, partition_counts, stage_parallel: bool = False,
                        precond_kind: str = "uncoupled", num_steps: int = 5, t0: float = 0.0,
                        newton_cfg: NewtonConfig | None = None, gmres_cfg: GmresConfig | None = None,
                        u0=None) -> list:
    """GMRES iterations vs partition count P (reference studies.py:204-242): the
    partitioned block ILU(0) drops cross-partition blocks; with ``stage_parallel``
    P workers leave P / s partitions."""
    tab = scheme if isinstance(scheme, Tableau) else builtin_tableau(scheme)
    T = problem.pattern.T
    records = []
    for P in partition_counts:
        if P < 1 or P > T:
            raise ValueError(f"partition count {P} outside [1, {T}]")
        if stage_parallel:
            if P % tab.s != 0:
                raise ValueError(f"worker count {P} not divisible by stage count {tab.s}")
            spec = PrecondSpec(kind=precond_kind, partitions=P // tab.s, stage_parallel=True)
        else:
            spec = PrecondSpec(kind=precond_kind, partitions=P)
        start = time.perf_counter()
        try:
            res = integrate(problem, tab, t0, t0 + num_steps * dt, dt, precond=spec, newton_cfg=newton_cfg,
                            gmres_cfg=gmres_cfg, keep_trajectory=False, u0=u0)
            records.append(_record(res, tab.name, precond_kind, P, dt, time.perf_counter() - start))
        except NewtonError:
            records.append(_failed(tab.name, precond_kind, P, dt, time.perf_counter() - start))
    return records
