"""Seeded synthetic inputs for the BASELINE configurations.

BASELINE.json names no dataset: meshes, Jacobians, mass matrices and
right-hand sides are generated here.  Values are
drawn in fixed element-row chunks, each chunk with its own seeded
``numpy.random.Generator``, so any contiguous element range (a GPU slab)
can be generated independently and bit-identically.

Value model (BASELINE.json configs[0]):
* J off-diagonal neighbour blocks i.i.d. N(0, sigma^2); diagonal blocks
  -(2I + N(0, sigma^2)).  ``jstd="nb"`` reads "N(0, 1/nb)" as sigma = 1/nb
  (SURVEY.md 8d recommendation: the solves converge in 4-9 iterations);
  ``jstd="sqrtnb"`` is the variance reading sigma = 1/sqrt(nb).
* M block-diagonal SPD, Q_e diag(U[0.5, 1.5]) Q_e^T with an independent
  seeded orthogonal Q_e per element (QR of a Gaussian matrix, sign-fixed).
* RHS N(0, 1).  dt = target / ||J||_2 (power iteration on J^T J).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .meshes import ElementGraph, build_mesh, mesh_table
from .tableau import builtin_tableau, derive

CHUNK = 256  # elements per RNG chunk


@dataclass
class Pattern:
    """CSR-of-blocks pattern: same arrays as the reference ``BlockSparseMatrix``
    (blocks.py:59-74): sorted columns per row with the diagonal included."""

    T: int
    indptr: np.ndarray
    indices: np.ndarray
    diag_pos: np.ndarray

    @property
    def nnzb(self) -> int:
        return int(self.indptr[-1])

    @classmethod
    def from_graph(cls, graph: ElementGraph) -> "Pattern":
        T = graph.num_elements
        degs = np.array([len(a) for a in graph.adjacency], dtype=np.int64)
        if T and np.all(degs == degs[0]):
            r = int(degs[0])
            table = np.array(graph.adjacency, dtype=np.int64).reshape(T, r)
            return cls.from_table(table)
        indptr = np.zeros(T + 1, dtype=np.int64)
        cols = []
        diag_pos = np.zeros(T, dtype=np.int64)
        for i in range(T):
            row = sorted(list(graph.adjacency[i]) + [i])
            diag_pos[i] = len(cols) + row.index(i)
            cols.extend(row)
            indptr[i + 1] = len(cols)
        return cls(T, indptr, np.array(cols, dtype=np.int64), diag_pos)

    @classmethod
    def from_table(cls, table: np.ndarray) -> "Pattern":
        T, r = table.shape
        rows = np.concatenate([table, np.arange(T)[:, None]], axis=1)
        rows.sort(axis=1)
        indptr = np.arange(T + 1, dtype=np.int64) * (r + 1)
        diag_pos = indptr[:-1] + np.argmax(rows == np.arange(T)[:, None], axis=1)
        return cls(T, indptr, rows.ravel().astype(np.int64), diag_pos.astype(np.int64))


def _chunks(T: int, lo: int = 0, hi: int | None = None):
    hi = T if hi is None else hi
    for c in range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK):
        a, b = c * CHUNK, min((c + 1) * CHUNK, T)
        yield c, max(a, lo), min(b, hi), a


def jacobian_blocks(pat: Pattern, nb: int, seed: int, jstd: str = "nb",
                    rows: tuple[int, int] | None = None) -> np.ndarray:
    """Synthetic J on ``pat`` for element rows [lo, hi) -> (nnzb_rows, nb, nb)."""
    sigma = 1.0 / nb if jstd == "nb" else 1.0 / np.sqrt(nb)
    lo, hi = rows if rows is not None else (0, pat.T)
    out = np.empty((int(pat.indptr[hi] - pat.indptr[lo]), nb, nb))
    base = int(pat.indptr[lo])
    eye2 = 2.0 * np.eye(nb)
    for c, a, b, c0 in _chunks(pat.T, lo, hi):
        rng = np.random.default_rng([seed, 0x4A, c])
        k0, k1 = int(pat.indptr[c0]), int(pat.indptr[min(c0 + CHUNK, pat.T)])
        vals = rng.standard_normal((k1 - k0, nb, nb))
        vals *= sigma
        d = pat.diag_pos[c0:min(c0 + CHUNK, pat.T)] - k0
        vals[d] = -(eye2 + vals[d])
        s0, s1 = int(pat.indptr[a]) - k0, int(pat.indptr[b]) - k0
        out[int(pat.indptr[a]) - base:int(pat.indptr[b]) - base] = vals[s0:s1]
    return out


def mass_blocks(T: int, nb: int, seed: int,
                rows: tuple[int, int] | None = None) -> np.ndarray:
    """SPD blocks Q diag(U[0.5,1.5]) Q^T for elements [lo, hi)."""
    lo, hi = rows if rows is not None else (0, T)
    out = np.empty((hi - lo, nb, nb))
    for c, a, b, c0 in _chunks(T, lo, hi):
        rng = np.random.default_rng([seed, 0x4D, c])
        n = min(c0 + CHUNK, T) - c0
        g = rng.standard_normal((n, nb, nb))
        lam = rng.uniform(0.5, 1.5, size=(n, nb))
        q, r = np.linalg.qr(g)
        q *= np.sign(np.diagonal(r, axis1=1, axis2=2))[:, None, :]
        blk = np.einsum("tij,tj,tkj->tik", q, lam, q)
        out[a - lo:b - lo] = blk[a - c0:b - c0]
    return out


def rhs_vector(s: int, T: int, nb: int, seed: int,
               rows: tuple[int, int] | None = None) -> np.ndarray:
    """N(0,1) stage-major right-hand side restricted to elements [lo, hi)."""
    lo, hi = rows if rows is not None else (0, T)
    out = np.empty((s, hi - lo, nb))
    for k in range(s):
        for c, a, b, c0 in _chunks(T, lo, hi):
            rng = np.random.default_rng([seed, 0x52, k, c])
            n = min(c0 + CHUNK, T) - c0
            v = rng.standard_normal((n, nb))
            out[k, a - lo:b - lo] = v[a - c0:b - c0]
    return out.reshape(-1)


def norm2_power_cpu(pat: Pattern, data: np.ndarray, iters: int = 60,
                    seed: int = 7) -> float:
    """||J||_2 by power iteration on J^T J (scipy BSR; small meshes only)."""
    import scipy.sparse as sp

    nb = data.shape[1]
    n = pat.T * nb
    A = sp.bsr_matrix((data, pat.indices, pat.indptr), shape=(n, n))
    At = A.T.tocsr()
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(iters):
        w = At @ (A @ v)
        lam = float(np.linalg.norm(w))
        v = w / lam
    return float(np.sqrt(lam))


@dataclass
class SolveConfig:
    """One BASELINE solve-level configuration (BASELINE.json configs)."""

    name: str
    mesh: str            # "tri2d" | "tet3d"
    N: int               # cells per side
    nb: int
    scheme: str          # RADAU23 / RADAU35 / DIRK33
    precond: str         # coupled | uncoupled | uncoupled-unshifted | block-jacobi | none
    restart: int
    rtol: float = 1e-8
    dt_norm: float = 100.0   # target dt * ||J||_2
    ordering: str = "natural"
    jstd: str = "nb"
    seed: int = 1701
    max_iters: int = 500
    extra: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return 2 * self.N ** 2 if self.mesh == "tri2d" else 6 * self.N ** 3

    @property
    def s(self) -> int:
        return builtin_tableau(self.scheme).s

    def scaled(self, **kw) -> "SolveConfig":
        d = dict(self.__dict__)
        d.update(kw)
        return SolveConfig(**d)


CONFIGS = {
    0: SolveConfig("cfg0", "tri2d", 16, 24, "RADAU23", "coupled", 30, dt_norm=20.0),
    1: SolveConfig("cfg1", "tri2d", 128, 40, "RADAU35", "uncoupled", 40, dt_norm=100.0),
    2: SolveConfig("cfg2", "tet3d", 32, 50, "RADAU35", "uncoupled", 40, dt_norm=100.0),
}


@dataclass
class Workload:
    cfg: SolveConfig
    table: np.ndarray
    pattern: Pattern
    J: np.ndarray
    M: np.ndarray
    rhs: np.ndarray
    a_inv: np.ndarray
    shifts: np.ndarray
    jnorm: float
    dt: float

    @property
    def graph(self) -> ElementGraph:
        return ElementGraph(num_elements=self.pattern.T,
                            adjacency=[list(map(int, r)) for r in self.table],
                            periodic=True, validate=False)


def relabel(table: np.ndarray, J: np.ndarray, M: np.ndarray, rhs: np.ndarray, s: int,
            new_of_old: np.ndarray):
    """The same block system under an element renumbering: returns the new
    neighbour table, pattern and (J, M, rhs) with block (i', j') = old block
    (old(i'), old(j')).  Numbering changes the ILU(0) factors, not B."""
    from .meshes import renumber_table
    T = table.shape[0]
    old_pat = Pattern.from_table(table)
    new_table = np.sort(renumber_table(table, new_of_old), axis=1)
    new_pat = Pattern.from_table(new_table)
    old_of_new = np.empty(T, dtype=np.int64)
    old_of_new[new_of_old] = np.arange(T)
    old_rows = np.repeat(np.arange(T), np.diff(old_pat.indptr))
    old_keys = old_rows * T + old_pat.indices
    new_rows = np.repeat(np.arange(T), np.diff(new_pat.indptr))
    want = old_of_new[new_rows] * T + old_of_new[new_pat.indices]
    pos = np.searchsorted(old_keys, want)
    assert np.array_equal(old_keys[pos], want)
    nb = J.shape[1]
    rhs_new = rhs.reshape(s, T, nb)[:, old_of_new].reshape(-1)
    return new_table, new_pat, J[pos], M[old_of_new], rhs_new


def make_workload(cfg: SolveConfig, jnorm: float | None = None,
                  norm_iters: int = 60) -> Workload:
    """Full single-process workload on the host (small/medium sizes).  Values
    are drawn in natural element order; ``ordering="color"`` relabels the same
    system colour-major."""
    from .meshes import color_major_permutation
    table = mesh_table(cfg.mesh, cfg.N, "natural")
    pat = Pattern.from_table(table)
    J = jacobian_blocks(pat, cfg.nb, cfg.seed, cfg.jstd)
    M = mass_blocks(pat.T, cfg.nb, cfg.seed)
    tab = builtin_tableau(cfg.scheme)
    der = derive(tab)
    s = tab.s
    rhs = rhs_vector(s, pat.T, cfg.nb, cfg.seed)
    if cfg.ordering == "color":
        from .meshes import slab_color_permutation
        parts = int(cfg.extra.get("parts", 1))
        table, pat, J, M, rhs = relabel(table, J, M, rhs, s, slab_color_permutation(table, parts))
    elif cfg.ordering != "natural":
        raise ValueError(f"unknown ordering {cfg.ordering!r}")
    if jnorm is None:
        jnorm = norm2_power_cpu(pat, J, iters=norm_iters)
    dt = cfg.dt_norm / jnorm
    return Workload(cfg, table, pat, J, M, rhs, der.a_inv, der.shifts, jnorm, dt)


def make_slab_workload(cfg: SolveConfig, P: int, rank: int):
    """Rank-local inputs for the element-partitioned solve: the global pattern
    (numbering per ``cfg.ordering``; colour ordering is applied inside each of
    the P slabs) plus only this rank's J rows, M blocks and rhs rows.  Values are
    generated for the rank's natural slab only (chunked generators), so no rank
    materialises the global matrix."""
    from .meshes import partition_bounds, renumber_table, slab_color_permutation
    table = mesh_table(cfg.mesh, cfg.N, "natural")
    T = table.shape[0]
    b = partition_bounds(T, P)
    lo, hi = int(b[rank]), int(b[rank + 1])
    nat = Pattern.from_table(table)
    s = builtin_tableau(cfg.scheme).s
    Jn = jacobian_blocks(nat, cfg.nb, cfg.seed, cfg.jstd, rows=(lo, hi))
    Mn = mass_blocks(T, cfg.nb, cfg.seed, rows=(lo, hi))
    rn = rhs_vector(s, T, cfg.nb, cfg.seed, rows=(lo, hi)).reshape(s, hi - lo, cfg.nb)
    if cfg.ordering == "color":
        new_of_old = slab_color_permutation(table, P)
    else:
        new_of_old = np.arange(T, dtype=np.int64)
    old_of_new = np.empty(T, dtype=np.int64)
    old_of_new[new_of_old] = np.arange(T)
    new_table = np.sort(renumber_table(table, new_of_old), axis=1)
    pat = Pattern.from_table(new_table)
    # local rows lo..hi of the new numbering are old rows of the same slab
    q0, q1 = int(pat.indptr[lo]), int(pat.indptr[hi])
    new_rows = np.repeat(np.arange(lo, hi), np.diff(pat.indptr[lo:hi + 1]))
    want = old_of_new[new_rows] * T + old_of_new[pat.indices[q0:q1]]
    oq0 = int(nat.indptr[lo])
    old_rows = np.repeat(np.arange(lo, hi), np.diff(nat.indptr[lo:hi + 1]))
    old_keys = old_rows * T + nat.indices[oq0:int(nat.indptr[hi])]
    pos = np.searchsorted(old_keys, want)
    J = Jn[pos]
    loc_old = old_of_new[lo:hi] - lo
    M = Mn[loc_old]
    rhs = np.ascontiguousarray(rn[:, loc_old]).reshape(-1)
    return pat, J, M, rhs
