"""Element graphs for the synthetic DG workloads.

Mirrors the reference's ``ElementGraph`` contract
(``/root/reference/pkg/src/irksolve/meshing.py:10-52``): a symmetric
adjacency without self loops, plus a ``partition_of`` map used to drop
cross-partition blocks from the factorization.  The reference only builds
1D line meshes (``meshing.py:55-73``); the 2D periodic triangle grid and the
3D periodic Kuhn-tetrahedron grid of BASELINE configs 0-2 are built here
(SURVEY.md section 8d gives the neighbour rules).

Element numbering is part of the input: the ILU(0) factors depend on it.
``ordering="natural"`` numbers elements cell by cell (z-major in 3D, so
contiguous index ranges are slabs); ``ordering="color"`` renumbers a
bipartite graph colour-major (all colour-0 elements first, natural order
inside each colour), which turns the ILU dependency DAG into two levels.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import permutations

import numpy as np


@dataclass
class ElementGraph:
    """Symmetric element adjacency; same fields as the reference type.

    ``adjacency`` is a list of sorted neighbour lists.  ``nbr`` optionally
    caches a dense (T, r) neighbour table for regular graphs (fast paths).
    """

    num_elements: int
    adjacency: list
    periodic: bool = False
    partition_of: np.ndarray = field(default=None)
    validate: bool = True

    def __post_init__(self):
        if self.partition_of is None:
            self.partition_of = np.zeros(self.num_elements, dtype=np.int64)
        if self.validate:
            # reference: meshing.py:22-30 (self-loop + symmetry check)
            adj_sets = [set(a) for a in self.adjacency]
            for i, nbrs in enumerate(self.adjacency):
                for j in nbrs:
                    if j == i:
                        raise ValueError(f"self-loop at element {i}")
                    if i not in adj_sets[j]:
                        raise ValueError(f"asymmetric adjacency: {i} -> {j}")

    @property
    def num_partitions(self) -> int:
        return int(self.partition_of.max()) + 1

    def degree(self, i: int) -> int:
        return len(self.adjacency[i])

    def num_blocks(self) -> int:
        return self.num_elements + sum(len(a) for a in self.adjacency)

    def satisfies_simplified_ilu_condition(self) -> bool:
        """True iff no two neighbours of any element are neighbours
        (reference: meshing.py:43-52)."""
        adj_sets = [set(a) for a in self.adjacency]
        for i in range(self.num_elements):
            nbrs = self.adjacency[i]
            for a in range(len(nbrs)):
                for b in range(a + 1, len(nbrs)):
                    if nbrs[b] in adj_sets[nbrs[a]]:
                        return False
        return True


def _from_table(nbr: np.ndarray, periodic: bool, validate: bool) -> ElementGraph:
    nbr = np.sort(nbr, axis=1)
    adjacency = [list(map(int, row)) for row in nbr]
    return ElementGraph(num_elements=len(adjacency), adjacency=adjacency,
                        periodic=periodic, validate=validate)


def line_mesh(T: int, periodic: bool = False) -> ElementGraph:
    """1D line; same contract as reference ``build_line_mesh`` (meshing.py:55-73)."""
    if T < 2:
        raise ValueError(f"need at least 2 elements, got {T}")
    if periodic and T < 4:
        raise ValueError(
            f"periodic line with T={T} violates the simplified-ILU neighbor condition")
    adjacency = []
    for i in range(T):
        if periodic:
            nbrs = sorted({(i - 1) % T, (i + 1) % T})
        else:
            nbrs = [j for j in (i - 1, i + 1) if 0 <= j < T]
        adjacency.append(nbrs)
    return ElementGraph(num_elements=T, adjacency=adjacency, periodic=periodic)


def tri2d_table(N: int) -> np.ndarray:
    """(2N^2, 3) neighbour table of the periodic N x N quad grid, each quad
    split into a lower-right triangle L(q)=2q and an upper-left U(q)=2q+1,
    q = iy*N + ix.  L(q) <-> {U(q), U(ix, iy-1), U(ix+1, iy)}."""
    if N < 2:
        raise ValueError("need N >= 2")
    iy, ix = np.divmod(np.arange(N * N), N)
    q = iy * N + ix
    below = ((iy - 1) % N) * N + ix
    right = iy * N + (ix + 1) % N
    above = ((iy + 1) % N) * N + ix
    left = iy * N + (ix - 1) % N
    nbr = np.empty((2 * N * N, 3), dtype=np.int64)
    nbr[2 * q] = np.stack([2 * q + 1, 2 * below + 1, 2 * right + 1], axis=1)
    nbr[2 * q + 1] = np.stack([2 * q, 2 * above, 2 * left], axis=1)
    return nbr


_PERMS = list(permutations(range(3)))          # local tet id -> axis order
_PERM_ID = {p: k for k, p in enumerate(_PERMS)}


def kuhn3d_table(N: int) -> np.ndarray:
    """(6N^3, 4) neighbour table of the periodic N^3 cube grid, each cube
    split into the 6 Kuhn tetrahedra {1 >= x_p0 >= x_p1 >= x_p2 >= 0}.
    Cube c = (iz*N + iy)*N + ix (z-major), element = 6c + local id.
    Facets: x_p0=x_p1 and x_p1=x_p2 are in-cube (swap neighbours); x_p0=1
    meets (p1,p2,p0) in cube +e_p0; x_p2=0 meets (p2,p0,p1) in cube -e_p2."""
    if N < 2:
        raise ValueError("need N >= 2")
    c = np.arange(N ** 3)
    iz, rem = np.divmod(c, N * N)
    iy, ix = np.divmod(rem, N)
    coords = [ix, iy, iz]

    def cube_shift(axis, d):
        cc = [coords[0].copy(), coords[1].copy(), coords[2].copy()]
        cc[axis] = (cc[axis] + d) % N
        return (cc[2] * N + cc[1]) * N + cc[0]

    nbr = np.empty((6 * N ** 3, 4), dtype=np.int64)
    for k, p in enumerate(_PERMS):
        p0, p1, p2 = p
        e = 6 * c + k
        sw01 = _PERM_ID[(p1, p0, p2)]
        sw12 = _PERM_ID[(p0, p2, p1)]
        up = _PERM_ID[(p1, p2, p0)]
        dn = _PERM_ID[(p2, p0, p1)]
        nbr[e, 0] = 6 * c + sw01
        nbr[e, 1] = 6 * c + sw12
        nbr[e, 2] = 6 * cube_shift(p0, +1) + up
        nbr[e, 3] = 6 * cube_shift(p2, -1) + dn
    return nbr


def two_coloring(nbr: np.ndarray) -> np.ndarray:
    """BFS 2-colouring of a connected-or-not graph given as a neighbour
    table; raises if the graph is not bipartite."""
    T = nbr.shape[0]
    color = -np.ones(T, dtype=np.int64)
    for start in range(T):
        if color[start] >= 0:
            continue
        color[start] = 0
        frontier = np.array([start])
        while frontier.size:
            nb = nbr[frontier].ravel()
            want = np.repeat(1 - color[frontier], nbr.shape[1])
            bad = (color[nb] >= 0) & (color[nb] != want)
            if bad.any():
                raise ValueError("graph is not bipartite")
            new = color[nb] < 0
            color[nb[new]] = want[new]
            frontier = np.unique(nb[new])
    return color


def renumber_table(nbr: np.ndarray, new_of_old: np.ndarray) -> np.ndarray:
    """Apply an element renumbering to a neighbour table."""
    T = nbr.shape[0]
    old_of_new = np.empty(T, dtype=np.int64)
    old_of_new[new_of_old] = np.arange(T)
    return new_of_old[nbr[old_of_new]]


def color_major_permutation(nbr: np.ndarray) -> np.ndarray:
    """new index of each old element: colour 0 first, natural order inside."""
    color = two_coloring(nbr)
    order = np.argsort(color, kind="stable")          # old ids in new order
    new_of_old = np.empty_like(order)
    new_of_old[order] = np.arange(len(order))
    return new_of_old


def slab_color_permutation(nbr: np.ndarray, parts: int) -> np.ndarray:
    """new index of each old (natural) element: the natural order is cut into
    ``parts`` contiguous slabs (``partition``), and inside each slab elements
    are ordered colour-major (colour 0 first, natural order inside a colour).
    parts=1 is the global colour-major numbering."""
    color = two_coloring(nbr)
    T = nbr.shape[0]
    b = partition_bounds(T, parts)
    new_of_old = np.empty(T, dtype=np.int64)
    for p in range(parts):
        lo, hi = int(b[p]), int(b[p + 1])
        order = lo + np.argsort(color[lo:hi], kind="stable")
        new_of_old[order] = np.arange(lo, hi)
    return new_of_old


def mesh_table(kind: str, N: int, ordering: str = "natural", parts: int = 1) -> np.ndarray:
    if kind == "tri2d":
        nbr = tri2d_table(N)
    elif kind == "tet3d":
        nbr = kuhn3d_table(N)
    else:
        raise ValueError(f"unknown mesh kind {kind!r}")
    if ordering == "natural":
        return np.sort(nbr, axis=1)
    if ordering == "color":
        return np.sort(renumber_table(nbr, slab_color_permutation(nbr, parts)), axis=1)
    raise ValueError(f"unknown ordering {ordering!r}")


def build_mesh(kind: str, N: int, ordering: str = "natural",
               validate: bool = True) -> ElementGraph:
    return _from_table(mesh_table(kind, N, ordering), periodic=True, validate=validate)


def partition(graph: ElementGraph, P: int) -> ElementGraph:
    """Contiguous element ranges, sizes differing by <= 1; same rule as the
    reference ``partition`` (meshing.py:81-90, np.array_split)."""
    T = graph.num_elements
    if not 1 <= P <= T:
        raise ValueError(f"partition count {P} outside [1, {T}]")
    part = np.empty(T, dtype=np.int64)
    for p, chunk in enumerate(np.array_split(np.arange(T), P)):
        part[chunk] = p
    return ElementGraph(num_elements=T, adjacency=graph.adjacency,
                        periodic=graph.periodic, partition_of=part, validate=False)


def partition_bounds(T: int, P: int) -> np.ndarray:
    """Start offsets (P+1) of the contiguous ranges ``partition`` produces."""
    sizes = [len(c) for c in np.array_split(np.arange(T), P)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
