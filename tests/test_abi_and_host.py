"""CPU-only checks: the C-ABI library loads and exports every declared symbol;
host-side logic (meshes, patterns, generators, keep masks) is correct."""

import os
import re
import subprocess

import numpy as np
import pytest

from paper_1701_07181_b200 import workloads as W
from paper_1701_07181_b200.meshes import (build_mesh, color_major_permutation, line_mesh,
                                          mesh_table, partition, partition_bounds, two_coloring)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(REPO, "include", "irkb200.h")).read()
    return sorted(set(re.findall(r"IRK_API\s+[\w\s\*]*?\b(irk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1701_07181_b200 import _lib
    from paper_1701_07181_b200 import build as B
    B.build()
    lib = _lib.load()
    decl = declared_symbols()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (irk_\w+)", out))
    assert set(decl) <= exported
    assert lib.irk_version() >= 10000


def test_library_is_sm100a():
    from paper_1701_07181_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1701_07181_b200 import IrkError, _lib
    with pytest.raises(IrkError):
        _lib.ctx()


@pytest.mark.parametrize("kind,N,deg", [("tri2d", 4, 3), ("tri2d", 16, 3), ("tet3d", 3, 4),
                                        ("tet3d", 4, 4)])
def test_mesh_structure(kind, N, deg):
    g = build_mesh(kind, N)  # validates symmetry / self loops
    assert all(len(a) == deg for a in g.adjacency)
    assert all(len(set(a)) == deg for a in g.adjacency)
    assert g.satisfies_simplified_ilu_condition()
    if N % 2 == 0:
        c = two_coloring(np.array(g.adjacency))
        assert set(np.unique(c)) == {0, 1}


def test_color_ordering_is_relabeling():
    nat = mesh_table("tri2d", 8, "natural")
    col = mesh_table("tri2d", 8, "color")
    perm = color_major_permutation(nat)
    T = len(nat)
    # colour-major: first half only neighbours second half
    assert np.all(col[: T // 2] >= T // 2) and np.all(col[T // 2:] < T // 2)
    # same edge set under the permutation
    e1 = {(perm[i], perm[j]) for i in range(T) for j in nat[i]}
    e2 = {(i, int(j)) for i in range(T) for j in col[i]}
    assert e1 == e2


def test_pattern_matches_reference_construction():
    from tests.helpers import pattern_of
    g = build_mesh("tet3d", 3)
    p = W.Pattern.from_graph(g)
    ip, ix, dp = pattern_of(g.adjacency)
    np.testing.assert_array_equal(p.indptr, ip)
    np.testing.assert_array_equal(p.indices, ix)
    np.testing.assert_array_equal(p.diag_pos, dp)


def test_chunked_generation_is_partition_independent():
    cfg = W.CONFIGS[2].scaled(N=4, nb=6)
    table = mesh_table(cfg.mesh, cfg.N)
    pat = W.Pattern.from_table(table)
    full = W.jacobian_blocks(pat, cfg.nb, 5)
    lo, hi = 100, 300
    part = W.jacobian_blocks(pat, cfg.nb, 5, rows=(lo, hi))
    np.testing.assert_array_equal(part, full[pat.indptr[lo]:pat.indptr[hi]])
    M = W.mass_blocks(pat.T, cfg.nb, 5)
    np.testing.assert_array_equal(W.mass_blocks(pat.T, cfg.nb, 5, rows=(lo, hi)), M[lo:hi])
    r = W.rhs_vector(3, pat.T, cfg.nb, 5).reshape(3, pat.T, cfg.nb)
    np.testing.assert_array_equal(W.rhs_vector(3, pat.T, cfg.nb, 5, rows=(lo, hi)).reshape(3, -1, cfg.nb),
                                  r[:, lo:hi])
    # mass blocks are SPD with eigenvalues in [0.5, 1.5]
    ev = np.linalg.eigvalsh(M)
    assert ev.min() >= 0.5 - 1e-12 and ev.max() <= 1.5 + 1e-12


def test_partition_bounds_match_array_split():
    g = line_mesh(10, periodic=True)
    for P in (1, 2, 3, 4, 7):
        b = partition_bounds(10, P)
        part = partition(g, P).partition_of
        for p in range(P):
            assert np.all(part[b[p]:b[p + 1]] == p)


def test_simplified_condition_vectorised():
    from paper_1701_07181_b200.precond import simplified_condition
    from tests.helpers import pattern_of

    class Pat:
        def __init__(self, adj):
            self.indptr, self.indices, _ = pattern_of(adj)

    assert simplified_condition(Pat(build_mesh("tri2d", 4).adjacency))
    assert simplified_condition(Pat(line_mesh(6, periodic=True).adjacency))
    assert not simplified_condition(Pat([[1, 2], [0, 2], [0, 1]]))


def test_keep_mask_vectorised_matches_loop():
    from paper_1701_07181_b200.precond import partition_keep_mask
    g = partition(build_mesh("tet3d", 4), 4)
    p = W.Pattern.from_graph(g)
    keep = partition_keep_mask(p, g.partition_of)
    loop = np.ones(p.nnzb, bool)
    for i in range(p.T):
        for k in range(p.indptr[i], p.indptr[i + 1]):
            j = p.indices[k]
            if j != i and g.partition_of[i] != g.partition_of[j]:
                loop[k] = False
    np.testing.assert_array_equal(keep, loop)
