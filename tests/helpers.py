"""Shared test fixtures (restated from the reference test suite)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pattern_of(adjacency):
    """CSR-of-blocks arrays exactly as reference BlockSparseMatrix builds them
    (blocks.py:59-74)."""
    T = len(adjacency)
    indptr = np.zeros(T + 1, dtype=np.int64)
    cols, diag_pos = [], np.zeros(T, dtype=np.int64)
    for i in range(T):
        row = sorted(list(adjacency[i]) + [i])
        diag_pos[i] = len(cols) + row.index(i)
        cols.extend(row)
        indptr[i + 1] = len(cols)
    return indptr, np.array(cols, dtype=np.int64), diag_pos


def random_blocks(adjacency, m, seed=0, diag_boost=3.0):
    """Block data of reference ``random_matrix`` (tests/test_meshing_blocks.py:9-16):
    same draw order (diagonal first, then neighbours in adjacency order)."""
    indptr, indices, diag_pos = pattern_of(adjacency)
    rng = np.random.default_rng(seed)
    data = np.zeros((len(indices), m, m))
    for i in range(len(adjacency)):
        data[diag_pos[i]] = diag_boost * np.eye(m) + rng.standard_normal((m, m))
        for j in adjacency[i]:
            k = indptr[i] + int(np.searchsorted(indices[indptr[i]:indptr[i + 1]], j))
            data[k] = rng.standard_normal((m, m))
    return data


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den else 1.0))
