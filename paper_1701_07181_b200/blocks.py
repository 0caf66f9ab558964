"""Device-resident block storage mirroring the reference ``blocks.py``.

* ``OpCounter`` -- same fields and semantics as reference blocks.py:18-53
  (block-operation counters for cost-model reconciliation).
* ``DevicePattern`` -- the CSR-of-blocks pattern (reference
  BlockSparseMatrix.indptr/indices/diag_pos, blocks.py:59-74) uploaded once.
* ``BlockSparseMatrix`` / ``BlockDiagonalMatrix`` -- device-resident block
  arrays with the reference's ``matvec(x, counter=None)`` API; ``matvec``
  accepts a CUDA tensor (returns a CUDA tensor) or a numpy array (returns a
  numpy array, copying through the device).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass
class OpCounter:
    block_multiplies: int = 0
    block_solves: int = 0
    block_factorizations: int = 0
    mass_multiplies: int = 0
    jacobian_multiplies: int = 0

    def reset(self) -> None:
        self.block_multiplies = self.block_solves = self.block_factorizations = 0
        self.mass_multiplies = self.jacobian_multiplies = 0

    def merge(self, other: "OpCounter") -> None:
        self.block_multiplies += other.block_multiplies
        self.block_solves += other.block_solves
        self.block_factorizations += other.block_factorizations
        self.mass_multiplies += other.mass_multiplies
        self.jacobian_multiplies += other.jacobian_multiplies

    def snapshot(self) -> dict:
        return dict(block_multiplies=self.block_multiplies, block_solves=self.block_solves,
                    block_factorizations=self.block_factorizations,
                    mass_multiplies=self.mass_multiplies,
                    jacobian_multiplies=self.jacobian_multiplies)


def pattern_arrays(graph):
    """indptr/indices/diag_pos exactly as the reference builds them (blocks.py:59-74)."""
    T = graph.num_elements
    degs = np.fromiter((len(a) for a in graph.adjacency), dtype=np.int64, count=T)
    if T and np.all(degs == degs[0]) and degs[0] > 0:
        r = int(degs[0])
        table = np.asarray(graph.adjacency, dtype=np.int64).reshape(T, r)
        rows = np.concatenate([table, np.arange(T)[:, None]], axis=1)
        rows.sort(axis=1)
        indptr = np.arange(T + 1, dtype=np.int64) * (r + 1)
        diag = indptr[:-1] + np.argmax(rows == np.arange(T)[:, None], axis=1)
        return indptr, rows.ravel().astype(np.int64), diag.astype(np.int64)
    indptr = np.zeros(T + 1, dtype=np.int64)
    cols, diag = [], np.zeros(T, dtype=np.int64)
    for i in range(T):
        row = sorted(list(graph.adjacency[i]) + [i])
        diag[i] = len(cols) + row.index(i)
        cols.extend(row)
        indptr[i + 1] = len(cols)
    return indptr, np.array(cols, dtype=np.int64), diag


class DevicePattern:
    """A block pattern uploaded to the GPU (owns an ``irk_pattern``)."""

    def __init__(self, indptr, indices, diag_pos, graph=None, device=None):
        self.indptr = L.i64_host(indptr)
        self.indices = L.i64_host(indices)
        self.diag_pos = L.i64_host(diag_pos)
        self.T = len(self.indptr) - 1
        self.nnzb = int(self.indptr[-1])
        self.graph = graph
        self.ctx = L.ctx(device)
        h = ctypes.c_void_p()
        L.check(L.lib().irk_pattern_create(self.ctx, self.T, L.ptr(self.indptr), L.ptr(self.indices),
                                           L.ptr(self.diag_pos), ctypes.byref(h)),
                "irk_pattern_create")
        self.handle = h.value
        self._rows = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and L._lib is not None:
            L._lib.irk_pattern_destroy(h)
            self.handle = None

    @property
    def rows(self) -> np.ndarray:
        if self._rows is None:
            self._rows = np.repeat(np.arange(self.T), np.diff(self.indptr))
        return self._rows

    def upper_count(self, keep: np.ndarray | None = None) -> int:
        mask = self.indices > self.rows
        if keep is not None:
            mask &= keep.astype(bool)
        return int(mask.sum())


_PATTERNS: dict = {}


def pattern_for(obj) -> DevicePattern:
    """Device pattern of a graph / reference matrix, cached per graph object."""
    graph = getattr(obj, "graph", obj)
    key = id(graph)
    hit = _PATTERNS.get(key)
    if hit is not None and hit[0]() is graph:
        return hit[1]
    if hasattr(obj, "indptr") and hasattr(obj, "diag_pos"):
        arrays = (obj.indptr, obj.indices, obj.diag_pos)
    else:
        arrays = pattern_arrays(graph)
    pat = DevicePattern(*arrays, graph=graph)
    try:
        _PATTERNS[key] = (weakref.ref(graph), pat)
    except TypeError:  # graph not weak-referenceable: no caching
        pass
    return pat


class DeviceBlocks:
    """``count`` nb x nb fp64 blocks in the device layout (owns ``irk_blocks``)."""

    def __init__(self, nb: int, count: int, device=None):
        self.nb = int(nb)
        self.count = int(count)
        self.ctx = L.ctx(device)
        h = ctypes.c_void_p()
        L.check(L.lib().irk_blocks_create(self.ctx, self.nb, self.count, ctypes.byref(h)),
                "irk_blocks_create")
        self.handle = h.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and L._lib is not None:
            L._lib.irk_blocks_destroy(h)
            self.handle = None

    def upload(self, data, first: int = 0) -> "DeviceBlocks":
        """data: (k, nb, nb) row-major numpy array or CUDA tensor."""
        t = L.torch()
        if isinstance(data, t.Tensor):
            if not data.is_cuda:
                data = data.numpy()
            else:
                data = data.contiguous().to(t.float64)
                cnt = data.numel() // (self.nb * self.nb)
                L.check(L.lib().irk_blocks_upload(self.handle, first, cnt, data.data_ptr(), 1,
                                                  L.stream_ptr()), "irk_blocks_upload")
                return self
        arr = L.f64_host(data)
        cnt = arr.size // (self.nb * self.nb)
        L.check(L.lib().irk_blocks_upload(self.handle, first, cnt, arr.ctypes.data, 0,
                                          L.stream_ptr()), "irk_blocks_upload")
        return self

    def download(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.count - first if count is None else count
        out = np.empty((count, self.nb, self.nb))
        L.check(L.lib().irk_blocks_download(self.handle, first, count, out.ctypes.data, 0,
                                            L.stream_ptr()), "irk_blocks_download")
        return out

    @classmethod
    def from_host(cls, data) -> "DeviceBlocks":
        data = np.asarray(data)
        b = cls(data.shape[-1], data.size // (data.shape[-1] ** 2))
        return b.upload(data)


# ---------------------------------------------------------------------------
# vector helpers
# ---------------------------------------------------------------------------

def to_device(x):
    """(cuda tensor, was_numpy) for a numpy array or tensor."""
    t = L.torch()
    if isinstance(x, t.Tensor):
        if x.is_cuda:
            return x.contiguous().to(t.float64), False
        return x.to(t.float64).cuda(), True
    return t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda(), True


def from_device(y, was_numpy: bool):
    return y.cpu().numpy() if was_numpy else y


def empty_like_dev(n: int):
    t = L.torch()
    return t.empty(n, dtype=t.float64, device="cuda")


class _Op:
    """RAII wrapper of an ``irk_stage_op`` handle."""

    def __init__(self, handle, keepalive):
        self.handle = handle
        self.keepalive = keepalive

    def __del__(self):
        if self.handle and L._lib is not None:
            L._lib.irk_stage_op_destroy(self.handle)
            self.handle = None


def make_stage_op(pattern: DevicePattern, s: int, jblocks: list, jfirst: list, mass, mix,
                  alpha: float) -> _Op:
    arr = (ctypes.c_void_p * s)(*[b.handle for b in jblocks])
    jf = (ctypes.c_int64 * s)(*[int(f) for f in jfirst])
    mixarr = None if mix is None else np.ascontiguousarray(mix, dtype=np.float64).ravel()
    h = ctypes.c_void_p()
    L.check(L.lib().irk_stage_op_create(pattern.ctx, pattern.handle, s, arr, jf,
                                        mass.handle if mass is not None else None,
                                        L.ptr(mixarr), float(alpha), ctypes.byref(h)),
            "irk_stage_op_create")
    return _Op(h.value, (pattern, jblocks, mass, mixarr, arr, jf))


class BlockSparseMatrix:
    """T x T matrix of dense m x m blocks on an element-graph pattern, resident
    on the GPU (reference blocks.py:56-132)."""

    def __init__(self, pattern: DevicePattern, blocks: DeviceBlocks, first: int = 0,
                 host=None):
        self.pattern = pattern
        self.graph = pattern.graph
        self.m = blocks.nb
        self.blocks = blocks
        self.first = int(first)
        self.indptr, self.indices, self.diag_pos = pattern.indptr, pattern.indices, pattern.diag_pos
        self._host = host
        self._op = None

    @classmethod
    def from_host(cls, graph_or_pattern, data) -> "BlockSparseMatrix":
        pat = graph_or_pattern if isinstance(graph_or_pattern, DevicePattern) else pattern_for(graph_or_pattern)
        data = np.asarray(data)
        if data.shape != (pat.nnzb, data.shape[1], data.shape[1]):
            raise ValueError(f"expected ({pat.nnzb}, m, m) block data, got {data.shape}")
        return cls(pat, DeviceBlocks.from_host(data), host=data)

    @classmethod
    def from_reference(cls, mat) -> "BlockSparseMatrix":
        """Upload a reference ``irksolve.BlockSparseMatrix`` (host numpy)."""
        return cls(pattern_for(mat), DeviceBlocks.from_host(mat.data), host=mat.data)

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
        """Host copy of the blocks (reference layout)."""
        if self._host is None:
            self._host = self.blocks.download(self.first, self.pattern.nnzb)
        return self._host

    def matvec(self, x, counter: OpCounter | None = None):
        if tuple(x.shape) != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {tuple(x.shape)}")
        if self._op is None:
            self._op = make_stage_op(self.pattern, 1, [self.blocks], [self.first], None, None, 1.0)
        xd, was_np = to_device(x)
        y = empty_like_dev(self.n)
        L.check(L.lib().irk_stage_op_apply(self._op.handle, xd.data_ptr(), y.data_ptr(),
                                           L.stream_ptr()), "irk_stage_op_apply")
        if counter is not None:
            counter.block_multiplies += self.nnz_blocks
        return from_device(y, was_np)

    def rhs_op(self, nrhs: int) -> _Op:
        """Native operator Y -> [J y_0, ..., J y_{nrhs-1}] (stage-major) that reads
        each block once for all right-hand sides (BASELINE config 3)."""
        ops = self.__dict__.setdefault("_rhs_ops", {})
        if nrhs not in ops:
            ops[nrhs] = make_stage_op(self.pattern, nrhs, [self.blocks] * nrhs, [self.first] * nrhs,
                                      None, None, 1.0)
        return ops[nrhs]

    def matvec_rhs(self, Y, counter: OpCounter | None = None):
        """J applied to the rows of Y (nrhs, n) in one sweep."""
        nrhs = int(Y.shape[0])
        if tuple(Y.shape) != (nrhs, self.n):
            raise ValueError(f"expected shape (nrhs, {self.n}), got {tuple(Y.shape)}")
        yd, was_np = to_device(Y.reshape(-1))
        out = empty_like_dev(nrhs * self.n)
        L.check(L.lib().irk_stage_op_apply(self.rhs_op(nrhs).handle, yd.data_ptr(), out.data_ptr(),
                                           L.stream_ptr()), "irk_stage_op_apply")
        if counter is not None:
            counter.block_multiplies += nrhs * self.nnz_blocks
        return from_device(out, was_np).reshape(nrhs, self.n)


class BlockDiagonalMatrix:
    """T dense m x m blocks on the diagonal (mass matrices), on the GPU."""

    def __init__(self, blocks):
        if isinstance(blocks, DeviceBlocks):
            self.device = blocks
            self._host = None
        else:
            arr = np.asarray(blocks, dtype=np.float64)
            if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
                raise ValueError("expected (T, m, m) block array")
            self.device = DeviceBlocks.from_host(arr)
            self._host = arr

    @classmethod
    def from_reference(cls, mass) -> "BlockDiagonalMatrix":
        return cls(mass.blocks)

    @property
    def blocks(self) -> np.ndarray:
        if self._host is None:
            self._host = self.device.download()
        return self._host

    @property
    def T_elems(self) -> int:
        return self.device.count

    @property
    def m(self) -> int:
        return self.device.nb

    @property
    def n(self) -> int:
        return self.T_elems * self.m

    def matvec(self, x, counter: OpCounter | None = None):
        """y_i = M_i x_i (reference blocks.py:164-170)."""
        if int(x.shape[0]) != self.n or len(x.shape) != 1:
            raise ValueError(f"expected vector of length {self.n}, got {tuple(x.shape)}")
        y = self._diag_matrix().matvec(x)
        if counter is not None:
            counter.block_multiplies += self.T_elems
        return y

    def _diag_matrix(self) -> "BlockSparseMatrix":
        if getattr(self, "_diag", None) is None:
            T = self.T_elems
            ar = np.arange(T, dtype=np.int64)
            pat = DevicePattern(np.arange(T + 1, dtype=np.int64), ar, ar)
            self._diag = BlockSparseMatrix(pat, self.device)
        return self._diag

    def solve(self, x, counter: OpCounter | None = None):
        """y_i = M_i^-1 x_i (reference blocks.py:172-176, np.linalg.solve per
        block): the block ILU(0) of M on the diagonal-only pattern, i.e. the
        device inverse of every M_i (partial-pivoting Gauss-Jordan, factor.cu /
        inverse.cu), built once, then one D^-1 gemv sweep.  Equal to the LU
        solve to rounding."""
        if int(x.shape[0]) != self.n or len(x.shape) != 1:
            raise ValueError(f"expected vector of length {self.n}, got {tuple(x.shape)}")
        if getattr(self, "_inv", None) is None:
            from .precond import ilu0_factorize
            self._inv = ilu0_factorize(self._diag_matrix())
        xd, was_np = to_device(x)
        y = empty_like_dev(self.n)
        self._inv.apply_device(xd, y)
        if counter is not None:
            counter.block_solves += self.T_elems
        return from_device(y, was_np)


# ---------------------------------------------------------------------------
# Line-oriented text exchange format (reference blocks.py:193-216)
# ---------------------------------------------------------------------------

def dump_matrix(mat, path: str) -> None:
    """Reference ``dump_matrix`` (blocks.py:193-201), byte-identical output:
    header ``T m nnz_blocks``, then per stored block (row-major pattern order) a
    line ``i j`` and a line of the m*m row-major values as ``repr(float)``.
    ``mat`` is a device ``BlockSparseMatrix`` (downloaded once) or any object
    with ``indptr / indices / data``."""
    indptr = np.asarray(mat.indptr)
    indices = np.asarray(mat.indices)
    data = np.asarray(mat.data)
    T = len(indptr) - 1
    m = data.shape[1]
    rows = np.repeat(np.arange(T), np.diff(indptr))
    with open(path, "w") as fh:
        fh.write(f"{T} {m} {len(indices)}\n")
        flat = data.reshape(len(indices), m * m).tolist()   # Python floats: repr is the shortest round trip
        for k in range(len(indices)):
            fh.write(f"{rows[k]} {indices[k]}\n")
            fh.write(" ".join(map(repr, flat[k])) + "\n")


def read_matrix_blocks(path: str, indptr, indices) -> np.ndarray:
    """Parse a ``dump_matrix`` file onto a pattern (host): the checks and the
    ``set_block`` placement of reference ``load_matrix`` (blocks.py:204-216)."""
    indptr, indices = np.asarray(indptr), np.asarray(indices)
    T_pat, nnzb = len(indptr) - 1, len(indices)
    with open(path) as fh:
        T, m, nnz = (int(tok) for tok in fh.readline().split())
        if T != T_pat:
            raise ValueError(f"file has T={T}, graph has {T_pat}")
        if nnz != nnzb:
            raise ValueError(f"file has {nnz} blocks, pattern expects {nnzb}")
        lines = fh.read().split("\n")
    ij = np.array([ln.split() for ln in lines[0:2 * nnz:2]], dtype=np.int64).reshape(nnz, 2)
    vals = np.array(" ".join(lines[1:2 * nnz:2]).split(), dtype=np.float64)
    if vals.size != nnz * m * m:
        raise ValueError("truncated block data")
    vals = vals.reshape(nnz, m, m)
    data = np.zeros((nnzb, m, m))
    for k in range(nnz):
        i, j = int(ij[k, 0]), int(ij[k, 1])
        lo, hi = indptr[i], indptr[i + 1]
        pos = int(np.searchsorted(indices[lo:hi], j)) + lo
        if pos >= hi or indices[pos] != j:
            raise KeyError(f"block ({i}, {j}) not in pattern")
        data[pos] = vals[k]   # later duplicates overwrite, as set_block does
    return data


def load_matrix(path: str, graph_or_pattern) -> "BlockSparseMatrix":
    """Reference ``load_matrix`` (blocks.py:204-216) into a device matrix."""
    pat = graph_or_pattern if isinstance(graph_or_pattern, DevicePattern) else pattern_for(graph_or_pattern)
    data = read_matrix_blocks(path, pat.indptr, pat.indices)
    return BlockSparseMatrix(pat, DeviceBlocks.from_host(data), host=data)
