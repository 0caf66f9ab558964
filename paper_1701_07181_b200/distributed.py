"""Element-partitioned (multi-GPU) transformed stage solve.

One process per GPU.  Elements are split into P contiguous index ranges
(reference ``meshing.partition``, meshing.py:81-90; z-major numbering makes
them slabs of the 3D cube).  Per GMRES iteration the ranks exchange:

* the halo: stage values of the elements a neighbouring slab's Jacobian rows
  touch (one grouped NCCL send/recv per peer, packed by an index gather), so
  every rank can apply its rows of B = A^-1 (x) M - dt blkdiag(J);
* the inner products of classical Gram-Schmidt and the norms -- allreduced from
  the native GMRES loop (``irk_comm_allreduce``: NCCL on the solve's stream).

The preconditioner is the *partitioned* block ILU(0): blocks coupling two
partitions are dropped (precond.py:26-45, the paper's parallel scheme,
PAPER.md:694-699), so its factorisation and apply are purely local -- each rank
factors the diagonal block of its slab.  The result equals the single-process
solve with ``partition_of = partition(graph, P).partition_of``.

``SlabPlan`` (index bookkeeping) and ``HaloExchange`` (a torch.distributed
restatement of the halo, used by the CPU gloo tests in tests/test_distributed.py)
are device-agnostic.  ``DistributedStageSolver`` runs on the native layer of
libirkb200 (csrc/comm.cu: ``irk_comm`` / ``irk_halo`` / ``irk_dist_op``, NCCL
loaded by the library itself); torch.distributed only broadcasts the NCCL
unique id, or -- for the host-staged transport -- carries the bytes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .meshes import partition_bounds


@dataclass
class SlabPlan:
    """Rank-local view of a CSR-of-blocks pattern under a contiguous partition.

    Local element ids: 0..T_local-1 are the owned elements (global
    lo..hi-1, same order); T_local.. are ghosts (neighbours owned by other
    ranks), sorted by global id.
    """

    rank: int
    P: int
    T: int
    lo: int
    hi: int
    ghosts: np.ndarray            # global ids of ghost elements
    ext_indptr: np.ndarray        # local rows, columns in extended numbering
    ext_indices: np.ndarray
    ext_diag: np.ndarray
    row_block_src: np.ndarray     # global block position of every local block
    loc_indptr: np.ndarray        # local rows, local columns only (factor pattern)
    loc_indices: np.ndarray
    loc_diag: np.ndarray
    loc_block_src: np.ndarray
    q0: int                       # global position of the rank's first block
    send: dict                    # peer -> local ids to send (ascending global id)
    recv: dict                    # peer -> ghost slots to fill (ascending global id)
    interior: tuple               # (r0, r1): rows with no ghost column

    @property
    def T_local(self) -> int:
        return self.hi - self.lo

    @property
    def n_ghost(self) -> int:
        return len(self.ghosts)

    @classmethod
    def build(cls, indptr, indices, diag_pos, P: int, rank: int) -> "SlabPlan":
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        T = len(indptr) - 1
        bounds = partition_bounds(T, P)
        owner = np.repeat(np.arange(P), np.diff(bounds))
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        q0, q1 = int(indptr[lo]), int(indptr[hi])
        cols = indices[q0:q1]
        rows = np.repeat(np.arange(lo, hi), np.diff(indptr[lo:hi + 1]))
        remote = (cols < lo) | (cols >= hi)
        ghosts = np.unique(cols[remote])
        # extended numbering: owned -> g - lo, ghost -> T_local + rank in ghosts
        ext_cols = np.where(remote, (hi - lo) + np.searchsorted(ghosts, cols), cols - lo)
        ext_indptr = indptr[lo:hi + 1] - q0
        src = np.arange(q0, q1, dtype=np.int64)
        # re-sort every row by extended column (ghost ids follow the owned ones)
        order = np.lexsort((ext_cols, rows))
        ext_cols, src, cols, rows, remote = ext_cols[order], src[order], cols[order], rows[order], remote[order]
        ext_diag = np.empty(hi - lo, dtype=np.int64)
        diag_hits = np.nonzero(ext_cols == rows - lo)[0]
        ext_diag[rows[diag_hits] - lo] = diag_hits
        # local factor pattern: drop the cross-partition blocks (they are not kept)
        keepm = ~remote
        loc_indices = (cols - lo)[keepm]
        loc_src = src[keepm]
        counts = np.add.reduceat(keepm.astype(np.int64), ext_indptr[:-1]) if hi > lo else np.zeros(0, np.int64)
        loc_indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        loc_rows = rows[keepm] - lo
        loc_diag = loc_indptr[:-1] + np.array(
            [np.searchsorted(loc_indices[loc_indptr[i]:loc_indptr[i + 1]], i) for i in range(hi - lo)],
            dtype=np.int64)
        del loc_rows
        # halo lists: what each peer needs from me / what I receive from each peer
        recv = {}
        gown = owner[ghosts]
        for p in np.unique(gown):
            recv[int(p)] = np.nonzero(gown == p)[0].astype(np.int64)
        send = {}
        for p in range(P):
            if p == rank:
                continue
            plo, phi = int(bounds[p]), int(bounds[p + 1])
            pc = indices[int(indptr[plo]):int(indptr[phi])]
            need = np.unique(pc[(pc >= lo) & (pc < hi)])
            if len(need):
                send[p] = (need - lo).astype(np.int64)
        # interior rows: rows whose columns are all owned (contiguous core when the
        # numbering is slab-major; computed as the longest owned-only run)
        has_remote = np.zeros(hi - lo, dtype=bool)
        np.logical_or.at(has_remote, rows - lo, remote)
        r0, r1 = _longest_false_run(has_remote)
        return cls(rank, P, T, lo, hi, ghosts, ext_indptr, ext_cols.astype(np.int64), ext_diag, src,
                   loc_indptr, loc_indices.astype(np.int64), loc_diag, loc_src, q0, send, recv, (r0, r1))


def _longest_false_run(mask: np.ndarray) -> tuple[int, int]:
    best = (0, 0)
    start = None
    for i, m in enumerate(list(mask) + [True]):
        if not m and start is None:
            start = i
        elif m and start is not None:
            if i - start > best[1] - best[0]:
                best = (start, i)
            start = None
    return best


class HaloExchange:
    """Ghost exchange of stage-major vectors over torch.distributed.

    ``exchange(x, ghost)``: x is the rank's (s, T_local, nb) vector (flat),
    ghost the (s, n_ghost, nb) receive buffer.  One grouped batch of isend /
    irecv per call (NCCL on GPU, gloo on CPU), packed with index_select.
    """

    def __init__(self, plan: SlabPlan, s: int, nb: int, device, group=None):
        import torch
        self.plan, self.s, self.nb, self.group = plan, s, nb, group
        self.torch = torch
        self.send_idx = {p: torch.as_tensor(v, device=device) for p, v in plan.send.items()}
        self.recv_idx = {p: torch.as_tensor(v, device=device) for p, v in plan.recv.items()}
        self.send_buf = {p: torch.empty((s, len(v), nb), dtype=torch.float64, device=device)
                         for p, v in plan.send.items()}
        self.recv_buf = {p: torch.empty((s, len(v), nb), dtype=torch.float64, device=device)
                         for p, v in plan.recv.items()}

    def start(self, x):
        """Pack and post the sends / receives; returns the pending work handles."""
        if self.plan.n_ghost == 0 and not self.send_idx:
            return []
        dist = self.torch.distributed
        xv = x.view(self.s, self.plan.T_local, self.nb)
        ops = []
        for p, idx in self.send_idx.items():
            self.torch.index_select(xv, 1, idx, out=self.send_buf[p])
            ops.append(dist.P2POp(dist.isend, self.send_buf[p], p, self.group))
        for p in self.recv_idx:
            ops.append(dist.P2POp(dist.irecv, self.recv_buf[p], p, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def finish(self, works, ghost) -> None:
        """Wait for the posted exchange and scatter the received values into ``ghost``."""
        for r in works:
            r.wait()
        if self.plan.n_ghost == 0:
            return
        gv = ghost.view(self.s, self.plan.n_ghost, self.nb)
        for p, idx in self.recv_idx.items():
            gv.index_copy_(1, idx, self.recv_buf[p])

    def exchange(self, x, ghost) -> None:
        self.finish(self.start(x), ghost)


def allreduce_sum(buf, group=None) -> None:
    import torch.distributed as dist
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def _stream_of(ptr):
    import torch
    return torch.cuda.ExternalStream(ptr) if ptr else torch.cuda.default_stream()


class Comm:
    """An ``irk_comm`` transport handle (comm.cu).

    * ``Comm.nccl(group)``: NCCL inside libirkb200 -- rank 0 draws the unique id,
      torch.distributed broadcasts it (plumbing only), every rank joins; halo
      send/recv and the GMRES allreduces then run natively on the solve's stream.
    * ``Comm.host(plan, s, nb, group)``: host-staged transport through
      torch.distributed on CPU tensors (gloo): the library calls back with the
      packed send buffer / the small allreduce buffers.  For machines without
      NCCL and for tests that put several ranks on one GPU (no kernel of one rank
      ever waits on another's: every exchange is completed on the host).
    * ``Comm.single()``: one rank, no exchange.
    """

    def __init__(self, handle: int, nranks: int, rank: int, keep=()):
        self.handle, self.nranks, self.rank, self._keep = handle, nranks, rank, list(keep)

    def __del__(self):
        h = getattr(self, "handle", None)
        from . import _lib as L
        if h and L._lib is not None:
            L._lib.irk_comm_destroy(h)
            self.handle = None

    @property
    def native_allreduce(self):
        import ctypes

        from . import _lib as L
        return ctypes.cast(L.lib().irk_comm_allreduce, ctypes.c_void_p).value, self.handle

    @classmethod
    def single(cls) -> "Comm":
        import ctypes

        from . import _lib as L
        h = ctypes.c_void_p()
        L.check(L.lib().irk_comm_create_callback(L.ctx(), 1, 0, None, None, None, ctypes.byref(h)),
                "irk_comm_create_callback")
        return cls(h.value, 1, 0)

    @classmethod
    def nccl(cls, group=None) -> "Comm":
        import ctypes

        import torch.distributed as dist

        from . import _lib as L
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (ctypes.c_ubyte * 128)()
        if rank == 0:
            L.check(L.lib().irk_comm_nccl_unique_id(buf, 128), "irk_comm_nccl_unique_id")
        obj = [bytes(buf)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        idb = (ctypes.c_ubyte * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        L.check(L.lib().irk_comm_create_nccl(L.ctx(), idb, world, rank, ctypes.byref(h)), "irk_comm_create_nccl")
        return cls(h.value, world, rank)

    @classmethod
    def host(cls, plan: "SlabPlan", s: int, nb: int, group=None) -> "Comm":
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib as L
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        peers = halo_peers(plan)
        ng = plan.n_ghost
        nsend = sum(len(plan.send.get(p, ())) for p in peers)
        errors = []

        def xfer(user, send_p, ghost_p, stream):
            try:
                st = _stream_of(stream)
                with torch.cuda.stream(st):
                    send = (L.wrap_device(send_p, s * nsend * nb).view(s, nsend, nb).cpu()
                            if nsend else None)
                    ops, recv, off = [], {}, 0
                    for p in peers:
                        cnt = len(plan.send.get(p, ()))
                        g = dist.get_global_rank(group, p) if group is not None else p
                        if cnt:
                            ops.append(dist.P2POp(dist.isend, send[:, off:off + cnt].contiguous(), g, group))
                        off += cnt
                        rc = len(plan.recv.get(p, ()))
                        if rc:
                            recv[p] = torch.empty((s, rc, nb), dtype=torch.float64)
                            ops.append(dist.P2POp(dist.irecv, recv[p], g, group))
                    for r in (dist.batch_isend_irecv(ops) if ops else []):
                        r.wait()
                    if ng:
                        gv = L.wrap_device(ghost_p, s * ng * nb).view(s, ng, nb)
                        for p, buf in recv.items():
                            first = int(plan.recv[p][0])
                            gv[:, first:first + buf.shape[1]].copy_(buf)
                        st.synchronize()
                return 0
            except BaseException as e:  # noqa: BLE001 -- surfaced through the C status
                errors.append(e)
                return 1

        def allreduce(user, buf_p, count, stream):
            try:
                st = _stream_of(stream)
                with torch.cuda.stream(st):
                    d = L.wrap_device(buf_p, count)
                    h = d.cpu()
                    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                    d.copy_(h)
                    st.synchronize()
                return 0
            except BaseException as e:  # noqa: BLE001
                errors.append(e)
                return 1

        xf, ar = L.XFER_FN(xfer), L.ALLREDUCE_FN(allreduce)
        h = ctypes.c_void_p()
        L.check(L.lib().irk_comm_create_callback(L.ctx(), world, rank, ctypes.cast(xf, ctypes.c_void_p).value,
                                                 ctypes.cast(ar, ctypes.c_void_p).value, None, ctypes.byref(h)),
                "irk_comm_create_callback")
        c = cls(h.value, world, rank, keep=(xf, ar))
        c.errors = errors
        return c


def halo_peers(plan: "SlabPlan") -> list:
    return sorted(set(plan.send) | set(plan.recv))


class DistributedStageSolver:
    """Rank-local device solver for the element-partitioned stage system, on the
    native layer of libirkb200 (comm.cu): ``irk_halo`` (pack kernel + grouped NCCL
    send/recv straight into the ghost buffer), ``irk_dist_op`` (the slab's rows of
    B, exchange overlapped with the interior rows) and ``irk_gmres`` with the
    native allreduce -- no Python in the GMRES loop.  Next to the slab's
    partitioned implicit-L factor the Arnoldi product P^-1 (B v) runs fused (halo
    mode of k_unc_fused_fwd) after the exchange.

    ``J_rows``: the rank's Jacobian block rows in global pattern order
    (positions plan.q0 .. plan.q0 + len, reference row-major layout);
    ``M_rows``: its mass blocks; ``a_inv``/``dt``/``shifts`` as in ``StageSolver``.
    ``transport``: "auto" (NCCL when the process group runs NCCL and has more than
    one rank, host-staged otherwise), "nccl", "host", or a ready ``Comm``.
    """

    def __init__(self, plan: SlabPlan, J_rows: np.ndarray, M_rows: np.ndarray, a_inv, dt: float,
                 kind: str = "uncoupled", shifts=None, gmres_cfg=None, group=None, transport="auto"):
        import ctypes

        import torch

        from . import _lib as L
        from .blocks import BlockDiagonalMatrix, BlockSparseMatrix, DeviceBlocks, DevicePattern
        from .krylov import GmresConfig
        from .precond import stage_coupled_factorize, stage_uncoupled_factorize
        from .stage_system import StageOperator

        self.plan, self.group, self.kind = plan, group, kind
        a_inv = np.asarray(a_inv, dtype=np.float64)
        s = a_inv.shape[0]
        nb = J_rows.shape[1]
        self.s, self.nb = s, nb
        self.cfg = gmres_cfg or GmresConfig(rel_tol=1e-8, restart=40)
        Tl, ng = plan.T_local, plan.n_ghost
        # operator pattern: local rows + one diagonal-only row per ghost (never computed)
        ip = np.concatenate([plan.ext_indptr, plan.ext_indptr[-1] + 1 + np.arange(ng)])
        ix = np.concatenate([plan.ext_indices, Tl + np.arange(ng)])
        dg = np.concatenate([plan.ext_diag, plan.ext_indptr[-1] + np.arange(ng)])
        self.op_pat = DevicePattern(ip, ix, dg)
        jb = DeviceBlocks(nb, len(ix))
        jb.upload(np.ascontiguousarray(J_rows[plan.row_block_src - plan.q0]))
        if ng:
            jb.upload(np.zeros((ng, nb, nb)), first=len(plan.ext_indices))
        Mext = np.concatenate([M_rows, np.broadcast_to(np.eye(nb), (ng, nb, nb))]) if ng else M_rows
        self.mass = BlockDiagonalMatrix(Mext)

        class _Der:
            pass

        der = _Der()
        der.a_inv = a_inv
        der.shifts = np.zeros(s) if shifts is None else np.asarray(shifts, dtype=np.float64)
        self.op = StageOperator(der, dt, self.mass, [BlockSparseMatrix(self.op_pat, jb)] * s)
        self.ghost = torch.zeros(max(s * ng * nb, 1), dtype=torch.float64, device="cuda")
        L.check(L.lib().irk_stage_op_set_halo(self.op._op.handle, Tl, self.ghost.data_ptr(), ng),
                "irk_stage_op_set_halo")
        # factor operator: local blocks only (cross-partition blocks are dropped)
        self.fac_pat = DevicePattern(plan.loc_indptr, plan.loc_indices, plan.loc_diag)
        fj = DeviceBlocks.from_host(np.ascontiguousarray(J_rows[plan.loc_block_src - plan.q0]))
        fm = BlockDiagonalMatrix(M_rows)
        self.fac_op = StageOperator(der, dt, fm, [BlockSparseMatrix(self.fac_pat, fj)] * s)
        self._factorize = (stage_coupled_factorize if kind.startswith("coupled") else
                           (lambda o: stage_uncoupled_factorize(o, der.shifts if kind == "uncoupled" else None)))
        self.fac = None
        self.n_local = s * Tl * nb
        # ---- native transport, halo and distributed operator --------------------
        self.comm = self._make_comm(transport, group, plan, s, nb)
        peers = halo_peers(plan)
        for p in peers:
            r = plan.recv.get(p)
            if r is not None and len(r) and not np.array_equal(r, np.arange(r[0], r[0] + len(r))):
                raise ValueError("ghosts of a peer must be contiguous (sorted global ids, contiguous slabs)")
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
        self._halo_arrays = (
            np.ascontiguousarray(peers, dtype=np.int32),
            i64([len(plan.send.get(p, ())) for p in peers]),
            i64(np.concatenate([plan.send[p] for p in peers if p in plan.send]) if plan.send else np.zeros(0)),
            i64([len(plan.recv.get(p, ())) for p in peers]),
            i64([int(plan.recv[p][0]) if len(plan.recv.get(p, ())) else 0 for p in peers]))
        pa, sc, se, rc, rf = self._halo_arrays
        h = ctypes.c_void_p()
        L.check(L.lib().irk_halo_create(self.comm.handle, s, nb, Tl, ng, len(peers), L.ptr(pa), L.ptr(sc),
                                        L.ptr(se), L.ptr(rc), L.ptr(rf), ctypes.byref(h)), "irk_halo_create")
        self.halo = h.value
        r0, r1 = plan.interior
        self.boundary = np.concatenate([np.arange(0, r0), np.arange(r1, Tl)]).astype(np.int32)
        d = ctypes.c_void_p()
        L.check(L.lib().irk_dist_op_create(self.op._op.handle, self.halo, self.ghost.data_ptr(), int(r0), int(r1),
                                           L.ptr(self.boundary), len(self.boundary), ctypes.byref(d)),
                "irk_dist_op_create")
        self.dist_op = d.value

    @staticmethod
    def _make_comm(transport, group, plan, s, nb):
        if isinstance(transport, Comm):
            return transport
        import torch.distributed as dist
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        if transport == "auto":
            transport = ("nccl" if dist.get_backend(group) == "nccl" else "host") if multi else "single"
        if transport == "single" or not multi:
            return Comm.single()
        if transport == "nccl":
            return Comm.nccl(group)
        if transport == "host":
            return Comm.host(plan, s, nb, group)
        raise ValueError(f"unknown transport {transport!r}")

    def __del__(self):
        from . import _lib as L
        if L._lib is None:
            return
        if getattr(self, "dist_op", None):
            L._lib.irk_dist_op_destroy(self.dist_op)
            self.dist_op = None
        if getattr(self, "halo", None):
            L._lib.irk_halo_destroy(self.halo)
            self.halo = None

    def factorize(self):
        """Local partitioned factor; re-factorised in place after the first call."""
        if self.fac is not None and hasattr(self.fac, "refactor"):
            if self.kind.startswith("coupled"):
                return self.fac.refactor(self.fac_op)
            return self.fac.refactor(self.fac_op, self.fac.shifts)
        self.fac = self._factorize(self.fac_op)
        return self.fac

    def native_linop(self):
        from . import _lib as L
        op = L.Linop()
        L.check(L.lib().irk_linop_dist_op(self.dist_op, op), "irk_linop_dist_op")
        return op, self

    def matvec(self, w):
        """This rank's rows of B w (irk_dist_op_apply: the exchange is in flight
        while the interior rows are computed, the boundary rows follow)."""
        from . import _lib as L
        y = self.torch_empty()
        L.check(L.lib().irk_dist_op_apply(self.dist_op, w.data_ptr(), y.data_ptr(), L.stream_ptr()),
                "irk_dist_op_apply")
        return y

    def product(self, v, x=None) -> bool:
        """x = P^-1 (B v) as the GMRES loop runs it; returns True if it ran fused."""
        import ctypes

        from . import _lib as L
        x = self.torch_empty() if x is None else x
        fused = ctypes.c_int(0)
        L.check(L.lib().irk_dist_op_factor_apply(self.dist_op, self.fac.handle, v.data_ptr(), x.data_ptr(),
                                                 ctypes.byref(fused), L.stream_ptr()), "irk_dist_op_factor_apply")
        return x, bool(fused.value)

    def torch_empty(self):
        import torch
        return torch.empty(self.n_local, dtype=torch.float64, device="cuda")

    def solve(self, rhs_local, x=None):
        from .krylov import gmres_device
        pre = None if self.fac is None else self.fac.apply
        out = gmres_device(self.matvec, pre, rhs_local, self.cfg, x=x,
                           native_allreduce=self.comm.native_allreduce if self.comm.nranks > 1 else None)
        for e in getattr(self.comm, "errors", ()):
            raise e
        return out
