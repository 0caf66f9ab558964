// Element-partitioned (multi-GPU) layer of the stage solve: the paper's
// parallel scheme -- elements cut into contiguous slabs
// (meshing.py:81-90), the partitioned block ILU(0) needs no communication
// (precond.py:26-45), the operator needs the neighbour halo, and the GMRES
// inner products are summed across ranks.
//
//   irk_comm   -- transport: NCCL (loaded at run time with dlopen, so the
//                 library has no link-time NCCL dependency and shares the
//                 process's libnccl.so.2 with PyTorch) or a host callback
//                 (host-staged exchange for tests / machines without NCCL).
//   irk_halo   -- one neighbour exchange of a stage-major vector: a pack
//                 kernel gathers the rows every peer needs into one send
//                 buffer ([stage][send element][nb], peers contiguous), then
//                 one NCCL group of s sends + s receives per peer, received
//                 straight into the ghost buffer ([stage][ghost][nb]; ghosts
//                 are sorted by global id, so each peer's range is contiguous).
//   irk_dist_op -- the slab's rows of B = A^-1 (x) M - dt blkdiag(J) as a
//                 native GMRES operator: with NCCL the exchange runs on a
//                 comm stream while the interior rows (no ghost column) are
//                 computed, the boundary rows after it lands.  irk_gmres
//                 recognises it next to a factor and runs the Arnoldi product
//                 P^-1 (B v) fused (apply.cu, halo mode) after the exchange.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "irk_internal.cuh"

namespace irk {

int factor_apply_fused(const irk_stage_op* op, const irk_factor* f, const double* v, double* x, cudaStream_t st);

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string where;
};

static NcclApi* nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = getenv("IRK_NCCL_LIB");
        const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* c : cands) {
            if (!c || !*c) continue;
            if ((api.h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) {
                api.where = c;
                break;
            }
        }
        if (!api.h) return;
        auto sym = [&](const char* n) { return dlsym(api.h, n); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.Send ||
            !api.Recv || !api.GroupStart || !api.GroupEnd) {
            dlclose(api.h);
            api.h = nullptr;
        }
    });
    return api.h ? &api : nullptr;
}

static int nccl_fail(ncclResult_t r, const char* what) {
    NcclApi* a = nccl_api();
    set_error(std::string(what) + ": " + (a && a->GetErrorString ? a->GetErrorString(r) : "NCCL error"));
    return IRK_ECUDA;
}
#define IRK_NCCL(call)                                                   \
    do {                                                                 \
        ncclResult_t _r = (call);                                        \
        if (_r != ncclSuccess) return ::irk::nccl_fail(_r, #call);       \
    } while (0)

// [stage][send element][nb] <- x[stage][elem][nb], 128-bit when nb is even
__global__ void k_halo_pack(const double* __restrict__ x, int64_t n, const int32_t* __restrict__ elems,
                            int64_t nsend, int nb, int s, double* __restrict__ out) {
    const int64_t per = nsend * nb;
    const int64_t total = per * s;
    if ((nb & 1) == 0) {
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total / 2;
             t += (int64_t)gridDim.x * blockDim.x) {
            const int64_t k = (2 * t) / per, r = (2 * t) % per, e = r / nb, c = (r % nb) >> 1;
            const double2 v = reinterpret_cast<const double2*>(x + k * n + (int64_t)elems[e] * nb)[c];
            reinterpret_cast<double2*>(out)[t] = v;
        }
    } else {
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
             t += (int64_t)gridDim.x * blockDim.x) {
            const int64_t k = t / per, r = t % per, e = r / nb, c = r % nb;
            out[t] = x[k * n + (int64_t)elems[e] * nb + c];
        }
    }
}

}  // namespace irk

using namespace irk;

struct irk_comm {
    irk_ctx* ctx = nullptr;
    int nranks = 1, rank = 0;
    int kind = 0;   // 0 nccl, 1 callback
    ncclComm_t nccl = nullptr;
    irk_halo_xfer_fn xfer = nullptr;
    irk_allreduce_fn ar = nullptr;
    void* user = nullptr;
};

struct irk_halo {
    irk_comm* comm = nullptr;
    int s = 0, nb = 0;
    int64_t T_local = 0, n_ghost = 0, nsend = 0;
    std::vector<int> peers;
    std::vector<int64_t> send_cnt, send_off, recv_cnt, recv_first;
    int32_t* d_elems = nullptr;
    double* d_send = nullptr;
    cudaStream_t cst = nullptr;          // comm stream (NCCL transport)
    cudaEvent_t ev_pack = nullptr, ev_recv = nullptr;
};

struct irk_dist_op {
    irk_stage_op* op = nullptr;
    irk_halo* halo = nullptr;
    double* ghost = nullptr;
    int64_t r0 = 0, r1 = 0;              // interior rows (no ghost column)
    int32_t* d_boundary = nullptr;
    int64_t nboundary = 0;
};

namespace irk {

static int halo_pack(irk_halo* h, const double* x, cudaStream_t st) {
    if (h->nsend == 0) return IRK_OK;
    const int64_t total = h->nsend * h->nb * h->s;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total / 2 + 255) / 256, 148 * 8));
    k_halo_pack<<<grid, 256, 0, st>>>(x, h->T_local * h->nb, h->d_elems, h->nsend, h->nb, h->s, h->d_send);
    IRK_LAUNCHED();
    return IRK_OK;
}

// NCCL group of s sends + s receives per peer on stream `cs`
static int halo_nccl(irk_halo* h, double* ghost, cudaStream_t cs) {
    NcclApi* a = nccl_api();
    irk_comm* c = h->comm;
    IRK_NCCL(a->GroupStart());
    for (size_t p = 0; p < h->peers.size(); ++p) {
        const int peer = h->peers[p];
        for (int k = 0; k < h->s; ++k) {
            if (h->send_cnt[p])
                IRK_NCCL(a->Send(h->d_send + (k * h->nsend + h->send_off[p]) * h->nb,
                                 (size_t)(h->send_cnt[p] * h->nb), ncclFloat64, peer, c->nccl, cs));
            if (h->recv_cnt[p])
                IRK_NCCL(a->Recv(ghost + (k * h->n_ghost + h->recv_first[p]) * h->nb,
                                 (size_t)(h->recv_cnt[p] * h->nb), ncclFloat64, peer, c->nccl, cs));
        }
    }
    IRK_NCCL(a->GroupEnd());
    return IRK_OK;
}

// Full exchange, stream-ordered on st (ghost valid for work enqueued on st after it)
int halo_exchange(irk_halo* h, const double* x, double* ghost, cudaStream_t st) {
    if (h->peers.empty()) return IRK_OK;
    IRK_TRY(halo_pack(h, x, st));
    if (h->comm->kind == 1) {
        const int rc = h->comm->xfer(h->comm->user, h->d_send, ghost, st);
        if (rc) { set_error("halo transfer callback failed"); return IRK_ECALLBACK; }
        return IRK_OK;
    }
    return halo_nccl(h, ghost, st);
}

int dist_op_exchange(const irk_dist_op* d, const double* w, cudaStream_t st) {
    return halo_exchange(d->halo, w, d->ghost, st);
}

const irk_stage_op* dist_op_stage_op(const irk_dist_op* d) { return d->op; }

// y = B w on the slab's rows: NCCL exchange overlapped with the interior rows
int dist_op_apply(const irk_dist_op* d, const double* w, double* y, cudaStream_t st) {
    irk_halo* h = d->halo;
    if (h->peers.empty()) return irk_stage_op_apply(d->op, w, y, st);
    if (h->comm->kind != 0) {
        IRK_TRY(halo_exchange(h, w, d->ghost, st));
        return irk_stage_op_apply(d->op, w, y, st);
    }
    IRK_TRY(halo_pack(h, w, st));
    IRK_CK(cudaEventRecord(h->ev_pack, st));
    IRK_CK(cudaStreamWaitEvent(h->cst, h->ev_pack, 0));
    IRK_TRY(halo_nccl(h, d->ghost, h->cst));
    IRK_CK(cudaEventRecord(h->ev_recv, h->cst));
    if (d->r1 > d->r0) IRK_TRY(irk_stage_op_apply_range(d->op, w, y, d->r0, d->r1, st));
    IRK_CK(cudaStreamWaitEvent(st, h->ev_recv, 0));
    if (d->nboundary) IRK_TRY(irk_stage_op_apply_rows(d->op, w, y, d->d_boundary, d->nboundary, st));
    return IRK_OK;
}

// One Arnoldi product x = P^-1 (B v) with the distributed operator: exchange, then
// the fused forward sweep over the operator's rows (own columns from v, ghosts from
// the halo buffer) + backward sweep.  Returns 1 (exchange done, nothing else) when
// the pair does not qualify; the caller then applies the operator locally.
int dist_op_fused_product(const irk_dist_op* d, const irk_factor* f, const double* v, double* x, cudaStream_t st) {
    IRK_TRY(dist_op_exchange(d, v, st));
    return factor_apply_fused(d->op, f, v, x, st);
}

}  // namespace irk

extern "C" {

int irk_comm_nccl_available(void) { return nccl_api() ? 1 : 0; }

int irk_comm_nccl_unique_id(unsigned char* id_out, int64_t cap) {
    IRK_ARG(id_out && cap >= (int64_t)sizeof(ncclUniqueId), "id buffer too small (NCCL_UNIQUE_ID_BYTES)");
    NcclApi* a = nccl_api();
    if (!a) { set_error("libnccl.so.2 could not be loaded (set IRK_NCCL_LIB)"); return IRK_EINVAL; }
    ncclUniqueId id;
    IRK_NCCL(a->GetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return IRK_OK;
}

int irk_comm_create_nccl(irk_ctx* ctx, const unsigned char* id, int nranks, int rank, irk_comm** out) {
    IRK_ARG(ctx && id && out, "NULL argument");
    IRK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    NcclApi* a = nccl_api();
    if (!a) { set_error("libnccl.so.2 could not be loaded (set IRK_NCCL_LIB)"); return IRK_EINVAL; }
    IRK_CK(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    auto* c = new irk_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->kind = 0;
    const ncclResult_t r = a->CommInitRank(&c->nccl, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return IRK_OK;
}

int irk_comm_create_callback(irk_ctx* ctx, int nranks, int rank, irk_halo_xfer_fn xfer, irk_allreduce_fn ar,
                             void* user, irk_comm** out) {
    IRK_ARG(ctx && out, "NULL argument");
    IRK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
    IRK_ARG(nranks == 1 || (xfer && ar), "a multi-rank callback transport needs xfer and allreduce");
    auto* c = new irk_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    c->kind = 1;
    c->xfer = xfer;
    c->ar = ar;
    c->user = user;
    *out = c;
    return IRK_OK;
}

void irk_comm_destroy(irk_comm* c) {
    if (!c) return;
    if (c->kind == 0 && c->nccl) {
        NcclApi* a = nccl_api();
        if (a) a->CommDestroy(c->nccl);
    }
    delete c;
}

int irk_comm_allreduce(void* comm, double* buf, int64_t count, void* stream) {
    auto* c = static_cast<irk_comm*>(comm);
    IRK_ARG(c && (buf || count == 0), "NULL argument");
    if (c->nranks == 1 || count == 0) return IRK_OK;
    if (c->kind == 1) {
        const int rc = c->ar(c->user, buf, count, stream);
        if (rc) { set_error("allreduce callback failed"); return IRK_ECALLBACK; }
        return IRK_OK;
    }
    IRK_NCCL(nccl_api()->AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c->nccl,
                                   (cudaStream_t)stream));
    return IRK_OK;
}

int irk_halo_create(irk_comm* comm, int s, int nb, int64_t T_local, int64_t n_ghost, int npeers,
                    const int32_t* peers, const int64_t* send_counts, const int64_t* send_elems,
                    const int64_t* recv_counts, const int64_t* recv_first, irk_halo** out) {
    IRK_ARG(comm && out, "NULL argument");
    IRK_ARG(s >= 1 && s <= IRK_MAX_STAGES && nb >= 1 && nb <= IRK_MAX_NB, "bad s / nb");
    IRK_ARG(T_local >= 1 && n_ghost >= 0 && npeers >= 0, "bad sizes");
    IRK_ARG(npeers == 0 || (peers && send_counts && recv_counts && recv_first), "NULL peer lists");
    auto* h = new irk_halo();
    h->comm = comm;
    h->s = s;
    h->nb = nb;
    h->T_local = T_local;
    h->n_ghost = n_ghost;
    std::vector<int32_t> elems;
    int64_t recv_total = 0;
    for (int p = 0; p < npeers; ++p) {
        if (peers[p] < 0 || peers[p] >= comm->nranks || peers[p] == comm->rank || send_counts[p] < 0 ||
            recv_counts[p] < 0 || recv_first[p] < 0 || recv_first[p] + recv_counts[p] > n_ghost) {
            delete h;
            set_error("invalid argument: bad halo peer list");
            return IRK_EINVAL;
        }
        h->peers.push_back(peers[p]);
        h->send_off.push_back(h->nsend);
        h->send_cnt.push_back(send_counts[p]);
        h->recv_cnt.push_back(recv_counts[p]);
        h->recv_first.push_back(recv_first[p]);
        for (int64_t e = 0; e < send_counts[p]; ++e) {
            const int64_t id = send_elems[h->nsend + e];
            if (id < 0 || id >= T_local) {
                delete h;
                set_error("invalid argument: halo send element out of range");
                return IRK_EINVAL;
            }
            elems.push_back((int32_t)id);
        }
        h->nsend += send_counts[p];
        recv_total += recv_counts[p];
    }
    if (recv_total != n_ghost) {
        delete h;
        set_error("invalid argument: halo receive counts do not cover the ghost buffer");
        return IRK_EINVAL;
    }
    int rc = IRK_OK;
    auto fail = [&](cudaError_t e, const char* what) {
        rc = fail_cuda(e, what, __FILE__, __LINE__);
        irk_halo_destroy(h);
        return rc;
    };
    cudaError_t e;
    if ((e = cudaSetDevice(comm->ctx->device)) != cudaSuccess) return fail(e, "cudaSetDevice");
    if (h->nsend) {
        if ((e = cudaMalloc(&h->d_elems, sizeof(int32_t) * h->nsend)) != cudaSuccess) return fail(e, "cudaMalloc");
        if ((e = cudaMemcpy(h->d_elems, elems.data(), sizeof(int32_t) * h->nsend, cudaMemcpyHostToDevice)) !=
            cudaSuccess)
            return fail(e, "cudaMemcpy");
        if ((e = cudaMalloc(&h->d_send, sizeof(double) * h->nsend * nb * s)) != cudaSuccess)
            return fail(e, "cudaMalloc");
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((e = cudaStreamCreateWithPriority(&h->cst, cudaStreamNonBlocking, hi)) != cudaSuccess)
        return fail(e, "cudaStreamCreate");
    if ((e = cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "cudaEventCreate");
    if ((e = cudaEventCreateWithFlags(&h->ev_recv, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "cudaEventCreate");
    *out = h;
    return IRK_OK;
}

void irk_halo_destroy(irk_halo* h) {
    if (!h) return;
    if (h->cst) cudaStreamSynchronize(h->cst);
    cudaFree(h->d_elems);
    cudaFree(h->d_send);
    if (h->ev_pack) cudaEventDestroy(h->ev_pack);
    if (h->ev_recv) cudaEventDestroy(h->ev_recv);
    if (h->cst) cudaStreamDestroy(h->cst);
    delete h;
}

int irk_halo_exchange(irk_halo* h, const double* x, double* ghost, void* stream) {
    IRK_ARG(h && x && (ghost || h->n_ghost == 0), "NULL argument");
    return halo_exchange(h, x, ghost, (cudaStream_t)stream);
}

int irk_dist_op_create(irk_stage_op* op, irk_halo* halo, double* ghost, int64_t interior_lo,
                       int64_t interior_hi, const int32_t* boundary_rows, int64_t nboundary, irk_dist_op** out) {
    IRK_ARG(op && halo && out, "NULL argument");
    IRK_ARG(op->s == halo->s && op->nb == halo->nb, "operator / halo stage count or block size differ");
    IRK_ARG(op->T_local == halo->T_local, "operator T_local differs from the halo's");
    IRK_ARG(op->n_ghost == halo->n_ghost && (halo->n_ghost == 0 || op->ghost == ghost),
            "operator ghost buffer differs (irk_stage_op_set_halo first)");
    IRK_ARG(0 <= interior_lo && interior_lo <= interior_hi && interior_hi <= op->T_local, "bad interior range");
    IRK_ARG(nboundary >= 0 && (nboundary == 0 || boundary_rows), "boundary rows missing");
    IRK_ARG(nboundary + (interior_hi - interior_lo) == op->T_local, "interior + boundary rows must cover the slab");
    auto* d = new irk_dist_op();
    d->op = op;
    d->halo = halo;
    d->ghost = ghost;
    d->r0 = interior_lo;
    d->r1 = interior_hi;
    d->nboundary = nboundary;
    if (nboundary) {
        cudaError_t e = cudaMalloc(&d->d_boundary, sizeof(int32_t) * nboundary);
        if (e == cudaSuccess)
            e = cudaMemcpy(d->d_boundary, boundary_rows, sizeof(int32_t) * nboundary, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(d->d_boundary);
            delete d;
            return fail_cuda(e, "boundary rows upload", __FILE__, __LINE__);
        }
    }
    *out = d;
    return IRK_OK;
}

void irk_dist_op_destroy(irk_dist_op* d) {
    if (!d) return;
    cudaFree(d->d_boundary);
    delete d;
}

int irk_dist_op_apply(const irk_dist_op* d, const double* w, double* y, void* stream) {
    IRK_ARG(d && w && y, "NULL argument");
    return dist_op_apply(d, w, y, (cudaStream_t)stream);
}

int irk_dist_op_factor_apply(const irk_dist_op* d, const irk_factor* f, const double* v, double* x, int* fused,
                             void* stream) {
    IRK_ARG(d && f && v && x, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int rc = dist_op_fused_product(d, f, v, x, st);
    if (rc < 0) return rc;
    if (fused) *fused = rc == 0 ? 1 : 0;
    if (rc == 0) return IRK_OK;
    // not fused: operator on the exchanged halo, then the preconditioner
    double* tmp = nullptr;
    const int64_t n = (int64_t)d->op->s * d->op->T_local * d->op->nb;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * n, st));
    int r2 = irk_stage_op_apply(d->op, v, tmp, st);
    if (r2 == IRK_OK) r2 = irk_factor_apply(f, tmp, x, st);
    cudaFreeAsync(tmp, st);
    return r2;
}

}  // extern "C"
