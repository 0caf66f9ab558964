// Block ILU(0) preconditioner apply: level-scheduled forward / backward
// block-triangular sweeps.
//
// Reference: ilu0_solve (numba_backend.py:75-91) -- unit-lower forward sweep,
// then x_i = D_i^-1 (z_i - sum_{j>i} U_ij x_j) with the explicit inverse --
// and coupled_solve (numba_backend.py:128-151) over the stage-major (k, i)
// grid.  Elements of one dependency level are independent; each level is one
// launch whose CTAs own one element (uncoupled: all s stages together, so a
// shared Jacobian upper block U_ij = -dt*J_ij is read once for s vectors) or
// one (stage, element) pair (coupled, stage-skewed levels lev(i)+k).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "blockops.cuh"
#include "irk_internal.cuh"
#include "pipeline.cuh"

namespace irk {

int choose_groups(int nb, int max_threads);
int permute_out(const double* src_dev, double* dst_dev, int nb, int64_t count, cudaStream_t st);
int permute_in(const double* src_dev, double* dst_dev, int nb, int64_t count, cudaStream_t st);

struct ApplyArgs {
    const int32_t *indptr, *indices, *diag, *lptr, *uptr;
    const uint8_t* keep;
    const double* L;
    const double* Dinv;
    const double* U;          // stored upper blocks [uq][k] or NULL
    const double* ubase[IRK_MAX_STAGES];
    double uscale;
    int u_shared;
    const double* G;          // coupled lower couplings [i][pair]
    const double* Cup;        // stored upper couplings [i][pair] or NULL
    const double* mass;       // implicit upper couplings
    double cup_scale[IRK_MAX_STAGES * IRK_MAX_STAGES];
    const double* y;
    double* x;
    double* W;                 // implicit-L forward sweep: w_i = Dinv_i z_i (s x n) or NULL
    double* Z;                 // deep sentinel sweeps: z_i of the forward sweep (s x n)
    const uint8_t* hasup;      // element has a kept upper block (implicit-L mode)
    unsigned* flags2;          // bwd flags, released by the implicit forward sweep for fused rows
    // persistent sweep: tasks in topological (level) order, claimed by ticket;
    // a task publishes flags[task] = epoch when its output is in memory
    const int32_t* order;
    int64_t ntasks;
    unsigned* flags;
    int* ticket;
    unsigned epoch;
    int64_t T, n;
    int s, nb, G_;
    int fac_shared;            // one factor (s = 1) applied to s right-hand sides
};

__device__ __forceinline__ int pidx(int hi, int lo) { return hi * (hi - 1) / 2 + lo; }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag(const unsigned* f, unsigned epoch) {
    while ((int)(ld_acquire(f) - epoch) < 0) __nanosleep(20);
}

// claim the next task (CTA-uniform); returns -1 when the sweep is done
__device__ __forceinline__ int64_t claim(const ApplyArgs& A, int* s_task) {
    if (threadIdx.x == 0) *s_task = atomicAdd(A.ticket, 1);
    __syncthreads();
    const int64_t t = *s_task;
    return t < A.ntasks ? t : -1;
}

// all writes of the CTA for this task are done -> publish the flag
__device__ __forceinline__ void publish(unsigned* f, unsigned epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release(f, epoch);
    }
}

// ---- uncoupled: one task = one element, all S stages ------------------------
template <int S, bool EVEN>
__global__ void __launch_bounds__(256) k_unc_fwd(ApplyArgs A) {
    extern __shared__ double red[];
    __shared__ int s_task;
    const Geo q = make_geo(A.nb, A.G_);
    const int64_t bsz = (int64_t)A.nb * 2 * q.P;
    for (;;) {
        const int64_t t = claim(A, &s_task);
        if (t < 0) break;
        const int64_t i = A.order[t];
        const int q0 = A.indptr[i], d = A.diag[i], l0 = A.lptr[i];
        if ((int)threadIdx.x < d - q0 && A.keep[q0 + threadIdx.x])
            wait_flag(A.flags + A.indices[q0 + threadIdx.x], A.epoch);
        __syncthreads();
        double part[S];
#pragma unroll
        for (int k = 0; k < S; ++k) part[k] = 0.0;
        if (q.active) {
            for (int qq = q0; qq < d; ++qq) {
                if (!A.keep[qq]) continue;
                const int64_t col = A.indices[qq];
                const double* Lb = A.L + (int64_t)(l0 + qq - q0) * S * bsz;
#pragma unroll
                for (int k = 0; k < S; ++k)
                    part[k] = gemv1<EVEN, true>(Lb + k * bsz, A.x + k * A.n + col * A.nb, q, part[k]);
            }
        }
        double tot[S];
        group_reduce(red, part, S, q, tot);
        if (q.active && q.g == 0) {
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const int64_t o = k * A.n + i * A.nb + q.a;
                A.x[o] = A.y[o] - tot[k];
            }
        }
        publish(A.flags + i, A.epoch);
    }
}

template <int S, bool EVEN>
__global__ void __launch_bounds__(256) k_unc_bwd(ApplyArgs A) {
    extern __shared__ double red[];
    __shared__ int s_task;
    double* tv = red + (int64_t)A.G_ * S * A.nb;   // [S][nb]
    const Geo q = make_geo(A.nb, A.G_);
    const int64_t bsz = (int64_t)A.nb * 2 * q.P;
    for (;;) {
        const int64_t t = claim(A, &s_task);
        if (t < 0) break;
        const int64_t i = A.order[t];
        const int d = A.diag[i], q1 = A.indptr[i + 1], u0 = A.uptr[i];
        if ((int)threadIdx.x < q1 - d - 1 && A.keep[d + 1 + threadIdx.x])
            wait_flag(A.flags + A.indices[d + 1 + threadIdx.x], A.epoch);
        __syncthreads();
        double part[S];
#pragma unroll
        for (int k = 0; k < S; ++k) part[k] = 0.0;
        if (q.active) {
            for (int qq = d + 1; qq < q1; ++qq) {
                if (!A.keep[qq]) continue;
                const int64_t col = A.indices[qq];
                const double* xs[S];
#pragma unroll
                for (int k = 0; k < S; ++k) xs[k] = A.x + k * A.n + col * A.nb;
                if (A.u_shared) {
                    gemv_shared<S, EVEN, true>(A.ubase[0] + qq * bsz, xs, q, part);
                } else if (A.U) {
                    const double* Ub = A.U + (int64_t)(u0 + qq - d - 1) * S * bsz;
#pragma unroll
                    for (int k = 0; k < S; ++k) part[k] = gemv1<EVEN, true>(Ub + k * bsz, xs[k], q, part[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        part[k] = gemv1<EVEN, true>(A.ubase[k] + qq * bsz, xs[k], q, part[k]);
                }
            }
        }
        double tot[S];
        group_reduce(red, part, S, q, tot);
        if (q.active && q.g == 0) {
#pragma unroll
            for (int k = 0; k < S; ++k)
                tv[k * A.nb + q.a] = ld_cg(A.x + k * A.n + i * A.nb + q.a) - A.uscale * tot[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < S; ++k) part[k] = 0.0;
        if (q.active) {
            const double* Db = A.Dinv + i * S * bsz;
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = gemv1<EVEN, false>(Db + k * bsz, tv + k * A.nb, q, part[k]);
        }
        group_reduce(red, part, S, q, tot);
        if (q.active && q.g == 0) {
#pragma unroll
            for (int k = 0; k < S; ++k) A.x[k * A.n + i * A.nb + q.a] = tot[k];
        }
        publish(A.flags + i, A.epoch);
    }
}

// ---- coupled: one task = (stage k, element i); flags indexed k*T + i --------
template <bool EVEN>
__global__ void __launch_bounds__(256) k_cpl_fwd(ApplyArgs A) {
    extern __shared__ double red[];
    __shared__ int s_task;
    const Geo q = make_geo(A.nb, A.G_);
    const int64_t bsz = (int64_t)A.nb * 2 * q.P;
    const int npairs = A.s * (A.s - 1) / 2;
    for (;;) {
        const int64_t t = claim(A, &s_task);
        if (t < 0) break;
        const int64_t code = A.order[t];
        const int k = (int)(code / A.T);
        const int64_t i = code - (int64_t)k * A.T;
        const int q0 = A.indptr[i], d = A.diag[i], l0 = A.lptr[i];
        const int nlo = d - q0;
        const int w = threadIdx.x;
        if (w < nlo) {
            if (A.keep[q0 + w]) wait_flag(A.flags + (int64_t)k * A.T + A.indices[q0 + w], A.epoch);
        } else if (w < nlo + k) {
            wait_flag(A.flags + (int64_t)(w - nlo) * A.T + i, A.epoch);
        }
        __syncthreads();
        double part = 0.0;
        if (q.active) {
            for (int qq = q0; qq < d; ++qq) {
                if (!A.keep[qq]) continue;
                const int64_t col = A.indices[qq];
                part = gemv1<EVEN, true>(A.L + ((int64_t)(l0 + qq - q0) * A.s + k) * bsz,
                                         A.x + k * A.n + col * A.nb, q, part);
            }
            for (int l = 0; l < k; ++l)
                part = gemv1<EVEN, true>(A.G + (i * npairs + pidx(k, l)) * bsz, A.x + l * A.n + i * A.nb, q, part);
        }
        double tot;
        group_reduce(red, &part, 1, q, &tot);
        if (q.active && q.g == 0) {
            const int64_t o = k * A.n + i * A.nb + q.a;
            A.x[o] = A.y[o] - tot;
        }
        publish(A.flags + code, A.epoch);
    }
}

template <bool EVEN>
__global__ void __launch_bounds__(256) k_cpl_bwd(ApplyArgs A) {
    extern __shared__ double red[];
    __shared__ int s_task;
    double* tv = red + (int64_t)A.G_ * 2 * A.nb;
    const Geo q = make_geo(A.nb, A.G_);
    const int64_t bsz = (int64_t)A.nb * 2 * q.P;
    const int npairs = A.s * (A.s - 1) / 2;
    for (;;) {
        const int64_t t = claim(A, &s_task);
        if (t < 0) break;
        const int64_t code = A.order[t];
        const int k = (int)(code / A.T);
        const int64_t i = code - (int64_t)k * A.T;
        const int d = A.diag[i], q1 = A.indptr[i + 1], u0 = A.uptr[i];
        const int nup = q1 - d - 1;
        const int w = threadIdx.x;
        if (w < nup) {
            if (A.keep[d + 1 + w]) wait_flag(A.flags + (int64_t)k * A.T + A.indices[d + 1 + w], A.epoch);
        } else if (w < nup + (A.s - 1 - k)) {
            wait_flag(A.flags + (int64_t)(k + 1 + w - nup) * A.T + i, A.epoch);
        }
        __syncthreads();
        double part[2] = {0.0, 0.0};
        if (q.active) {
            for (int qq = d + 1; qq < q1; ++qq) {
                if (!A.keep[qq]) continue;
                const int64_t col = A.indices[qq];
                const double* Ub = A.U ? A.U + ((int64_t)(u0 + qq - d - 1) * A.s + k) * bsz
                                       : A.ubase[k] + qq * bsz;
                part[0] = gemv1<EVEN, true>(Ub, A.x + k * A.n + col * A.nb, q, part[0]);
            }
            for (int l = k + 1; l < A.s; ++l) {
                const double* xl = A.x + l * A.n + i * A.nb;
                if (A.Cup) {
                    part[1] = gemv1<EVEN, true>(A.Cup + (i * npairs + pidx(l, k)) * bsz, xl, q, part[1]);
                } else {
                    const double v = gemv1<EVEN, true>(A.mass + i * bsz, xl, q, 0.0);
                    part[1] = fma(A.cup_scale[k * A.s + l], v, part[1]);
                }
            }
        }
        double tot[2];
        group_reduce(red, part, 2, q, tot);
        if (q.active && q.g == 0) {
            const double* xi = A.x + k * A.n + i * A.nb;
            tv[q.a] = ld_cg(xi + q.a) - (A.uscale * tot[0] + tot[1]);
        }
        __syncthreads();
        double p2 = 0.0;
        if (q.active) p2 = gemv1<EVEN, false>(A.Dinv + (i * A.s + k) * bsz, tv, q, 0.0);
        double t2;
        group_reduce(red, &p2, 1, q, &t2);
        if (q.active && q.g == 0) A.x[k * A.n + i * A.nb + q.a] = t2;
        publish(A.flags + code, A.epoch);
    }
}

// ---------------------------------------------------------------------------
// Bulk-copy pipelined persistent sweeps (uncoupled, nb even).
// Warp 0 lane 0 (producer) claims tasks in topological order.  For each task
// it (1) waits until the task's x double-buffer slot is free, (2) streams the
// task's factor blocks (fwd: L[lq][k]; bwd: U blocks then Dinv[i][k]) into the
// block ring with cp.async.bulk -- no dependency needed, so the next task's
// blocks are prefetched while the previous task finishes -- then (3) waits for
// the task's dependency flags (ld.acquire.gpu), issues fence.proxy.async and
// (4) bulk-copies the x segments the task multiplies into the x slot.
// Consumer warps take blocks in FIFO order, read x from the slot, reduce and
// store the task's output, publish its flag and free the x slot.
// Deadlock-free: tasks enter every ring in ticket order, dependencies have
// smaller tickets, and a task's x is loaded only after its dependencies.
// ---------------------------------------------------------------------------
enum { PD_FIRST = 1, PD_LAST = 2, PD_END = 4, PD_USH = 8, PD_U = 16, PD_DINV = 32, PD_L = 64, PD_SH = 128 };
// PD_SH: a factor block shared by all right-hand sides (fac_shared), applied to every k

struct PipeCfg {
    int nst;
    int stage_bytes;
    int block_bytes;
    int maxdeg;        // max lower/upper neighbours of a row
    int xslot_doubles; // (maxdeg + 1) * S * nb
};

struct PipeSmem {
    unsigned char* stages;
    uint64_t* full;
    uint64_t* empty;
    uint64_t* xfull;   // [2]
    uint64_t* xempty;  // [2]
    int4* desc;
    double* xs;        // [2][xslot]
    double* red;       // [2][G][S][nb] (task parity)
    double* tv;        // [S][nb]
};

template <int S>
__device__ __forceinline__ PipeSmem pipe_carve(unsigned char* raw, const PipeCfg& PC, int G, int nb) {
    PipeSmem P;
    P.stages = raw;
    P.full = reinterpret_cast<uint64_t*>(raw + (size_t)PC.nst * PC.stage_bytes);
    P.empty = P.full + PC.nst;
    P.xfull = P.empty + PC.nst;
    P.xempty = P.xfull + 2;
    P.desc = reinterpret_cast<int4*>(P.xempty + 2);
    P.xs = reinterpret_cast<double*>(P.desc + PC.nst);
    P.red = P.xs + 2 * (size_t)PC.xslot_doubles;
    P.tv = P.red + 2 * (size_t)G * S * nb;
    return P;
}

__device__ __forceinline__ void pipe_init(PipeSmem& P, int nst, int ncons_warps) {
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(P.full + i, 1);
            mbar_init(P.empty + i, ncons_warps);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(P.xfull + b, 1);
            mbar_init(P.xempty + b, ncons_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct Producer {
    PipeSmem* P;
    const PipeCfg* PC;
    int st = 0;
    uint32_t ph = 0;
    int xb = 0;          // x slot of the current task
    uint32_t xph = 0;    // phase of slot xb
    __device__ void push(int4 d, const double* blk) {
        mbar_wait(P->empty + st, ph ^ 1);
        P->desc[st] = d;
        if (blk) {
            mbar_expect_tx(P->full + st, PC->block_bytes);
            bulk_g2s(P->stages + (size_t)st * PC->stage_bytes, blk, PC->block_bytes, P->full + st);
        } else {
            mbar_expect_tx(P->full + st, 0);
        }
        if (++st == PC->nst) { st = 0; ph ^= 1; }
    }
    __device__ double* x_acquire() {   // wait for the task's x slot to be free
        mbar_wait(P->xempty + xb, xph ^ 1);
        return P->xs + (size_t)xb * PC->xslot_doubles;
    }
    __device__ void x_commit(uint32_t bytes) { mbar_expect_tx(P->xfull + xb, bytes); }
    __device__ void x_next() { xb ^= 1; if (xb == 0) xph ^= 1; }
};

struct Consumer {
    PipeSmem* P;
    const PipeCfg* PC;
    int st = 0;
    uint32_t ph = 0;
    int xb = 0;
    uint32_t xph = 0;
    __device__ int4 take() {
        mbar_wait(P->full + st, ph);
        return P->desc[st];
    }
    __device__ const double2* block() const {
        return reinterpret_cast<const double2*>(P->stages + (size_t)st * PC->stage_bytes);
    }
    __device__ void release() {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(P->empty + st);
        if (++st == PC->nst) { st = 0; ph ^= 1; }
    }
    __device__ const double* x_wait() {
        mbar_wait(P->xfull + xb, xph);
        return P->xs + (size_t)xb * PC->xslot_doubles;
    }
    __device__ void x_release() {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(P->xempty + xb);
        xb ^= 1;
        if (xb == 0) xph ^= 1;
    }
};

// acc += rows of a staged block times an x segment (smem); caller checks q.active
__device__ __forceinline__ double smem_gemv(const double2* B, const double* x, const Geo& q, double acc) {
    for (int p = q.g; p < q.P; p += q.G) {
        const double2 b = B[p * q.nb + q.a];
        const double2 v = *reinterpret_cast<const double2*>(x + 2 * p);
        acc = fma(b.x, v.x, acc);
        acc = fma(b.y, v.y, acc);
    }
    return acc;
}

// acc[k] += rows of a staged block times S x segments x + k * nb: every block
// pair is read from shared memory once for all S vectors
template <int S>
__device__ __forceinline__ void smem_gemv_all(const double2* B, const double* x, const Geo& q, double* acc) {
    for (int p = q.g; p < q.P; p += q.G) {
        const double2 b = B[p * q.nb + q.a];
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const double2 v = *reinterpret_cast<const double2*>(x + k * q.nb + 2 * p);
            acc[k] = fma(b.y, v.y, fma(b.x, v.x, acc[k]));
        }
    }
}

constexpr int MAXD = 8;   // neighbour metadata held in registers per task

// Task ranges: DEPS (persistent, many levels) -> batches of 32 tickets;
// !DEPS (one launch per level) -> a static contiguous slice per CTA.
template <bool DEPS>
__device__ __forceinline__ bool next_batch(const ApplyArgs& A, int& tb, int& tend, int& cur, int hi) {
    const int lane = threadIdx.x & 31;
    if (DEPS) {
        // one ticket at a time: consecutive tickets are mostly independent tasks
        // of one level, which must spread over CTAs for the wavefront to flow
        int v = 0;
        if (lane == 0) v = atomicAdd(A.ticket, 1);
        tb = __shfl_sync(0xffffffffu, v, 0);
        tend = min((int)A.ntasks, tb + 1);
    } else {
        tb = cur;
        cur += 32;
        tend = hi;
    }
    return tb < tend;
}

template <int S, bool DEPS>
__global__ void __launch_bounds__(288) k_unc_fwd_pipe(ApplyArgs A, PipeCfg PC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    PipeSmem P = pipe_carve<S>(smem_raw, PC, A.G_, nb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    pipe_init(P, PC.nst, ncons_warps);
    griddep_launch();
    const int64_t bsz = (int64_t)PC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    if (warp == 0) {
        Producer pr{&P, &PC};
        griddep_wait();   // PDL: CTA set up during the predecessor's drain
        int cur = (int)(A.ntasks * blockIdx.x / gridDim.x);
        const int hi = (int)(A.ntasks * (blockIdx.x + 1) / gridDim.x);
        int tb, tend;
        while (next_batch<DEPS>(A, tb, tend, cur, hi)) {
            // warp-parallel metadata prefetch: lane l <-> task tb + l
            const int tl = tb + lane;
            const bool valid = tl < tend;
            const int64_t il = valid ? A.order[tl] : 0;
            const int q0l = valid ? A.indptr[il] : 0, dl = valid ? A.diag[il] : 0, l0l = valid ? A.lptr[il] : 0;
            const int nnl = dl - q0l;
            int coll[MAXD];
            unsigned kml = 0;
#pragma unroll
            for (int m = 0; m < MAXD; ++m) {
                coll[m] = 0;
                if (m < nnl) { coll[m] = A.indices[q0l + m]; kml |= (A.keep[q0l + m] ? 1u : 0u) << m; }
            }
            for (int bt = 0; bt < 32 && tb + bt < tend; ++bt) {
                const int t = tb + bt;
                const int64_t i = __shfl_sync(0xffffffffu, il, bt);
                const int q0 = __shfl_sync(0xffffffffu, q0l, bt), nn = __shfl_sync(0xffffffffu, nnl, bt);
                const int l0 = __shfl_sync(0xffffffffu, l0l, bt);
                unsigned km = __shfl_sync(0xffffffffu, kml, bt);
                int col[MAXD];
#pragma unroll
                for (int m = 0; m < MAXD; ++m) col[m] = __shfl_sync(0xffffffffu, coll[m], bt);
                if (nn > MAXD) {   // rare: wide rows, read directly
                    km = 0;
                    for (int m = 0; m < nn && m < 32; ++m) km |= (A.keep[q0 + m] ? 1u : 0u) << m;
                }
                auto colm = [&](int m) -> int64_t {
                    if (m < MAXD) {
                        int v = 0;
#pragma unroll
                        for (int mm = 0; mm < MAXD; ++mm) v = (mm == m) ? col[mm] : v;
                        return v;
                    }
                    return A.indices[q0 + m];
                };
                auto kept = [&](int m) -> bool { return m < 32 ? ((km >> m) & 1u) : A.keep[q0 + m] != 0; };
                // item n of the task: (kept neighbour, stage) in order
                const int SF = A.fac_shared ? 1 : S;   // factor blocks per neighbour
                int nitems = 0;
                for (int m = 0; m < nn; ++m) nitems += kept(m) ? SF : 0;
                auto push_items = [&](int from, int to) {
                    if (nitems == 0) {
                        if (from == 0 && to > 0) pr.push(make_int4((int)i, -1, PD_FIRST | PD_LAST, nn), nullptr);
                        return;
                    }
                    int n = 0;
                    for (int m = 0; m < nn; ++m) {
                        if (!kept(m)) continue;
                        for (int k = 0; k < SF; ++k, ++n) {
                            if (n < from || n >= to) continue;
                            const int fl = PD_L | (n == 0 ? PD_FIRST : 0) | (n == nitems - 1 ? PD_LAST : 0) |
                                           (A.fac_shared ? PD_SH : 0);
                            pr.push(make_int4((int)i, m * S + k, fl, nn), A.L + ((int64_t)(l0 + m) * SF + k) * bsz);
                        }
                    }
                };
                const int ntot = nitems > 0 ? nitems : 1;
                // blocks pushed before x is committed: consumers block on x at the
                // task's first item, so at most nst - 1 may precede the commit
                const int npre = DEPS ? min(ntot, PC.nst - 1) : 0;
                double* xs = nullptr;
                int xb = 0;
                if (lane == 0) {
                    xs = pr.x_acquire();
                    xb = pr.xb;
                    push_items(0, npre);
                }
                // dependencies (one lane per neighbour), then the x segments z_{k,j}
                if (DEPS)
                    for (int m = lane; m < nn; m += 32)
                        if (kept(m)) wait_flag(A.flags + colm(m), A.epoch);
                __syncwarp();
                uint32_t bytes = S * seg;   // y_i (segments nn*S + k)
                for (int m = 0; m < nn; ++m) bytes += kept(m) ? S * seg : 0;
                if (lane == 0) {
                    if (DEPS) fence_proxy_async_global();
                    pr.x_commit(bytes);
                }
                xs = reinterpret_cast<double*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(xs), 0));
                xb = __shfl_sync(0xffffffffu, xb, 0);
                __syncwarp();
                for (int e = lane; e < (nn + 1) * S; e += 32) {
                    const int m = e / S, k = e - m * S;
                    if (m == nn) bulk_g2s(xs + e * nb, A.y + k * A.n + i * nb, seg, P.xfull + xb);
                    else if (kept(m)) bulk_g2s(xs + e * nb, A.x + k * A.n + colm(m) * nb, seg, P.xfull + xb);
                }
                if (lane == 0) push_items(npre, ntot);
                if (lane == 0) pr.x_next();
            }
        }
        if (lane == 0) pr.push(make_int4(-1, 0, PD_END, 0), nullptr);
        return;
    }
    const int c = threadIdx.x - 32;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = A.G_; q.g = c / nb; q.a = c - q.g * nb; q.active = q.g < q.G;
    Consumer cs{&P, &PC};
    griddep_wait();
    double part[S];
    const double* xs = nullptr;
    int par = 0;   // reduction buffer of the current task
    for (;;) {
        const int4 dsc = cs.take();
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;   // element id (descriptor)
        const int nn = dsc.w;      // lower neighbours: y_i sits at x-slot segment nn*S + k
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
            xs = cs.x_wait();
        }
        if (dsc.y >= 0 && q.active) {
            const int m = dsc.y / S, kk = dsc.y - m * S;
            const double2* B = cs.block();
            if (dsc.z & PD_SH) {
                smem_gemv_all<S>(B, xs + m * S * nb, q, part);
            } else {
#pragma unroll
                for (int k = 0; k < S; ++k)
                    if (k == kk) part[k] = smem_gemv(B, xs + (m * S + k) * nb, q, part[k]);
            }
        }
        cs.release();
        if (dsc.z & PD_LAST) {
            if (dsc.y < 0) {
                // no kept lower neighbour: z_i = y_i, no reduction
                if (q.active && q.g == 0)
#pragma unroll
                    for (int k = 0; k < S; ++k) A.x[k * A.n + i * nb + q.a] = xs[(nn * S + k) * nb + q.a];
                cs.x_release();
                if (DEPS) {
                    consumer_sync(1, ncons);
                    if (c == 0) { __threadfence(); st_release(A.flags + i, A.epoch); }
                }
                continue;
            }
            // one barrier per task: the reduction buffer alternates with the task
            // parity, and the next barrier orders the reads before its reuse
            double* red = P.red + (size_t)par * q.G * S * nb;
            par ^= 1;
            if (q.active)
#pragma unroll
                for (int k = 0; k < S; ++k) red[(q.g * S + k) * nb + q.a] = part[k];
            consumer_sync(1, ncons);
            if (q.active && q.g == 0) {
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    double sum = 0.0;
                    for (int gg = 0; gg < q.G; ++gg) sum += red[(gg * S + k) * nb + q.a];
                    A.x[k * A.n + i * nb + q.a] = xs[(nn * S + k) * nb + q.a] - sum;
                }
            }
            cs.x_release();
            if (DEPS) {
                consumer_sync(1, ncons);
                if (c == 0) { __threadfence(); st_release(A.flags + i, A.epoch); }
            }
        }
    }
}

// FWDI = false: backward sweep x_i = Dinv_i (z_i - uscale sum_{j>i} J_ij x_j).
// FWDI = true (implicit-L forward sweep, stage-shared J): t_i = y_i - alpha
// sum_{j<i} J_ij w_j with w_j = Dinv_j z_j; then z_i = t_i and w_i = Dinv_i z_i
// for rows with a kept upper block (their backward task follows), else the
// row is finished here: x_i = Dinv_i z_i (fused backward step).
template <int S, bool DEPS, bool FWDI>
__global__ void __launch_bounds__(288) k_unc_bwd_pipe(ApplyArgs A, PipeCfg PC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    PipeSmem P = pipe_carve<S>(smem_raw, PC, A.G_, nb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    pipe_init(P, PC.nst, ncons_warps);
    griddep_launch();
    const int64_t bsz = (int64_t)PC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    if (warp == 0) {
        Producer pr{&P, &PC};
        griddep_wait();   // PDL: CTA set up during the predecessor's drain
        int cur = (int)(A.ntasks * blockIdx.x / gridDim.x);
        const int hi = (int)(A.ntasks * (blockIdx.x + 1) / gridDim.x);
        int tb, tend;
        while (next_batch<DEPS>(A, tb, tend, cur, hi)) {
            const int tl = tb + lane;
            const bool valid = tl < tend;
            const int64_t il = valid ? A.order[tl] : 0;
            const int dl = valid ? A.diag[il] : 0, u0l = valid ? A.uptr[il] : 0;
            // neighbour range: upper (d, q1) for the backward sweep, lower [q0, d) for FWDI
            const int b0l = valid ? (FWDI ? A.indptr[il] : dl + 1) : 0;
            const int nnl = valid ? (FWDI ? dl : A.indptr[il + 1]) - b0l : 0;
            const int szl = (FWDI && valid && A.hasup[il]) ? 1 : 0;
            int coll[MAXD];
            unsigned kml = 0;
#pragma unroll
            for (int m = 0; m < MAXD; ++m) {
                coll[m] = 0;
                if (m < nnl) { coll[m] = A.indices[b0l + m]; kml |= (A.keep[b0l + m] ? 1u : 0u) << m; }
            }
            for (int bt = 0; bt < 32 && tb + bt < tend; ++bt) {
                const int t = tb + bt;
                const int64_t i = __shfl_sync(0xffffffffu, il, bt);
                const int nn = __shfl_sync(0xffffffffu, nnl, bt);
                const int b0 = __shfl_sync(0xffffffffu, b0l, bt);
                const int u0 = __shfl_sync(0xffffffffu, u0l, bt);
                const int store_z = __shfl_sync(0xffffffffu, szl, bt);
                unsigned km = __shfl_sync(0xffffffffu, kml, bt);
                int col[MAXD];
#pragma unroll
                for (int m = 0; m < MAXD; ++m) col[m] = __shfl_sync(0xffffffffu, coll[m], bt);
                if (nn > MAXD) {
                    km = 0;
                    for (int m = 0; m < nn && m < 32; ++m) km |= (A.keep[b0 + m] ? 1u : 0u) << m;
                }
                auto colm = [&](int m) -> int64_t {
                    if (m < MAXD) {
                        int v = 0;
#pragma unroll
                        for (int mm = 0; mm < MAXD; ++mm) v = (mm == m) ? col[mm] : v;
                        return v;
                    }
                    return A.indices[b0 + m];
                };
                auto kept = [&](int m) -> bool { return m < 32 ? ((km >> m) & 1u) : A.keep[b0 + m] != 0; };
                const bool ush = A.u_shared || A.fac_shared;
                const int nd = A.fac_shared ? 1 : S;   // Dinv items
                int nu = 0;
                for (int m = 0; m < nn; ++m) nu += kept(m) ? (ush ? 1 : S) : 0;
                const int ntot = nu + nd;
                auto push_items = [&](int from, int to) {
                    int n = 0;
                    for (int m = 0; m < nn; ++m) {
                        if (!kept(m)) continue;
                        const int qq = b0 + m;
                        if (ush) {
                            if (n >= from && n < to)
                                pr.push(make_int4((int)i, m * S, PD_USH | (n == 0 ? PD_FIRST : 0), nn << 2),
                                        A.U ? A.U + (int64_t)(u0 + m) * bsz : A.ubase[0] + qq * bsz);
                            ++n;
                        } else {
                            for (int k = 0; k < S; ++k, ++n) {
                                if (n < from || n >= to) continue;
                                const double* ub = A.U ? A.U + ((int64_t)(u0 + m) * S + k) * bsz : A.ubase[k] + qq * bsz;
                                pr.push(make_int4((int)i, m * S + k, PD_U | (n == 0 ? PD_FIRST : 0), nn << 2), ub);
                            }
                        }
                    }
                    for (int k = 0; k < nd; ++k, ++n) {
                        if (n < from || n >= to) continue;
                        const int fl = PD_DINV | (n == 0 ? PD_FIRST : 0) | (k == nd - 1 ? PD_LAST : 0) |
                                       (A.fac_shared ? PD_SH : 0);
                        pr.push(make_int4((int)i, k, fl, (nn << 2) | (store_z << 1) | (nu == 0 ? 1 : 0)), A.Dinv + (i * nd + k) * bsz);
                    }
                };
                const int npre = DEPS ? min(ntot, PC.nst - 1) : 0;
                double* xs = nullptr;
                int xb = 0;
                if (lane == 0) {
                    xs = pr.x_acquire();
                    xb = pr.xb;
                    push_items(0, npre);
                }
                if (DEPS)
                    for (int m = lane; m < nn; m += 32)
                        if (kept(m)) wait_flag(A.flags + colm(m), A.epoch);
                __syncwarp();
                uint32_t bytes = S * seg;
                for (int m = 0; m < nn; ++m) bytes += kept(m) ? S * seg : 0;
                if (lane == 0) {
                    if (DEPS) fence_proxy_async_global();
                    pr.x_commit(bytes);
                }
                xs = reinterpret_cast<double*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(xs), 0));
                xb = __shfl_sync(0xffffffffu, xb, 0);
                __syncwarp();
                for (int e = lane; e < (nn + 1) * S; e += 32) {
                    const int m = e / S, k = e - m * S;
                    // own segment: z_i (backward) or y_i (FWDI); neighbours: x_j (backward) or w_j (FWDI)
                    if (m == nn) bulk_g2s(xs + e * nb, (FWDI ? A.y : A.x) + k * A.n + i * nb, seg, P.xfull + xb);
                    else if (kept(m)) bulk_g2s(xs + e * nb, (FWDI ? A.W : A.x) + k * A.n + colm(m) * nb, seg, P.xfull + xb);
                }
                if (lane == 0) push_items(npre, ntot);
                if (lane == 0) pr.x_next();
            }
        }
        if (lane == 0) pr.push(make_int4(-1, 0, PD_END, 0), nullptr);
        return;
    }
    // Consumers: warp-shuffle reduction layout.  G (1, 2 or 4) groups split the column
    // pairs; warp w holds rows [R w, R w + R), R = 32 / G, lane = g R + (row - R w): every
    // quarter-warp reads 8 distinct block rows (conflict-free 128-bit LDS) and the G partial
    // sums of a row sit in lanes R apart (shfl_xor reduction, no shared-memory buffer).
    const int c = threadIdx.x - 32;
    const int G = A.G_, R = 32 / G;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = G;
    q.a = R * (c >> 5) + (c & (R - 1));
    q.g = (c & 31) / R;
    q.active = q.a < nb;
    auto group_sum = [&](double v) -> double {
        for (int o = R; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    Consumer cs{&P, &PC};
    griddep_wait();
    double part[S];
    const double* xs = nullptr;
    int par = 0;
    for (;;) {
        const int4 dsc = cs.take();
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;     // element id and upper-neighbour count from the descriptor
        double* tv = P.red + (size_t)par * S * nb;       // t of this task (task-parity double buffer)
        const int nup = dsc.w >> 2;                     // neighbour count: own segment index
        const bool store_z = FWDI && ((dsc.w >> 1) & 1);  // FWDI row with a backward task
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
            xs = cs.x_wait();
        }
        const double2* B = cs.block();
        if (dsc.z & PD_USH) {
            if (q.active) smem_gemv_all<S>(B, xs + (dsc.y / S) * S * nb, q, part);
        } else if (dsc.z & PD_U) {
            if (q.active) {
                const int m = dsc.y / S, kk = dsc.y - m * S;
#pragma unroll
                for (int k = 0; k < S; ++k)
                    if (k == kk) part[k] = smem_gemv(B, xs + (m * S + k) * nb, q, part[k]);
            }
        } else {  // Dinv item k
            const int kk = dsc.y;
            const bool no_upper = (dsc.z & PD_FIRST) || (dsc.w & 1);
            if (kk == 0 && no_upper) {
                // no kept neighbour block: t = own segment, read straight from the x slot
#pragma unroll
                for (int k = 0; k < S; ++k) part[k] = 0.0;
                if (store_z && q.active && q.g == 0)
#pragma unroll
                    for (int k = 0; k < S; ++k) A.x[k * A.n + i * nb + q.a] = xs[(nup * S + k) * nb + q.a];
            } else if (kk == 0) {
                // t_k = z_{i,k} - uscale * sum_j U_ij x_{j,k}  (all stages)
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    const double sum = group_sum(part[k]);
                    if (q.active && q.g == 0) {
                        const double tval = xs[(nup * S + k) * nb + q.a] - A.uscale * sum;
                        tv[k * nb + q.a] = tval;
                        if (store_z) A.x[k * A.n + i * nb + q.a] = tval;   // z_i for the backward sweep
                    }
                    part[k] = 0.0;
                }
                consumer_sync(1, ncons);
            }
            if (q.active) {
                const bool direct = (dsc.w & 1) != 0;
                const double* xv = direct ? xs + nup * S * nb : tv;
                if (dsc.z & PD_SH) {
                    smem_gemv_all<S>(B, xv, q, part);
                } else {
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        if (k == kk) part[k] = smem_gemv(B, xv + k * nb, q, part[k]);
                }
            }
        }
        cs.release();
        if (dsc.z & PD_LAST) {
            par ^= 1;
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const double sum = group_sum(part[k]);
                if (q.active && q.g == 0) (store_z ? A.W : A.x)[k * A.n + i * nb + q.a] = sum;
            }
            cs.x_release();
            if (DEPS) {
                consumer_sync(1, ncons);
                if (c == 0) {
                    __threadfence();
                    st_release(A.flags + i, A.epoch);
                    if (FWDI && !store_z) st_release(A.flags2 + i, A.epoch);   // row finished here
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Deep schedules (natural numbering: hundreds of dependency levels, ~T / levels tasks
// each): the sweep time is the level-to-level hand-over latency, not bandwidth.
// k_unc_bwd_pipe hands a task through a chain of hops -- producer polls the flags,
// bulk-copies the neighbours' segments into an x slot, the consumers take the ring
// items one by one with an mbarrier handshake each.  k_unc_deep is the short chain for
// the implicit-L, stage-shared-J case: a producer warp runs up to two tasks ahead
// (ticket, metadata, ALL blocks of the task in one shared-memory buffer, one mbarrier);
// thread (stage k, row a) of the consumers polls the flags itself, loads the neighbour
// segments straight from L2 (ld.cg: lines are shared with segments still being
// written), and does its row of both gemv phases from shared memory:
//   t = own - uscale sum_j B_ij v_j   (v = w_j forward / x_j backward),  out = Dinv_k t.
// Three CTA-wide barriers per task.  Deadlock-free: a CTA processes its tickets in
// order, so the smallest unfinished ticket is always some CTA's current task.
// ---------------------------------------------------------------------------
struct DeepCfg {
    int block_bytes;
    int buf_bytes;     // (maxdeg + S) blocks
    int maxdeg;
    int nbuf;          // task buffers (k_cpl_deep_sent; k_unc_deep* always use two)
};

struct DeepDesc {
    int i, nn, store_z;
    unsigned km;
    int col[MAXD];
};

template <int S, bool FWDI>
__global__ void __launch_bounds__(512) k_unc_deep(ApplyArgs A, DeepCfg DC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb, P = nb >> 1;
    unsigned char* bufs = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + 2 * (size_t)DC.buf_bytes);
    uint64_t* empty = full + 2;
    DeepDesc* desc = reinterpret_cast<DeepDesc*>(empty + 2);          // 2 x 48 B
    double* xs = reinterpret_cast<double*>(smem_raw + 2 * (size_t)DC.buf_bytes + 128);   // [maxdeg][S][nb]
    double* ts = xs + (size_t)DC.maxdeg * S * nb;                                         // [S][nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons = (int)blockDim.x - 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(full + b, 1);
            mbar_init(empty + b, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    const int64_t bsz = (int64_t)DC.block_bytes / 8;
    if (warp == 0) {
        griddep_wait();
        int b = 0;
        uint32_t ph = 0;
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(A.ticket, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            const bool end = t >= A.ntasks;
            int i = -1, b0 = 0, nn = 0, sz = 0;
            if (!end) {
                i = A.order[t];
                const int d = A.diag[i];
                b0 = FWDI ? A.indptr[i] : d + 1;
                nn = (FWDI ? d : A.indptr[i + 1]) - b0;
                sz = (FWDI && A.hasup[i]) ? 1 : 0;
            }
            int colm = 0, kp = 0;
            if (lane < nn && lane < MAXD) {
                colm = A.indices[b0 + lane];
                kp = A.keep[b0 + lane] ? 1 : 0;
            }
            const unsigned km = __ballot_sync(0xffffffffu, kp != 0);
            if (lane == 0) mbar_wait(empty + b, ph ^ 1);
            __syncwarp();
            if (lane == 0) {
                desc[b].i = i;
                desc[b].nn = nn;
                desc[b].store_z = sz;
                desc[b].km = km;
            }
            if (lane < MAXD) desc[b].col[lane] = colm;
            __syncwarp();
            if (lane == 0) {
                if (end) {
                    mbar_expect_tx(full + b, 0);
                } else {
                    const int nkept = __popc(km);
                    mbar_expect_tx(full + b, (uint32_t)(nkept + S) * (uint32_t)DC.block_bytes);
                    unsigned char* dst = bufs + (size_t)b * DC.buf_bytes;
                    for (int m = 0; m < nn; ++m)
                        if ((km >> m) & 1u) {
                            bulk_g2s(dst, A.ubase[0] + (int64_t)(b0 + m) * bsz, DC.block_bytes, full + b);
                            dst += DC.block_bytes;
                        }
                    for (int k = 0; k < S; ++k, dst += DC.block_bytes)
                        bulk_g2s(dst, A.Dinv + ((int64_t)i * S + k) * bsz, DC.block_bytes, full + b);
                }
            }
            if (end) break;
            b ^= 1;
            if (b == 0) ph ^= 1;
        }
        return;
    }
    const int c = threadIdx.x - 32;
    const int k = c / nb, a = c - k * nb;
    const bool act = k < S;
    // row a of a staged block times a shared-memory vector: four independent accumulators and
    // the loads of two column pairs ahead of their FMAs (these two gemv phases sit on the
    // level-to-level critical path: 0.95 + 0.49 us per task with a 2-accumulator loop)
    auto row_dot = [&](const unsigned char* blk, const double* xv) -> double {
        const double2* B = reinterpret_cast<const double2*>(blk) + a;
        const double2* X = reinterpret_cast<const double2*>(xv);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int p = 0;
#pragma unroll 5
        for (; p + 2 <= P; p += 2) {
            const double2 b0 = B[p * nb], b1 = B[(p + 1) * nb];
            const double2 v0 = X[p], v1 = X[p + 1];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
            s2 = fma(b1.x, v1.x, s2);
            s3 = fma(b1.y, v1.y, s3);
        }
        if (p < P) {
            const double2 b0 = B[p * nb];
            const double2 v0 = X[p];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
        }
        return (s0 + s1) + (s2 + s3);
    };
    griddep_wait();
    int b = 0;
    uint32_t ph = 0;
    for (;;) {
        mbar_wait(full + b, ph);
        const int64_t i = desc[b].i;
        if (i < 0) break;
        const int nn = desc[b].nn;
        const unsigned km = desc[b].km;
        const bool store_z = FWDI && desc[b].store_z != 0;
        const int nkept = __popc(km);
        // dependencies: consumer thread m polls neighbour m
        if (c < nn && ((km >> c) & 1u)) wait_flag(A.flags + desc[b].col[c], A.epoch);
        consumer_sync(1, ncons);
        double own = 0.0;
        if (act) {
            const double* vsrc = (FWDI ? A.W : A.x) + (int64_t)k * A.n + a;
            own = __ldcg((FWDI ? A.y : A.x) + (int64_t)k * A.n + i * nb + a);
            int slot = 0;
            for (int m = 0; m < nn; ++m)
                if ((km >> m) & 1u) {
                    xs[(slot * S + k) * nb + a] = __ldcg(vsrc + (int64_t)desc[b].col[m] * nb);
                    ++slot;
                }
        }
        consumer_sync(1, ncons);
        const unsigned char* buf = bufs + (size_t)b * DC.buf_bytes;
        if (act) {
            double sum = 0.0;
            for (int slot = 0; slot < nkept; ++slot)
                sum += row_dot(buf + (size_t)slot * DC.block_bytes, xs + (slot * S + k) * nb);
            const double tval = nkept ? own - A.uscale * sum : own;
            ts[k * nb + a] = tval;
            if (store_z) A.x[(int64_t)k * A.n + i * nb + a] = tval;   // z_i for the backward sweep
        }
        consumer_sync(1, ncons);
        if (act) {
            (store_z ? A.W : A.x)[(int64_t)k * A.n + i * nb + a] =
                row_dot(buf + (size_t)(nkept + k) * DC.block_bytes, ts + k * nb);
        }
        consumer_sync(1, ncons);   // outputs issued; buffer, xs and ts are free
        if (c == 0) {
            __threadfence();
            st_release(A.flags + i, A.epoch);
            if (FWDI && !store_z) st_release(A.flags2 + i, A.epoch);   // row finished here
            mbar_arrive(empty + b);
        }
        b ^= 1;
        if (b == 0) ph ^= 1;
    }
}

// k_unc_deep with self-validating values instead of flags.  The hand-over of k_unc_deep costs
// three L2 round trips per level -- the producer's __threadfence before the flag (0.83 us), the
// flag reaching the poller (~1.1 us), the segment load after it (0.83 us).  Here the outputs a
// sweep will write (w for the forward sweep, x for both) are pre-filled with a NaN bit pattern no
// computation produces, consumers spin on the VALUES they need (ld.relaxed.gpu, one per thread
// and neighbour; the addresses are spread over the vector, no hot line) and outputs are plain
// 8-byte stores: one round trip per level, no fence, no flag.  Every entry of w / x is written
// exactly once per apply, which is why z_i (needed by the backward sweep) goes to its own buffer
// Z instead of the x slot.  x must not alias y (the caller falls back to k_unc_deep).
constexpr unsigned long long DEEP_SENTINEL = 0xFFF8DEADBEEF5EEDULL;

__global__ void k_fill_sentinel(double* __restrict__ a, double* __restrict__ b, int64_t n) {
    const double sv = __longlong_as_double((long long)DEEP_SENTINEL);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        a[e] = sv;
        if (b) b[e] = sv;
    }
}

// Bounded spin (2^22 polls of ~0.7 us, normal waits are a few of them): a value that never arrives --
// only possible if an input vector carried the sentinel pattern itself, whose NaN payload the
// arithmetic would propagate into an output -- ends as NaN in the result instead of a hung GPU.
__device__ __forceinline__ double poll_value(const double* p) {
    unsigned long long v = DEEP_SENTINEL;
    for (int it = 0; it < (1 << 22) && v == DEEP_SENTINEL; ++it)
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void publish_value(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" :: "l"(p), "d"(v) : "memory");
}

template <int S, bool FWDI>
__global__ void __launch_bounds__(512) k_unc_deep_sent(ApplyArgs A, DeepCfg DC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb, P = nb >> 1;
    unsigned char* bufs = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + 2 * (size_t)DC.buf_bytes);
    uint64_t* empty = full + 2;
    DeepDesc* desc = reinterpret_cast<DeepDesc*>(empty + 2);
    double* xs = reinterpret_cast<double*>(smem_raw + 2 * (size_t)DC.buf_bytes + 128);   // [maxdeg][S][nb]
    double* ts = xs + (size_t)DC.maxdeg * S * nb;                                         // [S][nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons = (int)blockDim.x - 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(full + b, 1);
            mbar_init(empty + b, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    const int64_t bsz = (int64_t)DC.block_bytes / 8;
    if (warp == 0) {
        griddep_wait();
        int b = 0;
        uint32_t ph = 0;
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(A.ticket, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            const bool end = t >= A.ntasks;
            int i = -1, b0 = 0, nn = 0, sz = 0;
            if (!end) {
                i = A.order[t];
                const int d = A.diag[i];
                b0 = FWDI ? A.indptr[i] : d + 1;
                nn = (FWDI ? d : A.indptr[i + 1]) - b0;
                sz = (FWDI && A.hasup[i]) ? 1 : 0;
            }
            int colm = 0, kp = 0;
            if (lane < nn && lane < MAXD) {
                colm = A.indices[b0 + lane];
                kp = A.keep[b0 + lane] ? 1 : 0;
            }
            const unsigned km = __ballot_sync(0xffffffffu, kp != 0);
            if (lane == 0) mbar_wait(empty + b, ph ^ 1);
            __syncwarp();
            if (lane == 0) {
                desc[b].i = i;
                desc[b].nn = nn;
                desc[b].store_z = sz;
                desc[b].km = km;
            }
            if (lane < MAXD) desc[b].col[lane] = colm;
            __syncwarp();
            if (lane == 0) {
                if (end) {
                    mbar_expect_tx(full + b, 0);
                } else {
                    const int nkept = __popc(km);
                    mbar_expect_tx(full + b, (uint32_t)(nkept + S) * (uint32_t)DC.block_bytes);
                    unsigned char* dst = bufs + (size_t)b * DC.buf_bytes;
                    for (int m = 0; m < nn; ++m)
                        if ((km >> m) & 1u) {
                            bulk_g2s(dst, A.ubase[0] + (int64_t)(b0 + m) * bsz, DC.block_bytes, full + b);
                            dst += DC.block_bytes;
                        }
                    for (int k = 0; k < S; ++k, dst += DC.block_bytes)
                        bulk_g2s(dst, A.Dinv + ((int64_t)i * S + k) * bsz, DC.block_bytes, full + b);
                }
            }
            if (end) break;
            b ^= 1;
            if (b == 0) ph ^= 1;
        }
        return;
    }
    const int c = threadIdx.x - 32;
    const int k = c / nb, a = c - k * nb;
    const bool act = k < S;
    auto row_dot = [&](const unsigned char* blk, const double* xv) -> double {
        const double2* B = reinterpret_cast<const double2*>(blk) + a;
        const double2* X = reinterpret_cast<const double2*>(xv);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int p = 0;
#pragma unroll 5
        for (; p + 2 <= P; p += 2) {
            const double2 b0 = B[p * nb], b1 = B[(p + 1) * nb];
            const double2 v0 = X[p], v1 = X[p + 1];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
            s2 = fma(b1.x, v1.x, s2);
            s3 = fma(b1.y, v1.y, s3);
        }
        if (p < P) {
            const double2 b0 = B[p * nb];
            const double2 v0 = X[p];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
        }
        return (s0 + s1) + (s2 + s3);
    };
    griddep_wait();
    int b = 0;
    uint32_t ph = 0;
    for (;;) {
        mbar_wait(full + b, ph);
        const int64_t i = desc[b].i;
        if (i < 0) break;
        const int nn = desc[b].nn;
        const unsigned km = desc[b].km;
        const bool store_z = FWDI && desc[b].store_z != 0;
        const int nkept = __popc(km);
        // gather: the task's own segment (complete before this launch) and, by polling the values,
        // the neighbours' segments
        double own = 0.0;
        if (act) {
            own = __ldcg((FWDI ? A.y : A.Z) + (int64_t)k * A.n + i * nb + a);
            const double* vsrc = (FWDI ? A.W : A.x) + (int64_t)k * A.n + a;
            int slot = 0;
            for (int m = 0; m < nn; ++m)
                if ((km >> m) & 1u) {
                    xs[(slot * S + k) * nb + a] = poll_value(vsrc + (int64_t)desc[b].col[m] * nb);
                    ++slot;
                }
        }
        consumer_sync(1, ncons);
        const unsigned char* buf = bufs + (size_t)b * DC.buf_bytes;
        if (act) {
            double sum = 0.0;
            for (int slot = 0; slot < nkept; ++slot)
                sum += row_dot(buf + (size_t)slot * DC.block_bytes, xs + (slot * S + k) * nb);
            const double tval = nkept ? own - A.uscale * sum : own;
            ts[k * nb + a] = tval;
            if (store_z) A.Z[(int64_t)k * A.n + i * nb + a] = tval;   // z_i for the backward sweep
        }
        consumer_sync(1, ncons);
        if (act)
            publish_value((store_z ? A.W : A.x) + (int64_t)k * A.n + i * nb + a,
                          row_dot(buf + (size_t)(nkept + k) * DC.block_bytes, ts + k * nb));
        consumer_sync(1, ncons);   // buffer, xs and ts are free
        if (c == 0) mbar_arrive(empty + b);
        b ^= 1;
        if (b == 0) ph ^= 1;
    }
}

// Stage-coupled sweeps on a deep schedule with self-validating values (coupled_solve,
// numba_backend.py:128-151; the reference's default preconditioner on its natural numbering).
// Tasks are the (stage k, element i) pairs of the stage-skewed schedule (k_cpl_fwd / k_cpl_bwd
// semantics):
//   forward   z_ki = y_ki - sum_{j lower} L_{k,ij} z_kj - sum_{l<k} G_{kl,i} z_li
//   backward  x_ki = Dinv_ki ( z_ki - uscale sum_{j upper} U_ij x_kj - sum_{l>k} C_{kl,i} x_li ),
//             C_{kl,i} = cup_scale[k][l] M_i (implicit) or the stored blocks
// z goes to its own buffer Z, so that every entry of Z (forward) and x (backward) is written once
// and can be polled; both are pre-filled with the sentinel.  One thread per block row, a producer
// warp one task ahead (all blocks of the task in one buffer, one mbarrier).
struct CplDeepDesc {
    int k, i, nn;
    unsigned km;
    int col[MAXD];
};

template <bool FWD>
__global__ void __launch_bounds__(160) k_cpl_deep_sent(ApplyArgs A, DeepCfg DC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb, P = nb >> 1, S = A.s;
    const int npairs = S * (S - 1) / 2;
    unsigned char* bufs = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)DC.nbuf * DC.buf_bytes);
    uint64_t* empty = full + 2;
    CplDeepDesc* desc = reinterpret_cast<CplDeepDesc*>(empty + 2);   // 2 x 48 B
    double* xs = reinterpret_cast<double*>(smem_raw + (size_t)DC.nbuf * DC.buf_bytes + 128);   // [maxdeg + S][nb]
    double* tv = xs + (size_t)(DC.maxdeg + S) * nb;                                            // [nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons = (int)blockDim.x - 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(full + b, 1);
            mbar_init(empty + b, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t bsz = (int64_t)DC.block_bytes / 8;
    if (warp == 0) {
        int b = 0;
        uint32_t ph = 0;
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(A.ticket, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            const bool end = t >= A.ntasks;
            int k = 0, i = -1, b0 = 0, nn = 0, d = 0, l0 = 0, u0 = 0;
            if (!end) {
                const int64_t code = A.order[t];
                k = (int)(code / A.T);
                i = (int)(code - (int64_t)k * A.T);
                d = A.diag[i];
                b0 = FWD ? A.indptr[i] : d + 1;
                nn = (FWD ? d : A.indptr[i + 1]) - b0;
                l0 = A.lptr[i];
                u0 = A.uptr[i];
            }
            int colm = 0, kp = 0;
            if (lane < nn && lane < MAXD) {
                colm = A.indices[b0 + lane];
                kp = A.keep[b0 + lane] ? 1 : 0;
            }
            const unsigned km = __ballot_sync(0xffffffffu, kp != 0);
            if (lane == 0) mbar_wait(empty + b, ph ^ 1);
            __syncwarp();
            if (lane == 0) {
                desc[b].k = k;
                desc[b].i = i;
                desc[b].nn = nn;
                desc[b].km = km;
            }
            if (lane < MAXD) desc[b].col[lane] = colm;
            __syncwarp();
            if (lane == 0) {
                if (end) {
                    mbar_expect_tx(full + b, 0);
                } else {
                    const int nkept = __popc(km);
                    const int ncpl = FWD ? k : (A.Cup ? S - 1 - k : (k < S - 1 ? 1 : 0));
                    mbar_expect_tx(full + b, (uint32_t)(nkept + ncpl + (FWD ? 0 : 1)) * (uint32_t)DC.block_bytes);
                    unsigned char* dst = bufs + (size_t)b * DC.buf_bytes;
                    for (int m = 0; m < nn; ++m)
                        if ((km >> m) & 1u) {
                            const double* src = FWD ? A.L + ((int64_t)(l0 + m) * S + k) * bsz
                                                    : (A.U ? A.U + ((int64_t)(u0 + m) * S + k) * bsz
                                                           : A.ubase[k] + (int64_t)(b0 + m) * bsz);
                            bulk_g2s(dst, src, DC.block_bytes, full + b);
                            dst += DC.block_bytes;
                        }
                    if (FWD) {
                        for (int l = 0; l < k; ++l, dst += DC.block_bytes)
                            bulk_g2s(dst, A.G + ((int64_t)i * npairs + pidx(k, l)) * bsz, DC.block_bytes, full + b);
                    } else {
                        if (A.Cup) {
                            for (int l = k + 1; l < S; ++l, dst += DC.block_bytes)
                                bulk_g2s(dst, A.Cup + ((int64_t)i * npairs + pidx(l, k)) * bsz, DC.block_bytes, full + b);
                        } else if (k < S - 1) {
                            bulk_g2s(dst, A.mass + (int64_t)i * bsz, DC.block_bytes, full + b);
                            dst += DC.block_bytes;
                        }
                        bulk_g2s(dst, A.Dinv + ((int64_t)i * S + k) * bsz, DC.block_bytes, full + b);
                    }
                }
            }
            if (end) break;
            if (++b == DC.nbuf) { b = 0; ph ^= 1; }
        }
        return;
    }
    const int a = threadIdx.x - 32;
    const bool act = a < nb;
    auto row_dot = [&](const unsigned char* blk, const double* xv) -> double {
        const double2* B = reinterpret_cast<const double2*>(blk) + a;
        const double2* X = reinterpret_cast<const double2*>(xv);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int p = 0;
#pragma unroll 5
        for (; p + 2 <= P; p += 2) {
            const double2 b0 = B[p * nb], b1 = B[(p + 1) * nb];
            const double2 v0 = X[p], v1 = X[p + 1];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
            s2 = fma(b1.x, v1.x, s2);
            s3 = fma(b1.y, v1.y, s3);
        }
        if (p < P) {
            const double2 b0 = B[p * nb];
            const double2 v0 = X[p];
            s0 = fma(b0.x, v0.x, s0);
            s1 = fma(b0.y, v0.y, s1);
        }
        return (s0 + s1) + (s2 + s3);
    };
    int b = 0;
    uint32_t ph = 0;
    for (;;) {
        mbar_wait(full + b, ph);
        const int i = desc[b].i;
        if (i < 0) break;
        const int k = desc[b].k, nn = desc[b].nn;
        const unsigned km = desc[b].km;
        const int nkept = __popc(km);
        const double* vec = FWD ? A.Z : A.x;            // polled vector: z (forward) / x (backward)
        // gather by polling: the neighbours' stage-k segments, then the element's other stages
        double own = 0.0;
        int nseg = 0;
        if (act) {
            own = __ldcg((FWD ? A.y : A.Z) + (int64_t)k * A.n + (int64_t)i * nb + a);
            for (int m = 0; m < nn; ++m)
                if ((km >> m) & 1u) {
                    xs[nseg * nb + a] = poll_value(vec + (int64_t)k * A.n + (int64_t)desc[b].col[m] * nb + a);
                    ++nseg;
                }
            if (FWD) {
                for (int l = 0; l < k; ++l, ++nseg)
                    xs[nseg * nb + a] = poll_value(vec + (int64_t)l * A.n + (int64_t)i * nb + a);
            } else if (A.Cup) {
                for (int l = k + 1; l < S; ++l, ++nseg)
                    xs[nseg * nb + a] = poll_value(vec + (int64_t)l * A.n + (int64_t)i * nb + a);
            } else if (k < S - 1) {
                double cv = 0.0;      // combined coupling vector sum_{l>k} a_kl x_li (this row)
                for (int l = k + 1; l < S; ++l)
                    cv = fma(A.cup_scale[k * S + l], poll_value(vec + (int64_t)l * A.n + (int64_t)i * nb + a), cv);
                xs[nseg * nb + a] = cv;
                ++nseg;
            }
        }
        consumer_sync(1, ncons);
        const unsigned char* buf = bufs + (size_t)b * DC.buf_bytes;
        const int nblk = nkept + (FWD ? k : (A.Cup ? S - 1 - k : (k < S - 1 ? 1 : 0)));
        if (act) {
            double sn = 0.0, sc = 0.0;   // neighbour part, coupling part
            for (int m = 0; m < nkept; ++m) sn += row_dot(buf + (size_t)m * DC.block_bytes, xs + m * nb);
            for (int m = nkept; m < nblk; ++m) sc += row_dot(buf + (size_t)m * DC.block_bytes, xs + m * nb);
            if (FWD) {
                publish_value(A.Z + (int64_t)k * A.n + (int64_t)i * nb + a, own - (sn + sc));
            } else {
                tv[a] = own - (A.uscale * sn + sc);
            }
        }
        if (!FWD) {
            consumer_sync(1, ncons);
            if (act)
                publish_value(A.x + (int64_t)k * A.n + (int64_t)i * nb + a,
                              row_dot(buf + (size_t)nblk * DC.block_bytes, tv));
        }
        consumer_sync(1, ncons);   // buffer, xs and tv are free
        if (a == 0) mbar_arrive(empty + b);
        if (++b == DC.nbuf) { b = 0; ph ^= 1; }
    }
}

// ---------------------------------------------------------------------------
// Level-scheduled uncoupled sweep with the vector segments riding in the ring
// stages (matvec-style): every stage holds one factor / Jacobian block plus the
// x segments it multiplies (a neighbour's S stage segments, or the task's own S
// segments on its first Dinv item), so there is no separate x-slot double buffer
// and the shared memory of an SM goes to blocks in flight.  FWDI as in
// k_unc_bwd_pipe; stage-shared upper blocks (u_shared) or one factor for several
// right-hand sides (fac_shared).  One thread per block row (or 2 groups, shuffle
// reduction), task-parity double-buffered t vector.
// ---------------------------------------------------------------------------
struct SegCfg {
    int nst;
    int stage_bytes;   // block + S segments, 128-B aligned
    int block_bytes;
};

template <int S, bool FWDI>
__global__ void __launch_bounds__(288) k_unc_sweep_seg(ApplyArgs A, SegCfg SC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    unsigned char* stages = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)SC.nst * SC.stage_bytes);
    uint64_t* empty = full + SC.nst;
    int4* desc = reinterpret_cast<int4*>(empty + SC.nst);
    double* tvb = reinterpret_cast<double*>(desc + SC.nst);      // [2][S][nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SC.nst; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, ncons_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    const int64_t bsz = (int64_t)SC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    const bool ush = A.u_shared || A.fac_shared;
    const int nd = A.fac_shared ? 1 : S;
    if (warp == 0) {
        griddep_wait();
        if (lane != 0) return;
        int st = 0;
        uint32_t ph = 0;
        auto push = [&](int4 d, const double* blk, const double* segbase, int64_t segstride) {
            mbar_wait(empty + st, ph ^ 1);
            desc[st] = d;
            unsigned char* dst = stages + (size_t)st * SC.stage_bytes;
            const int nsg = segbase ? S : 0;
            mbar_expect_tx(full + st, SC.block_bytes + nsg * seg);
            bulk_g2s(dst, blk, SC.block_bytes, full + st);
            for (int k = 0; k < nsg; ++k)
                bulk_g2s(dst + SC.block_bytes + k * seg, segbase + k * segstride, seg, full + st);
            if (++st == SC.nst) { st = 0; ph ^= 1; }
        };
        const int64_t lo = A.ntasks * blockIdx.x / gridDim.x, hi = A.ntasks * (blockIdx.x + 1) / gridDim.x;
        for (int64_t t = lo; t < hi; ++t) {
            const int64_t i = A.order[t];
            const int d = A.diag[i];
            const int b0 = FWDI ? A.indptr[i] : d + 1;
            const int nn = (FWDI ? d : A.indptr[i + 1]) - b0;
            const int store_z = (FWDI && A.hasup[i]) ? 1 : 0;
            int n = 0;
            for (int m = 0; m < nn; ++m) {
                const int qq = b0 + m;
                if (!A.keep[qq]) continue;
                const int64_t col = A.indices[qq];
                const double* vsrc = (FWDI ? A.W : A.x) + col * nb;
                push(make_int4((int)i, 0, PD_USH | (n == 0 ? PD_FIRST : 0), 0),
                     A.U ? A.U + (int64_t)(A.uptr[i] + m) * bsz : A.ubase[0] + (int64_t)qq * bsz, vsrc, A.n);
                ++n;
            }
            const double* own = (FWDI ? A.y : A.x) + i * nb;
            for (int k = 0; k < nd; ++k) {
                const int fl = PD_DINV | (n == 0 ? PD_FIRST : 0) | (k == nd - 1 ? PD_LAST : 0) |
                               (A.fac_shared ? PD_SH : 0);
                push(make_int4((int)i, k, fl, store_z), A.Dinv + (i * nd + k) * bsz, k == 0 ? own : nullptr, A.n);
                ++n;
            }
        }
        push(make_int4(-1, 0, PD_END, 0), A.Dinv, nullptr, 0);   // block copy unused (harmless)
        return;
    }
    const int c = threadIdx.x - 32;
    const int G = A.G_, R = 32 / G;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = G;
    q.a = R * (c >> 5) + (c & (R - 1));
    q.g = (c & 31) / R;
    q.active = q.a < nb;
    auto group_sum = [&](double v) -> double {
        for (int o = R; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    griddep_wait();
    int st = 0;
    uint32_t ph = 0;
    double part[S];
    int par = 0;
    for (;;) {
        mbar_wait(full + st, ph);
        const int4 dsc = desc[st];
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;
        const unsigned char* base = stages + (size_t)st * SC.stage_bytes;
        const double2* B = reinterpret_cast<const double2*>(base);
        const double* segs = reinterpret_cast<const double*>(base + SC.block_bytes);
        double* tv = tvb + (size_t)par * S * nb;
        const bool store_z = FWDI && dsc.w;
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
        }
        if (dsc.z & PD_USH) {
            if (q.active) smem_gemv_all<S>(B, segs, q, part);
        } else {
            const int kk = dsc.y;
            if (kk == 0) {
                // t_k = own_k - uscale * sum_j U_ij x_{j,k}: own segments ride on this item
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    const double sum = group_sum(part[k]);
                    if (q.active && q.g == 0) {
                        const double tval = segs[k * nb + q.a] - A.uscale * sum;
                        tv[k * nb + q.a] = tval;
                        if (store_z) A.x[k * A.n + i * nb + q.a] = tval;   // z_i for the backward sweep
                    }
                    part[k] = 0.0;
                }
                consumer_sync(1, ncons);
            }
            if (q.active) {
                if (dsc.z & PD_SH) {
                    smem_gemv_all<S>(B, tv, q, part);
                } else {
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        if (k == kk) part[k] = smem_gemv(B, tv + k * nb, q, part[k]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == SC.nst) { st = 0; ph ^= 1; }
        if (dsc.z & PD_LAST) {
            par ^= 1;
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const double sum = group_sum(part[k]);
                if (q.active && q.g == 0) (store_z ? A.W : A.x)[k * A.n + i * nb + q.a] = sum;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Stage matvec fused into the implicit-L forward sweep (one GMRES Arnoldi
// product w = P^-1 (B v), krylov.py:88-89 with stage_system.py:52-70 and
// precond.py:222-241).  A task (row i) streams its Jacobian row once: every block
// J_ij multiplies the S stage segments of v (the matvec), and a kept lower block
// also the S segments of w_j = Dinv_j z_j (the sweep) -- one shared-memory block,
// two products, so the lower half of J is read once per iteration instead of
// twice.  Then M_i times v_i (mass mixing), y_i = alpha J v + mix (M v) formed in
// registers (never stored), t = y_i - uscale sum_j J_ij w_j, and the S Dinv items
// as in k_unc_sweep_seg<S, true>.  The backward sweep is unchanged.
// ---------------------------------------------------------------------------
enum { PD_MV = 1024, PD_FU2 = 2048, PD_MM = 4096 };

struct FusedMv {
    const double* J;    // operator blocks (== factor ubase[0], or the halo operator's own blocks)
    const double* M;
    const double* v;    // operator input (s, T, nb)
    double alpha;
    double mix[IRK_MAX_STAGES * IRK_MAX_STAGES];
    // element-partitioned operator (halo mode): its row i holds the factor's row i
    // (the slab's own columns, same order) followed by the ghost columns >= T_local,
    // whose segments come from the ghost buffer (s, n_ghost, nb).  NULL: the
    // operator's pattern is the factor's.
    const int32_t* op_indptr;
    const int32_t* op_indices;
    const double* ghost;
    int64_t T_local, n_ghost;
};

template <int S>
__global__ void __launch_bounds__(288) k_unc_fused_fwd(ApplyArgs A, SegCfg SC, FusedMv F) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    unsigned char* stages = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)SC.nst * SC.stage_bytes);
    uint64_t* empty = full + SC.nst;
    int4* desc = reinterpret_cast<int4*>(empty + SC.nst);
    double* tvb = reinterpret_cast<double*>(desc + SC.nst);      // [2][S][nb]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SC.nst; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, ncons_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    const int64_t bsz = (int64_t)SC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    if (warp == 0) {
        griddep_wait();
        if (lane != 0) return;
        int st = 0;
        uint32_t ph = 0;
        auto push = [&](int4 d, const double* blk, const double* s1, const double* s2, int64_t s1_stride) {
            mbar_wait(empty + st, ph ^ 1);
            desc[st] = d;
            unsigned char* dst = stages + (size_t)st * SC.stage_bytes;
            const int nsg = (s1 ? S : 0) + (s2 ? S : 0);
            mbar_expect_tx(full + st, SC.block_bytes + nsg * seg);
            bulk_g2s(dst, blk, SC.block_bytes, full + st);
            dst += SC.block_bytes;
            if (s1)
                for (int k = 0; k < S; ++k, dst += seg) bulk_g2s(dst, s1 + k * s1_stride, seg, full + st);
            if (s2)
                for (int k = 0; k < S; ++k, dst += seg) bulk_g2s(dst, s2 + k * A.n, seg, full + st);
            if (++st == SC.nst) { st = 0; ph ^= 1; }
        };
        const int64_t lo = A.ntasks * blockIdx.x / gridDim.x, hi = A.ntasks * (blockIdx.x + 1) / gridDim.x;
        for (int64_t t = lo; t < hi; ++t) {
            const int64_t i = A.order[t];
            const int d = A.diag[i];
            const int b0 = A.indptr[i], b1 = A.indptr[i + 1];
            const int store_z = A.hasup[i] ? 1 : 0;
            if (F.op_indptr) {
                // halo mode: the operator row = the factor row's own columns, then ghosts
                const int e0 = F.op_indptr[i], e1 = F.op_indptr[i + 1];
                const int64_t gstride = F.n_ghost * nb;
                for (int qe = e0; qe < e1; ++qe) {
                    const int64_t col = F.op_indices[qe];
                    const bool gh = col >= F.T_local;
                    const int qq = b0 + (qe - e0);
                    const bool low = !gh && qq < d && A.keep[qq];
                    push(make_int4((int)i, 0, (low ? PD_FU2 : PD_MV) | (qe == e0 ? PD_FIRST : 0), 0),
                         F.J + (int64_t)qe * bsz, gh ? F.ghost + (col - F.T_local) * nb : F.v + col * nb,
                         low ? A.W + col * nb : nullptr, gh ? gstride : A.n);
                }
            } else {
                for (int qq = b0; qq < b1; ++qq) {
                    const int64_t col = A.indices[qq];
                    const bool low = qq < d && A.keep[qq];
                    push(make_int4((int)i, 0, (low ? PD_FU2 : PD_MV) | (qq == b0 ? PD_FIRST : 0), 0),
                         F.J + (int64_t)qq * bsz, F.v + col * nb, low ? A.W + col * nb : nullptr, A.n);
                }
            }
            if (F.M) push(make_int4((int)i, 0, PD_MM, 0), F.M + i * bsz, F.v + i * nb, nullptr, A.n);
            for (int k = 0; k < S; ++k)
                push(make_int4((int)i, k, PD_DINV | (k == S - 1 ? PD_LAST : 0), store_z), A.Dinv + (i * S + k) * bsz,
                     nullptr, nullptr, A.n);
        }
        push(make_int4(-1, 0, PD_END, 0), A.Dinv, nullptr, nullptr, A.n);   // block copy unused (harmless)
        return;
    }
    const int c = threadIdx.x - 32;
    const int G = A.G_, R = 32 / G;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = G;
    q.a = R * (c >> 5) + (c & (R - 1));
    q.g = (c & 31) / R;
    q.active = q.a < nb;
    auto group_sum = [&](double v) -> double {
        for (int o = R; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    griddep_wait();
    int st = 0;
    uint32_t ph = 0;
    double pj[S], pm[S], pw[S];   // J v, M v, sum_j J_ij w_j
    int par = 0;
    for (;;) {
        mbar_wait(full + st, ph);
        const int4 dsc = desc[st];
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;
        const unsigned char* base = stages + (size_t)st * SC.stage_bytes;
        const double2* B = reinterpret_cast<const double2*>(base);
        const double* segs = reinterpret_cast<const double*>(base + SC.block_bytes);
        double* tv = tvb + (size_t)par * S * nb;
        const bool store_z = dsc.w != 0;
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) pj[k] = pm[k] = pw[k] = 0.0;
        }
        if (dsc.z & PD_FU2) {
            if (q.active)
                for (int p = q.g; p < q.P; p += q.G) {
                    const double2 b = B[p * nb + q.a];
#pragma unroll
                    for (int k = 0; k < S; ++k) {
                        const double2 v = *reinterpret_cast<const double2*>(segs + k * nb + 2 * p);
                        const double2 w = *reinterpret_cast<const double2*>(segs + (S + k) * nb + 2 * p);
                        pj[k] = fma(b.y, v.y, fma(b.x, v.x, pj[k]));
                        pw[k] = fma(b.y, w.y, fma(b.x, w.x, pw[k]));
                    }
                }
        } else if (dsc.z & PD_MV) {
            if (q.active) smem_gemv_all<S>(B, segs, q, pj);
        } else if (dsc.z & PD_MM) {
            if (q.active) smem_gemv_all<S>(B, segs, q, pm);
        } else {
            const int kk = dsc.y;
            if (kk == 0) {
                // y_k = alpha (J v)_k + sum_l mix_kl (M v)_l ; t_k = y_k - uscale sum_j J_ij w_jk
                double jv[S], mv[S];
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    jv[k] = group_sum(pj[k]);
                    mv[k] = F.M ? group_sum(pm[k]) : 0.0;
                    pw[k] = group_sum(pw[k]);
                }
                if (q.active && q.g == 0) {
#pragma unroll
                    for (int k = 0; k < S; ++k) {
                        double y = F.alpha * jv[k];
                        if (F.M) {
#pragma unroll
                            for (int l = 0; l < S; ++l) y += F.mix[k * S + l] * mv[l];
                        }
                        const double tval = y - A.uscale * pw[k];
                        tv[k * nb + q.a] = tval;
                        if (store_z) A.x[k * A.n + i * nb + q.a] = tval;   // z_i for the backward sweep
                    }
                }
#pragma unroll
                for (int k = 0; k < S; ++k) pj[k] = 0.0;   // reused as the Dinv accumulator
                consumer_sync(1, ncons);
            }
            if (q.active) {
#pragma unroll
                for (int k = 0; k < S; ++k)
                    if (k == kk) pj[k] = smem_gemv(B, tv + k * nb, q, pj[k]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == SC.nst) { st = 0; ph ^= 1; }
        if (dsc.z & PD_LAST) {
            par ^= 1;
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const double sum = group_sum(pj[k]);
                if (q.active && q.g == 0) (store_z ? A.W : A.x)[k * A.n + i * nb + q.a] = sum;
            }
        }
    }
}

// Occupancy of a sweep kernel at (threads, smem), with its dynamic-smem opt-in set once:
// the level launches sit on the critical path after every host wait of irk_gmres, so the
// driver queries are cached (mutex: the C ABI is called from several host threads).
static cudaError_t sweep_occupancy(const void* kernel, int threads, size_t smem, int optin, int* per_sm) {
    struct Entry { const void* k; int t; size_t s; int occ; };
    static std::mutex mu;
    static std::vector<Entry> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& e : cache)
        if (e.k == kernel && e.t == threads && e.s == smem) { *per_sm = e.occ; return cudaSuccess; }
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (err != cudaSuccess) return err;
    int occ = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (err != cudaSuccess) return err;
    cache.push_back({kernel, threads, smem, occ});
    *per_sm = occ;
    return cudaSuccess;
}

template <typename K>
static int run_seg(const irk_factor* f, K kernel, ApplyArgs& A, const irk_sched& S, int s, cudaStream_t st,
                   int extra_doubles = 0, bool pdl = true) {
    const int nb = A.nb;
    SegCfg SC;
    SC.block_bytes = (int)(block_doubles(nb) * 8);
    SC.stage_bytes = (SC.block_bytes + s * nb * 8 + 127) & ~127;
    static const int nst_env = getenv("IRK_SEG_NST") ? atoi(getenv("IRK_SEG_NST")) : 0;   // tuning knob
    SC.nst = nst_env > 1 ? nst_env : 2;
    const int threads = 32 + ((A.G_ * nb + 31) / 32) * 32;
    const size_t smem = (size_t)SC.nst * (SC.stage_bytes + 2 * sizeof(uint64_t) + sizeof(int4)) +
                        sizeof(double) * (2 * (size_t)s * nb + (size_t)extra_doubles) + 64;
    int per_sm = 1;
    IRK_CK(sweep_occupancy((const void*)kernel, threads, smem, (int)f->ctx->smem_optin, &per_sm));
    for (int64_t l = 0; l < S.nlevels; ++l) {
        const int64_t lo = S.h_lvl_ptr[l], hi = S.h_lvl_ptr[l + 1];
        if (hi == lo) continue;
        A.order = S.d_order + lo;
        A.ntasks = hi - lo;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(A.ntasks, (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
        IRK_CK(launch_pdl_if(pdl, kernel, dim3(grid), dim3(threads), smem, st, A, SC));
        IRK_LAUNCHED();
    }
    return IRK_OK;
}

// level launches of k_unc_fused_fwd: ring stages hold a block and up to 2 S segments
template <int S>
static int run_fused_fwd(const irk_factor* f, ApplyArgs& A, const FusedMv& F, cudaStream_t st) {
    const int nb = A.nb;
    const irk_sched& Sd = f->fwd;
    SegCfg SC;
    SC.block_bytes = (int)(block_doubles(nb) * 8);
    SC.stage_bytes = (SC.block_bytes + 2 * S * nb * 8 + 127) & ~127;
    static const int nst_env = getenv("IRK_FUSED_NST") ? atoi(getenv("IRK_FUSED_NST")) : 0;   // tuning knob
    SC.nst = nst_env > 1 ? nst_env : 2;
    const int threads = 32 + ((A.G_ * nb + 31) / 32) * 32;
    const size_t smem = (size_t)SC.nst * (SC.stage_bytes + 2 * sizeof(uint64_t) + sizeof(int4)) +
                        sizeof(double) * 2 * (size_t)S * nb + 64;
    int per_sm = 1;
    IRK_CK(sweep_occupancy((const void*)k_unc_fused_fwd<S>, threads, smem, (int)f->ctx->smem_optin, &per_sm));
    for (int64_t l = 0; l < Sd.nlevels; ++l) {
        const int64_t lo = Sd.h_lvl_ptr[l], hi = Sd.h_lvl_ptr[l + 1];
        if (hi == lo) continue;
        A.order = Sd.d_order + lo;
        A.ntasks = hi - lo;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(A.ntasks, (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
        static const bool pdl = !(getenv("IRK_PDL_FUSED") && atoi(getenv("IRK_PDL_FUSED")) == 0);   // A/B switch
        // the product's first launch is a plain one: with the PDL attribute its CTAs start during
        // the predecessor's drain and, when that predecessor is the previous product's backward
        // sweep (products issued back to back), park on the SMs holding shared memory
        static const bool pdl_first = getenv("IRK_PDL_FIRST") && atoi(getenv("IRK_PDL_FIRST")) != 0;
        const bool first = l == 0 || Sd.h_lvl_ptr[l] == 0;
        IRK_CK(launch_pdl_if(pdl && (!first || pdl_first), k_unc_fused_fwd<S>, dim3(grid), dim3(threads), smem, st, A, SC, F));
        IRK_LAUNCHED();
    }
    return IRK_OK;
}

// ---------------------------------------------------------------------------
// Stage-coupled sweeps on the bulk-copy pipeline (coupled_solve,
// numba_backend.py:128-151).  One task = one element i with ALL s stages: the
// element DAG is the uncoupled one (2 levels on the colour-ordered meshes instead
// of the s + 1 stage-skewed levels of (stage, element) tasks), a stage-shared
// upper block -dt J_ij is read once for s vectors, and the stage coupling of
// the element is solved inside the task:
//   forward  (k ascending):  z_k = (y_k - sum_j L_kij z_kj) - sum_{l<k} G_kl,i z_l
//   backward (k descending): x_k = Dinv_k ((z_k - sum_j U_ij x_kj) - sum_{l>k} C_kl,i x_l)
// with C_kl,i = A^-1_kl M_i (implicit: one M_i gemv per stage on sum_l a_kl x_l)
// or stored couplings.  Within-task stage dependencies go through shared
// memory (tv: z or t, xv: finished x_l, cv: the combined coupling vector).
// ---------------------------------------------------------------------------
enum { PD_G = 256, PD_C = 512 };

// reduce one value per (group, row) over the G groups into dst[a] (op: dst = base - sum)
__device__ __forceinline__ void group_sum_into(double* red, double v, const Geo& q, int ncons, const double* base,
                                               double* dst) {
    if (q.active) red[q.g * q.nb + q.a] = v;
    consumer_sync(1, ncons);
    if (q.active && q.g == 0) {
        double sum = 0.0;
        for (int gg = 0; gg < q.G; ++gg) sum += red[gg * q.nb + q.a];
        dst[q.a] = base[q.a] - sum;
    }
    consumer_sync(1, ncons);
}

template <int S, bool DEPS>
__global__ void __launch_bounds__(288) k_cpl_fwd_pipe(ApplyArgs A, PipeCfg PC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    PipeSmem P = pipe_carve<S>(smem_raw, PC, A.G_, nb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    pipe_init(P, PC.nst, ncons_warps);
    griddep_launch();
    const int64_t bsz = (int64_t)PC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    constexpr int NPAIRS = S * (S - 1) / 2;
    if (warp == 0) {
        Producer pr{&P, &PC};
        griddep_wait();   // PDL: CTA set up during the predecessor's drain
        int cur = (int)(A.ntasks * blockIdx.x / gridDim.x);
        const int hi = (int)(A.ntasks * (blockIdx.x + 1) / gridDim.x);
        int tb, tend;
        while (next_batch<DEPS>(A, tb, tend, cur, hi)) {
            const int tl = tb + lane;
            const bool valid = tl < tend;
            const int64_t il = valid ? A.order[tl] : 0;
            const int q0l = valid ? A.indptr[il] : 0, dl = valid ? A.diag[il] : 0, l0l = valid ? A.lptr[il] : 0;
            const int nnl = dl - q0l;
            for (int bt = 0; bt < 32 && tb + bt < tend; ++bt) {
                const int64_t i = __shfl_sync(0xffffffffu, il, bt);
                const int q0 = __shfl_sync(0xffffffffu, q0l, bt), nn = __shfl_sync(0xffffffffu, nnl, bt);
                const int l0 = __shfl_sync(0xffffffffu, l0l, bt);
                int nitems = NPAIRS;
                for (int m = 0; m < nn; ++m) nitems += A.keep[q0 + m] ? S : 0;
                const int ntot = nitems > 0 ? nitems : 1;
                auto push_items = [&](int from, int to) {
                    if (nitems == 0) {
                        if (from == 0 && to > 0) pr.push(make_int4((int)i, -1, PD_FIRST | PD_LAST, nn), nullptr);
                        return;
                    }
                    int n = 0;
                    for (int m = 0; m < nn; ++m) {
                        if (!A.keep[q0 + m]) continue;
                        for (int k = 0; k < S; ++k, ++n) {
                            if (n < from || n >= to) continue;
                            const int fl = PD_L | (n == 0 ? PD_FIRST : 0) | (n == nitems - 1 ? PD_LAST : 0);
                            pr.push(make_int4((int)i, m * S + k, fl, nn), A.L + ((int64_t)(l0 + m) * S + k) * bsz);
                        }
                    }
                    for (int k = 1; k < S; ++k)
                        for (int l = 0; l < k; ++l, ++n) {
                            if (n < from || n >= to) continue;
                            const int fl = PD_G | (n == 0 ? PD_FIRST : 0) | (n == nitems - 1 ? PD_LAST : 0);
                            pr.push(make_int4((int)i, k * S + l, fl, nn), A.G + (i * NPAIRS + pidx(k, l)) * bsz);
                        }
                };
                const int npre = DEPS ? min(ntot, PC.nst - 1) : 0;
                double* xs = nullptr;
                int xb = 0;
                if (lane == 0) {
                    xs = pr.x_acquire();
                    xb = pr.xb;
                    push_items(0, npre);
                }
                if (DEPS)
                    for (int m = lane; m < nn; m += 32)
                        if (A.keep[q0 + m]) wait_flag(A.flags + A.indices[q0 + m], A.epoch);
                __syncwarp();
                uint32_t bytes = S * seg;
                for (int m = 0; m < nn; ++m) bytes += A.keep[q0 + m] ? S * seg : 0;
                if (lane == 0) {
                    if (DEPS) fence_proxy_async_global();
                    pr.x_commit(bytes);
                }
                xs = reinterpret_cast<double*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(xs), 0));
                xb = __shfl_sync(0xffffffffu, xb, 0);
                __syncwarp();
                for (int e = lane; e < (nn + 1) * S; e += 32) {
                    const int m = e / S, k = e - m * S;
                    if (m == nn) bulk_g2s(xs + e * nb, A.y + k * A.n + i * nb, seg, P.xfull + xb);
                    else if (A.keep[q0 + m]) bulk_g2s(xs + e * nb, A.x + k * A.n + (int64_t)A.indices[q0 + m] * nb, seg, P.xfull + xb);
                }
                if (lane == 0) push_items(npre, ntot);
                if (lane == 0) pr.x_next();
            }
        }
        if (lane == 0) pr.push(make_int4(-1, 0, PD_END, 0), nullptr);
        return;
    }
    const int c = threadIdx.x - 32;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = A.G_; q.g = c / nb; q.a = c - q.g * nb; q.active = q.g < q.G;
    Consumer cs{&P, &PC};
    griddep_wait();
    double part[S];
    double gacc = 0.0;
    const double* xs = nullptr;
    bool t_done = false;
    double* tv = P.tv;   // [S][nb]: t_k, then z_k
    auto finalize_t = [&](int nn) {
        // t_k = y_k - sum_groups part_k for all stages
        if (q.active)
#pragma unroll
            for (int k = 0; k < S; ++k) P.red[(q.g * S + k) * nb + q.a] = part[k];
        consumer_sync(1, ncons);
        if (q.active && q.g == 0)
#pragma unroll
            for (int k = 0; k < S; ++k) {
                double sum = 0.0;
                for (int gg = 0; gg < q.G; ++gg) sum += P.red[(gg * S + k) * nb + q.a];
                tv[k * nb + q.a] = xs[(nn * S + k) * nb + q.a] - sum;
            }
        consumer_sync(1, ncons);
        t_done = true;
    };
    for (;;) {
        const int4 dsc = cs.take();
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;
        const int nn = dsc.w;
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
            gacc = 0.0;
            t_done = false;
            xs = cs.x_wait();
        }
        if (dsc.z & PD_L) {
            if (q.active) {
                const int m = dsc.y / S, kk = dsc.y - m * S;
                const double2* B = cs.block();
#pragma unroll
                for (int k = 0; k < S; ++k)
                    if (k == kk) part[k] = smem_gemv(B, xs + (m * S + k) * nb, q, part[k]);
            }
            cs.release();
        } else if (dsc.z & PD_G) {
            const int k = dsc.y / S, l = dsc.y - k * S;
            if (!t_done) finalize_t(nn);
            if (q.active) gacc = smem_gemv(cs.block(), tv + l * nb, q, gacc);
            cs.release();
            if (l == k - 1) {   // last coupling of stage k: z_k = t_k - sum_l G_kl z_l
                group_sum_into(P.red, gacc, q, ncons, tv + k * nb, tv + k * nb);
                gacc = 0.0;
            }
        } else {
            cs.release();
        }
        if (dsc.z & PD_LAST) {
            if (!t_done) finalize_t(nn);
            if (q.active && q.g == 0)
#pragma unroll
                for (int k = 0; k < S; ++k) A.x[k * A.n + i * nb + q.a] = tv[k * nb + q.a];
            cs.x_release();
            consumer_sync(1, ncons);   // tv / red reuse by the next task
            if (DEPS && c == 0) { __threadfence(); st_release(A.flags + i, A.epoch); }
        }
    }
}

template <int S, bool DEPS>
__global__ void __launch_bounds__(288) k_cpl_bwd_pipe(ApplyArgs A, PipeCfg PC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    PipeSmem P = pipe_carve<S>(smem_raw, PC, A.G_, nb);
    double* xv = P.tv + S * nb;   // [S][nb] finished x_l of the task
    double* cv = xv + S * nb;     // [nb] combined coupling vector
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    pipe_init(P, PC.nst, ncons_warps);
    griddep_launch();
    const int64_t bsz = (int64_t)PC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    constexpr int NPAIRS = S * (S - 1) / 2;
    const bool explicit_c = A.Cup != nullptr;
    if (warp == 0) {
        Producer pr{&P, &PC};
        griddep_wait();   // PDL: CTA set up during the predecessor's drain
        int cur = (int)(A.ntasks * blockIdx.x / gridDim.x);
        const int hi = (int)(A.ntasks * (blockIdx.x + 1) / gridDim.x);
        int tb, tend;
        while (next_batch<DEPS>(A, tb, tend, cur, hi)) {
            const int tl = tb + lane;
            const bool valid = tl < tend;
            const int64_t il = valid ? A.order[tl] : 0;
            const int dl = valid ? A.diag[il] : 0, u0l = valid ? A.uptr[il] : 0;
            const int nnl = valid ? A.indptr[il + 1] - dl - 1 : 0;
            for (int bt = 0; bt < 32 && tb + bt < tend; ++bt) {
                const int64_t i = __shfl_sync(0xffffffffu, il, bt);
                const int nn = __shfl_sync(0xffffffffu, nnl, bt);
                const int b0 = __shfl_sync(0xffffffffu, dl, bt) + 1;
                const int u0 = __shfl_sync(0xffffffffu, u0l, bt);
                const bool ush = A.u_shared != 0;
                int nu = 0;
                for (int m = 0; m < nn; ++m) nu += A.keep[b0 + m] ? (ush ? 1 : S) : 0;
                // stage chain: (couplings, Dinv) for k = S-1 .. 0
                const int nchain = S + (explicit_c ? NPAIRS : S - 1);
                const int ntot = nu + nchain;
                auto push_items = [&](int from, int to) {
                    int n = 0;
                    for (int m = 0; m < nn; ++m) {
                        if (!A.keep[b0 + m]) continue;
                        const int qq = b0 + m;
                        if (ush) {
                            if (n >= from && n < to)
                                pr.push(make_int4((int)i, m * S, PD_USH | (n == 0 ? PD_FIRST : 0), nn), A.ubase[0] + qq * bsz);
                            ++n;
                        } else {
                            for (int k = 0; k < S; ++k, ++n) {
                                if (n < from || n >= to) continue;
                                const double* ub = A.U ? A.U + ((int64_t)(u0 + m) * S + k) * bsz : A.ubase[k] + qq * bsz;
                                pr.push(make_int4((int)i, m * S + k, PD_U | (n == 0 ? PD_FIRST : 0), nn), ub);
                            }
                        }
                    }
                    for (int k = S - 1; k >= 0; --k) {
                        if (k < S - 1) {
                            if (explicit_c) {
                                for (int l = k + 1; l < S; ++l, ++n)
                                    if (n >= from && n < to)
                                        pr.push(make_int4((int)i, k * S + l, PD_C | (n == 0 ? PD_FIRST : 0), nn),
                                                A.Cup + (i * NPAIRS + pidx(l, k)) * bsz);
                            } else {
                                if (n >= from && n < to)
                                    pr.push(make_int4((int)i, k * S + S - 1, PD_C | (n == 0 ? PD_FIRST : 0), nn),
                                            A.mass + i * bsz);
                                ++n;
                            }
                        }
                        if (n >= from && n < to)
                            pr.push(make_int4((int)i, k, PD_DINV | (n == 0 ? PD_FIRST : 0) | (k == 0 ? PD_LAST : 0), nn),
                                    A.Dinv + (i * S + k) * bsz);
                        ++n;
                    }
                };
                const int npre = DEPS ? min(ntot, PC.nst - 1) : 0;
                double* xs = nullptr;
                int xb = 0;
                if (lane == 0) {
                    xs = pr.x_acquire();
                    xb = pr.xb;
                    push_items(0, npre);
                }
                if (DEPS)
                    for (int m = lane; m < nn; m += 32)
                        if (A.keep[b0 + m]) wait_flag(A.flags + A.indices[b0 + m], A.epoch);
                __syncwarp();
                uint32_t bytes = S * seg;
                for (int m = 0; m < nn; ++m) bytes += A.keep[b0 + m] ? S * seg : 0;
                if (lane == 0) {
                    if (DEPS) fence_proxy_async_global();
                    pr.x_commit(bytes);
                }
                xs = reinterpret_cast<double*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(xs), 0));
                xb = __shfl_sync(0xffffffffu, xb, 0);
                __syncwarp();
                for (int e = lane; e < (nn + 1) * S; e += 32) {
                    const int m = e / S, k = e - m * S;
                    if (m == nn) bulk_g2s(xs + e * nb, A.x + k * A.n + i * nb, seg, P.xfull + xb);   // z_i
                    else if (A.keep[b0 + m]) bulk_g2s(xs + e * nb, A.x + k * A.n + (int64_t)A.indices[b0 + m] * nb, seg, P.xfull + xb);
                }
                if (lane == 0) push_items(npre, ntot);
                if (lane == 0) pr.x_next();
            }
        }
        if (lane == 0) pr.push(make_int4(-1, 0, PD_END, 0), nullptr);
        return;
    }
    const int c = threadIdx.x - 32;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = A.G_; q.g = c / nb; q.a = c - q.g * nb; q.active = q.g < q.G;
    Consumer cs{&P, &PC};
    griddep_wait();
    double part[S];
    double acc = 0.0;
    const double* xs = nullptr;
    bool t_done = false;
    double* tv = P.tv;
    for (;;) {
        const int4 dsc = cs.take();
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;
        const int nn = dsc.w;
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
            acc = 0.0;
            t_done = false;
            xs = cs.x_wait();
        }
        const double2* B = cs.block();
        if (dsc.z & (PD_USH | PD_U)) {
            if (q.active) {
                const int m = dsc.y / S, kk = dsc.y - m * S;
                if (dsc.z & PD_USH) {
                    smem_gemv_all<S>(B, xs + m * S * nb, q, part);
                } else {
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        if (k == kk) part[k] = smem_gemv(B, xs + (m * S + k) * nb, q, part[k]);
                }
            }
            cs.release();
            continue;
        }
        if (!t_done) {
            // t_k = z_k - uscale * sum_j U_ij x_kj, all stages
            if (q.active)
#pragma unroll
                for (int k = 0; k < S; ++k) P.red[(q.g * S + k) * nb + q.a] = part[k];
            consumer_sync(1, ncons);
            if (q.active && q.g == 0)
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    double sum = 0.0;
                    for (int gg = 0; gg < q.G; ++gg) sum += P.red[(gg * S + k) * nb + q.a];
                    tv[k * nb + q.a] = xs[(nn * S + k) * nb + q.a] - A.uscale * sum;
                }
            consumer_sync(1, ncons);
            t_done = true;
        }
        if (dsc.z & PD_C) {
            const int k = dsc.y / S, l = dsc.y - k * S;
            if (explicit_c) {
                if (q.active) acc = smem_gemv(B, xv + l * nb, q, acc);
                cs.release();
                if (l == S - 1) {   // all l > k done: t_k -= sum_l C_kl x_l
                    group_sum_into(P.red, acc, q, ncons, tv + k * nb, tv + k * nb);
                    acc = 0.0;
                }
            } else {
                // implicit C_kl = a_kl M_i: cv = sum_{l>k} a_kl x_l, then t_k -= M_i cv
                for (int e = c; e < nb; e += ncons) {
                    double v = 0.0;
                    for (int ll = k + 1; ll < S; ++ll) v = fma(A.cup_scale[k * A.s + ll], xv[ll * nb + e], v);
                    cv[e] = v;
                }
                consumer_sync(1, ncons);
                double pm = 0.0;
                if (q.active) pm = smem_gemv(B, cv, q, 0.0);
                cs.release();
                group_sum_into(P.red, pm, q, ncons, tv + k * nb, tv + k * nb);
            }
            continue;
        }
        // Dinv item k: x_k = Dinv_k t_k
        {
            const int k = dsc.y;
            double pd = 0.0;
            if (q.active) pd = smem_gemv(B, tv + k * nb, q, 0.0);
            cs.release();
            if (q.active) P.red[q.g * nb + q.a] = pd;
            consumer_sync(1, ncons);
            if (q.active && q.g == 0) {
                double sum = 0.0;
                for (int gg = 0; gg < q.G; ++gg) sum += P.red[gg * nb + q.a];
                xv[k * nb + q.a] = sum;
                A.x[k * A.n + i * nb + q.a] = sum;
            }
            consumer_sync(1, ncons);
        }
        if (dsc.z & PD_LAST) {
            cs.x_release();
            if (DEPS && c == 0) { __threadfence(); st_release(A.flags + i, A.epoch); }
        }
    }
}

// ---------------------------------------------------------------------------
// Stage-coupled level sweeps with the vector segments in the ring stages (the
// k_unc_sweep_seg layout applied to coupled_solve, numba_backend.py:128-151).
// Element tasks, all stages; one thread per block row (G = 1) or 2 groups.
//   forward:  items L_{k,ij} (+ segment z_{k,j}), then G_{kl,i} (the first one carries the
//             own y_i segments); z_k = (y_k - sum L z) - sum_{l<k} G_kl z_l (in-task chain)
//   backward: items U_ij (+ the S segments x_{.,j}), then for k = S-1..0 the coupling item
//             (M_i with cv = sum_{l>k} a_kl x_l, or the stored C_kl blocks) and Dinv_k; the
//             first chain item carries the own z_i segments
// ---------------------------------------------------------------------------
template <int S, bool FWD>
__global__ void __launch_bounds__(288) k_cpl_sweep_seg(ApplyArgs A, SegCfg SC) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nb = A.nb;
    unsigned char* stages = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)SC.nst * SC.stage_bytes);
    uint64_t* empty = full + SC.nst;
    int4* desc = reinterpret_cast<int4*>(empty + SC.nst);
    double* tv = reinterpret_cast<double*>(desc + SC.nst);   // [S][nb]: t / z of the task
    double* xv = tv + S * nb;                                 // [S][nb]: finished x_l (backward)
    double* cv = xv + S * nb;                                 // [nb]: combined coupling vector
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1, ncons = ncons_warps * 32;
    constexpr int NPAIRS = S * (S - 1) / 2;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SC.nst; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, ncons_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    const int64_t bsz = (int64_t)SC.block_bytes / 8;
    const uint32_t seg = (uint32_t)nb * 8;
    const bool explicit_c = A.Cup != nullptr;
    if (warp == 0) {
        griddep_wait();   // PDL: the predecessor's output (y, x) is read from here on
        if (lane != 0) return;
        int st = 0;
        uint32_t ph = 0;
        auto push = [&](int4 d, const double* blk, const double* segbase, int64_t segstride, int nsg) {
            mbar_wait(empty + st, ph ^ 1);
            desc[st] = d;
            unsigned char* dst = stages + (size_t)st * SC.stage_bytes;
            mbar_expect_tx(full + st, SC.block_bytes + nsg * seg);
            bulk_g2s(dst, blk, SC.block_bytes, full + st);
            for (int k = 0; k < nsg; ++k)
                bulk_g2s(dst + SC.block_bytes + k * seg, segbase + k * segstride, seg, full + st);
            if (++st == SC.nst) { st = 0; ph ^= 1; }
        };
        const int64_t lo = A.ntasks * blockIdx.x / gridDim.x, hi = A.ntasks * (blockIdx.x + 1) / gridDim.x;
        for (int64_t t = lo; t < hi; ++t) {
            const int64_t i = A.order[t];
            const int d = A.diag[i];
            int n = 0;
            if (FWD) {
                const int q0 = A.indptr[i], l0 = A.lptr[i];
                for (int m = 0; m < d - q0; ++m) {
                    if (!A.keep[q0 + m]) continue;
                    const int64_t col = A.indices[q0 + m];
                    for (int k = 0; k < S; ++k, ++n)
                        push(make_int4((int)i, k, PD_L | (n == 0 ? PD_FIRST : 0), 0),
                             A.L + ((int64_t)(l0 + m) * S + k) * bsz, A.x + k * A.n + col * nb, 0, 1);
                }
                for (int k = 1; k < S; ++k)
                    for (int l = 0; l < k; ++l, ++n) {
                        const bool first_g = (k == 1 && l == 0);
                        const int fl = PD_G | (n == 0 ? PD_FIRST : 0) | (k == S - 1 && l == k - 1 ? PD_LAST : 0);
                        push(make_int4((int)i, k * S + l, fl, 0), A.G + (i * NPAIRS + pidx(k, l)) * bsz,
                             A.y + i * nb, A.n, first_g ? S : 0);
                    }
            } else {
                const int b0 = d + 1, nn = A.indptr[i + 1] - b0;
                for (int m = 0; m < nn; ++m) {
                    if (!A.keep[b0 + m]) continue;
                    const int qq = b0 + m;
                    const int64_t col = A.indices[qq];
                    push(make_int4((int)i, 0, PD_USH | (n == 0 ? PD_FIRST : 0), 0), A.ubase[0] + (int64_t)qq * bsz,
                         A.x + col * nb, A.n, S);
                    ++n;
                }
                bool first_chain = true;
                for (int k = S - 1; k >= 0; --k) {
                    if (k < S - 1) {
                        if (explicit_c) {
                            for (int l = k + 1; l < S; ++l, ++n)
                                push(make_int4((int)i, k * S + l, PD_C | (n == 0 ? PD_FIRST : 0), 0),
                                     A.Cup + (i * NPAIRS + pidx(l, k)) * bsz, nullptr, 0, 0);
                        } else {
                            push(make_int4((int)i, k * S + S - 1, PD_C | (n == 0 ? PD_FIRST : 0), 0),
                                 A.mass + i * bsz, nullptr, 0, 0);
                            ++n;
                        }
                    }
                    push(make_int4((int)i, k, PD_DINV | (n == 0 ? PD_FIRST : 0) | (k == 0 ? PD_LAST : 0), 0),
                         A.Dinv + (i * S + k) * bsz, A.x + i * nb, A.n, first_chain ? S : 0);
                    first_chain = false;
                    ++n;
                }
            }
        }
        push(make_int4(-1, 0, PD_END, 0), A.Dinv, nullptr, 0, 0);
        return;
    }
    const int c = threadIdx.x - 32;
    const int G = A.G_, R = 32 / G;
    Geo q;
    q.nb = nb; q.P = (nb + 1) >> 1; q.G = G;
    q.a = R * (c >> 5) + (c & (R - 1));
    q.g = (c & 31) / R;
    q.active = q.a < nb;
    auto group_sum = [&](double v) -> double {
        for (int o = R; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    griddep_wait();
    int st = 0;
    uint32_t ph = 0;
    double part[S];
    double acc = 0.0;
    bool t_done = false;
    for (;;) {
        mbar_wait(full + st, ph);
        const int4 dsc = desc[st];
        if (dsc.z & PD_END) break;
        const int64_t i = dsc.x;
        const unsigned char* base = stages + (size_t)st * SC.stage_bytes;
        const double2* B = reinterpret_cast<const double2*>(base);
        const double* segs = reinterpret_cast<const double*>(base + SC.block_bytes);
        if (dsc.z & PD_FIRST) {
#pragma unroll
            for (int k = 0; k < S; ++k) part[k] = 0.0;
            acc = 0.0;
            t_done = false;
        }
        auto release = [&]() {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
            if (++st == SC.nst) { st = 0; ph ^= 1; }
        };
        // t_k = own_k - uscale * sum part_k (own segments carried by this item)
        auto finalize_t = [&](double scale) {
#pragma unroll
            for (int k = 0; k < S; ++k) {
                const double sum = group_sum(part[k]);
                if (q.active && q.g == 0) tv[k * nb + q.a] = segs[k * nb + q.a] - scale * sum;
            }
            consumer_sync(1, ncons);
            t_done = true;
        };
        if (FWD) {
            if (dsc.z & PD_L) {
                const int kk = dsc.y;
                if (q.active)
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        if (k == kk) part[k] = smem_gemv(B, segs, q, part[k]);
                release();
            } else {   // G item (k, l): z_k -= G_kl z_l
                const int k = dsc.y / S, l = dsc.y - k * S;
                if (!t_done) finalize_t(1.0);
                if (q.active) acc = smem_gemv(B, tv + l * nb, q, acc);
                release();
                if (l == k - 1) {
                    const double sum = group_sum(acc);
                    if (q.active && q.g == 0) tv[k * nb + q.a] -= sum;
                    consumer_sync(1, ncons);
                    acc = 0.0;
                }
            }
            if (dsc.z & PD_LAST) {
                if (q.active && q.g == 0)
#pragma unroll
                    for (int k = 0; k < S; ++k) A.x[k * A.n + i * nb + q.a] = tv[k * nb + q.a];
                consumer_sync(1, ncons);   // tv reuse by the next task
            }
        } else {
            if (dsc.z & PD_USH) {
                if (q.active) smem_gemv_all<S>(B, segs, q, part);
                release();
                continue;
            }
            if (!t_done) finalize_t(A.uscale);
            if (dsc.z & PD_C) {
                const int k = dsc.y / S, l = dsc.y - k * S;
                if (explicit_c) {
                    if (q.active) acc = smem_gemv(B, xv + l * nb, q, acc);
                    release();
                    if (l == S - 1) {
                        const double sum = group_sum(acc);
                        if (q.active && q.g == 0) tv[k * nb + q.a] -= sum;
                        consumer_sync(1, ncons);
                        acc = 0.0;
                    }
                } else {
                    for (int e = c; e < nb; e += ncons) {
                        double v = 0.0;
                        for (int ll = k + 1; ll < S; ++ll) v = fma(A.cup_scale[k * A.s + ll], xv[ll * nb + e], v);
                        cv[e] = v;
                    }
                    consumer_sync(1, ncons);
                    double pm = 0.0;
                    if (q.active) pm = smem_gemv(B, cv, q, 0.0);
                    release();
                    const double sum = group_sum(pm);
                    if (q.active && q.g == 0) tv[k * nb + q.a] -= sum;
                    consumer_sync(1, ncons);
                }
                continue;
            }
            // Dinv item k: x_k = Dinv_k t_k
            const int k = dsc.y;
            double pd = 0.0;
            if (q.active) pd = smem_gemv(B, tv + k * nb, q, 0.0);
            release();
            const double sum = group_sum(pd);
            if (q.active && q.g == 0) {
                xv[k * nb + q.a] = sum;
                A.x[k * A.n + i * nb + q.a] = sum;
            }
            consumer_sync(1, ncons);
        }
    }
}

// x[k][i] = y[k][i] for the elements of a level with no kept lower neighbour
// (forward sweep: z_i = y_i) -- a plain vectorised row copy.
__global__ void k_copy_rows(const int32_t* __restrict__ rows, int64_t nrows, const double* __restrict__ y,
                            double* __restrict__ x, int s, int nb, int64_t n) {
    const int P = nb >> 1;   // nb even
    const int64_t tot = (int64_t)s * nrows * P;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(e % P);
        const int64_t rr = (e / P) % nrows;
        const int k = (int)(e / ((int64_t)P * nrows));
        const int64_t o = k * n + (int64_t)rows[rr] * nb + 2 * p;
        *reinterpret_cast<double2*>(x + o) = *reinterpret_cast<const double2*>(y + o);
    }
}

// Few levels (mesh-colouring schedule): one launch per level, static task
// slices, no flags.  Many levels (e.g. natural numbering): one persistent
// launch with tickets and dependency flags.
// schedules with at most this many levels run one launch per level (static task slices, no
// synchronisation inside the kernel); deeper ones run the persistent flag-synchronised sweeps.
// IRK_LEVEL_MAX overrides (A/B knob)
static const int64_t LEVEL_LAUNCH_MAX = getenv("IRK_LEVEL_MAX") ? atoll(getenv("IRK_LEVEL_MAX")) : 16;

template <typename K1, typename K2>
static int run_pipe(const irk_factor* f, K1 kernel_deps, K2 kernel_level, ApplyArgs& A, const irk_sched& S,
                    unsigned* flags, int* ticket, int s, cudaStream_t st, int extra_doubles = 0, int ctas_target = 4) {
    A.flags = flags;
    A.ticket = ticket;
    const int nb = A.nb;
    PipeCfg PC;
    PC.block_bytes = (int)(block_doubles(nb) * 8);
    PC.stage_bytes = (PC.block_bytes + 127) & ~127;
    PC.maxdeg = f->maxdeg;
    PC.xslot_doubles = (((PC.maxdeg + 1) * s * nb) + 15) & ~15;
    const int threads = 32 + ((A.G_ * nb + 31) / 32) * 32;
    const size_t fixed = sizeof(double) * (2 * (size_t)PC.xslot_doubles + 2 * (size_t)A.G_ * s * nb + (size_t)s * nb +
                                           (size_t)extra_doubles) + 4 * sizeof(uint64_t);
    // Each task is a short serial chain (x gather -> 3..12 blocks -> reduction),
    // so throughput comes from tasks in flight per SM, not ring depth: size the
    // ring so that >= 4 CTAs fit on an SM (tools/tune_apply.py: 2-3 stages of a
    // 40x40 block at 4-5 CTAs/SM run at 84% of HBM peak, 7 stages at 2 CTAs/SM
    // at 59%).  IRK_APPLY_NST overrides.
    const size_t per_stage = PC.stage_bytes + 2 * sizeof(uint64_t) + sizeof(int4);
    static const int ctas_env = getenv("IRK_APPLY_CTAS") ? atoi(getenv("IRK_APPLY_CTAS")) : 0;   // tuning knob
    const int ctas = ctas_env > 0 ? ctas_env : std::max(ctas_target, 1);
    const size_t per_cta = (size_t)f->ctx->smem_per_sm / ctas - 1024;
    PC.nst = (int)std::max<size_t>(2, std::min<size_t>(24, per_cta > fixed ? (per_cta - fixed) / per_stage : 0));
    if (ctas_target <= 0 && ctas_env <= 0) PC.nst = 2;   // as many 2-stage CTAs as fit (occupancy-limited grid)
    if (const char* ns = getenv("IRK_APPLY_NST")) PC.nst = std::max(2, atoi(ns));
    const size_t smem = (size_t)PC.nst * per_stage + fixed;
    // PDL for the uncoupled sweeps only: measured 7.8 -> 9.1 ms per RADAU23 coupled step with it
    const bool pdl = f->kind == IRK_FACTOR_UNCOUPLED;
    static const bool force_deps = getenv("IRK_APPLY_DEPS") && atoi(getenv("IRK_APPLY_DEPS")) != 0;
    const bool level_mode = S.nlevels <= LEVEL_LAUNCH_MAX && !force_deps;
    int per_sm = 1;
    if (level_mode) {
        IRK_CK(cudaFuncSetAttribute(kernel_level, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f->ctx->smem_optin));
        IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_level, threads, smem));
        for (int64_t l = 0; l < S.nlevels; ++l) {
            const int64_t lo = S.h_lvl_ptr[l], hi = S.h_lvl_ptr[l + 1];
            if (hi == lo) continue;
            A.order = S.d_order + lo;
            A.ntasks = hi - lo;
            if (l < (int64_t)S.h_trivial.size() && S.h_trivial[l]) {
                const int64_t tot = (int64_t)s * A.ntasks * (nb / 2);
                const int g = (int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)f->ctx->num_sms * 16));
                k_copy_rows<<<g, 256, 0, st>>>(A.order, A.ntasks, A.y, A.x, s, nb, A.n);
                IRK_LAUNCHED();
                continue;
            }
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((A.ntasks + 1) / 2,
                                                                        (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
            IRK_CK(launch_pdl_if(pdl, kernel_level, dim3(grid), dim3(threads), smem, st, A, PC));
            IRK_LAUNCHED();
        }
        return IRK_OK;
    }
    A.order = S.d_order;
    A.ntasks = S.h_lvl_ptr.empty() ? 0 : S.h_lvl_ptr.back();
    IRK_CK(cudaFuncSetAttribute(kernel_deps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f->ctx->smem_optin));
    IRK_CK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_deps, threads, smem));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(A.ntasks, (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
    IRK_CK(launch_pdl_if(pdl, kernel_deps, dim3(grid), dim3(threads), smem, st, A, PC));
    IRK_LAUNCHED();
    return IRK_OK;
}

// one persistent launch per sweep direction
template <typename K>
static int run_sweep(const irk_factor* f, K kernel, ApplyArgs& A, const irk_sched& S, unsigned* flags,
                     int* ticket, int threads, size_t smem, cudaStream_t st) {
    A.order = S.d_order;
    A.ntasks = S.h_lvl_ptr.empty() ? 0 : S.h_lvl_ptr.back();
    A.flags = flags;
    A.ticket = ticket;
    IRK_CK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    int per_sm = 0;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(A.ntasks, (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
    kernel<<<grid, threads, smem, st>>>(A);
    IRK_LAUNCHED();
    return IRK_OK;
}

// groups of the shuffle-reduction sweep layout (k_unc_bwd_pipe): a power of two
static int ws_groups(int nb, int s = 1) {
    static const int force = getenv("IRK_APPLY_WSG") ? atoi(getenv("IRK_APPLY_WSG")) : 0;   // tuning knob
    if (force == 1 || force == 2 || force == 4) return force;
    // small blocks carrying >= 3 vectors: the single consumer warp is the bottleneck (config 3,
    // nb = 24: 0.204 -> 0.173 ms at s = 4, 0.162 -> 0.150 ms at s = 3 with two groups)
    if (nb <= 32 && s >= 3) return 2;
    // one thread per block row: small CTAs, many tasks in flight per SM (measured best for
    // nb <= 64); two groups for the 100-row blocks of config 3
    return (nb > 64 && nb <= 128) ? 2 : 1;
}
// CTAs per SM the shared-memory ring is sized for (2-3 stages each): the sweeps are bound by
// tasks in flight, not by consumer width (tools/tune_apply.py: 0.57 ms at 6 vs 0.60 ms at 4)
static int ws_ctas(int G) { return G == 1 ? 0 : 4; }   // 0: 2-stage rings, occupancy-limited

// k_unc_deep applies: implicit-L factor on the stage-shared J, s factors for s vectors, even nb,
// <= MAXD neighbours per row, two task buffers within the shared memory of an SM
template <int S>
static size_t deep_smem(const irk_factor* f, const ApplyArgs& A) {
    const size_t blk = (size_t)block_doubles(A.nb) * 8;
    return 2 * (size_t)(f->maxdeg + S) * blk + 128 + sizeof(double) * ((size_t)f->maxdeg + 1) * S * A.nb;
}

template <int S>
static bool deep_ok(const irk_factor* f, const ApplyArgs& A) {
    static const bool off = getenv("IRK_DEEP") && atoi(getenv("IRK_DEEP")) == 0;   // A/B switch
    // narrow levels only (one CTA per SM, one task each): with wide levels the sweep is a throughput
    // problem again and the generic ring kernel wins (config 2 at N = 16, natural numbering: 67
    // levels of ~367 tasks, 1.51 ms vs 2.06 ms with a single-buffered k_unc_deep)
    const int64_t ntasks = f->fwd.h_lvl_ptr.empty() ? 0 : f->fwd.h_lvl_ptr.back();
    const bool narrow = f->fwd.nlevels > 0 && ntasks * 4 <= (int64_t)f->fwd.nlevels * f->ctx->num_sms * 5;
    return !off && narrow && A.u_shared && !A.fac_shared && A.U == nullptr && A.nb % 2 == 0 && f->maxdeg <= MAXD &&
           S * A.nb + 32 <= 512 && deep_smem<S>(f, A) <= (size_t)f->ctx->smem_optin;
}

template <int S, bool FWDI, bool SENT = false>
static int run_deep(const irk_factor* f, ApplyArgs& A, const irk_sched& Sd, unsigned* flags, int* ticket,
                    cudaStream_t st) {
    A.flags = flags;
    A.ticket = ticket;
    A.order = Sd.d_order;
    A.ntasks = Sd.h_lvl_ptr.empty() ? 0 : Sd.h_lvl_ptr.back();
    if (A.ntasks == 0) return IRK_OK;
    DeepCfg DC;
    DC.block_bytes = (int)(block_doubles(A.nb) * 8);
    DC.maxdeg = f->maxdeg;
    DC.buf_bytes = (f->maxdeg + S) * DC.block_bytes;
    DC.nbuf = 2;
    const int threads = 32 + ((S * A.nb + 31) / 32) * 32;
    const size_t smem = deep_smem<S>(f, A);
    int per_sm = 1;
    auto kernel = SENT ? k_unc_deep_sent<S, FWDI> : k_unc_deep<S, FWDI>;
    IRK_CK(sweep_occupancy((const void*)kernel, threads, smem, (int)f->ctx->smem_optin, &per_sm));
    IRK_CK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(A.ntasks, (int64_t)f->ctx->num_sms * std::max(per_sm, 1)));
    IRK_CK(launch_pdl_if(!SENT, kernel, dim3(grid), dim3(threads), smem, st, A, DC));
    IRK_LAUNCHED();
    return IRK_OK;
}

template <int S, bool EVEN>
static int unc_apply(const irk_factor* f, ApplyArgs& A0, cudaStream_t st) {
    ApplyArgs A = A0;
    // deep DAGs (persistent, flag-synchronised sweeps) prefer fewer, wider CTAs
    const bool deep = f->fwd.nlevels > LEVEL_LAUNCH_MAX || f->bwd.nlevels > LEVEL_LAUNCH_MAX;
    A.G_ = deep ? (A.nb <= 64 ? 4 : (A.nb <= 128 ? 2 : 1)) : ws_groups(A.nb, S);
    if (EVEN && S <= 4 && A.G_ * A.nb <= 256) {
        const int64_t nf = (int64_t)f->pat->T;
        static const bool seg_off = getenv("IRK_APPLY_SEG") && atoi(getenv("IRK_APPLY_SEG")) == 0;
        if (f->l_implicit && !deep && !seg_off && (A.u_shared || A.fac_shared) && A.G_ <= 2) {
            // level launches with the vector segments carried in the ring stages
            IRK_TRY(run_seg(f, k_unc_sweep_seg<S, true>, A, f->fwd, S, st));
            IRK_TRY(run_seg(f, k_unc_sweep_seg<S, false>, A, f->bwd, S, st));
            return IRK_OK;
        }
        if (f->l_implicit) {
            // implicit L: forward sweep streams the stage-shared J_ij with w_j = Dinv_j z_j and
            // finishes rows without upper blocks; the backward sweep covers the remaining rows
            A.flags2 = f->d_flags + nf;
            static const bool sent_off = getenv("IRK_DEEP_SENT") && atoi(getenv("IRK_DEEP_SENT")) == 0;   // A/B switch
            if (deep && !sent_off && deep_ok<S>(f, A) && A.x != A.y) {
                if (!f->d_Z) IRK_CK(cudaMalloc(&f->d_Z, sizeof(double) * (size_t)S * A.n));
                A.Z = f->d_Z;
                const int64_t tot = (int64_t)S * A.n;
                k_fill_sentinel<<<(int)std::min<int64_t>((tot + 255) / 256, (int64_t)f->ctx->num_sms * 8), 256, 0, st>>>(A.x, A.W, tot);
                IRK_LAUNCHED();
                IRK_TRY((run_deep<S, true, true>(f, A, f->fwd, f->d_flags, f->d_ticket, st)));
                IRK_TRY((run_deep<S, false, true>(f, A, f->bwd, f->d_flags + nf, f->d_ticket + 1, st)));
                return IRK_OK;
            }
            if (deep && deep_ok<S>(f, A)) {
                IRK_TRY((run_deep<S, true>(f, A, f->fwd, f->d_flags, f->d_ticket, st)));
                IRK_TRY((run_deep<S, false>(f, A, f->bwd, f->d_flags + nf, f->d_ticket + 1, st)));
                return IRK_OK;
            }
            IRK_TRY(run_pipe(f, k_unc_bwd_pipe<S, true, true>, k_unc_bwd_pipe<S, false, true>, A, f->fwd,
                             f->d_flags, f->d_ticket, S, st, 0, ws_ctas(A.G_)));
            IRK_TRY(run_pipe(f, k_unc_bwd_pipe<S, true, false>, k_unc_bwd_pipe<S, false, false>, A, f->bwd,
                             f->d_flags + nf, f->d_ticket + 1, S, st, 0, ws_ctas(A.G_)));
            return IRK_OK;
        }
        if (A0.G_ * A0.nb <= 256)
            IRK_TRY(run_pipe(f, k_unc_fwd_pipe<S, true>, k_unc_fwd_pipe<S, false>, A0, f->fwd, f->d_flags, f->d_ticket, S, st));
        else
            IRK_TRY(run_pipe(f, k_unc_fwd_pipe<S, true>, k_unc_fwd_pipe<S, false>, A, f->fwd, f->d_flags, f->d_ticket, S, st));
        IRK_TRY(run_pipe(f, k_unc_bwd_pipe<S, true, false>, k_unc_bwd_pipe<S, false, false>, A, f->bwd, f->d_flags + nf,
                         f->d_ticket + 1, S, st, 0, ws_ctas(A.G_)));
        return IRK_OK;
    }
    A = A0;
    const int threads = ((A.G_ * A.nb + 31) / 32) * 32;
    const size_t smem_f = sizeof(double) * A.G_ * S * A.nb;
    const size_t smem_b = smem_f + sizeof(double) * S * A.nb;
    const int64_t nf = (int64_t)f->pat->T;
    IRK_TRY(run_sweep(f, k_unc_fwd<S, EVEN>, A, f->fwd, f->d_flags, f->d_ticket, threads, smem_f, st));
    IRK_TRY(run_sweep(f, k_unc_bwd<S, EVEN>, A, f->bwd, f->d_flags + nf, f->d_ticket + 1, threads, smem_b, st));
    return IRK_OK;
}

template <int S>
static int cpl_apply_pipe(const irk_factor* f, ApplyArgs& A0, cudaStream_t st) {
    const int64_t nf = (int64_t)f->pat->T;
    static const bool seg_off = getenv("IRK_APPLY_SEG") && atoi(getenv("IRK_APPLY_SEG")) == 0;
    const bool level = f->fwd.nlevels <= LEVEL_LAUNCH_MAX && f->bwd.nlevels <= LEVEL_LAUNCH_MAX;
    if (level && !seg_off && f->u_shared && A0.nb <= 128) {
        ApplyArgs A = A0;
        A.G_ = ws_groups(A.nb);
        static const bool cpl_pdl = getenv("IRK_CPL_PDL") && atoi(getenv("IRK_CPL_PDL")) != 0;   // A/B knob
        IRK_TRY(run_seg(f, k_cpl_sweep_seg<S, true>, A, f->fwd, S, st, 0, cpl_pdl));
        IRK_TRY(run_seg(f, k_cpl_sweep_seg<S, false>, A, f->bwd, S, st, A.nb, cpl_pdl));
        return IRK_OK;
    }
    // narrower CTAs, more tasks in flight (config 4: 7.85 -> 7.70 ms per RADAU23 step)
    ApplyArgs A = A0;
    if (!getenv("IRK_APPLY_G") && 2 * A.nb <= 256) A.G_ = std::min(2, (A.nb + 1) / 2);
    IRK_TRY(run_pipe(f, k_cpl_fwd_pipe<S, true>, k_cpl_fwd_pipe<S, false>, A, f->fwd, f->d_flags, f->d_ticket, S, st,
                     0, 6));
    IRK_TRY(run_pipe(f, k_cpl_bwd_pipe<S, true>, k_cpl_bwd_pipe<S, false>, A, f->bwd, f->d_flags + nf, f->d_ticket + 1,
                     S, st, (S + 1) * A.nb, 6));
    return IRK_OK;
}

template <bool EVEN>
static int cpl_apply(const irk_factor* f, ApplyArgs& A, cudaStream_t st) {
    if (f->cpl_pipe) {
        switch (f->s) {
            case 2: return cpl_apply_pipe<2>(f, A, st);
            case 3: return cpl_apply_pipe<3>(f, A, st);
            case 4: return cpl_apply_pipe<4>(f, A, st);
            default: break;
        }
    }
    {
        // deep schedules (natural numbering): self-validating-value sweeps over the (stage, element) tasks
        static const bool sent_off = getenv("IRK_DEEP_SENT") && atoi(getenv("IRK_DEEP_SENT")) == 0;   // A/B switch
        const size_t blk = (size_t)block_doubles(A.nb) * 8;
        DeepCfg DC;
        DC.block_bytes = (int)blk;
        DC.maxdeg = f->maxdeg;
        DC.buf_bytes = (int)((f->maxdeg + f->s) * blk);
        DC.nbuf = 1;
        const size_t smem = (size_t)DC.nbuf * DC.buf_bytes + 128 + sizeof(double) * (size_t)(f->maxdeg + f->s + 1) * A.nb;
        const int64_t ntasks = f->fwd.h_lvl_ptr.empty() ? 0 : f->fwd.h_lvl_ptr.back();
        const int thr = 32 + ((A.nb + 31) / 32) * 32;
        if (EVEN && !sent_off && !f->cpl_pipe && f->fwd.nlevels > LEVEL_LAUNCH_MAX && f->maxdeg <= MAXD && thr <= 160 &&
            smem <= (size_t)f->ctx->smem_optin && A.x != A.y && ntasks > 0) {
            int occ_f = 1, occ_b = 1;
            IRK_CK(sweep_occupancy((const void*)k_cpl_deep_sent<true>, thr, smem, (int)f->ctx->smem_optin, &occ_f));
            IRK_CK(sweep_occupancy((const void*)k_cpl_deep_sent<false>, thr, smem, (int)f->ctx->smem_optin, &occ_b));
            const int64_t cap = (int64_t)f->ctx->num_sms * std::max(std::min(occ_f, occ_b), 1);
            // narrow levels only: at most two tasks of a level per resident CTA
            if (ntasks <= 2 * (int64_t)f->fwd.nlevels * cap) {
                if (!f->d_Z) IRK_CK(cudaMalloc(&f->d_Z, sizeof(double) * (size_t)A.s * A.n));
                A.Z = f->d_Z;
                const int64_t tot = (int64_t)A.s * A.n;
                k_fill_sentinel<<<(int)std::min<int64_t>((tot + 255) / 256, (int64_t)f->ctx->num_sms * 8), 256, 0, st>>>(A.x, A.Z, tot);
                IRK_LAUNCHED();
                IRK_CK(cudaMemsetAsync(f->d_ticket, 0, 2 * sizeof(int), st));
                const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntasks, cap));
                A.order = f->fwd.d_order;
                A.ntasks = ntasks;
                A.ticket = f->d_ticket;
                k_cpl_deep_sent<true><<<grid, thr, smem, st>>>(A, DC);
                IRK_LAUNCHED();
                A.order = f->bwd.d_order;
                A.ntasks = f->bwd.h_lvl_ptr.empty() ? 0 : f->bwd.h_lvl_ptr.back();
                A.ticket = f->d_ticket + 1;
                k_cpl_deep_sent<false><<<grid, thr, smem, st>>>(A, DC);
                IRK_LAUNCHED();
                return IRK_OK;
            }
        }
    }
    const int threads = ((A.G_ * A.nb + 31) / 32) * 32;
    const size_t smem_f = sizeof(double) * A.G_ * A.nb;
    const size_t smem_b = sizeof(double) * (A.G_ * 2 * A.nb + A.nb);
    const int64_t nf = (int64_t)f->s * f->pat->T;
    IRK_TRY(run_sweep(f, k_cpl_fwd<EVEN>, A, f->fwd, f->d_flags, f->d_ticket, threads, smem_f, st));
    IRK_TRY(run_sweep(f, k_cpl_bwd<EVEN>, A, f->bwd, f->d_flags + nf, f->d_ticket + 1, threads, smem_b, st));
    return IRK_OK;
}

static void fill_args(const irk_factor* f, ApplyArgs& A) {
    const irk_pattern* p = f->pat;
    A.indptr = p->d_indptr;
    A.indices = p->d_indices;
    A.diag = p->d_diag;
    A.lptr = p->d_lptr;
    A.uptr = p->d_uptr;
    A.keep = f->d_keep;
    A.L = f->d_L;
    A.W = f->d_W;
    A.hasup = f->d_hasup;
    A.flags2 = nullptr;
    A.Dinv = f->d_Dinv;
    A.U = f->u_stored ? f->d_U : nullptr;
    for (int k = 0; k < f->s; ++k) A.ubase[k] = f->ubase[k];
    A.uscale = f->uscale;
    A.u_shared = f->u_shared ? 1 : 0;
    A.G = f->d_G;
    A.Cup = f->d_Cup;
    A.mass = f->mass;
    for (int e = 0; e < f->s * f->s; ++e) A.cup_scale[e] = f->cup_scale[e];
    A.T = p->T;
    A.n = p->T * f->nb;
    A.s = f->s;
    A.nb = f->nb;
    // consumer groups: the multi-stage uncoupled sweeps read each block once for all stages and
    // run best with <= 4 consumer warps; the single-stage and coupled sweeps (more per-task
    // reductions) keep up to 8 (tools/tune_apply.py, tools/sweep.py config4)
    A.G_ = choose_groups(f->nb, (f->kind == IRK_FACTOR_UNCOUPLED && f->s > 1) ? 128 : 256);
    if (const char* g = getenv("IRK_APPLY_G")) A.G_ = std::max(1, std::min(atoi(g), (f->nb + 1) / 2));
}

int factor_materialize_L(const irk_factor* f, double** out, cudaStream_t st);   // factor.cu
int factor_form_level0_d(const irk_factor* f, cudaStream_t st);                // factor.cu

int factor_apply(const irk_factor* f, const double* y, double* x, cudaStream_t st) {
    ApplyArgs A{};
    fill_args(f, A);
    A.y = y;
    A.x = x;
    A.epoch = ++f->epoch;
    const bool even = (f->nb % 2) == 0;
    if (f->kind == IRK_FACTOR_COUPLED) return even ? cpl_apply<true>(f, A, st) : cpl_apply<false>(f, A, st);
    switch (f->s) {
#define CASE(S_) case S_: return even ? unc_apply<S_, true>(f, A, st) : unc_apply<S_, false>(f, A, st);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
        default: set_error("bad stage count"); return IRK_EINVAL;
    }
}

// x = P^-1 (B v): the stage operator fused into the forward sweep (k_unc_fused_fwd).
// Returns 1 (nothing launched) when the pair does not qualify: uncoupled implicit-L
// factor on the operator's own pattern and Jacobian blocks, colour (level-launch)
// schedule, shared J, no halo.  IRK_FUSED=0 disables it (A/B switch).
template <int S>
static int fused_apply_t(const irk_stage_op* op, const irk_factor* f, const double* v, double* x, cudaStream_t st) {
    ApplyArgs A{};
    fill_args(f, A);
    A.G_ = ws_groups(A.nb, S);
    if (A.G_ > 2 || A.G_ * A.nb > 256) return 1;
    A.y = nullptr;
    A.x = x;
    A.epoch = ++f->epoch;
    FusedMv F{};
    F.J = f->ubase[0];
    if (op->ghost) {
        F.J = op->J[0]->d + op->jfirst[0] * block_doubles(op->nb);
        F.op_indptr = op->pat->d_indptr;
        F.op_indices = op->pat->d_indices;
        F.ghost = op->ghost;
        F.T_local = op->T_local;
        F.n_ghost = op->n_ghost;
    }
    F.M = op->M ? op->M->d : nullptr;
    F.v = v;
    F.alpha = op->alpha;
    for (int e = 0; e < S * S; ++e) F.mix[e] = op->C[e];
    IRK_TRY(run_fused_fwd<S>(f, A, F, st));
    IRK_TRY(run_seg(f, k_unc_sweep_seg<S, false>, A, f->bwd, S, st));
    return IRK_OK;
}

// Compare the operator's own-column blocks of every row with the factor's source
// blocks at the corresponding factor position (bitwise); *bad = 1 on any mismatch.
__global__ void k_halo_blocks_equal(const double* __restrict__ opJ, const int32_t* __restrict__ op_indptr,
                                    const double* __restrict__ fJ, const int32_t* __restrict__ f_indptr,
                                    int64_t T, int64_t bsz, int* bad) {
    for (int64_t i = blockIdx.x; i < T; i += gridDim.x) {
        const int64_t e0 = op_indptr[i], q0 = f_indptr[i], cnt = f_indptr[i + 1] - q0;
        const double* a = opJ + e0 * bsz;
        const double* b = fJ + q0 * bsz;
        for (int64_t t = threadIdx.x; t < cnt * bsz; t += blockDim.x)
            if (__double_as_longlong(a[t]) != __double_as_longlong(b[t])) *bad = 1;
    }
}

static int halo_pair_ok(const irk_stage_op* op, const irk_factor* f, cudaStream_t st) {
    if (f->halo_op == op && f->halo_epoch == f->numeric_epoch) return f->halo_ok ? 0 : 1;
    f->halo_op = op;
    f->halo_epoch = f->numeric_epoch;
    f->halo_ok = false;
    const irk_pattern* po = op->pat;
    const irk_pattern* pf = f->pat;
    const int64_t T = op->T_local;
    if (po->T < T || pf->T != T || !f->ubase[0]) return 1;
    for (int64_t i = 0; i < T; ++i) {
        const int64_t e0 = po->h_indptr[i], e1 = po->h_indptr[i + 1];
        const int64_t q0 = pf->h_indptr[i], q1 = pf->h_indptr[i + 1];
        if (q1 - q0 > e1 - e0) return 1;
        for (int64_t k = 0; k < q1 - q0; ++k)
            if (po->h_indices[e0 + k] != pf->h_indices[q0 + k]) return 1;
        for (int64_t e = e0 + (q1 - q0); e < e1; ++e)
            if (po->h_indices[e] < T) return 1;
    }
    int* d_bad = nullptr;
    IRK_CK(cudaMallocAsync(&d_bad, sizeof(int), st));
    IRK_CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    const int64_t bsz = block_doubles(op->nb);
    k_halo_blocks_equal<<<(int)std::min<int64_t>(T, (int64_t)f->ctx->num_sms * 8), 256, 0, st>>>(
        op->J[0]->d + op->jfirst[0] * bsz, po->d_indptr, f->ubase[0], pf->d_indptr, T, bsz, d_bad);
    IRK_LAUNCHED();
    int bad = 1;
    IRK_CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    IRK_CK(cudaStreamSynchronize(st));
    IRK_CK(cudaFreeAsync(d_bad, st));
    f->halo_ok = bad == 0;
    return f->halo_ok ? 0 : 1;
}

int factor_apply_fused(const irk_stage_op* op, const irk_factor* f, const double* v, double* x, cudaStream_t st) {
    static const bool off = getenv("IRK_FUSED") && atoi(getenv("IRK_FUSED")) == 0;
    static const bool seg_off = getenv("IRK_APPLY_SEG") && atoi(getenv("IRK_APPLY_SEG")) == 0;
    if (off || seg_off || !op || !f) return 1;
    if (f->kind != IRK_FACTOR_UNCOUPLED || !f->l_implicit || f->u_stored || !f->u_shared) return 1;
    if (f->fwd.nlevels > LEVEL_LAUNCH_MAX || f->bwd.nlevels > LEVEL_LAUNCH_MAX) return 1;
    if (op->s != f->s || op->nb != f->nb || !op->shared_j || op->T_local != f->pat->T || f->nb % 2) return 1;
    if (op->ghost) {
        // element-partitioned operator (extended pattern, halo buffer) with the slab's
        // partitioned factor: checked once per (operator, factor) pair on the host
        // (patterns) and on the device (the operator's own-column blocks equal the
        // factor's upper source blocks), cached until the factor is re-factorised
        const int ok = halo_pair_ok(op, f, st);
        if (ok != 0) return ok < 0 ? ok : 1;
    } else {
        if (op->pat != f->pat) return 1;
        if (op->J[0]->d + op->jfirst[0] * block_doubles(op->nb) != f->ubase[0]) return 1;
    }
    switch (f->s) {
        case 1: return fused_apply_t<1>(op, f, v, x, st);
        case 2: return fused_apply_t<2>(op, f, v, x, st);
        case 3: return fused_apply_t<3>(op, f, v, x, st);
        case 4: return fused_apply_t<4>(op, f, v, x, st);
        default: return 1;
    }
}

// One factor (s = 1) applied to nrhs stage-major right-hand sides in one sweep:
// every factor block (Dinv_i, the implicit/stored upper blocks, stored L) is read
// once for all right-hand sides (BASELINE config 3: plain ILU(0) of J, s RHS).
int factor_apply_rhs(const irk_factor* f, int nrhs, const double* y, double* x, cudaStream_t st) {
    if (nrhs == 1) return factor_apply(f, y, x, st);
    if (f->kind != IRK_FACTOR_UNCOUPLED || f->s != 1) {
        set_error("multi-RHS apply needs a single uncoupled factor (s = 1)");
        return IRK_EINVAL;
    }
    ApplyArgs A{};
    fill_args(f, A);
    if (f->nb % 2 || nrhs > 4 || A.G_ * f->nb > 256) {
        set_error("multi-RHS apply needs even nb, nrhs <= 4 and nb <= 256");
        return IRK_EINVAL;
    }
    if (f->l_implicit && f->wrhs < nrhs) {
        cudaFree(f->d_Wrhs);
        f->d_Wrhs = nullptr;
        f->wrhs = 0;
        IRK_CK(cudaMalloc(&f->d_Wrhs, sizeof(double) * nrhs * f->pat->T * f->nb));
        f->wrhs = nrhs;
    }
    A.y = y;
    A.x = x;
    A.s = nrhs;
    A.fac_shared = 1;
    A.G_ = choose_groups(f->nb, 128);   // several right-hand sides per block: <= 4 consumer warps
    if (f->l_implicit) A.W = f->d_Wrhs;
    A.epoch = ++f->epoch;
    switch (nrhs) {
        case 2: return unc_apply<2, true>(f, A, st);
        case 3: return unc_apply<3, true>(f, A, st);
        case 4: return unc_apply<4, true>(f, A, st);
        default: set_error("nrhs out of range"); return IRK_EINVAL;
    }
}

// ---------------------------------------------------------------------------
// block gather/scatter used by export/import: dst[didx[e]] = scale*src[sidx[e]]
// (sidx < 0: zero block)
// ---------------------------------------------------------------------------
__global__ void k_copy_blocks(const double* __restrict__ src, const int64_t* __restrict__ sidx,
                              double* __restrict__ dst, const int64_t* __restrict__ didx, int64_t n,
                              int64_t bsz, double scale) {
    for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
        const int64_t si = sidx[e];
        double* d = dst + didx[e] * bsz;
        if (si < 0) {
            for (int64_t t = threadIdx.x; t < bsz; t += blockDim.x) d[t] = 0.0;
        } else {
            const double* s = src + si * bsz;
            for (int64_t t = threadIdx.x; t < bsz; t += blockDim.x) d[t] = scale * s[t];
        }
    }
}

int copy_blocks(const double* src, const std::vector<int64_t>& sidx, double* dst,
                const std::vector<int64_t>& didx, int64_t bsz, double scale, cudaStream_t st) {
    const int64_t n = (int64_t)sidx.size();
    if (n == 0) return IRK_OK;
    int64_t* d = nullptr;
    IRK_CK(cudaMallocAsync(&d, sizeof(int64_t) * 2 * n, st));
    IRK_CK(cudaMemcpyAsync(d, sidx.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    IRK_CK(cudaMemcpyAsync(d + n, didx.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    k_copy_blocks<<<(int)std::min<int64_t>(n, 148 * 16), 128, 0, st>>>(src, d, dst, d + n, n, bsz, scale);
    IRK_LAUNCHED();
    IRK_CK(cudaStreamSynchronize(st));  // host index vectors go out of scope
    IRK_CK(cudaFreeAsync(d, st));
    return IRK_OK;
}

int download_raw(const double* dev_layout, int nb, int64_t count, double* host, cudaStream_t st) {
    if (count == 0) return IRK_OK;
    double* tmp = nullptr;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * nb * nb * count, st));
    int rc = permute_out(dev_layout, tmp, nb, count, st);
    if (rc == IRK_OK) {
        cudaError_t e = cudaMemcpyAsync(host, tmp, sizeof(double) * nb * nb * count, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = fail_cuda(e, "D2H", __FILE__, __LINE__);
    }
    cudaFreeAsync(tmp, st);
    if (rc == IRK_OK) IRK_CK(cudaStreamSynchronize(st));
    return rc;
}

int upload_raw(const double* host, int nb, int64_t count, double* dev_layout, cudaStream_t st) {
    if (count == 0) return IRK_OK;
    double* tmp = nullptr;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * nb * nb * count, st));
    cudaError_t e = cudaMemcpyAsync(tmp, host, sizeof(double) * nb * nb * count, cudaMemcpyHostToDevice, st);
    int rc = e == cudaSuccess ? permute_in(tmp, dev_layout, nb, count, st) : fail_cuda(e, "H2D", __FILE__, __LINE__);
    cudaFreeAsync(tmp, st);
    return rc;
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_factor_apply(const irk_factor* f, const double* y, double* x, void* stream) {
    IRK_ARG(f && y && x, "NULL argument");
    IRK_ARG(y != x, "x must not alias y");
    return factor_apply(f, y, x, (cudaStream_t)stream);
}

int irk_op_factor_apply(const irk_stage_op* op, const irk_factor* f, const double* v, double* x, int* fused,
                        void* stream) {
    IRK_ARG(op && f && v && x, "NULL argument");
    IRK_ARG(v != x, "x must not alias v");
    IRK_ARG(op->s == f->s && op->nb == f->nb && op->T_local == f->pat->T, "operator and factor shapes differ");
    cudaStream_t st = (cudaStream_t)stream;
    const int rc = factor_apply_fused(op, f, v, x, st);
    if (rc < 0) return rc;
    if (fused) *fused = rc == 0 ? 1 : 0;
    if (rc == 0) return IRK_OK;
    double* tmp = nullptr;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * op->s * op->T_local * op->nb, st));
    int r = irk_stage_op_apply(op, v, tmp, stream);
    if (r == IRK_OK) r = factor_apply(f, tmp, x, st);
    cudaFreeAsync(tmp, st);
    return r;
}

int irk_factor_apply_rhs(const irk_factor* f, int nrhs, const double* y, double* x, void* stream) {
    IRK_ARG(f && y && x, "NULL argument");
    IRK_ARG(y != x, "x must not alias y");
    IRK_ARG(nrhs >= 1, "nrhs must be positive");
    return factor_apply_rhs(f, nrhs, y, x, (cudaStream_t)stream);
}

int irk_factor_export(const irk_factor* f, double* fstage, double* dinv, double* fcoupling, void* stream) {
    IRK_ARG(f, "NULL factor");
    IRK_ARG(f->d_D || !fstage, "factor was created without store_diag");
    cudaStream_t st = (cudaStream_t)stream;
    if (fstage) IRK_TRY(factor_form_level0_d(f, st));
    const irk_pattern* p = f->pat;
    const int s = f->s, nb = f->nb;
    const int64_t bsz = block_doubles(nb), T = p->T, nnzb = p->nnzb;
    std::vector<uint8_t> keep(nnzb);
    IRK_CK(cudaMemcpy(keep.data(), f->d_keep, nnzb, cudaMemcpyDeviceToHost));
    double* out = nullptr;
    const int64_t nout = std::max<int64_t>({s * nnzb, s * T, (int64_t)s * s * T});
    IRK_CK(cudaMallocAsync(&out, sizeof(double) * bsz * nout, st));
    int rc = IRK_OK;
    if (fstage) {
        std::vector<int64_t> sL, dL, sD, dD, sU, dU, zs, zd;
        for (int k = 0; k < s && !rc; ++k) {
            std::vector<int64_t> sJ, dJ;
            for (int64_t j = 0; j < T; ++j)
                for (int64_t q = p->h_indptr[j]; q < p->h_indptr[j + 1]; ++q) {
                    const int64_t o = k * nnzb + q;
                    if (q < p->h_diag[j]) { sL.push_back((p->h_lptr[j] + q - p->h_indptr[j]) * s + k); dL.push_back(o); }
                    else if (q == p->h_diag[j]) { sD.push_back(j * s + k); dD.push_back(o); }
                    else if (f->u_stored) { sU.push_back((p->h_uptr[j] + q - p->h_diag[j] - 1) * s + k); dU.push_back(o); }
                    else if (keep[q]) { sJ.push_back(q); dJ.push_back(o); }
                    else { zs.push_back(-1); zd.push_back(o); }
                }
            if (!f->u_stored) rc = copy_blocks(f->ubase[k], sJ, out, dJ, bsz, f->uscale, st);
        }
        double* Lm = f->d_L;
        if (!rc && f->l_implicit) rc = factor_materialize_L(f, &Lm, st);
        if (!rc) rc = copy_blocks(Lm, sL, out, dL, bsz, 1.0, st);
        if (f->l_implicit && Lm) cudaFreeAsync(Lm, st);
        if (!rc) rc = copy_blocks(f->d_D, sD, out, dD, bsz, 1.0, st);
        if (!rc && f->u_stored) rc = copy_blocks(f->d_U, sU, out, dU, bsz, 1.0, st);
        if (!rc) rc = copy_blocks(nullptr, zs, out, zd, bsz, 1.0, st);
        if (!rc) rc = download_raw(out, nb, s * nnzb, fstage, st);
    }
    if (!rc && dinv) {
        std::vector<int64_t> si, di;
        for (int k = 0; k < s; ++k)
            for (int64_t i = 0; i < T; ++i) { si.push_back(i * s + k); di.push_back(k * T + i); }
        rc = copy_blocks(f->d_Dinv, si, out, di, bsz, 1.0, st);
        if (!rc) rc = download_raw(out, nb, s * T, dinv, st);
    }
    if (!rc && fcoupling && f->kind == IRK_FACTOR_COUPLED) {
        const int npairs = s * (s - 1) / 2;
        for (int k = 0; k < s && !rc; ++k)
            for (int l = 0; l < s && !rc; ++l) {
                std::vector<int64_t> si, di;
                for (int64_t i = 0; i < T; ++i) {
                    di.push_back(((int64_t)k * s + l) * T + i);
                    if (k > l) si.push_back(i * npairs + (k * (k - 1) / 2 + l));
                    else if (k < l) si.push_back(f->d_Cup ? i * npairs + (l * (l - 1) / 2 + k) : i);
                    else si.push_back(-1);
                }
                if (k > l) rc = copy_blocks(f->d_G, si, out, di, bsz, 1.0, st);
                else if (k < l) rc = f->d_Cup ? copy_blocks(f->d_Cup, si, out, di, bsz, 1.0, st)
                                              : copy_blocks(f->mass, si, out, di, bsz, f->cup_scale[k * s + l], st);
                else rc = copy_blocks(nullptr, si, out, di, bsz, 1.0, st);
            }
        if (!rc) rc = download_raw(out, nb, (int64_t)s * s * T, fcoupling, st);
    }
    cudaFreeAsync(out, st);
    IRK_CK(cudaStreamSynchronize(st));
    return rc;
}

}  // extern "C"
