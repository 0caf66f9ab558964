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
#include <vector>

#include "blockops.cuh"
#include "irk_internal.cuh"

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
    // persistent sweep: tasks in topological (level) order, claimed by ticket;
    // a task publishes flags[task] = epoch when its output is in memory
    const int32_t* order;
    int64_t ntasks;
    unsigned* flags;
    int* ticket;
    unsigned epoch;
    int64_t T, n;
    int s, nb, G_;
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

template <int S, bool EVEN>
static int unc_apply(const irk_factor* f, ApplyArgs& A, cudaStream_t st) {
    const int threads = ((A.G_ * A.nb + 31) / 32) * 32;
    const size_t smem_f = sizeof(double) * A.G_ * S * A.nb;
    const size_t smem_b = smem_f + sizeof(double) * S * A.nb;
    const int64_t nf = (int64_t)f->pat->T;
    IRK_TRY(run_sweep(f, k_unc_fwd<S, EVEN>, A, f->fwd, f->d_flags, f->d_ticket, threads, smem_f, st));
    IRK_TRY(run_sweep(f, k_unc_bwd<S, EVEN>, A, f->bwd, f->d_flags + nf, f->d_ticket + 1, threads, smem_b, st));
    return IRK_OK;
}

template <bool EVEN>
static int cpl_apply(const irk_factor* f, ApplyArgs& A, cudaStream_t st) {
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
    A.G_ = choose_groups(f->nb, 256);
}

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

int irk_factor_export(const irk_factor* f, double* fstage, double* dinv, double* fcoupling, void* stream) {
    IRK_ARG(f, "NULL factor");
    IRK_ARG(f->d_D || !fstage, "factor was created without store_diag");
    cudaStream_t st = (cudaStream_t)stream;
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
        if (!rc) rc = copy_blocks(f->d_L, sL, out, dL, bsz, 1.0, st);
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
