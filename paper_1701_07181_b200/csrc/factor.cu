// Block ILU(0) factorisation on the GPU (pull / left-looking form).
//
// Reference (push form): numba_backend.py:43-72 (Alg. 1/2) and :94-125
// (Alg. 3, stage-coupled).  For pivot i ascending the reference inverts D_i,
// then for every upper neighbour j forms L_ji = B_ji D_i^-1 and updates
// D_j -= L_ji U_ij.  Pulled to the row being finalised, row j receives those
// updates in ascending i, exactly the order of the push form; the cross-stage
// Schur updates of Alg. 3 (from stages l < k) precede the within-stage ones,
// again as in the reference.  Row j only needs rows i < j that are complete,
// so rows are processed level by level (level(j) = 1 + max level of its
// lower neighbours); every (stage, row) task of a level runs as one CTA.
//
// A task: D = coef*M_j + alpha*J_jj; [coupled: G = C_lo * Dinv_{l,j},
// D -= G * C_up]; for each kept lower neighbour i: L = (alpha*J_ji) Dinv_i,
// D -= L U_ij [general: U_jk -= L U_ik fill updates]; Dinv_j = inv(D) by
// Gauss-Jordan with partial pivoting (same pivot rows as LAPACK getrf, so
// det = exp(sum log|pivot|) and the singular decision of
// numba_backend.py:33-40 carry over), cond_1 = |D|_1 |D^-1|_1 > 1e14 fails.
// Block products are FP64 4x4 register-tiled GEMMs from shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "irk_internal.cuh"
#include "pipeline.cuh"

namespace irk {


struct FactorArgs {
    const int32_t *indptr, *indices, *diag, *lptr, *uptr, *tpos;
    const uint8_t* keep;
    const double* J[IRK_MAX_STAGES];
    const double* M;
    const double* Cexp;       // explicit couplings (s*s*T blocks) or NULL
    double alpha;
    double coef[IRK_MAX_STAGES];
    double cmix[IRK_MAX_STAGES * IRK_MAX_STAGES];
    double* L;
    double* Dinv;
    double* Dst;
    double* U;                // stored upper blocks (general mode) or NULL
    double* G;
    unsigned long long* fail_key;
    const int32_t* tasks;
    int64_t ntasks;
    int64_t T;
    int s, nb, nbp4, ld, KC;
    int coupled, literal, simplified;
    int split;                // Schur phase: one CTA task per (element, stage) (k_schur<1, ..>), F.s stages
};

__device__ __forceinline__ int pair_index(int hi, int lo) { return hi * (hi - 1) / 2 + lo; }

// element (a,b) of a device-layout block
__device__ __forceinline__ int64_t lay(int a, int b, int nb) {
    return ((int64_t)(b >> 1) * nb + a) * 2 + (b & 1);
}

// smem tile At[c - c0][a] (k-major, ld) <- scale * A(a, c), c in [c0, c0+kc).
// One 16-byte load per (column pair, row): consecutive threads read
// consecutive rows of a pair (coalesced).  c0 and kc are even.
__device__ void load_At(double* At, const double* __restrict__ A, double scale, int c0, int kc,
                        const FactorArgs& F) {
    const int nb = F.nb, ld = F.ld, n4 = F.nbp4;
    const int tot = (kc >> 1) * n4;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int pp = e / n4, a = e - pp * n4;
        const int p = (c0 >> 1) + pp;
        double2 v = make_double2(0.0, 0.0);
        if (A && a < nb && 2 * p < nb) {
            v = reinterpret_cast<const double2*>(A)[(int64_t)p * nb + a];
            v.x *= scale;
            v.y *= scale;
        }
        At[(2 * pp) * ld + a] = v.x;
        At[(2 * pp + 1) * ld + a] = v.y;
    }
}

// smem tile Bs[c - c0][b] (k-major) <- scale * B(c, b), c in [c0, c0+kc)
__device__ void load_Bs(double* Bs, const double* __restrict__ B, double scale, int c0, int kc,
                        const FactorArgs& F) {
    const int nb = F.nb, ld = F.ld;
    const int tot = (F.nbp4 >> 1) * kc;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int p = e / kc, cc = e - p * kc;   // consecutive threads: consecutive rows c
        const int c = c0 + cc;
        double2 v = make_double2(0.0, 0.0);
        if (B && c < nb && 2 * p < nb) {
            v = reinterpret_cast<const double2*>(B)[(int64_t)p * nb + c];
            v.x *= scale;
            v.y *= scale;
        }
        *reinterpret_cast<double2*>(Bs + cc * ld + 2 * p) = v;
    }
}

// Block products on the FP64 tensor cores: mma.sync.m8n8k4.f64 (DMMA).
// The padded block (F.nbp4, a multiple of 8) is cut into 8x8 output tiles;
// warp w owns tiles w, w+8, ... (MAXT per warp).  Fragment layout of
// m8n8k4.f64: A[r=lane/4][k=lane%4], B[k=lane%4][c=lane/4],
// C[r=lane/4][c=2*(lane%4)+{0,1}].
template <int MAXT>
struct Tiles {
    double acc[MAXT][2];
    __device__ void zero() {
#pragma unroll
        for (int t = 0; t < MAXT; ++t) acc[t][0] = acc[t][1] = 0.0;
    }
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// acc(tile) += A(tile rows, k) B(k, tile cols) for k < kc (kc % 4 == 0);
// AT / BS are k-major with leading dimension ld.
template <int MAXT>
__device__ __forceinline__ void mma_chunk(Tiles<MAXT>& T, const double* AT, const double* BS,
                                          int kc, const FactorArgs& F) {
    const int tpr = F.nbp4 >> 3;
    const int ntile = tpr * tpr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int fr = lane >> 2, fk = lane & 3;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
        const int tile = warp + t * nw;
        if (tile >= ntile) break;
        const int r0 = (tile / tpr) * 8, c0 = (tile % tpr) * 8;
        const double* ap = AT + fk * F.ld + r0 + fr;
        const double* bp = BS + fk * F.ld + c0 + fr;
#pragma unroll 5
        for (int k = 0; k < kc; k += 4) dmma(T.acc[t][0], T.acc[t][1], ap[k * F.ld], bp[k * F.ld]);
    }
}

struct Smem {
    double* D;    // nbp4 x ld  (row-major D[a][b])
    double* Lt;   // nbp4 x ld  (k-major L^T: Lt[c][a] = L(a,c))
    double* At;   // KC x ld
    double* Bs;   // KC x ld
    double* colk; // nbp4
    double* red;  // 64
    int* piv;     // nbp4
    int* misc;    // 8
};

__device__ Smem carve(const FactorArgs& F) {
    extern __shared__ __align__(16) double smem[];
    Smem S;
    const int big = F.nbp4 * F.ld, chunk = F.KC * F.ld;
    S.D = smem;
    S.Lt = S.D + big;
    S.At = S.Lt + big;
    S.Bs = S.At + chunk;
    S.colk = S.Bs + chunk;
    S.red = S.colk + F.nbp4;
    S.piv = reinterpret_cast<int*>(S.red + 64);
    S.misc = S.piv + F.nbp4;
    return S;
}

// out = A * B (A scaled by sa, B scaled by sb): result stays in tiles
template <int MAXT>
__device__ void gemm_global(Tiles<MAXT>& T, const double* A, double sa, const double* B, double sb,
                            Smem& S, const FactorArgs& F) {
    T.zero();
    for (int c0 = 0; c0 < F.nbp4; c0 += F.KC) {
        const int kc = min(F.KC, F.nbp4 - c0);
        load_At(S.At, A, sa, c0, kc, F);
        load_Bs(S.Bs, B, sb, c0, kc, F);
        __syncthreads();
        mma_chunk<MAXT>(T, S.At, S.Bs, kc, F);
        __syncthreads();
    }
}

// tiles = Lt(smem, full) * B
template <int MAXT>
__device__ void gemm_lt(Tiles<MAXT>& T, const double* B, double sb, Smem& S, const FactorArgs& F) {
    T.zero();
    for (int c0 = 0; c0 < F.nbp4; c0 += F.KC) {
        const int kc = min(F.KC, F.nbp4 - c0);
        load_Bs(S.Bs, B, sb, c0, kc, F);
        __syncthreads();
        mma_chunk<MAXT>(T, S.Lt + c0 * F.ld, S.Bs, kc, F);
        __syncthreads();
    }
}

template <int MAXT, typename Fn>
__device__ __forceinline__ void for_tiles(Tiles<MAXT>& T, const FactorArgs& F, Fn fn) {
    const int tpr = F.nbp4 >> 3;
    const int ntile = tpr * tpr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
        const int tile = warp + t * nw;
        if (tile >= ntile) break;
        const int r = (tile / tpr) * 8 + (lane >> 2), c = (tile % tpr) * 8 + 2 * (lane & 3);
        fn(r, c, T.acc[t][0]);
        fn(r, c + 1, T.acc[t][1]);
    }
}

// store tiles as a device-layout block (rows/cols < nb) and as Lt in smem
template <int MAXT>
__device__ void store_L(Tiles<MAXT>& T, double* dst, Smem& S, const FactorArgs& F) {
    for_tiles<MAXT>(T, F, [&](int a, int b, double v) {
        S.Lt[b * F.ld + a] = v;
        if (dst && a < F.nb && b < F.nb) dst[lay(a, b, F.nb)] = v;
    });
    __syncthreads();
}

template <int MAXT>
__device__ void sub_into_D(Tiles<MAXT>& T, Smem& S, const FactorArgs& F) {
    for_tiles<MAXT>(T, F, [&](int a, int b, double v) { S.D[a * F.ld + b] -= v; });
    __syncthreads();
}

// copy smem rows of D (a<nb, b<nb) into a device-layout block
__device__ void store_D(const double* D, double* dst, const FactorArgs& F) {
    const int nb = F.nb, P = (nb + 1) >> 1;
    for (int e = threadIdx.x; e < nb * P; e += blockDim.x) {
        const int p = e / nb, a = e - p * nb;
        double2 v;
        v.x = D[a * F.ld + 2 * p];
        v.y = (2 * p + 1 < nb) ? D[a * F.ld + 2 * p + 1] : 0.0;
        reinterpret_cast<double2*>(dst)[e] = v;
    }
}

__device__ double block_norm1(const double* D, Smem& S, const FactorArgs& F) {
    // max column abs-sum, NaN propagating (np.abs(b).sum(axis=0).max())
    const int nb = F.nb;
    double v = -1.0;
    int isnan_flag = 0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        double s = 0.0;
        for (int a = 0; a < nb; ++a) s += fabs(D[a * F.ld + b]);
        if (s != s) isnan_flag = 1;
        v = fmax(v, s);
    }
    // block reduce max over warps
    for (int o = 16; o; o >>= 1) {
        v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        isnan_flag |= __shfl_xor_sync(0xffffffffu, isnan_flag, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { S.red[w] = isnan_flag ? __longlong_as_double(0x7ff8000000000000LL) : v; }
    __syncthreads();
    double r = -1.0;
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) {
        const double x = S.red[i];
        if (x != x) { r = x; break; }
        r = fmax(r, x);
    }
    __syncthreads();
    return r;
}

// Gauss-Jordan inverse of S.D (nb x nb) with partial pivoting (row
// interchanges, the pivot rows LAPACK getrf would pick: first max |a_rk|).
// One CTA barrier per pivot step: every warp finds the pivot redundantly from
// the current buffer, every thread writes its elements of the next buffer
// (S.D <-> S.Lt, Lt is free here); the column un-permutation is folded into
// the final store.  The inverse is written to `dst` (device layout).
// Returns (in all threads) whether the pivot passed the reference checks
// (numba_backend.py:33-40,53-55: det = exp(sum log|u_kk|) nonzero and finite,
// cond_1 <= 1e14).
__device__ bool gj_invert(Smem& S, const FactorArgs& F, double* dst) {
    const int nb = F.nb, ld = F.ld;
    const int lane = threadIdx.x & 31;
    const int nthr = blockDim.x;
    const int dr = nthr / nb, dc = nthr - (nthr / nb) * nb;   // stride of the flat (r,c) walk
    const int r0 = threadIdx.x / nb, c0 = threadIdx.x - (threadIdx.x / nb) * nb;
    const int tot = nb * nb;
    double* A = S.D;
    double* B = S.Lt;
    const double n1 = block_norm1(A, S, F);
    double logdet = 0.0;
    int zero = 0;
    for (int k = 0; k < nb; ++k) {
        double best = -1.0;
        int bi = k;
        for (int r = k + lane; r < nb; r += 32) {
            const double v = fabs(A[r * ld + k]);
            if (v > best) { best = v; bi = r; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        const int p = bi;
        const double piv = A[p * ld + k];
        const double inv = 1.0 / piv;
        if (threadIdx.x == 0) {
            S.piv[k] = p;
            logdet += log(fabs(piv));
            if (piv == 0.0) zero = 1;
        }
        const double* P = A + p * ld;
        int r = r0, c = c0;
        for (int e = threadIdx.x; e < tot; e += nthr) {
            double v;
            if (r == k) {
                v = (c == k) ? inv : P[c] * inv;
            } else {
                const int src = (r == p) ? k : r;   // row p receives the old row k
                const double f = A[src * ld + k];
                v = (c == k) ? -f * inv : fma(-f, P[c] * inv, A[src * ld + c]);
            }
            B[r * ld + c] = v;
            c += dc;
            r += dr;
            if (c >= nb) { c -= nb; r += 1; }
        }
        __syncthreads();
        double* t = A;
        A = B;
        B = t;
    }
    // column un-permutation: Y = X S_{n-1} ... S_0  ->  Y[:, c] = X[:, idx[c]]
    int* idx = S.misc + 8;
    if (threadIdx.x == 0) {
        for (int c = 0; c < nb; ++c) idx[c] = c;
        for (int k = nb - 1; k >= 0; --k) {
            const int p = S.piv[k];
            const int tmp = idx[k];
            idx[k] = idx[p];
            idx[p] = tmp;
        }
    }
    const double n2 = block_norm1(A, S, F);   // permutation invariant; has barriers
    {
        const int P2 = (nb + 1) >> 1;
        for (int e = threadIdx.x; e < nb * P2; e += nthr) {
            const int pp = e / nb, a = e - pp * nb;
            double2 v;
            v.x = A[a * ld + idx[2 * pp]];
            v.y = (2 * pp + 1 < nb) ? A[a * ld + idx[2 * pp + 1]] : 0.0;
            reinterpret_cast<double2*>(dst)[e] = v;
        }
    }
    if (threadIdx.x == 0) {
        const double det = exp(logdet);
        const double cond = n1 * n2;
        const bool bad = zero || det == 0.0 || !isfinite(det) || !(cond <= 1e14);
        S.misc[1] = bad ? 1 : 0;
    }
    __syncthreads();
    const bool ok = S.misc[1] == 0;
    __syncthreads();
    return ok;
}

// INVERT=false: Schur updates only; the updated pivot block goes to F.Dst and
// is inverted by the batched warp kernel (inverse.cu).
template <int MAXT, bool INVERT>
__global__ void __launch_bounds__(256) k_factor(FactorArgs F) {
    Smem S = carve(F);
    const int nb = F.nb, ld = F.ld;
    const int64_t bsz = (int64_t)nb * 2 * ((nb + 1) >> 1);
    const int npairs = F.s * (F.s - 1) / 2;
    Tiles<MAXT> T;
    for (int64_t t = blockIdx.x; t < F.ntasks; t += gridDim.x) {
        const int64_t code = F.tasks[t];
        const int k = (int)(code / F.T);
        const int j = (int)(code - (int64_t)k * F.T);
        const double* Jk = F.J[k];
        const int dpos = F.diag[j];
        const bool keep_d = F.keep[dpos] != 0;
        // D = fl(alpha*J_jj) + fl(coef*M_j)  (build_stage_matrix, precond.py:48-54)
        for (int e = threadIdx.x; e < F.nbp4 * ld; e += blockDim.x) S.D[e] = 0.0;
        __syncthreads();
        if (keep_d) {
            const int P = (nb + 1) >> 1;
            const double2* Jd = reinterpret_cast<const double2*>(Jk + (int64_t)dpos * bsz);
            const double2* Md = F.M ? reinterpret_cast<const double2*>(F.M + (int64_t)j * bsz) : nullptr;
            for (int e = threadIdx.x; e < nb * P; e += blockDim.x) {
                const int p = e / nb, a = e - p * nb;
                const double2 v = Jd[e];
                double x0 = __dmul_rn(F.alpha, v.x), x1 = __dmul_rn(F.alpha, v.y);
                if (Md) {
                    const double2 m = Md[e];
                    x0 = __dadd_rn(x0, __dmul_rn(F.coef[k], m.x));
                    x1 = __dadd_rn(x1, __dmul_rn(F.coef[k], m.y));
                }
                S.D[a * ld + 2 * p] = x0;
                if (2 * p + 1 < nb) S.D[a * ld + 2 * p + 1] = x1;
            }
        }
        __syncthreads();
        if (F.coupled) {
            // cross-stage Schur updates from earlier stages l < k (numba_backend.py:117-124)
            for (int l = 0; l < k; ++l) {
                const double* clo;
                double slo;
                if (F.Cexp) { clo = F.Cexp + (((int64_t)k * F.s + l) * F.T + j) * bsz; slo = 1.0; }
                else { clo = F.M + (int64_t)j * bsz; slo = F.cmix[k * F.s + l]; }
                gemm_global<MAXT>(T, clo, slo, F.Dinv + ((int64_t)j * F.s + l) * bsz, 1.0, S, F);
                store_L<MAXT>(T, F.G + ((int64_t)j * npairs + pair_index(k, l)) * bsz, S, F);
                const double* cup;
                double sup;
                if (F.literal) { cup = F.Dst + ((int64_t)j * F.s + l) * bsz; sup = 1.0; }
                else if (F.Cexp) { cup = F.Cexp + (((int64_t)l * F.s + k) * F.T + j) * bsz; sup = 1.0; }
                else { cup = F.M + (int64_t)j * bsz; sup = F.cmix[l * F.s + k]; }
                gemm_lt<MAXT>(T, cup, sup, S, F);
                sub_into_D<MAXT>(T, S, F);
            }
        }
        // within-stage updates from kept lower neighbours, ascending
        const int q0 = F.indptr[j];
        const int lq0 = F.lptr[j];
        for (int q = q0; q < dpos; ++q) {
            const int i = F.indices[q];
            const int tq = F.tpos[q];   // (i, j) block in row i
            const bool keep_lo = F.keep[q] != 0;
            const bool keep_up = tq >= 0 && F.keep[tq] != 0;
            double* Lout = F.L ? F.L + ((int64_t)(lq0 + (q - q0)) * F.s + k) * bsz : nullptr;
            if (!keep_up) {
                // reference never touches this block: it stays B_ji (or 0 if dropped)
                for (int e = threadIdx.x; Lout && e < nb * nb; e += blockDim.x) {
                    const int a = e / nb, b = e - a * nb;
                    Lout[lay(a, b, nb)] = keep_lo ? F.alpha * Jk[(int64_t)q * bsz + lay(a, b, nb)] : 0.0;
                }
                __syncthreads();
                continue;
            }
            gemm_global<MAXT>(T, keep_lo ? Jk + (int64_t)q * bsz : nullptr, F.alpha,
                              F.Dinv + ((int64_t)i * F.s + k) * bsz, 1.0, S, F);
            store_L<MAXT>(T, Lout, S, F);
            if (!keep_lo) continue;   // L == 0: D unchanged
            const double* Ub;
            double su;
            if (F.U) { Ub = F.U + ((int64_t)(F.uptr[i] + (tq - F.diag[i] - 1)) * F.s + k) * bsz; su = 1.0; }
            else { Ub = Jk + (int64_t)tq * bsz; su = F.alpha; }
            gemm_lt<MAXT>(T, Ub, su, S, F);
            sub_into_D<MAXT>(T, S, F);
            if (!F.simplified) {
                // fill-limited updates U_jk2 -= L U_ik2 (numba_backend.py:64-71)
                for (int kik = F.indptr[i]; kik < F.indptr[i + 1]; ++kik) {
                    const int k2 = F.indices[kik];
                    if (k2 <= j || k2 == i || !F.keep[kik]) continue;
                    int kjk = -1;
                    for (int qq = dpos + 1; qq < F.indptr[j + 1]; ++qq)
                        if (F.indices[qq] == k2) { kjk = qq; break; }
                    if (kjk < 0 || !F.keep[kjk]) continue;
                    const double* Uik = F.U + ((int64_t)(F.uptr[i] + (kik - F.diag[i] - 1)) * F.s + k) * bsz;
                    double* Ujk = F.U + ((int64_t)(F.uptr[j] + (kjk - dpos - 1)) * F.s + k) * bsz;
                    gemm_lt<MAXT>(T, Uik, 1.0, S, F);
                    for_tiles<MAXT>(T, F, [&](int a, int b, double v) {
                        if (a < nb && b < nb) Ujk[lay(a, b, nb)] -= v;
                    });
                    __syncthreads();
                }
            }
        }
        if (F.Dst) {
            store_D(S.D, F.Dst + ((int64_t)j * F.s + k) * bsz, F);
            __syncthreads();
        }
        if (INVERT) {
            const bool ok = gj_invert(S, F, F.Dinv + ((int64_t)j * F.s + k) * bsz);
            if (!ok && threadIdx.x == 0) atomicMin(F.fail_key, (unsigned long long)((int64_t)k * F.T + j));
            __syncthreads();
        }
    }
}

// U[uq][k] = keep ? alpha * J_k[q] : 0 for every upper block (general mode)
__global__ void k_init_upper(FactorArgs F, int64_t T) {
    const int nb = F.nb;
    const int64_t bsz = (int64_t)nb * 2 * ((nb + 1) >> 1);
    for (int64_t i = blockIdx.x; i < T; i += gridDim.x) {
        const int d = F.diag[i], q1 = F.indptr[i + 1], u0 = F.uptr[i];
        for (int q = d + 1; q < q1; ++q)
            for (int k = 0; k < F.s; ++k) {
                double* dst = F.U + ((int64_t)(u0 + q - d - 1) * F.s + k) * bsz;
                const double* src = F.J[k] + (int64_t)q * bsz;
                const bool kp = F.keep[q] != 0;
                for (int e = threadIdx.x; e < bsz; e += blockDim.x) dst[e] = kp ? F.alpha * src[e] : 0.0;
            }
    }
}

static void levels_forward(const irk_pattern* p, const std::vector<uint8_t>& keep, std::vector<int64_t>& lev) {
    const int64_t T = p->T;
    lev.assign(T, 0);
    std::vector<int32_t> tpos(p->nnzb);
    for (int64_t j = 0; j < T; ++j) {
        int64_t L = 0;
        for (int64_t q = p->h_indptr[j]; q < p->h_diag[j]; ++q) {
            const int64_t i = p->h_indices[q];
            // dependency if the reference reads row i for row j (either block kept)
            const int64_t* b = p->h_indices.data() + p->h_indptr[i];
            const int64_t* e = p->h_indices.data() + p->h_indptr[i + 1];
            const int64_t* f = std::lower_bound(b, e, j);
            const bool up = (f != e && *f == j) && keep[p->h_indptr[i] + (f - b)];
            if (keep[q] || up) L = std::max(L, lev[i] + 1);
        }
        lev[j] = L;
    }
}

static void levels_backward(const irk_pattern* p, const std::vector<uint8_t>& keep, std::vector<int64_t>& lev) {
    const int64_t T = p->T;
    lev.assign(T, 0);
    for (int64_t i = T - 1; i >= 0; --i) {
        int64_t L = 0;
        for (int64_t q = p->h_diag[i] + 1; q < p->h_indptr[i + 1]; ++q) {
            const int64_t j = p->h_indices[q];
            const int64_t* b = p->h_indices.data() + p->h_indptr[j];
            const int64_t* e = p->h_indices.data() + p->h_indptr[j + 1];
            const int64_t* f = std::lower_bound(b, e, i);
            const bool lo = (f != e && *f == i) && keep[p->h_indptr[j] + (f - b)];
            if (keep[q] || lo) L = std::max(L, lev[j] + 1);
        }
        lev[i] = L;
    }
}

// group task codes by level: tasks (k, elem) with level = lev[elem] + skew(k)
static int build_sched(irk_sched& S, const std::vector<int64_t>& lev, int64_t T, int s, bool per_stage,
                       int skew_dir, const std::vector<uint8_t>* include = nullptr) {
    int64_t maxl = 0;
    for (auto v : lev) maxl = std::max(maxl, v);
    const int kstages = per_stage ? s : 1;
    const int64_t nlev = maxl + 1 + (per_stage && skew_dir != 0 ? s - 1 : 0);
    std::vector<int64_t> cnt(nlev + 1, 0);
    auto level_of = [&](int k, int64_t e) -> int64_t {
        if (!per_stage || skew_dir == 0) return lev[e];
        return lev[e] + (skew_dir > 0 ? k : (s - 1 - k));
    };
    for (int k = 0; k < kstages; ++k)
        for (int64_t e = 0; e < T; ++e)
            if (!include || (*include)[e]) cnt[level_of(k, e) + 1]++;
    for (int64_t l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
    std::vector<int32_t> order(cnt[nlev]);
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int k = 0; k < kstages; ++k)
        for (int64_t e = 0; e < T; ++e)
            if (!include || (*include)[e]) order[pos[level_of(k, e)]++] = (int32_t)((int64_t)k * T + e);
    S.nlevels = nlev;
    S.h_lvl_ptr = cnt;
    IRK_CK(cudaMalloc(&S.d_order, sizeof(int32_t) * std::max<size_t>(order.size(), 1)));
    IRK_CK(cudaMemcpy(S.d_order, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice));
    return IRK_OK;
}

// apply schedules: uncoupled -> element tasks; coupled -> (stage, element)
// tasks on stage-skewed levels
int choose_groups(int nb, int max_threads);   // matvec.cu

int build_apply_schedules(irk_factor* f, const std::vector<uint8_t>& keep) {
    std::vector<int64_t> levf, levb;
    {
        const irk_pattern* p = f->pat;
        int md = 0;
        for (int64_t i = 0; i < p->T; ++i) {
            md = std::max<int>(md, (int)(p->h_diag[i] - p->h_indptr[i]));
            md = std::max<int>(md, (int)(p->h_indptr[i + 1] - p->h_diag[i] - 1));
        }
        f->maxdeg = md;
    }
    levels_forward(f->pat, keep, levf);
    levels_backward(f->pat, keep, levb);
    // coupled: (stage, element) tasks on stage-skewed levels for the generic kernels, or
    // element tasks (all stages, coupling solved in the task) for the pipelined sweeps
    // (a deep element DAG -- natural numbering -- keeps the stage-skewed tasks: s times more
    // tasks per level and a shorter critical path than element tasks with in-task coupling)
    const int64_t depth = std::max(levf.empty() ? 0 : *std::max_element(levf.begin(), levf.end()),
                                   levb.empty() ? 0 : *std::max_element(levb.begin(), levb.end())) + 1;
    f->cpl_pipe = f->kind == IRK_FACTOR_COUPLED && f->nb % 2 == 0 && f->s >= 2 && f->s <= 4 &&
                  choose_groups(f->nb, 256) * f->nb <= 256 && depth <= 16 && !getenv("IRK_CPL_GENERIC");
    const bool cpl = f->kind == IRK_FACTOR_COUPLED && !f->cpl_pipe;
    IRK_TRY(build_sched(f->fwd, levf, f->pat->T, f->s, cpl, +1));
    if (f->l_implicit) {
        // rows without a kept upper block are finished by the forward sweep
        const irk_pattern* p = f->pat;
        std::vector<uint8_t> hasup(p->T, 0);
        for (int64_t i = 0; i < p->T; ++i)
            for (int64_t q = p->h_diag[i] + 1; q < p->h_indptr[i + 1]; ++q)
                if (keep[q]) hasup[i] = 1;
        IRK_TRY(build_sched(f->bwd, levb, p->T, f->s, false, -1, &hasup));
        IRK_CK(cudaMalloc(&f->d_hasup, std::max<int64_t>(p->T, 1)));
        IRK_CK(cudaMemcpy(f->d_hasup, hasup.data(), p->T, cudaMemcpyHostToDevice));
    } else {
        IRK_TRY(build_sched(f->bwd, levb, f->pat->T, f->s, cpl, -1));
    }
    if (f->kind != IRK_FACTOR_COUPLED && !f->l_implicit) {
        // forward levels whose elements have no kept lower block: z_i = y_i (uncoupled only:
        // a coupled element still needs its stage coupling)
        const irk_pattern* p = f->pat;
        std::vector<char> has(f->fwd.nlevels, 0);
        for (int64_t i = 0; i < p->T; ++i)
            for (int64_t q = p->h_indptr[i]; q < p->h_diag[i]; ++q)
                if (keep[q]) has[levf[i]] = 1;
        f->fwd.h_trivial.assign(f->fwd.nlevels, 0);
        for (int64_t l = 0; l < f->fwd.nlevels; ++l) f->fwd.h_trivial[l] = !has[l];
    }
    const int64_t nflags = 2 * (cpl ? (int64_t)f->s : 1) * f->pat->T;
    IRK_CK(cudaMalloc(&f->d_flags, sizeof(unsigned) * nflags));
    IRK_CK(cudaMemset(f->d_flags, 0, sizeof(unsigned) * nflags));
    IRK_CK(cudaMalloc(&f->d_ticket, sizeof(int) * 2));
    return IRK_OK;
}

static size_t factor_smem(int nbp4, int ld, int KC) {
    return sizeof(double) * ((size_t)2 * nbp4 * ld + (size_t)2 * KC * ld + nbp4 + 64) +
           sizeof(int) * (2 * nbp4 + 16);
}

// ---------------------------------------------------------------------------
// Schur phase, stage-uncoupled simplified ILU(0) with stage-shared off-diagonal
// blocks (B_ji = alpha J_ji for every stage; the benchmark's path).
//
// One CTA per element j and all S stages; warp w owns the 8-row strip
// [8w, 8w+8) of every nb x nb block (NB = 8 * warps).  Per kept lower
// neighbour i the CTA bulk-copies J_ji, J_ij and Dinv_{k,i} (k < S) into
// shared memory -- one cp.async.bulk per column pair, at a pair stride of
// 2 NB + 8 doubles so that both DMMA operand fragments read conflict-free --
// then
//   T_k = J_ji Dinv_{k,i}          (DMMA m8n8k4, J_ji fragments shared by the S stages)
//   L_k = alpha T_k  -> global      (numba_backend.py:58-61, L_ji = B_ji D_i^-1)
//   D_k += (-alpha L_k) J_ij        (D_j -= L_ji U_ij, U_ij = alpha J_ij)
// with -alpha L_k staged back into the (consumed) Dinv slots as the A operand.
// The pivot accumulators D_k = fl(alpha J_jj) + fl(coef_k M_j) stay in
// registers across neighbours and are stored once for the batched inverse.
// ---------------------------------------------------------------------------
template <int NB>
struct SchurGeo {
    static constexpr int NT = NB / 8;          // 8x8 tiles per strip row = warps
    static constexpr int NP = NB / 2;          // column pairs
    static constexpr int LDP = 2 * NB + 8;     // pair stride (doubles), = 8 mod 16
    static constexpr int SLOT = NP * LDP;      // doubles per staged block
    // warp-private A' strip (8 x NB, row-major): row stride = 4 or 12 mod 16 makes
    // both the C-fragment double2 stores and the A-fragment loads conflict-free
    static constexpr int LDA = ((NB + 3) / 4 * 4) % 16 == 4 || ((NB + 3) / 4 * 4) % 16 == 12
                                   ? (NB + 3) / 4 * 4 : (NB + 3) / 4 * 4 + 4;
    static_assert(NT * 8 * LDA <= SLOT, "A' strips must fit in one staged block");
};

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TWO: two-phase unit -- GEMM1 of all stages (J_ji fragments loaded once for S stages), one
// barrier, A'_k into the consumed Dinv slots, GEMM2 of all stages (J_ij fragments loaded once),
// one barrier, refills: 2 barriers per unit instead of S + 1, fewer fragment loads
// MODE 2: no CTA barrier -- A'_k goes from the C fragments to the A fragments by shuffles (the
// staged blocks are read-only), every warp counts itself out of a slot when it has read it for
// the last time and the last warp out refills the slot with the next unit's block
// MODE 3 (S >= 2): MODE 2 with two Dinv slots used alternately (4 slots instead of S + 2): at
// NB = 56 (config 2, nb = 50) two CTAs fit on an SM instead of one.  (The register cap comes from
// __launch_bounds__' min-CTA argument; __maxnreg__(144) for the 224-thread CTAs was tried and
// drops a CTA per SM: registers are allocated per warp in larger units.)
// CTAs per SM that shared memory allows, capped so that a thread keeps >= 128 registers
template <int S, int NB, int NSL = S + 2>
constexpr int schur_min_ctas() {
    const int by_smem = 232448 / (NSL * SchurGeo<NB>::SLOT * 8 + 1280);
    // registers a thread needs: the pivot accumulators (S strips of NB / 8 tiles) + one product strip
    const int need = S >= 3 ? 128 : (S == 2 ? 112 : 80);
    const int by_regs = 65536 / (4 * NB * need);
    const int m = by_smem < by_regs ? by_smem : by_regs;
    return m < 1 ? 1 : m;
}

template <int S, int NB, int MODE = 0>
__global__ void __launch_bounds__(4 * NB, MODE == 1 ? 1 : schur_min_ctas<S, NB, (MODE == 3 ? 4 : S + 2)>()) k_schur(FactorArgs F, const int32_t* __restrict__ elems, int64_t nelem) {
    using Gm = SchurGeo<NB>;
    constexpr int NT = Gm::NT, LDP = Gm::LDP, SLOT = Gm::SLOT;
    // NB = nb rounded up to 8: the padding rows / columns of the staged blocks are
    // zero (slots zeroed once; bulk copies write only the nb x nb part), so the
    // padded DMMA tiles leave the nb x nb results exact
    const int nbv = F.nb, Pv = (nbv + 1) >> 1;
    // k-steps of 4 that hold data (nb = 50 runs 13 of 14); used by the two-phase units only: a
    // runtime bound in the NB = 40 barrier-free loops costs more than it saves (1.68 -> 1.88 ms)
    const int KK = (nbv + 3) >> 2;
    const int64_t BSZ = (int64_t)nbv * 2 * Pv;      // device block (column-pair layout)
    constexpr int SJ = 0, SU = 1;   // slots: J_ji, J_ij, then Dinv_k / A'_k at 2 + k
    extern __shared__ __align__(128) double shs[];
    __shared__ __align__(8) uint64_t bars[S + 2];
    __shared__ int outcnt[S + 2];   // MODE 2: warps that have left each slot
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fr = lane >> 2, fk = lane & 3;
    const int r0 = warp * 8;
    const double* J = F.J[0];
    // split mode (S == 1 instantiation over (element, stage) tasks, element-major so that the F.s
    // CTAs of an element run side by side and share its J blocks in L2): task it -> element
    // elems[it / ST], stage it % ST; otherwise one task per element with all S == ST stages
    const int ST = F.split ? F.s : S;
    auto elem_of = [&](int64_t it) -> int { return elems[F.split ? it / ST : it]; };
    auto stage_of = [&](int64_t it) -> int { return F.split ? (int)(it % ST) : 0; };
    constexpr int NSL = MODE == 3 ? 4 : S + 2;      // staged-block slots
    static_assert(MODE != 3 || S >= 2, "MODE 3 needs at least two stages");
    if (threadIdx.x < S + 2) outcnt[threadIdx.x] = 0;
    if (nbv != NB)
        for (int e = threadIdx.x; e < NSL * SLOT; e += blockDim.x) shs[e] = 0.0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < S + 2; ++b) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phases = 0;   // bit b: parity of the next completion of slot b
    auto wait_slot = [&](int b) {
        mbar_wait(&bars[b], (phases >> b) & 1u);
        phases ^= 1u << b;
    };
    // warp 0 refills slot b with a block (one bulk copy per column pair); the
    // caller has made every earlier generic access to the slot CTA-visible
    auto fill = [&](int b, const double* src) {
        if (warp == 0) {
            if (lane == 0) {
                fence_proxy_async_smem();
                mbar_expect_tx(&bars[b], (uint32_t)(Pv * nbv * 16));
            }
            __syncwarp();
            for (int p = lane; p < Pv; p += 32)
                bulk_g2s(shs + (size_t)b * SLOT + p * LDP, src + (int64_t)p * nbv * 2, nbv * 16, &bars[b]);
        }
    };
    // a "unit" is a (element, lower neighbour q) pair whose Schur update runs on
    // the tensor cores (both blocks kept); units are visited in CTA order
    struct Unit { int64_t it; int q; int i, tq; };
    auto find_unit = [&](int64_t it, int q) -> Unit {
        for (; it < nelem; it += gridDim.x) {
            const int j = elem_of(it);
            const int dpos = F.diag[j];
            if (q < 0) q = F.indptr[j];
            for (; q < dpos; ++q) {
                const int tq = F.tpos[q];
                if (F.keep[q] && tq >= 0 && F.keep[tq]) return Unit{it, q, F.indices[q], tq};
            }
            q = -1;
        }
        return Unit{-1, -1, -1, -1};
    };
    auto src_dinv = [&](const Unit& u, int k) { return F.Dinv + ((int64_t)u.i * ST + stage_of(u.it) + k) * BSZ; };
    Unit nxt = find_unit(blockIdx.x, -1);
    if (nxt.it >= 0) {
        fill(SJ, J + (int64_t)nxt.q * BSZ);
        fill(SU, J + (int64_t)nxt.tq * BSZ);
#pragma unroll
        for (int k = 0; k < (MODE == 3 ? 2 : S); ++k) fill(2 + k, src_dinv(nxt, k));
    }
    int dm = 0;   // MODE 3: Dinv blocks consumed so far (block m sits in slot 2 + (m & 1))
    auto frag_a = [&](const double* slotp, int kk) -> double {   // A(r0 + fr, 4kk + fk)
        return slotp[((4 * kk + fk) >> 1) * LDP + 2 * (r0 + fr) + (fk & 1)];
    };
    auto frag_b = [&](const double* slotp, int kk, int t) -> double {   // B(4kk + fk, 8t + fr)
        return slotp[((8 * t + fr) >> 1) * LDP + 2 * (4 * kk + fk) + (fr & 1)];
    };
    // double2 index of (row r0 + fr, column pair 4t + fk) in a device block; -1: padding
    auto gl_off = [&](int t) -> int64_t {
        const int pp = 4 * t + fk, a = r0 + fr;
        return (pp < Pv && a < nbv) ? (int64_t)pp * nbv + a : -1;
    };

    for (int64_t it = blockIdx.x; it < nelem; it += gridDim.x) {
        const int j = elem_of(it);
        const int ks = stage_of(it);
        const int dpos = F.diag[j];
        double dacc[S][NT][2];
        // ---- D_k = fl(alpha J_jj) + fl(coef_k M_j)  (build_stage_matrix, precond.py:48-54)
        {
            const bool keep_d = F.keep[dpos] != 0;
            const double2* Jd = reinterpret_cast<const double2*>(J + (int64_t)dpos * BSZ);
            const double2* Md = F.M ? reinterpret_cast<const double2*>(F.M + (int64_t)j * BSZ) : nullptr;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int64_t go = gl_off(t);
                const double2 jv = go >= 0 ? Jd[go] : make_double2(0.0, 0.0);
                const double2 mv = (Md && go >= 0) ? Md[go] : make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    double x0 = __dmul_rn(F.alpha, jv.x), x1 = __dmul_rn(F.alpha, jv.y);
                    if (Md) {
                        x0 = __dadd_rn(x0, __dmul_rn(F.coef[ks + k], mv.x));
                        x1 = __dadd_rn(x1, __dmul_rn(F.coef[ks + k], mv.y));
                    }
                    dacc[k][t][0] = keep_d ? x0 : 0.0;
                    dacc[k][t][1] = keep_d ? x1 : 0.0;
                }
            }
        }
        const int q0 = F.indptr[j];
        const int lq0 = F.lptr[j];
        for (int q = q0; q < dpos; ++q) {
            double* Lout = F.L ? F.L + ((int64_t)(lq0 + (q - q0)) * ST + ks) * BSZ : nullptr;   // NULL: implicit L
            if (!(nxt.it == it && nxt.q == q)) {
                // not a unit: the reference never forms L_ji D_i^-1 here, so L stays
                // B_ji (upper block dropped) or 0 (lower block dropped); D unchanged
                const int tq = F.tpos[q];
                const bool keep_lo = F.keep[q] != 0;
                const bool keep_up = tq >= 0 && F.keep[tq] != 0;
                const double* Jq = J + (int64_t)q * BSZ;
                if (F.L)
                    for (int64_t e = threadIdx.x; e < S * BSZ; e += blockDim.x) {
                        const int64_t o = e % BSZ;
                        Lout[e] = (keep_lo && !keep_up) ? F.alpha * Jq[o] : 0.0;
                    }
                continue;
            }
            const Unit cur = nxt;
            nxt = find_unit(it, q + 1);
            const bool more = nxt.it >= 0;
            if constexpr (MODE == 2 || MODE == 3) {
                // this warp is done with slot b: the last warp out refills it (src != NULL).
                // (Measured and dropped: rotating the slot roles so that each freed slot takes the
                // block the next unit needs first -- the mbarrier waits are gated by the slowest
                // warp of the CTA, not by the refill distance: 1.83 vs 1.68 ms.)
                auto release = [&](int b, const double* src) {
                    __syncwarp();
                    int old = 0;
                    if (lane == 0) {
                        __threadfence_block();
                        old = atomicAdd(&outcnt[b], 1);
                    }
                    old = __shfl_sync(0xffffffffu, old, 0);
                    if (old == NT - 1) {
                        if (lane == 0) {
                            outcnt[b] = 0;
                            if (src) {
                                fence_proxy_async_smem();
                                mbar_expect_tx(&bars[b], (uint32_t)(Pv * nbv * 16));
                            }
                        }
                        __syncwarp();
                        if (src)
                            for (int p = lane; p < Pv; p += 32)
                                bulk_g2s(shs + (size_t)b * SLOT + p * LDP, src + (int64_t)p * nbv * 2, nbv * 16, &bars[b]);
                    }
                };
                wait_slot(SJ);
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    const int dslot = MODE == 3 ? 2 + ((dm + k) & 1) : 2 + k;
                    wait_slot(dslot);
                    double acc[NT][2];
#pragma unroll
                    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
                    const double* Dk = shs + (size_t)dslot * SLOT;
#pragma unroll 2
                    for (int kk = 0; kk < NB / 4; ++kk) {
                        const double a = frag_a(shs + SJ * SLOT, kk);
#pragma unroll
                        for (int t = 0; t < NT; ++t) dmma(acc[t][0], acc[t][1], a, frag_b(Dk, kk, t));
                    }
                    if constexpr (MODE == 3) {
                        // the slot takes the Dinv block two ahead: this unit's D_{k+2}, else the next unit's
                        release(dslot, k + 2 < S ? src_dinv(cur, k + 2) : (more ? src_dinv(nxt, k + 2 - S) : nullptr));
                    } else {
                        release(2 + k, more ? src_dinv(nxt, k) : nullptr);
                    }
                    if (k == S - 1) release(SJ, more ? J + (int64_t)nxt.q * BSZ : nullptr);
                    // L_k = alpha T_k -> global (numba_backend.py:58-61) unless L is implicit;
                    // A'_k = -alpha L_k stays in the C fragments
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        acc[t][0] *= F.alpha;
                        acc[t][1] *= F.alpha;
                        if (Lout && gl_off(t) >= 0)
                            reinterpret_cast<double2*>(Lout + (int64_t)k * BSZ)[gl_off(t)] = make_double2(acc[t][0], acc[t][1]);
                        acc[t][0] *= -F.alpha;
                        acc[t][1] *= -F.alpha;
                    }
                    if (k == 0) wait_slot(SU);
                    // D_k += A'_k J_ij; A fragment (row fr, column 8 t2 + 4 h + fk) of A' sits in lane
                    // (fr, 2 h + fk / 2), register fk % 2 of C tile t2
#pragma unroll
                    for (int t2 = 0; t2 < NT; ++t2)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int srcl = (lane & ~3) | (2 * h + (fk >> 1));
                            const double x = __shfl_sync(0xffffffffu, acc[t2][0], srcl);
                            const double y = __shfl_sync(0xffffffffu, acc[t2][1], srcl);
                            const double a = (fk & 1) ? y : x;
#pragma unroll
                            for (int t = 0; t < NT; ++t)
                                dmma(dacc[k][t][0], dacc[k][t][1], a, frag_b(shs + SU * SLOT, 2 * t2 + h, t));
                        }
                    if (k == S - 1) release(SU, more ? J + (int64_t)nxt.tq * BSZ : nullptr);
                }
                dm += S;
                (void)cur;
                continue;
            }
            if constexpr (MODE == 1) {
                wait_slot(SJ);
#pragma unroll
                for (int k = 0; k < S; ++k) wait_slot(2 + k);
                double acc[S][NT][2];
#pragma unroll
                for (int k = 0; k < S; ++k)
#pragma unroll
                    for (int t = 0; t < NT; ++t) acc[k][t][0] = acc[k][t][1] = 0.0;
#pragma unroll 2
                for (int kk = 0; kk < KK; ++kk) {
                    const double a = frag_a(shs + SJ * SLOT, kk);
#pragma unroll
                    for (int k = 0; k < S; ++k)
#pragma unroll
                        for (int t = 0; t < NT; ++t)
                            dmma(acc[k][t][0], acc[k][t][1], a, frag_b(shs + (size_t)(2 + k) * SLOT, kk, t));
                }
#pragma unroll
                for (int k = 0; k < S; ++k)
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        acc[k][t][0] *= F.alpha;
                        acc[k][t][1] *= F.alpha;
                        if (Lout && gl_off(t) >= 0)
                            reinterpret_cast<double2*>(Lout + (int64_t)k * BSZ)[gl_off(t)] =
                                make_double2(acc[k][t][0], acc[k][t][1]);
                    }
                __syncthreads();   // all warps: GEMM1 done (J_ji and the Dinv slots)
                if (more) fill(SJ, J + (int64_t)nxt.q * BSZ);
#pragma unroll
                for (int k = 0; k < S; ++k) {
                    double* Ak = shs + (size_t)(2 + k) * SLOT + warp * 8 * Gm::LDA;
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        *reinterpret_cast<double2*>(Ak + fr * Gm::LDA + 8 * t + 2 * fk) =
                            make_double2(-F.alpha * acc[k][t][0], -F.alpha * acc[k][t][1]);
                }
                __syncwarp();
                wait_slot(SU);
#pragma unroll 2
                for (int kk = 0; kk < KK; ++kk) {
                    double a[S];
#pragma unroll
                    for (int k = 0; k < S; ++k)
                        a[k] = shs[(size_t)(2 + k) * SLOT + warp * 8 * Gm::LDA + fr * Gm::LDA + 4 * kk + fk];
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        const double b = frag_b(shs + SU * SLOT, kk, t);
#pragma unroll
                        for (int k = 0; k < S; ++k) dmma(dacc[k][t][0], dacc[k][t][1], a[k], b);
                    }
                }
                __syncthreads();   // all warps: GEMM2 done (A' slots, J_ij)
                if (more) {
#pragma unroll
                    for (int k = 0; k < S; ++k) fill(2 + k, src_dinv(nxt, k));
                    fill(SU, J + (int64_t)nxt.tq * BSZ);
                }
                (void)cur;
                continue;
            }
            // software-pipelined stages: phase k runs GEMM1_k (T_k = J_ji Dinv_k) interleaved with
            // GEMM2_{k-1} (D_{k-1} += A'_{k-1} J_ij), two independent accumulator sets per warp
            // between the same S + 1 barriers
            double acc[NT][2];
#pragma unroll
            for (int k = 0; k <= S; ++k) {
                const bool g1 = k < S, g2 = k > 0;
                if (k == 0) wait_slot(SJ);
                if (g1) wait_slot(2 + k);
                if (k == 1) wait_slot(SU);
#pragma unroll
                for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
                const double* Dk = shs + (size_t)(2 + (g1 ? k : 0)) * SLOT;
                const double* Ap = shs + (size_t)(2 + (g2 ? k - 1 : 0)) * SLOT + warp * 8 * Gm::LDA;
#pragma unroll 2
                for (int kk = 0; kk < NB / 4; ++kk) {
                    if (g1) {
                        const double a = frag_a(shs + SJ * SLOT, kk);
#pragma unroll
                        for (int t = 0; t < NT; ++t) dmma(acc[t][0], acc[t][1], a, frag_b(Dk, kk, t));
                    }
                    if (g2) {
                        const double a = Ap[fr * Gm::LDA + 4 * kk + fk];
#pragma unroll
                        for (int t = 0; t < NT; ++t)
                            dmma(dacc[g2 ? k - 1 : 0][t][0], dacc[g2 ? k - 1 : 0][t][1], a, frag_b(shs + SU * SLOT, kk, t));
                    }
                }
                if (g1) {
                    // L_k = alpha T_k -> global (numba_backend.py:58-61), unless L is implicit
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        acc[t][0] *= F.alpha;
                        acc[t][1] *= F.alpha;
                        if (Lout && gl_off(t) >= 0)
                            reinterpret_cast<double2*>(Lout + (int64_t)k * BSZ)[gl_off(t)] = make_double2(acc[t][0], acc[t][1]);
                    }
                }
                __syncthreads();   // all warps: GEMM1_k done (Dinv_k slot), GEMM2_{k-1} done (A'_{k-1})
                if (more && g2) fill(2 + k - 1, src_dinv(nxt, k - 1));
                if (more && k == S - 1) fill(SJ, J + (int64_t)nxt.q * BSZ);
                if (more && k == S) fill(SU, J + (int64_t)nxt.tq * BSZ);
                if (g1) {
                    // A'_k = -alpha L_k into the consumed Dinv_k slot (warp-private row-major strip)
                    double* Ak = shs + (size_t)(2 + k) * SLOT + warp * 8 * Gm::LDA;
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        *reinterpret_cast<double2*>(Ak + fr * Gm::LDA + 8 * t + 2 * fk) =
                            make_double2(-F.alpha * acc[t][0], -F.alpha * acc[t][1]);
                    __syncwarp();
                }
            }
            (void)cur;
        }
        // ---- pivot blocks -> F.Dst for the batched inverse
#pragma unroll
        for (int k = 0; k < S; ++k) {
            double2* Dk = reinterpret_cast<double2*>(F.Dst + ((int64_t)j * ST + ks + k) * BSZ);
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (gl_off(t) >= 0) Dk[gl_off(t)] = make_double2(dacc[k][t][0], dacc[k][t][1]);
        }
    }
}

template <int S, int NB, int MODE>
static int launch_schur_tt(const irk_ctx* ctx, const FactorArgs& F, const int32_t* elems, int64_t nelem,
                           cudaStream_t st, int cap_per_sm) {
    const size_t smem = sizeof(double) * (size_t)(MODE == 3 ? 4 : S + 2) * SchurGeo<NB>::SLOT;
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_schur<S, NB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        IRK_CK(cudaFuncSetAttribute(k_schur<S, NB, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr = true;
    }
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur<S, NB, MODE>, 4 * NB, smem));
    if (cap_per_sm > 0) per_sm = std::min(per_sm, cap_per_sm);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nelem, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_schur<S, NB, MODE><<<grid, 4 * NB, smem, st>>>(F, elems, nelem);
    IRK_LAUNCHED();
    return IRK_OK;
}

template <int S, int NB>
static int launch_schur_t(const irk_ctx* ctx, const FactorArgs& F, const int32_t* elems, int64_t nelem,
                          cudaStream_t st, int cap_per_sm) {
    // IRK_SCHUR_MODE (A/B knob): 0 per-stage software pipeline, S + 1 CTA barriers per unit;
    // 1 two-phase units (GEMM1 of all stages, GEMM2 of all stages: 2 barriers, more registers);
    // 2 barrier-free (A' by shuffles, last warp out of a slot refills it); 3 = 2 with two Dinv
    // slots (NB = 56, S >= 2 only)
    static const int env = getenv("IRK_SCHUR_MODE") ? atoi(getenv("IRK_SCHUR_MODE")) : -1;
    // measured: config 1 (NB 40, 3 CTAs/SM) 1.72 / - / 1.68 ms for modes 0 / 1 / 2; config 2 at N = 16
    // (NB 56): 4.86 ms for mode 1 and 5.14 ms for mode 2 (one CTA per SM), 4.46 ms for mode 3 (two)
    const int mode = env >= 0 ? env : (NB == 56 && S >= 2 ? 3 : (NB >= 56 ? 1 : 2));
    if constexpr (NB == 56 && S >= 2)
        if (mode == 3) return launch_schur_tt<S, NB, 3>(ctx, F, elems, nelem, st, cap_per_sm);
    if (mode == 1) return launch_schur_tt<S, NB, 1>(ctx, F, elems, nelem, st, cap_per_sm);
    if (mode == 0) return launch_schur_tt<S, NB, 0>(ctx, F, elems, nelem, st, cap_per_sm);
    return launch_schur_tt<S, NB, 2>(ctx, F, elems, nelem, st, cap_per_sm);
}

template <int S>
static int launch_schur_s(const irk_ctx* ctx, const FactorArgs& F, const int32_t* elems, int64_t nelem,
                          cudaStream_t st, int cap) {
    switch ((F.nb + 7) & ~7) {   // padded to the 8x8 DMMA tile
        case 16: return launch_schur_t<S, 16>(ctx, F, elems, nelem, st, cap);
        case 24: return launch_schur_t<S, 24>(ctx, F, elems, nelem, st, cap);
        case 32: return launch_schur_t<S, 32>(ctx, F, elems, nelem, st, cap);
        case 40: return launch_schur_t<S, 40>(ctx, F, elems, nelem, st, cap);
        case 48: return launch_schur_t<S, 48>(ctx, F, elems, nelem, st, cap);
        case 56: return launch_schur_t<S, 56>(ctx, F, elems, nelem, st, cap);
        case 64: return launch_schur_t<S, 64>(ctx, F, elems, nelem, st, cap);
        default: return IRK_EINVAL;
    }
}

static bool schur_eligible(const irk_factor* f, const FactorArgs& F) {
    if (getenv("IRK_NO_SCHUR")) return false;   // A/B switch for the generic kernel
    return f->kind == IRK_FACTOR_UNCOUPLED && f->simplified && f->u_shared && F.Dst != nullptr &&
           F.nb >= 12 && F.nb <= 64 && F.s <= 4;
}

static int launch_schur(const irk_ctx* ctx, const FactorArgs& F, const int32_t* elems, int64_t nelem,
                        cudaStream_t st, int cap = 0) {
    // Narrow levels (deep schedules: fewer elements than SMs) run one CTA task per (element,
    // stage) on the S = 1 instantiation: with one 5-warp CTA per element most of each SM idles and
    // the level's latency is the element's S x 2 GEMMs per unit; split, the stages run side by
    // side.  For full levels it loses (every stage re-stages the two J blocks: 1.95 vs 1.68 ms at
    // config 1, colour numbering).  IRK_SCHUR_SPLIT = 0 / 1 forces it off / on (A/B knob).
    static const int split_env = getenv("IRK_SCHUR_SPLIT") ? atoi(getenv("IRK_SCHUR_SPLIT")) : -1;
    const bool split = F.s >= 2 && (split_env >= 0 ? split_env != 0 : nelem <= (int64_t)ctx->num_sms);
    if (split) {
        FactorArgs Fs = F;
        Fs.split = 1;
        return launch_schur_s<1>(ctx, Fs, elems, nelem * F.s, st, cap);
    }
    switch (F.s) {
        case 1: return launch_schur_s<1>(ctx, F, elems, nelem, st, cap);
        case 2: return launch_schur_s<2>(ctx, F, elems, nelem, st, cap);
        case 3: return launch_schur_s<3>(ctx, F, elems, nelem, st, cap);
        case 4: return launch_schur_s<4>(ctx, F, elems, nelem, st, cap);
        default: return IRK_EINVAL;
    }
}

int launch_inverse(const irk_ctx* ctx, const int32_t* tasks, int64_t ntasks, int64_t T, int s, int nb,
                   const double* D, double* Dinv, unsigned long long* fail_key, int* fb, cudaStream_t st,
                   int cap_per_sm = 0, const InvForm* form = nullptr, bool optimistic = false);

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <int MAXT>
static int launch_levels(const irk_factor* f, FactorArgs& F, const irk_sched& sched, size_t smem,
                         cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        IRK_CK(cudaFuncSetAttribute(k_factor<MAXT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)f->ctx->smem_optin));
        IRK_CK(cudaFuncSetAttribute(k_factor<MAXT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)f->ctx->smem_optin));
        attr_set = true;
    }
    // batched warp inversion when nb has a specialisation (nb <= 64)
    const bool split = F.nb <= 64 && F.Dst != nullptr;
    for (int64_t l = 0; l < sched.nlevels; ++l) {
        const int64_t lo = sched.h_lvl_ptr[l], hi = sched.h_lvl_ptr[l + 1];
        if (hi == lo) continue;
        F.tasks = sched.d_order + lo;
        F.ntasks = hi - lo;
        const int grid = (int)std::min<int64_t>(hi - lo, (int64_t)f->ctx->num_sms * 8);
        if (split && schur_eligible(f, F) && f->d_fs_elems) {
            // the level's elements and their (element-major) stage tasks
            const int64_t e0 = f->h_fs_eptr[l], ne = f->h_fs_eptr[l + 1] - e0;
            const int32_t* el = f->d_fs_elems + e0;
            const int32_t* tk = f->d_fs_tasks + e0 * F.s;
            static const int nchunk = env_int("IRK_FACTOR_CHUNKS", 1);   // measured: no gain at config 1
            static const int schur_cap = env_int("IRK_SCHUR_CAP", 2);
            static const int inv_cap = env_int("IRK_INV_CAP", 1);
            // forming D inside the inverse needs the tensor-core inverse kernels
            static const bool form_off = env_int("IRK_FORM_D", 1) == 0 || env_int("IRK_INV_TC", 1) == 0;
            if (l == 0 && F.L == nullptr && !F.literal && F.nb > 16 && F.nb <= 64 && f->d_fb && !form_off) {
                // level 0 has no Schur update: the inverse kernel forms D = alpha J_jj + coef_k M_j itself
                InvForm fm;
                fm.J = F.J[0];
                fm.diag = F.diag;
                fm.keep = F.keep;
                fm.M = F.M;
                fm.Dst = F.Dst;
                fm.alpha = F.alpha;
                for (int k = 0; k < F.s; ++k) fm.coef[k] = F.coef[k];
                fm.store = f->store_d ? 1 : 0;
                IRK_TRY(launch_inverse(f->ctx, tk, ne * F.s, F.T, F.s, F.nb, F.Dst, F.Dinv, F.fail_key, f->d_fb, st,
                                       0, &fm, f->fb_optimistic != 0));
                f->d0_unstored = !f->store_d;
            } else if (l == 0 || nchunk <= 1 || ne < 4 * (int64_t)f->ctx->num_sms) {
                if (l == 0) f->d0_unstored = false;
                IRK_TRY(launch_schur(f->ctx, F, el, ne, st));
                IRK_TRY(launch_inverse(f->ctx, tk, ne * F.s, F.T, F.s, F.nb, F.Dst, F.Dinv, F.fail_key, f->d_fb, st,
                                       0, nullptr, f->fb_optimistic != 0));
            } else {
                // chunked: the latency-bound inverse of chunk c (side stream, capped grid) runs beside
                // the DMMA-bound Schur phase of chunk c+1 (main stream, capped at schur_cap CTAs/SM)
                if (!f->st2) {
                    IRK_CK(cudaStreamCreateWithFlags(&f->st2, cudaStreamNonBlocking));
                    f->ev.resize(nchunk + 1);
                    for (auto& e : f->ev) IRK_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                }
                for (int c = 0; c < nchunk; ++c) {
                    const int64_t a = ne * c / nchunk, b = ne * (c + 1) / nchunk;
                    if (b == a) continue;
                    IRK_TRY(launch_schur(f->ctx, F, el + a, b - a, st, schur_cap));
                    IRK_CK(cudaEventRecord(f->ev[c], st));
                    IRK_CK(cudaStreamWaitEvent(f->st2, f->ev[c], 0));
                    IRK_TRY(launch_inverse(f->ctx, tk + a * F.s, (b - a) * F.s, F.T, F.s, F.nb, F.Dst, F.Dinv,
                                           F.fail_key, f->d_fb, f->st2, inv_cap));
                }
                IRK_CK(cudaEventRecord(f->ev[nchunk], f->st2));
                IRK_CK(cudaStreamWaitEvent(st, f->ev[nchunk], 0));
            }
        } else if (split) {
            k_factor<MAXT, false><<<grid, 256, smem, st>>>(F);
            IRK_LAUNCHED();
            IRK_TRY(launch_inverse(f->ctx, F.tasks, F.ntasks, F.T, F.s, F.nb, F.Dst, F.Dinv, F.fail_key, f->d_fb, st,
                                   0, nullptr, f->fb_optimistic != 0));
        } else {
            k_factor<MAXT, true><<<grid, 256, smem, st>>>(F);
            IRK_LAUNCHED();
        }
    }
    return IRK_OK;
}

struct FactorSetup {
    int s;
    const irk_blocks* const* J;
    const int64_t* jfirst;
    const irk_blocks* M;
    const double* coef;     // uncoupled diag coefficients
    const double* a_inv;    // coupled mixing
    double alpha;
    const irk_blocks* coupling;
    const uint8_t* keep;
    int simplified, literal, store_diag, coupled;
};

// numeric values of a factorisation: operator sources and scalars (the
// structure -- pattern, keep, schedules, buffers -- is fixed at creation)
static int set_sources(irk_factor* f, const FactorSetup& P) {
    const irk_pattern* pat = f->pat;
    const int nb = f->nb;
    IRK_ARG(P.s == f->s, "stage count differs from the factor's");
    for (int k = 0; k < P.s; ++k) {
        IRK_ARG(P.J[k] && P.J[k]->nb == nb, "J blocks missing or nb mismatch");
        const int64_t jf = P.jfirst ? P.jfirst[k] : 0;
        IRK_ARG(jf >= 0 && jf + pat->nnzb <= P.J[k]->count, "J block range out of bounds");
    }
    IRK_ARG(!P.M || (P.M->nb == nb && P.M->count >= pat->T), "mass blocks mismatch");
    IRK_ARG(!P.coupling || (P.coupling->nb == nb && P.coupling->count >= (int64_t)P.s * P.s * pat->T),
            "coupling blocks mismatch");
    IRK_ARG(f->kind != IRK_FACTOR_COUPLED || P.M || P.coupling, "coupled factor needs M or explicit couplings");
    IRK_ARG(f->kind != IRK_FACTOR_COUPLED || f->s < 2 || (f->d_Cup != nullptr) == (P.coupling != nullptr),
            "explicit/implicit coupling mode differs from the factor's");
    const int64_t bsz = block_doubles(nb);
    FactorArgs& F = *static_cast<FactorArgs*>(f->fargs);
    bool shared = true;
    for (int k = 0; k < P.s; ++k) {
        f->ubase[k] = P.J[k]->d + (P.jfirst ? P.jfirst[k] : 0) * bsz;
        if (f->ubase[k] != f->ubase[0]) shared = false;
        F.J[k] = f->ubase[k];
    }
    f->u_shared = shared && !f->u_stored;
    f->uscale = f->u_stored ? 1.0 : P.alpha;
    F.M = P.M ? P.M->d : nullptr;
    F.Cexp = P.coupling ? P.coupling->d : nullptr;
    f->cpl_src = P.coupling ? P.coupling->d : nullptr;
    F.alpha = P.alpha;
    for (int k = 0; k < P.s; ++k)
        F.coef[k] = f->kind == IRK_FACTOR_COUPLED ? (P.a_inv ? P.a_inv[k * P.s + k] : 0.0)
                                                  : (P.coef ? P.coef[k] : 0.0);
    if (P.a_inv)
        for (int e = 0; e < P.s * P.s; ++e) F.cmix[e] = P.a_inv[e];
    if (f->kind == IRK_FACTOR_COUPLED && !P.coupling) {
        f->mass = P.M->d;
        for (int e = 0; e < P.s * P.s; ++e) f->cup_scale[e] = P.a_inv[e];
    }
    return IRK_OK;
}

struct FactorGraph {
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cap = nullptr;     // capture stream (the caller's may be the legacy default stream)
    FactorArgs key;                 // kernel arguments the graph was captured with
    long long launches = 0;         // kernel launches per replay (irk_launch_count)
    int calls = 0;
};

long long launch_count_now();          // common.cu
void count_launches(long long n);

static int factor_numeric(irk_factor* f, int64_t* fail_stage, int64_t* fail_elem, cudaStream_t st) {
    FactorArgs& F = *static_cast<FactorArgs*>(f->fargs);
    const irk_pattern* pat = f->pat;
    const int64_t bsz = block_doubles(f->nb);
    const int npairs = f->s * (f->s - 1) / 2;
    IRK_CK(cudaMemsetAsync(f->d_fail, 0xff, sizeof(unsigned long long), st));
    F.fail_key = f->d_fail;
    if (f->cpl_src && npairs > 0) {
        // explicit upper couplings C[k][l] (k<l) -> Cup[i][pair(l,k)], used unmodified by the apply
        for (int l = 1; l < f->s; ++l)
            for (int k = 0; k < l; ++k)
                IRK_CK(cudaMemcpy2DAsync(f->d_Cup + (int64_t)(l * (l - 1) / 2 + k) * bsz, sizeof(double) * bsz * npairs,
                                         f->cpl_src + ((int64_t)k * f->s + l) * pat->T * bsz, sizeof(double) * bsz,
                                         sizeof(double) * bsz, pat->T, cudaMemcpyDeviceToDevice, st));
    }
    if (f->u_stored) {
        k_init_upper<<<(int)std::min<int64_t>(pat->T, f->ctx->num_sms * 8), 256, 0, st>>>(F, pat->T);
        IRK_LAUNCHED();
    }
    int rc = IRK_OK;
    auto run_levels = [&](cudaStream_t s2) -> int {
        switch (f->maxt) {
            case 2: return launch_levels<2>(f, F, f->fsched, f->fsmem, s2);
            case 4: return launch_levels<4>(f, F, f->fsched, f->fsmem, s2);
            case 8: return launch_levels<8>(f, F, f->fsched, f->fsmem, s2);
            case 16: return launch_levels<16>(f, F, f->fsched, f->fsmem, s2);
            case 32: return launch_levels<32>(f, F, f->fsched, f->fsmem, s2);
            default: set_error("block size too large"); return IRK_EINVAL;
        }
    };
    // Deep schedules (natural numbering: 258 levels at config 1, 3-4 stream operations each) are
    // launch-bound: ~48 us per level for ~22 us of kernels.  The level loop is captured into a CUDA
    // graph on the second call (the first one sets the kernels' attributes) and replayed as long
    // as the kernel arguments are byte-identical (same buffers, coefficients and schedule: one
    // Newton iteration after the other); anything else re-captures.  Opt-in (IRK_FACTOR_GRAPH=1):
    // capturing and instantiating the ~1000-node graph costs tens of milliseconds once and a replay
    // saves 1 ms of 12.6 (config 1, natural numbering), so it pays off after a few dozen
    // re-factorisations of one structure only.
    static const bool graph_off = !(getenv("IRK_FACTOR_GRAPH") && atoi(getenv("IRK_FACTOR_GRAPH")) != 0);
    const bool deep = f->fsched.nlevels > 16 && !graph_off && f->kind == IRK_FACTOR_UNCOUPLED;
    if (deep) {
        if (!f->fgraph) f->fgraph = new FactorGraph();
        FactorGraph* g = static_cast<FactorGraph*>(f->fgraph);
        if (g->exec && std::memcmp(&g->key, &F, sizeof(FactorArgs)) == 0) {
            IRK_CK(cudaGraphLaunch(g->exec, st));
            count_launches(g->launches);
        } else if (g->calls++ == 0) {
            rc = run_levels(st);
        } else {
            if (g->exec) { cudaGraphExecDestroy(g->exec); g->exec = nullptr; }
            if (!g->cap) IRK_CK(cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking));
            const long long before = launch_count_now();
            IRK_CK(cudaStreamBeginCapture(g->cap, cudaStreamCaptureModeRelaxed));
            rc = run_levels(g->cap);
            cudaGraph_t graph = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(g->cap, &graph);
            g->launches = launch_count_now() - before;
            if (rc == IRK_OK && ce == cudaSuccess && graph) {
                if (cudaGraphInstantiate(&g->exec, graph, 0) == cudaSuccess) {
                    std::memcpy(&g->key, &F, sizeof(FactorArgs));
                    IRK_CK(cudaGraphLaunch(g->exec, st));
                } else {
                    g->exec = nullptr;
                }
            }
            if (graph) cudaGraphDestroy(graph);
            if (!g->exec) {   // capture not possible here: plain launches
                cudaGetLastError();
                rc = run_levels(st);
            }
        }
    } else {
        // Deep schedules pay two stream operations per level for the pivoted fallback (counter
        // reset + a launch that almost always finds an empty list): run the levels optimistically
        // -- one counter reset, no fallback launches, handed-back blocks pile up in the list -- and
        // repeat the factorisation the regular way if any block was handed back.
        static const bool opt_off = getenv("IRK_FB_OPTIMISTIC") && atoi(getenv("IRK_FB_OPTIMISTIC")) == 0;
        // (every path that batches its pivot inverses through launch_inverse: the DMMA Schur path and
        // the generic kernel's split form, which the coupled factor uses)
        const bool optimistic = f->fsched.nlevels > 16 && !opt_off && f->d_fb && F.nb > 16 && F.nb <= 64 &&
                                F.Dst != nullptr;
        if (optimistic) {
            IRK_CK(cudaMemsetAsync(f->d_fb, 0, sizeof(int), st));
            f->fb_optimistic = 1;
            rc = run_levels(st);
            f->fb_optimistic = 0;
            if (rc) return rc;
            int handed = 0;
            IRK_CK(cudaMemcpyAsync(&handed, f->d_fb, sizeof handed, cudaMemcpyDeviceToHost, st));
            IRK_CK(cudaStreamSynchronize(st));
            if (handed > 0) {
                IRK_CK(cudaMemsetAsync(f->d_fail, 0xff, sizeof(unsigned long long), st));
                rc = run_levels(st);
            }
        } else {
            rc = run_levels(st);
        }
    }
    if (rc) return rc;
    unsigned long long key = 0;
    IRK_CK(cudaMemcpyAsync(&key, f->d_fail, sizeof key, cudaMemcpyDeviceToHost, st));
    IRK_CK(cudaStreamSynchronize(st));
    if (fail_stage) *fail_stage = -1;
    if (fail_elem) *fail_elem = -1;
    if (key != ~0ULL) {
        if (fail_stage) *fail_stage = (int64_t)(key / pat->T);
        if (fail_elem) *fail_elem = (int64_t)(key % pat->T);
        set_error("numerically singular pivot block");
        return IRK_ESINGULAR;
    }
    return IRK_OK;
}


// Implicit L (never store L_ij = alpha J_ij Dinv_j) needs: stage-uncoupled
// simplified ILU, one J shared by all stages, a symmetric keep mask (so every
// kept lower block is a Schur pair), and the pipelined sweep kernels (even nb,
// s <= 4, G nb <= 256).  IRK_EXPLICIT_L=1 forces stored L (A/B comparisons).
static bool implicit_l_ok(const irk_pattern* pat, const FactorSetup& P, const std::vector<uint8_t>& keep,
                          int simplified) {
    if (P.coupled || !simplified || P.literal || getenv("IRK_EXPLICIT_L")) return false;
    const int nb = P.J[0]->nb;
    if (nb % 2 || P.s > 4 || choose_groups(nb, 256) * nb > 256) return false;
    const int64_t bsz = block_doubles(nb);
    const double* b0 = P.J[0]->d + (P.jfirst ? P.jfirst[0] : 0) * bsz;
    for (int k = 1; k < P.s; ++k)
        if (P.J[k]->d + (P.jfirst ? P.jfirst[k] : 0) * bsz != b0) return false;
    for (int64_t i = 0; i < pat->T; ++i)
        for (int64_t q = pat->h_indptr[i]; q < pat->h_indptr[i + 1]; ++q) {
            const int64_t j = pat->h_indices[q];
            const int64_t* b = pat->h_indices.data() + pat->h_indptr[j];
            const int64_t* e = pat->h_indices.data() + pat->h_indptr[j + 1];
            const int64_t* t = std::lower_bound(b, e, i);
            const bool kt = (t != e && *t == i) && keep[pat->h_indptr[j] + (t - b)];
            if (q != pat->h_diag[i] && (keep[q] != 0) != kt) return false;
        }
    return true;
}

static int factor_common(irk_ctx* ctx, const irk_pattern* pat, const FactorSetup& P, irk_factor** out,
                         int64_t* fail_stage, int64_t* fail_elem, cudaStream_t st) {
    IRK_ARG(ctx && pat && P.J && P.J[0] && out, "NULL argument");
    IRK_ARG(P.s >= 1 && P.s <= IRK_MAX_STAGES, "stage count out of range");
    IRK_ARG((int64_t)P.s * pat->T < INT_MAX, "s*T too large");
    const int nb = P.J[0]->nb;
    auto* f = new irk_factor();
    f->ctx = ctx;
    f->pat = pat;
    f->kind = P.coupled ? IRK_FACTOR_COUPLED : IRK_FACTOR_UNCOUPLED;
    f->s = P.s;
    f->nb = nb;
    f->simplified = P.coupled ? 1 : P.simplified;
    f->literal = P.literal;
    f->fargs = new FactorArgs{};
    std::vector<uint8_t> keep(pat->nnzb, 1);
    if (P.keep) std::memcpy(keep.data(), P.keep, pat->nnzb);
    const int64_t bsz = block_doubles(nb);
    int rc = IRK_OK;
    auto fail = [&](int code) { irk_factor_destroy(f); return code; };
#define FCK(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) return fail(fail_cuda(_e, #call, __FILE__, __LINE__)); } while (0)
    f->u_stored = !f->simplified;
    f->store_d = P.store_diag || P.literal;
    const int npairs = P.s * (P.s - 1) / 2;
    f->l_implicit = implicit_l_ok(pat, P, keep, f->simplified);
    FCK(cudaMalloc(&f->d_keep, pat->nnzb));
    FCK(cudaMemcpy(f->d_keep, keep.data(), pat->nnzb, cudaMemcpyHostToDevice));
    if (f->l_implicit) FCK(cudaMalloc(&f->d_W, sizeof(double) * bsz / nb * pat->T * P.s));   // s x T x nb
    else FCK(cudaMalloc(&f->d_L, sizeof(double) * bsz * std::max<int64_t>(pat->nlow * P.s, 1)));
    FCK(cudaMalloc(&f->d_Dinv, sizeof(double) * bsz * pat->T * P.s));
    // pivot blocks: needed for export/literal, and as the hand-off to the batched inverse
    if (P.store_diag || P.literal || nb <= 64) FCK(cudaMalloc(&f->d_D, sizeof(double) * bsz * pat->T * P.s));
    if (f->u_stored) FCK(cudaMalloc(&f->d_U, sizeof(double) * bsz * std::max<int64_t>(pat->nup * P.s, 1)));
    if (P.coupled && npairs > 0) FCK(cudaMalloc(&f->d_G, sizeof(double) * bsz * pat->T * npairs));
    if (P.coupled && P.coupling && npairs > 0) FCK(cudaMalloc(&f->d_Cup, sizeof(double) * bsz * pat->T * npairs));
    FCK(cudaMalloc(&f->d_fail, sizeof(unsigned long long)));
    // tensor-core inverse fallback list: [count | task codes]
    if (nb > 16 && nb <= 64) FCK(cudaMalloc(&f->d_fb, sizeof(int) * ((int64_t)P.s * pat->T + 1)));
    if ((rc = set_sources(f, P))) return fail(rc);
    std::vector<int64_t> levf;
    if ((rc = build_apply_schedules(f, keep))) return fail(rc);
    levels_forward(pat, keep, levf);
    // factor tasks: (stage, element) per level
    if ((rc = build_sched(f->fsched, levf, pat->T, P.s, true, P.coupled ? +1 : 0))) return fail(rc);
    if (!P.coupled) {
        // per-level element lists and element-major task codes for the Schur path
        const int64_t nl = f->fsched.nlevels;
        std::vector<int64_t> cnt(nl + 1, 0);
        for (int64_t e = 0; e < pat->T; ++e) cnt[levf[e] + 1]++;
        for (int64_t l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
        std::vector<int32_t> elems(pat->T), tasks((size_t)pat->T * P.s);
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t e = 0; e < pat->T; ++e) elems[pos[levf[e]]++] = (int32_t)e;
        for (int64_t q = 0; q < pat->T; ++q)
            for (int k = 0; k < P.s; ++k) tasks[q * P.s + k] = (int32_t)((int64_t)k * pat->T + elems[q]);
        f->h_fs_eptr = cnt;
        FCK(cudaMalloc(&f->d_fs_elems, sizeof(int32_t) * std::max<int64_t>(pat->T, 1)));
        FCK(cudaMalloc(&f->d_fs_tasks, sizeof(int32_t) * std::max<int64_t>(pat->T * P.s, 1)));
        FCK(cudaMemcpy(f->d_fs_elems, elems.data(), sizeof(int32_t) * pat->T, cudaMemcpyHostToDevice));
        FCK(cudaMemcpy(f->d_fs_tasks, tasks.data(), sizeof(int32_t) * pat->T * P.s, cudaMemcpyHostToDevice));
    }

    FactorArgs& F = *static_cast<FactorArgs*>(f->fargs);
    F.indptr = pat->d_indptr;
    F.indices = pat->d_indices;
    F.diag = pat->d_diag;
    F.lptr = pat->d_lptr;
    F.uptr = pat->d_uptr;
    F.tpos = pat->d_tpos;
    F.keep = f->d_keep;
    F.L = f->d_L;
    F.Dinv = f->d_Dinv;
    F.Dst = f->d_D;
    F.U = f->d_U;
    F.G = f->d_G;
    F.T = pat->T;
    F.s = P.s;
    F.nb = nb;
    F.nbp4 = (nb + 7) & ~7;                        // padded to the 8x8 DMMA tile
    F.ld = F.nbp4 + ((F.nbp4 % 16 == 0) ? 8 : 0);  // ld = 8 (mod 16): conflict-free fragments
    F.coupled = P.coupled;
    F.literal = P.literal;
    F.simplified = f->simplified;
    // shared memory budget: full D and L^T, K-chunked operand tiles
    F.KC = F.nbp4;
    while (factor_smem(F.nbp4, F.ld, F.KC) > ctx->smem_optin && F.KC > 8) F.KC = std::max(8, ((F.KC / 2) + 7) & ~7);
    f->fsmem = factor_smem(F.nbp4, F.ld, F.KC);
    if (f->fsmem > ctx->smem_optin) { set_error("block size too large for shared memory"); return fail(IRK_EINVAL); }
    const int tpr = F.nbp4 / 8;
    const int tiles_per_warp = (tpr * tpr + 7) / 8;
    f->maxt = tiles_per_warp <= 2 ? 2 : tiles_per_warp <= 4 ? 4 : tiles_per_warp <= 8 ? 8 : tiles_per_warp <= 16 ? 16 : 32;
#undef FCK
    rc = factor_numeric(f, fail_stage, fail_elem, st);
    if (rc < 0) return fail(rc);
    *out = f;
    return rc;
}

// Export of a factor whose level-0 pivot blocks were formed inside the inverse and
// not stored: re-form them (cold path), with the rounding of the Schur phase.
__global__ void k_form_d(FactorArgs F, const int32_t* tasks, int64_t ntasks) {
    const int nb = F.nb;
    const int64_t bsz = (int64_t)nb * 2 * ((nb + 1) >> 1);
    for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int64_t code = tasks[t];
        const int k = (int)(code / F.T);
        const int64_t j = code - (int64_t)k * F.T;
        const int dpos = F.diag[j];
        const bool keep_d = F.keep[dpos] != 0;
        double* dst = F.Dst + (j * F.s + k) * bsz;
        for (int64_t e = threadIdx.x; e < bsz; e += blockDim.x) {
            double x = __dmul_rn(F.alpha, F.J[0][(int64_t)dpos * bsz + e]);
            if (F.M) x = __dadd_rn(x, __dmul_rn(F.coef[k], F.M[j * bsz + e]));
            dst[e] = keep_d ? x : 0.0;
        }
    }
}

int factor_form_level0_d(const irk_factor* f, cudaStream_t st) {
    if (!f->d0_unstored || !f->d_fs_tasks || f->h_fs_eptr.size() < 2) return IRK_OK;
    const FactorArgs& F = *static_cast<const FactorArgs*>(f->fargs);
    const int64_t n = (f->h_fs_eptr[1] - f->h_fs_eptr[0]) * f->s;
    if (n <= 0) return IRK_OK;
    k_form_d<<<(int)std::min<int64_t>(n, (int64_t)f->ctx->num_sms * 8), 256, 0, st>>>(F, f->d_fs_tasks, n);
    IRK_LAUNCHED();
    f->d0_unstored = false;
    return IRK_OK;
}

// Implicit L, for export: L[lq][k] = alpha J_q Dinv_{j,k} (j = column of q) for
// kept lower blocks, 0 for dropped ones.  Cold path: one CTA per row, plain FMAs.
__global__ void k_materialize_L(FactorArgs F, double* out) {
    extern __shared__ double sm[];
    const int nb = F.nb;
    const int64_t bsz = (int64_t)nb * 2 * ((nb + 1) >> 1);
    double* Ja = sm;                 // nb x nb row-major
    double* Db = sm + nb * nb;
    for (int64_t i = blockIdx.x; i < F.T; i += gridDim.x) {
        const int q0 = F.indptr[i], d = F.diag[i], lq0 = F.lptr[i];
        for (int q = q0; q < d; ++q) {
            const int j = F.indices[q];
            for (int k = 0; k < F.s; ++k) {
                double* dst = out + ((int64_t)(lq0 + q - q0) * F.s + k) * bsz;
                if (!F.keep[q]) {
                    for (int e = threadIdx.x; e < bsz; e += blockDim.x) dst[e] = 0.0;
                    continue;
                }
                const double* Jq = F.J[0] + (int64_t)q * bsz;
                const double* Dk = F.Dinv + ((int64_t)j * F.s + k) * bsz;
                for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
                    const int a = e / nb, b = e - a * nb;
                    Ja[e] = Jq[lay(a, b, nb)];
                    Db[e] = Dk[lay(a, b, nb)];
                }
                __syncthreads();
                for (int e = threadIdx.x; e < bsz; e += blockDim.x) {
                    const int p = (int)(e >> 1) / nb, a = (int)(e >> 1) % nb, b = 2 * p + (int)(e & 1);
                    double acc = 0.0;
                    if (b < nb)
                        for (int c = 0; c < nb; ++c) acc = fma(Ja[a * nb + c], Db[c * nb + b], acc);
                    dst[e] = F.alpha * acc;
                }
                __syncthreads();
            }
        }
    }
}

int factor_materialize_L(const irk_factor* f, double** out, cudaStream_t st) {
    const FactorArgs& F = *static_cast<const FactorArgs*>(f->fargs);
    const int64_t bsz = block_doubles(f->nb);
    IRK_CK(cudaMallocAsync(out, sizeof(double) * bsz * std::max<int64_t>(f->pat->nlow * f->s, 1), st));
    const size_t smem = sizeof(double) * 2 * f->nb * f->nb;
    IRK_CK(cudaFuncSetAttribute(k_materialize_L, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_materialize_L<<<(int)std::min<int64_t>(f->pat->T, f->ctx->num_sms * 4), 256, smem, st>>>(F, *out);
    IRK_LAUNCHED();
    return IRK_OK;
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_factor_uncoupled(irk_ctx* ctx, const irk_pattern* pat, int s, const irk_blocks* const* J,
                         const int64_t* jfirst, const irk_blocks* M, const double* coef, double alpha,
                         const uint8_t* keep, int simplified, int store_diag, irk_factor** out,
                         int64_t* fail_stage, int64_t* fail_elem, void* stream) {
    IRK_ARG(!M || coef, "coef required with M");
    FactorSetup P{};
    P.s = s;
    P.J = J;
    P.jfirst = jfirst;
    P.M = M;
    P.coef = coef;
    P.alpha = alpha;
    P.keep = keep;
    P.simplified = simplified;
    P.store_diag = store_diag;
    P.coupled = 0;
    return factor_common(ctx, pat, P, out, fail_stage, fail_elem, (cudaStream_t)stream);
}

int irk_factor_coupled(irk_ctx* ctx, const irk_pattern* pat, int s, const irk_blocks* const* J,
                       const int64_t* jfirst, const irk_blocks* M, const double* a_inv, double alpha,
                       const irk_blocks* coupling, const uint8_t* keep, int literal, int store_diag,
                       irk_factor** out, int64_t* fail_stage, int64_t* fail_elem, void* stream) {
    IRK_ARG(a_inv || coupling, "a_inv or coupling required");
    IRK_ARG(!M || a_inv, "a_inv required with M");
    FactorSetup P{};
    P.s = s;
    P.J = J;
    P.jfirst = jfirst;
    P.M = M;
    P.a_inv = a_inv;
    P.alpha = alpha;
    P.coupling = coupling;
    P.keep = keep;
    P.simplified = 1;
    P.literal = literal;
    P.store_diag = store_diag;
    P.coupled = 1;
    return factor_common(ctx, pat, P, out, fail_stage, fail_elem, (cudaStream_t)stream);
}

int irk_factor_refactor(irk_factor* f, const irk_blocks* const* J, const int64_t* jfirst, const irk_blocks* M,
                        const double* coef, double alpha, const irk_blocks* coupling, int64_t* fail_stage,
                        int64_t* fail_elem, void* stream) {
    IRK_ARG(f && J, "NULL argument");
    IRK_ARG(f->kind == IRK_FACTOR_COUPLED || !M || coef, "coef required with M");
    FactorSetup P{};
    P.s = f->s;
    P.J = J;
    P.jfirst = jfirst;
    P.M = M;
    if (f->kind == IRK_FACTOR_COUPLED) P.a_inv = coef;
    else P.coef = coef;
    P.alpha = alpha;
    P.coupling = coupling;
    IRK_TRY(set_sources(f, P));
    IRK_ARG(!f->l_implicit || f->u_shared, "implicit-L factor: refactor needs one J shared by all stages");
    ++f->numeric_epoch;
    return factor_numeric(f, fail_stage, fail_elem, (cudaStream_t)stream);
}

void irk_factor_destroy(irk_factor* f) {
    if (!f) return;
    cudaFree(f->d_keep);
    cudaFree(f->d_L);
    cudaFree(f->d_W);
    cudaFree(f->d_Z);
    cudaFree(f->d_Wrhs);
    cudaFree(f->d_fb);
    cudaFree(f->d_fs_elems);
    cudaFree(f->d_fs_tasks);
    for (auto e : f->ev) cudaEventDestroy(e);
    if (f->st2) cudaStreamDestroy(f->st2);
    if (f->fgraph) {
        FactorGraph* g = static_cast<FactorGraph*>(f->fgraph);
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->cap) cudaStreamDestroy(g->cap);
        delete g;
    }
    cudaFree(f->d_hasup);
    cudaFree(f->d_Dinv);
    cudaFree(f->d_D);
    cudaFree(f->d_U);
    cudaFree(f->d_G);
    cudaFree(f->d_Cup);
    cudaFree(f->fwd.d_order);
    cudaFree(f->bwd.d_order);
    cudaFree(f->d_flags);
    cudaFree(f->d_ticket);
    cudaFree(f->d_fail);
    cudaFree(f->fsched.d_order);
    delete static_cast<FactorArgs*>(f->fargs);
    for (auto* b : f->owned) irk_blocks_destroy(b);
    delete f;
}

int irk_factor_levels(const irk_factor* f, int64_t* fwd_levels, int64_t* bwd_levels) {
    IRK_ARG(f, "NULL factor");
    if (fwd_levels) *fwd_levels = f->fwd.nlevels;
    if (bwd_levels) *bwd_levels = f->bwd.nlevels;
    return IRK_OK;
}

int irk_factor_implicit_l(const irk_factor* f) {
    IRK_ARG(f, "NULL factor");
    return f->l_implicit ? 1 : 0;
}

}  // extern "C"
