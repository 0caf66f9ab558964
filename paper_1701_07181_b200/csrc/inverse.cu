// Batched inversion of the ILU(0) pivot blocks: one warp per nb x nb block.
//
// Reference: _inv_with_cond (numba_backend.py:33-40) -- np.linalg.det via
// slogdet of the partial-pivoting LU, np.linalg.inv, 1-norm condition
// estimate cond = |D|_1 |D^-1|_1, failure when det == 0 / non-finite or
// cond > 1e14 (numba_backend.py:53-55).
//
// Gauss-Jordan with partial pivoting and *implicit* row interchanges: lane l
// keeps rows l and l+32 of the block in registers; at step k the warp finds
// the unused row p with the largest |D[p][k]| (first such row on ties -- the
// pivot sequence getrf would produce), broadcasts row p through shared
// memory and eliminates column k from every other row.  With the pivot rows
// p_0..p_{n-1} the result X satisfies inv(D)[k][p_m] = X[p_k][m]; the
// permutation is applied when the rows are staged through shared memory for
// the coalesced store.  det = exp(sum log|pivot|) as in slogdet.
#include <cuda_runtime.h>

#include <algorithm>

#include "irk_internal.cuh"

namespace irk {

struct InvArgs {
    const int32_t* tasks;     // task codes k*T + j
    int64_t ntasks;
    int64_t T;
    int s, nb;
    const double* D;          // pivot blocks D[j][k] (device layout)
    double* Dinv;             // inverses Dinv[j][k]
    unsigned long long* fail_key;
};

// EXACT: nb == NBT -- the pivot loop is fully unrolled, so every register
// index (column k, pivot column extraction) is a compile-time constant.
template <int NBT, bool EXACT>
__global__ void __launch_bounds__(128) k_inverse(InvArgs A) {
    constexpr int ROWS = (NBT + 31) / 32;
    constexpr int LDX = NBT + 1;
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    double* Xs = sm + (size_t)warp * (NBT * LDX + NBT);
    double* prow = Xs + NBT * LDX;                 // pivot row broadcast buffer
    int* ibuf = reinterpret_cast<int*>(sm + (size_t)wpb * (NBT * LDX + NBT)) + warp * 2 * NBT;
    int* piv = ibuf;                                // pivot row of each step
    int* invp = ibuf + NBT;                         // inverse permutation
    const int nb = EXACT ? NBT : A.nb;
    const int P = (nb + 1) >> 1;
    const int64_t bsz = (int64_t)nb * 2 * P;

    for (int64_t t = (int64_t)blockIdx.x * wpb + warp; t < A.ntasks; t += (int64_t)gridDim.x * wpb) {
        const int64_t code = A.tasks[t];
        const int k_st = (int)(code / A.T);
        const int64_t j = code - (int64_t)k_st * A.T;
        const double* src = A.D + (j * A.s + k_st) * bsz;
        double d[ROWS][NBT];
        // ---- load rows (coalesced: consecutive lanes = consecutive rows of a pair)
#pragma unroll
        for (int s = 0; s < ROWS; ++s) {
            const int r = lane + 32 * s;
#pragma unroll
            for (int p = 0; p < (NBT + 1) / 2; ++p) {
                double2 v = make_double2(0.0, 0.0);
                if (r < nb && p < P) v = reinterpret_cast<const double2*>(src)[(int64_t)p * nb + r];
                d[s][2 * p] = v.x;
                if (2 * p + 1 < NBT) d[s][2 * p + 1] = v.y;
            }
        }
        // ---- |D|_1 (max column abs sum, NaN propagating) through shared memory
        auto col_norm = [&]() -> double {
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const int r = lane + 32 * s;
                if (r < nb)
#pragma unroll
                    for (int c = 0; c < NBT; ++c) Xs[r * LDX + c] = fabs(d[s][c]);
            }
            __syncwarp();
            double mx = -1.0;
            int nan = 0;
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const int c = lane + 32 * s;
                if (c < nb) {
                    double sum = 0.0;
                    for (int r = 0; r < nb; ++r) sum += Xs[r * LDX + c];
                    if (sum != sum) nan = 1;
                    mx = fmax(mx, sum);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            }
            __syncwarp();
            return nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
        };
        const double n1 = col_norm();
        // ---- Gauss-Jordan, implicit pivoting
        int used[ROWS];
        int pstep[ROWS];
#pragma unroll
        for (int s = 0; s < ROWS; ++s) { used[s] = (lane + 32 * s) >= nb; pstep[s] = -1; }
        double logdet = 0.0;
        int zero = 0;
#pragma unroll(EXACT ? NBT : 1)
        for (int k = 0; k < nb; ++k) {
            // own entries of column k
            double ck[ROWS];
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                double v = 0.0;
#pragma unroll
                for (int c = 0; c < NBT; ++c) v = (c == k) ? d[s][c] : v;
                ck[s] = v;
            }
            // pivot: max |D[r][k]| over unused rows, smallest r on ties
            double best = -1.0;
            int br = 0x7fffffff;
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const double a = used[s] ? -1.0 : fabs(ck[s]);
                if (a > best) { best = a; br = lane + 32 * s; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int orr = __shfl_xor_sync(0xffffffffu, br, o);
                if (ob > best || (ob == best && orr < br)) { best = ob; br = orr; }
            }
            if (br == 0x7fffffff) br = k;   // all candidates NaN: mirror a zero pivot
            const int p = br;
            const int owner = p & 31, pslot = p >> 5;
            if (lane == owner) {
#pragma unroll
                for (int s = 0; s < ROWS; ++s)
                    if (s == pslot) {
#pragma unroll
                        for (int c = 0; c < NBT; c += 2)
                            *reinterpret_cast<double2*>(prow + c) = make_double2(d[s][c], c + 1 < NBT ? d[s][c + 1] : 0.0);
                    }
            }
            __syncwarp();
            const double pv = prow[k];
            const double inv = 1.0 / pv;
            if (lane == 0) {
                logdet += log(fabs(pv));
                if (pv == 0.0) zero = 1;
                piv[k] = p;
            }
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const int r = lane + 32 * s;
                const bool is_p = (r == p);
                if (is_p) { used[s] = 1; pstep[s] = k; }
                const double f = ck[s];
#pragma unroll
                for (int c = 0; c < NBT; c += 2) {
                    const double2 pc2 = *reinterpret_cast<const double2*>(prow + c);
                    const double pcs[2] = {pc2.x, pc2.y};
#pragma unroll
                    for (int e = 0; e < 2 && c + e < NBT; ++e) {
                        const int cc = c + e;
                        const double sc = pcs[e] * inv;
                        double v;
                        if (is_p) v = (cc == k) ? inv : sc;
                        else v = (cc == k) ? -f * inv : fma(-f, sc, d[s][cc]);
                        d[s][cc] = v;
                    }
                }
            }
            __syncwarp();
        }
        // ---- stage rows at their pivot step, then store inv(D)[k][c] = X[p_k][invp[c]]
#pragma unroll
        for (int s = 0; s < ROWS; ++s)
            if (pstep[s] >= 0)
#pragma unroll
                for (int c = 0; c < NBT; ++c) Xs[pstep[s] * LDX + c] = d[s][c];
        for (int m = lane; m < nb; m += 32) invp[piv[m]] = m;
        __syncwarp();
        double* dst = A.Dinv + (j * A.s + k_st) * bsz;
#pragma unroll
        for (int s = 0; s < ROWS; ++s) {
            const int r = lane + 32 * s;
            if (r < nb)
                for (int p = 0; p < P; ++p) {
                    double2 v;
                    v.x = Xs[r * LDX + invp[2 * p]];
                    v.y = (2 * p + 1 < nb) ? Xs[r * LDX + invp[2 * p + 1]] : 0.0;
                    reinterpret_cast<double2*>(dst)[(int64_t)p * nb + r] = v;
                }
        }
        __syncwarp();
        // |inv(D)|_1 = max column sum of X (a permutation of inv(D))
#pragma unroll
        for (int s = 0; s < ROWS; ++s)
            if (pstep[s] < 0) pstep[s] = lane + 32 * s;   // rows >= nb (unused)
        const double n2 = col_norm();
        if (lane == 0) {
            const double det = exp(logdet);
            const double cond = n1 * n2;
            const bool bad = zero || det == 0.0 || !isfinite(det) || !(cond <= 1e14);
            if (bad) atomicMin(A.fail_key, (unsigned long long)code);
        }
        __syncwarp();
    }
}

size_t inverse_smem(int nbt, int warps) {
    return (size_t)warps * (sizeof(double) * (nbt * (nbt + 1) + nbt) + sizeof(int) * 2 * nbt);
}

template <int NBT, bool EXACT>
static int launch_t(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    const int warps = 4;
    const size_t smem = inverse_smem(NBT, warps);
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_inverse<NBT, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inverse<NBT, EXACT>, warps * 32, smem));
    const int64_t need = (A.ntasks + warps - 1) / warps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_inverse<NBT, EXACT><<<grid, warps * 32, smem, st>>>(A);
    IRK_LAUNCHED();
    return IRK_OK;
}

// returns IRK_EINVAL if nb has no warp-inverse specialisation (caller falls back)
int launch_inverse(const irk_ctx* ctx, const int32_t* tasks, int64_t ntasks, int64_t T, int s, int nb,
                   const double* D, double* Dinv, unsigned long long* fail_key, cudaStream_t st) {
    if (ntasks <= 0) return IRK_OK;
    InvArgs A{tasks, ntasks, T, s, nb, D, Dinv, fail_key};
    if (nb == 24) return launch_t<24, true>(ctx, A, st);
    if (nb == 40) return launch_t<40, true>(ctx, A, st);
    if (nb == 50) return launch_t<50, true>(ctx, A, st);
    if (nb <= 16) return launch_t<16, false>(ctx, A, st);
    if (nb <= 32) return launch_t<32, false>(ctx, A, st);
    if (nb <= 64) return launch_t<64, false>(ctx, A, st);
    return IRK_EINVAL;
}

}  // namespace irk
