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
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "irk_internal.cuh"

namespace irk {

template <int K>
__host__ __device__ constexpr int kval(std::integral_constant<int, K>) { return K; }
__host__ __device__ constexpr int kval(int k) { return k; }

template <class F, int... K>
__device__ __forceinline__ void static_for(F&& f, std::integer_sequence<int, K...>) {
    (f(std::integral_constant<int, K>{}), ...);
}

// Warp argmax for partial pivoting: the largest |v| over lanes with a
// candidate, smallest row index on ties (the getrf rule).  For |v| >= 0 the
// IEEE bit pattern is monotonic, so three redux.sync reductions (high word,
// low word among the high-word winners, then row index) replace a 5-round
// shuffle butterfly.  Returns INT_MAX when no lane has a candidate.
__device__ __forceinline__ int warp_pivot(bool has, double absval, int row) {
    const unsigned hk = has ? (unsigned)__double2hiint(absval) + 1u : 0u;
    const unsigned lk = has ? (unsigned)__double2loint(absval) : 0u;
    const unsigned m1 = __reduce_max_sync(0xffffffffu, hk);
    const bool c1 = has && hk == m1;
    const unsigned m2 = __reduce_max_sync(0xffffffffu, c1 ? lk : 0u);
    const bool c2 = c1 && lk == m2;
    return (int)__reduce_min_sync(0xffffffffu, c2 ? (unsigned)row : 0x7fffffffu);
}

struct InvArgs {
    const int32_t* tasks;     // task codes k*T + j
    int64_t ntasks;
    int64_t T;
    int s, nb;
    const double* D;          // pivot blocks D[j][k] (device layout)
    double* Dinv;             // inverses Dinv[j][k]
    unsigned long long* fail_key;
    const int* ntasks_dev;    // non-NULL: task count on the device (<= ntasks), fallback lists
    int cap_per_sm;           // > 0: at most this many CTAs per SM (runs beside another kernel)
    InvForm form;             // form.J != NULL: build D from J and M (level 0) instead of reading it
};

// D_{j,k} formed from J and M, one element pair (double2 index p2 * nb + r of the device
// layout) at a time; the per-block pointers and scalars are resolved once per task
struct FormSrc {
    const double2* J;   // J_jj
    const double2* M;   // M_j or NULL
    double alpha, coef;
    bool keep;
};

__device__ __forceinline__ FormSrc form_src(const InvArgs& A, int64_t j, int k, int64_t bsz) {
    const InvForm& F = A.form;
    const int d = F.diag[j];
    FormSrc f;
    f.J = reinterpret_cast<const double2*>(F.J + (int64_t)d * bsz);
    f.M = F.M ? reinterpret_cast<const double2*>(F.M + j * bsz) : nullptr;
    f.alpha = F.alpha;
    f.coef = F.coef[k];
    f.keep = F.keep[d] != 0;
    return f;
}

__device__ __forceinline__ double2 form_pair(const FormSrc& f, int idx) {
    const double2 jv = f.J[idx];
    double x0 = __dmul_rn(f.alpha, jv.x), x1 = __dmul_rn(f.alpha, jv.y);
    if (f.M) {
        const double2 mv = f.M[idx];
        x0 = __dadd_rn(x0, __dmul_rn(f.coef, mv.x));
        x1 = __dadd_rn(x1, __dmul_rn(f.coef, mv.y));
    }
    return f.keep ? make_double2(x0, x1) : make_double2(0.0, 0.0);
}

// task count of a launch: the host bound, or the device count of a fallback list
__device__ __forceinline__ int64_t task_count(const InvArgs& A) {
    return A.ntasks_dev ? (int64_t)min((long long)*A.ntasks_dev, (long long)A.ntasks) : A.ntasks;
}

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

    for (int64_t t = (int64_t)blockIdx.x * wpb + warp; t < task_count(A); t += (int64_t)gridDim.x * wpb) {
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
        auto gj_step = [&](auto kc) {
            const int k = kval(kc);
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
                if (EXACT) {
                    // uniform row update new = a*P + g*old (no per-element select):
                    // pivot row a = 1/p, g = 0; other rows a = -f/p, g = 1;
                    // column k (static after unrolling) becomes a
                    const double a = is_p ? inv : -f * inv;
                    const double g = is_p ? 0.0 : 1.0;
#pragma unroll
                    for (int c = 0; c < NBT; c += 2) {
                        const double2 pc2 = *reinterpret_cast<const double2*>(prow + c);
                        const double pcs[2] = {pc2.x, pc2.y};
#pragma unroll
                        for (int e = 0; e < 2 && c + e < NBT; ++e) {
                            const int cc = c + e;
                            d[s][cc] = (cc == k) ? a : fma(a, pcs[e], g * d[s][cc]);
                        }
                    }
                } else {
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
            }
            __syncwarp();
        };
        if constexpr (EXACT) {
            static_for(gj_step, std::make_integer_sequence<int, NBT>{});   // k is a constant per step
        } else {
            for (int k = 0; k < nb; ++k) gj_step(k);
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

// ---------------------------------------------------------------------------
// 32 < nb <= 64: one row per lane.  A CTA inverts G = 32 / (nb-32) blocks with
// G "main" warps (rows 0..31 of block m in warp m) and one "extra" warp whose
// lane l holds row 32 + l % E of block l / E (E = nb - 32).  Each pivot step
// needs one CTA barrier: before it, every warp stages its best candidate row
// (per block) in a double-buffered shared slot; after it, every lane picks the
// winning candidate and reads the pivot row from the slot.
//
// Code size: a fully unrolled nb-step elimination is ~0.5 MB of SASS and
// thrashes the instruction cache.  Instead the row registers are rotated: the
// pivot steps run in chunks of 8 (unrolled), and after each chunk the row is
// rotated left by 8 columns, so the column eliminated in sub-step u always sits
// in register u (a compile-time index) and the loop body is one 8-step chunk.
// Rows are padded to NBR = ceil8(nb) zero columns; after NBR/8 chunks the
// rotation is back to the identity.
// ---------------------------------------------------------------------------
template <int NB>
struct Inv2Cfg {
    static constexpr int E = NB - 32;
    static constexpr int G = (32 / E) < 4 ? (32 / E) : 4;
    static constexpr int LDX = NB + 1;
    static constexpr int NBR = (NB + 7) & ~7;
};

template <int NB>
__host__ __device__ constexpr size_t inv2_smem_bytes() {
    using C = Inv2Cfg<NB>;
    return sizeof(double) * (2 * C::G * 2 * C::NBR + (size_t)C::G * NB * C::LDX + 2 * C::G * 2 + (size_t)C::G * NB) +
           sizeof(int) * (2 * C::G * 2 + 2 * C::G * NB);
}

template <int NB>
__global__ void __launch_bounds__(32 * (Inv2Cfg<NB>::G + 1), 2) k_inverse2(InvArgs A) {
    using C = Inv2Cfg<NB>;
    constexpr int E = C::E, G = C::G, LDX = C::LDX, NBR = C::NBR;
    extern __shared__ __align__(16) double sm2[];
    // layout: cand[2 bufs][G blocks][2 owners][NBR] | Xs[G][NB][LDX] | cval[2][G][2] | pvals[G][NB]
    //         | cidx[2][G][2] | piv[G][NB] | invp[G][NB]
    double* cand = sm2;
    double* Xs = cand + 2 * G * 2 * NBR;
    double* cval = Xs + (size_t)G * NB * LDX;
    double* pvals = cval + 2 * G * 2;
    int* cidx = reinterpret_cast<int*>(pvals + G * NB);
    int* pivs = cidx + 2 * G * 2;
    int* invp = pivs + G * NB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool extra = warp == G;
    const int blk = extra ? (lane / E) : warp;
    const int row = extra ? (32 + lane % E) : lane;
    const bool live = extra ? (lane < G * E) : true;
    const int P = NB / 2;
    const int64_t bsz = (int64_t)NB * 2 * ((NB + 1) / 2);
    const int64_t ntask = task_count(A);
    for (int64_t base = (int64_t)blockIdx.x * G; base < ntask; base += (int64_t)gridDim.x * G) {
        const int64_t t = base + blk;
        const bool valid = live && t < ntask;
        int64_t code = 0, j = 0;
        int k_st = 0;
        if (valid) {
            code = A.tasks[t];
            k_st = (int)(code / A.T);
            j = code - (int64_t)k_st * A.T;
        }
        double d[NBR];
        {
            const double2* src = reinterpret_cast<const double2*>(A.D + (j * A.s + k_st) * bsz);
#pragma unroll
            for (int p = 0; p < NBR / 2; ++p) {
                double2 v = make_double2(0.0, 0.0);
                if (valid && p < (NB + 1) / 2) v = src[(int64_t)p * NB + row];
                d[2 * p] = v.x;
                d[2 * p + 1] = (2 * p + 1 < NB) ? v.y : 0.0;
            }
        }
        double* X = Xs + (size_t)blk * NB * LDX;
        // |D|_1 via shared memory: every row stored, main-warp lanes sum columns
        auto colnorm = [&](double* out_norm) {
            if (live)
#pragma unroll
                for (int c = 0; c < NB; ++c) X[row * LDX + c] = fabs(d[c]);
            __syncthreads();
            if (!extra) {
                double mx = -1.0;
                int nan = 0;
                for (int c = lane; c < NB; c += 32) {
                    double sum = 0.0;
                    for (int r = 0; r < NB; ++r) sum += X[r * LDX + c];
                    if (sum != sum) nan = 1;
                    mx = fmax(mx, sum);
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
                }
                *out_norm = nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
            }
            __syncthreads();
        };
        double n1 = 0.0;
        colnorm(&n1);
        int used = live ? 0 : 1;
        int pstep = -1;
        int* piv = pivs + blk * NB;
        double* pvb = pvals + blk * NB;
        const int owner_slot = extra ? 1 : 0;
        // sub-step u of chunk ch eliminates column k = 8 ch + u, held in d[u]
        auto step = [&](int k, auto uc) {
            constexpr int u = decltype(uc)::value;
            const int buf = k & 1;
            double best = used ? -1.0 : fabs(d[u]);
            int br = used ? 0x7fffffff : row;
            // one branch-free butterfly for both warp kinds: main warps reduce over
            // all 32 lanes, the extra warp over its E-lane groups (then the group
            // leader's result is broadcast; E need not be a power of 2)
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int orr = __shfl_xor_sync(0xffffffffu, br, o);
                const int ol = lane ^ o;
                const bool same = !extra || ((ol / E == lane / E) && ol < G * E);
                if (same && (ob > best || (ob == best && orr < br))) { best = ob; br = orr; }
            }
            {
                const int leader = extra ? (lane / E) * E : lane;
                best = __shfl_sync(0xffffffffu, best, leader);
                br = __shfl_sync(0xffffffffu, br, leader);
            }
            if (live && br == row) {   // I hold this warp's candidate row for my block
                double* cr = cand + ((buf * G + blk) * 2 + owner_slot) * NBR;
#pragma unroll
                for (int c = 0; c < NBR; c += 2) *reinterpret_cast<double2*>(cr + c) = make_double2(d[c], d[c + 1]);
            }
            if (live && (extra ? (lane % E == 0) : (lane == 0))) {
                cval[(buf * G + blk) * 2 + owner_slot] = best;
                cidx[(buf * G + blk) * 2 + owner_slot] = br;
            }
            __syncthreads();
            // winner: main rows have smaller indices, so ties go to the main candidate
            const double v0 = cval[(buf * G + blk) * 2 + 0], v1 = cval[(buf * G + blk) * 2 + 1];
            const int i0 = cidx[(buf * G + blk) * 2 + 0], i1 = cidx[(buf * G + blk) * 2 + 1];
            const bool take1 = v1 > v0 || (v1 == v0 && i1 < i0);
            int p = take1 ? i1 : i0;
            if (p == 0x7fffffff) p = k;
            const double* pr = cand + ((buf * G + blk) * 2 + (take1 ? 1 : 0)) * NBR;
            const double pv = pr[u];
            const double inv = 1.0 / pv;
            if (!extra && lane == 0) {
                pvb[k] = pv;
                piv[k] = p;
            }
            const bool is_p = (row == p) && live;
            if (is_p) { used = 1; pstep = k; }
            // Unscaled pivot rows: the pivot row keeps its values (column k := 1)
            // and is scaled by 1/pivot once, when the rows are staged at the end;
            // every other row gets d + a * P with a = -d[k] / pivot (column k := a).
            // Rows that were pivots earlier carry their scale in f = d[k], so the
            // update is the scaled Gauss-Jordan step, one DFMA per element.
            const double a = is_p ? 0.0 : -d[u] * inv;
            const double ck = is_p ? 1.0 : a;
#pragma unroll
            for (int c = 0; c < NBR; c += 2) {
                const double2 pc = *reinterpret_cast<const double2*>(pr + c);
                d[c] = (c == u) ? ck : fma(a, pc.x, d[c]);
                d[c + 1] = (c + 1 == u) ? ck : fma(a, pc.y, d[c + 1]);
            }
        };
        // rotate left by 8: column 8(ch+1)+u moves to register u
        auto rotate8 = [&]() {
            double tmp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) tmp[u] = d[u];
#pragma unroll
            for (int c = 0; c < NBR - 8; ++c) d[c] = d[c + 8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d[NBR - 8 + u] = tmp[u];
        };
        // full chunks (no per-step guard: shuffles stay in provably converged code)
#pragma unroll 1
        for (int ch = 0; ch < NB / 8; ++ch) {
            static_for([&](auto uc) { step(ch * 8 + decltype(uc)::value, uc); },
                       std::make_integer_sequence<int, 8>{});
            rotate8();
        }
        if constexpr (NB % 8 != 0) {   // tail chunk: NB % 8 steps, then the last rotation
            static_for([&](auto uc) { step((NB / 8) * 8 + decltype(uc)::value, uc); },
                       std::make_integer_sequence<int, NB % 8>{});
            rotate8();
        }
        __syncthreads();
        // det = exp(sum_k log|pivot_k|) as slogdet: logs in parallel, summed in step order
        double logdet = 0.0;
        int zero = 0;
        if (!extra) {
            for (int m = lane; m < NB; m += 32) {
                const double pv = pvb[m];
                X[m] = log(fabs(pv));   // X is free until the rows are staged below
            }
            __syncwarp();
            if (lane == 0)
                for (int m = 0; m < NB; ++m) {
                    logdet += X[m];
                    if (pvb[m] == 0.0) zero = 1;
                }
        }
        __syncthreads();
        // stage rows at their pivot step (scaled by 1/pivot); inverse permutation; coalesced store
        if (live && pstep >= 0) {
            const double rs = 1.0 / pvb[pstep];
#pragma unroll
            for (int c = 0; c < NB; ++c) X[pstep * LDX + c] = d[c] * rs;
        }
        if (!extra)
            for (int m = lane; m < NB; m += 32) invp[blk * NB + piv[m]] = m;
        __syncthreads();
        if (valid) {
            double2* dst = reinterpret_cast<double2*>(A.Dinv + (j * A.s + k_st) * bsz);
            const int* ip = invp + blk * NB;
            for (int p = 0; p < P; ++p)
                dst[(int64_t)p * NB + row] = make_double2(X[row * LDX + ip[2 * p]], X[row * LDX + ip[2 * p + 1]]);
        }
        __syncthreads();
        double n2 = 0.0;
        colnorm(&n2);   // |inv|_1: column sums of the row-permuted X
        if (!extra && lane == 0 && base + blk < A.ntasks) {
            const double det = exp(logdet);
            const double cond = n1 * n2;
            const bool bad = zero || det == 0.0 || !isfinite(det) || !(cond <= 1e14);
            if (bad) atomicMin(A.fail_key, (unsigned long long)A.tasks[base + blk]);
        }
    }
}

// ---------------------------------------------------------------------------
// nb <= 40 (NBR = ceil8(nb) <= 40): one warp per block, no CTA barriers.
// Lane l holds rows l and l + 32 (ROWS = ceil(NBR/32) slots); the block is
// padded to NBR x NBR with an identity block, so the padded pivot steps pick
// their own padded row (pivot 1, zero multipliers) and change nothing -- the
// 8-step chunks need no runtime guard.  Same register rotation, unscaled pivot
// rows and pivot rule as k_inverse2; the pivot row is broadcast through a
// double-buffered per-warp shared row.
// ---------------------------------------------------------------------------
template <int NBR>
struct Inv3Cfg {
    static constexpr int ROWS = (NBR + 31) / 32;
    static constexpr int LDX = NBR + 1;
    static constexpr int WARPS = 4;
    // per warp: prow[2][NBR] | X[NBR][LDX] | pvals[NBR] doubles, piv/invp[NBR] ints
    static constexpr size_t warp_doubles = 2 * NBR + (size_t)NBR * LDX + NBR;
    static constexpr size_t smem = WARPS * (warp_doubles * sizeof(double) + 2 * NBR * sizeof(int));
};

template <int NBR>
__global__ void __launch_bounds__(32 * Inv3Cfg<NBR>::WARPS) k_inverse3(InvArgs A) {
    using C = Inv3Cfg<NBR>;
    constexpr int ROWS = C::ROWS, LDX = C::LDX;
    extern __shared__ __align__(16) double sm3[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* prow = sm3 + (size_t)warp * C::warp_doubles;
    double* X = prow + 2 * NBR;
    double* pvb = X + (size_t)NBR * LDX;
    int* piv = reinterpret_cast<int*>(sm3 + (size_t)C::WARPS * C::warp_doubles) + warp * 2 * NBR;
    int* invp = piv + NBR;
    const int nb = A.nb;
    const int P = (nb + 1) >> 1;
    const int64_t bsz = (int64_t)nb * 2 * P;
    for (int64_t t = (int64_t)blockIdx.x * C::WARPS + warp; t < task_count(A); t += (int64_t)gridDim.x * C::WARPS) {
        const int64_t code = A.tasks[t];
        const int k_st = (int)(code / A.T);
        const int64_t j = code - (int64_t)k_st * A.T;
        double d[ROWS][NBR];
        int used[ROWS], pstep[ROWS];
        {
            const double2* src = reinterpret_cast<const double2*>(A.D + (j * A.s + k_st) * bsz);
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const int r = lane + 32 * s;
                used[s] = r >= NBR;   // rows past the padded block never pivot
                pstep[s] = -1;
#pragma unroll
                for (int p = 0; p < NBR / 2; ++p) {
                    double2 v = make_double2(0.0, 0.0);
                    if (r < nb && p < P) v = src[(int64_t)p * nb + r];
                    if (2 * p + 1 >= nb) v.y = 0.0;
                    if (r >= nb) {   // identity padding
                        v.x = (2 * p == r) ? 1.0 : 0.0;
                        v.y = (2 * p + 1 == r) ? 1.0 : 0.0;
                    }
                    d[s][2 * p] = v.x;
                    d[s][2 * p + 1] = v.y;
                }
            }
        }
        // |.|_1 of the nb x nb part (max column abs-sum, NaN propagating)
        auto colnorm = [&]() -> double {
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const int r = lane + 32 * s;
                if (r < nb)
#pragma unroll
                    for (int c = 0; c < NBR; ++c) X[r * LDX + c] = fabs(d[s][c]);
            }
            __syncwarp();
            double mx = -1.0;
            int nan = 0;
            for (int c = lane; c < nb; c += 32) {
                double sum = 0.0;
                for (int r = 0; r < nb; ++r) sum += X[r * LDX + c];
                if (sum != sum) nan = 1;
                mx = fmax(mx, sum);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            }
            __syncwarp();
            return nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
        };
        const double n1 = colnorm();
        auto step = [&](int k, auto uc) {
            constexpr int u = decltype(uc)::value;
            bool has = false;
            double best = 0.0;
            int br = 0x7fffffff;
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const double a = fabs(d[s][u]);
                if (!used[s] && (!has || a > best)) { best = a; br = lane + 32 * s; has = true; }
            }
            const int pw = warp_pivot(has, best, br);
            const int p = (pw == 0x7fffffff) ? k : pw;
            double sv = d[0][u];
#pragma unroll
            for (int s = 1; s < ROWS; ++s) sv = ((p >> 5) == s) ? d[s][u] : sv;
            const double pv = __shfl_sync(0xffffffffu, sv, p & 31);
            const double inv = 1.0 / pv;
            double* pr = prow + (k & 1) * NBR;
            if (lane == (p & 31)) {
#pragma unroll
                for (int s = 0; s < ROWS; ++s)
                    if (s == (p >> 5))
#pragma unroll
                        for (int c = 0; c < NBR; c += 2)
                            *reinterpret_cast<double2*>(pr + c) = make_double2(d[s][c], d[s][c + 1]);
            }
            __syncwarp();
            if (lane == 0) { pvb[k] = pv; piv[k] = p; }
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                const bool is_p = (lane + 32 * s) == p;
                if (is_p) { used[s] = 1; pstep[s] = k; }
                const double a = is_p ? 0.0 : -d[s][u] * inv;
                const double ck = is_p ? 1.0 : a;
#pragma unroll
                for (int c = 0; c < NBR; c += 2) {
                    const double2 pc = *reinterpret_cast<const double2*>(pr + c);
                    d[s][c] = (c == u) ? ck : fma(a, pc.x, d[s][c]);
                    d[s][c + 1] = (c + 1 == u) ? ck : fma(a, pc.y, d[s][c + 1]);
                }
            }
        };
#pragma unroll 1
        for (int ch = 0; ch < NBR / 8; ++ch) {
            static_for([&](auto uc) { step(ch * 8 + decltype(uc)::value, uc); },
                       std::make_integer_sequence<int, 8>{});
#pragma unroll
            for (int s = 0; s < ROWS; ++s) {
                double tmp[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) tmp[u] = d[s][u];
#pragma unroll
                for (int c = 0; c < NBR - 8; ++c) d[s][c] = d[s][c + 8];
#pragma unroll
                for (int u = 0; u < 8; ++u) d[s][NBR - 8 + u] = tmp[u];
            }
        }
        __syncwarp();
        // det = exp(sum_k log|pivot_k|), k < nb, summed in step order
        for (int m = lane; m < nb; m += 32) X[m] = log(fabs(pvb[m]));
        __syncwarp();
        double logdet = 0.0;
        int zero = 0;
        if (lane == 0)
            for (int m = 0; m < nb; ++m) {
                logdet += X[m];
                if (pvb[m] == 0.0) zero = 1;
            }
        __syncwarp();
        // stage real rows at their pivot step (scaled by 1/pivot), then un-permute columns
#pragma unroll
        for (int s = 0; s < ROWS; ++s)
            if (pstep[s] >= 0 && pstep[s] < nb) {
                const double rs = 1.0 / pvb[pstep[s]];
#pragma unroll
                for (int c = 0; c < NBR; ++c) X[pstep[s] * LDX + c] = d[s][c] * rs;
            }
        for (int m = lane; m < nb; m += 32) invp[piv[m]] = m;
        __syncwarp();
        double2* dst = reinterpret_cast<double2*>(A.Dinv + (j * A.s + k_st) * bsz);
#pragma unroll
        for (int s = 0; s < ROWS; ++s) {
            const int r = lane + 32 * s;
            if (r < nb)
                for (int p = 0; p < P; ++p)
                    dst[(int64_t)p * nb + r] = make_double2(X[r * LDX + invp[2 * p]],
                                                            (2 * p + 1 < nb) ? X[r * LDX + invp[2 * p + 1]] : 0.0);
        }
        __syncwarp();
        // |inv|_1 from the staged rows (a row permutation of inv(D))
        double mx = -1.0;
        int nan = 0;
        for (int c = lane; c < nb; c += 32) {
            double sum = 0.0;
            for (int r = 0; r < nb; ++r) sum += fabs(X[r * LDX + c]);
            if (sum != sum) nan = 1;
            mx = fmax(mx, sum);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
        }
        const double n2 = nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
        if (lane == 0) {
            const double det = exp(logdet);
            const double cond = n1 * n2;
            const bool bad = zero || det == 0.0 || !isfinite(det) || !(cond <= 1e14);
            if (bad) atomicMin(A.fail_key, (unsigned long long)code);
        }
        __syncwarp();
    }
}

template <int NBR>
static int launch3(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    using C = Inv3Cfg<NBR>;
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_inverse3<NBR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem));
        IRK_CK(cudaFuncSetAttribute(k_inverse3<NBR>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr = true;
    }
    const int threads = 32 * C::WARPS;
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inverse3<NBR>, threads, C::smem));
    const int64_t need = (A.ntasks + C::WARPS - 1) / C::WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_inverse3<NBR><<<grid, threads, C::smem, st>>>(A);
    IRK_LAUNCHED();
    return IRK_OK;
}

// ---------------------------------------------------------------------------
// 32 < nb <= 40: one warp per block with a split layout.  Lane l holds row l
// (40 rotated positions, registers d[]) and a quarter of extra row 32 + l/4:
// positions [10q, 10q + 10) with q = l % 4 (registers x[]).  In pivot step u
// the extra-row entries of position u live in the lanes with q == u / 10 at
// x[u % 10] (a static index), and the extra row's multiplier is broadcast
// from that lane within its 4-lane group.  Rotating by 8 positions moves 8
// of the 10 quarter values in from the next lane of the group (shuffles).
// Rows nb..39 are identity padding, as in k_inverse3.
// ---------------------------------------------------------------------------
struct Inv4Cfg {
    static constexpr int NBR = 40, LDX = 42, WARPS = 4;
    static constexpr size_t warp_doubles = 2 * NBR + (size_t)NBR * LDX + NBR;
    static constexpr size_t smem = WARPS * (warp_doubles * sizeof(double) + 2 * NBR * sizeof(int));
};

template <int MINB>
__global__ void __launch_bounds__(32 * Inv4Cfg::WARPS, MINB) k_inverse4(InvArgs A) {
    using C = Inv4Cfg;
    constexpr int NBR = C::NBR, LDX = C::LDX;
    extern __shared__ __align__(16) double sm4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* prow = sm4 + (size_t)warp * C::warp_doubles;
    double* X = prow + 2 * NBR;
    double* pvb = X + (size_t)NBR * LDX;
    int* piv = reinterpret_cast<int*>(sm4 + (size_t)C::WARPS * C::warp_doubles) + warp * 2 * NBR;
    int* invp = piv + NBR;
    const int nb = A.nb;
    const int P = (nb + 1) >> 1;
    const int64_t bsz = (int64_t)nb * 2 * P;
    const int q = lane & 3, e = lane >> 2, re = 32 + e;
    const int gbase = lane & ~3, gnext = gbase | ((q + 1) & 3);
    for (int64_t t = (int64_t)blockIdx.x * C::WARPS + warp; t < task_count(A); t += (int64_t)gridDim.x * C::WARPS) {
        const int64_t code = A.tasks[t];
        const int k_st = (int)(code / A.T);
        const int64_t j = code - (int64_t)k_st * A.T;
        const double* srcd = A.D + (j * A.s + k_st) * bsz;
        double d[NBR], x[10];
        {
            const double2* src = reinterpret_cast<const double2*>(srcd);
#pragma unroll
            for (int p = 0; p < NBR / 2; ++p) {
                double2 v = make_double2(0.0, 0.0);
                if (p < P) v = src[(int64_t)p * nb + lane];
                if (2 * p + 1 >= nb) v.y = 0.0;
                d[2 * p] = v.x;
                d[2 * p + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 10; ++i) {
                const int c = 10 * q + i;
                double v;
                if (re < nb) v = (c < nb) ? srcd[((int64_t)(c >> 1) * nb + re) * 2 + (c & 1)] : 0.0;
                else v = (c == re) ? 1.0 : 0.0;   // identity padding
                x[i] = v;
            }
        }
        int used_m = 0, used_e = 0, pstep_m = -1, pstep_e = -1;
        // |.|_1 of the nb x nb part
        auto stage_abs = [&]() {
#pragma unroll
            for (int c = 0; c < NBR; ++c) X[lane * LDX + c] = fabs(d[c]);
#pragma unroll
            for (int i = 0; i < 10; ++i) X[re * LDX + 10 * q + i] = fabs(x[i]);
            __syncwarp();
        };
        auto norm_X = [&]() -> double {
            double mx = -1.0;
            int nan = 0;
            for (int c = lane; c < nb; c += 32) {
                double s4[4] = {0.0, 0.0, 0.0, 0.0};   // four independent chains
                int r = 0;
                for (; r + 4 <= nb; r += 4)
#pragma unroll
                    for (int h = 0; h < 4; ++h) s4[h] += fabs(X[(r + h) * LDX + c]);
                for (; r < nb; ++r) s4[0] += fabs(X[r * LDX + c]);
                const double sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                if (sum != sum) nan = 1;
                mx = fmax(mx, sum);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            }
            __syncwarp();
            return nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
        };
        stage_abs();
        const double n1 = norm_X();
        auto step = [&](int k, auto uc) {
            constexpr int u = decltype(uc)::value;
            constexpr int uq = u / 10, ui = u % 10;
            // candidates: own row first (smaller index wins ties), then the extra row
            bool has = !used_m;
            double best = fabs(d[u]);
            int br = lane;
            if (q == uq && !used_e) {
                const double a = fabs(x[ui]);
                if (!has || a > best) { best = a; br = re; has = true; }
            }
            const int pw = warp_pivot(has, best, br);
            const int p = (pw == 0x7fffffff) ? k : pw;
            // signed pivot straight from its owner lane: the reciprocal overlaps the row broadcast
            const double pv = __shfl_sync(0xffffffffu, p < 32 ? d[u] : x[ui], p < 32 ? p : (((p - 32) << 2) | uq));
            const double inv = 1.0 / pv;
            double* pr = prow + (k & 1) * NBR;
            if (p < 32) {
                if (lane == p)
#pragma unroll
                    for (int c = 0; c < NBR; c += 2) *reinterpret_cast<double2*>(pr + c) = make_double2(d[c], d[c + 1]);
            } else if (re == p) {
#pragma unroll
                for (int i = 0; i < 10; i += 2) *reinterpret_cast<double2*>(pr + 10 * q + i) = make_double2(x[i], x[i + 1]);
            }
            // extra row's column-u entry, from the group lane holding position u
            const double fe = __shfl_sync(0xffffffffu, x[ui], gbase | uq);
            __syncwarp();
            if (lane == 0) { pvb[k] = pv; piv[k] = p; }
            {
                const bool is_p = lane == p;
                if (is_p) { used_m = 1; pstep_m = k; }
                const double a = is_p ? 0.0 : -d[u] * inv;
                const double ck = is_p ? 1.0 : a;
#pragma unroll
                for (int c = 0; c < NBR; c += 2) {
                    const double2 pc = *reinterpret_cast<const double2*>(pr + c);
                    d[c] = (c == u) ? ck : fma(a, pc.x, d[c]);
                    d[c + 1] = (c + 1 == u) ? ck : fma(a, pc.y, d[c + 1]);
                }
            }
            {
                const bool is_p = re == p;
                if (is_p) { used_e = 1; pstep_e = k; }
                const double a = is_p ? 0.0 : -fe * inv;
                const double ck = is_p ? 1.0 : a;
                const double* pq = pr + 10 * q;
#pragma unroll
                for (int i = 0; i < 10; i += 2) {
                    const double2 pc = *reinterpret_cast<const double2*>(pq + i);
                    x[i] = (q == uq && i == ui) ? ck : fma(a, pc.x, x[i]);
                    x[i + 1] = (q == uq && i + 1 == ui) ? ck : fma(a, pc.y, x[i + 1]);
                }
            }
        };
#pragma unroll 1
        for (int ch = 0; ch < NBR / 8; ++ch) {
            static_for([&](auto uc) { step(ch * 8 + decltype(uc)::value, uc); },
                       std::make_integer_sequence<int, 8>{});
            double tmp[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) tmp[u] = d[u];
#pragma unroll
            for (int c = 0; c < NBR - 8; ++c) d[c] = d[c + 8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d[NBR - 8 + u] = tmp[u];
            // quarter rotation: new x[i] = position 10q + i + 8
            double nx[10];
            nx[0] = x[8];
            nx[1] = x[9];
#pragma unroll
            for (int i = 2; i < 10; ++i) nx[i] = __shfl_sync(0xffffffffu, x[i - 2], gnext);
#pragma unroll
            for (int i = 0; i < 10; ++i) x[i] = nx[i];
        }
        __syncwarp();
        // det = exp(sum log|pivot|) (slogdet); |pivot| == 0 -> singular
        double lg = 0.0;
        int zero = 0;
        for (int m = lane; m < nb; m += 32) {
            const double pv = pvb[m];
            lg += log(fabs(pv));
            zero |= pv == 0.0;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lg += __shfl_xor_sync(0xffffffffu, lg, o);
            zero |= __shfl_xor_sync(0xffffffffu, zero, o);
        }
        const double logdet = lg;
        // stage row k of inv(D) = (row pivoted at step k) / pivot_k with the column
        // permutation folded in: inv(D)[k][piv[m]] = X[p_k][m]
        int pc[NBR];
#pragma unroll
        for (int m = 0; m < NBR; m += 4) {
            const int4 v = *reinterpret_cast<const int4*>(piv + m);
            pc[m] = v.x; pc[m + 1] = v.y; pc[m + 2] = v.z; pc[m + 3] = v.w;
        }
        if (pstep_m >= 0 && pstep_m < nb) {
            const double rs = 1.0 / pvb[pstep_m];
#pragma unroll
            for (int c = 0; c < NBR; ++c)
                if (c < nb) X[pstep_m * LDX + pc[c]] = d[c] * rs;
        }
        if (pstep_e >= 0 && pstep_e < nb) {
            const double rs = 1.0 / pvb[pstep_e];
#pragma unroll
            for (int i = 0; i < 10; ++i)
                if (10 * q + i < nb) X[pstep_e * LDX + piv[10 * q + i]] = x[i] * rs;
        }
        __syncwarp();
        double2* dst = reinterpret_cast<double2*>(A.Dinv + (j * A.s + k_st) * bsz);
        for (int r = lane; r < nb; r += 32)
            for (int p = 0; p < P; ++p) {
                double2 v = *reinterpret_cast<const double2*>(X + r * LDX + 2 * p);
                if (2 * p + 1 >= nb) v.y = 0.0;
                dst[(int64_t)p * nb + r] = v;
            }
        __syncwarp();
        const double n2 = norm_X();
        if (lane == 0) {
            const double det = exp(logdet);
            const double cond = n1 * n2;
            const bool bad = zero || det == 0.0 || !isfinite(det) || !(cond <= 1e14);
            if (bad) atomicMin(A.fail_key, (unsigned long long)code);
        }
        __syncwarp();
    }
}

template <int MINB>
static int launch4_t(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    using C = Inv4Cfg;
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_inverse4<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem));
        IRK_CK(cudaFuncSetAttribute(k_inverse4<MINB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr = true;
    }
    const int threads = 32 * C::WARPS;
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inverse4<MINB>, threads, C::smem));
    const int64_t need = (A.ntasks + C::WARPS - 1) / C::WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_inverse4<MINB><<<grid, threads, C::smem, st>>>(A);
    IRK_LAUNCHED();
    return IRK_OK;
}

static int launch4(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    const char* e = getenv("IRK_INV4_MINB");   // tuning knob
    switch (e ? atoi(e) : 1) {
        case 2: return launch4_t<2>(ctx, A, st);
        case 3: return launch4_t<3>(ctx, A, st);
        case 4: return launch4_t<4>(ctx, A, st);
        default: return launch4_t<1>(ctx, A, st);
    }
}

template <int NB>
static int launch2(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    using C = Inv2Cfg<NB>;
    const size_t smem = inv2_smem_bytes<NB>();
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_inverse2<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int threads = 32 * (C::G + 1);
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inverse2<NB>, threads, smem));
    const int64_t need = (A.ntasks + C::G - 1) / C::G;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_inverse2<NB><<<grid, threads, smem, st>>>(A);
    IRK_LAUNCHED();
    return IRK_OK;
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

// ---------------------------------------------------------------------------
// Blocked Gauss-Jordan on the FP64 tensor cores (DMMA m8n8k4), 16 < nb <= 64.
//
// One warp per block, the block in shared memory (row-major, ld = NBT + 4:
// conflict-free A/B fragment loads).  Panels of 8 columns: the 8 scalar GJ
// steps run on the NBT x 8 panel in registers (lane = (column c = l&7, row
// group q = l>>3), rows q, q+4, ...), leaving [G; F] = in-place GJ values of
// the panel columns; the other columns get the rank-8 update
//     A_R <- [0; A_R'] + [G; F] * A_KR      (A_KR = the panel's rows, old)
// as 8x8 DMMA tiles.  2 nb^3 flops, ~80% of them on the tensor cores.
//
// No row interchanges: a block takes this path only if, at every step, the
// diagonal is a partial-pivoting choice (|a_kk| >= |a_rk| for all r > k; ties
// go to the smaller row, the getrf/idamax rule), i.e. getrf would not swap --
// then the elimination is exactly the pivoted one.  Any block where a swap
// would happen (or a zero / NaN pivot appears) is appended to a fallback list
// and re-done by the pivoted warp kernels.  det / cond as _inv_with_cond
// (numba_backend.py:33-40).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Reciprocal without the IEEE slow-path call: rcp.approx seed + two Newton steps (<= 1 ulp).
// Callers keep |x| inside [1e-30, 1e30] (anything else goes to the pivoted kernels).
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// not volatile: a pure function of its operands, so the scheduler may interleave independent tiles
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NT>
struct InvTcCfg {
    // ld = 8 (mod 16) doubles: conflict-free C-tile double2 accesses (the DMMA update's traffic)
    static constexpr int NBT = 8 * NT, LD = NBT + ((24 - NBT % 16) % 16), WARPS = 4;
    static constexpr int RL = (NBT + 31) / 32;    // panel rows per lane (row-per-lane layout)
    static constexpr size_t warp_doubles = (size_t)NBT * LD + 64;   // + 2 x 8 pivot-row buffer / 8 x 8 L scratch
    static constexpr size_t smem = WARPS * warp_doubles * sizeof(double);
};

// EXACT: nb == 8 NT (block index math and loops fold to constants); FORM: build D from
// J and M (factor level 0) instead of reading it
// row slot ks (0 or RL - 1, RL <= 2) of the lane's panel registers without dynamic register indexing
#define IRK_PK(ks_, c_) ((RL == 1 || (ks_) == 0) ? pa[0][c_] : pa[RL - 1][c_])

// BG (default): block Gauss-Jordan -- only the 8 x 8 pivot tile is eliminated with scalar
// arithmetic (two entries per lane in the DMMA C-fragment layout, shuffles only); the panel
// columns F_i = -X_ip P, the multipliers of the rows below (pivoting check) and the rank-8
// update all run as DMMA tiles.  !BG: the 8 scalar steps run on the whole NBT x 8 panel
// (kept for NT = 5 as the A/B alternative, IRK_INV_BG=0).
template <int NT, bool EXACT, bool FORM, bool BG = true>
__global__ void __launch_bounds__(32 * InvTcCfg<NT>::WARPS, NT <= 5 ? 4 : 1)
    k_inverse_tc(InvArgs A, int* fb_list, int* fb_count) {
    using C = InvTcCfg<NT>;
    constexpr int NBT = C::NBT, LD = C::LD, RL = C::RL;
    constexpr int NPAIR = NBT * NBT / 2;            // double2 per padded block
    extern __shared__ __align__(16) double smtc[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* X = smtc + (size_t)warp * C::warp_doubles;
    double* rowbuf = X + (size_t)NBT * LD;          // [2][8]: pivot row broadcast (alternating)
    const int nb = EXACT ? NBT : A.nb;
    const int P = (nb + 1) >> 1;
    const int64_t bsz = (int64_t)nb * 2 * P;
    const int fr = lane >> 2, fk = lane & 3;        // fragment layout
    // shared-memory position of element (r, c): 16-byte chunks XOR-swizzled by x(r) inside each
    // group of 4 chunks, so the row-per-lane panel / block accesses (32 rows of one column pair)
    // hit 8 distinct bank groups per phase instead of 2 (rows 2m, 2m + 1 share a swizzle: the
    // C-tile double2 accesses stay conflict-free)
    // x(r) = bits (r>>1)&1 and (r>>2)&1 swapped: rows 0, 2, 4, 6 still get four distinct chunk
    // permutations (row-per-lane / block load-store accesses), and rows r0 + 2, r0 + 3 of an aligned
    // 4 x 4 fragment (A / B operands, 64-bit loads of a half-warp) land on the other chunk pair of
    // the group -- with x = (r>>1)&3 they hit the same two chunks as rows r0, r0 + 1 (2-way conflicts
    // on every fragment load: 296 of 1890 shared-memory wavefronts per nb = 40 block)
    auto sw = [](int r, int c) -> int {
        const int x = (((r >> 1) & 1) << 1) | ((r >> 2) & 1);
        return r * LD + ((((c >> 1) ^ x) << 1) | (c & 1));
    };
    for (int64_t t = (int64_t)blockIdx.x * C::WARPS + warp; t < A.ntasks; t += (int64_t)gridDim.x * C::WARPS) {
        const int64_t code = A.tasks[t];
        const int k_st = (int)(code / A.T);
        const int64_t j = code - (int64_t)k_st * A.T;
        const double2* src = reinterpret_cast<const double2*>(A.D + (j * A.s + k_st) * bsz);
        double2* dst_d = FORM ? reinterpret_cast<double2*>(A.form.Dst + (j * A.s + k_st) * bsz) : nullptr;
        FormSrc fsrc{};
        if constexpr (FORM) fsrc = form_src(A, j, k_st, bsz);
        // ---- load: device pair p2 of row r is double2 index p2 * nb + r.  fsq: this lane's share of
        // |D|_F^2 over the nb x nb part (cheap bound for the condition check below)
        double fsq = 0.0;
        auto load_block = [&]() {
            if constexpr (EXACT && FORM) {
                // loads of J_jj and M_j issued in batches ahead of the arithmetic and the stores
                // (one load -> multiply -> store chain per pair stalled on every global load)
                constexpr int NE = (NPAIR + 31) / 32, BATCH = 5;
                const bool store = A.form.store;
    #pragma unroll
                for (int e0 = 0; e0 < NE; e0 += BATCH) {
                    double2 jv[BATCH], mv[BATCH];
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        jv[b] = mv[b] = make_double2(0.0, 0.0);
                        if (e0 + b < NE && (NPAIR % 32 == 0 || idx < NPAIR)) {
                            jv[b] = __ldg(fsrc.J + idx);
                            if (fsrc.M) mv[b] = __ldg(fsrc.M + idx);
                        }
                    }
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        if (e0 + b < NE && (NPAIR % 32 == 0 || idx < NPAIR)) {
                            const int p2 = idx / NBT, r = idx - p2 * NBT;
                            double x0 = __dmul_rn(fsrc.alpha, jv[b].x), x1 = __dmul_rn(fsrc.alpha, jv[b].y);
                            if (fsrc.M) {
                                x0 = __dadd_rn(x0, __dmul_rn(fsrc.coef, mv[b].x));
                                x1 = __dadd_rn(x1, __dmul_rn(fsrc.coef, mv[b].y));
                            }
                            const double2 v = fsrc.keep ? make_double2(x0, x1) : make_double2(0.0, 0.0);
                            if (store) dst_d[idx] = v;
                            fsq = fma(v.x, v.x, fma(v.y, v.y, fsq));
                            *reinterpret_cast<double2*>(X + sw(r, 2 * p2)) = v;
                        }
                    }
                }
            } else if constexpr (EXACT) {
                constexpr int NE = (NPAIR + 31) / 32, BATCH = 5;   // loads ahead of the shared-memory stores
    #pragma unroll
                for (int e0 = 0; e0 < NE; e0 += BATCH) {
                    double2 v[BATCH];
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        if (e0 + b < NE && (NPAIR % 32 == 0 || idx < NPAIR)) v[b] = __ldg(src + idx);
                    }
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        if (e0 + b < NE && (NPAIR % 32 == 0 || idx < NPAIR)) {
                            const int p2 = idx / NBT, r = idx - p2 * NBT;
                            fsq = fma(v[b].x, v[b].x, fma(v[b].y, v[b].y, fsq));
                            *reinterpret_cast<double2*>(X + sw(r, 2 * p2)) = v[b];
                        }
                    }
                }
            } else {
                // nb < NBT (identity padding): global loads issued in batches ahead of the arithmetic
                // and the shared-memory stores (one exposed DRAM latency per batch instead of one per
                // element pair: config 2, nb = 50, level-0 inverse 1.89 -> see DESIGN)
                constexpr int NE = (NPAIR + 31) / 32, BATCH = 7;
    #pragma unroll 1
                for (int e0 = 0; e0 < NE; e0 += BATCH) {
                    double2 jv[BATCH], mv[BATCH];
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        const int p2 = idx / NBT, r = idx - p2 * NBT;
                        jv[b] = mv[b] = make_double2(0.0, 0.0);
                        if (idx < NPAIR && r < nb && p2 < P) {
                            if constexpr (FORM) {
                                jv[b] = __ldg(fsrc.J + p2 * nb + r);
                                if (fsrc.M) mv[b] = __ldg(fsrc.M + p2 * nb + r);
                            } else {
                                jv[b] = __ldg(src + p2 * nb + r);
                            }
                        }
                    }
    #pragma unroll
                    for (int b = 0; b < BATCH; ++b) {
                        const int idx = lane + 32 * (e0 + b);
                        if (idx >= NPAIR) continue;
                        const int p2 = idx / NBT, r = idx - p2 * NBT;
                        double2 v;
                        if (r < nb && p2 < P) {
                            v = jv[b];
                            if constexpr (FORM) {
                                double x0 = __dmul_rn(fsrc.alpha, jv[b].x), x1 = __dmul_rn(fsrc.alpha, jv[b].y);
                                if (fsrc.M) {
                                    x0 = __dadd_rn(x0, __dmul_rn(fsrc.coef, mv[b].x));
                                    x1 = __dadd_rn(x1, __dmul_rn(fsrc.coef, mv[b].y));
                                }
                                v = fsrc.keep ? make_double2(x0, x1) : make_double2(0.0, 0.0);
                                if (A.form.store) dst_d[p2 * nb + r] = v;
                            }
                            if (2 * p2 + 1 >= nb) v.y = 0.0;
                            fsq = fma(v.x, v.x, fma(v.y, v.y, fsq));
                        } else {   // identity padding
                            v = make_double2(2 * p2 == r ? 1.0 : 0.0, 2 * p2 + 1 == r ? 1.0 : 0.0);
                        }
                        *reinterpret_cast<double2*>(X + sw(r, 2 * p2)) = v;
                    }
                }
            }
        };
        load_block();
        const double fsq1 = fsq;
        __syncwarp();
        // |.|_1: max column abs sum over the nb x nb part (NaN propagating)
        auto col_norm = [&]() -> double {
            double mx = -1.0;
            int nan = 0;
#pragma unroll
            for (int h = 0; h < (NBT + 31) / 32; ++h) {
                const int c = lane + 32 * h;
                if (c < nb) {
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
                    if constexpr (EXACT) {
#pragma unroll
                        for (int r = 0; r < NBT; ++r) s4[r & 3] += fabs(X[sw(r, c)]);
                    } else {
                        int r = 0;
                        for (; r + 4 <= nb; r += 4)
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4) s4[q4] += fabs(X[sw(r + q4, c)]);
                        for (; r < nb; ++r) s4[0] += fabs(X[sw(r, c)]);
                    }
                    const double sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
                    if (sum != sum) nan = 1;
                    mx = fmax(mx, sum);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            }
            return nan ? __longlong_as_double(0x7ff8000000000000LL) : mx;
        };
        // |pivot_k| kept by lane k mod 32 (log-determinant after the sweep)
        double apiv[(NBT + 31) / 32];
#pragma unroll
        for (int h = 0; h < (NBT + 31) / 32; ++h) apiv[h] = 1.0;
        bool swap = false;
        auto panel = [&](auto pv) {   // panel index: std::integral_constant (unrolled) or int (ROLL)
            const int p = pv;
            const int k0 = 8 * p;
            if (swap) return;
            // ---- panel to registers, one row per lane: pa[j][c] = X[lane + 32 j][k0 + c]
            double pa[RL][8];
#pragma unroll
            for (int j = 0; j < RL; ++j) {
                const int r = lane + 32 * j;
#pragma unroll
                for (int c = 0; c < 8; c += 2) {
                    double2 v = make_double2(0.0, 0.0);
                    if (r < NBT) v = *reinterpret_cast<const double2*>(X + sw(r, k0 + c));
                    pa[j][c] = v.x;
                    pa[j][c + 1] = v.y;
                }
            }
            // ---- 8 scalar GJ steps on the panel columns
            static_for([&](auto kc_) {
                constexpr int kk = decltype(kc_)::value;
                const int k = k0 + kk;
                const int ko = k & 31, ks = k >> 5;          // owner lane / slot of row k
                const bool own = lane == ko;
                const double piv = __shfl_sync(0xffffffffu, IRK_PK(ks, kk), ko);
                // partial-pivoting equivalence: no row r > k of column k beats the diagonal
                const double ap = fabs(piv);
                bool beat = false;
#pragma unroll
                for (int j = 0; j < RL; ++j)
                    if (lane + 32 * j > k && lane + 32 * j < NBT) beat |= fabs(pa[j][kk]) > ap;
                const bool ok = !__any_sync(0xffffffffu, beat) && piv != 0.0 && isfinite(piv);
                if (!ok) swap = true;
                const double inv = 1.0 / piv;
                if (k < nb && own) {
                    if (RL == 1 || ks == 0) apiv[0] = ap;
                    else apiv[RL - 1] = ap;
                }
                // new row k = a_k / piv (column k: 1 / piv), broadcast through shared memory
                double* rb = rowbuf + 8 * (kk & 1);
                if (own) {
#pragma unroll
                    for (int c = 0; c < 8; c += 2) {
                        double2 v = make_double2(c == kk ? inv : IRK_PK(ks, c) * inv, c + 1 == kk ? inv : IRK_PK(ks, c + 1) * inv);
                        *reinterpret_cast<double2*>(rb + c) = v;
                    }
                }
                __syncwarp();
                double rk[8];
#pragma unroll
                for (int c = 0; c < 8; c += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(rb + c);
                    rk[c] = v.x;
                    rk[c + 1] = v.y;
                }
                // other rows: a_rc - a_rk rk_c, column k: -a_rk / piv
#pragma unroll
                for (int j = 0; j < RL; ++j) {
                    const bool isk = own && j == ks;
                    const double f = pa[j][kk];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const double nv = (c == kk) ? -f * inv : fma(-f, rk[c], pa[j][c]);
                        pa[j][c] = isk ? rk[c] : nv;
                    }
                }
            }, std::make_integer_sequence<int, 8>{});
            if (swap) return;
            // ---- rank-8 update of the other column tiles (old panel rows as B)
            double bf[NT][2];
#pragma unroll
            for (int jt = 0; jt < NT; ++jt)
#pragma unroll
                for (int kc = 0; kc < 2; ++kc)
                    bf[jt][kc] = (jt == p) ? 0.0 : X[sw(k0 + 4 * kc + fk, 8 * jt + fr)];
            __syncwarp();
#pragma unroll
            for (int j = 0; j < RL; ++j) {
                const int r = lane + 32 * j;
                if (r < NBT)
#pragma unroll
                    for (int c = 0; c < 8; c += 2)
                        *reinterpret_cast<double2*>(X + sw(r, k0 + c)) = make_double2(pa[j][c], pa[j][c + 1]);
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                const double a0 = X[sw(8 * it + fr, k0 + fk)];
                const double a1 = X[sw(8 * it + fr, k0 + 4 + fk)];
#pragma unroll
                for (int jt = 0; jt < NT; ++jt) {
                    if (jt == p) continue;
                    double* cp = X + sw(8 * it + fr, 8 * jt + 2 * fk);
                    double2 c = (it == p) ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(cp);
                    dmma_f64(c.x, c.y, a0, bf[jt][0]);
                    dmma_f64(c.x, c.y, a1, bf[jt][1]);
                    *reinterpret_cast<double2*>(cp) = c;
                }
            }
            __syncwarp();
        };
        // ---- block Gauss-Jordan (BG).  Pivot tile state of the scalar elimination: lane (fr, fk)
        // holds X_pp[fr][2 fk], [2 fk + 1] (the DMMA C-fragment layout) in (v0, v1) and the
        // negated multipliers of its two columns in (l0, l1).
        double v0 = 0.0, v1 = 0.0, l0 = 0.0, l1 = 0.0;
        bool beat = false;
        // one Gauss-Jordan step on the 8 x 8 pivot tile of panel p (shuffles only)
        auto gj_step = [&](auto pv, auto kv) {
            constexpr int p = decltype(pv)::value;
            constexpr int k = decltype(kv)::value;
            constexpr int kh = k >> 1;
            constexpr bool odd = (k & 1) != 0;
            const double selv = odd ? v1 : v0;
            const double piv = __shfl_sync(0xffffffffu, selv, 4 * k + kh);        // X[k][k]
            const double f = __shfl_sync(0xffffffffu, selv, (lane & ~3) | kh);    // X[fr][k]
            const double rk0 = __shfl_sync(0xffffffffu, v0, 4 * k + fk);          // X[k][2 fk]
            const double rk1 = __shfl_sync(0xffffffffu, v1, 4 * k + fk);          // X[k][2 fk + 1]
            const double ap = fabs(piv);
            // partial-pivoting equivalence inside the tile: no row r > k of column k beats the
            // diagonal; pivots outside [1e-30, 1e30] (0, inf, NaN included) go to the pivoted kernels
            beat |= ((fr > k) && (fabs(f) > ap)) || !(ap >= 1e-30 && ap <= 1e30);
            if (8 * p + k < nb && lane == ((8 * p + k) & 31)) apiv[(8 * p + k) >> 5] = ap;
            const double inv = rcp_nr(piv);
            const bool isc = fk == kh, isr = fr == k;
            // scaled pivot row in this lane's columns; column k of the new row k is 1 / piv
            double s0 = rk0 * inv, s1 = rk1 * inv;
            double t0 = v0, t1 = v1;
            if (odd) {
                s1 = isc ? inv : s1;
                t1 = isc ? 0.0 : t1;
            } else {
                s0 = isc ? inv : s0;
                t0 = isc ? 0.0 : t0;
            }
            // other rows: a_rc - a_rk rk_c, column k: -a_rk / piv
            const double n0 = fma(-f, s0, t0), n1 = fma(-f, s1, t1);
            v0 = isr ? s0 : n0;
            v1 = isr ? s1 : n1;
            // column k now holds -l_rk for the rows below k (masked to the unit lower triangle later)
            if (odd) l1 = isc ? v1 : l1;
            else l0 = isc ? v0 : l0;
        };
        // P = inv(X_pp) -> X_pp, -L_pp (unit lower triangular factor of the unpivoted LU) -> scratch
        auto gj_store = [&](auto pv) {
            constexpr int k0 = 8 * decltype(pv)::value;
            *reinterpret_cast<double2*>(X + sw(k0 + fr, k0 + 2 * fk)) = make_double2(v0, v1);
            const int c0 = 2 * fk;
            *reinterpret_cast<double2*>(rowbuf + fr * 8 + c0) =
                make_double2(fr > c0 ? l0 : (fr == c0 ? -1.0 : 0.0), fr > c0 + 1 ? l1 : (fr == c0 + 1 ? -1.0 : 0.0));
        };
        if constexpr (BG) {
            // pivot tile of panel 0 (the later ones are eliminated during the previous panel's update)
            const double2 v = *reinterpret_cast<const double2*>(X + sw(fr, 2 * fk));
            v0 = v.x;
            v1 = v.y;
            static_for([&](auto kc_) { gj_step(std::integral_constant<int, 0>{}, kc_); }, std::make_integer_sequence<int, 8>{});
            gj_store(std::integral_constant<int, 0>{});
            if (__any_sync(0xffffffffu, beat)) swap = true;
            __syncwarp();
        }
        auto panel_bg = [&](auto pv) {
            constexpr int p = decltype(pv)::value;
            constexpr int k0 = 8 * p;
            constexpr bool LA = p + 1 < NT;          // look ahead: eliminate pivot tile p + 1 during this update
            if (swap) return;
            const double* Ls = rowbuf;
            // old row panel p as B fragments (read before row tile p is overwritten), old column
            // panel as A fragments, P and -L_pp as B fragments
            double bf[NT][2], af[NT][2];
#pragma unroll
            for (int jt = 0; jt < NT; ++jt)
#pragma unroll
                for (int kc = 0; kc < 2; ++kc)
                    bf[jt][kc] = (jt == p) ? 0.0 : X[sw(k0 + 4 * kc + fk, 8 * jt + fr)];
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                af[it][0] = (it == p) ? 0.0 : X[sw(8 * it + fr, k0 + fk)];
                af[it][1] = (it == p) ? 0.0 : X[sw(8 * it + fr, k0 + 4 + fk)];
            }
            const double pb0 = -X[sw(k0 + fk, k0 + fr)], pb1 = -X[sw(k0 + 4 + fk, k0 + fr)];
            const double lb0 = Ls[fk * 8 + fr], lb1 = Ls[(4 + fk) * 8 + fr];
            __syncwarp();
            // F_i = -X_ip P (the in-place Gauss-Jordan values of the panel columns)
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                if (it == p) continue;
                double2 c = make_double2(0.0, 0.0);
                dmma_nv(c.x, c.y, af[it][0], pb0);
                dmma_nv(c.x, c.y, af[it][1], pb1);
                *reinterpret_cast<double2*>(X + sw(8 * it + fr, k0 + 2 * fk)) = c;
            }
            __syncwarp();
            // [P; F] as A fragments
#pragma unroll
            for (int it = 0; it < NT; ++it) {
                af[it][0] = X[sw(8 * it + fr, k0 + fk)];
                af[it][1] = X[sw(8 * it + fr, k0 + 4 + fk)];
            }
            // multipliers of the row tiles below the pivot tile, X_ip inv(U_pp) = F_i (-L_pp): getrf
            // would not swap iff all |.| <= 1 (ties and rounding-level excesses keep the diagonal,
            // an equally valid partial-pivoting choice)
#pragma unroll
            for (int it = p + 1; it < NT; ++it) {
                double2 w = make_double2(0.0, 0.0);
                dmma_nv(w.x, w.y, af[it][0], lb0);
                dmma_nv(w.x, w.y, af[it][1], lb1);
                beat |= (fabs(w.x) > 1.0 + 1e-12) || (fabs(w.y) > 1.0 + 1e-12);
            }
            // rank-8 update A_R <- [0; A_R'] + [P; F] A_KR.  The next pivot tile goes first and stays
            // in registers; its 8 scalar elimination steps are spread over the other tile updates
            if constexpr (LA) {
                const double2 c = *reinterpret_cast<const double2*>(X + sw(k0 + 8 + fr, k0 + 8 + 2 * fk));
                v0 = c.x;
                v1 = c.y;
                dmma_nv(v0, v1, af[p + 1][0], bf[p + 1][0]);
                dmma_nv(v0, v1, af[p + 1][1], bf[p + 1][1]);
                l0 = l1 = 0.0;
            }
            constexpr int NTL = NT * (NT - 1);
            static_for([&](auto n_) {
                constexpr int n = decltype(n_)::value;
                constexpr int it = n / (NT - 1), jq = n % (NT - 1), jt = jq < p ? jq : jq + 1;
                if constexpr (LA) {
                    // step k goes before tile floor(k NTL / 8)
                    static_for([&](auto kc_) {
                        constexpr int k = decltype(kc_)::value;
                        if constexpr ((k * NTL) / 8 == n) gj_step(std::integral_constant<int, p + 1>{}, kc_);
                    }, std::make_integer_sequence<int, 8>{});
                }
                if constexpr (!(LA && it == p + 1 && jt == p + 1)) {
                    double* cp = X + sw(8 * it + fr, 8 * jt + 2 * fk);
                    double2 c = (it == p) ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(cp);
                    dmma_nv(c.x, c.y, af[it][0], bf[jt][0]);
                    dmma_nv(c.x, c.y, af[it][1], bf[jt][1]);
                    *reinterpret_cast<double2*>(cp) = c;
                }
            }, std::make_integer_sequence<int, NTL>{});
            if constexpr (LA) gj_store(std::integral_constant<int, p + 1>{});
            if (__any_sync(0xffffffffu, beat)) swap = true;
            __syncwarp();
        };
        if constexpr (BG) {
            static_for([&](auto pc_) { panel_bg(pc_); }, std::make_integer_sequence<int, NT>{});
        } else {
            static_for([&](auto pc_) { panel(pc_); }, std::make_integer_sequence<int, NT>{});
        }
        if (swap) {
            // the pivoted kernels read D from memory: write it unless already stored
            if (FORM && !A.form.store)
                for (int idx = lane; idx < P * nb; idx += 32) dst_d[idx] = form_pair(fsrc, idx);
            __threadfence();
            __syncwarp();
            if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = (int)code;
            __syncwarp();
            continue;
        }
        // ---- store inv(D) in the device layout and the condition check
        double2* dst = reinterpret_cast<double2*>(A.Dinv + (j * A.s + k_st) * bsz);
        double fsq2 = 0.0;
        if constexpr (EXACT) {
#pragma unroll
            for (int e = 0; e < (NPAIR + 31) / 32; ++e) {
                const int idx = lane + 32 * e;
                if (NPAIR % 32 == 0 || idx < NPAIR) {
                    const int p2 = idx / NBT, r = idx - p2 * NBT;
                    const double2 v = *reinterpret_cast<const double2*>(X + sw(r, 2 * p2));
                    fsq2 = fma(v.x, v.x, fma(v.y, v.y, fsq2));
                    dst[idx] = v;
                }
            }
        } else {
            for (int idx = lane; idx < P * nb; idx += 32) {
                const int p2 = idx / nb, r = idx - p2 * nb;
                double2 v = *reinterpret_cast<const double2*>(X + sw(r, 2 * p2));
                if (2 * p2 + 1 >= nb) v.y = 0.0;
                fsq2 = fma(v.x, v.x, fma(v.y, v.y, fsq2));
                dst[idx] = v;
            }
        }
        // cond_1 = |D|_1 |D^-1|_1 <= nb |D|_F |D^-1|_F: blocks whose Frobenius bound is already
        // <= 1e14 (all but pathological ones) skip the two exact column-norm passes (240 of ~1900
        // shared-memory wavefronts per nb = 40 block); the others get the exact check of
        // numba_backend.py:33-40 -- D is loaded again, the inverse is already in global memory
        double fa = fsq1, fb = fsq2;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            fa += __shfl_xor_sync(0xffffffffu, fa, o);
            fb += __shfl_xor_sync(0xffffffffu, fb, o);
        }
        bool cond_bad = false;
        if (!((double)nb * sqrt(fa) * sqrt(fb) <= 1e14)) {
            const double n2 = col_norm();
            __syncwarp();
            load_block();
            __syncwarp();
            const double n1 = col_norm();
            cond_bad = !(n1 * n2 <= 1e14);
        }
        double logdet = 0.0;
#pragma unroll
        for (int h = 0; h < (NBT + 31) / 32; ++h) logdet += log(apiv[h]);
#pragma unroll
        for (int o = 16; o; o >>= 1) logdet += __shfl_xor_sync(0xffffffffu, logdet, o);
        if (lane == 0) {
            const double det = exp(logdet);
            const bool bad = det == 0.0 || !isfinite(det) || cond_bad;
            if (bad) atomicMin(A.fail_key, (unsigned long long)code);
        }
        __syncwarp();
    }
}

template <int NT, bool EXACT, bool FORM, bool BG>
static int launch_tc_r(const irk_ctx* ctx, const InvArgs& A, int* fb_list, int* fb_count, cudaStream_t st) {
    using C = InvTcCfg<NT>;
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_inverse_tc<NT, EXACT, FORM, BG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem));
        IRK_CK(cudaFuncSetAttribute(k_inverse_tc<NT, EXACT, FORM, BG>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr = true;
    }
    const int threads = 32 * C::WARPS;
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inverse_tc<NT, EXACT, FORM, BG>, threads, C::smem));
    if (A.cap_per_sm > 0) per_sm = std::min(per_sm, A.cap_per_sm);
    const int64_t need = (A.ntasks + C::WARPS - 1) / C::WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->num_sms * std::max(per_sm, 1)));
    k_inverse_tc<NT, EXACT, FORM, BG><<<grid, threads, C::smem, st>>>(A, fb_list, fb_count);
    IRK_LAUNCHED();
    return IRK_OK;
}

template <int NT, bool EXACT, bool FORM>
static int launch_tc_t(const irk_ctx* ctx, const InvArgs& A, int* fb_list, int* fb_count, cudaStream_t st) {
    // A/B switch: the scalar-panel variant is instantiated for the config-1 tile count only
    // (nb 33..40) to bound build time.  (Two further variants were measured at config 1 and
    // dropped: two blocks per warp with the two pivot tiles eliminated side by side -- fewer
    // instructions but half the warps, 0.71-0.78 ms per level; the block held in registers in
    // the C-fragment layout -- half the shared-memory wavefronts but 12 warps per SM, 0.55-0.63
    // ms.  This kernel: 0.57-0.58 ms, the scalar-panel variant 0.69-0.70 ms.)
    static const bool scalar_panel = getenv("IRK_INV_BG") && atoi(getenv("IRK_INV_BG")) == 0;
    if constexpr (NT == 5)
        if (scalar_panel) return launch_tc_r<NT, EXACT, FORM, false>(ctx, A, fb_list, fb_count, st);
    return launch_tc_r<NT, EXACT, FORM, true>(ctx, A, fb_list, fb_count, st);
}

template <int NT>
static int launch_tc_n(const irk_ctx* ctx, const InvArgs& A, int* fb_list, int* fb_count, cudaStream_t st) {
    const bool form = A.form.J != nullptr;
    if (A.nb == 8 * NT)
        return form ? launch_tc_t<NT, true, true>(ctx, A, fb_list, fb_count, st)
                    : launch_tc_t<NT, true, false>(ctx, A, fb_list, fb_count, st);
    return form ? launch_tc_t<NT, false, true>(ctx, A, fb_list, fb_count, st)
                : launch_tc_t<NT, false, false>(ctx, A, fb_list, fb_count, st);
}

static int launch_pivoted(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st);

// tensor-core pass, then the pivoted kernels over the blocks it handed back
// (their count stays on the device: the fallback launch reads it)
// optimistic: no counter reset and no pivoted pass here -- the caller resets the counter once,
// lets the handed-back blocks of all launches pile up in the list and checks the count at the end
static int launch_tc(const irk_ctx* ctx, const InvArgs& A, int* fb, cudaStream_t st, bool optimistic = false) {
    int* fb_count = fb;
    int* fb_list = fb + 1;
    if (!optimistic) IRK_CK(cudaMemsetAsync(fb_count, 0, sizeof(int), st));
    const int nt = (A.nb + 7) / 8;
    int rc;
    switch (nt) {
        case 3: rc = launch_tc_n<3>(ctx, A, fb_list, fb_count, st); break;
        case 4: rc = launch_tc_n<4>(ctx, A, fb_list, fb_count, st); break;
        case 5: rc = launch_tc_n<5>(ctx, A, fb_list, fb_count, st); break;
        case 6: rc = launch_tc_n<6>(ctx, A, fb_list, fb_count, st); break;
        case 7: rc = launch_tc_n<7>(ctx, A, fb_list, fb_count, st); break;
        case 8: rc = launch_tc_n<8>(ctx, A, fb_list, fb_count, st); break;
        default: return IRK_EINVAL;
    }
    if (rc) return rc;
    if (optimistic) return IRK_OK;
    InvArgs B = A;
    B.tasks = fb_list;
    B.ntasks_dev = fb_count;
    B.form = InvForm{};
    return launch_pivoted(ctx, B, st);
}

// returns IRK_EINVAL if nb has no warp-inverse specialisation (caller falls back)
int launch_inverse(const irk_ctx* ctx, const int32_t* tasks, int64_t ntasks, int64_t T, int s, int nb,
                   const double* D, double* Dinv, unsigned long long* fail_key, int* fb, cudaStream_t st,
                   int cap_per_sm, const InvForm* form, bool optimistic) {
    if (ntasks <= 0) return IRK_OK;
    InvArgs A{tasks, ntasks, T, s, nb, D, Dinv, fail_key, nullptr, cap_per_sm, InvForm{}};
    static const bool tc_off = getenv("IRK_INV_TC") && atoi(getenv("IRK_INV_TC")) == 0;
    if (fb && !tc_off && nb > 16 && nb <= 64) {
        if (form) A.form = *form;
        return launch_tc(ctx, A, fb, st, optimistic);
    }
    if (form) return IRK_EINVAL;   // forming D needs the tensor-core path (caller runs the Schur phase)
    return launch_pivoted(ctx, A, st);
}

static int launch_pivoted(const irk_ctx* ctx, const InvArgs& A, cudaStream_t st) {
    const int nb = A.nb;
    if (nb <= 8) return launch3<8>(ctx, A, st);
    if (nb <= 16) return launch3<16>(ctx, A, st);
    if (nb <= 24) return launch3<24>(ctx, A, st);
    if (nb <= 32) return launch3<32>(ctx, A, st);
    if (nb <= 40) return launch4(ctx, A, st);
    if (nb == 50) return launch2<50>(ctx, A, st);
    if (nb <= 64) return launch_t<64, false>(ctx, A, st);
    return IRK_EINVAL;
}

}  // namespace irk
