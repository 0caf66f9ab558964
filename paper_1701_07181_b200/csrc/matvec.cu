// Fused transformed stage operator:
//   y_k = alpha * J_k w_k + sum_l mix[k][l] * (M w_l),   k = 0..s-1
// (reference StageOperator.matvec, stage_system.py:52-70, which does s
// Jacobian sweeps plus s^2 mass sweeps; here every J block and every M block
// is read from HBM exactly once per call and applied to all s stage vectors,
// and the s x s mixing is fused into the epilogue).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "blockops.cuh"
#include "irk_internal.cuh"
#include "pipeline.cuh"

namespace irk {

int choose_groups(int nb, int max_threads);  // defined below

struct MixParams {
    double c[IRK_MAX_STAGES * IRK_MAX_STAGES];
};

struct MatvecArgs {
    const int32_t* indptr;
    const int32_t* indices;
    const double* J[IRK_MAX_STAGES];   // per-stage block base (already offset by jfirst)
    const double* M;                   // NULL: no mass term
    const double* w;
    double* y;
    const double* ghost;               // halo values (s, n_ghost, nb) or NULL
    const int32_t* rows;               // row subset or NULL (all rows)
    int64_t nrows;
    int64_t row_lo, row_hi;            // pipelined kernel: contiguous row range
    int64_t n;                         // T_local * nb (stage stride of w, y)
    int64_t T_local;
    int64_t n_ghost;
    double alpha;
    int nb, G;
};

template <int S, bool SHARED, bool EVEN>
__global__ void __launch_bounds__(512) k_stage_matvec(MatvecArgs A, MixParams C) {
    extern __shared__ double red[];
    const Geo q = make_geo(A.nb, A.G);
    const int64_t bsz = (int64_t)A.nb * 2 * q.P;
    for (int64_t t = blockIdx.x; t < A.nrows; t += gridDim.x) {
        const int64_t i = A.rows ? A.rows[t] : t;
        double part[2 * S];
#pragma unroll
        for (int v = 0; v < 2 * S; ++v) part[v] = 0.0;
        if (q.active) {
            const int q0 = A.indptr[i], q1 = A.indptr[i + 1];
            for (int qq = q0; qq < q1; ++qq) {
                const int64_t col = A.indices[qq];
                const double* xs[S];
#pragma unroll
                for (int r = 0; r < S; ++r)
                    xs[r] = col < A.T_local ? A.w + r * A.n + col * A.nb
                                            : A.ghost + (r * A.n_ghost + (col - A.T_local)) * A.nb;
                if (SHARED) {
                    gemv_shared<S, EVEN, false>(A.J[0] + qq * bsz, xs, q, part);
                } else {
#pragma unroll
                    for (int r = 0; r < S; ++r)
                        part[r] = gemv1<EVEN, false>(A.J[r] + qq * bsz, xs[r], q, part[r]);
                }
            }
            if (A.M) {
                const double* xs[S];
#pragma unroll
                for (int r = 0; r < S; ++r) xs[r] = A.w + r * A.n + i * A.nb;
                gemv_shared<S, EVEN, false>(A.M + i * bsz, xs, q, part + S);
            }
        }
        double tot[2 * S];
        group_reduce(red, part, 2 * S, q, tot);
        if (q.active && q.g == 0) {
#pragma unroll
            for (int k = 0; k < S; ++k) {
                double acc = A.alpha * tot[k];
                if (A.M) {
#pragma unroll
                    for (int l = 0; l < S; ++l) acc += C.c[k * S + l] * tot[S + l];
                }
                A.y[k * A.n + i * A.nb + q.a] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised bulk-copy pipeline version (nb even, all rows).
// Warp 0 lane 0 is the producer: for the CTA's contiguous row range it streams
// every block of the row (J blocks in pattern order, then M_i) together with
// the x segments that block multiplies (s segments of nb doubles) into a ring
// of shared-memory stages with cp.async.bulk, completing on the stage's full
// mbarrier.  Warps 1.. are consumers: thread (g, a) multiplies row a of the
// staged block with the staged x pairs of its column pairs p = g (mod G) --
// 128-bit conflict-free LDS for the block, broadcast LDS for x -- and releases
// the stage on its empty mbarrier.  Row ends reduce the G groups through
// shared memory under a consumer-only named barrier.
// ---------------------------------------------------------------------------
struct PipeGeom {
    int nst;            // stages
    int stage_bytes;    // block + x segments, 128-B aligned
    int block_bytes;
    int seg_bytes;      // nb * 8
    int nseg;           // x segments per item (S shared, 1 distinct)
};

template <int S, bool SHARED>
__global__ void __launch_bounds__(288) k_stage_matvec_pipe(MatvecArgs A, MixParams C, PipeGeom PG) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* stages = smem_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)PG.nst * PG.stage_bytes);
    uint64_t* empty = full + PG.nst;
    double* red = reinterpret_cast<double*>(empty + PG.nst);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncons_warps = (blockDim.x >> 5) - 1;
    const int64_t T = A.row_hi - A.row_lo;
    const int64_t r0 = A.row_lo + T * blockIdx.x / gridDim.x, r1 = A.row_lo + T * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < PG.nst; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, ncons_warps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    griddep_launch();
    griddep_wait();   // PDL: pipeline set up during the predecessor's drain
    const int nb = A.nb;
    const int64_t bsz = (int64_t)PG.block_bytes / 8;
    if (warp == 0) {
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            auto push = [&](const double* blk, const double* const* segs, int nseg) {
                mbar_wait(empty + st, ph ^ 1);
                unsigned char* dst = stages + (size_t)st * PG.stage_bytes;
                mbar_expect_tx(full + st, PG.block_bytes + nseg * PG.seg_bytes);
                bulk_g2s(dst, blk, PG.block_bytes, full + st);
                for (int r = 0; r < nseg; ++r)
                    bulk_g2s(dst + PG.block_bytes + r * PG.seg_bytes, segs[r], PG.seg_bytes, full + st);
                if (++st == PG.nst) { st = 0; ph ^= 1; }
            };
            for (int64_t i = r0; i < r1; ++i) {
                const int q0 = A.indptr[i], q1 = A.indptr[i + 1];
                for (int qq = q0; qq < q1; ++qq) {
                    const int64_t col = A.indices[qq];
                    const double* xs[S];
#pragma unroll
                    for (int r = 0; r < S; ++r)
                        xs[r] = col < A.T_local ? A.w + r * A.n + col * nb
                                                : A.ghost + (r * A.n_ghost + (col - A.T_local)) * nb;
                    if (SHARED) {
                        push(A.J[0] + qq * bsz, xs, S);
                    } else {
#pragma unroll
                        for (int r = 0; r < S; ++r) push(A.J[r] + qq * bsz, xs + r, 1);
                    }
                }
                if (A.M) {
                    const double* xs[S];
#pragma unroll
                    for (int r = 0; r < S; ++r) xs[r] = A.w + r * A.n + i * nb;
                    push(A.M + i * bsz, xs, S);
                }
            }
        }
        return;
    }
    // ---- consumers
    const int c = threadIdx.x - 32;
    Geo q;
    q.nb = nb;
    q.P = (nb + 1) >> 1;
    q.G = A.G;
    q.g = c / nb;
    q.a = c - q.g * nb;
    q.active = q.g < q.G;
    const int ncons = ncons_warps * 32;
    int st = 0;
    uint32_t ph = 0;
    auto consume = [&](auto&& fn) {
        mbar_wait(full + st, ph);
        const unsigned char* base = stages + (size_t)st * PG.stage_bytes;
        if (q.active) fn(reinterpret_cast<const double2*>(base),
                         reinterpret_cast<const double*>(base + PG.block_bytes));
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == PG.nst) { st = 0; ph ^= 1; }
    };
    for (int64_t i = r0; i < r1; ++i) {
        double part[2 * S];
#pragma unroll
        for (int v = 0; v < 2 * S; ++v) part[v] = 0.0;
        const int q0 = A.indptr[i], q1 = A.indptr[i + 1];
        for (int qq = q0; qq < q1; ++qq) {
            if (SHARED) {
                consume([&](const double2* B, const double* X) {
                    for (int p = q.g; p < q.P; p += q.G) {
                        const double2 b = B[p * nb + q.a];
#pragma unroll
                        for (int r = 0; r < S; ++r) {
                            const double2 x = *reinterpret_cast<const double2*>(X + r * nb + 2 * p);
                            part[r] = fma(b.x, x.x, part[r]);
                            part[r] = fma(b.y, x.y, part[r]);
                        }
                    }
                });
            } else {
#pragma unroll
                for (int r = 0; r < S; ++r)
                    consume([&](const double2* B, const double* X) {
                        for (int p = q.g; p < q.P; p += q.G) {
                            const double2 b = B[p * nb + q.a];
                            const double2 x = *reinterpret_cast<const double2*>(X + 2 * p);
                            part[r] = fma(b.x, x.x, part[r]);
                            part[r] = fma(b.y, x.y, part[r]);
                        }
                    });
            }
        }
        if (A.M)
            consume([&](const double2* B, const double* X) {
                for (int p = q.g; p < q.P; p += q.G) {
                    const double2 b = B[p * nb + q.a];
#pragma unroll
                    for (int r = 0; r < S; ++r) {
                        const double2 x = *reinterpret_cast<const double2*>(X + r * nb + 2 * p);
                        part[S + r] = fma(b.x, x.x, part[S + r]);
                        part[S + r] = fma(b.y, x.y, part[S + r]);
                    }
                }
            });
        // reduce the G groups (consumer-only named barrier 1)
        if (q.active)
#pragma unroll
            for (int v = 0; v < 2 * S; ++v) red[(q.g * 2 * S + v) * nb + q.a] = part[v];
        consumer_sync(1, ncons);
        if (q.active && q.g == 0) {
            double tot[2 * S];
#pragma unroll
            for (int v = 0; v < 2 * S; ++v) {
                double sum = 0.0;
                for (int gg = 0; gg < q.G; ++gg) sum += red[(gg * 2 * S + v) * nb + q.a];
                tot[v] = sum;
            }
#pragma unroll
            for (int k = 0; k < S; ++k) {
                double acc = A.alpha * tot[k];
                if (A.M) {
#pragma unroll
                    for (int l = 0; l < S; ++l) acc += C.c[k * S + l] * tot[S + l];
                }
                A.y[k * A.n + i * nb + q.a] = acc;
            }
        }
        consumer_sync(1, ncons);
    }
}

template <int S, bool SHARED>
static int launch_pipe(const irk_stage_op* op, MatvecArgs& A, const MixParams& C, cudaStream_t st) {
    const int nb = A.nb;
    PipeGeom PG;
    PG.block_bytes = (int)(block_doubles(nb) * 8);
    PG.seg_bytes = nb * 8;
    PG.nseg = SHARED ? S : 1;
    PG.stage_bytes = ((PG.block_bytes + PG.nseg * PG.seg_bytes) + 127) & ~127;
    const int cons_threads = ((A.G * nb + 31) / 32) * 32;
    const int threads = 32 + cons_threads;
    const size_t red_bytes = sizeof(double) * A.G * 2 * S * nb;
    // ring budget per CTA: about two stages' worth of consumer work per S vectors -- small
    // blocks / few vectors run best as many small CTAs (config 3: nb=24 67% -> 96% of peak),
    // the s=3 nb=40 benchmark operator with ~7 stages per CTA (tools/sweep.py config3)
    static const int budget_kb = getenv("IRK_MATVEC_BUDGET_KB") ? atoi(getenv("IRK_MATVEC_BUDGET_KB")) : 0;   // tuning knob
    const size_t budget = budget_kb > 0 ? (size_t)budget_kb * 1024
                                        : std::min<size_t>(100 * 1024, std::max<size_t>(20 * 1024, (size_t)2 * S * PG.stage_bytes));
    PG.nst = (int)std::max<size_t>(2, std::min<size_t>(16, (budget - red_bytes) / PG.stage_bytes));
    const size_t smem = (size_t)PG.nst * PG.stage_bytes + 2 * sizeof(uint64_t) * PG.nst + red_bytes;
    static bool attr = false;
    if (!attr) {
        IRK_CK(cudaFuncSetAttribute(k_stage_matvec_pipe<S, SHARED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)std::min<size_t>(op->ctx->smem_optin, 200 * 1024)));
        attr = true;
    }
    int per_sm = 1;
    IRK_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stage_matvec_pipe<S, SHARED>, threads, smem));
    if (A.row_hi <= A.row_lo) return IRK_OK;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(A.row_hi - A.row_lo, (int64_t)op->ctx->num_sms * std::max(per_sm, 1)));
    IRK_CK(launch_pdl(k_stage_matvec_pipe<S, SHARED>, dim3((unsigned)grid), dim3(threads), smem, st, A, C, PG));
    IRK_LAUNCHED();
    return IRK_OK;
}

int choose_groups(int nb, int max_threads) {
    const int P = (nb + 1) / 2;
    int best = 1;
    double best_eff = -1.0;
    for (int G = 1; G <= P && G * nb <= max_threads; ++G) {
        const int thr = G * nb;
        const int warps = (thr + 31) / 32;
        const double e1 = (double)thr / (warps * 32);
        const int per = (P + G - 1) / G;
        const double e2 = (double)P / (G * per);
        // prefer more threads when efficiency ties (more memory parallelism)
        const double eff = e1 * e2 + 1e-4 * G;
        if (eff > best_eff) { best_eff = eff; best = G; }
    }
    return best;
}

template <int S, bool SHARED, bool EVEN>
static int launch_t(const irk_stage_op* op, MatvecArgs& A, const MixParams& C, cudaStream_t st) {
    const int threads = ((A.G * A.nb + 31) / 32) * 32;
    const size_t smem = sizeof(double) * A.G * 2 * S * A.nb;
    const int64_t grid = std::min<int64_t>(A.nrows, (int64_t)op->ctx->num_sms * 16);
    if (grid <= 0) return IRK_OK;
    k_stage_matvec<S, SHARED, EVEN><<<(int)grid, threads, smem, st>>>(A, C);
    IRK_LAUNCHED();
    return IRK_OK;
}

template <int S>
static int launch_s(const irk_stage_op* op, MatvecArgs& A, const MixParams& C, cudaStream_t st) {
    const bool even = (A.nb % 2) == 0;
    if (even && A.rows == nullptr && S <= 4 && A.G * A.nb <= 256)
        return op->shared_j ? launch_pipe<S, true>(op, A, C, st) : launch_pipe<S, false>(op, A, C, st);
    if (op->shared_j) return even ? launch_t<S, true, true>(op, A, C, st) : launch_t<S, true, false>(op, A, C, st);
    return even ? launch_t<S, false, true>(op, A, C, st) : launch_t<S, false, false>(op, A, C, st);
}

int stage_op_apply_rows(const irk_stage_op* op, const double* w, double* y, const int32_t* rows,
                        int64_t nrows, cudaStream_t st, int64_t row_lo = 0, int64_t row_hi = -1) {
    MatvecArgs A{};
    A.row_lo = row_lo;
    A.row_hi = row_hi < 0 ? op->T_local : row_hi;
    A.indptr = op->pat->d_indptr;
    A.indices = op->pat->d_indices;
    for (int k = 0; k < op->s; ++k) A.J[k] = op->J[k]->d + op->jfirst[k] * block_doubles(op->nb);
    A.M = op->M ? op->M->d : nullptr;
    A.w = w;
    A.y = y;
    A.ghost = op->ghost;
    A.rows = rows;
    A.nrows = nrows;
    A.T_local = op->T_local;
    A.n = op->T_local * op->nb;
    A.n_ghost = op->n_ghost;
    A.alpha = op->alpha;
    A.nb = op->nb;
    A.G = choose_groups(op->nb, 256);
    MixParams C{};
    for (int e = 0; e < op->s * op->s; ++e) C.c[e] = op->C[e];
    switch (op->s) {
        case 1: return launch_s<1>(op, A, C, st);
        case 2: return launch_s<2>(op, A, C, st);
        case 3: return launch_s<3>(op, A, C, st);
        case 4: return launch_s<4>(op, A, C, st);
        case 5: return launch_s<5>(op, A, C, st);
        default: set_error("stage count > 5 not supported by the fused matvec"); return IRK_EINVAL;
    }
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_stage_op_create(irk_ctx* ctx, const irk_pattern* pat, int s, const irk_blocks* const* J,
                        const int64_t* jfirst, const irk_blocks* M, const double* mix,
                        double alpha, irk_stage_op** out) {
    IRK_ARG(ctx && pat && J && out, "NULL argument");
    IRK_ARG(s >= 1 && s <= 5, "stage count must be in [1, 5]");
    auto* op = new irk_stage_op();
    op->ctx = ctx;
    op->pat = pat;
    op->s = s;
    op->nb = J[0]->nb;
    op->alpha = alpha;
    op->shared_j = true;
    for (int k = 0; k < s; ++k) {
        if (!J[k] || J[k]->nb != op->nb) { delete op; set_error("J blocks missing or nb mismatch"); return IRK_EINVAL; }
        op->J[k] = J[k];
        op->jfirst[k] = jfirst ? jfirst[k] : 0;
        if (op->jfirst[k] < 0 || op->jfirst[k] + pat->nnzb > J[k]->count) {
            delete op; set_error("J block range out of bounds"); return IRK_EINVAL;
        }
        if (J[k] != J[0] || op->jfirst[k] != op->jfirst[0]) op->shared_j = false;
    }
    op->M = M;
    if (M && (M->nb != op->nb || M->count < pat->T)) { delete op; set_error("mass blocks mismatch"); return IRK_EINVAL; }
    if (M) {
        if (!mix) { delete op; set_error("mix coefficients required with M"); return IRK_EINVAL; }
        for (int e = 0; e < s * s; ++e) op->C[e] = mix[e];
    }
    op->T_local = pat->T;
    *out = op;
    return IRK_OK;
}

void irk_stage_op_destroy(irk_stage_op* op) { delete op; }

int irk_stage_op_set_halo(irk_stage_op* op, int64_t T_local, const double* ghost, int64_t n_ghost) {
    IRK_ARG(op, "NULL op");
    IRK_ARG(T_local >= 1 && T_local <= op->pat->T, "T_local out of range");
    IRK_ARG(n_ghost >= 0 && (n_ghost == 0 || ghost), "ghost buffer missing");
    IRK_ARG(!op->M || op->M->count >= T_local, "mass blocks mismatch");
    op->T_local = T_local;
    op->ghost = ghost;
    op->n_ghost = n_ghost;
    return IRK_OK;
}

int irk_stage_op_apply(const irk_stage_op* op, const double* w, double* y, void* stream) {
    IRK_ARG(op && w && y, "NULL argument");
    return stage_op_apply_rows(op, w, y, nullptr, op->T_local, (cudaStream_t)stream);
}

int irk_stage_op_apply_range(const irk_stage_op* op, const double* w, double* y, int64_t row_lo, int64_t row_hi,
                             void* stream) {
    IRK_ARG(op && w && y, "NULL argument");
    IRK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= op->T_local, "row range out of bounds");
    if (row_hi == row_lo) return IRK_OK;
    const bool pipe_ok = op->nb % 2 == 0 && op->s <= 4 && choose_groups(op->nb, 256) * op->nb <= 256;
    if (pipe_ok) return stage_op_apply_rows(op, w, y, nullptr, row_hi - row_lo, (cudaStream_t)stream, row_lo, row_hi);
    // generic kernel: an explicit row list
    int32_t* d = nullptr;
    std::vector<int32_t> rows(row_hi - row_lo);
    for (int64_t r = row_lo; r < row_hi; ++r) rows[r - row_lo] = (int32_t)r;
    cudaStream_t st = (cudaStream_t)stream;
    IRK_CK(cudaMallocAsync(&d, sizeof(int32_t) * rows.size(), st));
    IRK_CK(cudaMemcpyAsync(d, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice, st));
    const int rc = stage_op_apply_rows(op, w, y, d, (int64_t)rows.size(), st);
    IRK_CK(cudaStreamSynchronize(st));   // host row list goes out of scope
    cudaFreeAsync(d, st);
    return rc;
}

int irk_stage_op_apply_rows(const irk_stage_op* op, const double* w, double* y, const int32_t* rows, int64_t nrows,
                            void* stream) {
    IRK_ARG(op && w && y && (rows || nrows == 0), "NULL argument");
    if (nrows == 0) return IRK_OK;
    return stage_op_apply_rows(op, w, y, rows, nrows, (cudaStream_t)stream);
}

}  // extern "C"
