/*
 * irkb200.h -- C ABI of the B200-native linear-solve hot path of the
 * transformed implicit Runge-Kutta method (Pazner & Persson, arXiv 1701.07181).
 *
 * libirkb200.so implements, in hand-written sm_100a CUDA:
 *   - the transformed stage operator  B = A^-1 (x) M - dt blkdiag(J_1..J_s)
 *     (reference: /root/reference/pkg/src/irksolve/stage_system.py:52-70),
 *   - block ILU(0): plain/shifted-uncoupled (precond.py:90-110, 244-280) and
 *     stage-coupled (precond.py:165-200), factorisation and apply,
 *   - left-preconditioned restarted GMRES (krylov.py:37-130) with fused
 *     classical Gram-Schmidt,
 *   - host-pointer shims with exactly the argument meaning of the reference's
 *     kernel-plugin protocol (kernels/numba_backend.py:21-151), so the library
 *     can be installed as ``irksolve.kernels._backend``.
 *
 * Conventions: every function returns an int status -- IRK_OK (0), a
 * positive status for a numerically singular pivot (IRK_ESINGULAR, with the
 * failing stage/element in out-params, the reference's SingularPivotError,
 * precond.py:16-23), or a negative error with a message in irk_last_error().
 * Plain pointers and sizes only; device pointers are CUDA global memory,
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Vectors are
 * stage-major then element-major fp64 (stage_system.py:6-7); block inputs are
 * row-major m x m fp64 and CSR-of-blocks indices are int64, as the reference
 * stores them (blocks.py:59-74).
 */
#ifndef IRKB200_H
#define IRKB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define IRK_API __attribute__((visibility("default")))
#else
#define IRK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define IRK_OK 0
#define IRK_ESINGULAR 1
#define IRK_EINVAL (-1)
#define IRK_ECUDA (-2)
#define IRK_ENOMEM (-3)
#define IRK_ECALLBACK (-4)

#define IRK_MAX_STAGES 8
#define IRK_MAX_NB 128

#define IRK_FACTOR_UNCOUPLED 0
#define IRK_FACTOR_COUPLED 1

typedef struct irk_ctx irk_ctx;
typedef struct irk_pattern irk_pattern;
typedef struct irk_blocks irk_blocks;
typedef struct irk_stage_op irk_stage_op;
typedef struct irk_factor irk_factor;
typedef struct irk_comm irk_comm;
typedef struct irk_halo irk_halo;
typedef struct irk_dist_op irk_dist_op;

/* ---- library / context ------------------------------------------------ */
IRK_API int irk_version(void);
IRK_API const char *irk_last_error(void);
/* number of CUDA kernels this library has launched in the process */
IRK_API int64_t irk_launch_count(void);
IRK_API int irk_ctx_create(int device, irk_ctx **out);
IRK_API void irk_ctx_destroy(irk_ctx *ctx);

/* ---- block pattern: reference BlockSparseMatrix.indptr/indices/diag_pos
 *      (blocks.py:59-74); sorted columns per row, diagonal present --------- */
IRK_API int irk_pattern_create(irk_ctx *ctx, int64_t T, const int64_t *indptr, const int64_t *indices,
                       const int64_t *diag_pos, irk_pattern **out);
IRK_API void irk_pattern_destroy(irk_pattern *pat);

/* ---- arrays of nb x nb fp64 blocks in device layout ---------------------- */
IRK_API int irk_blocks_create(irk_ctx *ctx, int nb, int64_t count, irk_blocks **out);
IRK_API void irk_blocks_destroy(irk_blocks *b);
/* copy `count` row-major blocks from `src` (host, or device if src_on_device)
 * into blocks [first, first+count) */
IRK_API int irk_blocks_upload(irk_blocks *b, int64_t first, int64_t count, const double *src,
                      int src_on_device, void *stream);
IRK_API int irk_blocks_download(const irk_blocks *b, int64_t first, int64_t count, double *dst,
                        int dst_on_device, void *stream);

/* ---- stage operator --------------------------------------------------------
 * y_k = alpha * J_k w_k + sum_l mix[k*s+l] * (M w_l)      k = 0..s-1
 * With alpha = -dt and mix = A^-1 this is StageOperator.matvec
 * (stage_system.py:52-70); with s=1, alpha=1, M=NULL it is bsr_matvec
 * (numba_backend.py:21-30); with s=1, mix={coef}, alpha=-dt it is the matvec of
 * build_stage_matrix(coef, M, J, dt) (precond.py:48-54).
 * J[k] (k<s) may repeat one object (shared Jacobian, read once per row);
 * jfirst[k] is the first block of stage k inside J[k] (NULL = 0). */
IRK_API int irk_stage_op_create(irk_ctx *ctx, const irk_pattern *pat, int s, const irk_blocks *const *J,
                        const int64_t *jfirst, const irk_blocks *M, const double *mix,
                        double alpha, irk_stage_op **out);
IRK_API void irk_stage_op_destroy(irk_stage_op *op);
IRK_API int irk_stage_op_apply(const irk_stage_op *op, const double *w, double *y, void *stream);
/* Rows [row_lo, row_hi) of y = B w (the rest of y untouched): the interior rows of a
 * slab, computed while its halo is in flight (multi-GPU). */
IRK_API int irk_stage_op_apply_range(const irk_stage_op *op, const double *w, double *y, int64_t row_lo,
                                     int64_t row_hi, void *stream);
/* Rows rows[0..nrows) (device int32 list) of y = B w: the slab's boundary rows. */
IRK_API int irk_stage_op_apply_rows(const irk_stage_op *op, const double *w, double *y, const int32_t *rows,
                                    int64_t nrows, void *stream);
/* element-partitioned operator: rows [0,T_local) of the pattern are local,
 * column indices >= T_local address `ghost` ((s, n_ghost, nb) device array) */
IRK_API int irk_stage_op_set_halo(irk_stage_op *op, int64_t T_local, const double *ghost, int64_t n_ghost);

/* ---- block ILU(0) -----------------------------------------------------------
 * Stage matrix k: B_k = coef[k] * M + alpha * J_k on J's pattern (alpha=-dt:
 * build_stage_matrix, precond.py:48-54; M=NULL, alpha=1: B_k = J_k as given).
 * keep: host uint8[nnzb] (NULL = all) -- partition_keep_mask (precond.py:26-45).
 * simplified: Alg. 2 sweep (1) or general Alg. 1 with fill-limited updates (0)
 * (numba_backend.py:43-72).  store_diag keeps the updated pivots for export.
 * Returns IRK_ESINGULAR with the first failing (stage, element) in
 * stage-major order, like SingularPivotError(element, stage). */
IRK_API int irk_factor_uncoupled(irk_ctx *ctx, const irk_pattern *pat, int s, const irk_blocks *const *J,
                         const int64_t *jfirst, const irk_blocks *M, const double *coef,
                         double alpha, const uint8_t *keep, int simplified, int store_diag,
                         irk_factor **out, int64_t *fail_stage, int64_t *fail_elem, void *stream);
/* Stage-coupled ILU(0), Alg. 3 (numba_backend.py:94-125): stage diagonals
 * a_inv[k][k]*M + alpha*J_k, cross-stage blocks a_inv[k][l]*M_i, or the
 * explicit `coupling` array ((s*s*T) blocks, index (k*s+l)*T+i) when given.
 * literal selects the printed update B_ll -= G_lk B_kk (numba_backend.py:120-123). */
IRK_API int irk_factor_coupled(irk_ctx *ctx, const irk_pattern *pat, int s, const irk_blocks *const *J,
                       const int64_t *jfirst, const irk_blocks *M, const double *a_inv,
                       double alpha, const irk_blocks *coupling, const uint8_t *keep,
                       int literal, int store_diag, irk_factor **out, int64_t *fail_stage,
                       int64_t *fail_elem, void *stream);
/* Re-factorise in place with new numeric values on the same structure
 * (pattern, keep mask, kind, stage count, explicit/implicit couplings):
 * coef = per-stage diagonal coefficients (uncoupled) or a_inv (coupled).
 * Reuses all device buffers and schedules (one Newton iteration's factor). */
IRK_API int irk_factor_refactor(irk_factor *f, const irk_blocks *const *J, const int64_t *jfirst,
                                const irk_blocks *M, const double *coef, double alpha,
                                const irk_blocks *coupling, int64_t *fail_stage, int64_t *fail_elem,
                                void *stream);
IRK_API void irk_factor_destroy(irk_factor *f);
/* x = P^-1 y for all s stages, (s,T,nb) device vectors (BlockIlu0.apply /
 * StageUncoupledIlu0.apply / StageCoupledIlu0.apply, precond.py:79-87,
 * 222-241, 152-162).  x may alias nothing else; y is not modified. */
IRK_API int irk_factor_apply(const irk_factor *f, const double *y, double *x, void *stream);
/* x = P^-1 (B v): one Arnoldi product of the left-preconditioned GMRES loop
 * (krylov.py:88-89: apply_precond(apply_operator(v))) with B the stage operator
 * (stage_system.py:52-70) and P the factor.  When the factor is the uncoupled
 * implicit-L ILU(0) of the operator's own Jacobian blocks on a colour schedule,
 * the matvec runs inside the forward sweep (each lower Jacobian block read once
 * for both products, B v never stored); otherwise the two calls run back to back
 * through a scratch vector.  *fused (optional) = 1 if the fused path ran.
 * irk_gmres takes the fused path itself for native (stage op, factor) pairs. */
IRK_API int irk_op_factor_apply(const irk_stage_op *op, const irk_factor *f, const double *v, double *x,
                                int *fused, void *stream);
/* One single-stage factor (s = 1, e.g. ilu0_factorize of J itself) applied to
 * nrhs stage-major right-hand sides y (nrhs, T, m) -> x in one sweep that reads
 * every factor block once (BASELINE config 3).  Same result as nrhs separate
 * irk_factor_apply calls (ilu0_solve, numba_backend.py:75-91, per column).
 * Needs even m, nrhs <= 4, m <= 256; IRK_EINVAL otherwise. */
IRK_API int irk_factor_apply_rhs(const irk_factor *f, int nrhs, const double *y, double *x, void *stream);
/* factor data in the reference's output layout (host, row-major):
 * fstage (s,nnzb,m,m): lower = L, diagonal = updated pivot, upper = U;
 * dinv (s,T,m,m); fcoupling (s,s,T,m,m) (coupled only, may be NULL).
 * Requires store_diag=1 at factorisation. */
IRK_API int irk_factor_export(const irk_factor *f, double *fstage, double *dinv, double *fcoupling,
                      void *stream);
IRK_API int irk_factor_levels(const irk_factor *f, int64_t *fwd_levels, int64_t *bwd_levels);
/* 1 if the factor keeps L implicit (L_ij = alpha J_ij Dinv_j is never stored;
 * uncoupled simplified ILU with one stage-shared J and a symmetric keep mask),
 * 0 if L is stored, <0 on error.  Results are the same either way. */
IRK_API int irk_factor_implicit_l(const irk_factor *f);

/* ---- GMRES ----------------------------------------------------------------- */
typedef int (*irk_apply_fn)(void *user, const double *in, double *out, void *stream);
typedef int (*irk_allreduce_fn)(void *user, double *buf_dev, int64_t count, void *stream);
typedef struct {
    irk_apply_fn fn;  /* NULL = identity */
    void *user;
} irk_linop;
typedef struct {
    double rel_tol;      /* GmresConfig.rel_tol (krylov.py:11) */
    int max_iters;       /* GmresConfig.max_iters */
    int restart;         /* <= 0: unrestarted */
    double reorth_eta;   /* CGS re-orthogonalisation threshold (DGKS); <=0: 1/sqrt(2) */
} irk_gmres_cfg;
typedef struct {
    int iterations;
    int operator_applies;
    int converged;
    int breakdown;
    int reorth_passes;
    int history_len;
    double b_norm;
    double final_true_residual;
} irk_gmres_stats;

IRK_API int irk_linop_stage_op(const irk_stage_op *op, irk_linop *out);
IRK_API int irk_linop_factor(const irk_factor *f, irk_linop *out);
/* Left-preconditioned restarted GMRES (krylov.py:37-130) on n local unknowns;
 * `allreduce` (may be NULL) sums small device arrays across ranks.  history
 * receives the residual history (capacity history_cap). */
IRK_API int irk_gmres(irk_ctx *ctx, int64_t n, irk_linop op, irk_linop pre, irk_allreduce_fn allreduce,
              void *ar_user, const double *rhs, double *x, const irk_gmres_cfg *cfg,
              irk_gmres_stats *stats, double *history, int history_cap, void *stream);

/* ---- fused Arnoldi primitives (classical Gram-Schmidt) --------------------
 * multidot: out[i] = V_i . w (i<nv), out[nv] = w . w          (device out)
 * update:   w -= sum_i h[i] V_i; out_nrm2[0] = w . w          (device h, out) */
IRK_API int irk_vec_multidot(irk_ctx *ctx, int64_t n, int nv, const double *V, int64_t ldv,
                     const double *w, double *out, void *stream);
IRK_API int irk_vec_update(irk_ctx *ctx, int64_t n, int nv, const double *V, int64_t ldv,
                   const double *h, double *w, double *out_nrm2, void *stream);

/* ---- element-partitioned (multi-GPU) layer ----------------------------------
 * The paper's parallel scheme: elements in P contiguous slabs
 * (partition, meshing.py:81-90), partitioned ILU(0) (precond.py:26-45, no
 * communication), a neighbour halo for the operator and summed GMRES inner
 * products.  One rank per GPU.  Replaces the reference's in-process partition
 * bookkeeping (precond.py:26-45 keep mask on one process); the reference has no
 * communication layer of its own.
 *
 * irk_comm: NCCL transport (libnccl.so.2 loaded at run time; the unique id is
 * produced on rank 0 and broadcast by the caller) or a host-callback transport
 * (host-staged exchange, e.g. for tests on one GPU).  irk_comm_allreduce has the
 * irk_allreduce_fn signature: pass it with user = the comm to irk_gmres. */
#define IRK_NCCL_ID_BYTES 128
/* move the packed send buffer ([stage][send element][nb], peers in creation
 * order, contiguous) to the peers and fill ghost ([stage][ghost][nb]) */
typedef int (*irk_halo_xfer_fn)(void *user, const double *send_dev, double *ghost_dev, void *stream);
IRK_API int irk_comm_nccl_available(void);
IRK_API int irk_comm_nccl_unique_id(unsigned char *id_out, int64_t cap);
IRK_API int irk_comm_create_nccl(irk_ctx *ctx, const unsigned char *id, int nranks, int rank, irk_comm **out);
IRK_API int irk_comm_create_callback(irk_ctx *ctx, int nranks, int rank, irk_halo_xfer_fn xfer,
                                     irk_allreduce_fn allreduce, void *user, irk_comm **out);
IRK_API void irk_comm_destroy(irk_comm *comm);
IRK_API int irk_comm_allreduce(void *comm, double *buf, int64_t count, void *stream);
/* halo of a stage-major (s, T_local, nb) vector: per peer, the local elements it
 * needs (send_elems, concatenated in peer order) and the contiguous ghost range
 * [recv_first, recv_first + recv_count) it fills (ghosts sorted by global id) */
IRK_API int irk_halo_create(irk_comm *comm, int s, int nb, int64_t T_local, int64_t n_ghost, int npeers,
                            const int32_t *peers, const int64_t *send_counts, const int64_t *send_elems,
                            const int64_t *recv_counts, const int64_t *recv_first, irk_halo **out);
IRK_API void irk_halo_destroy(irk_halo *h);
IRK_API int irk_halo_exchange(irk_halo *h, const double *x, double *ghost, void *stream);
/* the slab's rows of the stage operator (op after irk_stage_op_set_halo with the same
 * ghost buffer) as a GMRES operator: exchange overlapped with the interior rows
 * [interior_lo, interior_hi), then the boundary rows (host list) */
IRK_API int irk_dist_op_create(irk_stage_op *op, irk_halo *halo, double *ghost, int64_t interior_lo,
                               int64_t interior_hi, const int32_t *boundary_rows, int64_t nboundary,
                               irk_dist_op **out);
IRK_API void irk_dist_op_destroy(irk_dist_op *d);
IRK_API int irk_dist_op_apply(const irk_dist_op *d, const double *w, double *y, void *stream);
/* x = P^-1 (B v) with the distributed operator: exchange, then the fused Arnoldi
 * product over the slab's rows when the factor is the slab's partitioned implicit-L
 * ILU(0) on the same Jacobian values (*fused = 1), else operator then factor */
IRK_API int irk_dist_op_factor_apply(const irk_dist_op *d, const irk_factor *f, const double *v, double *x,
                                     int *fused, void *stream);
IRK_API int irk_linop_dist_op(const irk_dist_op *d, irk_linop *out);

/* ---- kernel-plugin protocol shims (host pointers; numba_backend.py) ------- */
IRK_API int irk_ref_bsr_matvec(irk_ctx *ctx, int64_t T, int m, const int64_t *indptr,
                       const int64_t *indices, const double *data, const double *x, double *y);
IRK_API int irk_ref_ilu0_factor(irk_ctx *ctx, int64_t T, int m, const int64_t *indptr,
                        const int64_t *indices, const int64_t *diag_pos, const double *data,
                        const uint8_t *keep, int simplified, double *f, double *dinv,
                        int64_t *fail);
IRK_API int irk_ref_ilu0_solve(irk_ctx *ctx, int64_t T, int m, const int64_t *indptr,
                       const int64_t *indices, const int64_t *diag_pos, const double *fdata,
                       const double *dinv, const uint8_t *keep, const double *y, double *x);
IRK_API int irk_ref_coupled_factor(irk_ctx *ctx, int s, int64_t T, int m, const int64_t *indptr,
                           const int64_t *indices, const int64_t *diag_pos,
                           const double *stage_data, const double *coupling, const uint8_t *keep,
                           int literal, double *f, double *g, double *dinv, int64_t *fail_stage,
                           int64_t *fail_elem);
IRK_API int irk_ref_coupled_solve(irk_ctx *ctx, int s, int64_t T, int m, const int64_t *indptr,
                          const int64_t *indices, const int64_t *diag_pos, const double *fstage,
                          const double *fcoupling, const double *dinv, const uint8_t *keep,
                          const double *y, double *x);

#ifdef __cplusplus
}
#endif
#endif /* IRKB200_H */
