/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle of the irk-b200 hot path.
 *
 * A plain-C restatement of the reference block kernels
 * (/root/reference/pkg/src/irksolve/kernels/numba_backend.py and its numpy
 * twin numpy_backend.py) plus the transformed stage matvec
 * (stage_system.py:52-70).  Same loop orders, same per-block operation
 * sequence (block product into a temporary, then add/subtract), row-major
 * m x m blocks, int64 CSR-of-blocks indices, uint8 keep mask.
 *
 * Used only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg as the checker / CPU reference arm.  The shipped GPU path never links
 * or calls this file.
 *
 * Parity is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py), see tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define COND_LIMIT 1e14 /* numba_backend.py:10 */

/* C = A @ B, m x m row-major (the reference's per-block `@`). */
static void gemm(int m, const double *A, const double *B, double *C) {
    for (int a = 0; a < m; ++a) {
        double *c = C + (size_t)a * m;
        for (int b = 0; b < m; ++b) c[b] = 0.0;
        for (int k = 0; k < m; ++k) {
            const double av = A[(size_t)a * m + k];
            const double *brow = B + (size_t)k * m;
            for (int b = 0; b < m; ++b) c[b] += av * brow[b];
        }
    }
}

/* y = A @ x. */
static void gemv(int m, const double *A, const double *x, double *y) {
    for (int a = 0; a < m; ++a) {
        const double *row = A + (size_t)a * m;
        double acc = 0.0;
        for (int b = 0; b < m; ++b) acc += row[b] * x[b];
        y[a] = acc;
    }
}

/* numba_backend.py:13-18 */
static int64_t block_pos(const int64_t *indptr, const int64_t *indices, int64_t i, int64_t j) {
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
        if (indices[k] == j) return k;
    return -1;
}

static double norm1(int m, const double *A) {
    /* np.abs(A).sum(axis=0).max(): NaN propagates */
    double best = -INFINITY;
    for (int b = 0; b < m; ++b) {
        double s = 0.0;
        for (int a = 0; a < m; ++a) s += fabs(A[(size_t)a * m + b]);
        if (isnan(s)) return s;
        if (s > best) best = s;
    }
    return best;
}

/*
 * numba_backend.py:33-40 (_inv_with_cond).  det is sign*exp(sum log|u_kk|)
 * over the partial-pivoting LU (numpy/numba slogdet path), so the singular
 * decision is "det == 0 or not finite".  The inverse solves LU X = P I.
 * Returns 1 and cond=inf when singular.  work: 2*m*m doubles + m ints.
 */
static int inv_with_cond(int m, const double *blk, double *inv, double *cond, double *lu, int *piv) {
    memcpy(lu, blk, sizeof(double) * (size_t)m * m);
    double logdet = 0.0;
    int zero = 0;
    for (int k = 0; k < m; ++k) {
        int p = k;
        double best = fabs(lu[(size_t)k * m + k]);
        for (int r = k + 1; r < m; ++r) {
            double v = fabs(lu[(size_t)r * m + k]);
            if (v > best) { best = v; p = r; }
        }
        piv[k] = p;
        if (p != k)
            for (int c = 0; c < m; ++c) {
                double t = lu[(size_t)k * m + c];
                lu[(size_t)k * m + c] = lu[(size_t)p * m + c];
                lu[(size_t)p * m + c] = t;
            }
        double d = lu[(size_t)k * m + k];
        logdet += log(fabs(d));
        if (d == 0.0) { zero = 1; continue; }
        for (int r = k + 1; r < m; ++r) {
            double l = lu[(size_t)r * m + k] / d;
            lu[(size_t)r * m + k] = l;
            for (int c = k + 1; c < m; ++c) lu[(size_t)r * m + c] -= l * lu[(size_t)k * m + c];
        }
    }
    double det = exp(logdet);
    if (zero || det == 0.0 || !isfinite(det)) {
        memset(inv, 0, sizeof(double) * (size_t)m * m);
        *cond = INFINITY;
        return 1;
    }
    /* X = U^-1 L^-1 P I, column by column */
    for (int col = 0; col < m; ++col) {
        double *x = inv; /* fill column col of inv, stride m */
        double tmp[512];
        double *v = (m <= 512) ? tmp : (double *)malloc(sizeof(double) * m);
        for (int a = 0; a < m; ++a) v[a] = (a == col) ? 1.0 : 0.0;
        for (int k = 0; k < m; ++k)
            if (piv[k] != k) { double t = v[k]; v[k] = v[piv[k]]; v[piv[k]] = t; }
        for (int a = 0; a < m; ++a) {
            double acc = v[a];
            for (int c = 0; c < a; ++c) acc -= lu[(size_t)a * m + c] * v[c];
            v[a] = acc;
        }
        for (int a = m - 1; a >= 0; --a) {
            double acc = v[a];
            for (int c = a + 1; c < m; ++c) acc -= lu[(size_t)a * m + c] * v[c];
            v[a] = acc / lu[(size_t)a * m + a];
        }
        for (int a = 0; a < m; ++a) x[(size_t)a * m + col] = v[a];
        if (v != tmp) free(v);
    }
    *cond = norm1(m, blk) * norm1(m, inv);
    return 0;
}

/* numba_backend.py:21-30 */
void orc_bsr_matvec(int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                    const double *data, const double *x, double *y) {
    const size_t bk = (size_t)m * m;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < T; ++i) {
        double tmp[512];
        double *yi = y + (size_t)i * m;
        for (int a = 0; a < m; ++a) yi[a] = 0.0;
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
            gemv(m, data + (size_t)k * bk, x + (size_t)indices[k] * m, tmp);
            for (int a = 0; a < m; ++a) yi[a] += tmp[a];
        }
    }
}

/*
 * stage_system.py:52-70: y_k = -dt * (J_k w_k) + sum_l a_inv[k,l] * (M w_l),
 * accumulated in that order.  J_k = J + k*jstride (jstride = 0: shared J).
 */
void orc_stage_matvec(int s, int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                      const double *J, int64_t jstride, const double *M, const double *a_inv,
                      double dt, const double *w, double *y) {
    const size_t n = (size_t)T * m;
    const size_t bk = (size_t)m * m;
    double *jw = (double *)malloc(sizeof(double) * n);
    double *mw = (double *)malloc(sizeof(double) * n * s);
    for (int l = 0; l < s; ++l) {
        const double *wl = w + l * n;
        double *out = mw + l * n;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < T; ++i) gemv(m, M + (size_t)i * bk, wl + (size_t)i * m, out + (size_t)i * m);
    }
    for (int k = 0; k < s; ++k) {
        orc_bsr_matvec(T, m, indptr, indices, J + (size_t)k * jstride, w + k * n, jw);
        double *yk = y + k * n;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < (int64_t)n; ++e) {
            double acc = -dt * jw[e];
            for (int l = 0; l < s; ++l) acc += a_inv[k * s + l] * mw[l * n + e];
            yk[e] = acc;
        }
    }
    free(jw);
    free(mw);
}

/* numba_backend.py:43-72.  f, dinv are outputs (f = data copy). Returns fail element or -1. */
int64_t orc_ilu0_factor(int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                        const int64_t *diag_pos, const double *data, const uint8_t *keep,
                        int simplified, double *f, double *dinv) {
    const size_t bk = (size_t)m * m;
    const int64_t nnzb = indptr[T];
    memcpy(f, data, sizeof(double) * bk * nnzb);
    for (int64_t k = 0; k < nnzb; ++k)
        if (!keep[k]) memset(f + k * bk, 0, sizeof(double) * bk);
    memset(dinv, 0, sizeof(double) * bk * T);
    double *inv = (double *)malloc(sizeof(double) * bk * 4);
    double *lu = inv + bk, *tmp = inv + 2 * bk, *tmp2 = inv + 3 * bk;
    int *piv = (int *)malloc(sizeof(int) * m);
    int64_t fail = -1;
    for (int64_t i = 0; i < T && fail < 0; ++i) {
        double cond;
        inv_with_cond(m, f + diag_pos[i] * bk, inv, &cond, lu, piv);
        if (!isfinite(cond) || cond > COND_LIMIT) { fail = i; break; }
        memcpy(dinv + i * bk, inv, sizeof(double) * bk);
        for (int64_t kij = diag_pos[i] + 1; kij < indptr[i + 1]; ++kij) {
            int64_t j = indices[kij];
            if (!keep[kij]) continue;
            int64_t kji = block_pos(indptr, indices, j, i);
            gemm(m, f + kji * bk, inv, tmp);
            memcpy(f + kji * bk, tmp, sizeof(double) * bk);
            gemm(m, f + kji * bk, f + kij * bk, tmp);
            double *dj = f + diag_pos[j] * bk;
            for (size_t e = 0; e < bk; ++e) dj[e] -= tmp[e];
            if (!simplified) {
                for (int64_t kik = indptr[i]; kik < indptr[i + 1]; ++kik) {
                    int64_t k2 = indices[kik];
                    if (k2 <= j || k2 == i || !keep[kik]) continue;
                    int64_t kjk = block_pos(indptr, indices, j, k2);
                    if (kjk >= 0 && keep[kjk]) {
                        gemm(m, f + kji * bk, f + kik * bk, tmp2);
                        double *fjk = f + kjk * bk;
                        for (size_t e = 0; e < bk; ++e) fjk[e] -= tmp2[e];
                    }
                }
            }
        }
    }
    free(inv);
    free(piv);
    return fail;
}

/* numba_backend.py:75-91.  y (T*m) -> x (T*m). */
void orc_ilu0_solve(int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                    const int64_t *diag_pos, const double *fdata, const double *dinv,
                    const uint8_t *keep, const double *y, double *x) {
    const size_t bk = (size_t)m * m;
    double tmp[512], acc[512];
    memcpy(x, y, sizeof(double) * (size_t)T * m);
    for (int64_t i = 0; i < T; ++i) {
        double *zi = x + i * m;
        for (int64_t k = indptr[i]; k < diag_pos[i]; ++k)
            if (keep[k]) {
                gemv(m, fdata + k * bk, x + indices[k] * m, tmp);
                for (int a = 0; a < m; ++a) zi[a] -= tmp[a];
            }
    }
    for (int64_t i = T - 1; i >= 0; --i) {
        double *xi = x + i * m;
        for (int a = 0; a < m; ++a) acc[a] = xi[a];
        for (int64_t k = diag_pos[i] + 1; k < indptr[i + 1]; ++k)
            if (keep[k]) {
                gemv(m, fdata + k * bk, x + indices[k] * m, tmp);
                for (int a = 0; a < m; ++a) acc[a] -= tmp[a];
            }
        gemv(m, dinv + i * bk, acc, xi);
    }
}

/* numba_backend.py:94-125.  Outputs f (s,nnzb,m,m), g (s,s,T,m,m), dinv (s,T,m,m). */
void orc_coupled_factor(int s, int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                        const int64_t *diag_pos, const double *stage_data, const double *coupling,
                        const uint8_t *keep, int literal, double *f, double *g, double *dinv,
                        int64_t *fail_stage, int64_t *fail_elem) {
    const size_t bk = (size_t)m * m;
    const int64_t nnzb = indptr[T];
    memcpy(f, stage_data, sizeof(double) * bk * nnzb * s);
    for (int64_t k = 0; k < nnzb; ++k)
        if (!keep[k])
            for (int st = 0; st < s; ++st) memset(f + ((size_t)st * nnzb + k) * bk, 0, sizeof(double) * bk);
    memcpy(g, coupling, sizeof(double) * bk * T * s * s);
    memset(dinv, 0, sizeof(double) * bk * T * s);
    double *inv = (double *)malloc(sizeof(double) * bk * 3);
    double *lu = inv + bk, *tmp = inv + 2 * bk;
    int *piv = (int *)malloc(sizeof(int) * m);
    *fail_stage = -1;
    *fail_elem = -1;
#define F(st, q) (f + ((size_t)(st) * nnzb + (q)) * bk)
#define G(k_, l_, i_) (g + ((((size_t)(k_) * s + (l_)) * T) + (i_)) * bk)
    for (int k = 0; k < s; ++k) {
        for (int64_t i = 0; i < T; ++i) {
            double cond;
            inv_with_cond(m, F(k, diag_pos[i]), inv, &cond, lu, piv);
            if (!isfinite(cond) || cond > COND_LIMIT) {
                *fail_stage = k;
                *fail_elem = i;
                goto done;
            }
            memcpy(dinv + ((size_t)k * T + i) * bk, inv, sizeof(double) * bk);
            for (int64_t kij = diag_pos[i] + 1; kij < indptr[i + 1]; ++kij) {
                if (!keep[kij]) continue;
                int64_t j = indices[kij];
                int64_t kji = block_pos(indptr, indices, j, i);
                gemm(m, F(k, kji), inv, tmp);
                memcpy(F(k, kji), tmp, sizeof(double) * bk);
                gemm(m, F(k, kji), F(k, kij), tmp);
                double *dj = F(k, diag_pos[j]);
                for (size_t e = 0; e < bk; ++e) dj[e] -= tmp[e];
            }
            for (int l = k + 1; l < s; ++l) {
                gemm(m, G(l, k, i), inv, tmp);
                memcpy(G(l, k, i), tmp, sizeof(double) * bk);
                if (literal) gemm(m, G(l, k, i), F(k, diag_pos[i]), tmp);
                else gemm(m, G(l, k, i), G(k, l, i), tmp);
                double *dl = F(l, diag_pos[i]);
                for (size_t e = 0; e < bk; ++e) dl[e] -= tmp[e];
            }
        }
    }
done:
#undef F
#undef G
    free(inv);
    free(piv);
}

/* numba_backend.py:128-151.  y (s*T*m) -> x. */
void orc_coupled_solve(int s, int64_t T, int m, const int64_t *indptr, const int64_t *indices,
                       const int64_t *diag_pos, const double *fstage, const double *fcoupling,
                       const double *dinv, const uint8_t *keep, const double *y, double *x) {
    const size_t bk = (size_t)m * m;
    const int64_t nnzb = indptr[T];
    double tmp[512], acc[512];
    memcpy(x, y, sizeof(double) * (size_t)s * T * m);
#define X(k_, i_) (x + ((size_t)(k_) * T + (i_)) * m)
#define F(st, q) (fstage + ((size_t)(st) * nnzb + (q)) * bk)
#define G(k_, l_, i_) (fcoupling + ((((size_t)(k_) * s + (l_)) * T) + (i_)) * bk)
    for (int k = 0; k < s; ++k)
        for (int64_t i = 0; i < T; ++i) {
            double *z = X(k, i);
            for (int64_t kk = indptr[i]; kk < diag_pos[i]; ++kk)
                if (keep[kk]) {
                    gemv(m, F(k, kk), X(k, indices[kk]), tmp);
                    for (int a = 0; a < m; ++a) z[a] -= tmp[a];
                }
            for (int l = 0; l < k; ++l) {
                gemv(m, G(k, l, i), X(l, i), tmp);
                for (int a = 0; a < m; ++a) z[a] -= tmp[a];
            }
        }
    for (int k = s - 1; k >= 0; --k)
        for (int64_t i = T - 1; i >= 0; --i) {
            double *xi = X(k, i);
            for (int a = 0; a < m; ++a) acc[a] = xi[a];
            for (int64_t kk = diag_pos[i] + 1; kk < indptr[i + 1]; ++kk)
                if (keep[kk]) {
                    gemv(m, F(k, kk), X(k, indices[kk]), tmp);
                    for (int a = 0; a < m; ++a) acc[a] -= tmp[a];
                }
            for (int l = k + 1; l < s; ++l) {
                gemv(m, G(k, l, i), X(l, i), tmp);
                for (int a = 0; a < m; ++a) acc[a] -= tmp[a];
            }
            gemv(m, dinv + ((size_t)k * T + i) * bk, acc, xi);
        }
#undef X
#undef F
#undef G
}
