// Host-pointer shims with the exact argument meaning of the reference's
// kernel-plugin protocol (kernels/numba_backend.py:21-151).  Each call copies
// its inputs to the device, runs the CUDA kernels, and copies fresh outputs
// back; inputs are never modified (the reference copies first too,
// numba_backend.py:47, 79, 99, 103, 133).  Every call uses its own stream and
// stream-ordered allocations, so the shims are reentrant (the reference may
// call ilu0_solve from up to s threads at once, precond.py:228-237).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "irk_internal.cuh"

namespace irk {
int build_apply_schedules(irk_factor* f, const std::vector<uint8_t>& keep);
int upload_raw(const double* host, int nb, int64_t count, double* dev_layout, cudaStream_t st);
int copy_blocks(const double* src, const std::vector<int64_t>& sidx, double* dst,
                const std::vector<int64_t>& didx, int64_t bsz, double scale, cudaStream_t st);
}  // namespace irk

using namespace irk;

namespace {

struct Scope {
    irk_ctx* ctx;
    cudaStream_t st = nullptr;
    irk_pattern* pat = nullptr;
    std::vector<irk_blocks*> blocks;
    irk_factor* fac = nullptr;
    irk_stage_op* op = nullptr;
    std::vector<void*> dev;
    explicit Scope(irk_ctx* c) : ctx(c) {}
    ~Scope() {
        if (st) cudaStreamSynchronize(st);
        for (void* p : dev) cudaFree(p);
        irk_stage_op_destroy(op);
        irk_factor_destroy(fac);
        for (auto* b : blocks) irk_blocks_destroy(b);
        irk_pattern_destroy(pat);
        if (st) cudaStreamDestroy(st);
    }
    int init() {
        IRK_CK(cudaSetDevice(ctx->device));
        IRK_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        return IRK_OK;
    }
    int pattern(int64_t T, const int64_t* indptr, const int64_t* indices, const int64_t* diag_pos) {
        std::vector<int64_t> dp;
        if (!diag_pos) {
            dp.resize(T);
            for (int64_t i = 0; i < T; ++i) {
                dp[i] = -1;
                for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
                    if (indices[k] == i) dp[i] = k;
                if (dp[i] < 0) { set_error("block row without a diagonal block is not supported"); return IRK_EINVAL; }
            }
            diag_pos = dp.data();
        }
        return irk_pattern_create(ctx, T, indptr, indices, diag_pos, &pat);
    }
    int upload(int nb, int64_t count, const double* host, irk_blocks** out) {
        IRK_TRY(irk_blocks_create(ctx, nb, count, out));
        blocks.push_back(*out);
        return irk_blocks_upload(*out, 0, count, host, 0, st);
    }
    int vec(size_t n, double** out, const double* host) {
        IRK_CK(cudaMalloc(out, sizeof(double) * std::max<size_t>(n, 1)));
        dev.push_back(*out);
        if (host) IRK_CK(cudaMemcpyAsync(*out, host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        return IRK_OK;
    }
};

// Build a factor object from reference-layout factor arrays (host).
int import_factor(Scope& S, int kind, int s, int m, const double* fstage, const double* fcoupling,
                  const double* dinv, const uint8_t* keep, irk_factor** out) {
    const irk_pattern* p = S.pat;
    const int64_t T = p->T, nnzb = p->nnzb, bsz = block_doubles(m);
    auto* f = new irk_factor();
    f->ctx = S.ctx;
    f->pat = p;
    f->kind = kind;
    f->s = s;
    f->nb = m;
    f->simplified = 0;
    f->u_stored = true;
    f->uscale = 1.0;
    S.fac = f;  // owned by the scope
    std::vector<uint8_t> kp(nnzb, 1);
    if (keep) std::memcpy(kp.data(), keep, nnzb);
    IRK_CK(cudaMalloc(&f->d_keep, nnzb));
    IRK_CK(cudaMemcpy(f->d_keep, kp.data(), nnzb, cudaMemcpyHostToDevice));
    IRK_CK(cudaMalloc(&f->d_L, sizeof(double) * bsz * std::max<int64_t>(p->nlow * s, 1)));
    IRK_CK(cudaMalloc(&f->d_U, sizeof(double) * bsz * std::max<int64_t>(p->nup * s, 1)));
    IRK_CK(cudaMalloc(&f->d_Dinv, sizeof(double) * bsz * T * s));
    irk_blocks *bf = nullptr, *bd = nullptr, *bc = nullptr;
    IRK_TRY(S.upload(m, (int64_t)s * nnzb, fstage, &bf));
    IRK_TRY(S.upload(m, (int64_t)s * T, dinv, &bd));
    std::vector<int64_t> sL, dL, sU, dU, sD, dD;
    for (int k = 0; k < s; ++k)
        for (int64_t j = 0; j < T; ++j) {
            for (int64_t q = p->h_indptr[j]; q < p->h_indptr[j + 1]; ++q) {
                if (q < p->h_diag[j]) { sL.push_back(k * nnzb + q); dL.push_back((p->h_lptr[j] + q - p->h_indptr[j]) * s + k); }
                else if (q > p->h_diag[j]) { sU.push_back(k * nnzb + q); dU.push_back((p->h_uptr[j] + q - p->h_diag[j] - 1) * s + k); }
            }
            sD.push_back(k * T + j);
            dD.push_back(j * s + k);
        }
    IRK_TRY(copy_blocks(bf->d, sL, f->d_L, dL, bsz, 1.0, S.st));
    IRK_TRY(copy_blocks(bf->d, sU, f->d_U, dU, bsz, 1.0, S.st));
    IRK_TRY(copy_blocks(bd->d, sD, f->d_Dinv, dD, bsz, 1.0, S.st));
    if (kind == IRK_FACTOR_COUPLED && s > 1) {
        const int npairs = s * (s - 1) / 2;
        IRK_TRY(S.upload(m, (int64_t)s * s * T, fcoupling, &bc));
        IRK_CK(cudaMalloc(&f->d_G, sizeof(double) * bsz * T * npairs));
        IRK_CK(cudaMalloc(&f->d_Cup, sizeof(double) * bsz * T * npairs));
        std::vector<int64_t> sg, dg, sc, dc;
        for (int k = 0; k < s; ++k)
            for (int l = 0; l < s; ++l)
                for (int64_t i = 0; i < T; ++i) {
                    const int64_t src = ((int64_t)k * s + l) * T + i;
                    if (k > l) { sg.push_back(src); dg.push_back(i * npairs + k * (k - 1) / 2 + l); }
                    else if (k < l) { sc.push_back(src); dc.push_back(i * npairs + l * (l - 1) / 2 + k); }
                }
        IRK_TRY(copy_blocks(bc->d, sg, f->d_G, dg, bsz, 1.0, S.st));
        IRK_TRY(copy_blocks(bc->d, sc, f->d_Cup, dc, bsz, 1.0, S.st));
    }
    IRK_TRY(build_apply_schedules(f, kp));
    *out = f;
    return IRK_OK;
}

}  // namespace

extern "C" {

int irk_ref_bsr_matvec(irk_ctx* ctx, int64_t T, int m, const int64_t* indptr, const int64_t* indices,
                       const double* data, const double* x, double* y) {
    IRK_ARG(ctx && indptr && indices && data && x && y, "NULL argument");
    Scope S(ctx);
    IRK_TRY(S.init());
    IRK_TRY(S.pattern(T, indptr, indices, nullptr));
    irk_blocks* J = nullptr;
    IRK_TRY(S.upload(m, S.pat->nnzb, data, &J));
    double *dx, *dy;
    IRK_TRY(S.vec(T * m, &dx, x));
    IRK_TRY(S.vec(T * m, &dy, nullptr));
    const irk_blocks* Js[1] = {J};
    IRK_TRY(irk_stage_op_create(ctx, S.pat, 1, Js, nullptr, nullptr, nullptr, 1.0, &S.op));
    IRK_TRY(irk_stage_op_apply(S.op, dx, dy, S.st));
    IRK_CK(cudaMemcpyAsync(y, dy, sizeof(double) * T * m, cudaMemcpyDeviceToHost, S.st));
    IRK_CK(cudaStreamSynchronize(S.st));
    return IRK_OK;
}

int irk_ref_ilu0_factor(irk_ctx* ctx, int64_t T, int m, const int64_t* indptr, const int64_t* indices,
                        const int64_t* diag_pos, const double* data, const uint8_t* keep, int simplified,
                        double* f, double* dinv, int64_t* fail) {
    IRK_ARG(ctx && indptr && indices && diag_pos && data && f && dinv && fail, "NULL argument");
    Scope S(ctx);
    IRK_TRY(S.init());
    IRK_TRY(S.pattern(T, indptr, indices, diag_pos));
    irk_blocks* J = nullptr;
    IRK_TRY(S.upload(m, S.pat->nnzb, data, &J));
    const irk_blocks* Js[1] = {J};
    int64_t fs = -1, fe = -1;
    int rc = irk_factor_uncoupled(ctx, S.pat, 1, Js, nullptr, nullptr, nullptr, 1.0, keep, simplified, 1,
                                  &S.fac, &fs, &fe, S.st);
    if (rc < 0) return rc;
    *fail = fe;
    IRK_TRY(irk_factor_export(S.fac, f, dinv, nullptr, S.st));
    return IRK_OK;
}

int irk_ref_ilu0_solve(irk_ctx* ctx, int64_t T, int m, const int64_t* indptr, const int64_t* indices,
                       const int64_t* diag_pos, const double* fdata, const double* dinv, const uint8_t* keep,
                       const double* y, double* x) {
    IRK_ARG(ctx && indptr && indices && diag_pos && fdata && dinv && y && x, "NULL argument");
    Scope S(ctx);
    IRK_TRY(S.init());
    IRK_TRY(S.pattern(T, indptr, indices, diag_pos));
    irk_factor* fac = nullptr;
    IRK_TRY(import_factor(S, IRK_FACTOR_UNCOUPLED, 1, m, fdata, nullptr, dinv, keep, &fac));
    double *dy, *dx;
    IRK_TRY(S.vec(T * m, &dy, y));
    IRK_TRY(S.vec(T * m, &dx, nullptr));
    IRK_TRY(irk_factor_apply(fac, dy, dx, S.st));
    IRK_CK(cudaMemcpyAsync(x, dx, sizeof(double) * T * m, cudaMemcpyDeviceToHost, S.st));
    IRK_CK(cudaStreamSynchronize(S.st));
    return IRK_OK;
}

int irk_ref_coupled_factor(irk_ctx* ctx, int s, int64_t T, int m, const int64_t* indptr, const int64_t* indices,
                           const int64_t* diag_pos, const double* stage_data, const double* coupling,
                           const uint8_t* keep, int literal, double* f, double* g, double* dinv,
                           int64_t* fail_stage, int64_t* fail_elem) {
    IRK_ARG(ctx && indptr && indices && diag_pos && stage_data && coupling && f && g && dinv && fail_stage &&
                fail_elem, "NULL argument");
    IRK_ARG(s >= 1 && s <= IRK_MAX_STAGES, "stage count out of range");
    Scope S(ctx);
    IRK_TRY(S.init());
    IRK_TRY(S.pattern(T, indptr, indices, diag_pos));
    const int64_t nnzb = S.pat->nnzb;
    irk_blocks *B = nullptr, *C = nullptr;
    IRK_TRY(S.upload(m, (int64_t)s * nnzb, stage_data, &B));
    IRK_TRY(S.upload(m, (int64_t)s * s * T, coupling, &C));
    const irk_blocks* Js[IRK_MAX_STAGES];
    int64_t jf[IRK_MAX_STAGES];
    for (int k = 0; k < s; ++k) { Js[k] = B; jf[k] = k * nnzb; }
    std::vector<double> eye(s * s, 0.0);
    int rc = irk_factor_coupled(ctx, S.pat, s, Js, jf, nullptr, eye.data(), 1.0, C, keep, literal, 1, &S.fac,
                                fail_stage, fail_elem, S.st);
    if (rc < 0) return rc;
    IRK_TRY(irk_factor_export(S.fac, f, dinv, g, S.st));
    // the reference returns the (unused) stage-diagonal coupling blocks unchanged
    const size_t bb = (size_t)m * m;
    for (int k = 0; k < s; ++k)
        std::memcpy(g + ((size_t)k * s + k) * T * bb, coupling + ((size_t)k * s + k) * T * bb, sizeof(double) * T * bb);
    return IRK_OK;
}

int irk_ref_coupled_solve(irk_ctx* ctx, int s, int64_t T, int m, const int64_t* indptr, const int64_t* indices,
                          const int64_t* diag_pos, const double* fstage, const double* fcoupling, const double* dinv,
                          const uint8_t* keep, const double* y, double* x) {
    IRK_ARG(ctx && indptr && indices && diag_pos && fstage && fcoupling && dinv && y && x, "NULL argument");
    IRK_ARG(s >= 1 && s <= IRK_MAX_STAGES, "stage count out of range");
    Scope S(ctx);
    IRK_TRY(S.init());
    IRK_TRY(S.pattern(T, indptr, indices, diag_pos));
    irk_factor* fac = nullptr;
    IRK_TRY(import_factor(S, IRK_FACTOR_COUPLED, s, m, fstage, fcoupling, dinv, keep, &fac));
    double *dy, *dx;
    const size_t n = (size_t)s * T * m;
    IRK_TRY(S.vec(n, &dy, y));
    IRK_TRY(S.vec(n, &dx, nullptr));
    IRK_TRY(irk_factor_apply(fac, dy, dx, S.st));
    IRK_CK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    IRK_CK(cudaStreamSynchronize(S.st));
    return IRK_OK;
}

}  // extern "C"
