// Context, error state, block pattern and block-array management + the
// row-major <-> device-layout permutation kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>

#include "irk_internal.cuh"

namespace irk {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("IRK_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}


static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count_now() { return g_launches.load(std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_err = msg; }

int fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
             cudaGetErrorString(e), what, file, line);
    g_err = buf;
    return e == cudaErrorMemoryAllocation ? IRK_ENOMEM : IRK_ECUDA;
}

// one CTA per block: coalesced row-major read into shared memory, coalesced
// 16-byte writes in the column-pair interleaved layout (and the reverse).
__global__ void k_rowmajor_to_layout(const double* __restrict__ src, double* __restrict__ dst,
                                     int nb, int64_t count) {
    extern __shared__ double sm[];
    const int P = (nb + 1) >> 1;
    const int64_t bsz_in = (int64_t)nb * nb, bsz_out = (int64_t)nb * 2 * P;
    for (int64_t b = blockIdx.x; b < count; b += gridDim.x) {
        const double* in = src + b * bsz_in;
        for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) sm[e] = in[e];
        __syncthreads();
        double2* out = reinterpret_cast<double2*>(dst + b * bsz_out);
        for (int e = threadIdx.x; e < nb * P; e += blockDim.x) {
            const int p = e / nb, a = e - p * nb;
            const int c = 2 * p;
            double2 v;
            v.x = sm[a * nb + c];
            v.y = (c + 1 < nb) ? sm[a * nb + c + 1] : 0.0;
            out[e] = v;
        }
        __syncthreads();
    }
}

__global__ void k_layout_to_rowmajor(const double* __restrict__ src, double* __restrict__ dst,
                                     int nb, int64_t count) {
    extern __shared__ double sm[];
    const int P = (nb + 1) >> 1;
    const int64_t bsz_in = (int64_t)nb * 2 * P, bsz_out = (int64_t)nb * nb;
    for (int64_t b = blockIdx.x; b < count; b += gridDim.x) {
        const double2* in = reinterpret_cast<const double2*>(src + b * bsz_in);
        for (int e = threadIdx.x; e < nb * P; e += blockDim.x) {
            const int p = e / nb, a = e - p * nb;
            const double2 v = in[e];
            sm[a * nb + 2 * p] = v.x;
            if (2 * p + 1 < nb) sm[a * nb + 2 * p + 1] = v.y;
        }
        __syncthreads();
        double* out = dst + b * bsz_out;
        for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) out[e] = sm[e];
        __syncthreads();
    }
}

int permute_in(const double* src_dev, double* dst_dev, int nb, int64_t count, cudaStream_t st) {
    if (count <= 0) return IRK_OK;
    const size_t smem = sizeof(double) * nb * nb;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(k_rowmajor_to_layout, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        cudaFuncSetAttribute(k_layout_to_rowmajor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    });
    const int grid = (int)std::min<int64_t>(count, 148 * 16);
    k_rowmajor_to_layout<<<grid, 256, smem, st>>>(src_dev, dst_dev, nb, count);
    IRK_LAUNCHED();
    return IRK_OK;
}

int permute_out(const double* src_dev, double* dst_dev, int nb, int64_t count, cudaStream_t st) {
    if (count <= 0) return IRK_OK;
    IRK_TRY(permute_in(nullptr, nullptr, nb, 0, st));  // attribute init
    const size_t smem = sizeof(double) * nb * nb;
    const int grid = (int)std::min<int64_t>(count, 148 * 16);
    k_layout_to_rowmajor<<<grid, 256, smem, st>>>(src_dev, dst_dev, nb, count);
    IRK_LAUNCHED();
    return IRK_OK;
}

}  // namespace irk

using namespace irk;

extern "C" {

int irk_version(void) { return 10000; }

int64_t irk_launch_count(void) { return (int64_t)g_launches.load(); }

const char* irk_last_error(void) { return g_err.c_str(); }

int irk_ctx_create(int device, irk_ctx** out) {
    IRK_ARG(out, "out is NULL");
    int n = 0;
    IRK_CK(cudaGetDeviceCount(&n));
    IRK_ARG(device >= 0 && device < n, "device index out of range");
    IRK_CK(cudaSetDevice(device));
    auto* c = new irk_ctx();
    c->device = device;
    cudaDeviceProp prop;
    IRK_CK(cudaGetDeviceProperties(&prop, device));
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    c->smem_per_sm = prop.sharedMemPerMultiprocessor;
    // keep stream-ordered allocations cached between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // no cross-stream reuse: a block freed on an upload stream must not be handed to a solve on
        // another stream with an implicit wait on that upload (double-buffered streaming, bench e2e)
        int off = 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseFollowEventDependencies, &off);
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &off);
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &off);
    }
    *out = c;
    return IRK_OK;
}

void irk_ctx_destroy(irk_ctx* ctx) { delete ctx; }

int irk_pattern_create(irk_ctx* ctx, int64_t T, const int64_t* indptr, const int64_t* indices,
                       const int64_t* diag_pos, irk_pattern** out) {
    IRK_ARG(ctx && out && indptr && indices && diag_pos, "NULL argument");
    IRK_ARG(T >= 1 && T < (1LL << 31), "T out of range");
    IRK_ARG(indptr[0] == 0, "indptr[0] != 0");
    const int64_t nnzb = indptr[T];
    IRK_ARG(nnzb >= T && nnzb < (1LL << 31), "nnzb out of range");
    for (int64_t i = 0; i < T; ++i) {
        IRK_ARG(indptr[i + 1] > indptr[i], "empty block row (diagonal missing)");
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
            IRK_ARG(indices[k] >= 0 && indices[k] < T, "column index out of range");
            if (k > indptr[i]) IRK_ARG(indices[k] > indices[k - 1], "columns not sorted/unique");
        }
        IRK_ARG(diag_pos[i] >= indptr[i] && diag_pos[i] < indptr[i + 1] &&
                    indices[diag_pos[i]] == i,
                "diag_pos does not point at the diagonal block");
    }
    auto* p = new irk_pattern();
    p->ctx = ctx;
    p->T = T;
    p->nnzb = nnzb;
    p->h_indptr.assign(indptr, indptr + T + 1);
    p->h_indices.assign(indices, indices + nnzb);
    p->h_diag.assign(diag_pos, diag_pos + T);
    p->h_lptr.assign(T + 1, 0);
    p->h_uptr.assign(T + 1, 0);
    std::vector<int32_t> ip(T + 1), ix(nnzb), dg(T), rowof(nnzb), lptr(T + 1), uptr(T + 1),
        tpos(nnzb);
    for (int64_t i = 0; i <= T; ++i) ip[i] = (int32_t)indptr[i];
    for (int64_t k = 0; k < nnzb; ++k) ix[k] = (int32_t)indices[k];
    for (int64_t i = 0; i < T; ++i) {
        dg[i] = (int32_t)diag_pos[i];
        p->h_lptr[i + 1] = p->h_lptr[i] + (diag_pos[i] - indptr[i]);
        p->h_uptr[i + 1] = p->h_uptr[i] + (indptr[i + 1] - diag_pos[i] - 1);
        for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
            rowof[k] = (int32_t)i;
            const int64_t j = indices[k];
            const int64_t* b = indices + indptr[j];
            const int64_t* e = indices + indptr[j + 1];
            const int64_t* f = std::lower_bound(b, e, i);
            tpos[k] = (f != e && *f == i) ? (int32_t)(indptr[j] + (f - b)) : -1;
        }
    }
    for (int64_t i = 0; i <= T; ++i) {
        lptr[i] = (int32_t)p->h_lptr[i];
        uptr[i] = (int32_t)p->h_uptr[i];
    }
    p->nlow = p->h_lptr[T];
    p->nup = p->h_uptr[T];
    auto up = [&](int32_t** d, const std::vector<int32_t>& h) -> int {
        IRK_CK(cudaMalloc(d, sizeof(int32_t) * std::max<size_t>(h.size(), 1)));
        IRK_CK(cudaMemcpy(*d, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice));
        return IRK_OK;
    };
    int rc = IRK_OK;
    if ((rc = up(&p->d_indptr, ip)) || (rc = up(&p->d_indices, ix)) || (rc = up(&p->d_diag, dg)) ||
        (rc = up(&p->d_rowof, rowof)) || (rc = up(&p->d_lptr, lptr)) ||
        (rc = up(&p->d_uptr, uptr)) || (rc = up(&p->d_tpos, tpos))) {
        irk_pattern_destroy(p);
        return rc;
    }
    *out = p;
    return IRK_OK;
}

void irk_pattern_destroy(irk_pattern* p) {
    if (!p) return;
    cudaFree(p->d_indptr);
    cudaFree(p->d_indices);
    cudaFree(p->d_diag);
    cudaFree(p->d_rowof);
    cudaFree(p->d_lptr);
    cudaFree(p->d_uptr);
    cudaFree(p->d_tpos);
    delete p;
}

int irk_blocks_create(irk_ctx* ctx, int nb, int64_t count, irk_blocks** out) {
    IRK_ARG(ctx && out, "NULL argument");
    IRK_ARG(nb >= 1 && nb <= IRK_MAX_NB, "block size out of range [1, 128]");
    IRK_ARG(count >= 0, "negative block count");
    auto* b = new irk_blocks();
    b->ctx = ctx;
    b->nb = nb;
    b->count = count;
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(count, 1) * block_doubles(nb);
    cudaError_t e = cudaMalloc(&b->d, bytes);
    if (e != cudaSuccess) {
        delete b;
        return fail_cuda(e, "cudaMalloc(blocks)", __FILE__, __LINE__);
    }
    *out = b;
    return IRK_OK;
}

void irk_blocks_destroy(irk_blocks* b) {
    if (!b) return;
    cudaFree(b->d);
    delete b;
}

int irk_blocks_upload(irk_blocks* b, int64_t first, int64_t count, const double* src,
                      int src_on_device, void* stream) {
    IRK_ARG(b && (src || count == 0), "NULL argument");
    IRK_ARG(first >= 0 && count >= 0 && first + count <= b->count, "block range out of bounds");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = b->nb;
    const int64_t bin = (int64_t)nb * nb;
    double* dst = b->d + first * block_doubles(nb);
    if (src_on_device) return permute_in(src, dst, nb, count, st);
    // stage host data through a device buffer in chunks of <= 256 MiB
    const int64_t chunk = std::max<int64_t>(1, (256LL << 20) / (8 * bin));
    if (count > chunk) {
        // several chunks: two staging buffers, H2D copies on the caller's stream and the layout
        // permutes on a helper stream, so the copy engine never waits for a permute (the upload is
        // PCIe-bound: 2.13 GB per config-1 system)
        cudaStream_t ps = nullptr;
        cudaEvent_t cp[2] = {}, pm[2] = {};
        double* buf[2] = {};
        IRK_CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            IRK_CK(cudaEventCreateWithFlags(&cp[b], cudaEventDisableTiming));
            IRK_CK(cudaEventCreateWithFlags(&pm[b], cudaEventDisableTiming));
            IRK_CK(cudaMallocAsync(&buf[b], sizeof(double) * bin * chunk, st));
        }
        int rc = IRK_OK;
        int64_t c = 0;
        for (int64_t c0 = 0; c0 < count && rc == IRK_OK; c0 += chunk, ++c) {
            const int b = (int)(c & 1);
            const int64_t n = std::min(chunk, count - c0);
            if (c >= 2) IRK_CK(cudaStreamWaitEvent(st, pm[b], 0));   // permute c-2 has drained buf[b]
            cudaError_t e = cudaMemcpyAsync(buf[b], src + c0 * bin, sizeof(double) * bin * n,
                                            cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) { rc = fail_cuda(e, "upload H2D", __FILE__, __LINE__); break; }
            IRK_CK(cudaEventRecord(cp[b], st));
            IRK_CK(cudaStreamWaitEvent(ps, cp[b], 0));
            rc = permute_in(buf[b], dst + c0 * block_doubles(nb), nb, n, ps);
            IRK_CK(cudaEventRecord(pm[b], ps));
        }
        for (int b = 0; b < 2 && b < c; ++b) IRK_CK(cudaStreamWaitEvent(st, pm[b], 0));
        for (int b = 0; b < 2; ++b) {
            cudaFreeAsync(buf[b], st);
            cudaEventDestroy(cp[b]);
            cudaEventDestroy(pm[b]);
        }
        cudaStreamDestroy(ps);
        return rc;
    }
    double* tmp = nullptr;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * bin * std::min(chunk, std::max<int64_t>(count, 1)), st));
    int rc = IRK_OK;
    for (int64_t c0 = 0; c0 < count && rc == IRK_OK; c0 += chunk) {
        const int64_t n = std::min(chunk, count - c0);
        cudaError_t e = cudaMemcpyAsync(tmp, src + c0 * bin, sizeof(double) * bin * n,
                                        cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) { rc = fail_cuda(e, "upload H2D", __FILE__, __LINE__); break; }
        rc = permute_in(tmp, dst + c0 * block_doubles(nb), nb, n, st);
    }
    cudaFreeAsync(tmp, st);
    return rc;
}

int irk_blocks_download(const irk_blocks* b, int64_t first, int64_t count, double* dst,
                        int dst_on_device, void* stream) {
    IRK_ARG(b && (dst || count == 0), "NULL argument");
    IRK_ARG(first >= 0 && count >= 0 && first + count <= b->count, "block range out of bounds");
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = b->nb;
    const int64_t bin = (int64_t)nb * nb;
    const double* src = b->d + first * block_doubles(nb);
    if (dst_on_device) return permute_out(src, dst, nb, count, st);
    const int64_t chunk = std::max<int64_t>(1, (256LL << 20) / (8 * bin));
    double* tmp = nullptr;
    IRK_CK(cudaMallocAsync(&tmp, sizeof(double) * bin * std::min(chunk, std::max<int64_t>(count, 1)), st));
    int rc = IRK_OK;
    for (int64_t c0 = 0; c0 < count && rc == IRK_OK; c0 += chunk) {
        const int64_t n = std::min(chunk, count - c0);
        rc = permute_out(src + c0 * block_doubles(nb), tmp, nb, n, st);
        if (rc) break;
        cudaError_t e = cudaMemcpyAsync(dst + c0 * bin, tmp, sizeof(double) * bin * n,
                                        cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) { rc = fail_cuda(e, "download D2H", __FILE__, __LINE__); break; }
    }
    cudaFreeAsync(tmp, st);
    if (rc == IRK_OK) IRK_CK(cudaStreamSynchronize(st));
    return rc;
}

}  // extern "C"
