// FP64 tensor-core (DMMA) peak on this GPU: the roofline denominator of the
// factorisation kernels (k_schur, k_inverse_tc), which run on
// mma.sync.aligned.m8n8k4.row.col.f64 tiles.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_peak tools/dmma_peak.cu
//   ./dmma_peak            -> one JSON line
//
// Every warp runs CHAINS independent accumulator chains of back-to-back DMMAs
// (512 flops each) entirely in registers; timed with CUDA events after a
// warm-up, best of REPS, grid = SMs x CTAS_PER_SM x WARPS warps. Also times
// plain FP64 FMA (DFMA) for the non-tensor pipe.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void k_dmma(int iters, double *sink) {
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    double c0[CHAINS], c1[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { c0[i] = 0.0; c1[i] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc += c0[i] + c1[i];
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}

template <int CHAINS>
__global__ void k_dfma(int iters, double *sink) {
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    double c[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = 1e-3 * i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc += c[i];
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    double *sink;
    CK(cudaMalloc(&sink, 1024 * sizeof(double)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int REPS = 5;
    double best_tc = 0, best_fma = 0;
    int best_cfg_tc = 0, best_cfg_fma = 0;
    const int threads_opts[] = {128, 256, 512};
    const int ctas_opts[] = {1, 2, 4};
    for (int ti = 0; ti < 3; ++ti)
        for (int ci = 0; ci < 3; ++ci) {
            int threads = threads_opts[ti], grid = sms * ctas_opts[ci];
            const int iters = 4096;
            k_dmma<8><<<grid, threads>>>(16, sink);
            CK(cudaDeviceSynchronize());
            for (int r = 0; r < REPS; ++r) {
                CK(cudaEventRecord(e0));
                k_dmma<8><<<grid, threads>>>(iters, sink);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                double warps = (double)grid * threads / 32;
                double fl = warps * iters * 8 * 512.0;
                double tf = fl / (ms * 1e-3) / 1e12;
                if (tf > best_tc) { best_tc = tf; best_cfg_tc = grid * 10000 + threads; }
            }
            k_dfma<8><<<grid, threads>>>(16, sink);
            CK(cudaDeviceSynchronize());
            for (int r = 0; r < REPS; ++r) {
                CK(cudaEventRecord(e0));
                k_dfma<8><<<grid, threads>>>(iters * 4, sink);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                double fl = (double)grid * threads * iters * 4 * 8 * 2.0;
                double tf = fl / (ms * 1e-3) / 1e12;
                if (tf > best_fma) { best_fma = tf; best_cfg_fma = grid * 10000 + threads; }
            }
        }
    printf("{\"fp64_dmma_tflops\": %.3f, \"dmma_grid\": %d, \"dmma_threads\": %d, "
           "\"fp64_dfma_tflops\": %.3f, \"dfma_grid\": %d, \"dfma_threads\": %d, \"sms\": %d, "
           "\"clock_khz_attr\": %d, \"how\": \"mma.sync.m8n8k4.f64 (512 flop) x 8 independent chains per "
           "warp / 8 independent DFMA chains per thread, CUDA events, best of %d per launch shape\"}\n",
           best_tc, best_cfg_tc / 10000, best_cfg_tc % 10000, best_fma, best_cfg_fma / 10000,
           best_cfg_fma % 10000, sms, clk, REPS);
    return 0;
}
