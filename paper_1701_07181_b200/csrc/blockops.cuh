// Device helpers for block products in the column-pair interleaved layout.
//
// Thread geometry used by every GEMV-type kernel: a CTA runs G groups of nb
// threads (plus idle padding up to a warp multiple).  Thread t owns row
// a = t % nb of group g = t / nb; group g handles column pairs p = g, g+G, ...
// A group's nb threads read one column pair of a block as nb consecutive
// 16-byte vectors, so a warp issues fully coalesced 128-bit loads; the
// matching x pair is one broadcast 16-byte load.  Partial sums of the G
// groups are reduced through shared memory in a fixed order (deterministic).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace irk {

struct Geo {
    int nb, P, G, a, g;
    bool active;
};

__device__ __forceinline__ Geo make_geo(int nb, int G) {
    Geo q;
    q.nb = nb;
    q.P = (nb + 1) >> 1;
    q.G = G;
    q.g = threadIdx.x / nb;
    q.a = threadIdx.x - q.g * nb;
    q.active = q.g < G;
    return q;
}

// streaming (read-once) 128-bit load that does not allocate in L1
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// coherent (L2) load of data produced by other CTAs of the running kernel
__device__ __forceinline__ double2 ld_cg2(const double* p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_cg(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// x pair (x[2p], x[2p+1]) with zero padding for odd nb
template <bool EVEN, bool COHERENT>
__device__ __forceinline__ double2 xpair(const double* x, int p, int nb) {
    if (EVEN) {
        if (COHERENT) return ld_cg2(x + 2 * p);
        return *reinterpret_cast<const double2*>(x + 2 * p);
    } else {
        double2 v;
        v.x = COHERENT ? ld_cg(x + 2 * p) : x[2 * p];
        v.y = (2 * p + 1 < nb) ? (COHERENT ? ld_cg(x + 2 * p + 1) : x[2 * p + 1]) : 0.0;
        return v;
    }
}

// acc[r] += (row a of blk) . xs[r]   for R vectors sharing one block
template <int R, bool EVEN, bool COHERENT>
__device__ __forceinline__ void gemv_shared(const double* __restrict__ blk, const double* const* xs,
                                            const Geo& q, double* acc) {
    const double2* B2 = reinterpret_cast<const double2*>(blk) + q.a;
#pragma unroll 4
    for (int p = q.g; p < q.P; p += q.G) {
        const double2 b = ld_stream(B2 + (size_t)p * q.nb);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 x = xpair<EVEN, COHERENT>(xs[r], p, q.nb);
            acc[r] = fma(b.x, x.x, acc[r]);
            acc[r] = fma(b.y, x.y, acc[r]);
        }
    }
}

// acc += (row a of blk) . x   (single vector)
template <bool EVEN, bool COHERENT>
__device__ __forceinline__ double gemv1(const double* __restrict__ blk, const double* x,
                                        const Geo& q, double acc) {
    const double2* B2 = reinterpret_cast<const double2*>(blk) + q.a;
#pragma unroll 4
    for (int p = q.g; p < q.P; p += q.G) {
        const double2 b = ld_stream(B2 + (size_t)p * q.nb);
        const double2 x2 = xpair<EVEN, COHERENT>(x, p, q.nb);
        acc = fma(b.x, x2.x, acc);
        acc = fma(b.y, x2.y, acc);
    }
    return acc;
}

// Reduce per-thread partials over the G groups: red is [G][nv][nb] in smem.
// After the call, thread (g=0, a) holds the totals in out[v] (v < nv).
// Contains __syncthreads(); every thread of the CTA must call it.
__device__ __forceinline__ void group_reduce(double* red, const double* part, int nv,
                                             const Geo& q, double* out) {
    if (q.active)
        for (int v = 0; v < nv; ++v) red[(q.g * nv + v) * q.nb + q.a] = part[v];
    __syncthreads();
    if (q.active && q.g == 0) {
        for (int v = 0; v < nv; ++v) {
            double s = 0.0;
            for (int gg = 0; gg < q.G; ++gg) s += red[(gg * nv + v) * q.nb + q.a];
            out[v] = s;
        }
    }
    __syncthreads();
}

}  // namespace irk
