// fp64 peak probes for the K4 roofline denominator: a DFMA
// chain kernel and a DMMA (mma.sync m8n8k4 f64) chain kernel, each with
// enough independent accumulators per thread/warp to saturate its pipe.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace qpk {

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) probe_dfma_kernel(double* sink, int iters) {
    double a[kChains];
    const double x = 0.9999999 + threadIdx.x * 1e-12, y = 1e-7;
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = c * 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], x, y);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c];
    if (s == 12345.678) sink[0] = s;  // never true; keeps the chains alive
}

__global__ void __launch_bounds__(256) probe_dmma_kernel(double* sink, int iters) {
    double d[kChains][2];
    const double a = 0.999 + (threadIdx.x & 31) * 1e-9, b = 1e-3;
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) sink[0] = s;
}

}  // namespace

cudaError_t launch_probe_dfma(double* sink, int iters, uint64_t* flops, cudaStream_t s) {
    const unsigned blocks = num_sms() * 8;
    probe_dfma_kernel<<<blocks, 256, 0, s>>>(sink, iters);
    *flops = uint64_t(2) * kChains * uint64_t(iters) * blocks * 256;
    return cudaGetLastError();
}

cudaError_t launch_probe_dmma(double* sink, int iters, uint64_t* flops, cudaStream_t s) {
    const unsigned blocks = num_sms() * 8;
    probe_dmma_kernel<<<blocks, 256, 0, s>>>(sink, iters);
    // each warp-level m8n8k4 is 8*8*4 = 256 FMAs
    *flops = uint64_t(2) * 256 * kChains * uint64_t(iters) * blocks * (256 / 32);
    return cudaGetLastError();
}

}  // namespace qpk
