// Two warps per SM sub-partition: warp w < 4 issues only DMMA, warp w >= 4
// (same sub-partition w%4) runs only an integer loop (or idles).  Does the
// integer warp slow the DMMA warp?  Development probe.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int MODE>  // 0: int warps idle, 1: int warps busy, 2: all 8 warps DMMA
__global__ void __launch_bounds__(256, 1) probe(double* sink, uint32_t* isink, int iters) {
    const int warp = threadIdx.x >> 5;
    if (warp < 4 || MODE == 2) {
        double d[16][2];
        const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
#pragma unroll
        for (int c = 0; c < 16; ++c) d[c][0] = d[c][1] = c;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int c = 0; c < 16; ++c)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(d[c][0]), "+d"(d[c][1])
                             : "d"(a), "d"(b));
        double s = 0;
#pragma unroll
        for (int c = 0; c < 16; ++c) s += d[c][0] + d[c][1];
        if (s == 1.2345) sink[0] = s;
    } else if (MODE == 1) {
        uint32_t x[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 7 + c;
        for (int it = 0; it < iters * 8; ++it)
#pragma unroll
            for (int c = 0; c < 16; ++c) x[c] = x[c] * 0x9E3779B1u + 0x7F4A7C15u;
        uint32_t t = 0;
#pragma unroll
        for (int c = 0; c < 16; ++c) t ^= x[c];
        if (t == 12345) isink[0] = t;
    }
}

template <int MODE>
float run(double* s, uint32_t* is, int iters) {
    probe<MODE><<<148, 256>>>(s, is, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<148, 256>>>(s, is, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    double* s;
    uint32_t* is;
    cudaMalloc(&s, 64);
    cudaMalloc(&is, 64);
    const int iters = 4000;
    const double dmma_warps = 148 * 4.0;
    for (int m = 0; m < 3; ++m) {
        float ms = m == 0 ? run<0>(s, is, iters) : m == 1 ? run<1>(s, is, iters) : run<2>(s, is, iters);
        const double flop = (m == 2 ? 2 : 1) * dmma_warps * iters * 16 * 512.0;
        printf("mode %d: %.3f ms  %.2f TFLOP/s  (%s)\n", m, ms, flop / (ms * 1e-3) / 1e12,
               m == 0 ? "1 DMMA warp per SMSP, partner idle"
                      : m == 1 ? "1 DMMA warp + 1 integer warp per SMSP" : "2 DMMA warps per SMSP");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
