// Does fp64 MMA (DMMA) or DFMA issue overlap with independent integer work
// on the same SM sub-partition?  Development probe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/overlap_probe.cu -o scripts/op_bin
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int NMMA, int NINT, bool DFMA_MODE>
__global__ void __launch_bounds__(256) probe(double* sink, uint32_t* isink, int iters) {
    double d[8][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = c;
    uint32_t x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 7 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < NMMA; ++m) {
            if (DFMA_MODE) {
                d[m & 7][0] = fma(d[m & 7][0], a, b);
                d[m & 7][1] = fma(d[m & 7][1], a, b);
            } else {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(d[m & 7][0]), "+d"(d[m & 7][1])
                             : "d"(a), "d"(b));
            }
#pragma unroll
            for (int k = 0; k < NINT; ++k) x[k & 7] = x[k & 7] * 0x9E3779B1u + (x[(k + 3) & 7] >> 7);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    uint32_t t = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) t ^= x[c];
    if (s == 1.2345) sink[0] = s;
    if (t == 12345) isink[0] = t;
}

template <int NMMA, int NINT, bool DF>
void run(const char* name, double* s, uint32_t* is) {
    const int iters = 2000, blocks = 148 * 2;
    probe<NMMA, NINT, DF><<<blocks, 256>>>(s, is, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<NMMA, NINT, DF><<<blocks, 256>>>(s, is, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // flop per launch: DMMA warp-instr = 512 flop; DFMA pair per thread = 4 flop
    const double warps = blocks * 8.0;
    const double flop = DF ? warps * 32 * iters * NMMA * 4.0 : warps * iters * NMMA * 512.0;
    printf("%-28s %8.3f ms  %6.2f TFLOP/s  int-ops/mma=%d\n", name, ms, flop / (ms * 1e-3) / 1e12, NINT);
}

int main() {
    double* s;
    uint32_t* is;
    cudaMalloc(&s, 64);
    cudaMalloc(&is, 64);
    run<32, 0, false>("dmma", s, is);
    run<32, 4, false>("dmma + 4 int/mma", s, is);
    run<32, 8, false>("dmma + 8 int/mma", s, is);
    run<32, 16, false>("dmma + 16 int/mma", s, is);
    run<8, 0, false>("int only (8 dmma/32 int)", s, is);
    run<32, 0, true>("dfma x2", s, is);
    run<32, 1, true>("dfma x2 + 1 int", s, is);
    run<32, 2, true>("dfma x2 + 2 int", s, is);
    run<32, 4, true>("dfma x2 + 4 int", s, is);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
