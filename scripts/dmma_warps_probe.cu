// Development probe: DMMA.8x8x4 throughput vs consumer warps per SM
// sub-partition (1 CTA per SM, W warps, each with 32 independent
// accumulator tiles like the K4 warp tile).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void probe(double* sink, int iters) {
    double acc[8][4][2];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double a = threadIdx.x * 1e-9, b = blockIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a + i, b + j);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
    if (s == 12345.0) sink[0] = s;
}

int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 12, 16}) {
        const int iters = 4000;
        probe<<<sms, warps * 32>>>(sink, 10);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<sms, warps * 32>>>(sink, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = double(sms) * warps * iters * 32 * 512;
        printf("warps/SM %2d (per SMSP %d): %.2f TFLOP/s\n", warps, warps / 4, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
