// Development probe: does scalar fp64 / integer work on the other warp of a
// sub-partition slow DMMA down?  Warps 0-3 run DMMA chains; warps 4-7 run
// `mode` work until they finish: 0 idle, 1 fp64 DADD/DMUL chains, 2 64-bit
// logic/shift/add, 3 64-bit multiply, 4 32-bit IMAD, 5 32-bit logic/shift/add.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void probe(double* sink, int iters, int mode) {
    const int warp = threadIdx.x >> 5;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp < 4) {
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
        __syncwarp();
        if ((threadIdx.x & 31) == 0) atomicAdd((int*)&done, 1);
    } else if (mode == 1) {
        double x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
        while (done < 4)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __dadd_rz(__dmul_ru(x[i], 0.3333333), 4503599627370496.0) - 4503599627370496.0;
        double s = 0;
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 12345.0) sink[1] = s;
    } else if (mode == 2) {
        unsigned long long x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
        while (done < 4)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = ((x[i] & 0x3333333333ull) + (x[i] >> 10)) ^ (x[i] << 3);
        unsigned long long s = 0;
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 12345) sink[2] = s;
    } else if (mode == 3) {
        unsigned long long x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
        while (done < 4)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = x[i] * 0x9E3779B97F4A7C15ull + 7;
        unsigned long long s = 0;
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 12345) sink[3] = s;
    } else if (mode == 4) {
        unsigned x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
        while (done < 4)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = x[i] * 0x9E3779B9u + 7;
        unsigned s = 0;
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 12345) sink[4] = s;
    } else if (mode == 5) {
        unsigned x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
        while (done < 4)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = ((x[i] & 0x33333333u) + (x[i] >> 10)) ^ (x[i] << 3);
        unsigned s = 0;
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 12345) sink[5] = s;
    }
}

int main() {
    double* sink;
    cudaMalloc(&sink, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode : {0, 1, 2, 3, 4, 5}) {
        const int iters = 4000;
        probe<<<sms, 256>>>(sink, 10, mode);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<sms, 256>>>(sink, iters, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = double(sms) * 4 * iters * 32 * 512;
        printf("mode %d: DMMA %.2f TFLOP/s (%.3f ms)  err=%s\n", mode, flops / (ms * 1e-3) / 1e12, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
