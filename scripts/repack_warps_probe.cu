// Development probe: does a third / fourth DMMA warp per sub-partition hide a
// warp's re-pack?  16 warps x 32 accumulators (32x32 warp tiles), re-packs of
// the four warps of a sub-partition in four different stages.
//   mode 0: no re-pack   1: canonical fold re-pack (24 instructions)   2: SWAR REDQ
#include <cstdio>
#include <cuda_runtime.h>

#include "gfq_matmul.cuh"
using namespace qpk;

template <int MODE, int NW>
__global__ void __launch_bounds__(NW * 32, 1) probe(double* sink, const double* frag, int stages) {
    __shared__ double sm[12 * 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 12 * 32; i += blockDim.x) sm[i] = frag[i];
    __syncthreads();
    constexpr int MT = NW == 16 ? 4 : 8;
    double acc[MT][4][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = kTwo52;
    const int phase = NW == 16 ? (warp >> 2) : 3 - ((warp & 3) + (warp >> 2) * 2) % 4;
    for (int s = 0; s < stages; ++s) {
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
            double af[MT], bf[4];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = sm[i * 32 + lane];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = sm[(8 + j) * 32 + lane];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (MODE != 0 && (s & 3) == phase) {
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        acc[i][j][h] = MODE == 1 ? redq_repack_canon3(acc[i][j][h]) : redq_repack_swar3<5, 10>(acc[i][j][h]);
        }
    }
    double sum = 0;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sum += acc[i][j][0] + acc[i][j][1];
    if (sum == 12345.0) sink[0] = sum;
}

template <int MODE, int NW>
void run(double* sink, const double* frag, int sms) {
    const int stages = 4096;
    probe<MODE, NW><<<sms, NW * 32>>>(sink, frag, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<MODE, NW><<<sms, NW * 32>>>(sink, frag, stages);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = double(sms) * NW * stages * 4.0 * (NW == 16 ? 16 : 32) * 512;
    printf("%2d warps, mode %d: %.3f ms, DMMA %.2f TFLOP/s  err=%s\n", NW, MODE, best, flops / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double *sink, *frag;
    cudaMalloc(&sink, 64);
    cudaMalloc(&frag, 12 * 32 * 8);
    cudaMemset(frag, 0, 12 * 32 * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 8>(sink, frag, sms);
    run<1, 8>(sink, frag, sms);
    run<2, 8>(sink, frag, sms);
    run<0, 16>(sink, frag, sms);
    run<1, 16>(sink, frag, sms);
    run<2, 16>(sink, frag, sms);
    return 0;
}
