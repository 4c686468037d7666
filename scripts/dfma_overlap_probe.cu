// Development probe: does integer work overlap a DFMA contraction (where it
// does not overlap DMMA)?  Per thread an 8x8 register tile updated by rank-1
// steps from shared memory (8 + 8 doubles per k as LDS.128), 8 warps per CTA;
// every 64 k-steps the canonical re-pack (24 integer instructions) of all 64
// accumulators.
//   mode 0: no re-pack   1: re-pack burst every 64 k   2: re-pack spread (one row of 8 accumulators per 8 k)
#include <cstdio>
#include <cuda_runtime.h>

#include "gfq_matmul.cuh"
using namespace qpk;

template <int MODE>
__global__ void __launch_bounds__(256, 1) probe(double* sink, const double* frag, int chunks) {
    __shared__ __align__(16) double sm[16 * 128];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) sm[i] = frag[i & 1023];
    __syncthreads();
    const int ty = lane >> 2, tx = lane & 3;
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = kTwo52;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll 1
        for (int k8 = 0; k8 < 8; ++k8) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const double2* pa = reinterpret_cast<const double2*>(sm + ((k8 * 8 + kk) & 15) * 128 + ty * 8);
                const double2* pb = reinterpret_cast<const double2*>(sm + ((k8 * 8 + kk) & 15) * 128 + 64 + tx * 8);
                double a[8], b[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 va = pa[i], vb = pb[i];
                    a[2 * i] = va.x, a[2 * i + 1] = va.y, b[2 * i] = vb.x, b[2 * i + 1] = vb.y;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
                if (MODE == 2) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[kk][j] = redq_repack_canon3(acc[kk][j]);
                }
            }
        }
        if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = redq_repack_canon3(acc[i][j]);
        }
    }
    double sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) sum += acc[i][j];
    if (sum == 12345.0) sink[0] = sum;
}

template <int MODE>
void run(double* sink, const double* frag, int sms, const char* what) {
    const int chunks = 2048;
    probe<MODE><<<sms, 256>>>(sink, frag, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<MODE><<<sms, 256>>>(sink, frag, chunks);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = double(sms) * 256 * chunks * 64.0 * 64 * 2;
    printf("mode %d (%s): %.3f ms, DFMA %.2f TFLOP/s  err=%s\n", MODE, what, best, flops / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double *sink, *frag;
    cudaMalloc(&sink, 64);
    cudaMalloc(&frag, 1024 * 8);
    cudaMemset(frag, 0, 1024 * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>(sink, frag, sms, "no re-pack");
    run<1>(sink, frag, sms, "canonical re-pack burst every 64 k");
    run<2>(sink, frag, sms, "canonical re-pack spread, 8 accumulators per k");
    return 0;
}
