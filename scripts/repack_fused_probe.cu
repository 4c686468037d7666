// Development probe: the REDQ re-pack spread over the k-steps of a chunk and
// issued inside the DMMA shadows of the same warp.  A chunk = 16 k-steps of
// 32 DMMAs; in k-step j the accumulator tiles {2j, 2j+1} are re-packed right
// before their DMMA, so each accumulator is re-packed every 64 K-steps and
// the integer work rides in the 14 idle issue cycles after every DMMA.
//   FUSED 0: no re-pack   1: fused swar3 REDQ   2: fused fold
// 256 threads (8 warps): 255-register cap.
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>

#include "gfq_matmul.cuh"
using namespace qpk;

#ifndef PROBE_THREADS
#define PROBE_THREADS 256
#endif

template <int FUSED>
__global__ void __launch_bounds__(PROBE_THREADS, 1) probe(double* sink, const double* frag, int chunks) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16 * 12 * 32; i += blockDim.x) sm[i] = frag[i & 1023];
    __syncthreads();
    if (warp >= 8) return;
    double acc[32][2];
#pragma unroll
    for (int t = 0; t < 32; ++t) acc[t][0] = acc[t][1] = kTwo52;
    for (int c = 0; c < chunks; ++c) {
        auto step = [&](auto jc) {
            constexpr int j = decltype(jc)::value;
            double af[8], bf[4];
            const double* p = sm + (j * 12) * 32 + lane;
#pragma unroll
            for (int i = 0; i < 8; ++i) af[i] = p[i * 32];
#pragma unroll
            for (int i = 0; i < 4; ++i) bf[i] = p[(8 + i) * 32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                if (FUSED && (t >> 1) == j) {
                    if (FUSED == 1) {
                        acc[t][0] = redq_repack_swar3<5, 10>(acc[t][0]);
                        acc[t][1] = redq_repack_swar3<5, 10>(acc[t][1]);
                    } else {
                        acc[t][0] = repack_fold3<5, 10, 6>(acc[t][0]);
                        acc[t][1] = repack_fold3<5, 10, 6>(acc[t][1]);
                    }
                }
                dmma884(acc[t][0], acc[t][1], af[t >> 2], bf[t & 3]);
            }
        };
        [&]<int... J>(std::integer_sequence<int, J...>) { (step(std::integral_constant<int, J>{}), ...); }
        (std::make_integer_sequence<int, 16>{});
    }
    double sum = 0;
#pragma unroll
    for (int t = 0; t < 32; ++t) sum += acc[t][0] + acc[t][1];
    if (sum == 12345.0) sink[0] = sum;
}

template <int FUSED>
void run(double* sink, const double* frag, int sms, const char* what) {
    const int chunks = 1024;
    const size_t smem = 16 * 12 * 32 * 8;
    cudaFuncSetAttribute(probe<FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<FUSED><<<sms, PROBE_THREADS, smem>>>(sink, frag, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<FUSED><<<sms, PROBE_THREADS, smem>>>(sink, frag, chunks);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = double(sms) * 8 * chunks * 16 * 32.0 * 512;
    printf("fused %d (%s): %.3f ms, DMMA %.2f TFLOP/s  err=%s\n", FUSED, what, best, flops / (best * 1e-3) / 1e12,
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
    run<1>(sink, frag, sms, "REDQ re-pack fused, 2 tiles per k-step");
    run<2>(sink, frag, sms, "fold fused");
    return 0;
}
