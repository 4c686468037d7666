// Development probe: how much of a warp's re-pack (integer work on its 64
// accumulators) does the sibling warp's DMMA stream hide?  The K4 consumer
// structure without memory: per warp a loop of "stages" of 128 DMMAs (4 k-steps
// x 32 tiles) and a re-pack of all accumulators every 4 stages.
//   mode 0: no re-pack            1: SWAR REDQ re-pack, warps w / w+4 two stages apart
//   mode 2: same, all warps in the same stage
//   mode 3: only warps 0-3 re-pack (4-7 run DMMA only)
//   mode 4: 4 warps only (one per sub-partition), with re-pack (nothing to overlap)
//   mode 5: lane fold, staggered   6: 4 warps only, no re-pack
//   mode 7: REDQ re-pack sprinkled: acc (i, j) re-packed right before its first
//           DMMA of the stage after the re-pack point (same warp interleave)
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_0710_0510_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "gfq_matmul.cuh"

using namespace qpk;

template <int MODE>
__global__ void __launch_bounds__(288, 1) probe(double* sink, int stages, double a0, double b0) {
    const int warp = threadIdx.x >> 5;
    if (warp >= ((MODE == 4 || MODE == 6) ? 4 : 8)) return;
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = kTwo52;
    double af[8], bf[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) af[i] = a0 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = b0 + j;
    int phase = 3;
    if (MODE == 1 || MODE == 5 || MODE == 7) phase = 3 - ((warp & 3) + (warp >> 2) * 2) % 4;
    const bool do_repack = MODE != 0 && MODE != 6 && !(MODE == 3 && warp >= 4);
    for (int s = 0; s < stages; ++s) {
        if (MODE == 7 && do_repack && s > 0 && ((s - 1) & 3) == phase) {
            // first k-step with the re-pack of each accumulator pair in front of its DMMA
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[i][j][0] = redq_repack_swar3<5, 10>(acc[i][j][0]);
                    acc[i][j][1] = redq_repack_swar3<5, 10>(acc[i][j][1]);
                    dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
                }
#pragma unroll 1
            for (int kk = 1; kk < 4; ++kk) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
            continue;
        }
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (MODE != 7 && do_repack && (s & 3) == phase) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (MODE == 5) {
                        acc[i][j][0] = repack_fold3<5, 10, 6>(acc[i][j][0]);
                        acc[i][j][1] = repack_fold3<5, 10, 6>(acc[i][j][1]);
                    } else {
                        acc[i][j][0] = redq_repack_swar3<5, 10>(acc[i][j][0]);
                        acc[i][j][1] = redq_repack_swar3<5, 10>(acc[i][j][1]);
                    }
                }
        }
    }
    double sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sum += acc[i][j][0] + acc[i][j][1];
    if (sum == 12345.0) sink[0] = sum;
}

template <int MODE>
void run(double* sink, int sms, const char* what) {
    const int stages = 4096;
    probe<MODE><<<sms, 288>>>(sink, 64, 1.0, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<MODE><<<sms, 288>>>(sink, stages, 1.0, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const int warps = (MODE == 4 || MODE == 6) ? 4 : 8;
    const double flops = double(sms) * warps * stages * 128.0 * 512;
    printf("mode %d (%s): %.3f ms, DMMA %.2f TFLOP/s  err=%s\n", MODE, what, best, flops / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* sink;
    cudaMalloc(&sink, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>(sink, sms, "8 warps, no re-pack");
    run<1>(sink, sms, "8 warps, REDQ re-pack staggered");
    run<2>(sink, sms, "8 warps, REDQ re-pack same stage");
    run<3>(sink, sms, "8 warps, only warps 0-3 re-pack");
    run<4>(sink, sms, "4 warps, REDQ re-pack");
    run<6>(sink, sms, "4 warps, no re-pack");
    run<5>(sink, sms, "8 warps, fold staggered");
    run<7>(sink, sms, "8 warps, REDQ re-pack inside the next stage's first k-step");
    return 0;
}
