// Development probe: what does integer work between DMMA stages cost the
// sibling warp's DMMA stream -- per instruction, by instruction type?  Same
// structure as repack_overlap_probe.cu (stages of 128 DMMAs, synthetic
// "re-pack" of all 64 accumulators every 4 stages, warps w / w+4 two stages
// apart).  TYPE 0: ALU rounds (SHF + LOP3 + IADD3 per 32-bit half), 1: IMAD
// rounds, 2: IMAD.HI rounds, 3: fp64 DADD rounds (one per accumulator).
#include <cstdio>
#include <cuda_runtime.h>

#include "gfq_matmul.cuh"
using namespace qpk;

template <int TYPE, int ROUNDS>
__device__ __forceinline__ double synth(double a) {
    uint64_t b = dbits(a);
    uint32_t lo = uint32_t(b), hi = uint32_t(b >> 32);
    if (TYPE == 3) {
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) a = __dadd_rz(a, 3.0);
        return a;
    }
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
        if (TYPE == 0) {
            lo = ((lo >> 3) ^ lo) + 0x1234567u;
            hi = ((hi >> 5) ^ hi) + 0x7654321u;
        } else if (TYPE == 1) {
            lo = lo * 0x9E3779B9u + 7u;
            hi = hi * 0x85EBCA6Bu + 5u;
        } else {
            lo = __umulhi(lo, 0xAAAAAAABu) + 0x40000000u;
            hi = __umulhi(hi, 0xAAAAAAABu) + 0x40000000u;
        }
    }
    return __longlong_as_double((long long)((uint64_t(hi) << 32) | lo));
}

template <int TYPE, int ROUNDS, int NW>
__global__ void __launch_bounds__(288, 1) probe(double* sink, int stages, double a0, double b0) {
    const int warp = threadIdx.x >> 5;
    if (warp >= NW) return;
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
    const int phase = 3 - ((warp & 3) + (warp >> 2) * 2) % 4;
    for (int s = 0; s < stages; ++s) {
#pragma unroll 1
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (ROUNDS > 0 && (s & 3) == phase) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[i][j][0] = synth<TYPE, ROUNDS>(acc[i][j][0]);
                    acc[i][j][1] = synth<TYPE, ROUNDS>(acc[i][j][1]);
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

template <int TYPE, int ROUNDS, int NW>
float run(double* sink, int sms) {
    const int stages = 4096;
    probe<TYPE, ROUNDS, NW><<<sms, 288>>>(sink, 64, 1.0, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<TYPE, ROUNDS, NW><<<sms, 288>>>(sink, stages, 1.0, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

template <int TYPE, int ROUNDS>
void both(double* sink, int sms, float b8, float b4, int per_round) {
    const float t8 = run<TYPE, ROUNDS, 8>(sink, sms), t4 = run<TYPE, ROUNDS, 4>(sink, sms);
    // per SMSP: 8-warp runs hold 2 x 1024 re-packs x 64 accumulators, 4-warp runs 1024 x 64
    const double clk = 1.965e6;  // clocks per ms
    const int n = per_round * ROUNDS;
    printf("type %d, %2d instr/acc: 8 warps %.3f ms (+%.1f%%, %.2f clk lost per instr) | 4 warps %.3f ms (%.2f clk per instr serial)\n",
           TYPE, n, t8, 100.0 * (t8 - b8) / b8, (t8 - b8) * clk / (2.0 * 1024 * 64 * n), t4,
           (t4 - b4) * clk / (1024.0 * 64 * n));
}

int main() {
    double* sink;
    cudaMalloc(&sink, 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const float b8 = run<0, 0, 8>(sink, sms), b4 = run<0, 0, 4>(sink, sms);
    printf("base: 8 warps %.3f ms, 4 warps %.3f ms\n", b8, b4);
    both<0, 2>(sink, sms, b8, b4, 6);
    both<0, 5>(sink, sms, b8, b4, 6);
    both<1, 6>(sink, sms, b8, b4, 2);
    both<1, 15>(sink, sms, b8, b4, 2);
    both<2, 3>(sink, sms, b8, b4, 4);
    both<2, 6>(sink, sms, b8, b4, 4);
    both<3, 2>(sink, sms, b8, b4, 1);
    both<3, 6>(sink, sms, b8, b4, 1);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
