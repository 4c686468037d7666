// Development probe for K5: read bandwidth of the GEMV access pattern (every
// warp streams its own contiguous segment) with per-lane 16-byte loads (4 in
// flight + 4 prefetched, as gfq_gemv_kernel) against a per-warp ring of TMA
// bulk copies (S stages of CH bytes, lane 0 issues, mbarrier completion).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_0710_0510_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "device_common.cuh"
using namespace qpk;

__device__ __forceinline__ uint4 ldg_stream(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__global__ void __launch_bounds__(256) lane_loads(const uint32_t* A, uint64_t seg_words, uint64_t nseg, uint32_t* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * 8 + warp; t < nseg; t += uint64_t(gridDim.x) * 8) {
        const uint32_t* row = A + t * seg_words;
        uint64_t j = 4 * lane;
        uint4 cur[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = ldg_stream(row + j + 128 * u);
        for (; j + 1024 - 128 < seg_words; j += 512) {
            uint4 nxt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) nxt[u] = ldg_stream(row + j + 512 + 128 * u);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += cur[u].x ^ cur[u].y ^ cur[u].z ^ cur[u].w;
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += cur[u].x ^ cur[u].y ^ cur[u].z ^ cur[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int S, int CH>
__global__ void __launch_bounds__(256) warp_tma(const uint32_t* A, uint64_t seg_words, uint64_t nseg, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ring = smem + size_t(warp) * S * CH;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(8) * S * CH) + warp * S;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t acc = 0, it = 0;
    constexpr uint64_t CW = CH / 4;
    for (uint64_t t = uint64_t(blockIdx.x) * 8 + warp; t < nseg; t += uint64_t(gridDim.x) * 8) {
        const uint32_t* row = A + t * seg_words;
        const uint64_t nch = seg_words / CW;
        auto issue = [&](uint64_t c, uint32_t slot) {
            mbar_expect_tx(&bars[slot], CH);
            bulk_g2s(ring + slot * CH, row + c * CW, CH, &bars[slot]);
        };
        if (lane == 0)
            for (uint64_t c = 0; c < nch && c < S; ++c) issue(c, (it + c) % S);
        for (uint64_t c = 0; c < nch; ++c, ++it) {
            const uint32_t slot = it % S;
            mbar_wait(&bars[slot], (it / S) & 1);
            const uint4* p = reinterpret_cast<const uint4*>(ring + slot * CH);
#pragma unroll
            for (int u = 0; u < CH / 512; ++u) {
                const uint4 v = p[u * 32 + lane];
                acc += v.x ^ v.y ^ v.z ^ v.w;
            }
            __syncwarp();
            if (lane == 0 && c + S < nch) issue(c + S, slot);
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <class F>
float timeit(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

template <int S, int CH>
void run_tma(const uint32_t* A, uint64_t seg_words, uint64_t nseg, uint32_t* out, int sms, int per_sm, double bytes) {
    const size_t smem = size_t(8) * S * CH + 8 * S * 8;
    cudaFuncSetAttribute(warp_tma<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const float ms = timeit([&] { warp_tma<S, CH><<<sms * per_sm, 256, smem>>>(A, seg_words, nseg, out); });
    printf("  warp TMA ring S=%d CH=%d, %d CTAs/SM: %.1f us  %.0f GB/s  (%s)\n", S, CH, per_sm, ms * 1e3, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t total_words = uint64_t(1) << 27;  // 512 MB
    uint32_t *A, *out;
    cudaMalloc(&A, total_words * 4);
    cudaMalloc(&out, 64);
    cudaMemset(A, 1, total_words * 4);
    for (uint64_t seg_words : {uint64_t(8192), uint64_t(1) << 15, uint64_t(1) << 17}) {
        const uint64_t nseg = total_words / seg_words;
        const double bytes = double(total_words) * 4;
        printf("segments of %llu KB:\n", (unsigned long long)(seg_words * 4 / 1024));
        for (int per_sm : {4, 8}) {
            const float ms = timeit([&] { lane_loads<<<sms * per_sm, 256>>>(A, seg_words, nseg, out); });
            printf("  per-lane LDG.128 x(4+4), %d CTAs/SM: %.1f us  %.0f GB/s\n", per_sm, ms * 1e3, bytes / ms / 1e6);
        }
        run_tma<4, 2048>(A, seg_words, nseg, out, sms, 3, bytes);
        run_tma<6, 2048>(A, seg_words, nseg, out, sms, 2, bytes);
        run_tma<3, 4096>(A, seg_words, nseg, out, sms, 2, bytes);
        run_tma<2, 8192>(A, seg_words, nseg, out, sms, 1, bytes);
        run_tma<4, 4096>(A, seg_words, nseg, out, sms, 1, bytes);
    }
    return 0;
}
