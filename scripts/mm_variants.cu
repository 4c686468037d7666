// Mainloop experiment for K4: fp64 DMMA throughput of pipeline variants
// (no REDQ, no epilogue beyond a checksum store).  Development tool only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/mm_variants.cu -o /tmp/mmv
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_0710_0510_b200/csrc/device_common.cuh"

using namespace qpk;

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, PAD = 4, LDS_ = BM + PAD;
constexpr int MT = 8, NT = 4;
constexpr size_t STAGE_DOUBLES = size_t(2) * BK * LDS_;

template <bool VOL>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    if (VOL)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    else
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// PRODUCER: dedicated 9th warp;  PREFETCH: double-buffered fragments;  VOL: volatile asm
template <bool PRODUCER, bool PREFETCH, bool VOL>
__global__ void __launch_bounds__(PRODUCER ? 288 : 256, 1)
    mm_kernel(const double* __restrict__ at, const double* __restrict__ bm, int K, int m_pad, int n_pad,
              double* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    double* stages = reinterpret_cast<double*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_DOUBLES * 8);
    uint64_t* empty = full + STAGES;
    uint32_t* freed = reinterpret_cast<uint32_t*>(empty + STAGES);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t m0 = uint64_t(blockIdx.y) * BM, n0 = uint64_t(blockIdx.x) * BN;
    const int KT = K / BK;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 8);
            freed[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    auto refill = [&](int s, int kt) {
        if (lane == 0) mbar_expect_tx(&full[s], 2 * BK * BM * 8);
        __syncwarp();
        double* sa = stages + s * STAGE_DOUBLES;
        double* sb = sa + BK * LDS_;
        const uint64_t k0 = uint64_t(kt) * BK;
        if (lane < BK)
            bulk_g2s(sa + lane * LDS_, at + (k0 + lane) * m_pad + m0, BM * 8, &full[s]);
        else
            bulk_g2s(sb + (lane - BK) * LDS_, bm + (k0 + lane - BK) * n_pad + n0, BN * 8, &full[s]);
    };
    if (PRODUCER) {
        if (warp == 8) {
            for (int kt = 0; kt < KT; ++kt) {
                const int s = kt % STAGES;
                if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
                refill(s, kt);
            }
            return;
        }
    } else if (warp == 0) {
        for (int s = 0; s < STAGES && s < KT; ++s) refill(s, s);
    }
    const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32, lr = lane >> 2, lc4 = lane & 3;
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double af[2][MT], bf[2][NT];
    auto load = [&](int buf, const double* sa, const double* sb, int kk) {
        const double* pa = sa + (kk * 4 + lc4) * LDS_ + wm + lr;
        const double* pb = sb + (kk * 4 + lc4) * LDS_ + wn + lr;
#pragma unroll
        for (int i = 0; i < MT; ++i) af[buf][i] = pa[i * 8];
#pragma unroll
        for (int j = 0; j < NT; ++j) bf[buf][j] = pb[j * 8];
    };
    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&full[s], (kt / STAGES) & 1);
        const double* sa = stages + s * STAGE_DOUBLES;
        const double* sb = sa + BK * LDS_;
        if (PREFETCH) {
            load(0, sa, sb, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int cur = kk & 1;
                if (kk < 3) load(cur ^ 1, sa, sb, kk + 1);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma<VOL>(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
            }
        } else {
#pragma unroll 1
            for (int kk = 0; kk < 4; ++kk) {
                load(0, sa, sb, kk);
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma<VOL>(acc[i][j][0], acc[i][j][1], af[0][i], bf[0][j]);
            }
        }
        __syncwarp();
        if (PRODUCER) {
            if (lane == 0) mbar_arrive(&empty[s]);
        } else {
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&freed[s], 1u) == 7;
                if (last) freed[s] = 0;
            }
            if (__shfl_sync(0xffffffffu, last, 0) && kt + STAGES < KT) refill(s, kt + STAGES);
        }
    }
    double sum = 0;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) sum += acc[i][j][0] + acc[i][j][1];
    out[(blockIdx.y * gridDim.x + blockIdx.x) * 256 + tid] = sum;
}

template <bool P, bool F, bool V>
void run(const char* name, const double* at, const double* b, int n, double* out) {
    auto kern = mm_kernel<P, F, V>;
    const size_t smem = STAGES * STAGE_DOUBLES * 8 + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    dim3 grid(n / BN, n / BM);
    const int threads = P ? 288 : 256;
    for (int w = 0; w < 2; ++w) kern<<<grid, threads, smem>>>(at, b, n, n, n, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int r = 0; r < reps; ++r) kern<<<grid, threads, smem>>>(at, b, n, n, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    printf("%-28s n=%d  %.3f ms  %.2f TFLOP/s  regs=%d local=%zu  err=%s\n", name, n, ms,
           2.0 * n * n * double(n) / (ms * 1e-3) / 1e12, fa.numRegs, fa.localSizeBytes,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 4096;
    double *at, *b, *out;
    cudaMalloc(&at, size_t(n) * n * 8);
    cudaMalloc(&b, size_t(n) * n * 8);
    cudaMalloc(&out, size_t(n) * n * 8);
    std::vector<double> h(size_t(n) * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = double((i * 2654435761u) % 7);
    cudaMemcpy(at, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    run<true, false, true>("producer/noprefetch/vol", at, b, n, out);
    run<true, false, false>("producer/noprefetch/novol", at, b, n, out);
    run<true, true, true>("producer/prefetch/vol", at, b, n, out);
    run<false, false, true>("lastarr/noprefetch/vol", at, b, n, out);
    run<false, true, true>("lastarr/prefetch/vol", at, b, n, out);
    run<false, true, false>("lastarr/prefetch/novol", at, b, n, out);
    return 0;
}
