// Pipeline experiment for the streaming kernels: the real C2 REDQ op under
// several CTA pipelines.  Development tool only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_0710_0510_b200/csrc \
//        scripts/stream_variants.cu -o scripts/sv_bin
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "stream_kernels.cuh"

using namespace qpk;
using Op = RedqOp<7, 4, CtConst<5, 7>>;

struct XorOp {
    static constexpr int IN0 = 3, IN1 = 3, OUT = 3, R = 4;
    __host__ __device__ uint32_t tables_words() const { return 0; }
    __host__ __device__ const uint32_t* tables_src() const { return nullptr; }
    __device__ void apply(const uint32_t* a, const uint32_t* b, uint32_t (&ow)[3], uint32_t, uint32_t&) const {
        ow[0] = a[0] ^ b[0], ow[1] = a[1] ^ b[1], ow[2] = a[2] ^ b[2];
    }
};

// V_CTA: all threads consume; thread 0 produces after a CTA barrier; the CTA
// stores one output tile.  NT threads, R records per thread, S stages.
template <class OpT, int NT, int RR, int S>
__global__ void __launch_bounds__(NT) v_cta(const OpT op, const uint8_t* __restrict__ in0,
                                            const uint8_t* __restrict__ in1, uint8_t* __restrict__ out,
                                            uint64_t n_tiles) {
    constexpr int R = 4, TILE = NT * R * RR;
    constexpr uint32_t B0 = OpT::IN0 * TILE, B1 = OpT::IN1 * TILE, BO = OpT::OUT * TILE;
    constexpr int W0 = R * OpT::IN0 / 4, W1 = R * OpT::IN1 / 4, WO = R * OpT::OUT / 4;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* s_in = smem;
    uint8_t* s_out = smem + S * (B0 + B1);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_out + 2 * BO);
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(bars + S);
    const uint32_t tab = smem_addr(s_tab);
    const int tid = threadIdx.x;
    for (uint32_t i = tid; i < op.tables_words(); i += NT) s_tab[i] = op.tables_src()[i];
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint64_t pol = 0;
    auto issue = [&](int s, uint64_t t) {
        mbar_expect_tx(&bars[s], B0 + B1);
        bulk_g2s_stream(s_in + s * (B0 + B1), in0 + t * B0, B0, &bars[s], pol);
        if (B1) bulk_g2s_stream(s_in + s * (B0 + B1) + B0, in1 + t * B1, B1, &bars[s], pol);
    };
    if (tid == 0) {
        pol = policy_evict_first();
        for (int s = 0; s < S; ++s)
            if (blockIdx.x + uint64_t(s) * gridDim.x < n_tiles) issue(s, blockIdx.x + uint64_t(s) * gridDim.x);
    }
    uint32_t err = 0, it = 0;
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int s = it % S, os = it & 1;
        if (tid == 0) bulk_wait_read<1>();
        mbar_wait(&bars[s], (it / S) & 1);
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
            const int run = rr * NT + tid;
            uint32_t a[W0 > 0 ? W0 : 1], b[W1 > 0 ? W1 : 1];
            lds_run<W0>(s_in + s * (B0 + B1) + run * (R * OpT::IN0), a);
            lds_run<W1>(s_in + s * (B0 + B1) + B0 + run * (R * OpT::IN1), b);
            uint32_t ow[WO];
            op.apply(a, b, ow, tab, err);
            uint32_t* d = reinterpret_cast<uint32_t*>(s_out + os * BO) + run * WO;
#pragma unroll
            for (int i = 0; i < WO; ++i) d[i] = ow[i];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            bulk_s2g(out + t * BO, s_out + os * BO, BO);
            bulk_commit();
            const uint64_t nx = t + uint64_t(S) * gridDim.x;
            if (nx < n_tiles) issue(s, nx);
        }
    }
    if (tid == 0) bulk_wait_all<0>();
}

// plain LDG/STG: each thread 4 consecutive words, vector loads, byte-packed
// stores through registers (no smem staging).  Grid-stride.
__global__ void __launch_bounds__(256) v_ldg(const Op op, const uint8_t* __restrict__ in0, uint8_t* __restrict__ out,
                                             uint64_t n_runs) {
    __shared__ uint32_t s_tab[1024];
    for (uint32_t i = threadIdx.x; i < op.tables_words(); i += 256) s_tab[i] = op.tables_src()[i];
    __syncthreads();
    const uint32_t tab = smem_addr(s_tab);
    uint32_t err = 0;
    for (uint64_t run = uint64_t(blockIdx.x) * 256 + threadIdx.x; run < n_runs; run += uint64_t(gridDim.x) * 256) {
        const uint4* p = reinterpret_cast<const uint4*>(in0 + run * 32);
        uint4 x = __ldcs(p), y = __ldcs(p + 1);
        uint32_t a[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}, b[1], ow[7];
        op.apply(a, b, ow, tab, err);
        uint32_t* d = reinterpret_cast<uint32_t*>(out + run * 28);
#pragma unroll
        for (int i = 0; i < 7; ++i) __stcs(d + i, ow[i]);
    }
}

template <class F>
float timeit(F f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10;
}

int main() {
    const uint64_t n = 1ull << 26;
    double* w;
    uint8_t* o;
    cudaMalloc(&w, n * 8);
    cudaMalloc(&o, n * 7);
    std::vector<double> h(n);
    for (uint64_t i = 0; i < n; ++i) h[i] = double((i * 0x9E3779B97F4A7C15ull) >> 15);
    cudaMemcpy(w, h.data(), n * 8, cudaMemcpyHostToDevice);
    // plan constants for p=5, q=2^7, d=6, window 4 (base-p table)
    RedqParams P{};
    P.p = 5;
    P.d = 6;
    P.qbits = 7;
    P.neg_q = 2;
    P.window = 4;
    P.radix = 5;
    P.n_entries = 625;
    P.mod_magic = uint32_t(((1ull << 32) + 4) / 5);
    P.float_mode = 1;
    P.inv_p = 0.2000000000000000111;  // RN(1/5) >= 1/5
    P.r_max = 1501199875790165.0;
    P.limit = double(1ull << 49);
    P.q = 128;
    std::vector<uint32_t> tabh(625);
    for (uint32_t idx = 0; idx < 625; ++idx) {
        uint32_t u[4], t = idx;
        for (int j = 0; j < 4; ++j) u[j] = t % 5, t /= 5;
        uint32_t e = 0;
        for (int j = 0; j < 4; ++j) e |= (j < 3 ? (u[j] + 2 * u[j + 1]) % 5 : u[j]) << (8 * j);
        tabh[idx] = e;
    }
    uint32_t* tabd;
    cudaMalloc(&tabd, 625 * 4);
    cudaMemcpy(tabd, tabh.data(), 625 * 4, cudaMemcpyHostToDevice);
    P.table = tabd;
    Op op{P};
    const double bytes = 15.0 * n;
    auto report = [&](const char* name, float ms) {
        printf("%-34s %.4f ms  %.1f GB/s  %s\n", name, ms, bytes / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
#define RUN_CTA(NT, RR, S, CPS)                                                                                 \
    {                                                                                                          \
        auto k = v_cta<Op, NT, RR, S>;                                                                         \
        const size_t sm = S * 8 * NT * 4 * RR + 2 * 7 * NT * 4 * RR + 64 + 2600;                               \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);                      \
        int per = 0;                                                                                           \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, sm);                                        \
        if (CPS) per = per < CPS ? per : CPS;                                                                  \
        const uint64_t tiles = n / (NT * 4 * RR);                                                              \
        const unsigned grid = unsigned(148 * per < tiles ? 148 * per : tiles);                                 \
        char nm[96];                                                                                           \
        snprintf(nm, 96, "cta NT=%d RR=%d S=%d cps=%d", NT, RR, S, per);                                       \
        report(nm, timeit([&] { k<<<grid, NT, sm>>>(op, reinterpret_cast<const uint8_t*>(w), nullptr, o, tiles); }));  \
    }
    RUN_CTA(256, 1, 4, 0)
    RUN_CTA(256, 1, 6, 0)
    RUN_CTA(256, 2, 4, 0)
    RUN_CTA(256, 2, 3, 0)
    RUN_CTA(512, 1, 4, 0)
    RUN_CTA(512, 2, 3, 0)
    RUN_CTA(128, 2, 4, 0)
    RUN_CTA(256, 1, 4, 2)
    RUN_CTA(256, 1, 8, 0)
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
        char nm[64];
        snprintf(nm, 64, "ldg grid=%d", g);
        report(nm, timeit([&] { v_ldg<<<g, 256>>>(op, reinterpret_cast<const uint8_t*>(w), o, n / 4); }));
    }
    // ---- C3: GF(7^3) packed path, 2^24 records of 3+3 -> 3 bytes
    {
        const uint64_t n3 = 1ull << 24;
        uint8_t *a3, *b3, *o3;
        cudaMalloc(&a3, n3 * 3);
        cudaMalloc(&b3, n3 * 3);
        cudaMalloc(&o3, n3 * 3);
        std::vector<uint8_t> hb(n3 * 3);
        for (uint64_t i = 0; i < hb.size(); ++i) hb[i] = uint8_t((i * 2654435761u >> 13) % 7);
        cudaMemcpy(a3, hb.data(), hb.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(b3, hb.data(), hb.size(), cudaMemcpyHostToDevice);
        // L/H coefficient tables for GF(7^3) are not needed for timing: zeros
        uint32_t* t3;
        cudaMalloc(&t3, 4 * 1372);
        cudaMemset(t3, 0, 4 * 1372);
        GfqElemParams E{};
        E.rq = P;
        E.rq.p = 7, E.rq.d = 4, E.rq.qbits = 8, E.rq.neg_q = 3, E.rq.window = 0, E.rq.q = 256;
        E.rq.mod_magic = uint32_t(((1ull << 32) + 6) / 7);
        E.rq.inv_p = 1.0 / 7.0 + 1e-17;
        E.rq.limit = double(1ull << 40);
        E.k = 3, E.p = 7, E.order = 343, E.group = 342, E.lh_radix = 7, E.qd = 256.0;
        E.lc = t3, E.hc = t3 + 343, E.log = t3 + 686, E.alog = t3 + 1029, E.tables_words = 1372, E.mode = 0;
        using Op3 = GfqElemOp<3, CtConst<7, 8>>;
        Op3 op3{E};
        const double b3y = 9.0 * n3;
        for (int mode = 0; mode < 2; ++mode) {
            op3.P.mode = mode;
#define RUN3(NT, RR, S)                                                                                          \
    {                                                                                                            \
        auto k = v_cta<Op3, NT, RR, S>;                                                                          \
        const size_t sm = S * 6 * NT * 4 * RR + 2 * 3 * NT * 4 * RR + 64 + 5600;                                 \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);                        \
        int per = 0;                                                                                             \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, sm);                                          \
        const uint64_t tiles = n3 / (NT * 4 * RR);                                                               \
        const unsigned grid = unsigned(148 * per < tiles ? 148 * per : tiles);                                   \
        float ms = timeit([&] { k<<<grid, NT, sm>>>(op3, a3, b3, o3, tiles); });                                 \
        printf("C3 mode %d cta NT=%d RR=%d S=%d cps=%d  %.4f ms  %.1f GB/s %s\n", mode, NT, RR, S, per, ms,       \
               b3y / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));                                 \
    }
            RUN3(256, 1, 4) RUN3(256, 2, 4) RUN3(256, 4, 3) RUN3(256, 4, 4) RUN3(256, 8, 3) RUN3(512, 4, 3)
        }
        // pipeline ceiling for 3+3 -> 3 byte records: out = a ^ b
        XorOp xop;
#define RUNX(NT, RR, S)                                                                                          \
    {                                                                                                            \
        auto k = v_cta<XorOp, NT, RR, S>;                                                                        \
        const size_t sm = S * 6 * NT * 4 * RR + 2 * 3 * NT * 4 * RR + 64;                                        \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);                        \
        int per = 0;                                                                                             \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NT, sm);                                          \
        const uint64_t tiles = n3 / (NT * 4 * RR);                                                               \
        const unsigned grid = unsigned(148 * per < tiles ? 148 * per : tiles);                                   \
        float ms = timeit([&] { k<<<grid, NT, sm>>>(xop, a3, b3, o3, tiles); });                                 \
        printf("C3 xor-copy cta NT=%d RR=%d S=%d cps=%d  %.4f ms  %.1f GB/s %s\n", NT, RR, S, per, ms,            \
               b3y / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));                                 \
    }
        RUNX(256, 1, 4) RUNX(256, 2, 4) RUNX(256, 4, 3) RUNX(256, 4, 4) RUNX(256, 8, 2) RUNX(128, 4, 4)
        RUNX(256, 2, 8) RUNX(512, 2, 4)
    }
    double* w2;
    cudaMalloc(&w2, n * 8);
    report("cudaMemcpy d2d 512MB (x16/15 bytes)",
           timeit([&] { cudaMemcpyAsync(w2, w, n * 8, cudaMemcpyDeviceToDevice); }) * 15.0f / 16.0f);
    return 0;
}
