// K1 (pack) and K4 (matrix product) of the q-adic pipeline for GF(p^k).
//
// K1a  DQT/Horner pack: coefficient records (k bytes) -> exact q-adic fp64
//      words, written transposed/padded for the GEMM (dqt.cpp:23-37).
// K1b  Zech/discrete-log tabulated pack: reps -> float_eval(rep) through the
//      float table staged in shared memory (gfq.cpp:194-207, 355).
// K4   C = A*B as an exact fp64 contraction on the packed words
//      (gfq.cpp:389-404 -> fgdp_dot, gfq.cpp:335-387):
//        * 128x128 CTA tile, 8 consumer warps each 64x32, fp64 tensor-core
//          MMA (mma.sync m8n8k4 f64 -> DMMA on sm_100a; tcgen05 has no f64
//          kind), accumulators in registers;
//        * a producer warp streams 16-deep K slices of A^T and B with TMA
//          bulk copies (one 1 KB row per lane) into padded shared rows
//          (conflict-free fragment loads), 4-stage mbarrier pipeline;
//        * delayed REDQ: every `chunk` K-steps a warp re-packs each
//          accumulator to sum(mu_i q^i) so digit sums stay below q and the
//          word below 2^53; warps are staggered so re-packs overlap the
//          other warps' MMAs;
//        * epilogue: final REDQ digits -> low/high half tables (Theorem 3,
//          gfq.cpp:218-248) in coefficient form -> bytes, or -> rep.
//
// Templates only; instantiated per k in gfq_matmul_inst.cu (-DQPK_INST=k).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, PAD = 4;
constexpr int LDS_ = BM + PAD;            // shared row stride in doubles (== BN + PAD)
constexpr int NCW = 8;                    // consumer warps
constexpr int THREADS = (NCW + 1) * 32;   // + producer warp
constexpr int WM = 64, WN = 32;           // warp tile
constexpr int MT = WM / 8, NT = WN / 8;   // 8 x 4 DMMA tiles per warp
constexpr size_t STAGE_DOUBLES = size_t(2) * BK * LDS_;
constexpr size_t SMEM_BYTES = STAGES * STAGE_DOUBLES * 8 + 2 * STAGES * 8;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

constexpr uint64_t kMask52 = (uint64_t(1) << 52) - 1;

// raw REDQ digits of an accumulated word (always < 2^53 and, for every
// supported field, <= r_max once the per-chunk bound holds)
template <int ND, bool POW2>
__device__ __forceinline__ void acc_digits(const RedqParams& P, double r, uint32_t (&u)[ND]) {
    const uint64_t rb = r < kTwo52 ? (dbits(r + kTwo52) & kMask52) : __double2ull_rz(r);
    const bool premul = r <= P.r_max;
    const uint64_t rop = premul ? floor_div_premul(r, P.inv_p) : rb / P.p;
    if constexpr (POW2) {
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            const uint32_t sh = P.qbits * i;
            u[i] = static_cast<uint32_t>(rb >> sh) - P.p * static_cast<uint32_t>(rop >> sh);
        }
    } else {
        const double ropd = static_cast<double>(rop);
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            uint64_t x, y;
            if (premul) {
                x = floor_div_premul(r, P.inv_q[i]);
                y = floor_div_premul(ropd, P.inv_q[i]);
            } else {
                x = rb / P.qpow[i];
                y = rop / P.qpow[i];
            }
            u[i] = static_cast<uint32_t>(x) - P.p * static_cast<uint32_t>(y);
        }
    }
}

// REDQ + re-pack (redq.cpp:178-182 `redq` + `assemble`): the word whose
// digit i is (digit i of r) mod p, returned as an exact double.
template <int ND, bool POW2>
__device__ __forceinline__ double redq_repack(const RedqParams& P, double r) {
    uint32_t u[ND];
    acc_digits<ND, POW2>(P, r, u);
    uint32_t mu[ND];
#pragma unroll
    for (int i = 0; i + 1 < ND; ++i) {
        const uint32_t t = u[i] + P.neg_q * u[i + 1];
        mu[i] = t - P.p * __umulhi(t, P.mod_magic);
    }
    mu[ND - 1] = u[ND - 1];
    if constexpr (POW2) {
        uint64_t v = 0;
#pragma unroll
        for (int i = ND - 1; i >= 0; --i) v = (v << P.qbits) | mu[i];
        return __longlong_as_double(static_cast<long long>(v | 0x4330000000000000ull)) - kTwo52;
    } else {
        double v = 0.0;
#pragma unroll
        for (int i = ND - 1; i >= 0; --i) v = fma(v, static_cast<double>(P.q), static_cast<double>(mu[i]));
        return v;
    }
}

__device__ __forceinline__ uint32_t add_mod_bytes(uint32_t x, uint32_t y, uint32_t p) {
    if (p < 128) {
        const uint32_t pp = p * 0x01010101u;
        const uint32_t s = __vadd4(x, y);
        return __vsub4(s, __vcmpgeu4(s, pp) & pp);
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t t = ((x >> (8 * i)) & 0xff) + ((y >> (8 * i)) & 0xff);
        if (t >= p) t -= p;
        r |= t << (8 * i);
    }
    return r;
}

// final conversion of one accumulated word to packed coefficient bytes
template <int K, bool POW2>
__device__ __forceinline__ uint32_t acc_to_coeffs(const GfqMatmulParams& P, double r, const uint32_t* lc,
                                                  const uint32_t* hc) {
    constexpr int ND = 2 * K - 1;
    uint32_t u[ND];
    acc_digits<ND, POW2>(P.rq, r, u);
    uint32_t il = 0, ih = 0;
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
        il = il * P.lh_radix + u[i];
        ih = ih * P.lh_radix + u[K - 1 + i];
    }
    return add_mod_bytes(lc[il], hc[ih], P.p);
}

template <int K, bool POW2>
__global__ void __launch_bounds__(THREADS, 1)
    gfq_matmul_kernel(const GfqMatmulParams P, const double* __restrict__ at, const double* __restrict__ bm,
                      uint64_t m, uint64_t n, uint64_t K_pad, uint64_t m_pad, uint64_t n_pad,
                      uint8_t* __restrict__ out_c, uint32_t* __restrict__ out_r) {
    constexpr int ND = 2 * K - 1;
    extern __shared__ __align__(128) uint8_t smem[];
    double* stages = reinterpret_cast<double*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_DOUBLES * 8);
    uint64_t* empty = full + STAGES;
    uint32_t* tabs = reinterpret_cast<uint32_t*>(empty + STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t m0 = uint64_t(blockIdx.y) * BM, n0 = uint64_t(blockIdx.x) * BN;
    const int KT = static_cast<int>(K_pad / BK);

    // epilogue tables (lc | hc | log) staged once per CTA
    uint32_t nlh = 1;
    for (int i = 0; i < K; ++i) nlh *= P.lh_radix;
    const uint32_t ntab = 2 * nlh + (out_r ? P.order : 0);
    for (uint32_t i = tid; i < 2 * nlh; i += blockDim.x) tabs[i] = i < nlh ? P.lc[i] : P.hc[i - nlh];
    if (out_r)
        for (uint32_t i = tid; i < P.order; i += blockDim.x) tabs[2 * nlh + i] = P.log[i];
    (void)ntab;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------- producer: one TMA bulk row copy per lane ----------
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
            if (lane == 0) mbar_expect_tx(&full[s], 2 * BK * BM * 8);
            __syncwarp();
            double* sa = stages + s * STAGE_DOUBLES;
            double* sb = sa + BK * LDS_;
            const uint64_t k0 = uint64_t(kt) * BK;
            if (lane < BK)
                bulk_g2s(sa + lane * LDS_, at + (k0 + lane) * m_pad + m0, BM * 8, &full[s]);
            else
                bulk_g2s(sb + (lane - BK) * LDS_, bm + (k0 + lane - BK) * n_pad + n0, BN * 8, &full[s]);
        }
        return;
    }

    // -------------------- consumers ---------------------------------------
    const int wm = (warp >> 2) * WM;  // 2 x 4 warp grid
    const int wn = (warp & 3) * WN;
    const int lr = lane >> 2, lc4 = lane & 3;
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // delayed REDQ schedule at 4-step granularity, staggered across warps
    const int chunk4 = static_cast<int>(P.chunk / 4);
    int countdown = chunk4 > 0 ? chunk4 - (warp * chunk4) / NCW : 0x7fffffff;

    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&full[s], (kt / STAGES) & 1);
        const double* sa = stages + s * STAGE_DOUBLES;
        const double* sb = sa + BK * LDS_;
#pragma unroll 1
        for (int kk = 0; kk < BK / 4; ++kk) {
            const double* pa = sa + (kk * 4 + lc4) * LDS_ + wm + lr;
            const double* pb = sb + (kk * 4 + lc4) * LDS_ + wn + lr;
            double af[MT], bf[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = pa[i * 8];
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = pb[j * 8];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            if (--countdown == 0) {
                countdown = chunk4;
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) {
                        acc[i][j][0] = redq_repack<ND, POW2>(P.rq, acc[i][j][0]);
                        acc[i][j][1] = redq_repack<ND, POW2>(P.rq, acc[i][j][1]);
                    }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ------------------------- epilogue ------------------------------------
    const uint32_t* lc = tabs;
    const uint32_t* hc = tabs + nlh;
    const uint32_t* lg = tabs + 2 * nlh;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const uint64_t row = m0 + wm + i * 8 + lr;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const uint64_t col = n0 + wn + j * 8 + lc4 * 2;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (row < m && col + h < n) {
                    const uint32_t c = acc_to_coeffs<K, POW2>(P, acc[i][j][h], lc, hc);
                    if (out_c) {
                        uint8_t* dst = out_c + (row * n + col + h) * K;
#pragma unroll
                        for (int t = 0; t < K; ++t) dst[t] = static_cast<uint8_t>(c >> (8 * t));
                    } else {
                        uint32_t idx = 0;
#pragma unroll
                        for (int t = K - 1; t >= 0; --t) idx = idx * P.p + ((c >> (8 * t)) & 0xff);
                        out_r[row * n + col + h] = lg[idx];
                    }
                }
            }
        }
    }
}

template <int K, bool POW2>
cudaError_t run_matmul(const GfqMatmulParams& P, const double* at, const double* b, uint64_t m, uint64_t n,
                       uint64_t K_pad, uint64_t m_pad, uint64_t n_pad, uint8_t* oc, uint32_t* orp, cudaStream_t s) {
    uint32_t nlh = 1;
    for (int i = 0; i < K; ++i) nlh *= P.lh_radix;
    const size_t smem = SMEM_BYTES + size_t(2 * nlh + P.order) * 4;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gfq_matmul_kernel<K, POW2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid(static_cast<unsigned>(n_pad / BN), static_cast<unsigned>(m_pad / BM));
    gfq_matmul_kernel<K, POW2><<<grid, THREADS, smem, s>>>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp);
    return cudaGetLastError();
}

}  // namespace

}  // namespace qpk
