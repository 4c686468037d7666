// K4: GF(p^k) matrix product as an exact fp64 contraction on q-packed
// operands (reference gfq.cpp:389-404 -> fgdp_dot, gfq.cpp:335-387; paper
// Alg. 4 and Theorem 3).
//
//  * 128x128 CTA tile, 8 consumer warps each 64x32, fp64 tensor-core MMA
//    (mma.sync m8n8k4 f64 -> DMMA on sm_100a; tcgen05 has no f64 kind),
//    accumulators in registers;
//  * a producer warp streams 16-deep K slices of A^T and B with TMA bulk
//    copies (one 1 KB row per lane) into padded shared rows (conflict-free
//    fragment loads), full/empty mbarrier pipeline (6 stages on the fast paths,
//    4 on the generic kernels).  (Measured on
//    B200, scripts/mm_variants.cu: the dedicated producer sustains 35.6
//    TFLOP/s = 96% of the DMMA probe; letting the last consumer warp refill
//    a stage instead reaches only 26.8 -- that warp becomes a straggler.);
//  * delayed REDQ: every `chunk` K-steps a warp re-packs each accumulator to
//    sum(mu_i q^i) (redq + assemble, redq.cpp:178-182) so digit sums stay
//    below q and the word below 2^53.  Re-packs run at stage granularity,
//    outside the stage loop (so they are never predicated into every stage)
//    and staggered so the two consumer warps of an SM sub-partition never
//    re-pack in the same stage.  Measured: integer
//    instructions do not hide behind the DMMAs -- each one costs the
//    sub-partition about one dispatch slot of the 16 a DMMA takes, wherever
//    it sits -- so the re-pack is written for instruction count.  On the fast
//    paths (p = 3, q = 2^(2m)) the accumulators carry a 2^52 bias so the word
//    is the accumulator's mantissa and the re-pack is integer-only: canonical
//    lane folds for C5 (24 instructions), the SWAR REDQ (floor(r/3) by
//    div3_u64) for the other fields, or, with repack = fold, a congruent lane
//    fold (7 instructions);
//  * the REDQ-re-pack kernel walks tiles in groups of 8 tile rows (L2 reuse
//    of B), the fold kernel row-major (measured best for each);
//  * epilogue: final REDQ digits -> low/high half tables in coefficient form
//    (gfq.cpp:218-248) -> bytes, or -> rep through the log table.
//
// Templates only; instantiated per (k, policy) in gfq_matmul_inst.cu.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"
#include "redq_core.cuh"

namespace qpk {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, PAD = 4;
static_assert(BK == kMatmulBK, "kernels.hpp kMatmulBK");
constexpr int LDS_ = BM + PAD;            // shared row stride in doubles (== BN + PAD)
constexpr int NCW = 8;                    // consumer warps
constexpr int THREADS = (NCW + 1) * 32;   // + producer warp
constexpr int WM = 64, WN = 32;           // warp tile
constexpr int MT = WM / 8, NT = WN / 8;   // 8 x 4 DMMA tiles per warp
constexpr size_t STAGE_DOUBLES = size_t(2) * BK * LDS_;
// NST pipeline stages: 6 for the compile-time fast paths (deeper buffering
// lets one warp of a sub-partition run ahead while the other re-packs), 4
// for the generic kernels (leaves shared memory for large field tables)
constexpr size_t smem_bytes(int nst) { return nst * STAGE_DOUBLES * 8 + 2 * nst * 8; }

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// REDQ + re-pack: the word whose digit i is (digit i of r) mod p, as an
// exact double (digits mu_i via the direct correction, then assembled)
template <int ND, class K>
__device__ __forceinline__ double redq_repack(const K& c, double r) {
    uint32_t u[ND], mu[ND];
    redq_raw_digits<ND>(c, r, u);
    redq_correct<ND, 0>(c, u, mu, [](uint32_t) { return 0u; });
    if constexpr (K::kPow2) {
        uint64_t v = 0;
#pragma unroll
        for (int i = ND - 1; i >= 0; --i) v = (v << c.qbits()) | mu[i];
        return __longlong_as_double(static_cast<long long>(v | 0x4330000000000000ull)) - kTwo52;
    } else {
        double v = 0.0;
        const double qd = static_cast<double>(c.P.q);
#pragma unroll
        for (int i = ND - 1; i >= 0; --i) v = fma(v, qd, static_cast<double>(mu[i]));
        return v;
    }
}

// Biased accumulators (the SWAR re-packs): the accumulator holds 2^52 + r,
// an integer in [2^52, 2^53) where fp64 is exact with ulp 1, so its 52
// mantissa bits are r itself -- the re-pack reads and writes r as bits with
// no fp64 <-> integer conversions.  Words stay below 2^52 (mm_plan_safe).
constexpr uint64_t kBiasBits = 0x4330000000000000ull;  // bits of 2^52

template <int ND, uint32_t B>
__host__ __device__ constexpr uint64_t lane_ones() {
    uint64_t m = 0;
    for (int i = 0; i < ND; ++i) m |= uint64_t(1) << (B * i);
    return m;
}

// The same REDQ + re-pack for p = 3 and q = 2^B with B even (q == 1 mod 3),
// computed lane-wise inside one 64-bit integer (lane i = bits [Bi, Bi+B)):
//  * u_i in [0, 2] is fixed by its value mod 4, and
//    u_i = (r >> Bi) - 3 (rop >> Bi) == a_i + b_i (mod 4) with a_i, b_i the
//    two low bits of lane i of r and rop (-3 == 1 mod 4): one masked add
//    produces every lane's u_i (lane sums <= 6 never reach the next lane);
//  * mu_i = u_i + neg_q u_{i+1} = u_i - u_{i+1} (mod 3): with
//    V = u_i + 8 - u_{i+1} in [6, 10] and g = [V >= 8], mu_i = V - 5 - 3g
//    (every lane stays non-negative, so no borrow crosses lanes);
//  * the mu lanes already sit at q^i: the re-packed word, no assembly.
// rop = floor(r/3) is exact integer arithmetic on the 32-bit halves of r
// (div3_u64), and r itself is the mantissa of the 2^52-biased accumulator:
// the re-pack issues no fp64 instruction.  (The Lemma-1 fp64 floor measured
// 42.6 ms for C5 against 40.1 ms here: its DMUL/DADD compete with the
// sibling warp's DMMA stream for the fp64 pipe.)
// floor(r/3) from the halves r = rh 2^32 + rl: with rh = 3 qh + mh and
// rl = 3 ql + rr, floor(r/3) = qh 2^32 + mh (2^32-1)/3 + ql + [mh + rr >= 3]
// (2^32 == 1 mod 3; the low part stays below 2^32).

// (Computing floor(r/3) by the fp64 floor for half of the accumulators and
// by div3_u64 for the other half measured 43.7 ms: worse than either.)
template <int ND, uint32_t B>
__device__ __forceinline__ double redq_repack_swar3(double acc) {
    static_assert(B % 2 == 0 && B >= 4 && B * (ND - 1) + 3 <= 52, "lanes of >= 4 bits below 2^52");
    constexpr uint64_t M1 = lane_ones<ND, B>();
    constexpr uint64_t M3 = 3 * M1;
    const uint64_t rb = dbits(acc) & ((uint64_t(1) << 52) - 1);  // acc = 2^52 + r: mantissa = r
    const uint64_t ob = div3_u64(rb);                               // floor(r/3)
    const uint64_t u = ((rb & M3) + (ob & M3)) & M3;                // lane i = u_i
    const uint64_t v = u + 8 * M1 - (u >> B);                       // u_i + 8 - u_{i+1}
    const uint64_t g = (v >> 3) & M1;                               // [u_i >= u_{i+1}]
    const uint64_t mu = v - 5 * M1 - 3 * g;                         // (u_i - u_{i+1}) mod 3
    return __longlong_as_double(static_cast<long long>(mu | kBiasBits));  // 2^52 + sum mu_i q^i
}

// The canonical re-pack for p = 3, q = 2^10, five digits (GF(3^3), C5), as
// lane folds on two 32-bit registers: digit i of the output is c_i mod 3, the
// same word redq_repack_swar3 and redq + assemble (redq.cpp:178-182) return
// whenever every digit c_i is below q (the chunk bound).  Every integer
// instruction issued between the MMAs costs the tensor pipe about one
// dispatch slot (measured with timing-only variants of this kernel, DESIGN
// section 5: ~0.2 ms of C5 per instruction per accumulator, IMAD.HI four
// times that), so the count is what matters: 24 instructions, no IMAD.HI,
// against 33 with two IMAD.HI for the SWAR REDQ with div3_u64.
//  * align: L = bits 0..29 (digits 0-2, bits 30-31 ride along and are masked
//    at the end), H = bits 30..49 (digits 3-4 at 0 and 10; the 2^52 bias
//    bits ride above bit 22 and come out as the bias of the result);
//  * 2^6 == 2^4 == 1 (mod 3): c -> (c & 63) + (c >> 6) <= 78, then
//    x -> (x & 15) + (x >> 4) <= 19, each as x - (2^s - 1) (x >> s) on all
//    lanes of a register at once (no lane borrows);
//  * x <= 19: floor(x/3) = (11 x) >> 5 (11 x <= 209 stays inside the lane),
//    x - 3 floor(x/3) is the canonical residue.
__host__ __device__ __forceinline__ uint64_t repack_canon3_bits(uint64_t bits) {
    const uint32_t lo = static_cast<uint32_t>(bits), hi = static_cast<uint32_t>(bits >> 32);
    constexpr uint32_t kH6 = 0x00F03C0Fu, kH4 = 0x00701C07u;  // (c >> 6), (x >> 4) and floor(x/3) lane masks
#ifdef __CUDA_ARCH__
    uint32_t xh = __funnelshift_l(lo, hi, 2);
#else
    uint32_t xh = (hi << 2) | (lo >> 30);
#endif
    uint32_t h = (lo >> 6) & kH6;
    uint32_t xl = lo - 63u * h;
    h = (xh >> 6) & (kH6 & 0xFFFFFu);
    xh -= 63u * h;
    h = (xl >> 4) & kH4;
    xl -= 15u * h;
    h = (xh >> 4) & (kH4 & 0xFFFFFu);
    xh -= 15u * h;
    h = ((xl * 11u) >> 5) & kH4;
    xl -= 3u * h;
    h = ((xh * 11u) >> 5) & (kH4 & 0xFFFFFu);
    xh -= 3u * h;
    // H carried (0x43300000 << 2) mod 2^32 = 0x0CC00000 untouched: >> 2 gives 0x03300000
    const uint32_t out_lo = (xl & 0x3FFFFFFFu) | (xh << 30);
#ifdef __CUDA_ARCH__
    const uint32_t out_hi = __funnelshift_r(xh, 1u, 2);  // (xh >> 2) | 0x40000000 in one SHF
#else
    const uint32_t out_hi = (xh >> 2) + 0x40000000u;
#endif
    return (static_cast<uint64_t>(out_hi) << 32) | out_lo;
}
__device__ __forceinline__ double redq_repack_canon3(double acc) {
    return __longlong_as_double(static_cast<long long>(repack_canon3_bits(dbits(acc))));
}

// Lane fold (repack mode QPK_REPACK_FOLD), p = 3 and q = 2^B: every digit
// c_i = l_i + 2^S h_i (l_i < 2^S) is replaced by l_i + h_i, which is
// congruent mod 3 because 2^S == 1 (mod 3) for even S.  Digits drop from
// < q to <= (2^S - 1) + (2^(B-S) - 1) (78 for B = 10, S = 6) -- not the
// canonical mu_i of REDQ, but the same value of every digit mod p, so the
// final REDQ and the output are identical; the host sizes the chunk for the
// larger post-fold digit bound.  On the biased accumulator this is pure
// integer lane arithmetic: 2 masks, 1 shift, 1 add (no fp64 work).
template <int ND, uint32_t B, uint32_t S>
__device__ __forceinline__ double repack_fold3(double acc) {
    static_assert(S % 2 == 0 && S < B && B * ND <= 52, "2^S == 1 mod 3, lanes below 2^52");
    constexpr uint64_t M1 = lane_ones<ND, B>();
    constexpr uint64_t ML = M1 * ((uint64_t(1) << S) - 1);
    constexpr uint64_t MH = M1 * ((uint64_t(1) << (B - S)) - 1);
    const uint64_t rb = dbits(acc);
    const uint64_t f = (rb & ML) + ((rb >> S) & MH);
    return __longlong_as_double(static_cast<long long>(f | kBiasBits));
}

#if defined(QPK_MM_EXP)
#include "../../scripts/mm_exp_repack.cuh"  // development: timing-only re-pack variants (scripts/mm_exp.sh)
#endif

// fold split S: the largest even S <= B - S + 2 (balances l_i and h_i)
template <uint32_t B>
constexpr uint32_t kFoldShift = ((B + 2) / 2) % 2 ? (B + 2) / 2 + 1 : (B + 2) / 2;

template <class K>
struct is_swar3 {
    static constexpr bool value = false;
};
template <uint32_t QB>
struct is_swar3<CtConst<3, QB>> {
    static constexpr bool value = (QB % 2 == 0) && QB >= 4;
};

// accumulators carry the 2^52 bias exactly on the SWAR re-pack fast paths
template <class K, bool FOLD>
struct mm_biased {
    static constexpr bool value = is_swar3<K>::value;  // both SWAR re-packs run on biased words
};

template <int ND, class K, bool FOLD>
__device__ __forceinline__ double repack_one(const K& c, double r) {
#if defined(QPK_MM_EXP)
    if constexpr (is_swar3<K>::value && !FOLD) return mm_exp_repack<ND, K::kQbits>(r);
#endif
    if constexpr (is_swar3<K>::value) {
        if constexpr (FOLD)
            return repack_fold3<ND, K::kQbits, kFoldShift<K::kQbits>>(r);
        else if constexpr (ND == 5 && K::kQbits == 10)
            return redq_repack_canon3(r);
        else
            return redq_repack_swar3<ND, K::kQbits>(r);
    } else {
        static_assert(!FOLD, "the lane fold is compiled for p = 3, q = 2^(2m) only");
        return redq_repack<ND>(c, r);
    }
}

__device__ __forceinline__ uint32_t add_mod_bytes_mm(uint32_t x, uint32_t y, uint32_t p) {
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
template <int KR, class K>
__device__ __forceinline__ uint32_t acc_to_coeffs(const K& c, uint32_t lh_radix, double r, uint32_t lc_s,
                                                  uint32_t hc_s) {
    constexpr int ND = 2 * KR - 1;
    uint32_t u[ND];
    redq_raw_digits<ND>(c, r, u);
    uint32_t il = 0, ih = 0;
#pragma unroll
    for (int i = KR - 1; i >= 0; --i) {
        il = il * lh_radix + u[i];
        ih = ih * lh_radix + u[KR - 1 + i];
    }
    return add_mod_bytes_mm(lds_u32(lc_s + 4 * il), lds_u32(hc_s + 4 * ih), c.p());
}

// REDQ_STAGE: re-pack at stage granularity (chunk a multiple of BK) rather
// than per 4-step MMA (fields whose safe chunk is below BK)
#ifndef QPK_MM_GROUP
#define QPK_MM_GROUP 8
#endif
// (9 warps: one SM sub-partition holds 3 of them, so 16384 / (3 * 32) caps
// the kernel at 168 registers per thread)
template <int KR, class K, bool REDQ_STAGE, int NST, bool FOLD, bool PAIR>
__global__ void __launch_bounds__(THREADS, 1)
    gfq_matmul_kernel(const GfqMatmulParams P, const double* __restrict__ at, const double* __restrict__ bm,
                      uint64_t m, uint64_t n, uint64_t K_pad, uint64_t m_pad, uint64_t n_pad,
                      uint8_t* __restrict__ out_c, uint32_t* __restrict__ out_r) {
    constexpr int ND = 2 * KR - 1;
    extern __shared__ __align__(128) uint8_t smem[];
    double* stages = reinterpret_cast<double*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE_DOUBLES * 8);
    uint64_t* empty = full + NST;
    uint32_t* tabs = reinterpret_cast<uint32_t*>(empty + NST);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // grouped rasterisation: consecutive CTAs walk GROUP tile rows column
    // by column, so a wave re-reads B's column slabs from L2 rather than DRAM
    // (row-major order streams all of B once per tile row).  Measured on C5:
    // REDQ re-pack 40.15 -> 39.37 ms with 8 rows, the fold 33.29 -> 34.07
    // (kept row-major there)
    constexpr uint32_t GROUP = FOLD ? 1u : uint32_t(QPK_MM_GROUP);
    uint32_t tm = blockIdx.y, tn = blockIdx.x;
    if constexpr (GROUP > 1) {
        const uint32_t num_n = gridDim.x, num_m = gridDim.y;
        const uint32_t bid = blockIdx.y * num_n + blockIdx.x, per = GROUP * num_n;
        const uint32_t first_m = (bid / per) * GROUP;
        const uint32_t gm = min(num_m - first_m, GROUP);
        tm = first_m + (bid % per) % gm;
        tn = (bid % per) / gm;
    }
    const uint64_t m0 = uint64_t(tm) * BM, n0 = uint64_t(tn) * BN;
    const int KT = static_cast<int>(K_pad / BK);

    // epilogue tables (lc | hc | log) staged once per CTA
    uint32_t nlh = 1;
    for (int i = 0; i < KR; ++i) nlh *= P.lh_radix;
    for (uint32_t i = tid; i < 2 * nlh; i += blockDim.x) tabs[i] = i < nlh ? P.lc[i] : P.hc[i - nlh];
    if (out_r)
        for (uint32_t i = tid; i < P.order; i += blockDim.x) tabs[2 * nlh + i] = P.log[i];
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------- producer: one TMA bulk row copy per lane ----------
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % NST;
            if (kt >= NST) mbar_wait(&empty[s], ((kt / NST) - 1) & 1);
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
    const K c{P.rq};
    const int wm = (warp >> 2) * WM;  // 2 x 4 warp grid; warps w, w+4 share SMSP w%4
    const int wn = (warp & 3) * WN;
    const int lr = lane >> 2, lc4 = lane & 3;
    constexpr double kBias = mm_biased<K, FOLD>::value ? kTwo52 : 0.0;
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = kBias;

    auto repack_all = [&]() {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                acc[i][j][0] = repack_one<ND, K, FOLD>(c, acc[i][j][0]);
                acc[i][j][1] = repack_one<ND, K, FOLD>(c, acc[i][j][1]);
            }
    };
    // 4 MMA k-steps of one stage; per step 8 A and 4 B fragments -> 32 DMMA
    // PAIR: the workspaces hold a thread's fragments 2t, 2t+1 next to each
    // other (kernels.hpp mm_col_a / mm_col_b): one 16-byte load for two
    auto mma_kstep = [&](const double* sa, const double* sb, int kk) {
        double af[MT], bf[NT];
        if constexpr (PAIR) {
            const double2* pa = reinterpret_cast<const double2*>(sa + (kk * 4 + lc4) * LDS_ + wm + 2 * lr);
            const double2* pb = reinterpret_cast<const double2*>(sb + (kk * 4 + lc4) * LDS_ + wn + 2 * lr);
#pragma unroll
            for (int t = 0; t < MT / 2; ++t) {
                const double2 v = pa[8 * t];
                af[2 * t] = v.x, af[2 * t + 1] = v.y;
            }
#pragma unroll
            for (int t = 0; t < NT / 2; ++t) {
                const double2 v = pb[8 * t];
                bf[2 * t] = v.x, bf[2 * t + 1] = v.y;
            }
        } else {
            const double* pa = sa + (kk * 4 + lc4) * LDS_ + wm + lr;
            const double* pb = sb + (kk * 4 + lc4) * LDS_ + wn + lr;
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = pa[i * 8];
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = pb[j * 8];
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    };

    if constexpr (REDQ_STAGE) {
        // (a register-lean fragment prefetch was measured here and gained
        // nothing while adding spills under the 168-register cap)
        auto stage = [&](int kt) {
            const int s = kt % NST;
            mbar_wait(&full[s], (kt / NST) & 1);
            const double* sa = stages + s * STAGE_DOUBLES;
#pragma unroll 1
            for (int kk = 0; kk < BK / 4; ++kk) mma_kstep(sa, sa + BK * LDS_, kk);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        };
        // re-pack after stage `next`, every cs stages; the phase offset keeps
        // warps w and w+4 (same sub-partition) cs/2 stages apart
        const int cs = static_cast<int>(P.chunk / BK);
        int next = KT;
        if (cs > 0) next = cs - 1 - ((warp & 3) + (warp >> 2) * (cs / 2)) % cs;
        int kt = 0;
        while (kt < KT) {
            const int end = next + 1 < KT ? next + 1 : KT;
            for (; kt < end; ++kt) stage(kt);
            if (kt == next + 1 && kt < KT) {
                repack_all();
                next += cs;
            }
        }
    } else {
        // generic small-chunk fields: re-pack every `chunk` MMA k-steps
        const int chunk4 = static_cast<int>(P.chunk / 4);
        int countdown = chunk4 > 0 ? chunk4 - (warp * chunk4) / NCW : 0x7fffffff;
        for (int kt = 0; kt < KT; ++kt) {
            const int s = kt % NST;
            mbar_wait(&full[s], (kt / NST) & 1);
            const double* sa = stages + s * STAGE_DOUBLES;
#pragma unroll 1
            for (int kk = 0; kk < BK / 4; ++kk) {
                mma_kstep(sa, sa + BK * LDS_, kk);
                if (--countdown == 0) {
                    countdown = chunk4;
                    repack_all();
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }

    // ------------------------- epilogue ------------------------------------
#if defined(QPK_MM_EXP)
    if constexpr (is_swar3<K>::value && !FOLD) {  // timing-only variants: keep the table indices in range
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[i][j][h] = redq_repack_swar3<ND, K::kQbits>(acc[i][j][h]);
    }
#endif
    const uint32_t lc_s = smem_addr(tabs), hc_s = lc_s + 4 * nlh, lg_s = lc_s + 8 * nlh;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const uint64_t row = m0 + wm + i * 8 + lr;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const uint64_t col = n0 + wn + j * 8 + lc4 * 2;
            // (storing a thread's two adjacent elements as 16-bit pieces measured slower:
            // C5 fold 33.03 -> 33.64 ms, the canonical re-pack 37.10 -> 37.17)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (row < m && col + h < n) {
                    const uint32_t cf = acc_to_coeffs<KR>(c, P.lh_radix, acc[i][j][h] - kBias, lc_s, hc_s);
                    if (out_c) {
                        uint8_t* dst = out_c + (row * n + col + h) * KR;
#pragma unroll
                        for (int t = 0; t < KR; ++t) dst[t] = static_cast<uint8_t>(cf >> (8 * t));
                    } else {
                        uint32_t idx = 0;
#pragma unroll
                        for (int t = KR - 1; t >= 0; --t) idx = idx * c.p() + ((cf >> (8 * t)) & 0xff);
                        out_r[row * n + col + h] = lds_u32(lg_s + 4 * idx);
                    }
                }
            }
        }
    }
}

template <int KR, class K, bool REDQ_STAGE, int NST = 4, bool FOLD = false, bool PAIR = false>
cudaError_t run_matmul_t(const GfqMatmulParams& P, const double* at, const double* b, uint64_t m, uint64_t n,
                         uint64_t K_pad, uint64_t m_pad, uint64_t n_pad, uint8_t* oc, uint32_t* orp, cudaStream_t s) {
    uint32_t nlh = 1;
    for (int i = 0; i < KR; ++i) nlh *= P.lh_radix;
    const size_t smem = smem_bytes(NST) + size_t(2 * nlh + P.order) * 4;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(gfq_matmul_kernel<KR, K, REDQ_STAGE, NST, FOLD, PAIR>),
                                        smem);
        e != cudaSuccess)
        return e;
    dim3 grid(static_cast<unsigned>(n_pad / BN), static_cast<unsigned>(m_pad / BM));
    gfq_matmul_kernel<KR, K, REDQ_STAGE, NST, FOLD, PAIR><<<grid, THREADS, smem, s>>>(P, at, b, m, n, K_pad, m_pad, n_pad,
                                                                                oc, orp);
    return cudaGetLastError();
}

// VARIANT 1: compile-time fast paths for the benchmark fields (C4 GF(3^2)
// at q = 2^16, C5 GF(3^3) at q = 2^10); returns cudaErrorNotSupported when
// the field is not one of them.  VARIANT 0: runtime-parameter kernels.
template <int KR, int VARIANT>
cudaError_t run_matmul(const GfqMatmulParams& P, const double* at, const double* b, uint64_t m, uint64_t n,
                       uint64_t K_pad, uint64_t m_pad, uint64_t n_pad, uint8_t* oc, uint32_t* orp, cudaStream_t s) {
    const bool stage_ok = P.chunk == 0 || P.chunk % BK == 0;
    if constexpr (VARIANT == 1) {
        if constexpr (KR == 2) {
            if (P.p == 3 && P.rq.qbits == 16 && mm_plan_safe(P.rq) && stage_ok)
                return run_matmul_t<2, CtConst<3, 16>, true, 6>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s);
        }
        if constexpr (KR == 3) {
            if (P.p == 3 && P.rq.qbits == 10 && mm_plan_safe(P.rq) && stage_ok) {
                // the workspaces were packed for the kernel mm_pair_layout names
                if ((P.repack != kRepackFold) != mm_pair_layout(P)) return cudaErrorInvalidValue;
                return P.repack == kRepackFold
                           ? run_matmul_t<3, CtConst<3, 10>, true, 6, true>(P, at, b, m, n, K_pad, m_pad, n_pad, oc,
                                                                            orp, s)
                           : run_matmul_t<3, CtConst<3, 10>, true, 6, false, true>(P, at, b, m, n, K_pad, m_pad, n_pad,
                                                                                   oc, orp, s);
            }
        }
        return cudaErrorNotSupported;
    } else {
        if (P.rq.qbits)
            return stage_ok ? run_matmul_t<KR, RtConst<true>, true>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s)
                            : run_matmul_t<KR, RtConst<true>, false>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s);
        return stage_ok ? run_matmul_t<KR, RtConst<false>, true>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s)
                        : run_matmul_t<KR, RtConst<false>, false>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s);
    }
}

}  // namespace

}  // namespace qpk
