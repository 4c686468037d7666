// REDQ on one exact-integer fp64 word (paper Alg. 2, Theorem 2;
// reference redq.cpp:31-100), parameterised by a constants policy:
//
//   RtConst<POW2>        p, q, neg_q read from the RedqParams block at run
//                        time; any word below 2^53 (premultiplied floor when
//                        r <= r_max, exact integer division otherwise).
//   CtConst<P, QBITS>    p and q = 2^QBITS fixed at compile time and the
//                        plan known to keep every word <= min(r_max, 2^52):
//                        no range branches, shifts and the mod-p correction
//                        fold into immediates.  Dispatched for the benchmark
//                        fields (C1-C5); everything else uses RtConst.
//
// Both produce identical digits: u_i = floor(r/q^i) - p*floor(rop/q^i) in
// [0, p-1], formed in wrapping 32-bit arithmetic.
#pragma once

#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

constexpr uint64_t kMask52 = (uint64_t(1) << 52) - 1;

// t mod p for 0 <= t < 2^16 and p <= 256 (floor(t/p) from a 32-bit
// multiply-high by ceil(2^32/p) is exact in that range)
__device__ __forceinline__ uint32_t mod_by_magic(uint32_t t, uint32_t p, uint32_t magic) {
    return t - p * __umulhi(t, magic);
}

template <bool POW2>
struct RtConst {
    static constexpr bool kSafe = false;
    static constexpr bool kPow2 = POW2;
    static constexpr uint32_t kQbitsCt = 0;  // not known at compile time
    const RedqParams& P;
    __device__ __forceinline__ uint32_t p() const { return P.p; }
    __device__ __forceinline__ uint32_t qbits() const { return P.qbits; }
    __device__ __forceinline__ uint32_t neg_q() const { return P.neg_q; }
    __device__ __forceinline__ uint32_t radix() const { return P.radix; }
    __device__ __forceinline__ uint32_t modp(uint32_t t) const { return mod_by_magic(t, P.p, P.mod_magic); }
};

template <uint32_t P_, uint32_t QBITS_>
struct CtConst {
    static constexpr bool kSafe = true;
    static constexpr bool kPow2 = true;
    static constexpr uint32_t kP = P_, kQbits = QBITS_, kQbitsCt = QBITS_;
    static constexpr uint32_t kNegQ = (P_ - (uint32_t(1) << QBITS_) % P_) % P_;
    const RedqParams& P;
    __device__ __forceinline__ static constexpr uint32_t p() { return P_; }
    __device__ __forceinline__ static constexpr uint32_t qbits() { return QBITS_; }
    __device__ __forceinline__ static constexpr uint32_t neg_q() { return kNegQ; }
    __device__ __forceinline__ static constexpr uint32_t radix() { return P_; }
    // t <= (p-1)(1+neg_q): a packed lookup constant when it fits 32 bits
    __device__ __forceinline__ static uint32_t modp(uint32_t t) {
        constexpr uint32_t tmax = (P_ - 1) * (1 + kNegQ);
        if constexpr (P_ <= 4 && tmax < 16) {
            constexpr uint32_t lut = [] {
                uint32_t v = 0;
                for (uint32_t i = 0; i <= tmax; ++i) v |= (i % P_) << (2 * i);
                return v;
            }();
            return (lut >> (2 * t)) & 3u;
        } else {
            return t % P_;
        }
    }
};

// Exact integer of a non-negative double below 2^52 in (lo, hi) halves.
__device__ __forceinline__ uint64_t int_bits52(double r) { return dbits(r + kTwo52) & kMask52; }

// Raw digits of r (an exact integer < 2^53; <= r_max and < 2^52 for CtConst).
template <int ND, class K>
__device__ __forceinline__ void redq_raw_digits(const K& c, double r, uint32_t (&u)[ND]) {
    const RedqParams& P = c.P;
    uint64_t rb, rop;
    bool premul = true;
    if constexpr (K::kSafe) {
        rb = int_bits52(r);
        rop = floor_div_premul(r, P.inv_p);
    } else {
        premul = r <= P.r_max;
        rb = r < kTwo52 ? int_bits52(r) : __double2ull_rz(r);
        rop = premul ? floor_div_premul(r, P.inv_p) : rb / P.p;
    }
    if constexpr (K::kPow2) {
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            const uint32_t sh = c.qbits() * i;
            u[i] = static_cast<uint32_t>(rb >> sh) - c.p() * static_cast<uint32_t>(rop >> sh);
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
            u[i] = static_cast<uint32_t>(x) - c.p() * static_cast<uint32_t>(y);
        }
    }
}

// Word validation with packed_from_double semantics (dqt.cpp:96-100) plus
// check_input (redq.cpp:22-29): returns trunc(w); sets kErrDomain when w is
// negative, NaN or not below min(q^(d+1), 2^53).  Invalid words still flow
// through the arithmetic (their residues are unspecified; the batch fails).
__device__ __forceinline__ double checked_word(const RedqParams& P, double w, uint32_t& err) {
    const double r = trunc(w);
    if (!(w >= 0.0 && r < P.limit)) err |= kErrDomain;
    return r;
}

// Correction mu from u (redq.cpp:61-100): W = 0 direct (identity when
// p | q), W = 2..4 windowed table of Alg. 3 with one byte per residue.
template <int ND, int W, class K, class TabLoad>
__device__ __forceinline__ void redq_correct(const K& c, const uint32_t (&u)[ND], uint32_t (&mu)[ND], TabLoad tab) {
    constexpr int D = ND - 1;
    if constexpr (W == 0 || D == 0) {
        if (D > 0 && c.neg_q() != 0) {
#pragma unroll
            for (int i = 0; i < D; ++i) mu[i] = c.modp(u[i] + c.neg_q() * u[i + 1]);
            mu[D] = u[D];
        } else {
#pragma unroll
            for (int i = 0; i < ND; ++i) mu[i] = u[i];
        }
    } else {
        constexpr int A = (D + W - 2) / (W - 1);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int s = a * (W - 1);
            uint32_t idx = 0;
#pragma unroll
            for (int j = W - 1; j >= 0; --j) idx = idx * c.radix() + (s + j <= D ? u[s + j] : 0u);
            const uint32_t e = tab(idx);
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (s + j <= D && (j + 1 < W || s + j == D)) mu[s + j] = byte_of(e, j);
        }
    }
}

// floor(r/3) for any 64-bit r in exact 32-bit integer arithmetic: with
// r = rh 2^32 + rl, rh = 3 qh + mh and rl = 3 ql + rr,
// floor(r/3) = qh 2^32 + mh (2^32-1)/3 + ql + [mh + rr >= 3]  (2^32 == 1 mod 3;
// the low part stays below 2^32).  No fp64 instruction (scripts/repack_int_probe.cpp).
__host__ __device__ __forceinline__ uint64_t div3_u64(uint64_t r) {
    const uint32_t rh = static_cast<uint32_t>(r >> 32), rl = static_cast<uint32_t>(r);
#ifdef __CUDA_ARCH__
    const uint32_t qh = __umulhi(rh, 0xAAAAAAABu) >> 1, ql = __umulhi(rl, 0xAAAAAAABu) >> 1;
#else
    const uint32_t qh = static_cast<uint32_t>((uint64_t(rh) * 0xAAAAAAABu) >> 33);
    const uint32_t ql = static_cast<uint32_t>((uint64_t(rl) * 0xAAAAAAABu) >> 33);
#endif
    const uint32_t mh = rh - 3 * qh, rr = rl - 3 * ql;
    const uint32_t lo = mh * 0x55555555u + ql + ((mh + rr + 1) >> 2);
    return (uint64_t(qh) << 32) | lo;
}

// REDQ for p = 3, q = 2^B (4 <= B <= 7) inside one 64-bit integer, lane i =
// bits [Bi, Bi+B) (the C5 re-pack trick, gfq_matmul.cuh, generalised to both
// signs of q mod 3):
//  * u_i = floor(r/q^i) mod 3 is fixed by its value mod 4, and
//    (r >> Bi) - 3 (rop >> Bi) == a_i + b_i (mod 4), a_i and b_i the two low
//    bits of lane i of r and rop (-3 == 1 mod 4);
//  * mu_i = (u_i + neg_q u_{i+1}) mod 3 lane-wise: neg_q = 2 (B even) as
//    V = u_i + 8 - u_{i+1}, neg_q = 1 (B odd) as V = u_i + u_{i+1} + 5, both in
//    [5, 10], then mu = V - 5 - 3 [V >= 8]; no lane ever borrows.
// Residues of many groups add up in the same lanes (<= 2 each) and are folded
// back below 3 (4 == 1 mod 3) before a lane can overflow.
template <int B, int ND>
struct Swar3 {
    static constexpr uint64_t M1 = [] {
        uint64_t m = 0;
        for (int i = 0; i < ND && B * i < 64; ++i) m |= uint64_t(1) << (B * i);
        return m;
    }();
    static constexpr uint64_t M3 = 3 * M1, Mlow = ((uint64_t(1) << (B - 2)) - 1) * M1;
    static constexpr uint32_t adds = ((1u << B) - 3) / 2;  // lanes stay below 2^B
    static constexpr bool negq1 = (B & 1) != 0;           // 2^B mod 3 = 2 for odd B: neg_q = 1
    __device__ __forceinline__ static uint64_t mu(double r, double inv_p) { return mu(dbits(r + kTwo52), r, inv_p); }
    // rb: the word as an integer (low 52 bits), r: the same word as a double
    __device__ __forceinline__ static uint64_t mu(uint64_t rb, double r, double inv_p) {
        const uint64_t ob = dbits(__dadd_rz(__dmul_ru(r, inv_p), kTwo52));  // low 52 bits = floor(r/3)
        const uint64_t u = ((rb & M3) + (ob & M3)) & M3;
        const uint64_t v = negq1 ? u + (u >> B) + 5 * M1 : u + 8 * M1 - (u >> B);
        return v - 5 * M1 - 3 * ((v >> 3) & M1);
    }
    __device__ __forceinline__ static uint64_t fold(uint64_t x) {
        x = ((x >> 2) & Mlow) + (x & M3);
        if constexpr (B > 5) x = ((x >> 2) & Mlow) + (x & M3);
        x = ((x >> 2) & M3) + (x & M3);  // lanes <= 5
        return x - 3 * (((x + 5 * M1) >> 3) & M1);
    }
};

// shared-memory u32 load at a 32-bit shared address
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

// shared-memory u16 load (zero-extended)
__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
    return v;
}

}  // namespace qpk
