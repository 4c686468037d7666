// HBM-streaming kernels of the q-adic pipeline on sm_100a:
//
//   K2  batched REDQ / FQT-inverse      fp64 words -> d+1 residues (uint8)
//   C1  fused DQT pack + fp64 product + REDQ (batched small polymul)
//   K3  GF(p^k) elementwise product, DQT/REDQ/L-H path or dlog/Zech path
//
// All three share one persistent TMA pipeline (stream_tma_kernel): a CTA
// owns tiles of THREADS*R records; one elected thread moves each input tile
// global->shared with cp.async.bulk (completion on an mbarrier, STAGES deep)
// and each finished output tile shared->global with a bulk store, so every
// HBM transfer is a long contiguous burst regardless of the awkward 7- or
// 3-byte record sizes.  Threads only touch shared memory, each one a run of R
// consecutive records, and all lookup tables (REDQ correction windows, L/H
// half tables, log/antilog) are staged in shared memory per CTA.
//
// (templates only: instantiated per digit count / record width in
// stream_inst.cu, compiled once per -DQPK_INST value so nvcc runs in parallel)
//
// Records that do not fill a whole tile, or buffers that are not 16-byte
// aligned, go through stream_tail_kernel (plain byte loads, same op).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.hpp"
#include "redq_core.cuh"

namespace qpk {

namespace {

constexpr int kThreads = 256;  // threads per CTA of the stream kernels (default)

// records -> contiguous byte stream -> u32 words (all indices constexpr)
template <int R, int OUT>
__device__ __forceinline__ void pack_records(const uint64_t (&rec)[R], uint32_t (&ow)[R * OUT / 4]) {
#pragma unroll
    for (int i = 0; i < R * OUT / 4; ++i) {
        uint32_t w = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int g = 4 * i + b;
            w |= static_cast<uint32_t>((rec[g / OUT] >> (8 * (g % OUT))) & 0xffu) << (8 * b);
        }
        ow[i] = w;
    }
}

// byte `i` of a run of packed u32 words
__device__ __forceinline__ uint32_t run_byte(const uint32_t* w, int i) { return byte_of(w[i >> 2], i & 3); }

// residues mu_0..mu_{ND-1} of one word, packed one per byte
template <int ND, int W, class K, class TabLoad>
__device__ __forceinline__ uint64_t redq_record(const K& c, double r, TabLoad tab_load) {
    uint32_t u[ND];
    redq_raw_digits<ND>(c, r, u);
    constexpr int D = ND - 1;
    if constexpr (W > 0 && D > 0) {
        if (c.neg_q() != 0) {
            // windowed table (Alg. 3): window a covers digits s..s+W-1,
            // s = a(W-1); its first W-1 residues are final, the last one only
            // at the top digit
            constexpr int A = (D + W - 2) / (W - 1);
            uint64_t rec = 0;
#pragma unroll
            for (int a = 0; a < A; ++a) {
                const int s = a * (W - 1);
                uint32_t idx = 0;
#pragma unroll
                for (int j = W - 1; j >= 0; --j) idx = idx * c.radix() + (s + j <= D ? u[s + j] : 0u);
                const uint32_t e = tab_load(idx);
                const int keep = (a == A - 1) ? (D - s + 1) : (W - 1);  // bytes of this window kept
                const uint32_t mask = keep >= 4 ? 0xffffffffu : ((1u << (8 * keep)) - 1);
                rec |= static_cast<uint64_t>(e & mask) << (8 * s);
            }
            return rec;
        }
    }
    uint32_t mu[ND];
    redq_correct<ND, 0>(c, u, mu, [](uint32_t) { return 0u; });
    uint64_t rec = 0;
#pragma unroll
    for (int j = 0; j < ND; ++j) rec |= static_cast<uint64_t>(mu[j]) << (8 * j);
    return rec;
}
// ... with the table staged in shared memory at byte address tab_saddr
template <int ND, int W, class K>
__device__ __forceinline__ uint64_t redq_record(const K& c, double r, uint32_t tab_saddr) {
    return redq_record<ND, W>(c, r, [tab_saddr](uint32_t idx) { return lds_u32(tab_saddr + 4 * idx); });
}

// ----------------------------------------------------------------- ops
// An op maps R consecutive records (IN0 + IN1 bytes each, as packed
// little-endian u32 words) to R output records of OUT bytes (packed u32).

template <int ND, int W, class K>
struct RedqOp {
    static constexpr int IN0 = 8, IN1 = 0, OUT = ND, R = 4, RR = 2, S = 3;
    RedqParams P;
    __host__ __device__ uint32_t tables_words() const { return W ? P.n_entries : 0u; }
    __host__ __device__ const uint32_t* tables_src() const { return P.table; }
    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t*, uint32_t (&ow)[R * OUT / 4],
                                          uint32_t tab, uint32_t& err) const {
        const K c{P};
        uint64_t rec[R];
        if constexpr (K::kSafe) {
            // the safe plans have a power-of-two limit 2^e (low word 0), so
            // 0 <= w < limit  <=>  hi32(w) < hi32(limit) as unsigned ints
            // (negatives carry the sign bit, NaN/inf the top exponent); one
            // compare for the whole run, the exact check only on a miss
            uint32_t hmax = a[1];
#pragma unroll
            for (int r = 1; r < R; ++r) hmax = max(hmax, a[2 * r + 1]);
            const uint32_t lim_hi = static_cast<uint32_t>(__double_as_longlong(P.limit) >> 32);
            if (hmax < lim_hi) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double w = __hiloint2double(static_cast<int>(a[2 * r + 1]), static_cast<int>(a[2 * r]));
                    rec[r] = redq_record<ND, W>(c, trunc(w), tab);
                }
                pack_records<R, OUT>(rec, ow);
                return;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double w = __hiloint2double(static_cast<int>(a[2 * r + 1]), static_cast<int>(a[2 * r]));
            uint32_t e = 0;
            double x = checked_word(P, w, e);
            if constexpr (K::kSafe) x = e ? 0.0 : x;  // keep table indices in range
            err |= e;
            rec[r] = redq_record<ND, W>(c, x, tab);
        }
        pack_records<R, OUT>(rec, ow);
    }
};

// coefficient records: reduce mod p (DensePoly, poly.hpp:19-21) unless every
// byte is already below p
template <int K_, class C>
__device__ __forceinline__ void record_coeffs(const C& c, uint32_t magic, const uint32_t* w, int rec,
                                              uint32_t (&cf)[K_]) {
#pragma unroll
    for (int i = 0; i < K_; ++i) cf[i] = run_byte(w, rec * K_ + i);
    bool clean = true;
#pragma unroll
    for (int i = 0; i < K_; ++i) clean &= cf[i] < c.p();
    if (!clean) {
#pragma unroll
        for (int i = 0; i < K_; ++i) cf[i] = mod_by_magic(cf[i], c.p(), magic);
    }
}

// DQT pack at q (dqt.cpp:23-37): exact integer as a double
template <int K_, class C>
__device__ __forceinline__ double pack_word(const C& c, double qd, const uint32_t (&cf)[K_]) {
    if constexpr (C::kPow2) {
        uint64_t v = 0;
#pragma unroll
        for (int i = K_ - 1; i >= 0; --i) v = (v << c.qbits()) | cf[i];
        // exact as a double below 2^52: a magic add instead of an I2F.F64
        // conversion (quarter-rate pipe)
        if constexpr (C::kSafe) return __longlong_as_double(static_cast<long long>(v | 0x4330000000000000ull)) - kTwo52;
        else return static_cast<double>(v);
    } else {
        double v = 0.0;
#pragma unroll
        for (int i = K_ - 1; i >= 0; --i) v = fma(v, qd, static_cast<double>(cf[i]));
        return v;
    }
}

// every byte of N packed words is below p (p < 128): b + 128 - p sets a
// byte's top bit iff p <= b < 128; bytes >= 128 carry it already.  Only
// such bytes can carry into a neighbour, so carries never hide a bad byte
// (at worst they flag a good one and the exact path runs).
template <int N>
__device__ __forceinline__ bool all_bytes_below(const uint32_t* w, uint32_t p) {
    const uint32_t add = (128u - p) * 0x01010101u;
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) bad |= w[i] | (w[i] + add);
    return (bad & 0x80808080u) == 0;
}

// record r (k bytes, little endian) of a packed run as an integer
template <int K_>
__device__ __forceinline__ uint32_t record_int(const uint32_t* w, int r) {
    const int byte = r * K_, i = byte >> 2, sh = 8 * (byte & 3);
    const uint32_t lo = w[i];
    const uint32_t hi = (sh + 8 * K_ > 32) ? w[i + 1] : 0u;
    const uint32_t v = sh ? __funnelshift_r(lo, hi, sh) : lo;
    return K_ == 4 ? v : (v & ((1u << (8 * K_)) - 1));
}

#ifndef QPK_PM_R  // tile geometry of the batched polynomial product
#define QPK_PM_R 4
#endif
#ifndef QPK_PM_RR
#define QPK_PM_RR 1
#endif
#ifndef QPK_PM_S
#define QPK_PM_S 2
#endif
// C1's field on byte lanes: F_3[X] products of degree < 4 at q = 2^5 (seven
// digits), the config's pipeline -- DQT pack (dqt.cpp:23-37), fp64 product,
// REDQ with the Lemma-1 floor (redq.cpp:31-60) and the mod-p correction
// (redq.cpp:63-65; neg_q = 1) -- with every step on all lanes of a register
// at once.  The generic path spends ~100 instructions per pair, most of them
// on the 16-lane ALU pipe (ncu r02 c1: ALU the busiest pipe, 102
// thread-instructions per pair); this one ~40, split between the ALU and FMA
// pipes.  xa, xb: the four coefficient bytes of each operand, all below 3
// (checked by the caller for the whole run).  Returns residue bytes 0-3 and
// (by reference) bytes 4-6.
//  * pack: moving a byte field left by s is x + (2^s - 1)(x & field): two
//    multiply-adds put byte i at bit 5i + 9, and the double with exponent
//    2^43 whose low mantissa word that is equals 2^43 + A exactly;
//  * u_i = floor(r/q^i) - 3 floor(rop/q^i) lies in [0, 2] and is fixed mod 4
//    by the low two bits of lane i of r and of rop (-3 == 1 mod 4); lane 6
//    starts at bit 30, so all seven 2-bit fields sit in the low words;
//  * mu_i = (u_i + u_{i+1}) mod 3 (mu_6 = u_6): v = u + (u >> 5) <= 4,
//    minus 3 where v >= 3;
//  * the 2-bit fields at 5i are spread to bytes by the same multiply-adds.
__device__ __forceinline__ uint32_t polymul_f3q32(double inv_p, uint32_t xa, uint32_t xb, uint32_t& hi3) {
    constexpr uint32_t kM1 = 0x42108421u, kM3 = 3u * kM1;  // bit 0 / bits 0-1 of every 5-bit lane
    const uint32_t ya = xa + 7u * (xa & 0x00030003u);      // bytes 0, 2 up by 3: fields at 3, 8, 19, 24
    const uint32_t yb = xb + 7u * (xb & 0x00030003u);
    const uint32_t pa = ya + 63u * (ya & 0x0000ffffu);     // low pair up by 6: fields at 9, 14, 19, 24
    const uint32_t pb = yb + 63u * (yb & 0x0000ffffu);
    const double da = __hiloint2double(0x42a00000, static_cast<int>(pa)) - 8796093022208.0;  // 2^43 + A - 2^43
    const double db = __hiloint2double(0x42a00000, static_cast<int>(pb)) - 8796093022208.0;
    const double r = da * db;  // exact, < 2^35
    const uint32_t rl = static_cast<uint32_t>(dbits(r + kTwo52));
    const uint32_t ol = static_cast<uint32_t>(dbits(__dadd_rz(__dmul_ru(r, inv_p), kTwo52)));
    const uint32_t u = ((rl & kM3) + (ol & kM3)) & kM3;
    const uint32_t v = u + (u >> 5);
    const uint32_t g = ((v + kM1) >> 2) & kM1;
    const uint32_t mu = v - 3u * g;
    uint32_t lo = mu & 0x00018c63u;          // residues 0-3 at 0, 5, 10, 15
    lo += 63u * (lo & 0x00018c00u);          // 2, 3 up by 6: 0, 5, 16, 21
    lo += 7u * (lo & 0x00600060u);           // 1, 3 up by 3: 0, 8, 16, 24
    uint32_t hi = mu >> 20;                  // residues 4-6 at 0, 5, 10
    hi += 63u * (hi & 0x00000c00u);          // 6 up by 6: 0, 5, 16
    hi += 7u * (hi & 0x00000060u);           // 5 up by 3: 0, 8, 16
    hi3 = hi;
    return lo;
}

template <class K>
constexpr bool is_f3_q32() {
    if constexpr (K::kSafe) return K::kP == 3 && K::kQbitsCt == 5;
    else return false;
}

template <int K_, int W, class K>
struct PolymulOp {
    static constexpr int ND = 2 * K_ - 1;
    static constexpr int IN0 = K_, IN1 = K_, OUT = ND, R = QPK_PM_R, RR = QPK_PM_RR, S = QPK_PM_S;
    PolymulParams P;
    // F_3, q = 2^5, k = 4 (C1): runs of clean bytes take polymul_f3q32, which
    // needs no table; the record-by-record path then reads the window table
    // from global memory, so no launch stages it (the staging and its CTA
    // barrier cost 0.26 us of a 4.8 us launch) and the one-wave direct kernel
    // is held to 7 CTAs per SM (32 registers: all 1024 CTAs of C1 resident)
    static constexpr bool kF3Q32 = K_ == 4 && R == 4 && W > 0 && is_f3_q32<K>();
    static constexpr int kDirectMinBlocks = kF3Q32 ? 7 : 1;
    __host__ __device__ uint32_t tables_words() const { return W && !kF3Q32 ? P.rq.n_entries : 0u; }
    __host__ __device__ const uint32_t* tables_src() const { return P.rq.table; }
    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t* b, uint32_t (&ow)[R * OUT / 4],
                                          uint32_t tab, uint32_t&) const {
        const K c{P.rq};
        const double qd = static_cast<double>(P.rq.q);
        uint64_t rec[R];
        // one range check for the whole run (bytes >= p are reduced mod p,
        // DensePoly, record by record on the slow path)
        bool clean = false;
        if constexpr (K::kSafe) {
            if constexpr ((R * K_) % 4 == 0 && K::kP < 128)
                clean = all_bytes_below<R * K_ / 4>(a, c.p()) && all_bytes_below<R * K_ / 4>(b, c.p());
            if constexpr (kF3Q32) {
                if (clean) {
                    uint32_t lo[R], hi[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) lo[r] = polymul_f3q32(P.rq.inv_p, a[r], b[r], hi[r]);
                    // four 7-byte records as seven words
                    ow[0] = lo[0];
                    ow[1] = __byte_perm(hi[0], lo[1], 0x4210);
                    ow[2] = __byte_perm(lo[1], hi[1], 0x4321);
                    ow[3] = __byte_perm(hi[1], lo[2], 0x5421);
                    ow[4] = __byte_perm(lo[2], hi[2], 0x5432);
                    ow[5] = __byte_perm(hi[2], lo[3], 0x6542);
                    ow[6] = __byte_perm(lo[3], hi[3], 0x6543);
                    return;
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t ca[K_], cb[K_];
            if (clean) {
#pragma unroll
                for (int i = 0; i < K_; ++i) ca[i] = run_byte(a, r * K_ + i), cb[i] = run_byte(b, r * K_ + i);
            } else {
                record_coeffs<K_>(c, P.rq.mod_magic, a, r, ca);
                record_coeffs<K_>(c, P.rq.mod_magic, b, r, cb);
            }
            // exact: q^(2k-1) < 2^53 (validated)
            const double word = pack_word<K_>(c, qd, ca) * pack_word<K_>(c, qd, cb);
            if constexpr (kF3Q32) {
                const uint32_t* gtab = P.rq.table;
                rec[r] = redq_record<ND, W>(c, word, [gtab](uint32_t idx) { return __ldg(gtab + idx); });
            } else {
                rec[r] = redq_record<ND, W>(c, word, tab);
            }
        }
        pack_records<R, OUT>(rec, ow);
    }
};

// bytewise (x + y) mod p of packed coefficient bytes, each < p
__device__ __forceinline__ uint32_t add_mod_bytes(uint32_t x, uint32_t y, uint32_t p, uint32_t k) {
    if (p < 128) {
        const uint32_t pp = p * 0x01010101u;
        const uint32_t s = __vadd4(x, y);
        return __vsub4(s, __vcmpgeu4(s, pp) & pp);
    }
    uint32_t r = 0;
    for (uint32_t i = 0; i < k; ++i) {
        uint32_t t = byte_of(x, i) + byte_of(y, i);
        if (t >= p) t -= p;
        r |= t << (8 * i);
    }
    return r;
}


__device__ __forceinline__ uint32_t add_mod_bytes_fast(uint32_t x, uint32_t y, uint32_t p);

// bytewise t mod p of a packed word (bytes may be any value)
__device__ __forceinline__ uint32_t bytes_mod_p(uint32_t w, uint32_t p, uint32_t magic) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) r |= mod_by_magic((w >> (8 * j)) & 0xffu, p, magic) << (8 * j);
    return r;
}

// GF(p^k) product for q = 2^8, k = 3, p < 8 through the reference's
// pipeline (gfq.cpp:353-384 with one term): DQT pack, fp64 product, REDQ,
// L/H tables.  A record of 3 coefficient bytes IS its DQT word at q = 2^8
// (dqt.cpp:23-37), exact as a double; the fp64 product is exact (< 2^48).
// REDQ: rop = floor(r/p) by the premultiplied reciprocal (Lemma 1, RU
// multiply + RZ magic add), then the raw digits u_i = (r >> 8i) - p (rop >> 8i)
// (redq.cpp:31-60).  u_i in [0, p-1] is fixed by its value mod 8, i.e. by the
// low 3 bits of byte i of r and rop: u_i == a_i + (-p mod 8) b_i (mod 8) --
// one masked multiply-add gives all five digits as byte lanes (no lane
// carries: 7 + 7*7 < 256).  The L and H tables are indexed by the base-p
// value of digit lanes 0..2 and 2..4 (one dp4a each; lane 3 has weight 0)
// in this lane's private copies (every lookup of a warp is one
// conflict-free wavefront): L as u16 (its low half has degree < k-1 = 2, so
// two coefficient bytes), entry e at byte 128 (e >> 1) + 2 (e & 1) + 4 lane;
// H as u32 coefficient bytes at byte hoff + 128 e + 4 lane.
template <class C>
__device__ __forceinline__ uint32_t lh_product_lane(double inv_p, uint32_t ra, uint32_t rb, uint32_t tb,
                                                    uint32_t hb) {
    constexpr uint32_t P = C::kP;
    constexpr uint32_t F = (8u - P % 8u) % 8u;
    constexpr uint32_t kWeights = 1u | (P << 8) | (P * P << 16);
    // the packed words as doubles (exact magic-add conversions) and their product
    // (I2F.F64 conversions measured 34.6 vs 34.1 us per C3 launch)
    const double wa = __hiloint2double(0x43300000, static_cast<int>(ra)) - kTwo52;
    const double wb = __hiloint2double(0x43300000, static_cast<int>(rb)) - kTwo52;
    const double r = wa * wb;
    const uint64_t rw = dbits(r + kTwo52);                             // low 52 bits: r as an integer
    const uint64_t ob = dbits(__dadd_rz(__dmul_ru(r, inv_p), kTwo52));  // low 52 bits: floor(r/p)
    const uint32_t lo = (static_cast<uint32_t>(rw) & 0x07070707u) + (static_cast<uint32_t>(ob) & 0x07070707u) * F;
    const uint32_t hi = static_cast<uint32_t>(rw >> 32) + static_cast<uint32_t>(ob >> 32) * F;  // lane 0: digit 4
    const uint32_t il = __dp4a(lo & 0x07070707u, kWeights, 0u);
    const uint32_t ih = __dp4a(__funnelshift_r(lo, hi, 16) & 0x07070707u, kWeights, 0u);
    const uint32_t lv = lds_u16(tb + (il << 6) - (il & 1u) * 62u);
    const uint32_t hv = lds_u32(hb + (ih << 7));
    return lv + hv;  // coefficient lanes < 2p: the caller reduces them mod p (bytes_below_2p_mod)
}

// bytewise t mod p for byte lanes below 2p <= 128 (carry-free)
__device__ __forceinline__ uint32_t bytes_below_2p_mod(uint32_t t, uint32_t p) {
    return t - p * (((t + (128u - p) * 0x01010101u) >> 7) & 0x01010101u);
}

// dlog product on the fast-path tables (gfq.cpp:260-264): the logs of both
// records (base-p index by one dp4a; byte lane 3 of y has weight 0) from
// this lane's private log copy, pre-scaled to antilog byte offsets with zero
// at 2g-1, so the sum indexes the doubled antilog table with no reduction
// mod g and any sum involving zero clamps to its zero entry
template <uint32_t P>
__device__ __forceinline__ uint32_t dlog_product_lane(uint32_t ya, uint32_t yb, uint32_t lg, uint32_t al,
                                                      uint32_t zero4) {
    constexpr uint32_t kWeights = 1u | (P << 8) | (P * P << 16);
    const uint32_t s = lds_u32(lg + 128u * __dp4a(ya, kWeights, 0u)) + lds_u32(lg + 128u * __dp4a(yb, kWeights, 0u));
    return lds_u32(al + min(s, zero4));
}

// GF(7^3) product on the integer DQT word (q = 2^8).  With coefficients
// below 7 the q-adic word product ra*rb has byte lanes c_0..c_4, c_j =
// sum a_i b_(j-i) <= 108 < q, so the convolution needs no carry handling in
// 64-bit integers (the fp64 product of the reference is the same exact
// integer).  Digit reduction mod p and reduction by the field polynomial are
// linear over GF(7): c_0..c_2 + (c_3 mod 7) x^3 + (c_4 mod 7) x^4 with x^3, x^4
// as packed coefficient bytes gives lanes <= 180, reduced by lanes_mod7.
__device__ __forceinline__ uint32_t gf73_lanes(uint32_t ra, uint32_t rb, uint32_t col3, uint32_t col4) {
    const uint64_t w = static_cast<uint64_t>(ra) * rb;
    const uint32_t lo = static_cast<uint32_t>(w), c4 = static_cast<uint32_t>(w >> 32);
    const uint32_t c3 = lo >> 24;
    constexpr uint32_t kMagic7 = 613566757u;  // ceil(2^32 / 7)
    return (lo & 0xffffffu) + mod_by_magic(c3, 7u, kMagic7) * col3 + mod_by_magic(c4, 7u, kMagic7) * col4;
}

// bytewise x mod 7 for any byte lanes (8 == 1 mod 7: x - 7 floor(x/8) keeps
// the residue and leaves each lane non-negative, so no borrow crosses a lane)
__device__ __forceinline__ uint32_t lanes_mod7(uint32_t t) {
    t -= 7u * ((t >> 3) & 0x1f1f1f1fu);  // lanes <= 7 + 31
    t -= 7u * ((t >> 3) & 0x07070707u);  // lanes <= 7 + 4
    const uint32_t ge = ((t + 0x79797979u) >> 7) & 0x01010101u;
    return t - 7u * ge;
}

// word holding record r of a packed 3-byte run in its low 24 bits (upper byte
// unspecified)
__device__ __forceinline__ uint32_t record24(const uint32_t* w, int r) {
    const int byte = 3 * r, i = byte >> 2, sh = 8 * (byte & 3);
    if (sh == 0) return w[i];
    if (sh == 8) return w[i] >> 8;
    return __funnelshift_r(w[i], w[i + 1], sh);
}

// the compile-time fast path (kernels.hpp gfq_fast_field): GF(7^3), q = 2^8
template <class K>
constexpr bool ct_fast_field() {
    if constexpr (K::kSafe) return K::kP == 7 && K::kQbitsCt == 8;
    else return false;
}


// coefficient index sum c_i p^i of a record integer (bytes c_i)
template <int K_, class C>
__device__ __forceinline__ uint32_t coeff_index(const C& c, uint32_t rec) {
    uint32_t idx = 0;
#pragma unroll
    for (int i = K_ - 1; i >= 0; --i) idx = idx * c.p() + ((rec >> (8 * i)) & 0xffu);
    return idx;
}

// (x + y) mod p bytewise for packed bytes below p < 128, carry-free
__device__ __forceinline__ uint32_t add_mod_bytes_fast(uint32_t x, uint32_t y, uint32_t p) {
    const uint32_t s = x + y;                                     // bytes < 2p <= 255
    const uint32_t ge = ((s + (128u - p) * 0x01010101u) >> 7) & 0x01010101u;  // byte >= p
    return s - ge * p;
}

// one GF(p^k) product through DQT/REDQ/L-H with q = 2^8 (record = word)
template <int K_, class C>
__device__ __forceinline__ uint32_t lh_product(const C& c, uint32_t ra, uint32_t rb, uint32_t lc, uint32_t hc) {
    constexpr int ND = 2 * K_ - 1;
    const double prod = static_cast<double>(ra) * static_cast<double>(rb);  // exact, < 2^(16k)
    uint32_t u[ND];
    redq_raw_digits<ND>(c, prod, u);
    uint32_t il = 0, ih = 0;
#pragma unroll
    for (int i = K_ - 1; i >= 0; --i) {
        il = il * c.p() + u[i];
        ih = ih * c.p() + u[K_ - 1 + i];
    }
    return add_mod_bytes_fast(lds_u32(lc + 4 * il), lds_u32(hc + 4 * ih), c.p());
}

// one GF(p^k) product in the dlog representation (gfq.cpp:260-264)
template <int K_, class C>
__device__ __forceinline__ uint32_t dlog_product(const C&, uint32_t ia, uint32_t ib, uint32_t lg, uint32_t al,
                                                 uint32_t group) {
    const uint32_t ra = lds_u32(lg + 4 * ia), rb = lds_u32(lg + 4 * ib);
    uint32_t rc = ra + rb;
    rc = rc >= group ? rc - group : rc;
    rc = (ra == group || rb == group) ? group : rc;
    return lds_u32(al + 4 * rc);
}

#ifndef QPK_GFE_R  // tile geometry of the GF elementwise op (records/run, runs/tile, stages)
#define QPK_GFE_R 8
#endif
#ifndef QPK_GFE_RR
#define QPK_GFE_RR 2
#endif
#ifndef QPK_GFE_S
#define QPK_GFE_S 2
#endif
// MODE: kGfqPacked / kGfqDlog / kGfqLinear as a compile-time choice (fast
// paths), -1 = P.mode
// ... and of the fast field's REDQ/L-H (PK) and dlog (DL) paths: 66 / 88 KB
// of lane-private tables, outputs stored straight from registers (kDirectStore),
// one CTA of 512 consumer threads (+ the producer warp) per SM, 8-record
// runs x 4 stages.  Measured over rotating buffers larger than L2 (C3, 2^24
// products, scripts/c3_sweep.py, PK / DL): two CTAs of 256 threads, 16-record
// runs x 2 stages, CTA-barrier pipeline 31.3 / 28.1 us; with the producer
// warp 30.7 / 28.1; one CTA of 512, 8-record runs x 4 stages 29.8 / 27.0
// (16 antilog copies); x 5-6 stages, 4-record runs x 8 stages, 16-record
// runs x 2 stages and 768 threads all measured slower.
#ifndef QPK_GFE_PK_RR
#define QPK_GFE_PK_RR 1
#endif
#ifndef QPK_GFE_PK_R
#define QPK_GFE_PK_R 8
#endif
#ifndef QPK_GFE_PK_S
#define QPK_GFE_PK_S 4
#endif
#ifndef QPK_GFE_PK_T
#define QPK_GFE_PK_T 512
#endif
#ifndef QPK_GFE_DL_R
#define QPK_GFE_DL_R 8
#endif
#ifndef QPK_GFE_DL_S
#define QPK_GFE_DL_S 4
#endif
#ifndef QPK_GFE_DL_T
#define QPK_GFE_DL_T 512
#endif
// the fast field's linear path (no tables): measured (c3_sweep) 26.5 us with
// the generic geometry; direct stores + producer warp at 512 x 8 x 6 stages
// 26.7-27.2, 256 x 16 x 4 28.7-29.1, bulk stores at 256 x 8 x 2 x 4 34.5
#ifndef QPK_GFE_LN_R
#define QPK_GFE_LN_R QPK_GFE_R
#endif
#ifndef QPK_GFE_LN_RR
#define QPK_GFE_LN_RR QPK_GFE_RR
#endif
#ifndef QPK_GFE_LN_S
#define QPK_GFE_LN_S QPK_GFE_S
#endif
#ifndef QPK_GFE_LN_T
#define QPK_GFE_LN_T kThreads
#endif
template <int K_, class K, int MODE = -1>
struct GfqElemOp {
    static constexpr int ND = 2 * K_ - 1;
    // fast path (GF(7^3), q = 2^8) when the host built its block
    static constexpr bool kFast = K_ == 3 && ct_fast_field<K>();
    static constexpr bool kFastDlog = kFast && MODE == kGfqDlog;
    static constexpr int IN0 = K_, IN1 = K_, OUT = K_;
    static constexpr bool kFastLin = kFast && MODE == kGfqLinear;
    static constexpr int R = kFastDlog ? QPK_GFE_DL_R : (kFast && MODE == kGfqPacked) ? QPK_GFE_PK_R
                             : kFastLin ? QPK_GFE_LN_R : QPK_GFE_R;
    static_assert(!kFast || R % 4 == 0, "the fast path handles groups of 4 records");
    static constexpr uint32_t kP = [] {
        if constexpr (kFast) return K::kP;
        else return 0u;
    }();
    static constexpr uint32_t kP3 = kP * kP * kP;
    // its REDQ/L-H and dlog paths stage 66 / 88 KB of tables (lane-private
    // copies, kernels.hpp fast_off) beside 4 input stages of 24 KB
    static constexpr bool kLanePriv = kFast && (MODE == kGfqPacked || MODE == kGfqDlog);
    static constexpr int RR = kLanePriv ? QPK_GFE_PK_RR : kFastLin ? QPK_GFE_LN_RR : QPK_GFE_RR;
    static constexpr int S = kFastDlog ? QPK_GFE_DL_S : kLanePriv ? QPK_GFE_PK_S : kFastLin ? QPK_GFE_LN_S : QPK_GFE_S;
    static constexpr int THREADS = kFastDlog ? QPK_GFE_DL_T : kLanePriv ? QPK_GFE_PK_T : kFastLin ? QPK_GFE_LN_T : kThreads;
    // block words: L16 | H | LOG | ALOG copies
    static constexpr uint32_t kLWords = (kP3 + 1) / 2, kHOff = kLWords, kLogOff = kLWords + kP3,
                              kAlogOff = (kLWords + 2 * kP3 + 3) / 4 * 4;  // 16-byte aligned
    static constexpr bool kCustomStage = kFast;
#ifndef QPK_GFE_DS
#define QPK_GFE_DS 1
#endif
#ifndef QPK_GFE_LIN_DS
#define QPK_GFE_LIN_DS 0
#endif
    static constexpr bool kDirectStore = (kLanePriv && QPK_GFE_DS) || (kFast && MODE == kGfqLinear && QPK_GFE_LIN_DS);
    GfqElemParams P;
    __host__ __device__ bool fast() const { return kFast && P.fast_off != 0; }
    __host__ __device__ __forceinline__ int mode() const {
        const int m = MODE < 0 ? P.mode : MODE;
        return (m == kGfqLinear && !kFast) ? kGfqPacked : m;  // linear: the fast field only
    }
    __host__ __device__ __forceinline__ bool packed() const { return mode() != kGfqDlog; }
    __host__ __device__ bool custom_stage() const { return fast() && mode() != kGfqLinear; }
    __host__ __device__ uint32_t alog_words() const { return 2 * P.group * kDlogCopies; }
    // staged tables: lc|hc|log|alog, or on the fast field what its path reads:
    // lane-private L|H (packed), lane-private log + the antilog copies (dlog),
    // nothing (linear)
    __host__ __device__ uint32_t tables_words() const {
        if (fast()) {
            if (mode() == kGfqLinear) return 0u;
            return mode() == kGfqDlog ? 32u * kP3 + alog_words() : 32u * (kLWords + kP3);
        }
        return P.fast_off ? P.fast_off : P.tables_words;
    }
    __host__ __device__ const uint32_t* tables_src() const { return P.lc + (fast() ? P.fast_off : 0u); }
    // lane-private copies: warp w moves block words [32c, 32c + 32) for
    // c = w, w + 8, ... (one coalesced load, then word j goes to 32 j + lane);
    // the dlog path then copies the interleaved antilog block behind them
    __device__ void stage_custom(uint32_t* dst) const {
        const bool dl = mode() == kGfqDlog;
        const uint32_t* src = P.lc + P.fast_off + (dl ? kLogOff : 0u);
        const uint32_t n = dl ? kP3 : kLWords + kP3;
        const uint32_t lane = threadIdx.x & 31u, nw = blockDim.x >> 5;
        for (uint32_t c = threadIdx.x >> 5; 32 * c < n; c += nw) {
            const uint32_t j0 = 32 * c;
            const uint32_t mine = j0 + lane < n ? __ldg(src + j0 + lane) : 0u;
#pragma unroll 8
            for (uint32_t j = 0; j < 32; ++j) {
                const uint32_t v = __shfl_sync(0xffffffffu, mine, j);
                if (j0 + j < n) dst[32 * (j0 + j) + lane] = v;
            }
        }
        if (dl) {
            const uint4* a = reinterpret_cast<const uint4*>(P.lc + P.fast_off + kAlogOff);  // 16-byte aligned
            uint4* d = reinterpret_cast<uint4*>(dst + 32 * kP3);
            for (uint32_t i = threadIdx.x; i < alog_words() / 4; i += blockDim.x) d[i] = __ldg(a + i);
        }
    }

    // groups of 4 records = 3 packed words
    __device__ __forceinline__ void apply_fast(const uint32_t* a, const uint32_t* b, uint32_t (&ow)[R * OUT / 4],
                                                 uint32_t tab) const {
        const K c{P.rq};
        constexpr int NW = R * 3 / 4;
        uint32_t aw[NW], bw[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) aw[i] = a[i], bw[i] = b[i];
        if (!(all_bytes_below<NW>(aw, c.p()) && all_bytes_below<NW>(bw, c.p()))) {
            // coefficient bytes >= p are reduced mod p, as record_coeffs does
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                aw[i] = bytes_mod_p(aw[i], c.p(), P.rq.mod_magic);
                bw[i] = bytes_mod_p(bw[i], c.p(), P.rq.mod_magic);
            }
        }
        if constexpr (kFast) {
            if (mode() == kGfqLinear) {
#pragma unroll
                for (int g = 0; g < R / 4; ++g) {
                    uint32_t t[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        t[r] = gf73_lanes(record24(aw + 3 * g, r) & 0xffffffu, record24(bw + 3 * g, r) & 0xffffffu,
                                          P.col3, P.col4);
                    ow[3 * g] = lanes_mod7(t[0] | (t[1] << 24));
                    ow[3 * g + 1] = lanes_mod7((t[1] >> 8) | (t[2] << 16));
                    ow[3 * g + 2] = lanes_mod7((t[2] >> 16) | (t[3] << 8));
                }
                return;
            }
        }
        const bool pk = packed();
        // this lane's private copies: packed L16 at tb, H at hb; dlog log at tb
        const uint32_t tb = tab + 4 * (threadIdx.x & 31u), hb = tb + 128 * kHOff;
        // dlog: lane l reads antilog copy l mod n
        constexpr uint32_t nc = kDlogCopies;
        const uint32_t al = tab + 128 * kP3 + 4 * (threadIdx.x % nc);
        const uint32_t zero4 = 4 * (2 * P.group - 1) * nc;
#pragma unroll
        for (int g = 0; g < R / 4; ++g) {
            uint32_t res[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t ya = record24(aw + 3 * g, r), yb = record24(bw + 3 * g, r);
                if (pk) {
                    res[r] = lh_product_lane<K>(P.rq.inv_p, ya & 0xffffffu, yb & 0xffffffu, tb, hb);
                } else {
                    res[r] = dlog_product_lane<kP>(ya, yb, tb, al, zero4);
                }
            }
            ow[3 * g] = res[0] | (res[1] << 24);
            ow[3 * g + 1] = (res[1] >> 8) | (res[2] << 16);
            ow[3 * g + 2] = (res[2] >> 16) | (res[3] << 8);
            if (pk) {  // L + H lanes, four records at a time
#pragma unroll
                for (int i = 0; i < 3; ++i) ow[3 * g + i] = bytes_below_2p_mod(ow[3 * g + i], K::kP);
            }
        }
    }

    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t* b, uint32_t (&ow)[R * OUT / 4],
                                          uint32_t tab, uint32_t&) const {
        if constexpr (kFast) {
            if (P.fast_off) {
                apply_fast(a, b, ow, tab);
                return;
            }
        }
        const K c{P.rq};
        uint32_t nlh = 1;
#pragma unroll
        for (int i = 0; i < K_; ++i) nlh *= P.lh_radix;
        const uint32_t lc = tab, hc = tab + 4 * nlh, lg = tab + 8 * nlh, al = tab + 8 * nlh + 4 * P.order;
        uint64_t rec[R];
        if constexpr (K::kSafe && K::kQbitsCt == 8) {
            // q = 2^8: a record of k coefficient bytes IS its DQT word, so
            // packing is a byte-run extract; taken when every byte is < p
            if (all_bytes_below<R * K_ / 4>(a, c.p()) && all_bytes_below<R * K_ / 4>(b, c.p())) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint32_t ra = record_int<K_>(a, r), rb = record_int<K_>(b, r);
                    uint32_t res;
                    if (packed()) {
                        res = lh_product<K_>(c, ra, rb, lc, hc);
                    } else {
                        res = dlog_product<K_>(c, coeff_index<K_>(c, ra), coeff_index<K_>(c, rb), lg, al, P.group);
                    }
                    rec[r] = res;
                }
                pack_records<R, OUT>(rec, ow);
                return;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t ca[K_], cb[K_];
            record_coeffs<K_>(c, P.rq.mod_magic, a, r, ca);
            record_coeffs<K_>(c, P.rq.mod_magic, b, r, cb);
            uint32_t res;
            if (packed()) {
                // paper Alg. 4 with one term: pack, fp64 product, REDQ digits,
                // low/high half tables (gfq.cpp:353-381); the tables give
                // coefficient vectors, so the halves add coefficient-wise
                uint32_t u[ND];
                redq_raw_digits<ND>(c, pack_word<K_>(c, P.qd, ca) * pack_word<K_>(c, P.qd, cb), u);
                uint32_t il = 0, ih = 0;
#pragma unroll
                for (int i = K_ - 1; i >= 0; --i) {
                    il = il * P.lh_radix + u[i];
                    ih = ih * P.lh_radix + u[K_ - 1 + i];
                }
                res = add_mod_bytes(lds_u32(lc + 4 * il), lds_u32(hc + 4 * ih), c.p(), K_);
            } else {
                // dlog representation: rep(a*b) = rep(a) + rep(b) mod p^k-1,
                // zero sentinel (gfq.cpp:260-264), then back to coefficients
                uint32_t ia = 0, ib = 0;
#pragma unroll
                for (int i = K_ - 1; i >= 0; --i) {
                    ia = ia * c.p() + ca[i];
                    ib = ib * c.p() + cb[i];
                }
                const uint32_t ra = lds_u32(lg + 4 * ia), rb = lds_u32(lg + 4 * ib);
                uint32_t rc = ra + rb;
                if (rc >= P.group) rc -= P.group;
                if (ra == P.group || rb == P.group) rc = P.group;
                res = lds_u32(al + 4 * rc);
            }
            rec[r] = res;
        }
        pack_records<R, OUT>(rec, ow);
    }
};

// ------------------------------------------------------------- the pipeline
// stream_tma_kernel: a CTA of 256 threads owns tiles of 256*R*RR records.
// Thread 0 keeps S input stages in flight (bulk copies completing on
// mbarriers) and bulk-stores each finished output tile from a double
// buffer; every thread processes RR runs of R consecutive records per tile.
// Tile size (RR) and depth (S) per op come from a sweep on B200
// (scripts/stream_variants.cu): for C2, 16 KB tiles x 3 stages at 2 CTAs/SM
// reach 98% of cudaMemcpy device-to-device bandwidth; a warp-specialised
// variant with per-warp output stores was slower.
// threads per CTA of the TMA pipeline: Op::THREADS when the op sets it
template <class Op, class = void>
struct op_threads : std::integral_constant<int, kThreads> {};
template <class Op>
struct op_threads<Op, std::void_t<decltype(Op::THREADS)>> : std::integral_constant<int, Op::THREADS> {};

// ops with kDirectStore store their output runs straight from registers
// (vector st.global, a warp's runs are contiguous) instead of staging the
// output tile for a bulk store: no output buffers in shared memory, so an op
// with large tables keeps one more input stage in flight
template <class Op, class = void>
struct op_direct_store : std::false_type {};
template <class Op>
struct op_direct_store<Op, std::enable_if_t<Op::kDirectStore>> : std::true_type {};

#ifndef QPK_DS_PRODUCER
#define QPK_DS_PRODUCER 1
#endif
// measured C3 REDQ/L-H 29.7 -> 28.4 us, dlog 27.0 -> 26.6; the same trigger
// in the bulk-store pipeline left C3 linear unchanged and cost C2 2%
#ifndef QPK_WS_TRIGGER
#define QPK_WS_TRIGGER 1
#endif


template <class Op>
struct Geometry {
    static constexpr int R = Op::R, RR = Op::RR, S = Op::S;
    static constexpr int THREADS = op_threads<Op>::value;
    static constexpr bool DS = op_direct_store<Op>::value;
    // direct-store ops with a producer warp: one extra warp keeps the input
    // stages in flight, released per consumer warp through "empty"
    // mbarriers, so the consumer warps never meet at a CTA barrier
    static constexpr bool WS = DS && QPK_DS_PRODUCER;
    static constexpr int BLOCK = THREADS + (WS ? 32 : 0);  // launched threads
    static constexpr int TILE = THREADS * R * RR;  // records per tile
    static constexpr uint32_t B0 = Op::IN0 * TILE, B1 = Op::IN1 * TILE, BO = Op::OUT * TILE;
    static constexpr int W0 = R * Op::IN0 / 4, W1 = R * Op::IN1 / 4, WO = R * Op::OUT / 4;
    static_assert((R * Op::IN0) % 4 == 0 && (R * Op::IN1) % 4 == 0 && (R * Op::OUT) % 4 == 0, "u32 runs");
    static_assert(B0 % 16 == 0 && B1 % 16 == 0 && BO % 16 == 0, "bulk copies move multiples of 16 bytes");
    // stage buffers | output double buffer | S (2S with WS) mbarriers | (16-aligned) tables
    static constexpr size_t tab_off =
        (size_t(S) * (B0 + B1) + (DS ? 0 : 2 * size_t(BO)) + (WS ? 2 : 1) * S * 8 + 15) / 16 * 16;
    static constexpr size_t smem_pipe = tab_off;
};

// `N` u32 words from shared memory with the widest vector that divides N
template <int N>
__device__ __forceinline__ void lds_run(const uint8_t* base, uint32_t (&w)[N > 0 ? N : 1]) {
    if constexpr (N == 0) {
        w[0] = 0;
    } else if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const uint4 v = reinterpret_cast<const uint4*>(base)[i];
            w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = reinterpret_cast<const uint32_t*>(base)[i];
    }
}

__device__ __forceinline__ void report(uint32_t err, uint32_t* status) {
    err = __reduce_or_sync(0xffffffffu, err);
    if (err && (threadIdx.x & 31) == 0 && status) atomicOr(status, err);
}

// ASYNC: 16-byte cp.async copies (the TMA kernel, where a CTA streams for
// tens of microseconds); the one-pass direct/tail kernels keep the plain
// loop (measured: cp.async cost C1's hot launch 6.31 -> 6.65 us)
// WAIT = false leaves the cp.async copies in flight (the caller waits)
template <class Op, bool ASYNC = true, bool WAIT = true>
__device__ __forceinline__ void stage_tables(const Op& op, uint32_t* dst) {
    // 16-byte cp.async copies, every one in flight at once (a per-thread
    // load/store loop serialises one L2 round trip per 256 words: measured
    // C3 packed 29.1 -> 28.1 us), then the unaligned remainder
    const uint32_t nt = op.tables_words();
    const uint32_t* src = op.tables_src();
    uint32_t head = 0;
    if (ASYNC && ((reinterpret_cast<uintptr_t>(src) | smem_addr(dst)) & 15u) == 0) {
        const uint32_t n4 = nt / 4;
        for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + 4 * i)), "l"(src + 4 * i)
                         : "memory");
        head = 4 * n4;
    }
    for (uint32_t i = head + threadIdx.x; i < nt; i += blockDim.x) dst[i] = src[i];
    if (ASYNC && WAIT) asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void stg_run(uint8_t* base, const uint32_t (&w)[N]) {
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i)
            reinterpret_cast<uint4*>(base)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
    } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) reinterpret_cast<uint2*>(base)[i] = make_uint2(w[2 * i], w[2 * i + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) reinterpret_cast<uint32_t*>(base)[i] = w[i];
    }
}

// The same 32 runs of one warp (N words each, N not a multiple of 4: a
// thread's own stores are 4 bytes wide and N * 4 bytes apart across lanes,
// 7+ cache lines per instruction) written as 16-byte chunks of the warp's
// contiguous output range, transposed through a per-warp shared buffer
// (stride N words: conflict-free for odd N).  `warp_out` is 16-byte aligned.
template <int N>
__device__ __forceinline__ void stg_run_warp(uint8_t* warp_out, uint32_t* wbuf, const uint32_t (&w)[N], int lane) {
#pragma unroll
    for (int i = 0; i < N; ++i) wbuf[lane * N + i] = w[i];
    __syncwarp();
    constexpr int V = 32 * N / 4;
#pragma unroll
    for (int j = 0; j < (V + 31) / 32; ++j) {
        const int ch = j * 32 + lane;
        if (ch < V) reinterpret_cast<uint4*>(warp_out)[ch] = reinterpret_cast<const uint4*>(wbuf)[ch];
    }
    __syncwarp();
}

template <class Op, class = void>
struct has_custom_stage : std::false_type {};
template <class Op>
struct has_custom_stage<Op, std::enable_if_t<Op::kCustomStage>> : std::true_type {};

// an op's tables: its own staging (lane-private copies built from a compact
// table) or the plain copy
template <class Op, bool ASYNC = true, bool WAIT = true>
__device__ __forceinline__ void stage_op_tables(const Op& op, uint32_t* dst) {
    if constexpr (has_custom_stage<Op>::value) {
        if (op.custom_stage()) {
            op.stage_custom(dst);
            return;
        }
    }
    stage_tables<Op, ASYNC, WAIT>(op, dst);
}

template <class Op>
__global__ void __launch_bounds__(Geometry<Op>::BLOCK) stream_tma_kernel(const Op op, const uint8_t* __restrict__ in0,
                                                              const uint8_t* __restrict__ in1,
                                                              uint8_t* __restrict__ out, uint64_t n_tiles,
                                                              uint32_t* status) {
    using G = Geometry<Op>;
    constexpr int S = G::S;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* s_in = smem;
    uint8_t* s_out = smem + size_t(S) * (G::B0 + G::B1);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_out + (G::DS ? 0 : 2 * size_t(G::BO)));
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(smem + G::tab_off);  // 16-byte aligned
    const uint32_t tab = smem_addr(s_tab);
    const int tid = threadIdx.x;

    uint64_t policy = 0;
    auto issue = [&](int s, uint64_t tile) {
        uint8_t* dst = s_in + size_t(s) * (G::B0 + G::B1);
        mbar_expect_tx(&bars[s], G::B0 + G::B1);
        bulk_g2s_stream(dst, in0 + tile * G::B0, G::B0, &bars[s], policy);
        if constexpr (G::B1 > 0) bulk_g2s_stream(dst + G::B0, in1 + tile * G::B1, G::B1, &bars[s], policy);
    };
    // barrier setup (and the staging of large tables) run before pdl_wait,
    // overlapping the previous kernel's tail: the tables are plan constants,
    // uploaded when the plan or field was built, never written by a preceding
    // launch; thread 0 puts the first S tiles in flight while the table
    // copies complete
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        if constexpr (G::WS)
            for (int s = 0; s < S; ++s) mbar_init(&bars[S + s], G::THREADS / 32);
        fence_mbar_init();
        policy = policy_evict_first();
    }
#ifndef QPK_EARLY_STAGE_WORDS
#define QPK_EARLY_STAGE_WORDS 4096
#endif
    // large tables only (C3 dlog copies, 38 KB: 32.7 -> 32.0 us); C2's
    // 2.5 KB table measured 0.4% slower staged early (0.1584 vs 0.1590 ms)
    const bool early = op.tables_words() >= QPK_EARLY_STAGE_WORDS;
    if (early) stage_op_tables<Op, true, false>(op, s_tab);
    pdl_wait();
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            const uint64_t t = blockIdx.x + uint64_t(s) * gridDim.x;
            if (t < n_tiles) issue(s, t);
        }
    }
    if (!early) stage_op_tables<Op, true, false>(op, s_tab);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    uint32_t err = 0;
    uint32_t it = 0;
    if constexpr (G::WS) {
        const int warp = tid >> 5, lane = tid & 31;
        if (warp == G::THREADS / 32) {
            // producer: refill stage s once every consumer warp released it
            if (lane == 0) {
                policy = policy_evict_first();
                for (uint64_t tile = blockIdx.x + uint64_t(S) * gridDim.x; tile < n_tiles; tile += gridDim.x, ++it) {
                    const int s = it % S;
                    mbar_wait(&bars[S + s], (it / S) & 1);
                    issue(s, tile);
                }
            }
            return;
        }
        for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int s = it % S;
            const uint8_t* src = s_in + size_t(s) * (G::B0 + G::B1);
#if QPK_WS_TRIGGER
            // the CTA's last tile: the next kernel may launch (its CTAs land
            // on the SMs this grid leaves and stage their tables during its
            // tail; their data accesses still follow pdl_wait)
            if (tile + gridDim.x >= n_tiles) pdl_trigger();
#endif
            mbar_wait(&bars[s], (it / S) & 1);
#pragma unroll
            for (int rr = 0; rr < G::RR; ++rr) {
                const int run = rr * G::THREADS + tid;
                uint32_t a[G::W0 > 0 ? G::W0 : 1], b[G::W1 > 0 ? G::W1 : 1];
                lds_run<G::W0>(src + run * (G::R * Op::IN0), a);
                lds_run<G::W1>(src + G::B0 + run * (G::R * Op::IN1), b);
                uint32_t ow[G::WO];
                op.apply(a, b, ow, tab, err);
                stg_run<G::WO>(out + tile * G::BO + size_t(run) * (G::R * Op::OUT), ow);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[S + s]);
        }
        report(err, status);
    } else {
        for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int s = it % S;
            const uint8_t* src = s_in + size_t(s) * (G::B0 + G::B1);
            if constexpr (G::DS) {
                // every thread waits on the stage's mbarrier (the TMA writes are
                // visible to it); one barrier per tile frees the stage
                mbar_wait(&bars[s], (it / S) & 1);
#pragma unroll
                for (int rr = 0; rr < G::RR; ++rr) {
                    const int run = rr * G::THREADS + tid;
                    uint32_t a[G::W0 > 0 ? G::W0 : 1], b[G::W1 > 0 ? G::W1 : 1];
                    lds_run<G::W0>(src + run * (G::R * Op::IN0), a);
                    lds_run<G::W1>(src + G::B0 + run * (G::R * Op::IN1), b);
                    uint32_t ow[G::WO];
                    op.apply(a, b, ow, tab, err);
                    stg_run<G::WO>(out + tile * G::BO + size_t(run) * (G::R * Op::OUT), ow);
                }
                __syncthreads();
                if (tid == 0) {
                    const uint64_t next = tile + uint64_t(S) * gridDim.x;
                    if (next < n_tiles) issue(s, next);
                }
                continue;
            }
            const int os = it & 1;
            if (tid == 0) bulk_wait_read<1>();  // output buffer `os` (two tiles ago) drained
            mbar_wait(&bars[s], (it / S) & 1);
            __syncthreads();

            uint32_t* obuf = reinterpret_cast<uint32_t*>(s_out + size_t(os) * G::BO);
#pragma unroll
            for (int rr = 0; rr < G::RR; ++rr) {
                const int run = rr * G::THREADS + tid;  // R consecutive records
                uint32_t a[G::W0 > 0 ? G::W0 : 1], b[G::W1 > 0 ? G::W1 : 1];
                lds_run<G::W0>(src + run * (G::R * Op::IN0), a);
                lds_run<G::W1>(src + G::B0 + run * (G::R * Op::IN1), b);
                uint32_t ow[G::WO];
                op.apply(a, b, ow, tab, err);
#pragma unroll
                for (int i = 0; i < G::WO; ++i) obuf[run * G::WO + i] = ow[i];
            }
            fence_proxy_async_smem();
            __syncthreads();

            if (tid == 0) {
                bulk_s2g(out + tile * G::BO, s_out + size_t(os) * G::BO, G::BO);
                bulk_commit();
                const uint64_t next = tile + uint64_t(S) * gridDim.x;
                if (next < n_tiles) issue(s, next);
            }
        }
        if (tid == 0) bulk_wait_all<0>();
        report(err, status);
    }
}

// Small batches (one wave of CTAs): every thread loads its runs straight
// from global memory with the widest aligned vectors and stores its output
// run -- no pipeline prologue, every load in flight at once.  Used below
// kDirectMax records (measured: C1's 2^20 pairs, a latency-bound 15.7 MB).
template <int N>
__device__ __forceinline__ void ldg_run(const uint8_t* base, uint32_t (&w)[N > 0 ? N : 1]) {
    if constexpr (N == 0) {
        w[0] = 0;
    } else if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + i);
            w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
        }
    } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(base) + i);
            w[2 * i] = v.x, w[2 * i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = __ldg(reinterpret_cast<const uint32_t*>(base) + i);
    }
}

template <class Op, class = void>
struct op_direct_min_blocks : std::integral_constant<int, 1> {};
template <class Op>
struct op_direct_min_blocks<Op, std::enable_if_t<(Op::kDirectMinBlocks > 1)>>
    : std::integral_constant<int, Op::kDirectMinBlocks> {};

template <class Op>
__global__ void __launch_bounds__(kThreads, op_direct_min_blocks<Op>::value) stream_direct_kernel(const Op op, const uint8_t* __restrict__ in0,
                                                                 const uint8_t* __restrict__ in1,
                                                                 uint8_t* __restrict__ out, uint64_t n_runs,
                                                                 uint32_t* status) {
    using G = Geometry<Op>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(smem);
    // first loads before the table staging, so both overlap
    pdl_wait();
    uint64_t run = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t a[G::W0 > 0 ? G::W0 : 1], b[G::W1 > 0 ? G::W1 : 1];
    if (run < n_runs) {
        ldg_run<G::W0>(in0 + run * (G::R * Op::IN0), a);
        ldg_run<G::W1>(in1 + run * (G::R * Op::IN1), b);
    }
    if (op.tables_words() > 0) {  // CTA-uniform
        stage_op_tables<Op, false>(op, s_tab);
        __syncthreads();
    }
    const uint32_t tab = smem_addr(s_tab);
    uint32_t err = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    constexpr bool kWarpStore = G::WO % 4 != 0;
    __shared__ __align__(16) uint32_t s_wout[kWarpStore ? kThreads * G::WO : 4];
    const int lane = threadIdx.x & 31;
    const bool out_aligned = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (; run < n_runs; run += stride) {
        uint32_t ow[G::WO];
        op.apply(a, b, ow, tab, err);
        if (kWarpStore && out_aligned && run - lane + 31 < n_runs)  // warp-uniform: all 32 runs exist
            stg_run_warp<G::WO>(out + (run - lane) * (G::R * Op::OUT), s_wout + (threadIdx.x - lane) * G::WO, ow, lane);
        else
            stg_run<G::WO>(out + run * (G::R * Op::OUT), ow);
        if (run + stride < n_runs) {
            ldg_run<G::W0>(in0 + (run + stride) * (G::R * Op::IN0), a);
            ldg_run<G::W1>(in1 + (run + stride) * (G::R * Op::IN1), b);
        }
    }
    report(err, status);
}

// Records [first, n) with byte-granular global loads (tails, unaligned buffers).
template <class Op>
__global__ void __launch_bounds__(kThreads) stream_tail_kernel(const Op op, const uint8_t* __restrict__ in0,
                                                               const uint8_t* __restrict__ in1,
                                                               uint8_t* __restrict__ out, uint64_t first,
                                                               uint64_t n, uint32_t* status) {
    using G = Geometry<Op>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(smem);
    stage_op_tables<Op, false>(op, s_tab);
    pdl_wait();
    __syncthreads();
    const uint32_t tab = smem_addr(s_tab);
    uint32_t err = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G::R;
    for (uint64_t base = first + (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * G::R; base < n;
         base += stride) {
        const int cnt = n - base < uint64_t(G::R) ? static_cast<int>(n - base) : G::R;
        uint32_t a[G::W0 > 0 ? G::W0 : 1] = {}, b[G::W1 > 0 ? G::W1 : 1] = {};
        for (int i = 0; i < cnt * Op::IN0; ++i) a[i >> 2] |= uint32_t(in0[base * Op::IN0 + i]) << (8 * (i & 3));
        for (int i = 0; i < cnt * Op::IN1; ++i) b[i >> 2] |= uint32_t(in1[base * Op::IN1 + i]) << (8 * (i & 3));
        uint32_t ow[G::WO];
        // zero padding is a valid input for every op, so it never raises
        op.apply(a, b, ow, tab, err);
        for (int i = 0; i < cnt * Op::OUT; ++i) out[base * Op::OUT + i] = static_cast<uint8_t>(ow[i >> 2] >> (8 * (i & 3)));
    }
    report(err, status);
}

#ifndef QPK_DIRECT_MAX
#define QPK_DIRECT_MAX (1u << 21)
#endif
constexpr uint64_t kDirectMax = QPK_DIRECT_MAX;  // records: below this the direct kernel runs

template <class Op>
cudaError_t run_tail(const Op& op, const uint8_t* in0, const uint8_t* in1, uint8_t* out, uint64_t first, uint64_t n,
                     uint32_t* status, cudaStream_t s) {
    using G = Geometry<Op>;
    const size_t tab_bytes = size_t(op.tables_words()) * 4;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(stream_tail_kernel<Op>), tab_bytes);
        e != cudaSuccess)
        return e;
    const uint64_t groups = (n - first + G::R - 1) / G::R;
    const uint64_t grid = std::min<uint64_t>((groups + kThreads - 1) / kThreads, uint64_t(num_sms()) * 8);
    return launch_pdl(stream_tail_kernel<Op>, dim3(static_cast<unsigned>(grid)), dim3(kThreads), tab_bytes, s, op, in0,
                      in1, out, first, n, status);
}

template <class Op>
cudaError_t run_stream(const Op& op, const uint8_t* in0, const uint8_t* in1, uint8_t* out, uint64_t n,
                       uint32_t* status, cudaStream_t s) {
    using G = Geometry<Op>;
    if (n == 0) return cudaSuccess;
    const size_t tab_bytes = size_t(op.tables_words()) * 4;
    const bool aligned = (reinterpret_cast<uintptr_t>(in0) % 16 == 0) &&
                         (G::B1 == 0 || reinterpret_cast<uintptr_t>(in1) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    const int sms = num_sms();
    // small batches: the direct kernel over whole runs, then the tail
    if (aligned && n < kDirectMax && n >= uint64_t(G::R)) {
        const uint64_t n_runs = n / G::R;
        // (the direct kernel's static buffer of the warp-transposed stores counts against the 48 KB default)
        constexpr size_t kStatic = G::WO % 4 != 0 ? size_t(kThreads) * G::WO * 4 : 16;
        if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(stream_direct_kernel<Op>), tab_bytes, kStatic);
            e != cudaSuccess)
            return e;
        const uint64_t grid = std::min<uint64_t>((n_runs + kThreads - 1) / kThreads, uint64_t(sms) * 16);
        if (cudaError_t e = launch_pdl(stream_direct_kernel<Op>, dim3(static_cast<unsigned>(grid)), dim3(kThreads),
                                       tab_bytes, s, op, in0, in1, out, n_runs, status);
            e != cudaSuccess)
            return e;
        const uint64_t first = n_runs * G::R;
        if (first == n) return cudaSuccess;
        return run_tail(op, in0, in1, out, first, n, status, s);
    }
    const uint64_t n_tiles = aligned ? n / G::TILE : 0;
    if (n_tiles > 0) {
        const size_t smem = G::smem_pipe + tab_bytes;
        if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(stream_tma_kernel<Op>), smem);
            e != cudaSuccess)
            return e;
        // occupancy per instantiation, device and table size (a per-call
        // query costs microseconds of host time, comparable to a small launch)
        static thread_local size_t occ_smem = 0;
        static thread_local int occ_dev = -1;
        static thread_local int occ_per_sm = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (occ_smem != smem || occ_dev != dev) {
            int v = 0;
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, stream_tma_kernel<Op>, G::BLOCK, smem);
            if (e != cudaSuccess) return e;
            occ_smem = smem;
            occ_dev = dev;
            occ_per_sm = std::max(v, 1);
        }
        const uint64_t grid = std::min<uint64_t>(n_tiles, uint64_t(sms) * occ_per_sm);
        const cudaError_t e = launch_pdl(stream_tma_kernel<Op>, dim3(static_cast<unsigned>(grid)), dim3(G::BLOCK),
                                         smem, s, op, in0, in1, out, n_tiles, status);
        if (e != cudaSuccess) return e;
    }
    const uint64_t first = n_tiles * G::TILE;
    if (first < n) return run_tail(op, in0, in1, out, first, n, status, s);
    return cudaSuccess;
}

// compile-time fast paths for the benchmark fields (BASELINE configs):
//   C2  REDQ   p=5, q=2^7,  7 digits, window 4
//   C1  polymul p=3, q=2^5,  k=4, window 4
//   C3  GF(7^3) p=7, q=2^8,  k=3
// safe = every word of the plan stays <= min(r_max, 2^52)
inline bool plan_is_safe(const RedqParams& P) {
    return P.qbits && P.limit <= P.r_max + 1.0 && P.limit <= kTwo52;
}

template <int ND, bool POW2>
cudaError_t redq_dispatch_pow2(const RedqParams& P, const double* w, uint64_t n, uint8_t* out, uint32_t* st,
                            cudaStream_t s) {
    const auto* in = reinterpret_cast<const uint8_t*>(w);
    if constexpr (ND == 7 && POW2) {
        if (P.p == 5 && P.qbits == 7 && P.window == 4 && P.radix == 5 && plan_is_safe(P))
            return run_stream(RedqOp<7, 4, CtConst<5, 7>>{P}, in, nullptr, out, n, st, s);
    }
    switch (P.window) {
        case 2: return run_stream(RedqOp<ND, 2, RtConst<POW2>>{P}, in, nullptr, out, n, st, s);
        case 3: return run_stream(RedqOp<ND, 3, RtConst<POW2>>{P}, in, nullptr, out, n, st, s);
        case 4: return run_stream(RedqOp<ND, 4, RtConst<POW2>>{P}, in, nullptr, out, n, st, s);
        default: return run_stream(RedqOp<ND, 0, RtConst<POW2>>{P}, in, nullptr, out, n, st, s);
    }
}

template <int ND>
cudaError_t redq_dispatch_q(const RedqParams& P, const double* w, uint64_t n, uint8_t* out, uint32_t* st,
                            cudaStream_t s) {
    return P.qbits ? redq_dispatch_pow2<ND, true>(P, w, n, out, st, s)
                   : redq_dispatch_pow2<ND, false>(P, w, n, out, st, s);
}

template <int K_, bool POW2>
cudaError_t polymul_dispatch_w(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                               uint32_t* st, cudaStream_t s) {
    if constexpr (K_ == 4 && POW2) {
        if (P.rq.p == 3 && P.rq.qbits == 5 && P.rq.window == 4 && P.rq.radix == 3 && plan_is_safe(P.rq))
            return run_stream(PolymulOp<4, 4, CtConst<3, 5>>{P}, a, b, out, n, st, s);
    }
    switch (P.rq.window) {
        case 2: return run_stream(PolymulOp<K_, 2, RtConst<POW2>>{P}, a, b, out, n, st, s);
        case 3: return run_stream(PolymulOp<K_, 3, RtConst<POW2>>{P}, a, b, out, n, st, s);
        case 4: return run_stream(PolymulOp<K_, 4, RtConst<POW2>>{P}, a, b, out, n, st, s);
        default: return run_stream(PolymulOp<K_, 0, RtConst<POW2>>{P}, a, b, out, n, st, s);
    }
}

template <int K_>
cudaError_t polymul_dispatch_q(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                               uint8_t* out, uint32_t* st, cudaStream_t s) {
    return P.rq.qbits ? polymul_dispatch_w<K_, true>(P, a, b, n, out, st, s)
                      : polymul_dispatch_w<K_, false>(P, a, b, n, out, st, s);
}

template <int K_>
cudaError_t gfq_elem_dispatch(const GfqElemParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                              uint8_t* out, cudaStream_t s) {
    if constexpr (K_ == 3) {
        if (P.p == 7 && P.rq.qbits == 8 && plan_is_safe(P.rq)) switch (P.mode) {
                case kGfqDlog: return run_stream(GfqElemOp<3, CtConst<7, 8>, kGfqDlog>{P}, a, b, out, n, nullptr, s);
                case kGfqLinear:
                    return run_stream(GfqElemOp<3, CtConst<7, 8>, kGfqLinear>{P}, a, b, out, n, nullptr, s);
                default: return run_stream(GfqElemOp<3, CtConst<7, 8>, kGfqPacked>{P}, a, b, out, n, nullptr, s);
            }
    }
    return P.rq.qbits ? run_stream(GfqElemOp<K_, RtConst<true>>{P}, a, b, out, n, nullptr, s)
                      : run_stream(GfqElemOp<K_, RtConst<false>>{P}, a, b, out, n, nullptr, s);
}

}  // namespace

}  // namespace qpk
