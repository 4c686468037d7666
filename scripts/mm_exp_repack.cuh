// Development only (scripts/mm_exp.sh): timing-only re-pack variants of the K4
// fast path, compiled in with -DQPK_MM_EXP=n.  They measure what one more
// integer instruction per accumulator per re-pack costs the DMMA stream
// ("dispatch-slot cost"); the results are wrong on purpose
// (the epilogue re-canonicalises so table indices stay in range).
#pragma once
template <int ND, uint32_t B>
__device__ __forceinline__ double mm_exp_repack(double acc) {
#if QPK_MM_EXP == 1
    return acc;  // no re-pack at all
#elif QPK_MM_EXP == 2
    return __longlong_as_double(static_cast<long long>(dbits(acc) & 0xFFFFFFFFFFFFFFFEull));  // one LOP3
#elif QPK_MM_EXP == 3
    const uint64_t b = dbits(acc);  // one LOP3 per half
    return __longlong_as_double(static_cast<long long>(b & 0xFFFFFFFEFFFFFFFEull));
#elif QPK_MM_EXP == 4  // 8 ALU-pipe instructions (LOP3 / IADD3 alternating, 4 per half)
    uint64_t b = dbits(acc);
    uint32_t lo = uint32_t(b), hi = uint32_t(b >> 32);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        lo = (lo ^ 0x1234567u) + 0x89abcdu;
        hi = (hi ^ 0x7654321u) + 0xfedcbau;
    }
    return __longlong_as_double(static_cast<long long>((uint64_t(hi) << 32) | lo));
#elif QPK_MM_EXP == 5  // 8 IMAD (FMA pipe), not affine-foldable
    uint64_t b = dbits(acc);
    uint32_t lo = uint32_t(b), hi = uint32_t(b >> 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        lo = lo * lo + 0x89abcdu;
        hi = hi * hi + 0xfedcbau;
    }
    return __longlong_as_double(static_cast<long long>((uint64_t(hi) << 32) | lo));
#elif QPK_MM_EXP == 6  // 8 FFMA (fp32 pipe)
    uint64_t b = dbits(acc);
    float lo = __uint_as_float(uint32_t(b)), hi = __uint_as_float(uint32_t(b >> 32));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        lo = fmaf(lo, lo, 1.5f);
        hi = fmaf(hi, hi, 2.5f);
    }
    return __longlong_as_double(static_cast<long long>((uint64_t(__float_as_uint(hi)) << 32) | __float_as_uint(lo)));
#elif QPK_MM_EXP == 7  // 8 SHF (funnel shifts, ALU pipe)
    uint64_t b = dbits(acc);
    uint32_t lo = uint32_t(b), hi = uint32_t(b >> 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        lo = __funnelshift_l(hi, lo, 3);
        hi = __funnelshift_l(lo, hi, 5);
    }
    return __longlong_as_double(static_cast<long long>((uint64_t(hi) << 32) | lo));
#elif QPK_MM_EXP == 8  // 8 IMAD.HI
    uint64_t b = dbits(acc);
    uint32_t lo = uint32_t(b), hi = uint32_t(b >> 32);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        lo = __umulhi(lo, lo) + 0x40000000u;
        hi = __umulhi(hi, hi) + 0x40000000u;
    }
    return __longlong_as_double(static_cast<long long>((uint64_t(hi) << 32) | lo));
#else
    return redq_repack_swar3<ND, B>(acc);
#endif
}
