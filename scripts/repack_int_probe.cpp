// Host check of the integer-only REDQ re-pack (gfq_matmul.cuh div3_u64 +
// redq_repack_swar3): 2e8 random 50-bit words and q-adic words with 10-bit
// digits against floor(r/3) and the digit-wise mod 3.  g++ -O2 this; run.
#include <cstdint>
#include <cstdio>
#include <random>
// host copy of the device function (same arithmetic)
static inline uint32_t umulhi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
template <int ND, uint32_t B> constexpr uint64_t lane_ones() { uint64_t m = 0; for (int i = 0; i < ND; ++i) m |= uint64_t(1) << (B * i); return m; }
// floor(r / 3) for r < 2^50 from 32-bit halves
static inline uint64_t div3_u50(uint64_t r) {
    const uint32_t rh = (uint32_t)(r >> 32), rl = (uint32_t)r;
    const uint32_t qh = umulhi(rh, 0xAAAAAAABu) >> 1, mh = rh - 3 * qh;
    const uint32_t ql = umulhi(rl, 0xAAAAAAABu) >> 1, rr = rl - 3 * ql;
    const uint32_t lo = mh * 0x55555555u + ql + ((mh + rr + 1) >> 2);
    return ((uint64_t)qh << 32) | lo;
}
template <int ND, uint32_t B> static inline uint64_t repack(uint64_t rb) {
    constexpr uint64_t M1 = lane_ones<ND, B>(), M3 = 3 * M1;
    const uint64_t ob = div3_u50(rb);
    const uint64_t u = ((rb & M3) + (ob & M3)) & M3;
    const uint64_t v = u + 8 * M1 - (u >> B);
    const uint64_t g = (v >> 3) & M1;
    return v - 5 * M1 - 3 * g;
}
int main() {
    std::mt19937_64 g(1);
    uint64_t bad = 0, n = 0;
    for (uint64_t it = 0; it < 200000000ull; ++it) {
        uint64_t r;
        if (it % 2) r = g() & ((uint64_t(1) << 50) - 1);
        else { r = 0; for (int i = 4; i >= 0; --i) r = (r << 10) | (g() % 1024); }
        if (div3_u50(r) != r / 3) { if (bad++ < 5) printf("div3 bad %llu\n", (unsigned long long)r); }
        uint64_t want = 0; for (int i = 4; i >= 0; --i) want = (want << 10) | (((r >> (10 * i)) & 1023) % 3);
        if (repack<5, 10>(r) != want) { if (bad++ < 5) printf("repack bad %llu\n", (unsigned long long)r); }
        ++n;
    }
    // edge values
    for (uint64_t r : {0ull, 1ull, 2ull, 3ull, (1ull << 32) - 1, 1ull << 32, (1ull << 50) - 1, 0x3ffffffffffffull})
        if (div3_u50(r) != r / 3) printf("edge bad %llu\n", (unsigned long long)r), ++bad;
    printf("checked %llu, bad %llu\n", (unsigned long long)n, (unsigned long long)bad);
}
