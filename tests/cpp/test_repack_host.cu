// Host check of the K4 re-packs (paper_0710_0510_b200/csrc/gfq_matmul.cuh):
// the canonical lane-fold re-pack of C5 (p = 3, q = 2^10, five digits) must
// return, for every word whose digits are all below q, the word whose digit
// i is (digit i) mod 3 -- what redq + assemble give (reference
// redq.cpp:178-182) -- with the 2^52 bias of the accumulator in place.
// Every digit value in every lane (other lanes zero and all-ones) and
// 2 * 10^7 random 50-bit words.  Built with nvcc, runs on the host.
#include <cstdint>
#include <cstdio>

#include "gfq_matmul.cuh"

int main() {
    using namespace qpk;
    unsigned long long bad = 0, n = 0;
    auto check = [&](uint64_t r) {
        uint64_t want = 0;
        for (int i = 0; i < 5; ++i) want |= (((r >> (10 * i)) & 1023) % 3) << (10 * i);
        const uint64_t got = repack_canon3_bits(r | kBiasBits);
        bad += got != (want | kBiasBits);
        ++n;
    };
    const uint64_t all = (uint64_t(1) << 50) - 1;
    for (int lane = 0; lane < 5; ++lane)
        for (uint64_t c = 0; c < 1024; ++c) {
            check(c << (10 * lane));
            check((c << (10 * lane)) | (all & ~(uint64_t(1023) << (10 * lane))));
        }
    uint64_t x = 0x9e3779b97f4a7c15ull;
    for (long i = 0; i < 20000000; ++i) {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;  // xorshift64
        check(x & all);
    }
    std::printf("%llu words, %llu mismatches\n", n, bad);
    return bad != 0;
}
