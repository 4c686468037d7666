// SplitMix64 with modulo reduction, pinned so seeded fixtures agree across
// implementations (reference: proj/include/qpack/rng.hpp:13-31).  The n-th
// call returns mix(seed + n * 0x9e3779b97f4a7c15), which is what lets the GPU
// generate the same streams in parallel (qpk_gen_* in qpack_b200.h).
#pragma once

#include "qpack/common.hpp"

namespace qpack {

class SplitMix64 {
  public:
    explicit SplitMix64(u64 seed) : s_(seed) {}

    u64 next() {
        s_ += 0x9e3779b97f4a7c15ULL;
        u64 z = s_;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }

    // value in [0, n) by plain modulo; n must be nonzero
    u64 below(u64 n) { return next() % n; }

    u128 next_u128() {
        u128 hi = next();
        return (hi << 64) | next();
    }

  private:
    u64 s_;
};

}  // namespace qpack
