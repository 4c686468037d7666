// Exact floor division by a premultiplied reciprocal (paper Lemma 1;
// reference: proj/include/qpack/fpdiv.hpp:19-37).
//
// inv_up >= 1/p is 1/p rounded upward; floor(r*inv_up rounded up) equals
// floor(r/p) for every r <= r_max, r_max being the largest r with
// r*(2e+e^2) < 1 at e = 3*2^-53.  The GPU kernels use the same constants.
#pragma once

#include "qpack/common.hpp"

namespace qpack {

struct ReciprocalDivisor {
    u64 p = 0;
    double inv_up = 0.0;
    double epsilon = 0.0;  // 2^-53
    u64 r_max = 0;

    static ReciprocalDivisor make(u64 p);
};

u64 floor_div_rn(u64 r, u64 p);
u64 floor_div_premul(u64 r, const ReciprocalDivisor& d);
u64 premul_floor_bound(double epsilon);

}  // namespace qpack
