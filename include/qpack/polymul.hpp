// FQT chunked polynomial product (reference: proj/include/qpack/polymul.hpp:18-47;
// paper §5).  Batched single-chunk products on the GPU: qpack::gpu::polymul_batch.
#pragma once

#include <vector>

#include "qpack/counters.hpp"
#include "qpack/dqt.hpp"
#include "qpack/params.hpp"
#include "qpack/poly.hpp"
#include "qpack/redq.hpp"

namespace qpack {

// chunk i holds the coefficients of X^(i(d+1)) .. X^(i(d+1)+d)
struct FqtPoly {
    std::vector<Packed> chunks;
    u32 d = 0;
    QadicParams params;
};

FqtPoly fqt_encode(const DensePoly& poly, u32 d, const QadicParams& params);
DensePoly fqt_decode(const FqtPoly& enc, std::size_t coeff_len);
u64 packed_degree(u64 n_degree, u32 d);                 // ceil((N+1)/(d+1)) - 1
RedqPlan fqt_reduction_plan(const QadicParams& params, u32 d);

DensePoly fqt_mul(const DensePoly& P, const DensePoly& Q, u32 d, const QadicParams& params,
                  CostReport* cost = nullptr);
DensePoly fqt_mul(const DensePoly& P, const DensePoly& Q, u32 d, const QadicParams& params,
                  const RedqPlan& plan, CostReport* cost = nullptr);

}  // namespace qpack
