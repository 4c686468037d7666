// K4 instantiation for one record width, selected with -DQPK_INST=k (1..4);
// build.py compiles this file once per k so the unrolled kernels build in
// parallel.
#include "gfq_matmul.cuh"

#ifndef QPK_INST
#error "compile with -DQPK_INST=<1..4>"
#endif

#define QPK_CAT2(a, b) a##b
#define QPK_CAT(a, b) QPK_CAT2(a, b)

namespace qpk {

cudaError_t QPK_CAT(matmul_launch_k, QPK_INST)(const GfqMatmulParams& P, const double* at, const double* b,
                                               uint64_t m, uint64_t n, uint64_t K_pad, uint64_t m_pad,
                                               uint64_t n_pad, uint8_t* oc, uint32_t* orp, cudaStream_t s) {
    return P.rq.qbits ? run_matmul<QPK_INST, true>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s)
                      : run_matmul<QPK_INST, false>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s);
}

}  // namespace qpk
