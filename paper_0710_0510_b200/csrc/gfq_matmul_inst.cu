// K4 instantiations for one record width k and one policy variant, selected
// with -DQPK_INST=k (1..4) and -DQPK_VARIANT=v (0 runtime-parameter kernels,
// 1 compile-time fast paths); build.py compiles this file once per (k, v)
// so the unrolled kernels build in parallel.
#include "gfq_matmul.cuh"

#if !defined(QPK_INST) || !defined(QPK_VARIANT)
#error "compile with -DQPK_INST=<1..4> -DQPK_VARIANT=<0|1>"
#endif

#define QPK_CAT2(a, b, c, d) a##b##c##d
#define QPK_CAT(a, b, c, d) QPK_CAT2(a, b, c, d)

namespace qpk {

cudaError_t QPK_CAT(matmul_launch_k, QPK_INST, _v, QPK_VARIANT)(const GfqMatmulParams& P, const double* at,
                                                                 const double* b, uint64_t m, uint64_t n,
                                                                 uint64_t K_pad, uint64_t m_pad, uint64_t n_pad,
                                                                 uint8_t* oc, uint32_t* orp, cudaStream_t s) {
    return run_matmul<QPK_INST, QPK_VARIANT>(P, at, b, m, n, K_pad, m_pad, n_pad, oc, orp, s);
}

}  // namespace qpk
