// One slice of the streaming-kernel instantiations, selected with
// -DQPK_INST=N (1..8): REDQ with N digits per word and, for N <= 4, the
// k = N polymul and GF(p^k) elementwise kernels.  build.py compiles this file
// once per N so the expensive template instantiations build in parallel.
#include "stream_inst.hpp"
#include "stream_kernels.cuh"

#ifndef QPK_INST
#error "compile with -DQPK_INST=<1..8>"
#endif

#define QPK_CAT2(a, b) a##b
#define QPK_CAT(a, b) QPK_CAT2(a, b)

namespace qpk {

cudaError_t QPK_CAT(redq_launch_nd, QPK_INST)(const RedqParams& P, const double* w, uint64_t n, uint8_t* out,
                                              uint32_t* st, cudaStream_t s) {
    return redq_dispatch_q<QPK_INST>(P, w, n, out, st, s);
}

#if QPK_INST <= 4
cudaError_t QPK_CAT(polymul_launch_k, QPK_INST)(const PolymulParams& P, const uint8_t* a, const uint8_t* b,
                                                uint64_t n, uint8_t* out, uint32_t* st, cudaStream_t s) {
    return polymul_dispatch_q<QPK_INST>(P, a, b, n, out, st, s);
}

cudaError_t QPK_CAT(gfq_elem_launch_k, QPK_INST)(const GfqElemParams& P, const uint8_t* a, const uint8_t* b,
                                                 uint64_t n, uint8_t* out, cudaStream_t s) {
    return gfq_elem_dispatch<QPK_INST>(P, a, b, n, out, s);
}
#endif

}  // namespace qpk
