// One chunk width of the K6 convolution kernels, selected with -DQPK_INST=ND
// (2k-1 residues per product chunk: 1, 3, ..., 15); build.py compiles this
// file once per width so the template instantiations build in parallel.
#include "fqt_conv.cuh"

#ifndef QPK_INST
#error "compile with -DQPK_INST=<1|3|...|15>"
#endif

#define QPK_CAT2(a, b) a##b
#define QPK_CAT(a, b) QPK_CAT2(a, b)

namespace qpk {

cudaError_t QPK_CAT(fqt_conv_nd, QPK_INST)(const FqtParams& P, const double* pw, uint64_t L1, const double* qw,
                                           uint64_t L2, uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res,
                                           cudaStream_t s) {
    return run_conv<QPK_INST>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
}

}  // namespace qpk
