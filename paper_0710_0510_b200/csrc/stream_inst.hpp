// Per-width instantiations of the TMA streaming pipeline (stream_inst.cu).
#pragma once

#include <cuda_runtime.h>

#include "kernels.hpp"

namespace qpk {

#define QPK_DECL_REDQ(N)                                                                                   \
    cudaError_t redq_launch_nd##N(const RedqParams& P, const double* w, uint64_t n, uint8_t* out, uint32_t* st, \
                                  cudaStream_t s);
#define QPK_DECL_K(K)                                                                                        \
    cudaError_t polymul_launch_k##K(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, \
                                    uint8_t* out, uint32_t* st, cudaStream_t s);                            \
    cudaError_t gfq_elem_launch_k##K(const GfqElemParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, \
                                     uint8_t* out, cudaStream_t s);

QPK_DECL_REDQ(1)
QPK_DECL_REDQ(2)
QPK_DECL_REDQ(3)
QPK_DECL_REDQ(4)
QPK_DECL_REDQ(5)
QPK_DECL_REDQ(6)
QPK_DECL_REDQ(7)
QPK_DECL_REDQ(8)
QPK_DECL_K(1)
QPK_DECL_K(2)
QPK_DECL_K(3)
QPK_DECL_K(4)

#undef QPK_DECL_REDQ
#undef QPK_DECL_K

}  // namespace qpk
