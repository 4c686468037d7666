// Internal GPU entry points shared by the C++ API (gpu_api.cpp) and the
// C-ABI (capi.cpp).  Device-pointer variants are asynchronous on `s`;
// *_host variants take host buffers and return when results are visible.
#pragma once

#include <cuda_runtime.h>

#include "device_state.hpp"
#include "qpack/counters.hpp"
#include "qpack/gfq.hpp"
#include "qpack/params.hpp"
#include "qpack/redq.hpp"

namespace qpack::gpu {

uint32_t take_status(detail::DevicePlanCache& dp, cudaStream_t s);
void raise_status(uint32_t st);
// the field's error word (kErrRep, kErrDomain): wait for `s`, read, clear
uint32_t take_field_status(detail::DeviceFieldCache& F, cudaStream_t s);
void raise_field_status(uint32_t st);

void redq_device(detail::DevicePlanCache& dp, const double* d_words, u64 n, uint8_t* d_out, cudaStream_t s);
void redq_host(detail::DevicePlanCache& dp, const double* h_words, u64 n, uint8_t* h_out);
void redq_device_u64(detail::DevicePlanCache& dp, const uint64_t* d_words, u64 n, uint8_t* d_out, cudaStream_t s);
void redq_host_u64(detail::DevicePlanCache& dp, const uint64_t* h_words, u64 n, uint8_t* h_out);
void redq_device_u128(detail::DevicePlanCache& dp, const uint64_t* d_words, u64 n, uint8_t* d_out, cudaStream_t s);
void redq_host_u128(detail::DevicePlanCache& dp, const uint64_t* h_words, u64 n, uint8_t* h_out);

// fqt_mul / dqt_mul_poly over a batch of single-chunk pairs
struct PolymulPlan {
    QadicParams params;
    RedqPlan redq;  // fqt_reduction_plan(params, k-1)
    qpk::PolymulParams P{};
    explicit PolymulPlan(const QadicParams& pr);
};
void polymul_device(PolymulPlan& pl, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, cudaStream_t s);
void polymul_host(PolymulPlan& pl, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out);
CostReport polymul_cost(const PolymulPlan& pl, u64 n);

// K6: chunked FQT product of long polynomials (uint8 coefficients, p <= 256)
void fqt_mul_device(const RedqPlan& plan, const QadicParams& params, const uint8_t* a, u64 na, const uint8_t* b,
                    u64 nb, uint8_t* out, cudaStream_t s);
void fqt_mul_host(const RedqPlan& plan, const QadicParams& params, const uint8_t* a, u64 na, const uint8_t* b, u64 nb,
                  uint8_t* out);
// any p (u64 coefficients, reduced mod p; the reference's DensePoly range)
void fqt_mul_device_u64(const RedqPlan& plan, const QadicParams& params, const uint64_t* a, u64 na, const uint64_t* b,
                        u64 nb, uint64_t* out, cudaStream_t s);
void fqt_mul_host_u64(const RedqPlan& plan, const QadicParams& params, const uint64_t* a, u64 na, const uint64_t* b,
                      u64 nb, uint64_t* out);
CostReport fqt_cost(const RedqPlan& plan, const QadicParams& params, u64 na, u64 nb);

void gfq_mul_device(detail::DeviceFieldCache& F, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, int path,
                    cudaStream_t s);
void gfq_mul_host(detail::DeviceFieldCache& F, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, int path);
void gfq_mul_rep_host(detail::DeviceFieldCache& F, const uint32_t* a, const uint32_t* b, u64 n, uint32_t* out);
void gfq_rep_op_host(detail::DeviceFieldCache& F, const GfqField& field, int op, const uint32_t* a, const uint32_t* b,
                     u64 n, uint32_t* out);

// repack: qpk::kRepackRedq (canonical REDQ re-pack) or qpk::kRepackFold
uint32_t resolve_chunk(const detail::DeviceFieldCache& F, const GfqField& field, u64 K, uint32_t chunk,
                       uint32_t repack = 0);
void gfq_matmul_device(detail::DeviceFieldCache& F, const GfqField& field, const void* A, const void* B, u64 m, u64 K,
                       u64 n, uint32_t chunk, void* C, bool reps, cudaStream_t s, uint32_t repack = 0,
                       const double* packed_b = nullptr);
// zech_reads: when given, also the reference's data-dependent counter part (K7)
void gfq_matmul_host(detail::DeviceFieldCache& F, const GfqField& field, const void* A, const void* B, u64 m, u64 K,
                     u64 n, uint32_t chunk, void* C, bool reps, uint32_t repack = 0, u64* zech_reads = nullptr);
CostReport matmul_cost(const GfqField& field, u64 m, u64 K, u64 n);
// fgdp_dot's data-dependent Zech reads summed over C = A*B (K7), A and B
// device rep arrays (m x K, K x n); synchronous on stream s
u64 zech_reads_device(detail::DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* B, u64 m,
                      u64 K, u64 n, cudaStream_t s);

void gfq_gemv_device(detail::DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* x, u64 m,
                     u64 K, uint32_t* y_rep, uint8_t* y_coeff, cudaStream_t s);
void gfq_gemv_host(detail::DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* x, u64 m,
                   u64 K, uint32_t* y_rep, uint8_t* y_coeff, u64* zech_reads = nullptr);
CostReport gemv_cost(const GfqField& field, u64 m, u64 K);

}  // namespace qpack::gpu
