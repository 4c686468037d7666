// Batched GPU entry points of qpack-b200 (C++ face of include/qpack_b200.h).
//
// The reference's per-word calls (redq_residues_into, dqt_mul_poly, fgdp_dot
// on length-1 vectors, GfqField::mul) cannot be accelerated one word at a
// time; these overloads take whole batches and run the sm_100a kernels.
// Pointers are HOST memory; results are visible on return, exactly like the
// reference.  Errors throw the reference's exception types.
#pragma once

#include <cstdint>
#include <span>

#include "qpack/counters.hpp"
#include "qpack/gfq.hpp"
#include "qpack/params.hpp"
#include "qpack/redq.hpp"

namespace qpack::gpu {

// redq_residues_into over words given as exact doubles; out has n*(d+1)
// residues (p <= 256).  (redq.hpp:73-74)
void redq_residues_batch(std::span<const double> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost = nullptr);
// the same over integer words below min(q^(d+1), 2^64) (the reference's u128
// integer mode, restricted to 64-bit words)
void redq_residues_batch(std::span<const std::uint64_t> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost = nullptr);
// ... and over u128 words below q^(d+1) (the reference's integer mode in
// full, redq.cpp:44-58)
void redq_residues_batch(std::span<const u128> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost = nullptr);

// n products of degree-<k polynomials (records of k coefficients) -> n*(2k-1)
// residues, via pack -> fp64 product -> REDQ.  (dqt_mul_poly dqt.hpp:46,
// fqt_mul single chunk polymul.hpp:42)
void polymul_batch(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b, const QadicParams& params,
                   std::span<std::uint8_t> out, CostReport* cost = nullptr);

// packed: DQT pack, fp64 product, REDQ, L/H tables (gfq.cpp:353-384);
// dlog: GfqField::mul on the Zech/discrete-log representation (gfq.cpp:260-264);
// linear: GF(7^3) at q = 2^8 only -- integer word product and lane-wise mod 7
// through x^3, x^4 (an extra; every other field runs `packed`)
enum class GfqPath { packed = 0, dlog = 1, linear = 2 };

// elementwise GF(p^k) products of coefficient records (k bytes each)
void gfq_mul_batch(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b, const GfqField& field,
                   std::span<std::uint8_t> out, GfqPath path = GfqPath::packed);

// elementwise GfqField::mul over reps
void gfq_mul_batch(std::span<const GfqElt> a, std::span<const GfqElt> b, const GfqField& field,
                   std::span<GfqElt> out);

// Delayed re-pack between K-chunks: `redq` re-packs every accumulated word
// to sum mu_i q^i (REDQ + assemble, redq.cpp:178-182); `fold` (GF(3^3) at
// q = 2^10) replaces each digit by a smaller one congruent mod p (see
// DESIGN.md 5).  Both give the same product.
enum class Repack : std::uint32_t { redq = 0, fold = 1 };

// C = A*B of coefficient records: A is m x K x k, B is K x n x k, C m x n x k
void gfq_matmul_coeffs(std::span<const std::uint8_t> A, std::span<const std::uint8_t> B, std::size_t m,
                       std::size_t K, std::size_t n, const GfqField& field, std::span<std::uint8_t> C,
                       std::uint32_t chunk = 0, CostReport* cost = nullptr, Repack repack = Repack::redq);

// y = A x over GF(p^k) on reps: A is m x K (row-major), x has K entries, y
// gets m.  Each y_i is fgdp_dot(A[i,:], x) (gfq.hpp:98-99, gfq.cpp:335-387).
void gfq_gemv(std::span<const GfqElt> A, std::span<const GfqElt> x, std::size_t m, const GfqField& field,
              std::span<GfqElt> y, CostReport* cost = nullptr);

// fgdp_dot of two long vectors on the GPU (one row of gfq_gemv, split over
// the whole device)
GfqElt fgdp_dot(std::span<const GfqElt> v1, std::span<const GfqElt> v2, const GfqField& field,
                CostReport* cost = nullptr);

}  // namespace qpack::gpu
