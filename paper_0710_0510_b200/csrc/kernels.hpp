// Host-visible parameter blocks and launchers for the sm_100a kernels.
// Everything here is plain data: the C-ABI (capi.cpp) fills these from the
// host-side plan/field objects and calls the launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qpk {

constexpr int kMaxFastDigits = 8;   // templated fast path: d+1 <= 8
constexpr int kMaxDigits = 64;      // generic path
constexpr int kMaxGfqK = 4;         // coefficient records up to 4 bytes

// status bits OR-ed into a device word by the kernels
enum : uint32_t {
    kErrDomain = 1u,      // word outside [0, min(q^(d+1), 2^53))  (redq.cpp:22-29, dqt.cpp:96-97)
    kErrOutOfRange = 2u,  // premultiplied floor outside r_max     (fpdiv.cpp:133-135)
    kErrRep = 4u,         // field element rep >= p^k: read as the zero element (gfq.cpp:317-320
                          // from_index, gfq_matmul's GfqMatrix reps: std::out_of_range)
};

// One REDQ plan as the device sees it (RedqPlan, redq.hpp:46-61).
struct RedqParams {
    uint32_t p;
    uint32_t d;           // highest digit index
    uint32_t qbits;       // log2(q) when q is a power of two, else 0
    uint32_t neg_q;       // (p - q mod p) mod p
    uint32_t window;      // 0 = direct/identity correction, else table window (2..4)
    uint32_t radix;       // table index radix (p or 2^ceil(log2 p))
    uint32_t n_entries;   // radix^window
    uint32_t mod_magic;   // ceil(2^32 / p), exact mod for t < 2^16 when p <= 256
    uint32_t float_mode;  // RedqMode::float_premul
    double inv_p;         // ReciprocalDivisor(p).inv_up
    double r_max;         // premul exactness bound (as an exact double)
    double limit;         // min(q^(d+1), 2^53): words must lie below
    uint64_t q;
    uint64_t qpow[kMaxDigits];
    uint64_t qpow64[kMaxDigits];  // q^i exactly when < 2^64, else 0 (u64 words: floor(r / q^i) = 0)
    uint64_t limit_u64;           // q^(d+1) when < 2^64, else 0 (every u64 word is in range)
    double inv_q[kMaxDigits];  // ReciprocalDivisor(q^i).inv_up, general q
    const uint32_t* table;     // device table, byte-packed windows (mu_j in byte j)
};

// Batched small polynomial product (config 1): pack, fp64 product, REDQ.
struct PolymulParams {
    RedqParams rq;  // d = 2k-2
    uint32_t k;
};

// The compile-time fast path of the GF elementwise product: GF(7^3) at
// q = 2^8 (BASELINE config 3).  Its dlog path reads the antilog table from
// kDlogCopies interleaved copies (entry e, copy c at word e*kDlogCopies + c;
// lane l reads copy l mod kDlogCopies, so only the 32/kDlogCopies lanes of
// one copy share its banks).  16 copies (44 KB, two lanes per copy) with the
// producer-warp pipeline measured 27.0-27.2 us for C3 dlog against 27.6-27.8
// with 8 (scripts/c3_sweep.py, round 2).
#ifndef QPK_DLOG_COPIES
#define QPK_DLOG_COPIES 16
#endif
constexpr uint32_t kDlogCopies = QPK_DLOG_COPIES;
constexpr bool gfq_fast_field(uint64_t p, uint32_t k, uint64_t q) { return p == 7 && k == 3 && q == 256; }

// GF elementwise product paths (qpk_gfq_mul_batch `path`)
constexpr int kGfqPacked = 0;  // DQT pack, fp64 product, REDQ, L/H tables (gfq.cpp:353-384)
constexpr int kGfqDlog = 1;    // dlog/Zech representation (gfq.cpp:260-264)
constexpr int kGfqLinear = 2;  // GF(7^3), q = 2^8 only: integer word product + lane-wise mod 7 (an extra;
                               // other fields run kGfqPacked)

// GF(p^k) elementwise product (config 3).
struct GfqElemParams {
    RedqParams rq;          // d = 2k-2, mode float
    uint32_t k, p, order, group, lh_radix;
    double qd;              // q as double (Horner)
    const uint32_t* lc;     // lh^k: corrected low half  -> coefficient bytes
    const uint32_t* hc;     // lh^k: corrected high half -> coefficient bytes (reduced by the modulus)
    const uint32_t* log;    // p^k: coefficient index -> rep
    const uint32_t* alog;   // p^k: rep -> coefficient bytes (sentinel -> 0)
    uint32_t tables_words;  // all tables, contiguous from lc (for smem staging)
    uint32_t fast_off;      // word offset of the fast-path block (gfq_fast_field), else 0; at the
                            // base-p index e of three coefficients or digits:
                            //   L16[p^3] (low half: coefficient bytes 0, 1; padded to whole words)
                            //   | H[p^3] (coefficient bytes) | LOG[p^3] (4*kDlogCopies*log, zero ->
                            //   4*kDlogCopies*(2g-1)) | (16-byte aligned) ALOG[2g * kDlogCopies] (rep i mod g as
                            //   coefficient bytes, zero at 2g-1; copies interleaved)
    uint32_t col3, col4;    // k = 3: coefficient bytes of x^3 and x^4 mod the field polynomial
    int mode;               // kGfqPacked, kGfqDlog or kGfqLinear
};

// GF(p^k) matrix product (configs 4/5).
constexpr uint32_t kRepackRedq = 0, kRepackFold = 1;
constexpr uint32_t kMatmulBK = 16;  // K-steps per shared-memory stage (gfq_matmul.cuh BK)

// Post-re-pack digit bound of the lane fold for q = 2^B (gfq_matmul.cuh
// repack_fold3): S = the even split kFoldShift<B>, bound (2^S-1) + (2^(B-S)-1).
inline uint32_t fold_digit_bound(uint32_t B) {
    uint32_t S = (B + 2) / 2;
    if (S % 2) ++S;
    return ((1u << S) - 1) + ((1u << (B - S)) - 1);
}

struct GfqMatmulParams {
    RedqParams rq;        // d = 2k-2, digits of one accumulated word
    uint32_t k, p, order, group, lh_radix;
    uint32_t chunk;       // delayed REDQ re-pack every `chunk` K-steps (0 = never)
    uint32_t repack;      // kRepackRedq (canonical mu_i) or kRepackFold (lane fold, p = 3, q = 2^(2m))
    double qd;
    const uint32_t* lc;   // as GfqElemParams
    const uint32_t* hc;
    const uint32_t* log;  // for rep output
    const double* fval;   // rep -> q-adic evaluation (float_eval, gfq.cpp:194-207)
};

// GF(p^k) matrix-vector product / long dot product on dlog reps (K5).
struct GfqGemvParams {
    RedqParams rq;        // d = 2k-2
    uint32_t k, p, order, lh_radix;
    uint32_t chunk;       // products per lane per REDQ group (<= n_q; 0 = one group)
    uint32_t vals32;      // every packed value (fval) is below 2^32: u32 values, exact u64 MAC
    const uint32_t* lc;   // lc | hc contiguous (lh_radix^k words each), as GfqElemParams
    const uint32_t* log;  // p^k: coefficient index -> rep
    const double* fval;   // rep -> q-adic evaluation (float_eval, gfq.cpp:194-207)
    uint32_t* status;     // the field's error word: kErrRep for reps >= order (read as zero)
};

// GF(p^k) outside the byte-packed fast form (k > 4 or p > 255), rep domain
// throughout (gfq_wide.cu).
constexpr uint32_t kMaxWideK = 8;  // q^(2k-1) < 2^53 with q > k (p-1)^2 allows k <= 8
struct GfqWideParams {
    uint32_t p, k, order, group, lh_radix, qbits;  // qbits: log2 q for q = 2^b, else 0
    uint32_t chunk;                                // products per lane per REDQ group (n_q)
    uint64_t qpow[2 * kMaxWideK - 1];              // q^i
    const double* fval;                            // rep -> q-adic evaluation
    const uint32_t* log;                           // polynomial index -> rep
    const uint32_t* antilog;                       // rep -> polynomial index
    const uint32_t* low;                           // lh^k reps
    const uint32_t* high;                          // lh^k reps
    const uint32_t* zech;                          // order reps (plus-one table)
    uint32_t* status;                              // kErrRep
};
// elementwise products of k-byte coefficient records (p < 256); path kGfqDlog
// or the DQT/REDQ/L-H pipeline (kGfqPacked, kGfqLinear)
cudaError_t launch_gfq_wide_mul(const GfqWideParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                                int path, cudaStream_t s);
// y = A x on reps; ws: gfq_wide_workspace_bytes
uint64_t gfq_wide_workspace_bytes(uint64_t m, uint64_t K);
cudaError_t launch_gfq_wide_gemv(const GfqWideParams& P, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                                 void* ws, uint32_t* out_rep, uint8_t* out_coeff, cudaStream_t s);
cudaError_t launch_gfq_wide_reps_to_coeffs(const GfqWideParams& P, const uint32_t* reps, uint64_t n, uint8_t* out,
                                           cudaStream_t s);

// K7: fgdp_dot's data-dependent Zech reads, replayed per gfq_matmul output.
constexpr uint32_t kMaxCountK = 8;
struct GfqCountParams {
    uint32_t p, k, group, lh_radix, qbits;  // qbits: log2 q for q = 2^b, else 0
    uint64_t n_q;
    uint64_t qpow[2 * kMaxCountK - 1];      // q^i
    const double* fval;                     // rep -> q-adic evaluation
    const uint32_t* low;                    // lh^k reps (GfqField low table)
    const uint32_t* high;                   // lh^k reps
    const uint32_t* zech;                   // order reps (plus-one table)
};

// Chunked FQT product of two long polynomials (K6, fqt_mul polymul.cpp:81-147).
struct FqtParams {
    RedqParams rq;  // fqt_reduction_plan: d = 2k-2 (ND = 2k-1 <= 15)
    uint32_t k;     // coefficients per chunk (d+1)
    uint32_t nq;    // products per REDQ group (params.n_q)
    // DMMA kernel, q = 2^b with q^(2k-1) <= 2^52: accumulators biased by 2^52
    // and the group REDQ in integers, floor(r/p) = mulhi64(r, p_magic)
    uint32_t mma_int;
    uint64_t p_magic;  // ceil(2^64 / p)
};

// ---- launchers (return cudaError_t of the launch) ----
cudaError_t launch_redq_f64(const RedqParams& P, const double* words, uint64_t n, uint8_t* out,
                            uint32_t* status, cudaStream_t s);
// REDQ of integer words (u64; the reference's integer mode beyond fp64):
// floor(r/p) as (hi/p) 2^32 + premul floor of (hi mod p) 2^32 + lo (< 2^40 <= r_max)
cudaError_t launch_redq_u64(const RedqParams& P, const uint64_t* words, uint64_t n, uint8_t* out,
                            uint32_t* status, cudaStream_t s);
cudaError_t launch_polymul(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                           uint8_t* out, uint32_t* status, cudaStream_t s);
cudaError_t launch_gfq_elem(const GfqElemParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                            uint8_t* out, cudaStream_t s);
// GfqField::mul over reps; reps above g latch kErrRep in *status (read as zero)
cudaError_t launch_gfq_mul_rep(uint32_t group, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out,
                               uint32_t* status, cudaStream_t s);

// DQT pack of coefficient records into q-adic doubles (K1a): src is
// rows x cols x k bytes; dst element (r, c) goes to dst[c*ld + r] when
// `transpose`, else dst[r*ld + c].  dst must be pre-zeroed for padding.
// pair_layout: K4 fragment column order (mm_col_a for the transposed operand A,
// mm_col_b for B)
cudaError_t launch_pack_coeffs(uint32_t p, uint32_t k, double qd, const uint8_t* src, uint64_t rows,
                               uint64_t cols, double* dst, uint64_t ld, bool transpose, bool pair_layout,
                               cudaStream_t s);
// Zech/dlog tabulated pack (K1b): reps -> float_eval(rep) via a smem table;
// reps >= order are packed as zero and latch kErrRep in *status.
// layout helpers of the GEMV-column matmul route (fields whose n_q is below
// one fp64 MMA step): u32 transpose, coefficient records <-> reps through
// the field's log / antilog-to-bytes tables (GfqElemParams log, alog)
cudaError_t launch_transpose_u32(const uint32_t* src, uint64_t rows, uint64_t cols, uint32_t* dst, cudaStream_t s);
cudaError_t launch_coeffs_to_reps(uint32_t p, uint32_t k, const uint32_t* log, const uint8_t* src, uint64_t n,
                                  uint32_t* dst, cudaStream_t s);
cudaError_t launch_reps_to_coeffs(uint32_t k, const uint32_t* alog, const uint32_t* src, uint64_t n, uint8_t* dst,
                                  cudaStream_t s);
cudaError_t launch_pack_reps(const double* fval, uint32_t order, const uint32_t* src, uint64_t rows,
                             uint64_t cols, double* dst, uint64_t ld, bool transpose, bool pair_layout,
                             uint32_t* status, cudaStream_t s);

// Column order of the K4 operand workspaces when mm_pair_layout(P) holds (the
// C5 fast path with the canonical re-pack).  A thread of the fp64 MMA takes
// the elements 8 i + lr of its warp's 64 rows of A^T (i = 0..7) and of its
// warp's 32 columns of B (i = 0..3).  Inside every 64-block of A^T columns
// and every 32-block of B columns, element 8 i + lr is stored at
// 16 (i / 2) + 2 lr + (i % 2): a thread's fragment pairs are adjacent (one
// 16-byte shared load for two fragments: 6 loads per k-step instead of 12)
// and the eight lanes of a quarter warp read eight different 16-byte bank
// groups (row stride 132 doubles == 32 bytes mod 128).  Every instruction
// next to the DMMAs costs a dispatch slot: C5 37.10 ->
// 36.54 ms.  Not used by the other K4 kernels: at the 168-register cap the
// aligned register quads of the 16-byte loads make ptxas spill in the fold
// kernel (33.0 -> 36.4 ms) and gain nothing for C4.
__host__ __device__ constexpr uint64_t mm_col_a(uint64_t x) {
    return (x & ~uint64_t(63)) | (((x >> 4) & 3) << 4) | ((x & 7) << 1) | ((x >> 3) & 1);
}
__host__ __device__ constexpr uint64_t mm_col_b(uint64_t x) {
    return (x & ~uint64_t(31)) | (((x >> 4) & 1) << 4) | ((x & 7) << 1) | ((x >> 3) & 1);
}
// a plan is "safe" when every accumulated word stays <= min(r_max, 2^52)
inline bool mm_plan_safe(const RedqParams& R) {
    return R.qbits && R.limit <= R.r_max + 1.0 && R.limit <= 4503599627370496.0;
}
// the launch that takes the paired column order (P with chunk and repack resolved)
inline bool mm_pair_layout(const GfqMatmulParams& P) {
    return P.k == 3 && P.p == 3 && P.rq.qbits == 10 && mm_plan_safe(P.rq) &&
           (P.chunk == 0 || P.chunk % kMatmulBK == 0) && P.repack != kRepackFold;
}

// K4: C = A*B on packed operands.  at is K x m_pad (A transposed), b is
// K x n_pad, both zero padded (m_pad, n_pad multiples of 128, K_pad of 16),
// packed with pair_layout = mm_pair_layout(P).
// Output either coefficient bytes (m x n x k) or reps (m x n u32).
cudaError_t launch_gfq_matmul(const GfqMatmulParams& P, const double* at, const double* b, uint64_t m,
                              uint64_t n, uint64_t K_pad, uint64_t m_pad, uint64_t n_pad, uint8_t* out_coeffs,
                              uint32_t* out_reps, cudaStream_t s);

// K5: y = A x over GF(p^k), A m x K reps (row-major), x K reps; `splits`
// K-ranges per row (gemv_splits); ws: gemv_workspace_bytes (packed x and
// split partials, 16-byte aligned).  Either output may be null: y_rep (m
// reps) and/or y_coeff (m x k bytes).
uint32_t gemv_splits(uint64_t m, uint64_t K);
uint64_t gemv_workspace_bytes(uint64_t m, uint64_t K, uint32_t splits);
cudaError_t launch_gfq_gemv(const GfqGemvParams& P, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                            uint32_t splits, void* ws, uint32_t* y_rep, uint8_t* y_coeff, cudaStream_t s);

// K6: out (na+nb-1 coefficients) = a * b mod p, coefficients as uint8;
// REDQ of u128 integer words ((lo, hi) u64 pairs, the reference's integer
// mode up to q^(d+1) <= 2^128, redq.cpp:44-58): u128 arithmetic, direct
// correction.  limit: q^(d+1) as (lo, hi), or 0/0 when it exceeds 2^128.
// GfqField::mul / add / neg / inverse over reps (gfq.cpp:260-294), op 0..3;
// add reads the Zech (plus-one) table zech[g+1] (zero sentinel g); inverse
// of zero latches kErrDomain in *status
cudaError_t launch_gfq_rep_op(int op, uint32_t p, uint32_t group, const uint32_t* zech, const uint32_t* a,
                              const uint32_t* b, uint64_t n, uint32_t* out, uint32_t* status, cudaStream_t s);
cudaError_t launch_redq_u128(const RedqParams& P, const uint64_t* words, uint64_t n, uint8_t* out, uint32_t* status,
                             cudaStream_t s);

// FQT product with integer words beyond fp64 (the reference's u128 mode,
// m up to 128: polymul.cpp:97-146 with u128 MAC): packed words and group
// sums as unsigned __int128, integer-mode REDQ per group (redq.cpp:44-58)
// and the direct correction.  ws: fqt_wide_workspace_bytes.
uint64_t fqt_wide_workspace_bytes(uint32_t k, uint64_t na, uint64_t nb);
cudaError_t launch_fqt_mul_wide(uint32_t p, uint64_t q, uint32_t k, uint32_t nq, const uint8_t* a, uint64_t na,
                                const uint8_t* b, uint64_t nb, uint8_t* out, void* ws, cudaStream_t s);

// FQT product for p > 256 (any p < 2^63; the uint8 kernels above cover
// p <= 256): u64 coefficients in and out (reduced mod p), u128 words and
// group sums, integer-mode REDQ per group with the direct correction, one
// thread per output chunk.  ws: fqt_widep_workspace_bytes.
uint64_t fqt_widep_workspace_bytes(uint32_t k, uint64_t na, uint64_t nb);
cudaError_t launch_fqt_mul_widep(uint64_t p, uint64_t q, uint32_t k, uint32_t nq, const uint64_t* a, uint64_t na,
                                 const uint64_t* b, uint64_t nb, uint64_t* out, void* ws, cudaStream_t s);

// ws: fqt_workspace_bytes (packed chunks and per-chunk residue partials).
uint64_t fqt_workspace_bytes(uint32_t k, uint32_t nq, uint64_t na, uint64_t nb);
cudaError_t launch_fqt_mul(const FqtParams& P, const uint8_t* a, uint64_t na, const uint8_t* b, uint64_t nb,
                           uint8_t* out, void* ws, cudaStream_t s);

// Synthetic inputs: out[i] = SplitMix64(seed) draw (start+i+1) mod bound.
cudaError_t launch_gen_draws(uint64_t seed, uint64_t start, uint64_t count, uint32_t bound, uint8_t* out,
                             cudaStream_t s);
// q-adic words: out[i] = word first+i, word w = sum_j (draw w*(d+1)+j+1 mod q) * q^(d-j)
cudaError_t launch_gen_words(uint64_t seed, uint64_t first, uint64_t n, uint64_t q, uint32_t d, double* out,
                             cudaStream_t s);
// record pairs: a[i] = draws 2k*i+1..2k*i+k, b[i] = the next k
cudaError_t launch_gen_pairs(uint64_t seed, uint64_t n, uint32_t k, uint32_t bound, uint8_t* a, uint8_t* b,
                             cudaStream_t s);

// total (added atomically) += Zech-table reads of fgdp_dot(A[i,:], B[:,j]) over
// all outputs; A m x K and B K x n reps, row-major
cudaError_t launch_gfq_count(const GfqCountParams& P, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K,
                             uint64_t n, unsigned long long* total, cudaStream_t s);

// fp64 peak probes (roofline denominators): returns flop count per launch
cudaError_t launch_probe_dfma(double* sink, int iters, uint64_t* flops, cudaStream_t s);
cudaError_t launch_probe_dmma(double* sink, int iters, uint64_t* flops, cudaStream_t s);

int num_sms();  // of the current device

// Raise `kernel`'s dynamic shared-memory limit to at least `bytes` on the
// current device (a per-device function attribute: recorded per (kernel,
// device), thread-safe; a no-op below the 48 KB default).
cudaError_t ensure_dyn_smem(const void* kernel, size_t bytes, size_t static_bytes = 0);

}  // namespace qpk
