/* qpack-b200 C-ABI — the drop-in boundary of the q-adic transform pipeline
 * (arXiv 0710.0510) on B200 / sm_100a.
 *
 * Plain C types only: integers, doubles, raw pointers, opaque handles.  Each
 * entry point names the reference interface it replaces (paths relative to
 * the reference's proj/).  The reference itself is a C++ header API with no
 * FFI; INTEGRATION.md shows the ctypes / C++ bindings a maintainer adds.
 *
 * Errors: every call returns a qpk_status that maps 1:1 onto the exception
 * class the reference throws for the same condition; the
 * message is in qpk_last_error() (thread-local, valid until the next call on
 * the same thread).
 *
 * Pointer conventions: functions WITHOUT a `_host` suffix take DEVICE
 * pointers and a `stream` (a cudaStream_t, NULL = legacy default stream);
 * they are asynchronous and latch data errors on the plan or field
 * (qpk_redq_sync / qpk_polymul_sync / qpk_field_sync report them).  `_host` functions take HOST pointers
 * (pinned memory gives the full PCIe overlap), copy in and out internally
 * and return only when results are visible — the reference's synchronous
 * semantics.  There is no CPU fallback: without a usable CUDA device every
 * compute entry point returns QPK_ERR_CUDA.
 */
#ifndef QPACK_B200_H
#define QPACK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QPK_API __attribute__((visibility("default")))
#define QPK_ABI_VERSION 1

typedef enum qpk_status {
    QPK_OK = 0,
    QPK_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    QPK_ERR_DOMAIN = 2,           /* std::domain_error     */
    QPK_ERR_LENGTH = 3,           /* std::length_error     */
    QPK_ERR_OUT_OF_RANGE = 4,     /* std::out_of_range     */
    QPK_ERR_OVERFLOW = 5,         /* std::overflow_error   */
    QPK_ERR_RUNTIME = 6,          /* std::runtime_error    */
    QPK_ERR_LOGIC = 7,            /* std::logic_error      */
    QPK_ERR_CUDA = 8              /* device failure / no device (no reference counterpart) */
} qpk_status;

/* CostReport (counters.hpp:20-33) */
typedef struct qpk_cost {
    uint64_t mul_add, divisions, table_accesses, reduction_calls;
} qpk_cost;

QPK_API const char* qpk_last_error(void);
QPK_API int qpk_abi_version(void);
/* SM count and compute capability of the current device */
QPK_API qpk_status qpk_device_info(int* sms, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------- REDQ (K2) */
typedef struct qpk_redq_plan_s* qpk_redq_plan;

/* RedqPlan::build(p, q, d, mode)            redq.hpp:57, redq.cpp:115-146
 * mode 0 = RedqMode::integer, 1 = RedqMode::float_premul */
QPK_API qpk_status qpk_redq_plan_create(uint64_t p, uint64_t q, uint32_t d, int mode, qpk_redq_plan* out);
/* plan.attach_correction(build_correction_table(p, q, window, indexing))
 *                                            redq.hpp:60, 93-94; redq.cpp:148-152, 203-245
 * indexing 0 = TableIndexing::base_p, 1 = binary_shift */
QPK_API qpk_status qpk_redq_plan_attach_table(qpk_redq_plan plan, uint32_t window, int indexing);
/* attach_correction(load_correction_table(bytes))   redq.hpp:108, redq.cpp:299-323 ("QPKT" v1) */
QPK_API qpk_status qpk_redq_plan_attach_table_bytes(qpk_redq_plan plan, const uint8_t* qpkt, uint64_t len);
QPK_API void qpk_redq_plan_destroy(qpk_redq_plan plan);

/* redq_residues_into over a batch             redq.hpp:73-74, redq.cpp:162-170
 * words: n exact-integer doubles (packed_from_double semantics, dqt.cpp:96-100),
 * residues: n*(d+1) uint8, record i = (mu_0..mu_d) of word i.  p <= 256. */
QPK_API qpk_status qpk_redq_residues_f64(qpk_redq_plan plan, const double* words, uint64_t n, uint8_t* residues,
                                         void* stream);
QPK_API qpk_status qpk_redq_residues_f64_host(qpk_redq_plan plan, const double* words, uint64_t n,
                                              uint8_t* residues, qpk_cost* cost);
/* the same for integer words (RedqMode::integer beyond fp64, redq.cpp:44-51):
 * u64 words below min(q^(d+1), 2^64), any d and q                     */
QPK_API qpk_status qpk_redq_residues_u64(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                         void* stream);
QPK_API qpk_status qpk_redq_residues_u64_host(qpk_redq_plan plan, const uint64_t* words, uint64_t n,
                                              uint8_t* residues, qpk_cost* cost);
/* u128 words as (lo, hi) uint64 pairs, below q^(d+1) <= 2^128: the
 * reference's integer mode in full (redq.cpp:44-58)                       */
QPK_API qpk_status qpk_redq_residues_u128(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                          void* stream);
QPK_API qpk_status qpk_redq_residues_u128_host(qpk_redq_plan plan, const uint64_t* words, uint64_t n,
                                               uint8_t* residues, qpk_cost* cost);
/* wait for `stream`, then report (and clear) latched data errors:
 * QPK_ERR_DOMAIN = a word not below q^(d+1) / not an exact double (redq.cpp:27-28).
 * The error word is per plan: it collects what every launch on the plan
 * latched, on any stream (a caller that shares one plan across streams sees
 * the union; use one plan per stream to attribute errors to one stream). */
QPK_API qpk_status qpk_redq_sync(qpk_redq_plan plan, void* stream);
/* closed-form counters of n reductions (divisions, reduction_calls, table_accesses) */
QPK_API qpk_status qpk_redq_cost(qpk_redq_plan plan, uint64_t n, qpk_cost* cost);

/* ------------------------------------ batched DQT products (K1a + fp64 + K2) */
typedef struct qpk_polymul_plan_s* qpk_polymul_plan;

/* params (p, q, k, n_q, m=53) checked as dqt_mul_poly / fqt_mul do
 *                                            dqt.cpp:81-83, polymul.cpp:81-89 */
QPK_API qpk_status qpk_polymul_plan_create(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, qpk_polymul_plan* out);
/* as above with the word width m (QadicParams::m, params.hpp:23-31): m > 53
 * selects integer (u128) words for qpk_fqt_mul -- the reference's integer
 * mode; the batched qpk_polymul_batch needs q^(2k-1) <= 2^53 */
QPK_API qpk_status qpk_polymul_plan_create_m(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, uint32_t m,
                                             qpk_polymul_plan* out);
QPK_API void qpk_polymul_plan_destroy(qpk_polymul_plan plan);
/* n pairs of k-coefficient records -> n records of 2k-1 residues
 * = fqt_mul(a_i, b_i, k-1, params, fqt_reduction_plan)   polymul.hpp:42-47
 * = dqt_mul_poly(a_i, b_i, params)                        dqt.hpp:46 */
QPK_API qpk_status qpk_polymul_batch(qpk_polymul_plan plan, const uint8_t* a, const uint8_t* b, uint64_t n,
                                     uint8_t* out, void* stream);
QPK_API qpk_status qpk_polymul_batch_host(qpk_polymul_plan plan, const uint8_t* a, const uint8_t* b, uint64_t n,
                                          uint8_t* out, qpk_cost* cost);
QPK_API qpk_status qpk_polymul_sync(qpk_polymul_plan plan, void* stream);
/* one product of two long polynomials (na, nb coefficients, uint8 < 256,
 * reduced mod p) -> na+nb-1 coefficients: chunked FQT (K6)
 * = fqt_mul(a, b, k-1, params, fqt_reduction_plan)          polymul.hpp:42-47, polymul.cpp:81-147
 * k <= 8; counters (host variant) are the reference's closed form */
QPK_API qpk_status qpk_fqt_mul(qpk_polymul_plan plan, const uint8_t* a, uint64_t na, const uint8_t* b, uint64_t nb,
                               uint8_t* out, void* stream);
QPK_API qpk_status qpk_fqt_mul_host(qpk_polymul_plan plan, const uint8_t* a, uint64_t na, const uint8_t* b,
                                    uint64_t nb, uint8_t* out, qpk_cost* cost);
/* the same product with u64 coefficients (reduced mod p on input), for any p
 * the plan accepts -- the uint8 entry points above need p <= 256
 * (DensePoly's u64 coefficients, poly.hpp; polymul.cpp:81-147) */
QPK_API qpk_status qpk_fqt_mul_u64(qpk_polymul_plan plan, const uint64_t* a, uint64_t na, const uint64_t* b,
                                   uint64_t nb, uint64_t* out, void* stream);
QPK_API qpk_status qpk_fqt_mul_u64_host(qpk_polymul_plan plan, const uint64_t* a, uint64_t na, const uint64_t* b,
                                        uint64_t nb, uint64_t* out, qpk_cost* cost);

/* --------------------------------------------------------------- GF(p^k) */
typedef struct qpk_field_s* qpk_field;

/* GfqField::build(p, k, q, indexing)          gfq.hpp:33-34, gfq.cpp:132-258 */
QPK_API qpk_status qpk_field_create(uint64_t p, uint32_t k, uint64_t q, int indexing, qpk_field* out);
QPK_API void qpk_field_destroy(qpk_field f);
/* modulus_poly() (k+1), to_coeffs(generator()) (k), params().n_q, memory_entries()   gfq.hpp:40-66 */
QPK_API qpk_status qpk_field_info(qpk_field f, uint64_t* modulus, uint64_t* generator, uint32_t* n_q,
                                  uint64_t* memory_entries);
/* describe()                                   gfq.hpp:67, gfq.cpp:321-333 */
QPK_API qpk_status qpk_field_describe(qpk_field f, char* buf, uint64_t cap);
/* host copies of the field tables, p^k entries each (L/H: lh_radix^k) */
QPK_API qpk_status qpk_field_tables(qpk_field f, uint32_t* log, uint64_t* antilog, uint32_t* plus1, double* fval,
                                    uint32_t* low, uint32_t* high);
/* GfqField::mul / add / neg / inverse on reps         gfq.cpp:260-294
 * op 0 mul, 1 add, 2 neg, 3 inverse.  qpk_field_op: n elements on the
 * device (host buffers in and out); qpk_field_op1: one element, the
 * reference's scalar call (host code, like every per-element call) */
QPK_API qpk_status qpk_field_op(qpk_field f, int op, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out);
QPK_API qpk_status qpk_field_op1(qpk_field f, int op, uint32_t a, uint32_t b, uint32_t* out);
/* Device-pointer rep entry points (qpk_gfq_matmul_rep, qpk_gfq_gemv) run
 * asynchronously: a rep >= p^k is read as the zero element and latched on
 * the field.  qpk_field_sync waits for `stream` and reports (then clears)
 * what any launch on the field latched, whatever its stream:
 * QPK_ERR_OUT_OF_RANGE for reps outside the field (gfq.cpp:317-320).  The
 * _host entry points check it themselves before returning. */
QPK_API qpk_status qpk_field_sync(qpk_field f, void* stream);
/* fgdp_dot on reps (host, reference Alg. 4)     gfq.hpp:98-99, gfq.cpp:335-387 */
QPK_API qpk_status qpk_fgdp_dot(qpk_field f, const uint32_t* v1, const uint32_t* v2, uint64_t n, uint32_t* out,
                                qpk_cost* cost);

/* elementwise products of k-byte coefficient records (K3)
 * path 0 = DQT/REDQ/L-H   (fgdp_dot on length-1 vectors, gfq.cpp:335-387)
 * path 1 = dlog/Zech      (GfqField::mul, gfq.cpp:260-264)
 * path 2 = linear         (GF(7^3) at q = 2^8: integer word product, lane-wise
 *                          mod 7 through x^3, x^4; other fields run path 0)  */
QPK_API qpk_status qpk_gfq_mul_batch(qpk_field f, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                                     int path, void* stream);
QPK_API qpk_status qpk_gfq_mul_batch_host(qpk_field f, const uint8_t* a, const uint8_t* b, uint64_t n,
                                          uint8_t* out, int path);
/* GfqField::mul over reps (host buffers) */
QPK_API qpk_status qpk_gfq_mul_rep_host(qpk_field f, const uint32_t* a, const uint32_t* b, uint64_t n,
                                        uint32_t* out);

/* C = A*B (K1 pack + K4 contraction)            gfq.hpp:113-114, gfq.cpp:389-404
 * coefficient records: A m x K x k, B K x n x k, C m x n x k (uint8);
 * chunk = K-steps between delayed REDQ re-packs (0 = automatic: never when
 * K <= n_q, else the largest safe chunk). */
QPK_API qpk_status qpk_gfq_matmul(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K,
                                  uint64_t n, uint32_t chunk, uint8_t* C, void* stream);
QPK_API qpk_status qpk_gfq_matmul_host(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K,
                                       uint64_t n, uint32_t chunk, uint8_t* C, qpk_cost* cost);
/* as qpk_gfq_matmul with the delayed re-pack chosen: QPK_REPACK_REDQ (every
 * word re-packed to sum mu_i q^i, redq + assemble, redq.cpp:178-182) or
 * QPK_REPACK_FOLD (GF(3^3) at q = 2^10: digits folded to smaller values
 * congruent mod p, chunk sized for the fold's digit bound); same C. */
#define QPK_REPACK_REDQ 0u
#define QPK_REPACK_FOLD 1u
QPK_API qpk_status qpk_gfq_matmul_repack(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K,
                                         uint64_t n, uint32_t chunk, uint32_t repack, uint8_t* C, void* stream);
QPK_API qpk_status qpk_gfq_matmul_repack_host(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m,
                                              uint64_t K, uint64_t n, uint32_t chunk, uint32_t repack, uint8_t* C,
                                              qpk_cost* cost);
/* the reference signature on GfqMatrix data: reps (u32) in, reps out */
QPK_API qpk_status qpk_gfq_matmul_rep(qpk_field f, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K,
                                      uint64_t n, uint32_t* C, void* stream);
QPK_API qpk_status qpk_gfq_matmul_rep_host(qpk_field f, const uint32_t* A, const uint32_t* B, uint64_t m,
                                           uint64_t K, uint64_t n, uint32_t* C, qpk_cost* cost);

/* y = A x on reps: y_i = fgdp_dot(A[i,:], x)    gfq.hpp:98-99, gfq.cpp:335-387
 * A m x K u32 reps (row-major), x K reps; outputs (either may be NULL):
 * y_rep m reps, y_coeff m x k coefficient bytes.  m = 1 is a long fgdp_dot
 * split over the whole device. */
QPK_API qpk_status qpk_gfq_gemv(qpk_field f, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                                uint32_t* y_rep, uint8_t* y_coeff, void* stream);
QPK_API qpk_status qpk_gfq_gemv_host(qpk_field f, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                                     uint32_t* y_rep, uint8_t* y_coeff, qpk_cost* cost);

/* ------------------------------------- seeded synthetic inputs (rng.hpp) */
/* out[i] = SplitMix64(seed): draw number start+i+1, mod bound (below()) */
QPK_API qpk_status qpk_gen_draws(uint64_t seed, uint64_t start, uint64_t count, uint32_t bound, uint8_t* out,
                                 void* stream);
/* out[i] = word first+i, word w = sum_j below(q) * q^(d-j) over draws
 * w*(d+1)+1 .. (first draw = top digit; the acceptance suite's
 * random_digit_safe_word, acceptance.cpp:52-56) */
QPK_API qpk_status qpk_gen_words(uint64_t seed, uint64_t first, uint64_t n, uint64_t q, uint32_t d, double* out,
                                 void* stream);
/* record pairs: a[i] = draws 2k*i+1..2k*i+k, b[i] = the next k, each below(bound) */
QPK_API qpk_status qpk_gen_pairs(uint64_t seed, uint64_t n, uint32_t k, uint32_t bound, uint8_t* a, uint8_t* b,
                                 void* stream);

/* ---------------------------------------------------------- measurement */
/* fp64 peak probe: which 0 = DFMA chains, 1 = DMMA (mma.sync f64) chains;
 * returns achieved TFLOP/s (CUDA events, after a warm-up launch) */
QPK_API qpk_status qpk_probe_fp64(int which, int iters, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* QPACK_B200_H */
