/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference algorithms.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load this
 * library, and only as the checker.  The product (libqpack_b200.so) never
 * links or calls it.
 *
 * Parity pinning: every function here is checked in tests/test_oracle.py
 * against (a) the known-answer vectors of the reference's own tests
 * (proj/tests/acceptance.cpp, proj/tests/test_*.cpp; values cited there) and
 * (b) the unmodified reference compiled into oracle/_ref/libqpack_ref.so.
 */
#ifndef QPACK_ORACLE_H
#define QPACK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned __int128 qo_u128;

/* status codes match include/qpack_b200.h's qpk_status */
enum {
    QO_OK = 0,
    QO_INVALID_ARGUMENT = 1,
    QO_DOMAIN = 2,
    QO_LENGTH = 3,
    QO_OUT_OF_RANGE = 4,
    QO_OVERFLOW = 5,
    QO_RUNTIME = 6,
    QO_LOGIC = 7
};

const char* qo_last_error(void);

/* ---- SplitMix64 (rng.hpp:13-31), counter-addressed ---- */
uint64_t qo_splitmix_at(uint64_t seed, uint64_t j); /* j-th output, 1-based */
void qo_draws_u8(uint64_t seed, uint64_t start, uint64_t count, uint64_t bound, uint8_t* out);

/* ---- fpdiv (fpdiv.cpp) ---- */
int qo_premul_floor_bound(double eps, uint64_t* out);
int qo_reciprocal(uint64_t p, double* inv_up, uint64_t* r_max);
int qo_floor_div_premul(uint64_t r, double inv_up, uint64_t r_max, uint64_t* out);

/* ---- params (params.cpp) ---- */
int qo_is_prime(uint64_t n);
int qo_validate(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, uint32_t m); /* 0 ok, 1..4 violation, <0 error */
int qo_qadic_for_degree(uint64_t p, uint32_t d, uint32_t m, uint64_t* q, uint32_t* k, uint32_t* n_q);

/* ---- REDQ (redq.cpp) ---- */
#define QO_MAX_DIGITS 64
typedef struct {
    uint64_t p, q;
    uint32_t d;
    int float_mode;
    uint64_t neg_q;
    qo_u128 qpow[QO_MAX_DIGITS];
    double inv_p;
    uint64_t r_max;
    double inv_qpow[QO_MAX_DIGITS];
    /* optional correction table */
    uint32_t window;
    uint64_t radix;
    uint64_t n_entries;
    uint64_t* entries;
} qo_redq_plan;

int qo_redq_plan_build(uint64_t p, uint64_t q, uint32_t d, int float_mode, qo_redq_plan* plan);
int qo_correction_table(uint64_t p, uint64_t q, uint32_t w, int binary_shift, uint64_t max_entries,
                        uint64_t** entries, uint64_t* n, uint64_t* radix);
int qo_redq_attach_table(qo_redq_plan* plan, uint32_t w, int binary_shift);
void qo_redq_plan_free(qo_redq_plan* plan);
/* u: raw digits (may be NULL), mu: residues; d+1 each */
int qo_redq_word(const qo_redq_plan* plan, qo_u128 r, uint64_t* u, uint64_t* mu);
int qo_redq_batch_f64(const qo_redq_plan* plan, const double* words, uint64_t n, uint8_t* out);
/* convenience: build plan + run, for ctypes */
int qo_redq_run_f64(uint64_t p, uint64_t q, uint32_t d, int float_mode, uint32_t window, int binary_shift,
                    const double* words, uint64_t n, uint8_t* out);
int qo_redq_trace(uint64_t p, uint64_t q, uint32_t d, uint64_t r_lo, uint64_t r_hi, uint64_t* rop_lo,
                  uint64_t* rop_hi, uint64_t* u, uint64_t* mu);
int qo_redq_run_u64(uint64_t p, uint64_t q, uint32_t d, int float_mode, uint32_t window, int binary_shift,
                    const uint64_t* words, uint64_t n, uint64_t* out);
int qo_redq_run_u128(uint64_t p, uint64_t q, uint32_t d, int float_mode, uint32_t window, int binary_shift,
                     const uint64_t* words, uint64_t n, uint64_t* out);

/* ---- DQT + FQT (dqt.cpp, polymul.cpp) ---- */
int qo_polymul_batch(uint64_t p, uint32_t d, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out);
int qo_fqt_mul(uint64_t p, uint32_t d, uint64_t q, uint32_t n_q, const uint64_t* a, uint64_t la,
               const uint64_t* b, uint64_t lb, uint64_t* out, uint64_t* cost);
/* the same with the word width m (u128 words up to m = 128) */
int qo_fqt_mul_m(uint64_t p, uint32_t d, uint64_t q, uint32_t n_q, uint32_t m, const uint64_t* a, uint64_t la,
                 const uint64_t* b, uint64_t lb, uint64_t* out, uint64_t* cost);

/* ---- GF(p^k) (gfq.cpp) ---- */
typedef struct {
    uint64_t p, q, order, group, lh_radix, lh_size;
    uint32_t k, n_q;
    int binary_shift;
    uint64_t modulus[33];
    uint64_t generator_index;
    uint32_t* log;      /* poly index -> rep */
    uint64_t* antilog;  /* rep -> poly index */
    uint32_t* plus1;
    double* fval;
    uint32_t* ltab;
    uint32_t* htab;
    double inv_p;
    uint64_t r_max;
} qo_field;

qo_field* qo_field_build(uint64_t p, uint32_t k, uint64_t q, int binary_shift);
void qo_field_free(qo_field* f);
uint32_t qo_field_mul(const qo_field* f, uint32_t a, uint32_t b);
uint32_t qo_field_add(const qo_field* f, uint32_t a, uint32_t b);
uint32_t qo_fgdp_dot(const qo_field* f, const uint32_t* v1, const uint32_t* v2, uint64_t n, uint64_t stride2,
                     uint64_t* cost);
uint32_t qo_rep_from_bytes(const qo_field* f, const uint8_t* c);
void qo_rep_to_bytes(const qo_field* f, uint32_t rep, uint8_t* c);
/* algo 0 = fgdp_dot length 1; 1 = dlog mul */
int qo_gfq_mul_batch(const qo_field* f, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out, int algo);
/* C rows [row_lo,row_hi) of A(m x K) * B(K x n), coefficient records; threads >= 1 */
int qo_gfq_matmul(const qo_field* f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K, uint64_t n,
                  uint64_t row_lo, uint64_t row_hi, uint8_t* C, int threads);
/* Freivalds: returns 1 if C*x == A*(B*x) for `trials` random x (seeded), 0 otherwise */
int qo_gfq_freivalds(const qo_field* f, const uint8_t* A, const uint8_t* B, const uint8_t* C, uint64_t m,
                     uint64_t K, uint64_t n, uint64_t seed, int trials);

/* ---- naive oracles (oracle.cpp) ---- */
int qo_poly_mod(const uint64_t* a, uint64_t la, const uint64_t* modulus, uint32_t k, uint64_t p, uint64_t* out);
int qo_naive_gfq_dot(const uint64_t* v1, const uint64_t* v2, uint64_t n, uint32_t k, const uint64_t* modulus,
                     uint64_t p, uint64_t* out);

/* ---- checksum (common.cpp:51-61), streaming over bytes promoted to u64 ---- */
uint64_t qo_fold_checksum_u8(const uint8_t* data, uint64_t n, uint64_t state);
uint64_t qo_fold_checksum_u64(const uint64_t* data, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
