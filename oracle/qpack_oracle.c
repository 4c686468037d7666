/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * q-adic pipeline (arXiv 0710.0510; reference library `qpack`).
 *
 * This is the CHECKER for the CUDA product path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It is written for clarity, not speed (scalar, u128), except
 * that the matrix product can split output rows across pthreads.
 *
 * Each function cites the reference file:line whose behaviour it restates
 * (paths relative to /root/reference/proj).  Pinned by tests/test_oracle.py
 * against the reference's own known-answer vectors and against the unmodified
 * reference built in oracle/_ref/.
 */
#include "qpack_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef qo_u128 u128;

static __thread char g_err[256];

static int err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* qo_last_error(void) { return g_err; }

static int is_pow2(u128 v) { return v != 0 && (v & (v - 1)) == 0; }

static unsigned bitlen(u128 v) {
    unsigned n = 0;
    while (v) {
        v >>= 1;
        ++n;
    }
    return n;
}

/* v^e < 2^128 ? (common.cpp:43-49) */
static int pow_fits(u128 v, unsigned e, u128* out) {
    u128 r = 1;
    for (unsigned i = 0; i < e; ++i) {
        if (v != 0 && r > (~(u128)0) / v) return 0;
        r *= v;
    }
    if (out) *out = r;
    return 1;
}

/* ------------------------------------------------------------------ rng */
/* rng.hpp:17-22: state += gamma, then the splitmix64 finaliser.  The n-th
 * call therefore returns mix(seed + n*gamma); rng.hpp:25 below(n) = next % n. */
u64 qo_splitmix_at(u64 seed, u64 j) {
    u64 z = seed + j * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void qo_draws_u8(u64 seed, u64 start, u64 count, u64 bound, uint8_t* out) {
    for (u64 i = 0; i < count; ++i) out[i] = (uint8_t)(qo_splitmix_at(seed, start + i + 1) % bound);
}

/* --------------------------------------------------------------- fpdiv */
/* 256-bit little-endian helpers for the exact Lemma-1 bound. */
typedef struct {
    u64 w[5];
} big;

static big big_mul_u64(big a, u64 m) {
    big r;
    u128 c = 0;
    for (int i = 0; i < 5; ++i) {
        u128 s = (u128)a.w[i] * m + c;
        r.w[i] = (u64)s;
        c = s >> 64;
    }
    return r;
}

static big big_add(big a, big b) {
    big r;
    u128 c = 0;
    for (int i = 0; i < 5; ++i) {
        u128 s = (u128)a.w[i] + b.w[i] + c;
        r.w[i] = (u64)s;
        c = s >> 64;
    }
    return r;
}

static big big_shl(u64 v, unsigned sh) { /* v * 2^sh, sh < 256 */
    big r;
    memset(&r, 0, sizeof r);
    unsigned limb = sh / 64, off = sh % 64;
    r.w[limb] = v << off;
    if (off && limb + 1 < 5) r.w[limb + 1] = v >> (64 - off);
    return r;
}

static int big_lt_pow2(big a, unsigned bits) { /* a < 2^bits */
    for (int i = 4; i >= 0; --i) {
        unsigned lo = 64u * (unsigned)i;
        if (bits <= lo) {
            if (a.w[i]) return 0;
        } else if (bits < lo + 64) {
            return (a.w[i] >> (bits - lo)) == 0;
        } else {
            return 1;
        }
    }
    return 1;
}

/* fpdiv.cpp:53-97 — largest r with r*(2e+e^2) < 1, exactly.  With
 * e = mant/2^s the condition is r*mant*(2^(s+1)+mant) < 2^(2s); the answer
 * is found by bisection on r. */
int qo_premul_floor_bound(double eps, u64* out) {
    if (!(eps > 0.0) || !(eps < 1.0)) return err(QO_DOMAIN, "premul_floor_bound: epsilon must be in (0, 1)");
    int e2 = 0;
    double f = frexp(eps, &e2);
    u64 mant = (u64)ldexp(f, 53);
    unsigned s = (unsigned)(53 - e2);
    if (s > 120) {
        *out = ~(u64)0;
        return QO_OK;
    }
    /* denom = mant*2^(s+1) + mant^2 */
    big m2;
    memset(&m2, 0, sizeof m2);
    u128 sq = (u128)mant * mant;
    m2.w[0] = (u64)sq;
    m2.w[1] = (u64)(sq >> 64);
    big denom = big_add(big_shl(mant, s + 1), m2);
    u64 lo = 0, hi = ~(u64)0;
    if (big_lt_pow2(big_mul_u64(denom, hi), 2 * s)) {
        *out = hi;
        return QO_OK;
    }
    while (lo + 1 < hi) { /* invariant: lo ok, hi not ok */
        u64 mid = lo + (hi - lo) / 2;
        if (big_lt_pow2(big_mul_u64(denom, mid), 2 * s))
            lo = mid;
        else
            hi = mid;
    }
    *out = lo;
    return QO_OK;
}

/* fpdiv.cpp:99-123 — RN(1/p), bumped one ulp up unless already >= 1/p
 * (exact comparison mant*p >= 2^(53-e2)); r_max = bound(3*2^-53). */
int qo_reciprocal(u64 p, double* inv_up, u64* r_max) {
    if (p == 0) return err(QO_DOMAIN, "ReciprocalDivisor: divisor must be positive");
    if (p >= ((u64)1 << 53)) return err(QO_DOMAIN, "ReciprocalDivisor: divisor exceeds exact double range");
    double z = 1.0 / (double)p;
    int e2 = 0;
    double f = frexp(z, &e2);
    u64 mant = (u64)ldexp(f, 53);
    unsigned sh = (unsigned)(53 - e2);
    int ge = sh <= 127 ? ((u128)mant * p >= ((u128)1 << sh)) : 0;
    *inv_up = ge ? z : nextafter(z, INFINITY);
    return qo_premul_floor_bound(3.0 * 0x1p-53, r_max);
}

/* fpdiv.cpp:132-139 */
int qo_floor_div_premul(u64 r, double inv_up, u64 r_max, u64* out) {
    if (r > r_max) return err(QO_OUT_OF_RANGE, "floor_div_premul: numerator exceeds guaranteed range r_max");
    double t = (double)r * inv_up;
    *out = (u64)nextafter(t, INFINITY);
    return QO_OK;
}

/* -------------------------------------------------------------- params */
/* params.cpp:36-42 */
int qo_is_prime(u64 n) {
    if (n < 2) return 0;
    if (n % 2 == 0) return n == 2;
    for (u64 d = 3; d * d <= n; d += 2)
        if (n % d == 0) return 0;
    return 1;
}

static u128 digit_load(u64 p, u32 k, u32 n_q) { return (u128)(p - 1) * (p - 1) * k * n_q; }

/* q^(2k-1) < 2^m (params.cpp:21-26) */
static int word_ok(u64 q, u32 k, u32 m) {
    u128 v;
    if (!pow_fits(q, 2 * k - 1, &v)) return 0;
    if (m >= 128) return 1;
    return v < ((u128)1 << m);
}

/* params.cpp:42-59: 0 = ok, 1 non_prime, 2 q_too_small, 3 word_overflow,
 * 4 q_unrepresentable (ParamViolation order, params.hpp:39-45). */
int qo_validate(u64 p, u64 q, u32 k, u32 n_q, u32 m) {
    if (!p || !q || !k || !n_q || !m) return -err(QO_INVALID_ARGUMENT, "validate: all parameters must be positive");
    if (!qo_is_prime(p)) return 1;
    if (bitlen(q) > m) return 4;
    if ((u128)q <= digit_load(p, k, n_q)) return 2;
    if (!word_ok(q, k, m)) return 3;
    return 0;
}

/* params.cpp:103-116 with prefer_power_of_two = true: smallest 2^b above
 * the one-product digit load, n_q the largest count that q still clears. */
int qo_qadic_for_degree(u64 p, u32 d, u32 m, u64* q_out, u32* k_out, u32* nq_out) {
    if (m != 24 && m != 53 && m != 64 && m != 128) return err(QO_INVALID_ARGUMENT, "m must be one of 24, 53, 64, 128");
    u32 k = d + 1;
    u128 load = digit_load(p, k, 1);
    unsigned b = bitlen(load);
    if (b >= 64 || b + 1 > m) return err(QO_DOMAIN, "qadic_for_degree: degree does not fit");
    u64 q = (u64)1 << b;
    if (!word_ok(q, k, m)) return err(QO_DOMAIN, "qadic_for_degree: degree does not fit");
    u64 n_q = (u64)((q - 1) / load);
    if (qo_validate(p, q, k, (u32)n_q, m) != 0) return err(QO_DOMAIN, "qadic_for_degree: invalid params");
    *q_out = q;
    *k_out = k;
    *nq_out = (u32)n_q;
    return QO_OK;
}

/* ---------------------------------------------------------------- REDQ */
/* redq.cpp:115-146 */
int qo_redq_plan_build(u64 p, u64 q, u32 d, int float_mode, qo_redq_plan* pl) {
    memset(pl, 0, sizeof *pl);
    if (p < 2) return err(QO_INVALID_ARGUMENT, "RedqPlan: p must be >= 2");
    if (q < 2) return err(QO_INVALID_ARGUMENT, "RedqPlan: q must be >= 2");
    if (d + 1 > QO_MAX_DIGITS || !pow_fits(q, d, NULL))
        return err(QO_INVALID_ARGUMENT, "RedqPlan: q^d exceeds 128 bits; no word holds d+1 digits");
    pl->p = p;
    pl->q = q;
    pl->d = d;
    pl->float_mode = float_mode;
    pl->neg_q = (p - q % p) % p;
    u128 pw = 1;
    for (u32 i = 0; i <= d; ++i) {
        pl->qpow[i] = pw;
        if (i < d) pw *= q;
    }
    int rc = qo_reciprocal(p, &pl->inv_p, &pl->r_max);
    if (rc) return rc;
    if (float_mode) {
        u128 top;
        if (!pow_fits(q, d + 1, &top) || top - 1 > pl->r_max)
            return err(QO_INVALID_ARGUMENT, "RedqPlan: float mode needs q^(d+1)-1 <= r_max");
        for (u32 i = 0; i <= d; ++i) {
            u64 rm;
            rc = qo_reciprocal((u64)pl->qpow[i], &pl->inv_qpow[i], &rm);
            if (rc) return rc;
        }
    }
    return QO_OK;
}

/* redq.cpp:203-245: entry for tuple (u_0..u_{w-1}) packs
 * (mu_0..mu_{w-1}) base radix, mu_j = u_j + neg_q*u_{j+1} mod p (j<w-1),
 * mu_{w-1} = u_{w-1}; tuples index base radix as well. */
int qo_correction_table(u64 p, u64 q, u32 w, int binary_shift, u64 max_entries, u64** entries, u64* n,
                        u64* radix_out) {
    if (p < 2) return err(QO_INVALID_ARGUMENT, "build_correction_table: p must be >= 2");
    if (w < 2) return err(QO_INVALID_ARGUMENT, "build_correction_table: window must cover >= 2 digits");
    u64 radix = p;
    if (binary_shift) {
        unsigned c = 0;
        while (((u64)1 << c) < p) ++c;
        radix = (u64)1 << c;
    }
    u128 size;
    if (!pow_fits(radix, w, &size) || size > max_entries)
        return err(QO_LENGTH, "build_correction_table: table exceeds the entry budget");
    if (bitlen(size) > 63) return err(QO_LENGTH, "build_correction_table: packed window exceeds 63 bits");
    u64* t = (u64*)calloc((size_t)size, sizeof(u64));
    u64 neg_q = (p - q % p) % p;
    u64 tup[64] = {0};
    for (;;) {
        u64 idx = 0, ent = 0, sc = 1;
        for (u32 j = 0; j < w; ++j) {
            u64 mu = (j + 1 < w) ? (tup[j] + neg_q * tup[j + 1]) % p : tup[j];
            idx += tup[j] * sc;
            ent += mu * sc;
            sc *= radix;
        }
        t[idx] = ent;
        u32 j = 0;
        while (j < w && ++tup[j] == p) tup[j++] = 0;
        if (j == w) break;
    }
    *entries = t;
    *n = (u64)size;
    *radix_out = radix;
    return QO_OK;
}

int qo_redq_attach_table(qo_redq_plan* pl, u32 w, int binary_shift) {
    u64* e;
    u64 n, radix;
    int rc = qo_correction_table(pl->p, pl->q, w, binary_shift, (u64)1 << 26, &e, &n, &radix);
    if (rc) return rc;
    free(pl->entries);
    pl->entries = e;
    pl->n_entries = n;
    pl->radix = radix;
    pl->window = w;
    return QO_OK;
}

void qo_redq_plan_free(qo_redq_plan* pl) {
    free(pl->entries);
    pl->entries = NULL;
}

/* redq.cpp:22-100 + 162-170: check r < q^(d+1); rop = floor(r/p) (float:
 * premultiplied reciprocal; integer: u128 division); raw digits
 * u_i = floor(r/q^i) - p*floor(rop/q^i); then the ascending correction,
 * either direct or through the windowed table. */
int qo_redq_word(const qo_redq_plan* pl, u128 r, u64* u_out, u64* mu) {
    const u32 d = pl->d, nd = d + 1;
    const int p2 = is_pow2(pl->q);
    const unsigned b = p2 ? bitlen(pl->q) - 1 : 0;
    u128 top = p2 ? (r >> (b * d)) : r / pl->qpow[d];
    if (top >= pl->q) return err(QO_DOMAIN, "redq: input exceeds q^(d+1), digits are not all below q");
    u64 u[QO_MAX_DIGITS];
    if (pl->float_mode) {
        u64 r64 = (u64)r, rop, x, y;
        int rc = qo_floor_div_premul(r64, pl->inv_p, pl->r_max, &rop);
        if (rc) return rc;
        for (u32 i = 0; i < nd; ++i) {
            if ((rc = qo_floor_div_premul(r64, pl->inv_qpow[i], pl->r_max, &x))) return rc;
            if ((rc = qo_floor_div_premul(rop, pl->inv_qpow[i], pl->r_max, &y))) return rc;
            u[i] = x - pl->p * y;
        }
    } else {
        u128 rop = r / pl->p;
        for (u32 i = 0; i < nd; ++i) {
            u128 x = p2 ? (r >> (b * i)) : r / pl->qpow[i];
            u128 y = p2 ? (rop >> (b * i)) : rop / pl->qpow[i];
            u[i] = (u64)(x - (u128)pl->p * y);
        }
    }
    if (u_out) memcpy(u_out, u, nd * sizeof(u64));
    memcpy(mu, u, nd * sizeof(u64));
    if (pl->neg_q == 0 || d == 0) return QO_OK;
    if (!pl->entries) {
        for (u32 i = 0; i < d; ++i) mu[i] = (mu[i] + pl->neg_q * mu[i + 1]) % pl->p;
        return QO_OK;
    }
    const u32 w = pl->window;
    const u32 acc = (d + w - 2) / (w - 1);
    for (u32 a = 0; a < acc; ++a) {
        u32 s = a * (w - 1);
        u64 idx = 0, sc = 1;
        for (u32 j = 0; j < w; ++j) {
            idx += (s + j <= d ? mu[s + j] : 0) * sc;
            sc *= pl->radix;
        }
        u64 ent = pl->entries[idx];
        for (u32 j = 0; j < w && s + j <= d; ++j) {
            u64 m = ent % pl->radix;
            ent /= pl->radix;
            if (j + 1 < w || s + j == d) mu[s + j] = m;
        }
    }
    return QO_OK;
}

static int f64_to_word(double x, u128* r) {
    if (!(x >= 0.0) || x >= 9007199254740992.0 || x != floor(x))
        return err(QO_DOMAIN, "redq: word is not an exact non-negative integer double");
    *r = (u128)(u64)x;
    return QO_OK;
}

int qo_redq_batch_f64(const qo_redq_plan* pl, const double* words, u64 n, uint8_t* out) {
    u64 mu[QO_MAX_DIGITS];
    const u32 nd = pl->d + 1;
    for (u64 i = 0; i < n; ++i) {
        u128 r;
        int rc = f64_to_word(words[i], &r);
        if (rc) return rc;
        if ((rc = qo_redq_word(pl, r, NULL, mu))) return rc;
        for (u32 j = 0; j < nd; ++j) out[i * nd + j] = (uint8_t)mu[j];
    }
    return QO_OK;
}

int qo_redq_run_f64(u64 p, u64 q, u32 d, int float_mode, u32 window, int binary_shift, const double* words, u64 n,
                    uint8_t* out) {
    qo_redq_plan pl;
    int rc = qo_redq_plan_build(p, q, d, float_mode, &pl);
    if (!rc && window) rc = qo_redq_attach_table(&pl, window, binary_shift);
    if (!rc) rc = qo_redq_batch_f64(&pl, words, n, out);
    qo_redq_plan_free(&pl);
    return rc;
}

int qo_redq_run_u64(u64 p, u64 q, u32 d, int float_mode, u32 window, int binary_shift, const u64* words, u64 n,
                    u64* out) {
    qo_redq_plan pl;
    int rc = qo_redq_plan_build(p, q, d, float_mode, &pl);
    if (!rc && window) rc = qo_redq_attach_table(&pl, window, binary_shift);
    for (u64 i = 0; !rc && i < n; ++i) rc = qo_redq_word(&pl, words[i], NULL, out + i * (d + 1));
    qo_redq_plan_free(&pl);
    return rc;
}

/* the same over u128 words given as (lo, hi) u64 pairs */
int qo_redq_run_u128(u64 p, u64 q, u32 d, int float_mode, u32 window, int binary_shift, const u64* words, u64 n,
                     u64* out) {
    qo_redq_plan pl;
    int rc = qo_redq_plan_build(p, q, d, float_mode, &pl);
    if (!rc && window) rc = qo_redq_attach_table(&pl, window, binary_shift);
    for (u64 i = 0; !rc && i < n; ++i)
        rc = qo_redq_word(&pl, ((u128)words[2 * i + 1] << 64) | words[2 * i], NULL, out + i * (d + 1));
    qo_redq_plan_free(&pl);
    return rc;
}

/* ------------------------------------------------------------ DQT / FQT */
/* polymul.cpp:18-23: largest window w in 4..2 with p^w <= 2^20 */
static u32 choose_window(u64 p) {
    for (u32 w = 4; w >= 2; --w) {
        u128 v;
        if (pow_fits(p, w, &v) && v <= ((u128)1 << 20)) return w;
    }
    return 0;
}

/* dqt.cpp:23-37: sum c_i q^i (shifts when q = 2^b) */
static u128 pack_digits(const u64* c, u32 n, u64 q) {
    u128 v = 0;
    for (u32 i = n; i-- > 0;) v = v * q + c[i];
    return v;
}

/* polymul.cpp:81-147 — chunked FQT product.  Chunks of d+1 coefficients,
 * padded chunk span 2*Dq+1 on both sides, u128 accumulation of up to n_q
 * chunk products per group, one REDQ(d'=2d) per group with the plan of
 * fqt_reduction_plan (polymul.cpp:67-74: integer mode, windowed table when
 * p does not divide q), overlap-add of the residues mod p. */
int qo_fqt_mul(u64 p, u32 d, u64 q, u32 n_q, const u64* a, u64 la, const u64* b, u64 lb, u64* out, u64* cost) {
    return qo_fqt_mul_m(p, d, q, n_q, 53, a, la, b, lb, out, cost);
}

/* fqt_mul with word width m (u128 words up to m = 128, polymul.cpp u128 MAC) */
int qo_fqt_mul_m(u64 p, u32 d, u64 q, u32 n_q, u32 m, const u64* a, u64 la, const u64* b, u64 lb, u64* out,
                 u64* cost) {
    if (qo_validate(p, q, d + 1, n_q, m) != 0) return err(QO_INVALID_ARGUMENT, "fqt_mul: invalid params");
    if (la == 0 || lb == 0) return QO_OK;
    qo_redq_plan pl;
    int rc = qo_redq_plan_build(p, q, 2 * d, 0, &pl);
    if (rc) return rc;
    if (pl.neg_q) {
        u32 w = choose_window(p);
        if (w && (rc = qo_redq_attach_table(&pl, w, 0))) return rc;
    }
    u64 nmax = (la > lb ? la : lb) - 1;
    u64 dq = (nmax + 1 + d) / (d + 1) - 1;
    u64 span = 2 * dq + 1;
    u128* pw = (u128*)calloc(span, sizeof(u128));
    u128* qw = (u128*)calloc(span, sizeof(u128));
    u64 tmp[64];
    for (u64 c = 0; c * (d + 1) < la; ++c) {
        for (u32 j = 0; j <= d; ++j) tmp[j] = c * (d + 1) + j < la ? a[c * (d + 1) + j] % p : 0;
        pw[c] = pack_digits(tmp, d + 1, q);
    }
    for (u64 c = 0; c * (d + 1) < lb; ++c) {
        for (u32 j = 0; j <= d; ++j) tmp[j] = c * (d + 1) + j < lb ? b[c * (d + 1) + j] % p : 0;
        qw[c] = pack_digits(tmp, d + 1, q);
    }
    u64 lout = la + lb - 1;
    memset(out, 0, lout * sizeof(u64));
    u64 groups = (span + n_q - 1) / n_q;
    u64 mu[QO_MAX_DIGITS];
    for (u64 t = 0; t < span && !rc; ++t) {
        for (u64 g = 0; g < groups && !rc; ++g) {
            u64 lo = g * n_q, hi = lo + n_q < span ? lo + n_q : span;
            u128 acc = 0;
            for (u64 i = lo; i < hi; ++i) {
                acc += pw[i] * ((t >= i && t - i < span) ? qw[t - i] : 0);
                if (cost) cost[0] += 1;
            }
            rc = qo_redq_word(&pl, acc, NULL, mu);
            if (cost) {
                cost[1] += 1;
                cost[3] += 1;
                if (pl.entries && 2 * d > 0) cost[2] += (2 * d + pl.window - 2) / (pl.window - 1);
            }
            for (u32 j = 0; j <= 2 * d; ++j) {
                u64 idx = t * (d + 1) + j;
                if (idx < lout) out[idx] = (out[idx] + mu[j]) % p;
            }
        }
    }
    free(pw);
    free(qw);
    qo_redq_plan_free(&pl);
    return rc;
}

/* Batched single-chunk products (config 1): params = qadic_for_degree(p,d,53),
 * pairs of degree-<=d polynomials → 2d+1 residues each. */
int qo_polymul_batch(u64 p, u32 d, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out) {
    u64 q;
    u32 k, n_q;
    int rc = qo_qadic_for_degree(p, d, 53, &q, &k, &n_q);
    if (rc) return rc;
    u64 ca[64], cb[64], r[130];
    for (u64 i = 0; i < n; ++i) {
        for (u32 j = 0; j < k; ++j) {
            ca[j] = a[i * k + j];
            cb[j] = b[i * k + j];
        }
        if ((rc = qo_fqt_mul(p, d, q, n_q, ca, k, cb, k, r, NULL))) return rc;
        for (u32 j = 0; j < 2 * d + 1; ++j) out[i * (2 * d + 1) + j] = (uint8_t)r[j];
    }
    return QO_OK;
}

/* ------------------------------------------------------------- GF(p^k) */
static void idx_to_coeffs(u64 idx, u32 k, u64 p, u64* c) {
    for (u32 i = 0; i < k; ++i) {
        c[i] = idx % p;
        idx /= p;
    }
}

static u64 coeffs_to_idx(const u64* c, u32 n, u64 p) {
    u64 v = 0;
    for (u32 i = n; i-- > 0;) v = v * p + c[i] % p;
    return v;
}

/* remainder of a (len la, in place) by the monic polynomial m of degree k;
 * returns the new length (<= k).  Same long division as gfq.cpp:55-69. */
static u32 prem(u64* a, u32 la, const u64* m, u32 k, u64 p) {
    while (la > k) {
        u64 lead = a[la - 1];
        u32 sh = la - 1 - k;
        if (lead)
            for (u32 i = 0; i < k; ++i) a[sh + i] = (a[sh + i] + p - (lead * m[i]) % p) % p;
        --la;
    }
    return la;
}

/* product mod the modulus (gfq.cpp:32-52), result padded to k coeffs */
static void pmulmod(const u64* a, const u64* b, const u64* m, u32 k, u64 p, u64* out) {
    u64 prod[66] = {0};
    for (u32 i = 0; i < k; ++i)
        for (u32 j = 0; j < k; ++j) prod[i + j] = (prod[i + j] + a[i] * b[j]) % p;
    u32 l = prem(prod, 2 * k - 1, m, k, p);
    for (u32 i = 0; i < k; ++i) out[i] = i < l ? prod[i] : 0;
}

/* gfq.cpp:76-89: trial division by every monic polynomial of degree 1..k/2 */
static int irreducible(const u64* poly, u32 k, u64 p) {
    if (k == 1) return 1;
    for (u32 t = 1; 2 * t <= k; ++t) {
        u64 cnt = 1;
        for (u32 i = 0; i < t; ++i) cnt *= p;
        for (u64 idx = 0; idx < cnt; ++idx) {
            u64 dv[33], a[33];
            idx_to_coeffs(idx, t, p, dv);
            dv[t] = 1;
            memcpy(a, poly, (k + 1) * sizeof(u64));
            u32 l = prem(a, k + 1, dv, t, p);
            int zero = 1;
            for (u32 i = 0; i < l; ++i) zero &= a[i] == 0;
            if (zero) return 0;
        }
    }
    return 1;
}

static void ppow(const u64* base, u64 e, const u64* m, u32 k, u64 p, u64* out) {
    u64 r[33] = {0}, b[33];
    r[0] = 1 % p;
    memcpy(b, base, k * sizeof(u64));
    while (e) {
        if (e & 1) pmulmod(r, b, m, k, p, r);
        pmulmod(b, b, m, k, p, b);
        e >>= 1;
    }
    memcpy(out, r, k * sizeof(u64));
}

/* gfq.cpp:132-258 */
qo_field* qo_field_build(u64 p, u32 k, u64 q, int binary_shift) {
    if (!qo_is_prime(p)) {
        err(QO_DOMAIN, "GfqField: p is not prime");
        return NULL;
    }
    if (k == 0 || k > 32) {
        err(QO_INVALID_ARGUMENT, "GfqField: bad k");
        return NULL;
    }
    u128 order;
    if (!pow_fits(p, k, &order) || order > ((u128)1 << 20)) {
        err(QO_LENGTH, "GfqField: table budget exceeded");
        return NULL;
    }
    qo_field* f = (qo_field*)calloc(1, sizeof *f);
    f->p = p;
    f->k = k;
    f->q = q;
    f->order = (u64)order;
    f->group = f->order - 1;
    f->binary_shift = binary_shift;
    u128 unit = (u128)(p - 1) * (p - 1) * k;
    u128 nq = (q - 1) / unit;
    if (nq > ((u128)1 << 30)) nq = (u128)1 << 30;
    f->n_q = (u32)nq;
    if (f->n_q == 0 || qo_validate(p, q, k, f->n_q, 53) != 0) {
        err(QO_DOMAIN, "GfqField: q fails the packing bounds");
        free(f);
        return NULL;
    }
    /* smallest monic irreducible in index order */
    int found = 0;
    for (u64 idx = 0; idx < f->order && !found; ++idx) {
        idx_to_coeffs(idx, k, p, f->modulus);
        f->modulus[k] = 1;
        found = irreducible(f->modulus, k, p);
    }
    /* smallest primitive element: g^(group/f) != 1 for each prime f */
    u64 fac[64], nf = 0, g = f->group;
    for (u64 dd = 2; dd * dd <= g; ++dd)
        if (g % dd == 0) {
            fac[nf++] = dd;
            while (g % dd == 0) g /= dd;
        }
    if (g > 1) fac[nf++] = g;
    for (u64 idx = 1; idx < f->order && !f->generator_index; ++idx) {
        u64 c[33], r[33];
        idx_to_coeffs(idx, k, p, c);
        int ok = 1;
        for (u64 i = 0; i < nf && ok; ++i) {
            ppow(c, f->group / fac[i], f->modulus, k, p, r);
            int one = r[0] == 1;
            for (u32 j = 1; j < k; ++j) one &= r[j] == 0;
            if (one) ok = 0;
        }
        if (ok) f->generator_index = idx;
    }
    const u32 sentinel = (u32)f->group;
    f->log = (u32*)malloc(f->order * sizeof(u32));
    f->antilog = (u64*)calloc(f->order, sizeof(u64));
    f->fval = (double*)calloc(f->order, sizeof(double));
    f->plus1 = (u32*)malloc(f->order * sizeof(u32));
    for (u64 i = 0; i < f->order; ++i) f->log[i] = sentinel;
    u64 gc[33], cur[33] = {0};
    idx_to_coeffs(f->generator_index, k, p, gc);
    cur[0] = 1 % p;
    for (u64 e = 0; e < f->group; ++e) {
        u64 idx = coeffs_to_idx(cur, k, p);
        f->antilog[e] = idx;
        f->log[idx] = (u32)e;
        double v = 0.0;
        for (u32 i = k; i-- > 0;) v = v * (double)q + (double)cur[i];
        f->fval[e] = v;
        pmulmod(cur, gc, f->modulus, k, p, cur);
    }
    f->fval[sentinel] = 0.0;
    /* Zech / plus-one: rep of (g^e + 1); entry `sentinel` is rep of 1 */
    for (u64 e = 0; e <= f->group; ++e) {
        u64 idx = e == f->group ? 0 : f->antilog[e];
        u64 c0 = idx % p;
        f->plus1[e] = f->log[idx - c0 + (c0 + 1) % p];
    }
    /* L/H half-window tables (Theorem 3): tuple (u_0..u_{k-1}) indexed base
     * lh_radix; L gives the rep of the corrected low half, H the rep of the
     * corrected high half shifted up by k-1 and reduced by the modulus. */
    u64 lh = p;
    if (binary_shift) {
        unsigned c = 0;
        while (((u64)1 << c) < p) ++c;
        lh = (u64)1 << c;
    }
    f->lh_radix = lh;
    u128 lsz = 0;
    pow_fits(lh, k, &lsz);
    f->lh_size = (u64)lsz;
    f->ltab = (u32*)malloc(f->lh_size * sizeof(u32));
    f->htab = (u32*)malloc(f->lh_size * sizeof(u32));
    for (u64 i = 0; i < f->lh_size; ++i) f->ltab[i] = f->htab[i] = sentinel;
    u64 neg_q = (p - q % p) % p;
    u64 tup[33] = {0};
    for (;;) {
        u64 idx = 0, sc = 1;
        for (u32 j = 0; j < k; ++j) {
            idx += tup[j] * sc;
            sc *= lh;
        }
        u64 low[66] = {0}, high[66] = {0};
        for (u32 i = 0; i + 1 < k; ++i) low[i] = high[k - 1 + i] = (tup[i] + neg_q * tup[i + 1]) % p;
        high[2 * k - 2] = tup[k - 1];
        u32 ll = k >= 2 ? k - 1 : 1;
        f->ltab[idx] = f->log[coeffs_to_idx(low, prem(low, ll, f->modulus, k, p), p)];
        f->htab[idx] = f->log[coeffs_to_idx(high, prem(high, 2 * k - 1, f->modulus, k, p), p)];
        u32 j = 0;
        while (j < k && ++tup[j] == p) tup[j++] = 0;
        if (j == k) break;
    }
    qo_reciprocal(p, &f->inv_p, &f->r_max);
    return f;
}

void qo_field_free(qo_field* f) {
    if (!f) return;
    free(f->log);
    free(f->antilog);
    free(f->fval);
    free(f->plus1);
    free(f->ltab);
    free(f->htab);
    free(f);
}

/* gfq.cpp:260-264 */
uint32_t qo_field_mul(const qo_field* f, u32 a, u32 b) {
    if (a == f->group || b == f->group) return (u32)f->group;
    return (u32)(((u64)a + b) % f->group);
}

/* gfq.cpp:266-275 (Zech addition) */
uint32_t qo_field_add(const qo_field* f, u32 a, u32 b) {
    if (a == f->group) return b;
    if (b == f->group) return a;
    u64 diff = ((u64)b + f->group - a) % f->group;
    u32 t = f->plus1[diff];
    if (t == f->group) return (u32)f->group;
    return (u32)(((u64)a + t) % f->group);
}

/* gfq.cpp:335-387 (paper Alg. 4).  v2 is read with stride `stride2` so a
 * column of a row-major matrix can be passed without a gather. */
uint32_t qo_fgdp_dot(const qo_field* f, const u32* v1, const u32* v2, u64 n, u64 stride2, u64* cost) {
    const u64 p = f->p;
    const u32 k = f->k;
    const int p2 = is_pow2(f->q);
    const unsigned b = p2 ? bitlen(f->q) - 1 : 0;
    u32 result = (u32)f->group;
    for (u64 lo = 0; lo < n; lo += f->n_q) {
        u64 hi = lo + f->n_q < n ? lo + f->n_q : n;
        double acc = 0.0;
        for (u64 i = lo; i < hi; ++i) acc += f->fval[v1[i]] * f->fval[v2[i * stride2]];
        u64 r = (u64)acc, rop;
        if (r <= f->r_max)
            qo_floor_div_premul(r, f->inv_p, f->r_max, &rop);
        else
            rop = r / p;
        u64 u[66];
        u64 qp = 1;
        for (u32 i = 0; i < 2 * k - 1; ++i) {
            u64 x = p2 ? r >> (b * i) : r / qp;
            u64 y = p2 ? rop >> (b * i) : rop / qp;
            u[i] = x - p * y;
            if (!p2) qp *= f->q;
        }
        u64 il = 0, ih = 0, sc = 1;
        for (u32 i = 0; i < k; ++i) {
            il += u[i] * sc;
            ih += u[k - 1 + i] * sc;
            sc *= f->lh_radix;
        }
        u32 g = qo_field_add(f, f->htab[ih], f->ltab[il]);
        result = qo_field_add(f, result, g);
        if (cost) {
            cost[0] += hi - lo;
            cost[1] += 1;
            cost[3] += 1;
        }
    }
    return result;
}

uint32_t qo_rep_from_bytes(const qo_field* f, const uint8_t* c) {
    u64 idx = 0;
    for (u32 i = f->k; i-- > 0;) idx = idx * f->p + c[i];
    return f->log[idx];
}

void qo_rep_to_bytes(const qo_field* f, u32 rep, uint8_t* c) {
    u64 idx = rep == f->group ? 0 : f->antilog[rep];
    for (u32 i = 0; i < f->k; ++i) {
        c[i] = (uint8_t)(idx % f->p);
        idx /= f->p;
    }
}

int qo_gfq_mul_batch(const qo_field* f, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, int algo) {
    const u32 k = f->k;
    for (u64 i = 0; i < n; ++i) {
        u32 ra = qo_rep_from_bytes(f, a + i * k), rb = qo_rep_from_bytes(f, b + i * k);
        u32 rc = algo == 0 ? qo_fgdp_dot(f, &ra, &rb, 1, 1, NULL) : qo_field_mul(f, ra, rb);
        qo_rep_to_bytes(f, rc, out + i * k);
    }
    return QO_OK;
}

typedef struct {
    const qo_field* f;
    const u32 *ra, *rbt;
    u64 K, n, lo, hi;
    uint8_t* C;
} mm_job;

static void* mm_worker(void* arg) {
    mm_job* j = (mm_job*)arg;
    for (u64 i = j->lo; i < j->hi; ++i)
        for (u64 c = 0; c < j->n; ++c)
            qo_rep_to_bytes(j->f, qo_fgdp_dot(j->f, j->ra + i * j->K, j->rbt + c * j->K, j->K, 1, NULL),
                            j->C + (i * j->n + c) * j->f->k);
    return NULL;
}

/* gfq.cpp:389-404: every C[i][j] is one fgdp_dot of row i and column j;
 * B is transposed once so columns are contiguous. */
int qo_gfq_matmul(const qo_field* f, const uint8_t* A, const uint8_t* B, u64 m, u64 K, u64 n, u64 row_lo,
                  u64 row_hi, uint8_t* C, int threads) {
    if (row_hi > m || row_lo > row_hi) return err(QO_INVALID_ARGUMENT, "gfq_matmul: bad row range");
    const u32 k = f->k;
    u32* ra = (u32*)malloc((m ? m : 1) * (K ? K : 1) * sizeof(u32));
    u32* rbt = (u32*)malloc((n ? n : 1) * (K ? K : 1) * sizeof(u32));
    for (u64 i = row_lo; i < row_hi; ++i)
        for (u64 l = 0; l < K; ++l) ra[i * K + l] = qo_rep_from_bytes(f, A + (i * K + l) * k);
    for (u64 l = 0; l < K; ++l)
        for (u64 c = 0; c < n; ++c) rbt[c * K + l] = qo_rep_from_bytes(f, B + (l * n + c) * k);
    if (threads < 1) threads = 1;
    pthread_t th[256];
    mm_job jobs[256];
    if (threads > 256) threads = 256;
    u64 rows = row_hi - row_lo;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (mm_job){f, ra, rbt, K, n, row_lo + rows * t / threads, row_lo + rows * (t + 1) / threads, C};
        pthread_create(&th[t], NULL, mm_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(ra);
    free(rbt);
    return QO_OK;
}

/* Freivalds' check in the coefficient domain: y = C x and z = A (B x),
 * products accumulated as unreduced integer coefficient sums, reduced by the
 * modulus at the end.  Independent of the table machinery above. */
static void gf_matvec(const qo_field* f, const uint8_t* M, u64 rows, u64 cols, const uint8_t* x, uint8_t* y) {
    const u32 k = f->k;
    const u64 p = f->p;
    u64* acc = (u64*)malloc((2 * k - 1) * sizeof(u64));
    for (u64 i = 0; i < rows; ++i) {
        memset(acc, 0, (2 * k - 1) * sizeof(u64));
        const uint8_t* row = M + i * cols * k;
        for (u64 j = 0; j < cols; ++j)
            for (u32 s = 0; s < k; ++s) {
                u64 a = row[j * k + s];
                if (!a) continue;
                for (u32 t = 0; t < k; ++t) acc[s + t] += a * x[j * k + t];
            }
        u64 red[66];
        for (u32 s = 0; s < 2 * k - 1; ++s) red[s] = acc[s] % p;
        u32 l = prem(red, 2 * k - 1, f->modulus, k, p);
        for (u32 s = 0; s < k; ++s) y[i * k + s] = (uint8_t)(s < l ? red[s] : 0);
    }
    free(acc);
}

int qo_gfq_freivalds(const qo_field* f, const uint8_t* A, const uint8_t* B, const uint8_t* C, u64 m, u64 K, u64 n,
                     u64 seed, int trials) {
    const u32 k = f->k;
    uint8_t* x = (uint8_t*)malloc(n * k);
    uint8_t* bx = (uint8_t*)malloc(K * k);
    uint8_t* abx = (uint8_t*)malloc(m * k);
    uint8_t* cx = (uint8_t*)malloc(m * k);
    int ok = 1;
    for (int t = 0; t < trials && ok; ++t) {
        qo_draws_u8(seed + (u64)t, 0, n * k, f->p, x);
        gf_matvec(f, B, K, n, x, bx);
        gf_matvec(f, A, m, K, bx, abx);
        gf_matvec(f, C, m, n, x, cx);
        ok = memcmp(abx, cx, m * k) == 0;
    }
    free(x);
    free(bx);
    free(abx);
    free(cx);
    return ok;
}

/* -------------------------------------------------------- naive oracles */
/* oracle.cpp:144-163 */
int qo_poly_mod(const u64* a, u64 la, const u64* modulus, u32 k, u64 p, u64* out) {
    u64* r = (u64*)malloc((la + k + 1) * sizeof(u64));
    for (u64 i = 0; i < la; ++i) r[i] = a[i] % p;
    u32 l = la > k ? prem(r, (u32)la, modulus, k, p) : (u32)la;
    for (u32 i = 0; i < k; ++i) out[i] = i < l ? r[i] : 0;
    free(r);
    return QO_OK;
}

/* oracle.cpp:165-182: schoolbook products reduced by the modulus, summed */
int qo_naive_gfq_dot(const u64* v1, const u64* v2, u64 n, u32 k, const u64* modulus, u64 p, u64* out) {
    memset(out, 0, k * sizeof(u64));
    for (u64 t = 0; t < n; ++t) {
        u64 prod[66] = {0}, red[33];
        for (u32 i = 0; i < k; ++i)
            for (u32 j = 0; j < k; ++j) prod[i + j] = (prod[i + j] + (v1[t * k + i] % p) * (v2[t * k + j] % p)) % p;
        qo_poly_mod(prod, 2 * k - 1, modulus, k, p, red);
        for (u32 i = 0; i < k; ++i) out[i] = (out[i] + red[i]) % p;
    }
    return QO_OK;
}

/* ------------------------------------------------------------- checksum */
/* common.cpp:51-61: FNV-1a over the 8 little-endian bytes of each value.
 * Byte inputs are promoted to u64; `state` chains calls (start with
 * 0xcbf29ce484222325). */
u64 qo_fold_checksum_u8(const uint8_t* data, u64 n, u64 h) {
    /* the seven zero high bytes only multiply: fold them into P^8 */
    u64 p8 = 1;
    for (int b = 0; b < 8; ++b) p8 *= 0x100000001b3ULL;
    for (u64 i = 0; i < n; ++i) h = (h ^ data[i]) * p8;
    return h;
}

u64 qo_fold_checksum_u64(const u64* data, u64 n) {
    u64 h = 0xcbf29ce484222325ULL;
    for (u64 i = 0; i < n; ++i)
        for (int b = 0; b < 8; ++b) {
            h ^= (data[i] >> (8 * b)) & 0xff;
            h *= 0x100000001b3ULL;
        }
    return h;
}

/* redq_trace (redq.cpp:184-195) for u128 words given as two halves, integer
 * mode plan (p, q, d) without table: rop, raw digits u, residues mu. */
int qo_redq_trace(u64 p, u64 q, u32 d, u64 r_lo, u64 r_hi, u64* rop_lo, u64* rop_hi, u64* u, u64* mu) {
    qo_redq_plan pl;
    int rc = qo_redq_plan_build(p, q, d, 0, &pl);
    if (rc) return rc;
    u128 r = ((u128)r_hi << 64) | r_lo;
    u128 rop = r / p;
    *rop_lo = (u64)rop;
    *rop_hi = (u64)(rop >> 64);
    rc = qo_redq_word(&pl, r, u, mu);
    qo_redq_plan_free(&pl);
    return rc;
}
