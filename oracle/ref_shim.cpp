// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" batch drivers around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp compiled with -Dqpack=qpack_ref by
// oracle/Makefile into oracle/_ref/libqpack_ref.so).  The reference API is
// per-word / per-pair scalar C++; these loops drive it exactly the way the
// reference's own acceptance suite does (proj/tests/acceptance.cpp:46-56)
// and the survey's CPU-baseline protocol prescribes: inputs
// are converted before the clock starts, each thread owns a contiguous index
// range, its own CostReport and its own output slice.
//
// Used by: tests/ (golden generation and parity), bench.py --impl reference
// and bench.py's cpu_baseline leg.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "qpack/dqt.hpp"
#include "qpack/fpdiv.hpp"
#include "qpack/gfq.hpp"
#include "qpack/oracle.hpp"
#include "qpack/params.hpp"
#include "qpack/polymul.hpp"
#include "qpack/redq.hpp"
#include "qpack/rng.hpp"

using namespace qpack;  // renamed to qpack_ref by the build

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::domain_error*>(&e)) return 2;
    if (dynamic_cast<const std::length_error*>(&e)) return 3;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 4;
    if (dynamic_cast<const std::overflow_error*>(&e)) return 5;
    if (dynamic_cast<const std::runtime_error*>(&e)) return 6;
    if (dynamic_cast<const std::logic_error*>(&e)) return 7;
    return 6;
}

using Clock = std::chrono::steady_clock;

// Run body(lo, hi, cost) over [0, n) on `threads` workers; returns ns of the
// parallel region and the summed counters.
template <typename Body>
uint64_t run_split(uint64_t n, int threads, uint64_t* cost_out, Body body) {
    if (threads < 1) threads = 1;
    if (static_cast<uint64_t>(threads) > n && n > 0) threads = static_cast<int>(n);
    std::vector<CostReport> costs(threads);
    std::vector<std::exception_ptr> errs(threads);
    auto t0 = Clock::now();
    if (threads == 1) {
        body(0, n, costs[0]);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            uint64_t lo = n * t / threads, hi = n * (t + 1) / threads;
            pool.emplace_back([&, t, lo, hi] {
                try {
                    body(lo, hi, costs[t]);
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
    }
    auto t1 = Clock::now();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    if (cost_out) {
        CostReport tot;
        for (auto& c : costs) tot += c;
        cost_out[0] = tot.mul_add;
        cost_out[1] = tot.divisions;
        cost_out[2] = tot.table_accesses;
        cost_out[3] = tot.reduction_calls;
    }
    return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
}

struct FieldBox {
    GfqField f;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- inputs
// Sequential draws from the reference generator (rng.hpp:13-31):
// out[j] = SplitMix64(seed).below(bound) for the (j+1)-th call.
int ref_draws_u8(uint64_t seed, uint64_t count, uint64_t bound, uint8_t* out) {
    SplitMix64 rng(seed);
    for (uint64_t j = 0; j < count; ++j) out[j] = static_cast<uint8_t>(rng.below(bound));
    return 0;
}

uint64_t ref_splitmix_next(uint64_t seed, uint64_t skip) {
    SplitMix64 rng(seed);
    for (uint64_t j = 0; j < skip; ++j) rng.next();
    return rng.next();
}

// ---------------------------------------------------------------- fpdiv
int ref_reciprocal(uint64_t p, double* inv_up, uint64_t* r_max) {
    try {
        ReciprocalDivisor d = ReciprocalDivisor::make(p);
        *inv_up = d.inv_up;
        *r_max = d.r_max;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_premul_floor_bound(double eps, uint64_t* out) {
    try {
        *out = premul_floor_bound(eps);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_floor_div_premul(uint64_t r, uint64_t p, uint64_t* out) {
    try {
        *out = floor_div_premul(r, ReciprocalDivisor::make(p));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- params
int ref_qadic_for_degree(uint64_t p, uint32_t d, uint32_t m, uint64_t* q, uint32_t* k, uint32_t* n_q) {
    try {
        QadicParams pr = qadic_for_degree(p, d, m);
        *q = pr.q;
        *k = pr.k;
        *n_q = pr.n_q;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_validate(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, uint32_t m) {
    try {
        return static_cast<int>(validate(p, q, k, n_q, m).violation) + 100;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- REDQ
// Correction table entries (build_correction_table, redq.cpp:203-245).
int ref_correction_table(uint64_t p, uint64_t q, uint32_t w, int indexing, uint64_t* out, uint64_t cap,
                         uint64_t* n_out, uint64_t* radix) {
    try {
        CorrectionTable t = build_correction_table(p, q, w, static_cast<TableIndexing>(indexing));
        *n_out = t.entries.size();
        *radix = t.radix;
        if (out) std::memcpy(out, t.entries.data(), std::min<uint64_t>(cap, t.entries.size()) * 8);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// REDQ over a batch of words given as exact doubles (the survey's C2 input).
// mode 0 = RedqMode::integer, 1 = RedqMode::float_premul; window 0 = direct
// correction, else attach build_correction_table(p,q,window,indexing).
int ref_redq_batch(uint64_t p, uint64_t q, uint32_t d, int mode, uint32_t window, int indexing,
                   const double* words, uint64_t n, uint8_t* out, int threads, uint64_t* ns,
                   uint64_t* cost) {
    try {
        RedqPlan plan = RedqPlan::build(p, q, d, mode ? RedqMode::float_premul : RedqMode::integer);
        if (window) plan.attach_correction(build_correction_table(p, q, window, static_cast<TableIndexing>(indexing)));
        const unsigned nd = d + 1;
        // input conversion outside the clock: the reference takes u128 words
        std::vector<u128> w(n);
        for (uint64_t i = 0; i < n; ++i) w[i] = static_cast<u128>(static_cast<uint64_t>(words[i]));
        uint64_t t = run_split(n, threads, cost, [&](uint64_t lo, uint64_t hi, CostReport& c) {
            std::vector<u64> mu;
            for (uint64_t i = lo; i < hi; ++i) {
                redq_residues_into(w[i], plan, mu, &c);
                for (unsigned j = 0; j < nd; ++j) out[i * nd + j] = static_cast<uint8_t>(mu[j]);
            }
        });
        if (ns) *ns = t;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// u64-word variant with u64 residues (wide primes), integer/float mode.
int ref_redq_batch_u64(uint64_t p, uint64_t q, uint32_t d, int mode, uint32_t window, int indexing,
                       const uint64_t* words, uint64_t n, uint64_t* out) {
    try {
        RedqPlan plan = RedqPlan::build(p, q, d, mode ? RedqMode::float_premul : RedqMode::integer);
        if (window) plan.attach_correction(build_correction_table(p, q, window, static_cast<TableIndexing>(indexing)));
        std::vector<u64> mu;
        for (uint64_t i = 0; i < n; ++i) {
            redq_residues_into(static_cast<u128>(words[i]), plan, mu);
            for (unsigned j = 0; j <= d; ++j) out[i * (d + 1) + j] = mu[j];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// redq_trace (redq.cpp:184-195) for the worked examples; u128 words as two u64 halves.
int ref_redq_trace(uint64_t p, uint64_t q, uint32_t d, uint64_t r_lo, uint64_t r_hi, uint64_t* rop_lo,
                   uint64_t* rop_hi, uint64_t* u, uint64_t* mu, uint64_t* word_lo, uint64_t* word_hi) {
    try {
        RedqPlan plan = RedqPlan::build(p, q, d);
        u128 r = (static_cast<u128>(r_hi) << 64) | r_lo;
        RedqTrace t = redq_trace(r, plan);
        *rop_lo = static_cast<uint64_t>(t.rop);
        *rop_hi = static_cast<uint64_t>(t.rop >> 64);
        for (unsigned i = 0; i <= d; ++i) {
            u[i] = t.u[i];
            mu[i] = t.mu[i];
        }
        *word_lo = static_cast<uint64_t>(t.word);
        *word_hi = static_cast<uint64_t>(t.word >> 64);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- C1
// Batched small polynomial products over F_p: a, b are n x (d+1) coefficient
// records, out is n x (2d+1).  algo 0 = fqt_mul with qadic_for_degree(p,d,53)
// and a prebuilt fqt_reduction_plan; algo 1 = dqt_mul_poly.
int ref_polymul_batch(uint64_t p, uint32_t d, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                      int algo, int threads, uint64_t* ns, uint64_t* cost) {
    try {
        QadicParams params = qadic_for_degree(p, d, 53);
        RedqPlan plan = fqt_reduction_plan(params, d);
        const unsigned k = d + 1, ko = 2 * d + 1;
        std::vector<DensePoly> pa(n), pb(n);
        for (uint64_t i = 0; i < n; ++i) {
            pa[i] = DensePoly{p, std::vector<u64>(a + i * k, a + i * k + k)};
            pb[i] = DensePoly{p, std::vector<u64>(b + i * k, b + i * k + k)};
        }
        uint64_t t = run_split(n, threads, cost, [&](uint64_t lo, uint64_t hi, CostReport& c) {
            for (uint64_t i = lo; i < hi; ++i) {
                DensePoly r = algo == 0 ? fqt_mul(pa[i], pb[i], d, params, plan, &c)
                                        : dqt_mul_poly(pa[i], pb[i], params);
                for (unsigned j = 0; j < ko; ++j) out[i * ko + j] = static_cast<uint8_t>(j < r.coeffs.size() ? r.coeffs[j] : 0);
            }
        });
        if (ns) *ns = t;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// General fqt_mul on one pair of polynomials (any length), for chunked-FQT parity.
int ref_fqt_mul_m(uint64_t p, uint32_t d, uint64_t q, uint32_t n_q, uint32_t m, const uint64_t* a, uint64_t la,
                  const uint64_t* b, uint64_t lb, uint64_t* out, uint64_t* cost);

int ref_fqt_mul(uint64_t p, uint32_t d, uint64_t q, uint32_t n_q, const uint64_t* a, uint64_t la,
                const uint64_t* b, uint64_t lb, uint64_t* out, uint64_t* cost) {
    return ref_fqt_mul_m(p, d, q, n_q, 53, a, la, b, lb, out, cost);
}

// fqt_mul with word width m (the reference's u128 words up to m = 128)
int ref_fqt_mul_m(uint64_t p, uint32_t d, uint64_t q, uint32_t n_q, uint32_t m, const uint64_t* a, uint64_t la,
                  const uint64_t* b, uint64_t lb, uint64_t* out, uint64_t* cost) {
    try {
        QadicParams params{p, q, d + 1, n_q, m};
        DensePoly pa{p, std::vector<u64>(a, a + la)}, pb{p, std::vector<u64>(b, b + lb)};
        CostReport c;
        DensePoly r = fqt_mul(pa, pb, d, params, &c);
        for (uint64_t i = 0; i < r.coeffs.size(); ++i) out[i] = r.coeffs[i];
        if (cost) {
            cost[0] = c.mul_add;
            cost[1] = c.divisions;
            cost[2] = c.table_accesses;
            cost[3] = c.reduction_calls;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---------------------------------------------------------------- GF(p^k)
void* ref_field_build(uint64_t p, uint32_t k, uint64_t q, int indexing) {
    try {
        return new FieldBox{GfqField::build(p, k, q, static_cast<TableIndexing>(indexing))};
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_field_free(void* h) { delete static_cast<FieldBox*>(h); }

// Public field description: modulus (k+1 coeffs), generator coeffs (k),
// n_q, memory_entries, and the describe() text.
int ref_field_info(void* h, uint64_t* modulus, uint64_t* generator, uint32_t* n_q, uint64_t* mem_entries,
                   char* text, uint64_t text_cap) {
    const GfqField& f = static_cast<FieldBox*>(h)->f;
    for (size_t i = 0; i < f.modulus_poly().size(); ++i) modulus[i] = f.modulus_poly()[i];
    std::vector<u64> g = f.to_coeffs(f.generator());
    for (size_t i = 0; i < g.size(); ++i) generator[i] = g[i];
    *n_q = f.params().n_q;
    *mem_entries = f.memory_entries();
    std::string s = f.describe();
    if (text && text_cap) {
        std::size_t m = std::min<std::size_t>(text_cap - 1, s.size());
        std::memcpy(text, s.data(), m);
        text[m] = 0;
    }
    return 0;
}

// Per-rep tables through the public API: antilog index (to_index), float_eval.
int ref_field_tables(void* h, uint64_t* to_index, double* float_eval, uint32_t* from_index) {
    const GfqField& f = static_cast<FieldBox*>(h)->f;
    for (u64 r = 0; r < f.order(); ++r) {
        to_index[r] = f.to_index(GfqElt{static_cast<u32>(r)});
        float_eval[r] = f.float_eval(GfqElt{static_cast<u32>(r)});
        from_index[r] = f.from_index(r).rep;
    }
    return 0;
}

// Field ops on reps: op 0 mul, 1 add, 2 neg, 3 inverse.
int ref_field_op(void* h, int op, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out) {
    try {
        const GfqField& f = static_cast<FieldBox*>(h)->f;
        for (uint64_t i = 0; i < n; ++i) {
            GfqElt x{a[i]}, y{b ? b[i] : 0};
            GfqElt r = op == 0 ? f.mul(x, y) : op == 1 ? f.add(x, y) : op == 2 ? f.neg(x) : f.inverse(x);
            out[i] = r.rep;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

namespace {
inline GfqElt elt_from_bytes(const GfqField& f, const uint8_t* c, uint32_t k) {
    u64 idx = 0;
    for (uint32_t i = k; i-- > 0;) idx = idx * f.p() + c[i];
    return f.from_index(idx);
}
inline void elt_to_bytes(const GfqField& f, GfqElt e, uint8_t* c, uint32_t k) {
    u64 idx = f.to_index(e);
    for (uint32_t i = 0; i < k; ++i) {
        c[i] = static_cast<uint8_t>(idx % f.p());
        idx /= f.p();
    }
}
}  // namespace

// Elementwise GF(p^k) product of coefficient records (n x k uint8 each).
// algo 0 = fgdp_dot on length-1 vectors (DQT/REDQ/L-H path, gfq.cpp:335-387),
// algo 1 = GfqField::mul (dlog/Zech path, gfq.cpp:260-264).
int ref_gfq_mul_batch(void* h, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out, int algo,
                      int threads, uint64_t* ns, uint64_t* cost) {
    try {
        const GfqField& f = static_cast<FieldBox*>(h)->f;
        const uint32_t k = f.k();
        std::vector<GfqElt> ea(n), eb(n), ec(n);
        for (uint64_t i = 0; i < n; ++i) {
            ea[i] = elt_from_bytes(f, a + i * k, k);
            eb[i] = elt_from_bytes(f, b + i * k, k);
        }
        uint64_t t = run_split(n, threads, cost, [&](uint64_t lo, uint64_t hi, CostReport& c) {
            for (uint64_t i = lo; i < hi; ++i) {
                if (algo == 0)
                    ec[i] = fgdp_dot(std::span<const GfqElt>(&ea[i], 1), std::span<const GfqElt>(&eb[i], 1), f, &c);
                else
                    ec[i] = f.mul(ea[i], eb[i]);
            }
        });
        for (uint64_t i = 0; i < n; ++i) elt_to_bytes(f, ec[i], out + i * k, k);
        if (ns) *ns = t;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// C = A*B over GF(p^k), coefficient records.  A is m x K x k, B is K x n x k,
// C is m x n x k (uint8).  Only output rows [row_lo, row_hi) are computed.
// algo 0 = gfq_matmul as shipped (gfq.cpp:389-404) on row slabs;
// algo 1 = fgdp_dot over a pre-transposed B (same arithmetic, no strided
// gather; the survey's fast golden path).
int ref_gfq_matmul(void* h, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K, uint64_t n,
                   uint64_t row_lo, uint64_t row_hi, uint8_t* C, int algo, int threads, uint64_t* ns,
                   uint64_t* cost) {
    try {
        const GfqField& f = static_cast<FieldBox*>(h)->f;
        const uint32_t k = f.k();
        if (row_hi > m || row_lo > row_hi) throw std::invalid_argument("ref_gfq_matmul: bad row range");
        uint64_t rows = row_hi - row_lo;
        GfqMatrix a{rows, K, std::vector<GfqElt>(rows * K)};
        for (uint64_t i = 0; i < rows; ++i)
            for (uint64_t l = 0; l < K; ++l) a.data[i * K + l] = elt_from_bytes(f, A + ((row_lo + i) * K + l) * k, k);
        GfqMatrix b{K, n, std::vector<GfqElt>(K * n)};
        for (uint64_t l = 0; l < K * n; ++l) b.data[l] = elt_from_bytes(f, B + l * k, k);
        std::vector<GfqElt> bt;
        if (algo == 1) {
            bt.resize(K * n);
            for (uint64_t l = 0; l < K; ++l)
                for (uint64_t j = 0; j < n; ++j) bt[j * K + l] = b.data[l * n + j];
        }
        std::vector<GfqElt> c(rows * n);
        uint64_t t = run_split(rows, threads, cost, [&](uint64_t lo, uint64_t hi, CostReport& cr) {
            if (algo == 0) {
                GfqMatrix slab{hi - lo, K, std::vector<GfqElt>(a.data.begin() + lo * K, a.data.begin() + hi * K)};
                GfqMatrix r = gfq_matmul(slab, b, f, &cr);
                std::copy(r.data.begin(), r.data.end(), c.begin() + lo * n);
            } else {
                for (uint64_t i = lo; i < hi; ++i)
                    for (uint64_t j = 0; j < n; ++j)
                        c[i * n + j] = fgdp_dot(std::span<const GfqElt>(&a.data[i * K], K),
                                                std::span<const GfqElt>(&bt[j * K], K), f, &cr);
            }
        });
        for (uint64_t i = 0; i < rows * n; ++i) elt_to_bytes(f, c[i], C + (row_lo * n + i) * k, k);
        if (ns) *ns = t;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Reference-API gfq_matmul directly on reps (GfqMatrix of GfqElt), m x K by K x n.
int ref_gfq_matmul_rep(void* h, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K, uint64_t n,
                       uint32_t* C, uint64_t* cost) {
    try {
        const GfqField& f = static_cast<FieldBox*>(h)->f;
        GfqMatrix a{m, K, std::vector<GfqElt>(m * K)}, b{K, n, std::vector<GfqElt>(K * n)};
        for (uint64_t i = 0; i < m * K; ++i) a.data[i] = GfqElt{A[i]};
        for (uint64_t i = 0; i < K * n; ++i) b.data[i] = GfqElt{B[i]};
        CostReport cr;
        GfqMatrix r = gfq_matmul(a, b, f, &cr);
        for (uint64_t i = 0; i < m * n; ++i) C[i] = r.data[i].rep;
        if (cost) {
            cost[0] = cr.mul_add;
            cost[1] = cr.divisions;
            cost[2] = cr.table_accesses;
            cost[3] = cr.reduction_calls;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// fgdp_dot on reps (one dot product), for dot/GEMV parity.
int ref_fgdp_dot(void* h, const uint32_t* v1, const uint32_t* v2, uint64_t n, uint32_t* out, uint64_t* cost) {
    try {
        const GfqField& f = static_cast<FieldBox*>(h)->f;
        std::vector<GfqElt> a(n), b(n);
        for (uint64_t i = 0; i < n; ++i) {
            a[i] = GfqElt{v1[i]};
            b[i] = GfqElt{v2[i]};
        }
        CostReport cr;
        *out = fgdp_dot(a, b, f, &cr).rep;
        if (cost) {
            cost[0] = cr.mul_add;
            cost[1] = cr.divisions;
            cost[2] = cr.table_accesses;
            cost[3] = cr.reduction_calls;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// FNV-1a fold exactly as the reference computes it (common.cpp:51-61); used
// to pin the oracle's streaming checksum restatement.
uint64_t ref_fold_checksum(const uint64_t* data, uint64_t n) { return fold_checksum(data, n); }

}  // extern "C"
