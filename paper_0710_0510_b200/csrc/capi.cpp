// extern "C" boundary of libqpack_b200.so: thin wrappers that translate the
// C++ exceptions of the host library / GPU layer into qpk_status codes.
#include "qpack_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "host/device_state.hpp"
#include "host/gpu_internal.hpp"
#include "kernels.hpp"
#include "qpack/gfq.hpp"
#include "qpack/polymul.hpp"
#include "qpack/redq.hpp"

struct qpk_redq_plan_s {
    qpack::RedqPlan plan;
};
struct qpk_polymul_plan_s {
    std::unique_ptr<qpack::gpu::PolymulPlan> pl;
};
struct qpk_field_s {
    qpack::GfqField f;
};

namespace {

thread_local std::string g_msg;

qpk_status fail(qpk_status st, const char* what) {
    g_msg = what;
    return st;
}

template <class Fn>
qpk_status guard(Fn&& fn) {
    try {
        fn();
        g_msg.clear();
        return QPK_OK;
    } catch (const qpack::gpu::device_error& e) {
        return fail(QPK_ERR_CUDA, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(QPK_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::domain_error& e) {
        return fail(QPK_ERR_DOMAIN, e.what());
    } catch (const std::length_error& e) {
        return fail(QPK_ERR_LENGTH, e.what());
    } catch (const std::out_of_range& e) {
        return fail(QPK_ERR_OUT_OF_RANGE, e.what());
    } catch (const std::overflow_error& e) {
        return fail(QPK_ERR_OVERFLOW, e.what());
    } catch (const std::logic_error& e) {
        return fail(QPK_ERR_LOGIC, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(QPK_ERR_RUNTIME, "out of host memory");
    } catch (const std::exception& e) {
        return fail(QPK_ERR_RUNTIME, e.what());
    }
}

void need(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void put_cost(qpk_cost* out, const qpack::CostReport& c) {
    if (!out) return;
    out->mul_add = c.mul_add;
    out->divisions = c.divisions;
    out->table_accesses = c.table_accesses;
    out->reduction_calls = c.reduction_calls;
}

}  // namespace

extern "C" {

const char* qpk_last_error(void) { return g_msg.c_str(); }

int qpk_abi_version(void) { return QPK_ABI_VERSION; }

qpk_status qpk_device_info(int* sms, int* cc_major, int* cc_minor) {
    return guard([&] {
        qpack::gpu::require_device();
        int dev = 0;
        qpack::gpu::check(cudaGetDevice(&dev), "cudaGetDevice");
        if (sms) qpack::gpu::check(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev), "attr");
        if (cc_major) qpack::gpu::check(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev), "attr");
        if (cc_minor) qpack::gpu::check(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev), "attr");
    });
}

// ------------------------------------------------------------------ REDQ
qpk_status qpk_redq_plan_create(uint64_t p, uint64_t q, uint32_t d, int mode, qpk_redq_plan* out) {
    return guard([&] {
        need(out != nullptr, "qpk_redq_plan_create: null output handle");
        auto h = std::make_unique<qpk_redq_plan_s>();
        h->plan = qpack::RedqPlan::build(p, q, d, mode ? qpack::RedqMode::float_premul : qpack::RedqMode::integer);
        *out = h.release();
    });
}

qpk_status qpk_redq_plan_attach_table(qpk_redq_plan plan, uint32_t window, int indexing) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(indexing == 0 || indexing == 1, "indexing must be 0 (base_p) or 1 (binary_shift)");
        plan->plan.attach_correction(qpack::build_correction_table(
            plan->plan.p, plan->plan.q, window, static_cast<qpack::TableIndexing>(indexing)));
    });
}

qpk_status qpk_redq_plan_attach_table_bytes(qpk_redq_plan plan, const uint8_t* qpkt, uint64_t len) {
    return guard([&] {
        need(plan != nullptr && (qpkt != nullptr || len == 0), "null argument");
        std::istringstream in(std::string(reinterpret_cast<const char*>(qpkt), len));
        plan->plan.attach_correction(qpack::load_correction_table(in));
    });
}

void qpk_redq_plan_destroy(qpk_redq_plan plan) { delete plan; }

qpk_status qpk_redq_residues_f64(qpk_redq_plan plan, const double* words, uint64_t n, uint8_t* residues,
                                 void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        auto& dp = qpack::detail::device_plan(plan->plan);
        qpack::gpu::redq_device(dp, words, n, residues, as_stream(stream));
    });
}

qpk_status qpk_redq_residues_f64_host(qpk_redq_plan plan, const double* words, uint64_t n, uint8_t* residues,
                                      qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        qpack::gpu::redq_host(qpack::detail::device_plan(plan->plan), words, n, residues);
        put_cost(cost, qpack::detail::redq_batch_cost(plan->plan, n));
    });
}

qpk_status qpk_redq_residues_u64(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                 void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        auto& dp = qpack::detail::device_plan(plan->plan);
        qpack::gpu::redq_device_u64(dp, words, n, residues, as_stream(stream));
    });
}

qpk_status qpk_redq_residues_u64_host(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                      qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        qpack::gpu::redq_host_u64(qpack::detail::device_plan(plan->plan), words, n, residues);
        put_cost(cost, qpack::detail::redq_batch_cost(plan->plan, n));
    });
}

qpk_status qpk_redq_residues_u128(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                  void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        need(plan->plan.p <= 256, "residues are uint8: p must be <= 256");
        auto& dp = qpack::detail::device_plan(plan->plan);
        qpack::gpu::redq_device_u128(dp, words, n, residues, as_stream(stream));
    });
}

qpk_status qpk_redq_residues_u128_host(qpk_redq_plan plan, const uint64_t* words, uint64_t n, uint8_t* residues,
                                       qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (words && residues), "null buffer");
        need(plan->plan.p <= 256, "residues are uint8: p must be <= 256");
        qpack::gpu::redq_host_u128(qpack::detail::device_plan(plan->plan), words, n, residues);
        put_cost(cost, qpack::detail::redq_batch_cost(plan->plan, n));
    });
}

qpk_status qpk_redq_sync(qpk_redq_plan plan, void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        auto& dp = qpack::detail::device_plan(plan->plan);
        qpack::gpu::raise_status(qpack::gpu::take_status(dp, as_stream(stream)));
    });
}

qpk_status qpk_redq_cost(qpk_redq_plan plan, uint64_t n, qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr && cost != nullptr, "null argument");
        put_cost(cost, qpack::detail::redq_batch_cost(plan->plan, n));
    });
}

// --------------------------------------------------------------- polymul
qpk_status qpk_polymul_plan_create(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, qpk_polymul_plan* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        auto h = std::make_unique<qpk_polymul_plan_s>();
        h->pl = std::make_unique<qpack::gpu::PolymulPlan>(qpack::QadicParams{p, q, k, n_q, 53});
        *out = h.release();
    });
}

qpk_status qpk_polymul_plan_create_m(uint64_t p, uint64_t q, uint32_t k, uint32_t n_q, uint32_t m,
                                     qpk_polymul_plan* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        auto h = std::make_unique<qpk_polymul_plan_s>();
        h->pl = std::make_unique<qpack::gpu::PolymulPlan>(qpack::QadicParams{p, q, k, n_q, m});
        *out = h.release();
    });
}

void qpk_polymul_plan_destroy(qpk_polymul_plan plan) { delete plan; }

qpk_status qpk_fqt_mul(qpk_polymul_plan plan, const uint8_t* a, uint64_t na, const uint8_t* b, uint64_t nb,
                       uint8_t* out, void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(na == 0 || nb == 0 || (a && b && out), "null buffer");
        qpack::gpu::fqt_mul_device(plan->pl->redq, plan->pl->params, a, na, b, nb, out, as_stream(stream));
    });
}

qpk_status qpk_fqt_mul_host(qpk_polymul_plan plan, const uint8_t* a, uint64_t na, const uint8_t* b, uint64_t nb,
                            uint8_t* out, qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(na == 0 || nb == 0 || (a && b && out), "null buffer");
        qpack::gpu::fqt_mul_host(plan->pl->redq, plan->pl->params, a, na, b, nb, out);
        put_cost(cost, qpack::gpu::fqt_cost(plan->pl->redq, plan->pl->params, na, nb));
    });
}

qpk_status qpk_fqt_mul_u64(qpk_polymul_plan plan, const uint64_t* a, uint64_t na, const uint64_t* b, uint64_t nb,
                           uint64_t* out, void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(na == 0 || nb == 0 || (a && b && out), "null buffer");
        qpack::gpu::fqt_mul_device_u64(plan->pl->redq, plan->pl->params, a, na, b, nb, out, as_stream(stream));
    });
}

qpk_status qpk_fqt_mul_u64_host(qpk_polymul_plan plan, const uint64_t* a, uint64_t na, const uint64_t* b,
                                uint64_t nb, uint64_t* out, qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(na == 0 || nb == 0 || (a && b && out), "null buffer");
        qpack::gpu::fqt_mul_host_u64(plan->pl->redq, plan->pl->params, a, na, b, nb, out);
        put_cost(cost, qpack::gpu::fqt_cost(plan->pl->redq, plan->pl->params, na, nb));
    });
}

qpk_status qpk_polymul_batch(qpk_polymul_plan plan, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                             void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (a && b && out), "null buffer");
        qpack::gpu::polymul_device(*plan->pl, a, b, n, out, as_stream(stream));
    });
}

qpk_status qpk_polymul_batch_host(qpk_polymul_plan plan, const uint8_t* a, const uint8_t* b, uint64_t n,
                                  uint8_t* out, qpk_cost* cost) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        need(n == 0 || (a && b && out), "null buffer");
        qpack::gpu::polymul_host(*plan->pl, a, b, n, out);
        put_cost(cost, qpack::gpu::polymul_cost(*plan->pl, n));
    });
}

qpk_status qpk_polymul_sync(qpk_polymul_plan plan, void* stream) {
    return guard([&] {
        need(plan != nullptr, "null plan");
        auto& dp = qpack::detail::device_plan(plan->pl->redq);
        qpack::gpu::raise_status(qpack::gpu::take_status(dp, as_stream(stream)));
    });
}

// ------------------------------------------------------------------ field
qpk_status qpk_field_create(uint64_t p, uint32_t k, uint64_t q, int indexing, qpk_field* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        need(indexing == 0 || indexing == 1, "indexing must be 0 (base_p) or 1 (binary_shift)");
        auto h = std::make_unique<qpk_field_s>(
            qpk_field_s{qpack::GfqField::build(p, k, q, static_cast<qpack::TableIndexing>(indexing))});
        *out = h.release();
    });
}

void qpk_field_destroy(qpk_field f) { delete f; }

qpk_status qpk_field_info(qpk_field f, uint64_t* modulus, uint64_t* generator, uint32_t* n_q,
                          uint64_t* memory_entries) {
    return guard([&] {
        need(f != nullptr, "null field");
        const auto& F = f->f;
        if (modulus) std::memcpy(modulus, F.modulus_poly().data(), F.modulus_poly().size() * 8);
        if (generator) {
            const auto g = F.to_coeffs(F.generator());
            std::memcpy(generator, g.data(), g.size() * 8);
        }
        if (n_q) *n_q = F.params().n_q;
        if (memory_entries) *memory_entries = F.memory_entries();
    });
}

qpk_status qpk_field_describe(qpk_field f, char* buf, uint64_t cap) {
    return guard([&] {
        need(f != nullptr && buf != nullptr && cap > 0, "null argument");
        const std::string s = f->f.describe();
        const std::size_t m = std::min<std::size_t>(cap - 1, s.size());
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    });
}

qpk_status qpk_field_tables(qpk_field f, uint32_t* log, uint64_t* antilog, uint32_t* plus1, double* fval,
                            uint32_t* low, uint32_t* high) {
    return guard([&] {
        need(f != nullptr, "null field");
        using A = qpack::detail::FieldAccess;
        const auto& F = f->f;
        auto cp = [](auto* dst, const auto& v) {
            if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
        };
        cp(log, A::log(F));
        cp(antilog, A::antilog(F));
        cp(plus1, A::zech(F));
        cp(fval, A::fval(F));
        cp(low, A::low(F));
        cp(high, A::high(F));
    });
}

qpk_status qpk_field_op(qpk_field f, int op, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out) {
    return guard([&] {
        need(f != nullptr && (n == 0 || (a && out)), "null argument");
        need(op >= 0 && op <= 3, "op must be 0..3");
        need(op >= 2 || n == 0 || b != nullptr, "binary op needs b");
        const auto& F = f->f;
        // reps must name field elements (GfqElt contract): checked on the device
        qpack::gpu::gfq_rep_op_host(qpack::detail::device_field(F), F, op, a, op < 2 ? b : nullptr, n, out);
    });
}

qpk_status qpk_field_sync(qpk_field f, void* stream) {
    return guard([&] {
        need(f != nullptr, "null field");
        auto& F = qpack::detail::device_field(f->f);
        qpack::gpu::raise_field_status(qpack::gpu::take_field_status(F, as_stream(stream)));
    });
}

qpk_status qpk_field_op1(qpk_field f, int op, uint32_t a, uint32_t b, uint32_t* out) {
    return guard([&] {
        need(f != nullptr && out != nullptr, "null argument");
        need(op >= 0 && op <= 3, "op must be 0..3");
        const auto& F = f->f;
        const qpack::GfqElt x{a};
        qpack::GfqElt r;
        if (op == 0)
            r = F.mul(x, qpack::GfqElt{b});
        else if (op == 1)
            r = F.add(x, qpack::GfqElt{b});
        else if (op == 2)
            r = F.neg(x);
        else
            r = F.inverse(x);
        *out = r.rep;
    });
}

qpk_status qpk_fgdp_dot(qpk_field f, const uint32_t* v1, const uint32_t* v2, uint64_t n, uint32_t* out,
                        qpk_cost* cost) {
    return guard([&] {
        need(f != nullptr && out != nullptr && (n == 0 || (v1 && v2)), "null argument");
        qpack::CostReport c;
        const auto* x = reinterpret_cast<const qpack::GfqElt*>(v1);
        const auto* y = reinterpret_cast<const qpack::GfqElt*>(v2);
        *out = qpack::fgdp_dot(std::span<const qpack::GfqElt>(x, n), std::span<const qpack::GfqElt>(y, n), f->f, &c)
                   .rep;
        put_cost(cost, c);
    });
}

qpk_status qpk_gfq_mul_batch(qpk_field f, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out, int path,
                             void* stream) {
    return guard([&] {
        need(f != nullptr && (n == 0 || (a && b && out)), "null argument");
        need(path >= 0 && path <= 2, "path must be 0 (packed), 1 (dlog) or 2 (linear)");
        qpack::gpu::gfq_mul_device(qpack::detail::device_field(f->f), a, b, n, out, path, as_stream(stream));
    });
}

qpk_status qpk_gfq_mul_batch_host(qpk_field f, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                                  int path) {
    return guard([&] {
        need(f != nullptr && (n == 0 || (a && b && out)), "null argument");
        need(path >= 0 && path <= 2, "path must be 0 (packed), 1 (dlog) or 2 (linear)");
        qpack::gpu::gfq_mul_host(qpack::detail::device_field(f->f), a, b, n, out, path);
    });
}

qpk_status qpk_gfq_mul_rep_host(qpk_field f, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out) {
    return guard([&] {
        need(f != nullptr && (n == 0 || (a && b && out)), "null argument");
        // reps outside the field: out_of_range, detected on the device
        if (n) qpack::gpu::gfq_mul_rep_host(qpack::detail::device_field(f->f), a, b, n, out);
    });
}

qpk_status qpk_gfq_matmul(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K, uint64_t n,
                          uint32_t chunk, uint8_t* C, void* stream) {
    return guard([&] {
        need(f != nullptr, "null field");
        need((m == 0 || n == 0) || (A && B && C) || K == 0, "null buffer");
        if (K == 0 && m && n) {
            qpack::gpu::check(cudaMemsetAsync(C, 0, m * n * f->f.k(), as_stream(stream)), "memset");
            return;
        }
        qpack::gpu::gfq_matmul_device(qpack::detail::device_field(f->f), f->f, A, B, m, K, n, chunk, C, false,
                                      as_stream(stream));
    });
}

// counters of C = A*B: the reference's closed-form part plus, when the
// caller asked for them, the data-dependent Zech reads (K7)
static void put_matmul_cost(qpk_cost* cost, const qpack::GfqField& f, uint64_t m, uint64_t K, uint64_t n, uint64_t zech) {
    if (!cost) return;
    qpack::CostReport c = qpack::gpu::matmul_cost(f, m, K, n);
    c.table_accesses += zech;
    put_cost(cost, c);
}

qpk_status qpk_gfq_matmul_host(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K, uint64_t n,
                               uint32_t chunk, uint8_t* C, qpk_cost* cost) {
    return qpk_gfq_matmul_repack_host(f, A, B, m, K, n, chunk, qpk::kRepackRedq, C, cost);
}

qpk_status qpk_gfq_matmul_repack(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K,
                                 uint64_t n, uint32_t chunk, uint32_t repack, uint8_t* C, void* stream) {
    return guard([&] {
        need(f != nullptr, "null field");
        need((m == 0 || n == 0) || (A && B && C) || K == 0, "null buffer");
        if (K == 0 && m && n) {
            qpack::gpu::check(cudaMemsetAsync(C, 0, m * n * f->f.k(), as_stream(stream)), "memset");
            return;
        }
        qpack::gpu::gfq_matmul_device(qpack::detail::device_field(f->f), f->f, A, B, m, K, n, chunk, C, false,
                                      as_stream(stream), repack);
    });
}

qpk_status qpk_gfq_matmul_repack_host(qpk_field f, const uint8_t* A, const uint8_t* B, uint64_t m, uint64_t K,
                                      uint64_t n, uint32_t chunk, uint32_t repack, uint8_t* C, qpk_cost* cost) {
    return guard([&] {
        need(f != nullptr, "null field");
        need((m == 0 || n == 0) || (A && B && C) || K == 0, "null buffer");
        uint64_t zech = 0;
        if (m && n) {
            if (K == 0)
                std::memset(C, 0, m * n * f->f.k());
            else
                qpack::gpu::gfq_matmul_host(qpack::detail::device_field(f->f), f->f, A, B, m, K, n, chunk, C, false,
                                            repack, cost ? &zech : nullptr);
        }
        put_matmul_cost(cost, f->f, m, K, n, zech);
    });
}

qpk_status qpk_gfq_matmul_rep(qpk_field f, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K, uint64_t n,
                              uint32_t* C, void* stream) {
    return guard([&] {
        need(f != nullptr, "null field");
        need((m == 0 || n == 0) || (A && B && C) || K == 0, "null buffer");
        if (m == 0 || n == 0) return;
        if (K == 0) {
            // every entry is the field's zero sentinel
            std::vector<uint32_t> z(m * n, static_cast<uint32_t>(f->f.order() - 1));
            qpack::gpu::check(cudaMemcpyAsync(C, z.data(), z.size() * 4, cudaMemcpyHostToDevice, as_stream(stream)),
                              "fill");
            qpack::gpu::check(cudaStreamSynchronize(as_stream(stream)), "sync");
            return;
        }
        qpack::gpu::gfq_matmul_device(qpack::detail::device_field(f->f), f->f, A, B, m, K, n, 0, C, true,
                                      as_stream(stream));
    });
}

qpk_status qpk_gfq_matmul_rep_host(qpk_field f, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K,
                                   uint64_t n, uint32_t* C, qpk_cost* cost) {
    return guard([&] {
        need(f != nullptr, "null field");
        need((m == 0 || n == 0) || (A && B && C) || K == 0, "null buffer");
        // gfq_matmul(GfqMatrix...) on the caller's rep arrays in place (no
        // GfqMatrix copies); reps outside the field are detected on the
        // device (the K1 pack) and raise out_of_range like the reference
        uint64_t zech = 0;
        if (m != 0 && n != 0) {
            if (K == 0) {
                const uint32_t zero = static_cast<uint32_t>(f->f.order() - 1);
                std::fill(C, C + m * n, zero);
            } else {
                qpack::gpu::gfq_matmul_host(qpack::detail::device_field(f->f), f->f, A, B, m, K, n, 0, C, true,
                                            qpk::kRepackRedq, cost ? &zech : nullptr);
            }
        }
        put_matmul_cost(cost, f->f, m, K, n, zech);
    });
}

qpk_status qpk_gfq_gemv(qpk_field f, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K, uint32_t* y_rep,
                        uint8_t* y_coeff, void* stream) {
    return guard([&] {
        need(f != nullptr, "null field");
        need(m == 0 || ((A || K == 0) && (x || K == 0) && (y_rep || y_coeff)), "null buffer");
        qpack::gpu::gfq_gemv_device(qpack::detail::device_field(f->f), f->f, A, x, m, K, y_rep, y_coeff,
                                    as_stream(stream));
    });
}

qpk_status qpk_gfq_gemv_host(qpk_field f, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                             uint32_t* y_rep, uint8_t* y_coeff, qpk_cost* cost) {
    return guard([&] {
        need(f != nullptr, "null field");
        need(m == 0 || ((A || K == 0) && (x || K == 0) && (y_rep || y_coeff)), "null buffer");
        // reps outside the field are detected on the device (out_of_range)
        uint64_t zech = 0;
        if (m) qpack::gpu::gfq_gemv_host(qpack::detail::device_field(f->f), f->f, A, x, m, K, y_rep, y_coeff,
                                         cost ? &zech : nullptr);
        put_matmul_cost(cost, f->f, m, K, 1, zech);
    });
}

// ---------------------------------------------------------------- inputs
qpk_status qpk_gen_draws(uint64_t seed, uint64_t start, uint64_t count, uint32_t bound, uint8_t* out, void* stream) {
    return guard([&] {
        need(bound >= 1 && bound <= 256, "bound must be in [1, 256]");
        need(count == 0 || out, "null buffer");
        qpack::gpu::require_device();
        qpack::gpu::check(qpk::launch_gen_draws(seed, start, count, bound, out, as_stream(stream)), "gen_draws");
    });
}

qpk_status qpk_gen_words(uint64_t seed, uint64_t first, uint64_t n, uint64_t q, uint32_t d, double* out,
                         void* stream) {
    return guard([&] {
        need(q >= 2, "q must be >= 2");
        need(qpack::pow_fits_u128(q, d + 1) && qpack::checked_pow_u128(q, d + 1) <= (qpack::u128(1) << 53),
             "q^(d+1) must not exceed 2^53");
        need(n == 0 || out, "null buffer");
        qpack::gpu::require_device();
        qpack::gpu::check(qpk::launch_gen_words(seed, first, n, q, d, out, as_stream(stream)), "gen_words");
    });
}

qpk_status qpk_gen_pairs(uint64_t seed, uint64_t n, uint32_t k, uint32_t bound, uint8_t* a, uint8_t* b,
                         void* stream) {
    return guard([&] {
        need(bound >= 1 && bound <= 256 && k >= 1, "bound must be in [1, 256], k >= 1");
        need(n == 0 || (a && b), "null buffer");
        qpack::gpu::require_device();
        qpack::gpu::check(qpk::launch_gen_pairs(seed, n, k, bound, a, b, as_stream(stream)), "gen_pairs");
    });
}

// ----------------------------------------------------------- measurement
qpk_status qpk_probe_fp64(int which, int iters, double* tflops) {
    return guard([&] {
        need(tflops != nullptr && iters > 0 && (which == 0 || which == 1), "bad argument");
        qpack::gpu::require_device();
        qpack::gpu::DevBuf sink;
        sink.ensure(64);
        uint64_t flops = 0;
        auto launch = [&] {
            qpack::gpu::check(which ? qpk::launch_probe_dmma(sink.as<double>(), iters, &flops, 0)
                                    : qpk::launch_probe_dfma(sink.as<double>(), iters, &flops, 0),
                              "probe");
        };
        launch();  // warm-up
        cudaEvent_t e0, e1;
        qpack::gpu::check(cudaEventCreate(&e0), "event");
        qpack::gpu::check(cudaEventCreate(&e1), "event");
        cudaEventRecord(e0, 0);
        launch();
        cudaEventRecord(e1, 0);
        qpack::gpu::check(cudaEventSynchronize(e1), "probe sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tflops = static_cast<double>(flops) / (static_cast<double>(ms) * 1e-3) / 1e12;
    });
}

}  // extern "C"
