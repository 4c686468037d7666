// Drop-in check of the C++ API in include/qpack (the reference's public API,
// proj/include/qpack) against the reference's own known answers.  Built and
// run by tests/test_dropin_cpp.py; `./test_dropin gpu` adds the GPU-backed
// calls (gfq_matmul, qpack::gpu::*).
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "qpack/dqt.hpp"
#include "qpack/fpdiv.hpp"
#include "qpack/gfq.hpp"
#include "qpack/gpu.hpp"
#include "qpack/params.hpp"
#include "qpack/polymul.hpp"
#include "qpack/redq.hpp"
#include "qpack/rng.hpp"

using namespace qpack;

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);    \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

template <class E, class F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void host_tests() {
    // params (test_params.cpp:54-60, 140-152)
    CHECK(validate(3, 100, 2, 1, 53).ok());
    CHECK(validate(3, 16, 4, 1, 53).violation == ParamViolation::q_too_small);
    CHECK(validate(3, 16, 4, 1, 53).detail.find("n_q*k*(p-1)^2") != std::string::npos);
    CHECK(validate(3, 1 << 20, 4, 1, 53).violation == ParamViolation::word_overflow);
    CHECK(validate(3, u64(1) << 60, 2, 1, 53).violation == ParamViolation::q_unrepresentable);
    CHECK(throws<std::invalid_argument>([] { validate(0, 2, 1, 1, 53); }));
    QadicParams pd = qadic_for_degree(3, 4, 53);
    CHECK(pd.k == 5 && pd.q == 32 && pd.n_q == 1);
    QadicParams b3 = best_qadic(3, 53, 1, true);
    CHECK(b3.k == 5 && b3.q == 32);
    CHECK(delayed_bound(1009, 24) == 33);

    // fpdiv (test_fpdiv.cpp:13-36)
    CHECK(floor_div_rn(10302, 3) == 3434);
    CHECK(premul_floor_bound(0x1p-53) == (u64(1) << 52) - 1);
    CHECK(premul_floor_bound(0x1p-24) == (u64(1) << 23) - 1);
    CHECK(ReciprocalDivisor::make(3).r_max == 1501199875790165ull);
    CHECK(throws<std::out_of_range>([] {
        ReciprocalDivisor d = ReciprocalDivisor::make(3);
        floor_div_premul(d.r_max + 1, d);
    }));

    // DQT (test_dqt.cpp:26-71; acceptance.cpp:61-68)
    const QadicParams p100{3, 100, 2, 1, 53};
    CHECK(pack(DensePoly{3, {1, 1}}, p100).value == 101);
    CHECK(dqt_mul(pack(DensePoly{3, {1, 1}}, p100), pack(DensePoly{3, {2, 1}}, p100)).value == 10302);
    CHECK((unpack(Packed{10302, p100}, 3) == std::vector<u64>{2, 3, 1}));
    CHECK((dqt_mul_poly(DensePoly{3, {1, 1}}, DensePoly{3, {2, 1}}, p100) == DensePoly{3, {2, 0, 1}}));
    CHECK(throws<std::length_error>([&] { pack(DensePoly{3, {1, 1, 1}}, p100); }));
    CHECK((unpack_value(40013002800270018ull, 10000, 5) == std::vector<u64>{18, 27, 28, 13, 4}));

    // REDQ (test_redq.cpp:26-58, 161-167, 237-247)
    RedqPlan id = RedqPlan::build(5, 10000, 4);
    CHECK(redq(40013002800270018ull, id) == 40003000300020003ull);
    RedqPlan w = RedqPlan::build(23, 1000000, 3);
    CHECK(w.neg_q_mod_p == 17);
    RedqTrace t = redq_trace(parse_u128("1234005678009123004567"), w);
    CHECK(to_string(t.rop) == "53652420783005348024");
    CHECK((t.u == std::vector<u64>{15, 8, 18, 15}));
    CHECK((t.mu == std::vector<u64>{13, 15, 20, 15}));
    CHECK(t.word == parse_u128("15000020000015000013"));
    CHECK(build_correction_table(5, 10000, 3, TableIndexing::base_p).entries.size() == 125);
    CHECK(build_correction_table(5, 10000, 3, TableIndexing::binary_shift).entries.size() == 512);
    CHECK(throws<std::domain_error>([] { redq(u128(100 * 100 * 100), RedqPlan::build(3, 100, 2)); }));
    CHECK(throws<std::invalid_argument>([] { RedqPlan::build(3, u64(1) << 20, 3, RedqMode::float_premul); }));
    {
        CorrectionTable tb = build_correction_table(3, 4, 2, TableIndexing::base_p);
        std::stringstream buf;
        save_correction_table(tb, buf);
        const std::string bytes = buf.str();
        CHECK(bytes.size() == 40 + 8 * 9);
        CHECK(bytes.substr(0, 4) == "QPKT");
        CHECK(static_cast<unsigned char>(bytes[8]) == 3 && static_cast<unsigned char>(bytes[16]) == 4);
        CorrectionTable back = load_correction_table(buf);
        CHECK(back.entries == tb.entries && back.radix == tb.radix);
    }
    // tabulated == direct == integer == float (test_redq.cpp:77-126)
    {
        SplitMix64 rng(36);
        RedqPlan direct = RedqPlan::build(23, 1 << 10, 6);
        RedqPlan tabled = RedqPlan::build(23, 1 << 10, 6);
        tabled.attach_correction(build_correction_table(23, 1 << 10, 3, TableIndexing::base_p));
        for (int it = 0; it < 2000; ++it) {
            u128 r = 0;
            for (int i = 0; i < 7; ++i) r = r * 1024 + rng.below(1024);
            CostReport c;
            CHECK(redq(r, tabled, &c) == redq(r, direct));
            CHECK(c.table_accesses == 3);
        }
    }

    // FQT: every word width runs on the device (gpu_tests)
    CHECK(packed_degree(500, 4) == 100);

    // GF(9) (test_gfq.cpp:23-36, 108-115)
    GfqField f9 = GfqField::build(3, 2, gfq_default_q(3, 2));
    CHECK((f9.modulus_poly() == std::vector<u64>{1, 0, 1}));
    CHECK((f9.to_coeffs(f9.generator()) == std::vector<u64>{1, 1}));
    GfqElt x = f9.from_coeffs(std::vector<u64>{0, 1});
    CHECK((f9.to_coeffs(f9.mul(x, x)) == std::vector<u64>{2, 0}));
    std::vector<GfqElt> v1 = {f9.from_coeffs(std::vector<u64>{1, 1}), f9.from_coeffs(std::vector<u64>{0, 2})};
    std::vector<GfqElt> v2 = {f9.from_coeffs(std::vector<u64>{2, 1}), f9.from_coeffs(std::vector<u64>{0, 1})};
    CHECK((f9.to_coeffs(fgdp_dot(v1, v2, f9)) == std::vector<u64>{2, 0}));
    CHECK(f9.memory_entries() == 6 * 9);
    CHECK(throws<std::domain_error>([] { GfqField::build(4, 2, 64); }));
    CHECK(throws<std::length_error>([] { GfqField::build(3, 30, 1 << 16); }));
}

static void gpu_tests() {
    SplitMix64 rng(77);
    // FQT on the device (K6) behind the unchanged signature
    CHECK((fqt_mul(DensePoly{3, {1, 1}}, DensePoly{3, {1, 1}}, 1, QadicParams{3, 32, 2, 1, 53}) ==
           DensePoly{3, {1, 2, 1}}));
    {
        DensePoly a{3, {}}, b{3, {}};
        for (int i = 0; i < 3000; ++i) a.coeffs.push_back(rng.below(3));
        for (int i = 0; i < 1777; ++i) b.coeffs.push_back(rng.below(3));
        const QadicParams pr = qadic_for_degree(3, 3, 53);
        CostReport c;
        const DensePoly got = fqt_mul(a, b, 3, pr, &c);
        DensePoly want = DensePoly::zero(3, a.coeffs.size() + b.coeffs.size() - 1);
        for (std::size_t i = 0; i < a.coeffs.size(); ++i)
            for (std::size_t j = 0; j < b.coeffs.size(); ++j)
                want.coeffs[i + j] = (want.coeffs[i + j] + a.coeffs[i] * b.coeffs[j]) % 3;
        CHECK(got == want);
        const u64 span = 2 * packed_degree(2999, 3) + 1;
        CHECK(c.mul_add == span * span && c.divisions == span * span);  // n_q = 1
    }
    // batched REDQ == per-word host REDQ
    RedqPlan plan = RedqPlan::build(5, 128, 6, RedqMode::float_premul);
    plan.attach_correction(build_correction_table(5, 128, 4, TableIndexing::base_p));
    std::vector<double> words(100003);
    for (auto& wd : words) wd = static_cast<double>(rng.next() >> 15);
    std::vector<std::uint8_t> res(words.size() * 7);
    CostReport cost;
    gpu::redq_residues_batch(words, plan, res, &cost);
    bool same = true;
    for (std::size_t i = 0; i < words.size(); ++i) {
        const std::vector<u64> mu = redq_residues(static_cast<u128>(static_cast<u64>(words[i])), plan);
        for (int j = 0; j < 7; ++j) same &= res[i * 7 + j] == mu[j];
    }
    CHECK(same);
    CHECK(cost.divisions == words.size() && cost.table_accesses == 2 * words.size());
    words[5] = 1e300;
    CHECK(throws<std::domain_error>([&] { gpu::redq_residues_batch(words, plan, res); }));

    // u128 words (the reference's integer mode, p = 23, q = 10^6, d = 3:
    // words up to 10^24 > 2^64) == the scalar redq_residues per word
    {
        const RedqPlan wide = RedqPlan::build(23, 1000000, 3);
        std::vector<u128> w128(3001);
        for (auto& w : w128) w = (u128(rng.next()) << 64 | rng.next()) % (u128(1000000) * 1000000 * 1000000 * 1000000);
        w128[0] = 0;
        w128[1] = u128(1000000) * 1000000 * 1000000 * 1000000 - 1;
        std::vector<std::uint8_t> r128(w128.size() * 4);
        gpu::redq_residues_batch(std::span<const u128>(w128), wide, r128);
        bool ok = true;
        for (std::size_t i = 0; i < w128.size(); ++i) {
            const std::vector<u64> mu = redq_residues(w128[i], wide);
            for (int j = 0; j < 4; ++j) ok &= r128[i * 4 + j] == mu[j];
        }
        CHECK(ok);
        w128[9] = u128(1000000) * 1000000 * 1000000 * 1000000;
        CHECK(throws<std::domain_error>([&] { gpu::redq_residues_batch(std::span<const u128>(w128), wide, r128); }));
    }

    // FQT with u128 words (test_polymul.cpp:42-58, m = 128): the device's
    // integer-word kernel
    CHECK((fqt_mul(DensePoly{5, {3, 2, 1}}, DensePoly{5, {1, 0, 4}}, 2, QadicParams{5, 10000, 3, 1, 128}) ==
           DensePoly{5, {3, 2, 3, 3, 4}}));

    // GPU gfq_matmul == the triple loop of field ops (acceptance.cpp:361-374)
    GfqField f = GfqField::build(3, 3, 1024);
    const std::size_t n = 40, K = 300;
    GfqMatrix a = GfqMatrix::zero(f, n, K), b = GfqMatrix::zero(f, K, n);
    for (auto& e : a.data) e = f.from_index(rng.below(f.order()));
    for (auto& e : b.data) e = f.from_index(rng.below(f.order()));
    CostReport mc;
    GfqMatrix c = gfq_matmul(a, b, f, &mc);
    bool mm = true;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            GfqElt acc = f.zero();
            for (std::size_t l = 0; l < K; ++l) acc = f.add(acc, f.mul(a.at(i, l), b.at(l, j)));
            mm &= c.at(i, j) == acc;
        }
    CHECK(mm);
    CHECK(mc.mul_add == n * n * K && mc.divisions == n * n * ((K + f.params().n_q - 1) / f.params().n_q));

    // coefficient-record API, both delayed re-packs (chunk 64, K > n_q): same C
    {
        std::vector<std::uint8_t> A(n * K * 3), B(K * n * 3), C1(n * n * 3), C2(n * n * 3);
        for (std::size_t i = 0; i < n * K; ++i) {
            const std::vector<u64> x = f.to_coeffs(a.data[i]), y = f.to_coeffs(b.data[i]);
            for (int t = 0; t < 3; ++t) A[i * 3 + t] = static_cast<std::uint8_t>(x[t]), B[i * 3 + t] = static_cast<std::uint8_t>(y[t]);
        }
        gpu::gfq_matmul_coeffs(A, B, n, K, n, f, C1, 64, nullptr, gpu::Repack::redq);
        gpu::gfq_matmul_coeffs(A, B, n, K, n, f, C2, 64, nullptr, gpu::Repack::fold);
        bool same_c = C1 == C2;
        for (std::size_t i = 0; i < n * n; ++i) {
            const std::vector<u64> want = f.to_coeffs(c.data[i]);
            for (int t = 0; t < 3; ++t) same_c &= C1[i * 3 + t] == want[t];
        }
        CHECK(same_c);
        GfqField f9 = GfqField::build(3, 2, 64);
        std::vector<std::uint8_t> A9(4 * 8 * 2), C9(4 * 4 * 2);
        CHECK(throws<std::invalid_argument>(
            [&] { gpu::gfq_matmul_coeffs(A9, A9, 4, 8, 4, f9, C9, 0, nullptr, gpu::Repack::fold); }));
    }

    // elementwise GF products, both device paths == fgdp_dot on one pair
    GfqField f343 = GfqField::build(7, 3, 256);
    const std::size_t m = 5000;
    std::vector<std::uint8_t> ca(m * 3), cb(m * 3), out(m * 3);
    for (auto& v : ca) v = static_cast<std::uint8_t>(rng.below(7));
    for (auto& v : cb) v = static_cast<std::uint8_t>(rng.below(7));
    for (auto path : {gpu::GfqPath::packed, gpu::GfqPath::dlog}) {
        gpu::gfq_mul_batch(ca, cb, f343, out, path);
        bool ok = true;
        for (std::size_t i = 0; i < m; ++i) {
            std::vector<u64> x3(ca.begin() + i * 3, ca.begin() + i * 3 + 3), y3(cb.begin() + i * 3, cb.begin() + i * 3 + 3);
            GfqElt ea = f343.from_coeffs(x3), eb = f343.from_coeffs(y3);
            const std::vector<u64> want = f343.to_coeffs(fgdp_dot(std::span<const GfqElt>(&ea, 1),
                                                                  std::span<const GfqElt>(&eb, 1), f343));
            for (int j = 0; j < 3; ++j) ok &= out[i * 3 + j] == want[j];
        }
        CHECK(ok);
    }
}

int main(int argc, char** argv) {
    host_tests();
    if (argc > 1 && std::string(argv[1]) == "gpu") gpu_tests();
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
