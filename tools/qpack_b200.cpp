// qpack_b200: the reference's benchmark / regression CLI surface
// (proj/tools/qpack.cpp, proj/README.md:52-97) over the qpack-b200 drop-in
// API, whose batch-shaped calls run on the B200 kernels.
//
//   qpack_b200 mulpoly --p P --n N [--d D] [--algo fqt] [--seed S] [--repeat R]
//                      [--csv FILE] [--m M] [--no-verify] [--a LIST --b LIST]
//   qpack_b200 paper-examples [--inject-fault]
//   qpack_b200 gfq --p P --k K [--op dot|matmul] [--len L] [--size S]
//                  [--seed S] [--csv FILE] [--indexing base_p|binary_shift]
//                  [--dump-field]
//
// CSV rows keep the reference schema (qpack.cpp:9-14, README "CSV schema"):
//   algo,p,q,k,d,N,n_q,n_d,mul_add,divisions,table_accesses,wall_time_ns,checksum
// with the same seeded inputs (splitmix64, below(n) = next() % n), the same
// counters (closed forms of the reference loops) and the same FNV-1a
// checksum of the output coefficients, so rows compare byte-for-byte with
// the reference's except wall_time_ns and the algo tag: device rows are
// tagged `<algo>_b200`, host verification rows keep the reference's name.
// QPACK_TABLE_CACHE reuses serialized correction tables (qpack.cpp:80-98).
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "qpack/common.hpp"
#include "qpack/counters.hpp"
#include "qpack/dqt.hpp"
#include "qpack/gfq.hpp"
#include "qpack/gpu.hpp"
#include "qpack/params.hpp"
#include "qpack/polymul.hpp"
#include "qpack/redq.hpp"
#include "qpack/rng.hpp"

namespace fs = std::filesystem;
using namespace qpack;

namespace {

std::string hex16(u64 v) {
    char buf[17];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
    return buf;
}

std::string hex(u64 v) {
    char buf[17];
    std::snprintf(buf, sizeof buf, "%llx", static_cast<unsigned long long>(v));
    return buf;
}

// one CSV row: what ran (tag, field and shape), what it counted, how long it
// took, and the FNV-1a fold of its output
struct Measurement {
    std::string tag;
    u64 prime = 0, radix = 0, size = 0, group = 0, delay = 0;
    u32 chunk = 0, degree = 0;
    CostReport counted;
    u64 elapsed_ns = 0, fnv = 0;
};

class CsvLog {
public:
    explicit CsvLog(std::string file) : file_(std::move(file)) {}
    void add(const Measurement& m) const {
        if (file_.empty()) return;
        std::error_code ec;
        const bool header = !fs::exists(file_, ec) || fs::file_size(file_, ec) == 0;
        std::ofstream f(file_, std::ios::app);
        if (!f) throw std::runtime_error("cannot open csv file " + file_);
        if (header) f << kColumns << '\n';
        const std::array<u64, 11> nums{m.prime, m.radix,          m.chunk,
                                       m.degree, m.size,          m.group,
                                       m.delay,  m.counted.mul_add, m.counted.divisions,
                                       m.counted.table_accesses,  m.elapsed_ns};
        f << m.tag;
        for (u64 v : nums) f << ',' << v;
        f << ',' << hex16(m.fnv) << '\n';
    }

private:
    static constexpr const char* kColumns =
        "algo,p,q,k,d,N,n_q,n_d,mul_add,divisions,table_accesses,wall_time_ns,checksum";
    std::string file_;
};

class Stopwatch {
public:
    Stopwatch() : t0_(clock::now()) {}
    u64 ns() const {
        return static_cast<u64>(std::chrono::duration_cast<std::chrono::nanoseconds>(clock::now() - t0_).count());
    }

private:
    using clock = std::chrono::steady_clock;
    clock::time_point t0_;
};

// QPACK_TABLE_CACHE: a plan's correction table is read back from the cache
// directory when a file for (p, q, window, indexing) exists, stored otherwise
void reuse_cached_table(RedqPlan& plan) {
    const char* root = std::getenv("QPACK_TABLE_CACHE");
    if (root == nullptr || !plan.correction.has_value()) return;
    const CorrectionTable& tab = *plan.correction;
    const std::string leaf = "redq_p" + std::to_string(tab.p) + "_q" + std::to_string(tab.q) + "_w" +
                             std::to_string(tab.k_window) +
                             (tab.indexing == TableIndexing::base_p ? "_basep.tbl" : "_shift.tbl");
    const fs::path where = fs::path(root) / leaf;
    if (std::ifstream cached(where, std::ios::binary); cached) {
        plan.attach_correction(load_correction_table(cached));
    } else {
        fs::create_directories(root);
        std::ofstream fresh(where, std::ios::binary);
        save_correction_table(tab, fresh);
    }
}

std::vector<u64> coefficients_of(const std::string& text, u64 p) {
    std::vector<u64> out;
    std::size_t at = 0;
    while (at <= text.size() && !text.empty()) {
        const std::size_t comma = std::min(text.find(',', at), text.size());
        if (comma > at) out.push_back(std::stoull(text.substr(at, comma - at)) % p);
        at = comma + 1;
    }
    return out;
}

// plain schoolbook product mod p: the CLI's own verification
DensePoly schoolbook(const DensePoly& a, const DensePoly& b) {
    DensePoly r = DensePoly::zero(a.p, a.coeffs.size() + b.coeffs.size() - 1);
    for (std::size_t i = 0; i < a.coeffs.size(); ++i)
        for (std::size_t j = 0; j < b.coeffs.size(); ++j)
            r.coeffs[i + j] = (r.coeffs[i + j] + a.coeffs[i] * b.coeffs[j]) % a.p;
    return r;
}

struct Args {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    u64 u(const std::string& k, u64 def) const { return has(k) ? std::stoull(kv.at(k)) : def; }
    bool flag(const std::string& k) const { return flags.count(k) != 0; }
};

int cmd_mulpoly(const Args& a) {
    if (!a.has("p") || !a.has("n")) throw std::invalid_argument("mulpoly: --p and --n are required");
    const u64 p = a.u("p", 3), n = a.u("n", 100);
    const u32 m = static_cast<u32>(a.u("m", 53));
    const std::string algo = a.str("algo", "fqt");
    const CsvLog log(a.str("csv"));
    const bool on_device = algo == "fqt", verify = on_device && !a.flag("no-verify");
    if (algo == "delayed") throw std::domain_error("--algo delayed is not part of qpack-b200 (host-only variant)");
    if (!on_device && algo != "oracle") throw std::domain_error("unknown --algo " + algo);
    QadicParams shape{};
    RedqPlan reducer;
    if (on_device) {
        shape = a.has("d") ? qadic_for_degree(p, static_cast<u32>(a.u("d", 0)), m) : best_qadic(p, m, 1, true);
        reducer = fqt_reduction_plan(shape, shape.k - 1);
        reuse_cached_table(reducer);
    }
    SplitMix64 draws(a.u("seed", 42));
    const bool fixed = a.has("a") || a.has("b");
    for (u64 rep = 0, reps = a.u("repeat", 1); rep < reps; ++rep) {
        DensePoly lhs{p, {}}, rhs{p, {}};
        if (fixed) {
            lhs.coeffs = coefficients_of(a.str("a"), p);
            rhs.coeffs = coefficients_of(a.str("b"), p);
            if (lhs.coeffs.empty() || rhs.coeffs.empty())
                throw std::domain_error("--a and --b must both be given for fixed inputs");
        } else {
            for (DensePoly* poly : {&lhs, &rhs})
                for (u64 i = 0; i <= n; ++i) poly->coeffs.push_back(draws.below(p));
        }
        Measurement row;
        row.tag = on_device ? "fqt_b200" : "oracle";
        row.prime = p;
        row.size = n;
        if (on_device) {
            row.radix = shape.q;
            row.chunk = shape.k;
            row.degree = shape.k - 1;
            row.group = shape.n_q;
        }
        const Stopwatch clock;
        // K6 on the device (m <= 53), or the host schoolbook product
        const DensePoly product =
            on_device ? fqt_mul(lhs, rhs, shape.k - 1, shape, reducer, &row.counted) : schoolbook(lhs, rhs);
        row.elapsed_ns = clock.ns();
        row.fnv = fold_checksum(product.coeffs.data(), product.coeffs.size());
        if (verify && !(product == schoolbook(lhs, rhs))) {
            std::cerr << "verification FAILED against the schoolbook product\n";
            return 3;
        }
        log.add(row);
        std::cout << row.tag << " p=" << p << " N=" << n << " rep=" << rep << " mul_add=" << row.counted.mul_add
                  << " divisions=" << row.counted.divisions << " table_accesses=" << row.counted.table_accesses
                  << " wall_ns=" << row.elapsed_ns << " checksum=" << hex(row.fnv) << (verify ? " verified=ok" : "")
                  << "\n";
    }
    return 0;
}

std::string bracketed(const std::vector<u64>& v) {
    std::string s;
    for (u64 x : v) s += (s.empty() ? "[" : ",") + std::to_string(x);
    return (s.empty() ? "[" : s) + "]";
}

// The worked examples of the paper (PAPER.md sections 2-4) as exhibits of
// (label, computed, expected) lines, then the same reductions on the device.
int cmd_paper_examples(const Args& a) {
    using Line = std::tuple<std::string, std::string, std::string>;
    struct Exhibit {
        std::string title;
        std::function<std::vector<Line>()> lines;
    };
    const bool corrupt = a.flag("inject-fault");
    const std::vector<Exhibit> exhibits = {
        {"[1] radix-100 product over Z/3Z",
         [] {
             const QadicParams radix100{3, 100, 2, 1, 53};
             const DensePoly x_plus_1{3, {1, 1}}, x_plus_2{3, {2, 1}};
             const Packed word = dqt_mul(pack(x_plus_1, radix100), pack(x_plus_2, radix100));
             const bool reduced = dqt_mul_poly(x_plus_1, x_plus_2, radix100) == DensePoly{3, {2, 0, 1}};
             return std::vector<Line>{{"101 x 102", to_string(word.value), "10302"},
                                      {"digits", bracketed(unpack(word, 3)), "[2,3,1]"},
                                      {"reduced", reduced ? "X^2+2" : "?", "X^2+2"}};
         }},
        {"[2] five residues reduced at once (p | q)",
         [] {
             const u128 word = static_cast<u128>(100020003) * 400050006;
             return std::vector<Line>{
                 {"packed product", to_string(word), "40013002800270018"},
                 {"reduced word", to_string(redq(word, RedqPlan::build(5, 10000, 4))), "40003000300020003"}};
         }},
        {"[3] full correction at p=23, q=10^6",
         [] {
             const RedqTrace tr = redq_trace(parse_u128("1234005678009123004567"), RedqPlan::build(23, 1000000, 3));
             return std::vector<Line>{{"rop", to_string(tr.rop), "53652420783005348024"},
                                      {"u", bracketed(tr.u), "[15,8,18,15]"},
                                      {"mu", bracketed(tr.mu), "[13,15,20,15]"}};
         }},
        {"[4] degree-6 correction through three window lookups",
         [corrupt] {
             CorrectionTable window3 = build_correction_table(23, 1000000, 3, TableIndexing::base_p);
             if (corrupt)
                 for (u64& e : window3.entries) e ^= 1;  // a corrupted cache must be detected
             const RedqPlan direct = RedqPlan::build(23, 1000000, 6);
             SplitMix64 draws(4);
             u64 lookups = 0, disagreements = 0;
             std::vector<u64> raw(7);
             for (int trial = 0; trial < 500; ++trial) {
                 for (u64& digit : raw) digit = draws.below(23);
                 CostReport tally;
                 disagreements += correct_tabulated(raw, window3, &tally) != correct_direct(raw, direct);
                 lookups = tally.table_accesses;
             }
             return std::vector<Line>{{"window accesses", std::to_string(lookups), "3"},
                                      {"tabulated == direct", disagreements == 0 ? "yes" : "no", "yes"}};
         }},
        {"[5] the same reductions on the device (batched REDQ kernels)",
         [] {
             // random words at p=23, q=2^7, d=6 through the windowed device
             // table (Alg. 3), against the host REDQ of each word
             RedqPlan pd = RedqPlan::build(23, 1 << 7, 6, RedqMode::float_premul);
             pd.attach_correction(build_correction_table(23, 1 << 7, 3, TableIndexing::base_p));
             std::vector<double> words(4096);
             SplitMix64 wr(5);
             for (double& w : words) {
                 u64 r = 0;
                 for (int i = 0; i < 7; ++i) r = r * 128 + wr.below(128);
                 w = static_cast<double>(r);
             }
             std::vector<std::uint8_t> res(words.size() * 7);
             gpu::redq_residues_batch(words, pd, res);
             bool same = true;
             for (std::size_t i = 0; i < words.size(); ++i) {
                 const std::vector<u64> mu = redq_residues(static_cast<u128>(static_cast<u64>(words[i])), pd);
                 for (int j = 0; j < 7; ++j) same &= res[i * 7 + j] == mu[j];
             }
             return std::vector<Line>{{"device residues == host", same ? "yes" : "no", "yes"}};
         }},
    };
    int misses = 0;
    for (const Exhibit& ex : exhibits) {
        std::cout << ex.title << "\n";
        for (const auto& [label, got, want] : ex.lines()) {
            if (got == want) {
                std::cout << "  ok   " << label << ": " << got << "\n";
            } else {
                std::cout << "  FAIL " << label << ": " << got << " (expected " << want << ")\n";
                ++misses;
            }
        }
    }
    std::cout << (misses ? "MISMATCHES FOUND\n" : "all examples reproduced\n");
    return misses ? 4 : 0;
}

int cmd_gfq(const Args& a) {
    if (!a.has("p") || !a.has("k")) throw std::invalid_argument("gfq: --p and --k are required");
    const u64 p = a.u("p", 3);
    const u32 k = static_cast<u32>(a.u("k", 2));
    const std::string op = a.str("op", "dot");
    if (op != "dot" && op != "matmul" && !a.flag("dump-field")) throw std::domain_error("unknown --op " + op);
    const bool shifted = a.str("indexing", "base_p") == "binary_shift";
    const GfqField F =
        GfqField::build(p, k, gfq_default_q(p, k), shifted ? TableIndexing::binary_shift : TableIndexing::base_p);
    if (a.flag("dump-field")) {
        std::cout << F.describe();
        return 0;
    }
    const CsvLog log(a.str("csv"));
    SplitMix64 draws(a.u("seed", 42));
    auto random_element = [&] { return F.from_index(draws.below(F.order())); };
    // the device row and the host row of one comparison share shape and checksum rules
    auto rows = [&](u64 n) {
        Measurement dev;
        dev.prime = p;
        dev.radix = F.params().q;
        dev.chunk = k;
        dev.size = n;
        dev.group = F.params().n_q;
        Measurement host = dev;
        dev.tag = "fgdp_b200";
        host.tag = "naive_dot";
        return std::pair<Measurement, Measurement>{dev, host};
    };
    auto field_dot = [&](auto&& lhs_at, auto&& rhs_at, u64 terms) {
        GfqElt sum = F.zero();
        for (u64 l = 0; l < terms; ++l) sum = F.add(sum, F.mul(lhs_at(l), rhs_at(l)));
        return sum;
    };
    if (op == "dot") {
        const u64 len = a.u("len", 100);
        std::vector<GfqElt> lhs(len), rhs(len);
        for (u64 i = 0; i < len; ++i) {
            lhs[i] = random_element();
            rhs[i] = random_element();
        }
        auto [dev, host] = rows(len);
        const Stopwatch t_dev;
        const GfqElt got = gpu::fgdp_dot(lhs, rhs, F, &dev.counted);  // K5 on the device
        dev.elapsed_ns = t_dev.ns();
        const Stopwatch t_host;
        const GfqElt want = field_dot([&](u64 l) { return lhs[l]; }, [&](u64 l) { return rhs[l]; }, len);
        host.elapsed_ns = t_host.ns();
        const std::vector<u64> got_c = F.to_coeffs(got), want_c = F.to_coeffs(want);
        dev.fnv = fold_checksum(got_c.data(), got_c.size());
        host.fnv = fold_checksum(want_c.data(), want_c.size());
        log.add(dev);
        log.add(host);
        const u64 groups = (len + F.params().n_q - 1) / F.params().n_q;
        std::cout << "gfq dot p=" << p << " k=" << k << " len=" << len << " divisions=" << dev.counted.divisions
                  << " (expected " << groups << ") table_accesses=" << dev.counted.table_accesses
                  << " agreement=" << (got_c == want_c ? "ok" : "MISMATCH") << "\n";
        return got_c == want_c ? 0 : 3;
    }
    const u64 side = a.u("size", 8);
    GfqMatrix lhs = GfqMatrix::zero(F, side, side), rhs = GfqMatrix::zero(F, side, side);
    for (GfqMatrix* mat : {&lhs, &rhs})
        for (GfqElt& e : mat->data) e = random_element();
    auto [dev, host] = rows(side);
    const Stopwatch t_dev;
    const GfqMatrix got = gfq_matmul(lhs, rhs, F, &dev.counted);  // K1 + K4 on the device
    dev.elapsed_ns = t_dev.ns();
    const Stopwatch t_host;
    std::vector<u64> want_index;
    bool agree = true;
    for (u64 i = 0; i < side; ++i)
        for (u64 j = 0; j < side; ++j) {
            const GfqElt e = field_dot([&](u64 l) { return lhs.at(i, l); }, [&](u64 l) { return rhs.at(l, j); }, side);
            agree = agree && got.at(i, j) == e;
            want_index.push_back(F.to_index(e));
        }
    host.elapsed_ns = t_host.ns();
    dev.fnv = host.fnv = fold_checksum(want_index.data(), want_index.size());
    log.add(dev);
    log.add(host);
    std::cout << "gfq matmul p=" << p << " k=" << k << " size=" << side << " divisions=" << dev.counted.divisions
              << " agreement=" << (agree ? "ok" : "MISMATCH") << "\n";
    return agree ? 0 : 3;
}

const char* kUsage =
    "usage: qpack_b200 <mulpoly|paper-examples|gfq> [options]\n"
    "  mulpoly --p P --n N [--d D] [--algo fqt|oracle] [--seed S] [--repeat R] [--csv F] [--m M]\n"
    "          [--no-verify] [--a c0,c1,.. --b c0,c1,..]\n"
    "  paper-examples [--inject-fault]\n"
    "  gfq --p P --k K [--op dot|matmul] [--len L] [--size S] [--seed S] [--csv F]\n"
    "      [--indexing base_p|binary_shift] [--dump-field]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << kUsage;
        return 1;
    }
    const std::string sub = argv[1];
    Args args;
    static const char* kFlags[] = {"no-verify", "inject-fault", "dump-field"};
    for (int i = 2; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) {
            std::cerr << "unexpected argument " << t << "\n" << kUsage;
            return 1;
        }
        t = t.substr(2);
        bool is_flag = false;
        for (const char* f : kFlags) is_flag |= t == f;
        if (is_flag) {
            args.flags[t] = true;
        } else if (const auto eq = t.find('='); eq != std::string::npos) {
            args.kv[t.substr(0, eq)] = t.substr(eq + 1);
        } else if (i + 1 < argc) {
            args.kv[t] = argv[++i];
        } else {
            std::cerr << "missing value for --" << t << "\n";
            return 1;
        }
    }
    try {
        if (sub == "mulpoly") return cmd_mulpoly(args);
        if (sub == "paper-examples") return cmd_paper_examples(args);
        if (sub == "gfq") return cmd_gfq(args);
        std::cerr << kUsage;
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
