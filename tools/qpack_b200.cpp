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
#include <chrono>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
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

using namespace qpack;

namespace {

struct Row {
    std::string algo;
    u64 p = 0, q = 0;
    u32 k = 0, d = 0;
    u64 n = 0, n_q = 0, n_d = 0;
    CostReport cost;
    u64 wall_ns = 0;
    u64 checksum = 0;
};

void append_csv(const std::string& path, const Row& r) {
    if (path.empty()) return;
    const bool fresh = !std::filesystem::exists(path) || std::filesystem::file_size(path) == 0;
    std::ofstream out(path, std::ios::app);
    if (!out) throw std::runtime_error("cannot open csv file " + path);
    if (fresh) out << "algo,p,q,k,d,N,n_q,n_d,mul_add,divisions,table_accesses,wall_time_ns,checksum\n";
    out << r.algo << ',' << r.p << ',' << r.q << ',' << r.k << ',' << r.d << ',' << r.n << ',' << r.n_q << ','
        << r.n_d << ',' << r.cost.mul_add << ',' << r.cost.divisions << ',' << r.cost.table_accesses << ','
        << r.wall_ns << ',' << std::hex << std::setw(16) << std::setfill('0') << r.checksum << std::dec
        << std::setfill(' ') << '\n';
}

u64 now_ns() {
    return static_cast<u64>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
            .count());
}

// QPACK_TABLE_CACHE: load the plan's table if cached, else save it
void wire_table_cache(RedqPlan& plan) {
    const char* dir = std::getenv("QPACK_TABLE_CACHE");
    if (!dir || !plan.correction) return;
    const CorrectionTable& t = *plan.correction;
    std::ostringstream name;
    name << dir << "/redq_p" << t.p << "_q" << t.q << "_w" << t.k_window << "_"
         << (t.indexing == TableIndexing::base_p ? "basep" : "shift") << ".tbl";
    const std::string path = name.str();
    if (std::filesystem::exists(path)) {
        std::ifstream in(path, std::ios::binary);
        plan.attach_correction(load_correction_table(in));
        return;
    }
    std::filesystem::create_directories(dir);
    std::ofstream out(path, std::ios::binary);
    save_correction_table(t, out);
}

std::vector<u64> parse_list(const std::string& s, u64 p) {
    std::vector<u64> v;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) v.push_back(std::stoull(item) % p);
    return v;
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
    const u64 p = a.u("p", 3), n = a.u("n", 100), seed = a.u("seed", 42);
    const u32 m = static_cast<u32>(a.u("m", 53));
    const unsigned repeat = static_cast<unsigned>(a.u("repeat", 1));
    const std::string algo = a.str("algo", "fqt"), csv = a.str("csv");
    const bool no_verify = a.flag("no-verify");
    if (algo == "delayed") throw std::domain_error("--algo delayed is not part of qpack-b200 (host-only variant)");
    if (algo != "fqt" && algo != "oracle") throw std::domain_error("unknown --algo " + algo);
    SplitMix64 rng(seed);
    QadicParams params{};
    RedqPlan plan;
    if (algo == "fqt") {
        params = a.has("d") ? qadic_for_degree(p, static_cast<u32>(a.u("d", 0)), m) : best_qadic(p, m, 1, true);
        plan = fqt_reduction_plan(params, params.k - 1);
        wire_table_cache(plan);
    }
    for (unsigned rep = 0; rep < repeat; ++rep) {
        DensePoly x{p, {}}, y{p, {}};
        if (a.has("a") || a.has("b")) {
            x.coeffs = parse_list(a.str("a"), p);
            y.coeffs = parse_list(a.str("b"), p);
            if (x.coeffs.empty() || y.coeffs.empty())
                throw std::domain_error("--a and --b must both be given for fixed inputs");
        } else {
            for (u64 i = 0; i <= n; ++i) x.coeffs.push_back(rng.below(p));
            for (u64 i = 0; i <= n; ++i) y.coeffs.push_back(rng.below(p));
        }
        Row r;
        r.algo = algo == "fqt" ? "fqt_b200" : "oracle";
        r.p = p;
        r.n = n;
        DensePoly out{p, {}};
        const u64 t0 = now_ns();
        if (algo == "fqt") {
            out = fqt_mul(x, y, params.k - 1, params, plan, &r.cost);  // K6 on the device (m <= 53)
            r.q = params.q;
            r.k = params.k;
            r.d = params.k - 1;
            r.n_q = params.n_q;
        } else {
            out = schoolbook(x, y);
        }
        r.wall_ns = now_ns() - t0;
        r.checksum = fold_checksum(out.coeffs.data(), out.coeffs.size());
        if (!no_verify && algo != "oracle" && !(out == schoolbook(x, y))) {
            std::cerr << "verification FAILED against the schoolbook product\n";
            return 3;
        }
        append_csv(csv, r);
        std::cout << r.algo << " p=" << p << " N=" << n << " rep=" << rep << " mul_add=" << r.cost.mul_add
                  << " divisions=" << r.cost.divisions << " table_accesses=" << r.cost.table_accesses
                  << " wall_ns=" << r.wall_ns << " checksum=" << std::hex << r.checksum << std::dec
                  << (no_verify || algo == "oracle" ? "" : " verified=ok") << "\n";
    }
    return 0;
}

int cmd_paper_examples(const Args& a) {
    int bad = 0;
    auto check = [&](const std::string& what, const std::string& got, const std::string& want) {
        const bool ok = got == want;
        std::cout << (ok ? "  ok   " : "  FAIL ") << what << ": " << got;
        if (!ok) std::cout << " (expected " << want << ")";
        std::cout << "\n";
        bad += ok ? 0 : 1;
    };
    auto fmt = [](const std::vector<u64>& v) {
        std::string s = "[";
        for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
        return s + "]";
    };
    std::cout << "[1] radix-100 product over Z/3Z\n";
    const QadicParams ex1{3, 100, 2, 1, 53};
    const Packed prod1 = dqt_mul(pack(DensePoly{3, {1, 1}}, ex1), pack(DensePoly{3, {2, 1}}, ex1));
    check("101 x 102", to_string(prod1.value), "10302");
    check("digits", fmt(unpack(prod1, 3)), "[2,3,1]");
    check("reduced", dqt_mul_poly(DensePoly{3, {1, 1}}, DensePoly{3, {2, 1}}, ex1) == DensePoly{3, {2, 0, 1}}
                         ? "X^2+2" : "?",
          "X^2+2");

    std::cout << "[2] five residues reduced at once (p | q)\n";
    const u128 prod2 = static_cast<u128>(100020003) * 400050006;
    check("packed product", to_string(prod2), "40013002800270018");
    check("reduced word", to_string(redq(prod2, RedqPlan::build(5, 10000, 4))), "40003000300020003");

    std::cout << "[3] full correction at p=23, q=10^6\n";
    const RedqTrace t3 = redq_trace(parse_u128("1234005678009123004567"), RedqPlan::build(23, 1000000, 3));
    check("rop", to_string(t3.rop), "53652420783005348024");
    check("u", fmt(t3.u), "[15,8,18,15]");
    check("mu", fmt(t3.mu), "[13,15,20,15]");

    std::cout << "[4] degree-6 correction through three window lookups\n";
    CorrectionTable q2 = build_correction_table(23, 1000000, 3, TableIndexing::base_p);
    if (a.flag("inject-fault"))
        for (u64& e : q2.entries) e ^= 1;  // a corrupted cache must be detected
    const RedqPlan plan4 = RedqPlan::build(23, 1000000, 6);
    SplitMix64 rng(4);
    bool windows_ok = true;
    u64 accesses = 0;
    for (int it = 0; it < 500; ++it) {
        std::vector<u64> u(7);
        for (u64& v : u) v = rng.below(23);
        CostReport cost;
        if (correct_tabulated(u, q2, &cost) != correct_direct(u, plan4)) windows_ok = false;
        accesses = cost.table_accesses;
    }
    check("window accesses", std::to_string(accesses), "3");
    check("tabulated == direct", windows_ok ? "yes" : "no", "yes");

    std::cout << "[5] the same reductions on the device (batched REDQ kernels)\n";
    {
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
        check("device residues == host", same ? "yes" : "no", "yes");
    }
    std::cout << (bad == 0 ? "all examples reproduced\n" : "MISMATCHES FOUND\n");
    return bad == 0 ? 0 : 4;
}

int cmd_gfq(const Args& a) {
    if (!a.has("p") || !a.has("k")) throw std::invalid_argument("gfq: --p and --k are required");
    const u64 p = a.u("p", 3), len = a.u("len", 100), size = a.u("size", 8), seed = a.u("seed", 42);
    const u32 k = static_cast<u32>(a.u("k", 2));
    const std::string op = a.str("op", "dot"), csv = a.str("csv");
    const TableIndexing idx =
        a.str("indexing", "base_p") == "binary_shift" ? TableIndexing::binary_shift : TableIndexing::base_p;
    const GfqField field = GfqField::build(p, k, gfq_default_q(p, k), idx);
    if (a.flag("dump-field")) {
        std::cout << field.describe();
        return 0;
    }
    SplitMix64 rng(seed);
    auto fill = [&](Row& r, u64 n) {
        r.p = p;
        r.q = field.params().q;
        r.k = k;
        r.n = n;
        r.n_q = field.params().n_q;
    };
    if (op == "dot") {
        std::vector<GfqElt> v1(len), v2(len);
        for (u64 i = 0; i < len; ++i) {
            v1[i] = field.from_index(rng.below(field.order()));
            v2[i] = field.from_index(rng.below(field.order()));
        }
        Row packed, naive;
        packed.algo = "fgdp_b200";
        naive.algo = "naive_dot";
        u64 t0 = now_ns();
        const GfqElt got = gpu::fgdp_dot(v1, v2, field, &packed.cost);  // K5 on the device
        packed.wall_ns = now_ns() - t0;
        t0 = now_ns();
        GfqElt want = field.zero();
        for (u64 i = 0; i < len; ++i) want = field.add(want, field.mul(v1[i], v2[i]));
        naive.wall_ns = now_ns() - t0;
        const std::vector<u64> gc = field.to_coeffs(got), wc = field.to_coeffs(want);
        fill(packed, len);
        fill(naive, len);
        packed.checksum = fold_checksum(gc.data(), gc.size());
        naive.checksum = fold_checksum(wc.data(), wc.size());
        append_csv(csv, packed);
        append_csv(csv, naive);
        const bool agree = gc == wc;
        const u64 expected = len == 0 ? 0 : (len + field.params().n_q - 1) / field.params().n_q;
        std::cout << "gfq dot p=" << p << " k=" << k << " len=" << len << " divisions=" << packed.cost.divisions
                  << " (expected " << expected << ") table_accesses=" << packed.cost.table_accesses
                  << " agreement=" << (agree ? "ok" : "MISMATCH") << "\n";
        return agree ? 0 : 3;
    }
    if (op == "matmul") {
        GfqMatrix x = GfqMatrix::zero(field, size, size), y = GfqMatrix::zero(field, size, size);
        for (GfqElt& e : x.data) e = field.from_index(rng.below(field.order()));
        for (GfqElt& e : y.data) e = field.from_index(rng.below(field.order()));
        Row packed, naive;
        packed.algo = "fgdp_b200";
        naive.algo = "naive_dot";
        u64 t0 = now_ns();
        const GfqMatrix c = gfq_matmul(x, y, field, &packed.cost);  // K1 + K4 on the device
        packed.wall_ns = now_ns() - t0;
        t0 = now_ns();
        GfqMatrix want = GfqMatrix::zero(field, size, size);
        for (u64 i = 0; i < size; ++i)
            for (u64 j = 0; j < size; ++j) {
                GfqElt acc = field.zero();
                for (u64 l = 0; l < size; ++l) acc = field.add(acc, field.mul(x.at(i, l), y.at(l, j)));
                want.at(i, j) = acc;
            }
        naive.wall_ns = now_ns() - t0;
        const bool agree = c.data == want.data;
        std::vector<u64> folded;
        for (const GfqElt& e : want.data) folded.push_back(field.to_index(e));
        fill(packed, size);
        fill(naive, size);
        packed.checksum = naive.checksum = fold_checksum(folded.data(), folded.size());
        append_csv(csv, packed);
        append_csv(csv, naive);
        std::cout << "gfq matmul p=" << p << " k=" << k << " size=" << size << " divisions=" << packed.cost.divisions
                  << " agreement=" << (agree ? "ok" : "MISMATCH") << "\n";
        return agree ? 0 : 3;
    }
    throw std::domain_error("unknown --op " + op);
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
