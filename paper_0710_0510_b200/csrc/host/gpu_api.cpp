// GPU layer of qpack-b200: device mirrors of plans and fields, the batched
// qpack::gpu entry points and the gfq_matmul drop-in.  No CPU fallback: every
// entry point here runs the sm_100a kernels or throws.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <tuple>

#include "device_state.hpp"
#include "gpu_internal.hpp"
#include "qpack/gpu.hpp"
#include "qpack/polymul.hpp"

namespace qpack::gpu {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw device_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw device_error(std::string("qpack-b200: no CUDA device available (") + cudaGetErrorString(e) + ")");
}

DevBuf::~DevBuf() {
    if (ptr) cudaFree(ptr);
}

void* DevBuf::ensure(std::size_t n) {
    if (n <= bytes && ptr) return ptr;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    check(cudaMalloc(&ptr, std::max<std::size_t>(n, 16)), "cudaMalloc");
    bytes = std::max<std::size_t>(n, 16);
    return ptr;
}

StreamBuf::StreamBuf(std::size_t bytes, cudaStream_t stream) : s(stream) {
    // keep freed workspace in the device's default pool across calls (the
    // default release threshold of 0 would hand it back to the OS at every
    // synchronisation, and re-mapping 1 GB costs milliseconds)
    static const bool pool_kept = [] {
        int dev = 0;
        cudaMemPool_t pool = nullptr;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return true;
    }();
    (void)pool_kept;
    if (bytes) check(cudaMallocAsync(&ptr, bytes, s), "cudaMallocAsync");
}

StreamBuf::~StreamBuf() {
    if (ptr) cudaFreeAsync(ptr, s);
}

Staging::Staging() {
    for (cudaStream_t* s : {&sh, &sk, &sd, &sk2})
        check(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking), "cudaStreamCreate");
    check(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming), "cudaEventCreate");
    for (int i = 0; i < kSlots; ++i)
        for (cudaEvent_t* e : {&ev_in[i], &ev_k[i], &ev_out[i]})
            check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
}

Staging::~Staging() {
    for (int i = 0; i < kSlots; ++i)
        for (cudaEvent_t e : {ev_in[i], ev_k[i], ev_out[i]})
            if (e) cudaEventDestroy(e);
    if (ev_aux) cudaEventDestroy(ev_aux);
    for (cudaStream_t s : {sh, sk, sd, sk2})
        if (s) cudaStreamDestroy(s);
}

}  // namespace qpack::gpu

namespace qpack::detail {

using gpu::check;

// Plan/field constants and status words are written by cudaMemcpy/cudaMemset
// on the legacy stream; a pageable cudaMemcpy may return before its DMA lands
// and cudaMemset is asynchronous, while the kernels that read them run on the
// caller's (possibly non-blocking) stream -- and the stream kernels stage
// their tables before the PDL wait.  Wait for those writes once, at build.
void settle_uploads() { check(cudaStreamSynchronize(nullptr), "upload sync"); }

qpk::RedqParams make_redq_params(const RedqPlan& plan, gpu::DevBuf* table) {
    if (plan.p > 256) throw std::invalid_argument("qpack-b200 REDQ: residues are emitted as uint8, p must be <= 256");
    if (plan.d + 1 > static_cast<unsigned>(qpk::kMaxDigits))
        throw std::invalid_argument("qpack-b200 REDQ: at most 64 digits per word");
    qpk::RedqParams P{};
    P.p = static_cast<uint32_t>(plan.p);
    P.d = plan.d;
    P.qbits = is_pow2(plan.q) ? bit_width_u128(plan.q) - 1 : 0;
    P.neg_q = static_cast<uint32_t>(plan.neg_q_mod_p);
    P.mod_magic = static_cast<uint32_t>(((u64(1) << 32) + plan.p - 1) / plan.p);
    P.float_mode = plan.mode == RedqMode::float_premul;
    P.inv_p = plan.inv_p.inv_up;
    P.r_max = static_cast<double>(plan.inv_p.r_max);
    P.q = plan.q;
    // words must lie below min(q^(d+1), 2^53)
    const u128 two53 = u128(1) << 53;
    P.limit = (pow_fits_u128(plan.q, plan.d + 1) && checked_pow_u128(plan.q, plan.d + 1) < two53)
                  ? static_cast<double>(static_cast<u64>(checked_pow_u128(plan.q, plan.d + 1)))
                  : 9007199254740992.0;
    const u128 two64 = u128(1) << 64;
    P.limit_u64 = (pow_fits_u128(plan.q, plan.d + 1) && checked_pow_u128(plan.q, plan.d + 1) < two64)
                      ? static_cast<u64>(checked_pow_u128(plan.q, plan.d + 1))
                      : 0;
    {
        u128 pw64 = 1;
        for (unsigned i = 0; i <= plan.d; ++i) {
            P.qpow64[i] = pw64 < two64 ? static_cast<u64>(pw64) : 0;
            if (pw64 < two64) pw64 *= plan.q;
        }
    }
    u128 pw = 1;
    for (unsigned i = 0; i <= plan.d; ++i) {
        const bool small = pw < two53;
        P.qpow[i] = small ? static_cast<uint64_t>(pw) : (uint64_t(1) << 63);
        P.inv_q[i] = small ? ReciprocalDivisor::make(static_cast<u64>(pw)).inv_up : 0.0;  // r < 2^53 <= q^i -> 0
        if (pw < two53) pw *= plan.q;
    }
    // tabulated correction on the device when the window table fits shared memory
    P.window = 0;
    if (plan.neg_q_mod_p != 0 && plan.correction && plan.d > 0) {
        const CorrectionTable& t = *plan.correction;
        if (t.k_window >= 2 && t.k_window <= 4 && t.entries.size() <= 16384 && table) {
            std::vector<uint32_t> packed(t.entries.size());
            for (std::size_t idx = 0; idx < t.entries.size(); ++idx) {
                u64 e = t.entries[idx];
                uint32_t w = 0;
                for (u32 j = 0; j < t.k_window; ++j, e /= t.radix) w |= static_cast<uint32_t>(e % t.radix) << (8 * j);
                packed[idx] = w;
            }
            table->ensure(packed.size() * 4);
            check(cudaMemcpy(table->ptr, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice), "table upload");
            P.window = t.k_window;
            P.radix = static_cast<uint32_t>(t.radix);
            P.n_entries = static_cast<uint32_t>(t.entries.size());
            P.table = table->as<uint32_t>();
        }
        // otherwise: direct correction on the device (identical residues,
        // test_redq.cpp "correction table reproduces the direct formula")
    }
    return P;
}

// The device mirrors hang off const plans and fields (the reference
// functions are reentrant on shared const objects): their lazy creation is
// serialised by one process-wide lock, held for every lookup.
std::mutex g_mirror_mu;

DevicePlanCache& device_plan(const RedqPlan& plan) {
    std::lock_guard<std::mutex> lock(g_mirror_mu);
    if (!plan.device) {
        gpu::require_device();
        auto c = std::make_shared<DevicePlanCache>();
        c->prm = make_redq_params(plan, &c->table);
        c->gen = plan.correction_gen;
        c->status.ensure(4);
        check(cudaMemset(c->status.ptr, 0, 4), "status init");
        settle_uploads();
        plan.device = std::move(c);
    } else if (plan.device->gen != plan.correction_gen) {
        // a table was attached since the upload: launches still in flight may
        // read the old table, so the device drains before it is replaced; the
        // latched error word is kept
        DevicePlanCache& c = *plan.device;
        std::lock_guard<std::mutex> lk(c.mu);
        check(cudaDeviceSynchronize(), "drain before a table swap");
        c.prm = make_redq_params(plan, &c.table);
        c.gen = plan.correction_gen;
        settle_uploads();
    }
    return *plan.device;
}

CostReport redq_batch_cost(const RedqPlan& plan, u64 n) {
    CostReport c;
    c.divisions = n;
    c.reduction_calls = n;
    if (plan.neg_q_mod_p != 0 && plan.correction && plan.d > 0) {
        const u64 w = plan.correction->k_window;
        c.table_accesses = n * ((plan.d + w - 2) / (w - 1));
    }
    return c;
}

// GF(p^k) outside the byte-packed form (k > 4 or p > 255): the rep-domain
// tables of gfq_wide.cu in global memory (they may exceed shared memory)
std::shared_ptr<DeviceFieldCache> build_wide_field(const GfqField& f) {
    const u64 p = f.p(), q = FieldAccess::q(f), order = f.order();
    const u32 k = f.k();
    if (k > qpk::kMaxWideK) throw std::invalid_argument("qpack-b200 GF(p^k): k <= 8 (every field with q^(2k-1) < 2^53)");
    auto c = std::make_shared<DeviceFieldCache>();
    c->wide = true;
    std::vector<uint32_t> host;
    const std::vector<u32>& lg = FieldAccess::log(f);
    const std::vector<u64>& al = FieldAccess::antilog(f);
    const std::vector<u32>& lo = FieldAccess::low(f);
    const std::vector<u32>& hi = FieldAccess::high(f);
    const std::vector<u32>& z = FieldAccess::zech(f);
    host.insert(host.end(), lg.begin(), lg.end());
    for (const u64 v : al) host.push_back(static_cast<uint32_t>(v));
    host.insert(host.end(), lo.begin(), lo.end());
    host.insert(host.end(), hi.begin(), hi.end());
    host.insert(host.end(), z.begin(), z.end());
    c->wide_tabs.ensure(host.size() * 4);
    check(cudaMemcpy(c->wide_tabs.ptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice), "field tables upload");
    c->fval.ensure(order * 8);
    check(cudaMemcpy(c->fval.ptr, FieldAccess::fval(f).data(), order * 8, cudaMemcpyHostToDevice), "fval upload");
    c->status.ensure(4);
    check(cudaMemset(c->status.ptr, 0, 4), "status init");
    settle_uploads();
    qpk::GfqWideParams& W = c->wp;
    W.p = static_cast<uint32_t>(p);
    W.k = k;
    W.order = static_cast<uint32_t>(order);
    W.group = static_cast<uint32_t>(order - 1);
    W.lh_radix = static_cast<uint32_t>(FieldAccess::lh_radix(f));
    W.qbits = is_pow2(q) ? bit_width_u128(q) - 1 : 0;
    W.chunk = static_cast<uint32_t>(f.params().n_q);
    u64 qi = 1;
    for (u32 i = 0; i < 2 * k - 1; ++i, qi *= q) W.qpow[i] = qi;
    W.qpow[1] = q;  // also for k = 1 (the DQT pack reads it)
    W.fval = c->fval.as<double>();
    const uint32_t* t = c->wide_tabs.as<uint32_t>();
    W.log = t;
    W.antilog = t + order;
    W.low = t + 2 * order;
    W.high = W.low + lo.size();
    W.zech = W.high + hi.size();
    W.status = c->status.as<uint32_t>();
    // the generic helpers (coefficient records -> reps, rep ops) read these
    c->elem.p = W.p;
    c->elem.k = k;
    c->elem.order = W.order;
    c->elem.group = W.group;
    c->elem.log = W.log;
    return c;
}

DeviceFieldCache& device_field(const GfqField& f) {
    std::lock_guard<std::mutex> lock(g_mirror_mu);
    auto& slot = FieldAccess::device(f);
    if (slot) return *slot;
    gpu::require_device();
    const u64 p = f.p();
    const u32 k = f.k();
    if (p > 255 || k > static_cast<u32>(qpk::kMaxGfqK)) {
        slot = build_wide_field(f);
        return *slot;
    }
    auto c = std::make_shared<DeviceFieldCache>();
    const u64 lh = FieldAccess::lh_radix(f);
    u64 nlh = 1;
    for (u32 i = 0; i < k; ++i) nlh *= lh;
    const u64 order = f.order();
    // the compile-time fast path (GF(7^3) at q = 2^8, stream_kernels.cuh
    // GfqElemOp::fast) gets one more block, at the base-p index of three
    // coefficients or digits: L as u16 | H | log (pre-scaled antilog byte
    // offsets) | kDlogCopies interleaved copies of the doubled antilog table
    const bool fast = qpk::gfq_fast_field(p, k, FieldAccess::q(f));
    const u64 base_words = 2 * nlh + 2 * order;
    const u64 group = order - 1;
    const u64 nc = qpk::kDlogCopies;
    const u64 p3 = p * p * p;
    const u64 fast_off = (base_words + 3) / 4 * 4;  // 16-byte aligned
    const u64 alog_off = ((p3 + 1) / 2 + 2 * p3 + 3) / 4 * 4;  // 16-byte aligned (vector staging)
    const u64 fast_words = alog_off + 2 * group * nc;
    const u64 words = fast ? fast_off + fast_words : base_words;
    // a launch stages the tables its path reads (the fast path: 32
    // lane-private copies of L|H, or of log plus the antilog copies)
    const u64 staged = fast ? 32 * ((p3 + 1) / 2 + p3) : base_words;
    if (staged * 4 > 96 * 1024)
        throw std::invalid_argument("qpack-b200 GF(p^k): field tables exceed the shared-memory budget");
    // coefficient-form tables: rep -> packed coefficient bytes
    auto bytes_of = [&](u32 rep) {
        uint32_t w = 0;
        const std::vector<u64> cf = f.to_coeffs(GfqElt{rep});
        for (u32 i = 0; i < k; ++i) w |= static_cast<uint32_t>(cf[i]) << (8 * i);
        return w;
    };
    std::vector<uint32_t> host(words);
    for (u64 i = 0; i < nlh; ++i) {
        host[i] = bytes_of(FieldAccess::low(f)[i]);
        host[nlh + i] = bytes_of(FieldAccess::high(f)[i]);
    }
    for (u64 i = 0; i < order; ++i) {
        host[2 * nlh + i] = FieldAccess::log(f)[i];
        host[2 * nlh + order + i] = bytes_of(static_cast<u32>(i));
    }
    if (fast) {
        auto* l16 = reinterpret_cast<uint16_t*>(host.data() + fast_off);
        uint32_t* h32 = host.data() + fast_off + (p3 + 1) / 2;
        uint32_t* lg32 = h32 + p3;
        uint32_t* alR = host.data() + fast_off + alog_off;
        for (u64 d2 = 0; d2 < p; ++d2)
            for (u64 d1 = 0; d1 < p; ++d1)
                for (u64 d0 = 0; d0 < p; ++d0) {
                    const u64 lh_idx = d0 + lh * (d1 + lh * d2);
                    const u64 e = d0 + p * (d1 + p * d2);
                    // the low half has degree < k-1 = 2: two coefficient bytes
                    if (host[lh_idx] >> 16) throw std::logic_error("qpack-b200: low-half table entry of degree >= 2");
                    l16[e] = static_cast<uint16_t>(host[lh_idx]);
                    h32[e] = host[nlh + lh_idx];
                    const u64 lg = FieldAccess::log(f)[e];  // zero -> the sentinel g
                    lg32[e] = static_cast<uint32_t>(4 * nc * (lg == group ? 2 * group - 1 : lg));
                }
        // rep i mod g for i < 2g-1, zero at 2g-1: a sum of two logs indexes it
        // with no reduction mod g, and any sum involving zero clamps to 2g-1
        for (u64 i = 0; i < 2 * group; ++i) {
            const uint32_t v = i + 1 < 2 * group ? bytes_of(static_cast<u32>(i % group)) : 0u;
            for (u64 cp = 0; cp < nc; ++cp) alR[i * nc + cp] = v;
        }
    }
    c->tables.ensure(words * 4);
    check(cudaMemcpy(c->tables.ptr, host.data(), words * 4, cudaMemcpyHostToDevice), "field tables upload");
    c->fval.ensure(order * 8);
    check(cudaMemcpy(c->fval.ptr, FieldAccess::fval(f).data(), order * 8, cudaMemcpyHostToDevice), "fval upload");
    c->status.ensure(4);
    check(cudaMemset(c->status.ptr, 0, 4), "status init");
    settle_uploads();
    c->nlh = static_cast<uint32_t>(nlh);

    const RedqPlan digits = RedqPlan::build(p, FieldAccess::q(f), 2 * k - 2, RedqMode::integer);
    const qpk::RedqParams rq = make_redq_params(digits, nullptr);
    const uint32_t* tb = c->tables.as<uint32_t>();
    qpk::GfqElemParams& E = c->elem;
    E.rq = rq;
    E.k = k;
    E.p = static_cast<uint32_t>(p);
    E.order = static_cast<uint32_t>(order);
    E.group = static_cast<uint32_t>(order - 1);
    E.lh_radix = static_cast<uint32_t>(lh);
    E.qd = static_cast<double>(FieldAccess::q(f));
    E.lc = tb;
    E.hc = tb + nlh;
    E.log = tb + 2 * nlh;
    E.alog = tb + 2 * nlh + order;
    E.tables_words = static_cast<uint32_t>(words);
    E.fast_off = fast ? static_cast<uint32_t>(fast_off) : 0u;
    if (k == 3) {
        const std::vector<u64> xv = {0, 1, 0};
        const GfqElt x = f.from_coeffs(xv);
        E.col3 = bytes_of(f.pow(x, 3).rep);
        E.col4 = bytes_of(f.pow(x, 4).rep);
    }
    qpk::GfqMatmulParams& M = c->mm;
    M.rq = rq;
    M.k = k;
    M.p = E.p;
    M.order = E.order;
    M.group = E.group;
    M.lh_radix = E.lh_radix;
    M.qd = E.qd;
    M.lc = E.lc;
    M.hc = E.hc;
    M.log = E.log;
    M.fval = c->fval.as<double>();
    qpk::GfqGemvParams& G = c->gemv;
    G.rq = rq;
    G.k = k;
    G.p = E.p;
    G.order = E.order;
    G.lh_radix = E.lh_radix;
    G.lc = E.lc;
    G.log = E.log;
    G.fval = M.fval;
    G.status = c->status.as<uint32_t>();
    G.vals32 = 1;
    for (const double v : FieldAccess::fval(f)) G.vals32 &= v < 4294967296.0 ? 1u : 0u;
    slot = std::move(c);
    return *slot;
}

}  // namespace qpack::detail

namespace qpack::gpu {

using detail::DeviceFieldCache;
using detail::DevicePlanCache;

uint32_t take_status(DevicePlanCache& dp, cudaStream_t s) {
    check(cudaStreamSynchronize(s), "stream sync");
    uint32_t st = 0;
    check(cudaMemcpy(&st, dp.status.ptr, 4, cudaMemcpyDeviceToHost), "status read");
    if (st) {
        check(cudaMemset(dp.status.ptr, 0, 4), "status clear");
        detail::settle_uploads();
    }
    return st;
}

void raise_status(uint32_t st) {
    if (st & qpk::kErrDomain) throw std::domain_error("redq: input exceeds q^(d+1), digits are not all below q");
    if (st & qpk::kErrOutOfRange) throw std::out_of_range("floor_div_premul: numerator exceeds guaranteed range r_max");
}

// The field's error word (kErrRep: a rep >= p^k, read as zero; kErrDomain:
// the inverse of zero): every launch on the field ORs into it, whatever its
// stream; reading it waits for stream `s` and clears it.
uint32_t take_field_status(DeviceFieldCache& F, cudaStream_t s) {
    check(cudaStreamSynchronize(s), "stream sync");
    uint32_t st = 0;
    check(cudaMemcpy(&st, F.status.ptr, 4, cudaMemcpyDeviceToHost), "status read");
    if (st) {
        check(cudaMemset(F.status.ptr, 0, 4), "status clear");
        detail::settle_uploads();
    }
    return st;
}

void raise_field_status(uint32_t st) {
    if (st & qpk::kErrRep) throw std::out_of_range("GfqField: rep outside the field");
    if (st & qpk::kErrDomain) throw std::domain_error("GfqField: zero has no inverse");
}

void redq_device(DevicePlanCache& dp, const double* d_words, u64 n, uint8_t* d_out, cudaStream_t s) {
    check(qpk::launch_redq_f64(dp.prm, d_words, n, d_out, dp.status.as<uint32_t>(), s), "redq launch");
}

void redq_device_u64(DevicePlanCache& dp, const uint64_t* d_words, u64 n, uint8_t* d_out, cudaStream_t s) {
    check(qpk::launch_redq_u64(dp.prm, d_words, n, d_out, dp.status.as<uint32_t>(), s), "redq launch");
}

void redq_device_u128(DevicePlanCache& dp, const uint64_t* d_words, u64 n, uint8_t* d_out, cudaStream_t s) {
    check(qpk::launch_redq_u128(dp.prm, d_words, n, d_out, dp.status.as<uint32_t>(), s), "redq launch");
}

// u128 words as (lo, hi) pairs, same chunked pipeline as the u64 words
void redq_host_u128(DevicePlanCache& dp, const uint64_t* h_words, u64 n, uint8_t* h_out) {
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.staging) dp.staging = std::make_unique<Staging>();
    Staging& S = *dp.staging;
    const u64 nd = dp.prm.d + 1, chunk = u64(1) << 20;
    for (int sl = 0; sl < Staging::kSlots; ++sl) {
        S.in0[sl].ensure(chunk * 16);
        S.out[sl].ensure(chunk * nd);
    }
    S.run(
        n, chunk,
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(S.in0[sl].ptr, h_words + 2 * off, cnt * 16, cudaMemcpyHostToDevice, s), "H2D");
        },
        [&](int sl, u64, u64 cnt, cudaStream_t s) {
            redq_device_u128(dp, S.in0[sl].as<uint64_t>(), cnt, S.out[sl].as<uint8_t>(), s);
        },
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(h_out + off * nd, S.out[sl].ptr, cnt * nd, cudaMemcpyDeviceToHost, s), "D2H");
        });
    raise_status(take_status(dp, S.sk));
}

void redq_host_u64(DevicePlanCache& dp, const uint64_t* h_words, u64 n, uint8_t* h_out) {
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.staging) dp.staging = std::make_unique<Staging>();
    Staging& S = *dp.staging;
    const u64 nd = dp.prm.d + 1, chunk = u64(1) << 21;
    for (int sl = 0; sl < Staging::kSlots; ++sl) {
        S.in0[sl].ensure(chunk * 8);
        S.out[sl].ensure(chunk * nd);
    }
    S.run(
        n, chunk,
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(S.in0[sl].ptr, h_words + off, cnt * 8, cudaMemcpyHostToDevice, s), "H2D");
        },
        [&](int sl, u64, u64 cnt, cudaStream_t s) {
            redq_device_u64(dp, S.in0[sl].as<uint64_t>(), cnt, S.out[sl].as<uint8_t>(), s);
        },
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(h_out + off * nd, S.out[sl].ptr, cnt * nd, cudaMemcpyDeviceToHost, s), "D2H");
        });
    raise_status(take_status(dp, S.sk));
}

// Host buffers in, host buffers out: H2D / kernel / D2H of consecutive
// chunks on three streams so the copies of one chunk overlap the others.
void redq_host(DevicePlanCache& dp, const double* h_words, u64 n, uint8_t* h_out) {
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.staging) dp.staging = std::make_unique<Staging>();
    Staging& S = *dp.staging;
    const u64 nd = dp.prm.d + 1;
    // 16 MB of words per chunk: short pipeline fill/drain against PCIe
    // (measured Gen5 x16: 55.6 GB/s H2D, 57.2 D2H, 100 GB/s both ways)
    static const u64 chunk = [] {
        const char* e = std::getenv("QPK_HOST_CHUNK_LOG2");  // dev knob (scripts/pcie_probe.py)
        return u64(1) << (e ? std::clamp(std::atoi(e), 16, 26) : 21);
    }();
    for (int sl = 0; sl < Staging::kSlots; ++sl) {
        S.in0[sl].ensure(chunk * 8);
        S.out[sl].ensure(chunk * nd);
    }
    S.run(
        n, chunk,
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(S.in0[sl].ptr, h_words + off, cnt * 8, cudaMemcpyHostToDevice, s), "H2D");
        },
        [&](int sl, u64, u64 cnt, cudaStream_t s) {
            redq_device(dp, S.in0[sl].as<double>(), cnt, S.out[sl].as<uint8_t>(), s);
        },
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(h_out + off * nd, S.out[sl].ptr, cnt * nd, cudaMemcpyDeviceToHost, s), "D2H");
        });
    raise_status(take_status(dp, S.sk));
}

void redq_residues_batch(std::span<const double> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost) {
    if (out.size() < words.size() * (plan.d + 1))
        throw std::invalid_argument("redq_residues_batch: output span holds fewer than n*(d+1) residues");
    DevicePlanCache& dp = detail::device_plan(plan);
    redq_host(dp, words.data(), words.size(), out.data());
    if (cost) *cost += detail::redq_batch_cost(plan, words.size());
}

void redq_residues_batch(std::span<const std::uint64_t> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost) {
    if (out.size() < words.size() * (plan.d + 1))
        throw std::invalid_argument("redq_residues_batch: output span holds fewer than n*(d+1) residues");
    DevicePlanCache& dp = detail::device_plan(plan);
    redq_host_u64(dp, words.data(), words.size(), out.data());
    if (cost) *cost += detail::redq_batch_cost(plan, words.size());
}

void redq_residues_batch(std::span<const u128> words, const RedqPlan& plan, std::span<std::uint8_t> out,
                         CostReport* cost) {
    if (out.size() < words.size() * (plan.d + 1))
        throw std::invalid_argument("redq_residues_batch: output span holds fewer than n*(d+1) residues");
    if (plan.p > 256) throw std::invalid_argument("qpack-b200 redq: residues are uint8, p must be <= 256");
    std::vector<uint64_t> halves(2 * words.size());
    for (std::size_t i = 0; i < words.size(); ++i) {
        halves[2 * i] = static_cast<uint64_t>(words[i]);
        halves[2 * i + 1] = static_cast<uint64_t>(words[i] >> 64);
    }
    DevicePlanCache& dp = detail::device_plan(plan);
    redq_host_u128(dp, halves.data(), words.size(), out.data());
    if (cost) *cost += detail::redq_batch_cost(plan, words.size());
}

// ------------------------------------------------------------ polymul plans
PolymulPlan::PolymulPlan(const QadicParams& pr) : params(pr) {
    const ValidationResult vr = validate(pr);
    if (!vr.ok()) throw std::invalid_argument("dqt_mul_poly: " + vr.detail);
    if (pr.k > 8) throw std::invalid_argument("qpack-b200 polymul: device path packs at most k = 8 coefficients");
    redq = fqt_reduction_plan(pr, pr.k - 1);
    P.k = pr.k;
    // p > 256: only the u64-coefficient FQT entry points (no uint8 residues,
    // no device REDQ mirror)
    if (pr.p > 256) return;
    DevicePlanCache& dp = detail::device_plan(redq);
    P.rq = dp.prm;
}

void polymul_device(PolymulPlan& pl, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, cudaStream_t s) {
    if (pl.params.p > 256) throw std::invalid_argument("qpack-b200 polymul: residues are uint8, p must be <= 256");
    if (pl.params.k > static_cast<u32>(qpk::kMaxGfqK))
        throw std::invalid_argument("qpack-b200 polymul: the batched path packs at most k = 4 coefficients");
    // the batched kernel multiplies packed words in fp64: exact while the
    // product word q^(2k-1) fits 53 bits (m <= 53 guarantees it)
    if (pl.params.m > 53 && (!pow_fits_u128(pl.params.q, 2 * pl.params.k - 1) ||
                             checked_pow_u128(pl.params.q, 2 * pl.params.k - 1) > (u128(1) << 53)))
        throw std::invalid_argument("qpack-b200 polymul: the batched path computes in fp64 words (q^(2k-1) <= 2^53)");
    DevicePlanCache& dp = detail::device_plan(pl.redq);
    check(qpk::launch_polymul(pl.P, a, b, n, out, dp.status.as<uint32_t>(), s), "polymul launch");
}

void polymul_host(PolymulPlan& pl, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out) {
    if (pl.params.p > 256) throw std::invalid_argument("qpack-b200 polymul: residues are uint8, p must be <= 256");
    DevicePlanCache& dp = detail::device_plan(pl.redq);
    std::lock_guard<std::mutex> lock(dp.mu);
    if (!dp.staging) dp.staging = std::make_unique<Staging>();
    Staging& S = *dp.staging;
    // up to 2^22 pairs per chunk; a batch smaller than four such chunks is cut
    // in four (64 Ki granules) so the D2H of one quarter still overlaps the
    // H2D of the next (C1's 2^20 pairs: one serial H2D + kernel + D2H before)
    const u64 k = pl.params.k, ko = 2 * k - 1;
    u64 chunk = std::clamp<u64>((n / 4 + 0xffff) & ~u64(0xffff), u64(1) << 16, u64(1) << 22);
    if (const char* e = std::getenv("QPK_PM_CHUNK_LOG2")) chunk = u64(1) << std::clamp(std::atoi(e), 12, 22);  // dev knob
    for (int sl = 0; sl < Staging::kSlots; ++sl) {
        S.in0[sl].ensure(chunk * k);
        S.in1[sl].ensure(chunk * k);
        S.out[sl].ensure(chunk * ko);
    }
    S.run(
        n, chunk,
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(S.in0[sl].ptr, a + off * k, cnt * k, cudaMemcpyHostToDevice, s), "H2D");
            check(cudaMemcpyAsync(S.in1[sl].ptr, b + off * k, cnt * k, cudaMemcpyHostToDevice, s), "H2D");
        },
        [&](int sl, u64, u64 cnt, cudaStream_t s) {
            polymul_device(pl, S.in0[sl].as<uint8_t>(), S.in1[sl].as<uint8_t>(), cnt, S.out[sl].as<uint8_t>(), s);
        },
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(out + off * ko, S.out[sl].ptr, cnt * ko, cudaMemcpyDeviceToHost, s), "D2H");
        });
    raise_status(take_status(dp, S.sk));
}

// ---- chunked FQT product (K6) ----
void fqt_check(const RedqPlan& plan, const QadicParams& params, bool wide_p = false) {
    if (!wide_p && params.p > 256)
        throw std::invalid_argument("qpack-b200 fqt_mul: uint8 coefficients need p <= 256 (u64 entry points: any p)");
    if (params.k < 1 || params.k > 8)
        throw std::invalid_argument("qpack-b200 fqt_mul: the device path packs 1..8 coefficients per chunk");
    if (plan.p != params.p || plan.q != params.q || plan.d != 2 * (params.k - 1))
        throw std::invalid_argument("fqt_mul: reduction plan does not match the params");
}

void fqt_mul_device(const RedqPlan& plan, const QadicParams& params, const uint8_t* a, u64 na, const uint8_t* b,
                    u64 nb, uint8_t* out, cudaStream_t s) {
    fqt_check(plan, params);
    if (na == 0 || nb == 0) return;
    if (params.m > 53) {
        // integer words beyond fp64 (the reference's u128 mode): u128 kernel
        StreamBuf ws(qpk::fqt_wide_workspace_bytes(params.k, na, nb), s);
        check(qpk::launch_fqt_mul_wide(static_cast<uint32_t>(params.p), params.q, params.k,
                                       static_cast<uint32_t>(std::max<u64>(params.n_q, 1)), a, na, b, nb, out, ws.ptr, s),
              "fqt_mul (u128 words) launch");
        return;
    }
    DevicePlanCache& dp = detail::device_plan(plan);
    qpk::FqtParams F{};
    F.rq = dp.prm;
    F.k = params.k;
    F.nq = static_cast<uint32_t>(std::max<u64>(params.n_q, 1));
    // integer group REDQ in the DMMA kernel: q = 2^b and every group word
    // below 2^52 (biased accumulators), p <= 256 (mulhi floor exact)
    const u64 nd = 2 * u64(params.k) - 1;
    F.mma_int = (dp.prm.qbits != 0 && dp.prm.qbits * nd <= 52) ? 1u : 0u;
    F.p_magic = ~u64(0) / params.p + 1;  // ceil(2^64 / p) for p not a power of two; 2^64/p exactly otherwise
    StreamBuf ws(qpk::fqt_workspace_bytes(params.k, F.nq, na, nb), s);
    check(qpk::launch_fqt_mul(F, a, na, b, nb, out, ws.ptr, s), "fqt_mul launch");
}

void fqt_mul_host(const RedqPlan& plan, const QadicParams& params, const uint8_t* a, u64 na, const uint8_t* b, u64 nb,
                  uint8_t* out) {
    fqt_check(plan, params);
    if (na == 0 || nb == 0) return;
    DevicePlanCache& dp = detail::device_plan(plan);
    std::lock_guard<std::mutex> lock(dp.mu);
    auto* da = static_cast<uint8_t*>(dp.io_a.ensure(na));
    auto* db = static_cast<uint8_t*>(dp.io_b.ensure(nb));
    auto* dc = static_cast<uint8_t*>(dp.io_c.ensure(na + nb - 1));
    check(cudaMemcpy(da, a, na, cudaMemcpyHostToDevice), "H2D");
    check(cudaMemcpy(db, b, nb, cudaMemcpyHostToDevice), "H2D");
    fqt_mul_device(plan, params, da, na, db, nb, dc, 0);
    check(cudaMemcpy(out, dc, na + nb - 1, cudaMemcpyDeviceToHost), "D2H");
}

// p > 256 (or any p): u64 coefficients, u128 words (launch_fqt_mul_widep)
void fqt_mul_device_u64(const RedqPlan& plan, const QadicParams& params, const uint64_t* a, u64 na, const uint64_t* b,
                        u64 nb, uint64_t* out, cudaStream_t s) {
    fqt_check(plan, params, true);
    if (na == 0 || nb == 0) return;
    gpu::require_device();
    StreamBuf ws(qpk::fqt_widep_workspace_bytes(params.k, na, nb), s);
    check(qpk::launch_fqt_mul_widep(params.p, params.q, params.k, static_cast<uint32_t>(std::max<u64>(params.n_q, 1)),
                                    a, na, b, nb, out, ws.ptr, s),
          "fqt_mul (u64 coefficients) launch");
}

void fqt_mul_host_u64(const RedqPlan& plan, const QadicParams& params, const uint64_t* a, u64 na, const uint64_t* b,
                      u64 nb, uint64_t* out) {
    fqt_check(plan, params, true);
    if (na == 0 || nb == 0) return;
    gpu::require_device();
    DevBuf da, db, dc;  // per call: no device plan mirror for p > 256
    da.ensure(na * 8);
    db.ensure(nb * 8);
    dc.ensure((na + nb - 1) * 8);
    check(cudaMemcpy(da.ptr, a, na * 8, cudaMemcpyHostToDevice), "H2D");
    check(cudaMemcpy(db.ptr, b, nb * 8, cudaMemcpyHostToDevice), "H2D");
    fqt_mul_device_u64(plan, params, da.as<uint64_t>(), na, db.as<uint64_t>(), nb, dc.as<uint64_t>(), 0);
    check(cudaMemcpy(out, dc.ptr, (na + nb - 1) * 8, cudaMemcpyDeviceToHost), "D2H");
}

CostReport fqt_cost(const RedqPlan& plan, const QadicParams& params, u64 na, u64 nb) {
    // the reference loop (polymul.cpp:106-146) runs every (t, i) of the
    // zero-padded span and one REDQ per (t, group)
    if (na == 0 || nb == 0) return {};
    const u64 d = params.k - 1;
    const u64 dq = packed_degree(std::max(na, nb) - 1, static_cast<u32>(d));
    const u64 span = 2 * dq + 1;
    const u64 groups = (span + params.n_q - 1) / params.n_q;
    CostReport c = detail::redq_batch_cost(plan, span * groups);
    c.mul_add = span * span;
    return c;
}

CostReport polymul_cost(const PolymulPlan& pl, u64 n) {
    // fqt_mul with one chunk per operand: one product, one REDQ per pair
    CostReport c = detail::redq_batch_cost(pl.redq, n);
    c.mul_add = n;
    return c;
}

void polymul_batch(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b, const QadicParams& params,
                   std::span<std::uint8_t> out, CostReport* cost) {
    static std::mutex mu;
    static std::map<std::tuple<u64, u64, u32, u32, u32>, std::unique_ptr<PolymulPlan>> cache;
    PolymulPlan* pl;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto& slot = cache[{params.p, params.q, params.k, params.n_q, params.m}];
        if (!slot) slot = std::make_unique<PolymulPlan>(params);
        pl = slot.get();
    }
    const u64 n = a.size() / params.k;
    if (a.size() != b.size() || a.size() % params.k || out.size() < n * (2 * params.k - 1))
        throw std::invalid_argument("polymul_batch: spans do not hold n records of k coefficients / 2k-1 residues");
    polymul_host(*pl, a.data(), b.data(), n, out.data());
    if (cost) *cost += polymul_cost(*pl, n);
}

// ------------------------------------------------------------------ GF(p^k)
// coefficient records hold one byte per coefficient
void require_byte_coeffs(const DeviceFieldCache& F) {
    if (F.elem.p > 255)
        throw std::invalid_argument("qpack-b200 GF(p^k): coefficient records are bytes (p < 256); p = " +
                                    std::to_string(F.elem.p) + " takes the rep entry points");
}

void gfq_mul_device(DeviceFieldCache& F, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, int path,
                    cudaStream_t s) {
    if (path < qpk::kGfqPacked || path > qpk::kGfqLinear)
        throw std::invalid_argument("gfq_mul: path must be 0 (packed), 1 (dlog) or 2 (linear)");
    require_byte_coeffs(F);
    if (F.wide) {
        check(qpk::launch_gfq_wide_mul(F.wp, a, b, n, out, path, s), "gfq_mul (rep domain) launch");
        return;
    }
    qpk::GfqElemParams E = F.elem;
    E.mode = path;
    check(qpk::launch_gfq_elem(E, a, b, n, out, s), "gfq_mul launch");
}

void gfq_mul_host(DeviceFieldCache& F, const uint8_t* a, const uint8_t* b, u64 n, uint8_t* out, int path) {
    std::lock_guard<std::mutex> lock(F.mu);
    if (!F.staging) F.staging = std::make_unique<Staging>();
    Staging& S = *F.staging;
    const u64 k = F.elem.k, chunk = u64(1) << 22;
    for (int sl = 0; sl < Staging::kSlots; ++sl) {
        S.in0[sl].ensure(chunk * k);
        S.in1[sl].ensure(chunk * k);
        S.out[sl].ensure(chunk * k);
    }
    S.run(
        n, chunk,
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(S.in0[sl].ptr, a + off * k, cnt * k, cudaMemcpyHostToDevice, s), "H2D");
            check(cudaMemcpyAsync(S.in1[sl].ptr, b + off * k, cnt * k, cudaMemcpyHostToDevice, s), "H2D");
        },
        [&](int sl, u64, u64 cnt, cudaStream_t s) {
            gfq_mul_device(F, S.in0[sl].as<uint8_t>(), S.in1[sl].as<uint8_t>(), cnt, S.out[sl].as<uint8_t>(), path, s);
        },
        [&](int sl, u64 off, u64 cnt, cudaStream_t s) {
            check(cudaMemcpyAsync(out + off * k, S.out[sl].ptr, cnt * k, cudaMemcpyDeviceToHost, s), "D2H");
        });
}

void gfq_mul_batch(std::span<const std::uint8_t> a, std::span<const std::uint8_t> b, const GfqField& field,
                   std::span<std::uint8_t> out, GfqPath path) {
    const u64 k = field.k();
    if (a.size() != b.size() || a.size() % k || out.size() < a.size())
        throw std::invalid_argument("gfq_mul_batch: spans do not hold n records of k coefficients");
    gfq_mul_host(detail::device_field(field), a.data(), b.data(), a.size() / k, out.data(), static_cast<int>(path));
}

void gfq_mul_rep_host(DeviceFieldCache& F, const uint32_t* a, const uint32_t* b, u64 n, uint32_t* out) {
    std::lock_guard<std::mutex> lock(F.mu);
    DevBuf& da = F.io_a;
    DevBuf& db = F.io_b;
    DevBuf& dc = F.io_c;
    da.ensure(n * 4);
    db.ensure(n * 4);
    dc.ensure(n * 4);
    check(cudaMemcpy(da.ptr, a, n * 4, cudaMemcpyHostToDevice), "H2D");
    check(cudaMemcpy(db.ptr, b, n * 4, cudaMemcpyHostToDevice), "H2D");
    check(qpk::launch_gfq_mul_rep(F.elem.group, da.as<uint32_t>(), db.as<uint32_t>(), n, dc.as<uint32_t>(),
                                  F.status.as<uint32_t>(), 0),
          "gfq_mul_rep launch");
    check(cudaMemcpy(out, dc.ptr, n * 4, cudaMemcpyDeviceToHost), "D2H");
    raise_field_status(take_field_status(F, 0));
}

// GfqField::mul / add / neg / inverse over host rep arrays, on the device
void gfq_rep_op_host(DeviceFieldCache& F, const GfqField& field, int op, const uint32_t* a, const uint32_t* b, u64 n,
                     uint32_t* out) {
    if (n == 0) return;
    std::lock_guard<std::mutex> lock(F.mu);
    const u64 group = field.order() - 1;
    if (op == 1 && !F.zech.ptr) {
        const std::vector<u32>& z = detail::FieldAccess::zech(field);
        F.zech.ensure(z.size() * 4);
        check(cudaMemcpy(F.zech.ptr, z.data(), z.size() * 4, cudaMemcpyHostToDevice), "zech upload");
        detail::settle_uploads();
    }
    F.io_a.ensure(n * 4);
    F.io_b.ensure(n * 4);
    F.io_c.ensure(n * 4);
    check(cudaMemcpy(F.io_a.ptr, a, n * 4, cudaMemcpyHostToDevice), "H2D");
    if (op < 2) check(cudaMemcpy(F.io_b.ptr, b, n * 4, cudaMemcpyHostToDevice), "H2D");
    check(qpk::launch_gfq_rep_op(op, static_cast<uint32_t>(field.p()), static_cast<uint32_t>(group),
                                 F.zech.as<uint32_t>(), F.io_a.as<uint32_t>(), F.io_b.as<uint32_t>(), n,
                                 F.io_c.as<uint32_t>(), F.status.as<uint32_t>(), 0),
          "gfq rep op launch");
    check(cudaMemcpy(out, F.io_c.ptr, n * 4, cudaMemcpyDeviceToHost), "D2H");
    raise_field_status(take_field_status(F, 0));
}

void gfq_mul_batch(std::span<const GfqElt> a, std::span<const GfqElt> b, const GfqField& field,
                   std::span<GfqElt> out) {
    if (a.size() != b.size() || out.size() < a.size()) throw std::invalid_argument("gfq_mul_batch: length mismatch");
    if (a.empty()) return;
    for (const auto* v : {&a, &b})
        for (const GfqElt& e : *v)
            if (e.rep >= field.order()) throw std::out_of_range("gfq_mul_batch: rep outside the field");
    gfq_mul_rep_host(detail::device_field(field), reinterpret_cast<const uint32_t*>(a.data()),
                     reinterpret_cast<const uint32_t*>(b.data()), a.size(), reinterpret_cast<uint32_t*>(out.data()));
}

// ---- matmul ----
namespace {
u64 round_up(u64 v, u64 m) { return (v + m - 1) / m * m; }
}  // namespace

uint32_t resolve_chunk(const DeviceFieldCache& F, const GfqField& field, u64 K, uint32_t chunk, uint32_t repack) {
    const u64 p = field.p(), k = field.k(), q = field.params().q;
    const u64 unit = k * (p - 1) * (p - 1);
    if (repack > qpk::kRepackFold) throw std::invalid_argument("gfq_matmul: unknown re-pack mode");
    // the lane fold is compiled for the GF(3^3), q = 2^10 fast path (p = 3:
    // 2^S == 1 mod 3 for even S)
    if (repack == qpk::kRepackFold && !(p == 3 && k == 3 && q == 1024))
        throw std::invalid_argument("gfq_matmul: the fold re-pack is provided for GF(3^3) at q = 2^10 only");
    // after a re-pack every digit is <= p-1 (REDQ) or <= the fold bound;
    // `safe` more products keep it < q
    const u64 post = repack == qpk::kRepackFold ? qpk::fold_digit_bound(10) : p - 1;
    const u64 safe = unit ? (q - 1 - post) / unit : K;
    (void)F;
    if (chunk == 0) {
        if (K <= field.params().n_q) return 0;  // one accumulation group: never reduce
        chunk = static_cast<uint32_t>(std::min<u64>(safe, 1u << 30));
        // a whole number of K-stages re-packs between stages (the fast
        // kernels; C5's field: 85 -> 80, measured 90 -> ~40 ms at 8192^3)
        if (chunk >= qpk::kMatmulBK) chunk -= chunk % qpk::kMatmulBK;
    }
    if (chunk > safe)
        throw std::invalid_argument("gfq_matmul: chunk " + std::to_string(chunk) + " lets digit sums reach q (max " +
                                    std::to_string(safe) + ")");
    chunk -= chunk % 4;  // the kernel re-packs at 4-step granularity
    if (chunk == 0) throw std::invalid_argument("gfq_matmul: field admits fewer than 4 products between reductions");
    return chunk;
}

// A, B, C device pointers: coefficient records (reps when `reps`)
// Fields whose safe group is below one fp64 MMA step (4 products, e.g.
// GF(7^3) at q = 2^8, n_q = 2): C = A B as n GEMVs (K5, groups of n_q
// products per lane like the reference's fgdp_dot) over B's columns,
// through rep layouts: A as reps, B^T as reps, C^T rows, transposed back.
void gfq_matmul_by_columns(DeviceFieldCache& F, const GfqField& field, const void* A, const void* B, u64 m, u64 K,
                           u64 n, void* C, bool reps, cudaStream_t s) {
    const qpk::GfqElemParams& E = F.elem;
    StreamBuf wa(reps ? 0 : m * K * 4, s), wb(reps ? 0 : K * n * 4, s), wbt(n * K * 4, s), wct(n * m * 4, s),
        wc(reps ? 0 : m * n * 4, s);
    const uint32_t* ar = static_cast<const uint32_t*>(A);
    const uint32_t* br = static_cast<const uint32_t*>(B);
    if (!reps) {
        check(qpk::launch_coeffs_to_reps(E.p, E.k, E.log, static_cast<const uint8_t*>(A), m * K, wa.as<uint32_t>(), s),
              "coeffs -> reps");
        check(qpk::launch_coeffs_to_reps(E.p, E.k, E.log, static_cast<const uint8_t*>(B), K * n, wb.as<uint32_t>(), s),
              "coeffs -> reps");
        ar = wa.as<uint32_t>();
        br = wb.as<uint32_t>();
    }
    check(qpk::launch_transpose_u32(br, K, n, wbt.as<uint32_t>(), s), "transpose B");
    for (u64 j = 0; j < n; ++j)
        gfq_gemv_device(F, field, ar, wbt.as<uint32_t>() + j * K, m, K, wct.as<uint32_t>() + j * m, nullptr, s);
    uint32_t* cr = reps ? static_cast<uint32_t*>(C) : wc.as<uint32_t>();
    check(qpk::launch_transpose_u32(wct.as<uint32_t>(), n, m, cr, s), "transpose C");
    if (!reps) {
        if (F.wide)
            check(qpk::launch_gfq_wide_reps_to_coeffs(F.wp, cr, m * n, static_cast<uint8_t*>(C), s), "reps -> coeffs");
        else
            check(qpk::launch_reps_to_coeffs(E.k, E.alog, cr, m * n, static_cast<uint8_t*>(C), s), "reps -> coeffs");
    }
}

namespace {

// the fp64 MMA route of gfq_matmul (else: rep-domain or per-column GEMVs)
bool matmul_mma_route(const DeviceFieldCache& F, const GfqField& field, u64 K) {
    if (F.wide) return false;
    const u64 p = field.p(), unit = field.k() * (p - 1) * (p - 1), q = field.params().q;
    const u64 safe = unit ? (q - 1 - (p - 1)) / unit : K;
    return !(K > field.params().n_q && safe < 4);
}

// kernel parameters of one launch (chunk and re-pack resolved)
qpk::GfqMatmulParams matmul_params(const DeviceFieldCache& F, const GfqField& field, u64 K, uint32_t chunk,
                                   uint32_t repack) {
    qpk::GfqMatmulParams M = F.mm;
    M.chunk = resolve_chunk(F, field, K, chunk, repack);
    M.repack = M.chunk ? repack : qpk::kRepackRedq;
    return M;
}

// operand B (K x n records or reps) -> the K4 workspace bt (kp x np doubles)
void matmul_pack_b(DeviceFieldCache& F, const qpk::GfqMatmulParams& M, const void* B, u64 K, u64 n, bool reps,
                   double* bt, cudaStream_t s) {
    const u64 np = round_up(n, 128), kp = round_up(std::max<u64>(K, 1), 16);
    const bool pair = qpk::mm_pair_layout(M);
    if (np != n || kp != K) check(cudaMemsetAsync(bt, 0, kp * np * 8, s), "memset");
    if (reps)
        check(qpk::launch_pack_reps(F.mm.fval, F.mm.order, static_cast<const uint32_t*>(B), K, n, bt, np, false, pair,
                                    F.status.as<uint32_t>(), s),
              "pack B");
    else
        check(qpk::launch_pack_coeffs(F.mm.p, F.mm.k, F.mm.qd, static_cast<const uint8_t*>(B), K, n, bt, np, false,
                                      pair, s),
              "pack B");
}

}  // namespace

// packed_b: operand B already in the K4 workspace form (matmul_pack_b with
// the same field, K, chunk and repack), shared by the row bands of one product
void gfq_matmul_device(DeviceFieldCache& F, const GfqField& field, const void* A, const void* B, u64 m, u64 K, u64 n,
                       uint32_t chunk, void* C, bool reps, cudaStream_t s, uint32_t repack, const double* packed_b) {
    if (m == 0 || n == 0) return;
    if (!reps) require_byte_coeffs(F);
    if (F.wide) {
        // rep-domain GEMVs over B's columns (the fp64 MMA kernels pack at most
        // four byte coefficients per word)
        if (repack != qpk::kRepackRedq)
            throw std::invalid_argument("gfq_matmul: the fold re-pack is provided for GF(3^3) at q = 2^10 only");
        gfq_matmul_by_columns(F, field, A, B, m, K, n, C, reps, s);
        return;
    }
    {
        const u64 p = field.p(), unit = field.k() * (p - 1) * (p - 1), q = field.params().q;
        const u64 safe = unit ? (q - 1 - (p - 1)) / unit : K;
        if (K > field.params().n_q && safe < 4) {
            if (chunk > safe)
                throw std::invalid_argument("gfq_matmul: chunk " + std::to_string(chunk) +
                                            " lets digit sums reach q (max " + std::to_string(safe) + ")");
            if (repack != qpk::kRepackRedq)
                throw std::invalid_argument("gfq_matmul: the fold re-pack is provided for GF(3^3) at q = 2^10 only");
            gfq_matmul_by_columns(F, field, A, B, m, K, n, C, reps, s);
            return;
        }
    }
    const u64 mp = round_up(m, 128), np = round_up(n, 128), kp = round_up(std::max<u64>(K, 1), 16);
    StreamBuf wa(kp * mp * 8, s), wb(packed_b ? 0 : kp * np * 8, s);
    auto* at = wa.as<double>();
    const qpk::GfqMatmulParams M = matmul_params(F, field, K, chunk, repack);
    const bool pair = qpk::mm_pair_layout(M);  // the column order the kernel this launch selects reads
    if (mp != m || kp != K) check(cudaMemsetAsync(at, 0, kp * mp * 8, s), "memset");
    if (reps)
        check(qpk::launch_pack_reps(F.mm.fval, F.mm.order, static_cast<const uint32_t*>(A), m, K, at, mp, true, pair,
                                    F.status.as<uint32_t>(), s),
              "pack A");
    else
        check(qpk::launch_pack_coeffs(F.mm.p, F.mm.k, F.mm.qd, static_cast<const uint8_t*>(A), m, K, at, mp, true, pair,
                                      s),
              "pack A");
    const double* bt = packed_b;
    if (!bt) {
        matmul_pack_b(F, M, B, K, n, reps, wb.as<double>(), s);
        bt = wb.as<double>();
    }
    check(qpk::launch_gfq_matmul(M, at, bt, m, n, kp, mp, np, reps ? nullptr : static_cast<uint8_t*>(C),
                                 reps ? static_cast<uint32_t*>(C) : nullptr, s),
          "gfq_matmul launch");
}

void gfq_matmul_host(DeviceFieldCache& F, const GfqField& field, const void* A, const void* B, u64 m, u64 K, u64 n,
                     uint32_t chunk, void* C, bool reps, uint32_t repack, u64* zech_reads) {
    std::lock_guard<std::mutex> lock(F.mu);
    const u64 es = reps ? 4 : field.k();
    auto* da = F.io_a.ensure(m * K * es);
    auto* db = F.io_b.ensure(K * n * es);
    auto* dc = F.io_c.ensure(m * n * es);
    // Large products on the MMA route run as row bands of A and C: B goes up
    // and is packed once, then band i's rows of A go up while band i-1
    // multiplies and band i-2's rows of C come back (streams chained by
    // events) -- the copies of all but the first and last band hide behind
    // the contraction.  Consecutive bands run on two alternating compute
    // streams so a band's last, partly filled wave of tiles overlaps the next
    // band's first.  Small or other-route products: copy, multiply, copy.
    const u64 bands = (matmul_mma_route(F, field, K) && K && m >= 1024 && m * K * es >= (u64(16) << 20))
                          ? std::min<u64>(8, m / 512)
                          : 1;
    if (bands > 1) {
        if (!F.staging) F.staging = std::make_unique<Staging>();
        Staging& S = *F.staging;
        const u64 np = round_up(n, 128), kp = round_up(K, 16);
        const qpk::GfqMatmulParams M = matmul_params(F, field, K, chunk, repack);
        StreamBuf bt(kp * np * 8, S.sk);
        // every stream drains before bt is released, also when a launch below throws
        struct Drain {
            Staging& st;
            ~Drain() {
                for (cudaStream_t q : {st.sh, st.sk, st.sk2, st.sd}) cudaStreamSynchronize(q);
            }
        } drain{S};
        check(cudaMemcpyAsync(db, B, K * n * es, cudaMemcpyHostToDevice, S.sh), "H2D");
        check(cudaEventRecord(S.ev_in[0], S.sh), "event");
        check(cudaStreamWaitEvent(S.sk, S.ev_in[0], 0), "wait B");
        matmul_pack_b(F, M, db, K, n, reps, bt.as<double>(), S.sk);
        check(cudaEventRecord(S.ev_aux, S.sk), "event");
        check(cudaStreamWaitEvent(S.sk2, S.ev_aux, 0), "wait packed B");
        const u64 rows_per = round_up((m + bands - 1) / bands, 128);
        auto* a8 = static_cast<uint8_t*>(da);
        auto* c8 = static_cast<uint8_t*>(dc);
        for (u64 r0 = 0, i = 0; r0 < m; r0 += rows_per, ++i) {
            const u64 rows = std::min(rows_per, m - r0);
            const int sl = static_cast<int>(i % Staging::kSlots);
            check(cudaMemcpyAsync(a8 + r0 * K * es, static_cast<const uint8_t*>(A) + r0 * K * es, rows * K * es,
                                  cudaMemcpyHostToDevice, S.sh),
                  "H2D");
            check(cudaEventRecord(S.ev_in[sl], S.sh), "event");
            const cudaStream_t ks = (i & 1) ? S.sk2 : S.sk;
            check(cudaStreamWaitEvent(ks, S.ev_in[sl], 0), "wait A band");
            gfq_matmul_device(F, field, a8 + r0 * K * es, db, rows, K, n, chunk, c8 + r0 * n * es, reps, ks, repack,
                              bt.as<double>());
            check(cudaEventRecord(S.ev_k[sl], ks), "event");
            check(cudaStreamWaitEvent(S.sd, S.ev_k[sl], 0), "wait band");
            check(cudaMemcpyAsync(static_cast<uint8_t*>(C) + r0 * n * es, c8 + r0 * n * es, rows * n * es,
                                  cudaMemcpyDeviceToHost, S.sd),
                  "D2H");
        }
        check(cudaStreamSynchronize(S.sd), "sync");
        check(cudaStreamSynchronize(S.sk), "sync");
        check(cudaStreamSynchronize(S.sk2), "sync");
    } else {
        check(cudaMemcpy(da, A, m * K * es, cudaMemcpyHostToDevice), "H2D");
        check(cudaMemcpy(db, B, K * n * es, cudaMemcpyHostToDevice), "H2D");
        gfq_matmul_device(F, field, da, db, m, K, n, chunk, dc, reps, 0, repack);
        check(cudaMemcpy(C, dc, m * n * es, cudaMemcpyDeviceToHost), "D2H");
    }
    if (reps) raise_field_status(take_field_status(F, 0));
    if (zech_reads && m && n && K) {
        // the reference's data-dependent counter part (K7), on rep operands
        const uint32_t* ra = static_cast<const uint32_t*>(da);
        const uint32_t* rb = static_cast<const uint32_t*>(db);
        StreamBuf wa(reps ? 0 : m * K * 4, 0), wb(reps ? 0 : K * n * 4, 0);
        if (!reps) {
            const qpk::GfqElemParams& E = F.elem;
            check(qpk::launch_coeffs_to_reps(E.p, E.k, E.log, static_cast<const uint8_t*>(da), m * K, wa.as<uint32_t>(), 0),
                  "coeffs -> reps");
            check(qpk::launch_coeffs_to_reps(E.p, E.k, E.log, static_cast<const uint8_t*>(db), K * n, wb.as<uint32_t>(), 0),
                  "coeffs -> reps");
            ra = wa.as<uint32_t>();
            rb = wb.as<uint32_t>();
        }
        *zech_reads = zech_reads_device(F, field, ra, rb, m, K, n, 0);
    }
}

u64 zech_reads_device(DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* B, u64 m, u64 K,
                      u64 n, cudaStream_t s) {
    if (m == 0 || n == 0 || K == 0) return 0;
    if (field.k() > qpk::kMaxCountK) throw std::invalid_argument("qpack-b200 counters: k <= 8");
    const std::vector<u32>& lo = detail::FieldAccess::low(field);
    const std::vector<u32>& hi = detail::FieldAccess::high(field);
    const std::vector<u32>& z = detail::FieldAccess::zech(field);
    if (!F.lh_reps.ptr) {
        std::vector<uint32_t> host(lo.begin(), lo.end());
        host.insert(host.end(), hi.begin(), hi.end());
        host.insert(host.end(), z.begin(), z.end());
        F.lh_reps.ensure(host.size() * 4);
        check(cudaMemcpy(F.lh_reps.ptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice), "counter tables upload");
        F.counter.ensure(8);
        detail::settle_uploads();
    }
    qpk::GfqCountParams P{};
    P.p = static_cast<uint32_t>(field.p());
    P.k = field.k();
    P.group = static_cast<uint32_t>(field.order() - 1);
    P.lh_radix = static_cast<uint32_t>(detail::FieldAccess::lh_radix(field));
    const u64 q = detail::FieldAccess::q(field);
    P.qbits = is_pow2(q) ? bit_width_u128(q) - 1 : 0;
    P.n_q = field.params().n_q;
    u64 qi = 1;
    for (u32 i = 0; i < 2 * field.k() - 1; ++i, qi *= q) P.qpow[i] = qi;
    P.fval = F.fval.as<double>();
    P.low = F.lh_reps.as<uint32_t>();
    P.high = P.low + lo.size();
    P.zech = P.high + hi.size();
    auto* total = F.counter.as<unsigned long long>();
    check(cudaMemsetAsync(total, 0, 8, s), "counter clear");
    check(qpk::launch_gfq_count(P, A, B, m, K, n, total, s), "gfq counter launch");
    unsigned long long v = 0;
    check(cudaMemcpyAsync(&v, total, 8, cudaMemcpyDeviceToHost, s), "counter read");
    check(cudaStreamSynchronize(s), "counter sync");
    return v;
}

CostReport matmul_cost(const GfqField& field, u64 m, u64 K, u64 n) {
    // reference grouping (gfq.cpp:346-385): ceil(K/n_q) groups per entry;
    // table_accesses here counts the operand and L/H lookups; the Zech reads
    // of the two additions per group depend on the data: callers that report
    // counters add zech_reads_device (K7)
    const u64 groups = K ? (K + field.params().n_q - 1) / field.params().n_q : 0;
    CostReport c;
    c.mul_add = m * n * K;
    c.divisions = c.reduction_calls = m * n * groups;
    c.table_accesses = 2 * m * n * K + 2 * m * n * groups;
    return c;
}

// ---- GEMV / long dot (K5) ----
void gfq_gemv_device(DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* x, u64 m, u64 K,
                     uint32_t* y_rep, uint8_t* y_coeff, cudaStream_t s) {
    if (m == 0) return;
    if (y_coeff) require_byte_coeffs(F);
    if (F.wide) {
        StreamBuf ws(qpk::gfq_wide_workspace_bytes(m, K), s);
        check(qpk::launch_gfq_wide_gemv(F.wp, A, x, m, K, ws.ptr, y_rep, y_coeff, s), "gfq_gemv (rep domain) launch");
        return;
    }
    uint32_t splits = qpk::gemv_splits(m, K);
    if (const char* e = std::getenv("QPK_GEMV_SPLITS")) splits = static_cast<uint32_t>(std::max(1, std::atoi(e)));  // dev knob
    // products one lane accumulates: a split is rounded up to 128 elements,
    // 4 per lane per 128
    const u64 ksplit = (K + splits - 1) / splits;
    const u64 lane_terms = (ksplit + 127) / 128 * 4;
    // groups of at most n_q products per lane, as the reference's grouping
    // (gfq.cpp:346-385); multiples of 4 keep the 16-byte vector path
    const u64 n_q = field.params().n_q;
    qpk::GfqGemvParams G = F.gemv;
    G.chunk = lane_terms <= n_q ? 0u : static_cast<uint32_t>(n_q >= 4 ? n_q - n_q % 4 : n_q);
    StreamBuf ws(qpk::gemv_workspace_bytes(m, K, splits), s);
    check(qpk::launch_gfq_gemv(G, A, x, m, K, splits, ws.ptr, y_rep, y_coeff, s), "gfq_gemv launch");
}

void gfq_gemv_host(DeviceFieldCache& F, const GfqField& field, const uint32_t* A, const uint32_t* x, u64 m, u64 K,
                   uint32_t* y_rep, uint8_t* y_coeff, u64* zech_reads) {
    std::lock_guard<std::mutex> lock(F.mu);
    auto* da = static_cast<uint32_t*>(F.io_a.ensure(std::max<u64>(m * K, 1) * 4));
    auto* dx = static_cast<uint32_t*>(F.io_b.ensure(std::max<u64>(K, 1) * 4));
    auto* dy = static_cast<uint8_t*>(F.io_c.ensure(m * (4 + field.k())));
    if (m * K != 0) check(cudaMemcpy(da, A, m * K * 4, cudaMemcpyHostToDevice), "H2D");
    if (K) check(cudaMemcpy(dx, x, K * 4, cudaMemcpyHostToDevice), "H2D");
    uint32_t* dr = reinterpret_cast<uint32_t*>(dy);
    uint8_t* dc = dy + m * 4;
    gfq_gemv_device(F, field, da, dx, m, K, y_rep ? dr : nullptr, y_coeff ? dc : nullptr, 0);
    if (y_rep) check(cudaMemcpy(y_rep, dr, m * 4, cudaMemcpyDeviceToHost), "D2H");
    if (y_coeff) check(cudaMemcpy(y_coeff, dc, m * field.k(), cudaMemcpyDeviceToHost), "D2H");
    raise_field_status(take_field_status(F, 0));
    if (zech_reads) *zech_reads = zech_reads_device(F, field, da, dx, m, K, 1, 0);
}

CostReport gemv_cost(const GfqField& field, u64 m, u64 K) {
    // per row the reference fgdp_dot's counters (gfq.cpp:346-385) minus the
    // data-dependent Zech additions, as matmul_cost
    return matmul_cost(field, m, K, 1);
}

void gfq_gemv(std::span<const GfqElt> A, std::span<const GfqElt> x, std::size_t m, const GfqField& field,
              std::span<GfqElt> y, CostReport* cost) {
    const u64 K = x.size();
    if (A.size() != m * K || y.size() < m)
        throw std::invalid_argument("gfq_gemv: span sizes do not match m x K / K / m");
    for (const auto& v : {A, x})
        for (const GfqElt& e : v)
            if (e.rep >= field.order()) throw std::out_of_range("gfq_gemv: rep outside the field");
    static_assert(sizeof(GfqElt) == 4, "GfqElt is one u32 rep");
    u64 zech = 0;
    gfq_gemv_host(detail::device_field(field), field, reinterpret_cast<const uint32_t*>(A.data()),
                  reinterpret_cast<const uint32_t*>(x.data()), m, K, reinterpret_cast<uint32_t*>(y.data()), nullptr,
                  cost ? &zech : nullptr);
    if (cost) {
        *cost += gemv_cost(field, m, K);
        cost->table_accesses += zech;
    }
}

GfqElt fgdp_dot(std::span<const GfqElt> v1, std::span<const GfqElt> v2, const GfqField& field, CostReport* cost) {
    if (v1.size() != v2.size()) throw std::invalid_argument("fgdp_dot: vector length mismatch");
    GfqElt r{};
    gfq_gemv(v1, v2, 1, field, std::span<GfqElt>(&r, 1), cost);
    return r;
}

void gfq_matmul_coeffs(std::span<const std::uint8_t> A, std::span<const std::uint8_t> B, std::size_t m, std::size_t K,
                       std::size_t n, const GfqField& field, std::span<std::uint8_t> C, std::uint32_t chunk,
                       CostReport* cost, Repack repack) {
    const u64 k = field.k();
    if (A.size() != m * K * k || B.size() != K * n * k || C.size() < m * n * k)
        throw std::invalid_argument("gfq_matmul_coeffs: span sizes do not match m x K x k / K x n x k / m x n x k");
    u64 zech = 0;
    gfq_matmul_host(detail::device_field(field), field, A.data(), B.data(), m, K, n, chunk, C.data(), false,
                    static_cast<std::uint32_t>(repack), cost ? &zech : nullptr);
    if (cost) {
        *cost += matmul_cost(field, m, K, n);
        cost->table_accesses += zech;
    }
}

}  // namespace qpack::gpu

namespace qpack {

GfqMatrix gfq_matmul(const GfqMatrix& a, const GfqMatrix& b, const GfqField& field, CostReport* cost) {
    if (a.cols != b.rows) throw std::invalid_argument("gfq_matmul: inner dimensions differ");
    GfqMatrix c = GfqMatrix::zero(field, a.rows, b.cols);
    if (a.rows == 0 || b.cols == 0) return c;
    if (a.cols == 0) return c;
    for (const auto* mtx : {&a, &b})
        for (const GfqElt& e : mtx->data)
            if (e.rep >= field.order()) throw std::out_of_range("gfq_matmul: rep outside the field");
    u64 zech = 0;
    gpu::gfq_matmul_host(detail::device_field(field), field, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, 0,
                         c.data.data(), true, qpk::kRepackRedq, cost ? &zech : nullptr);
    if (cost) {
        *cost += gpu::matmul_cost(field, a.rows, a.cols, b.cols);
        cost->table_accesses += zech;  // the reference's Zech reads, replayed on the device (K7)
    }
    return c;
}

}  // namespace qpack
