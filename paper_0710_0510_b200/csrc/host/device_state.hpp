// Device mirrors of the host plan objects (internal to libqpack_b200.so).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels.hpp"
#include "qpack/gfq.hpp"
#include "qpack/params.hpp"
#include "qpack/redq.hpp"

namespace qpack::gpu {

// any CUDA failure (maps to QPK_ERR_CUDA in the C-ABI)
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what);
void require_device();

// grow-only device allocation
struct DevBuf {
    void* ptr = nullptr;
    std::size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    void* ensure(std::size_t n);
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

// Per-call device workspace in stream order (cudaMallocAsync / cudaFreeAsync
// from the default pool): concurrent calls on different streams never share
// scratch, like the reference's pure functions (SURVEY 8(b) "Threading"),
// and the pool keeps repeated calls allocation-free.
struct StreamBuf {
    void* ptr = nullptr;
    cudaStream_t s = nullptr;
    StreamBuf(std::size_t bytes, cudaStream_t stream);
    StreamBuf(const StreamBuf&) = delete;
    StreamBuf& operator=(const StreamBuf&) = delete;
    ~StreamBuf();
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

// Chunked host<->device pipeline for the `_host` entry points.  Chunk c's
// inputs go up on the H2D stream, its kernel runs on the compute stream and
// its outputs come back on the D2H stream; events chain the three and
// recycle one of kSlots device buffer sets, so each copy engine sees an
// uninterrupted queue of its own direction.  (Measured on B200, C2 e2e:
// 4 round-robin streams each running H2D->kernel->D2H left the two
// directions partly serialised.)
struct Staging {
    static constexpr int kSlots = 4;
    cudaStream_t sh = nullptr, sk = nullptr, sd = nullptr;
    cudaStream_t sk2 = nullptr;  // second compute stream (row bands of a matrix product alternate)
    cudaEvent_t ev_aux = nullptr;
    cudaEvent_t ev_in[kSlots] = {}, ev_k[kSlots] = {}, ev_out[kSlots] = {};
    DevBuf in0[kSlots], in1[kSlots], out[kSlots];
    Staging();
    ~Staging();
    // h2d(slot, off, cnt, stream), kern(slot, off, cnt, stream),
    // d2h(slot, off, cnt, stream) for chunks [off, off+cnt) of n records;
    // returns after the last D2H completed
    template <class H, class K, class O>
    void run(std::uint64_t n, std::uint64_t chunk, H h2d, K kern, O d2h) {
        for (std::uint64_t off = 0, c = 0; off < n; off += chunk, ++c) {
            const int sl = static_cast<int>(c % kSlots);
            const std::uint64_t cnt = n - off < chunk ? n - off : chunk;
            if (c >= kSlots) check(cudaStreamWaitEvent(sh, ev_out[sl], 0), "wait slot");
            h2d(sl, off, cnt, sh);
            check(cudaEventRecord(ev_in[sl], sh), "event");
            check(cudaStreamWaitEvent(sk, ev_in[sl], 0), "wait h2d");
            kern(sl, off, cnt, sk);
            check(cudaEventRecord(ev_k[sl], sk), "event");
            check(cudaStreamWaitEvent(sd, ev_k[sl], 0), "wait kernel");
            d2h(sl, off, cnt, sd);
            check(cudaEventRecord(ev_out[sl], sd), "event");
        }
        check(cudaStreamSynchronize(sd), "sync");
        check(cudaStreamSynchronize(sk), "sync");
    }
};

}  // namespace qpack::gpu

namespace qpack::detail {

struct DevicePlanCache {
    std::uint64_t gen = 0;  // RedqPlan::correction_gen the constants were built from
    qpk::RedqParams prm{};
    gpu::DevBuf table;   // byte-packed correction windows
    gpu::DevBuf status;  // latched kErr* bits
    gpu::DevBuf io_a, io_b, io_c;
    std::mutex mu;
    std::unique_ptr<gpu::Staging> staging;
};

struct DeviceFieldCache {
    gpu::DevBuf tables;  // lc | hc | log | alog  (u32)
    gpu::DevBuf fval;    // rep -> q-adic double
    gpu::DevBuf zech;    // plus-one table (GfqField::add), uploaded on first use
    gpu::DevBuf status;  // data-error flag of the rep ops (inverse of zero)
    gpu::DevBuf lh_reps; // low | high as reps, for the K7 counter (uploaded on first use)
    // fields outside the byte-packed form (k > 4 or p > 255): rep-domain
    // kernels (gfq_wide.cu) over log | antilog | low | high | zech
    bool wide = false;
    gpu::DevBuf wide_tabs;
    qpk::GfqWideParams wp{};
    gpu::DevBuf counter; // K7 total
    qpk::GfqElemParams elem{};
    qpk::GfqMatmulParams mm{};
    qpk::GfqGemvParams gemv{};
    uint32_t nlh = 0;
    gpu::DevBuf io_a, io_b, io_c;
    std::mutex mu;
    std::unique_ptr<gpu::Staging> staging;
};

struct FieldAccess {
    static const std::vector<u32>& log(const GfqField& f) { return f.log_; }
    static const std::vector<u64>& antilog(const GfqField& f) { return f.antilog_; }
    static const std::vector<u32>& zech(const GfqField& f) { return f.zech_; }
    static const std::vector<double>& fval(const GfqField& f) { return f.fval_; }
    static const std::vector<u32>& low(const GfqField& f) { return f.low_; }
    static const std::vector<u32>& high(const GfqField& f) { return f.high_; }
    static u64 lh_radix(const GfqField& f) { return f.lh_radix_; }
    static u64 q(const GfqField& f) { return f.q_; }
    static std::shared_ptr<DeviceFieldCache>& device(const GfqField& f) { return f.device_; }
};

// Device parameter block of a REDQ plan; uploads its table into `table`.
qpk::RedqParams make_redq_params(const RedqPlan& plan, gpu::DevBuf* table);
DevicePlanCache& device_plan(const RedqPlan& plan);
DeviceFieldCache& device_field(const GfqField& f);

// closed-form reference counters
CostReport redq_batch_cost(const RedqPlan& plan, u64 n);

}  // namespace qpack::detail
