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

// pinned-free chunked host<->device pipeline resources
struct Staging {
    static constexpr int kStreams = 4;
    cudaStream_t streams[kStreams] = {};
    DevBuf in0[kStreams], in1[kStreams], out[kStreams];
    Staging();
    ~Staging();
};

}  // namespace qpack::gpu

namespace qpack::detail {

struct DevicePlanCache {
    qpk::RedqParams prm{};
    gpu::DevBuf table;   // byte-packed correction windows
    gpu::DevBuf status;  // latched kErr* bits
    gpu::DevBuf ws_fqt;  // K6 packed chunks and residue partials
    gpu::DevBuf io_a, io_b, io_c;
    std::mutex mu;
    std::unique_ptr<gpu::Staging> staging;
};

struct DeviceFieldCache {
    gpu::DevBuf tables;  // lc | hc | log | alog  (u32)
    gpu::DevBuf fval;    // rep -> q-adic double
    qpk::GfqElemParams elem{};
    qpk::GfqMatmulParams mm{};
    qpk::GfqGemvParams gemv{};
    uint32_t nlh = 0;
    gpu::DevBuf ws_a, ws_b;  // packed A^T and B
    gpu::DevBuf ws_gemv;     // GEMV split partials
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
