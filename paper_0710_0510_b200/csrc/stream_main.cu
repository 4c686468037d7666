// Non-templated streaming kernels (generic-width REDQ, input generators,
// rep products), the launch dispatchers, and the device SM count.  The
// templated TMA pipeline lives in stream_kernels.cuh and is instantiated in
// stream_inst.cu.
#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"
#include "stream_inst.hpp"

namespace qpk {

namespace {


__device__ __forceinline__ uint32_t mod_small_g(uint32_t t, uint32_t p, uint32_t magic) {
    return t - p * __umulhi(t, magic);
}

__device__ __forceinline__ void report_g(uint32_t err, uint32_t* status) { report_status(err, status); }

// Generic REDQ for d+1 > kMaxFastDigits: one word per thread, runtime loops.
__global__ void redq_generic_kernel(const RedqParams P, const double* __restrict__ words, uint64_t n,
                                    uint8_t* __restrict__ out, uint32_t* status) {
    uint32_t err = 0;
    const uint32_t nd = P.d + 1;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double w = words[i];
        double r = trunc(w);
        if (!(w >= 0.0 && r < P.limit)) {
            err |= kErrDomain;
            r = 0.0;
        }
        const bool premul = r <= P.r_max;
        const uint64_t rb = __double2ull_rz(r);
        const uint64_t rop = premul ? floor_div_premul(r, P.inv_p) : rb / P.p;
        uint32_t u[kMaxDigits];
        for (uint32_t j = 0; j < nd; ++j) {
            uint64_t x, y;
            if (P.qbits) {
                x = rb >> (P.qbits * j);
                y = rop >> (P.qbits * j);
            } else {
                x = rb / P.qpow[j];
                y = rop / P.qpow[j];
            }
            u[j] = static_cast<uint32_t>(x) - P.p * static_cast<uint32_t>(y);
        }
        // direct correction (results equal the tabulated one, redq tests)
        if (P.neg_q)
            for (uint32_t j = 0; j + 1 < nd; ++j) u[j] = mod_small_g(u[j] + P.neg_q * u[j + 1], P.p, P.mod_magic);
        for (uint32_t j = 0; j < nd; ++j) out[i * nd + j] = static_cast<uint8_t>(u[j]);
    }
    report_g(err, status);
}

// REDQ of u64 integer words (any d, any q): one word per thread.  rop =
// floor(r/p) from a 32-bit division of the high half and the premultiplied
// fp64 floor (Lemma 1) of (hi mod p) 2^32 + lo < p 2^32 <= 2^40 <= r_max, so
// no 64-bit division runs for p; digits by shifts (q = 2^b) or by exact u64
// divisions by q^i.  The direct correction equals the tabulated one.
__global__ void redq_u64_kernel(const RedqParams P, const uint64_t* __restrict__ words, uint64_t n,
                                uint8_t* __restrict__ out, uint32_t* status) {
    uint32_t err = 0;
    const uint32_t nd = P.d + 1;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t r = words[i];
        if (P.limit_u64 && r >= P.limit_u64) {
            err |= kErrDomain;
            r = 0;
        }
        const uint32_t hi = static_cast<uint32_t>(r >> 32), lo = static_cast<uint32_t>(r);
        const uint32_t q1 = hi / P.p;
        const uint64_t t = (static_cast<uint64_t>(hi - q1 * P.p) << 32) | lo;
        const uint64_t rop = (static_cast<uint64_t>(q1) << 32) + floor_div_premul(static_cast<double>(t), P.inv_p);
        uint32_t u[kMaxDigits];
        for (uint32_t j = 0; j < nd; ++j) {
            uint64_t x, y;
            if (P.qbits) {
                const uint32_t sh = P.qbits * j;
                x = sh < 64 ? r >> sh : 0;
                y = sh < 64 ? rop >> sh : 0;
            } else if (P.qpow64[j]) {
                x = r / P.qpow64[j];
                y = rop / P.qpow64[j];
            } else {
                x = y = 0;
            }
            u[j] = static_cast<uint32_t>(x) - P.p * static_cast<uint32_t>(y);
        }
        if (P.neg_q)
            for (uint32_t j = 0; j + 1 < nd; ++j) u[j] = mod_small_g(u[j] + P.neg_q * u[j + 1], P.p, P.mod_magic);
        for (uint32_t j = 0; j < nd; ++j) out[i * nd + j] = static_cast<uint8_t>(u[j]);
    }
    report_g(err, status);
}

// REDQ of u128 words (one per thread): rop = r / p, u_j = r/q^j - p (rop/q^j)
// (shifts for q = 2^b, u128 divisions by q^j otherwise), direct correction
__global__ void redq_u128_kernel(const RedqParams P, const unsigned __int128* __restrict__ words, uint64_t n,
                                 unsigned __int128 limit, uint8_t* __restrict__ out, uint32_t* status) {
    using u128d = unsigned __int128;
    pdl_wait();
    uint32_t err = 0;
    const uint32_t nd = P.d + 1;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        u128d r = words[i];
        if (limit && r >= limit) {
            err |= kErrDomain;
            r = 0;
        }
        const u128d rop = r / P.p;
        uint32_t u[kMaxDigits];
        u128d qj = 1;
        for (uint32_t j = 0; j < nd; ++j) {
            u128d x, y;
            if (P.qbits) {
                const uint32_t sh = P.qbits * j;
                x = sh < 128 ? r >> sh : 0;
                y = sh < 128 ? rop >> sh : 0;
            } else {
                x = r / qj;
                y = rop / qj;
                qj *= P.q;
            }
            u[j] = static_cast<uint32_t>(static_cast<uint64_t>(x) - P.p * static_cast<uint64_t>(y));
        }
        if (P.neg_q)
            for (uint32_t j = 0; j + 1 < nd; ++j) u[j] = mod_small_g(u[j] + P.neg_q * u[j + 1], P.p, P.mod_magic);
        for (uint32_t j = 0; j < nd; ++j) out[i * nd + j] = static_cast<uint8_t>(u[j]);
    }
    report_g(err, status);
}

// field ops over reps (gfq.cpp:260-294); the zero element is rep g; reps
// above g latch kErrRep and are read as zero
__global__ void gfq_rep_op_kernel(int op, uint32_t p, uint32_t group, const uint32_t* __restrict__ zech,
                                  const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                                  uint32_t* __restrict__ out, uint32_t* status) {
    pdl_wait();
    uint32_t err = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t x = a[i];
        if (x > group) err |= kErrRep, x = group;
        uint32_t r;
        if (op == 0) {  // mul: (a + b) mod g, zero absorbs
            uint32_t y = b[i];
            if (y > group) err |= kErrRep, y = group;
            r = (x == group || y == group) ? group : (x + y >= group ? x + y - group : x + y);
        } else if (op == 1) {  // add through the Zech table: a + plus1[(b - a) mod g]
            uint32_t y = b[i];
            if (y > group) err |= kErrRep, y = group;
            if (x == group) {
                r = y;
            } else if (y == group) {
                r = x;
            } else {
                const uint32_t t = zech[y >= x ? y - x : y + group - x];
                r = t == group ? group : (x + t >= group ? x + t - group : x + t);
            }
        } else if (op == 2) {  // neg: a + g/2 (p odd), identity for p = 2
            r = (x == group || p == 2) ? x : (x + group / 2 >= group ? x + group / 2 - group : x + group / 2);
        } else {  // inverse: (g - a) mod g
            if (x == group) err |= kErrDomain;
            r = x == 0 ? 0 : group - x;
        }
        out[i] = r;
    }
    report_g(err, status);
}

__global__ void gfq_mul_rep_kernel(uint32_t group, const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                   uint64_t n, uint32_t* __restrict__ out, uint32_t* status) {
    uint32_t err = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t x = a[i], y = b[i];
        if (x > group || y > group) err |= kErrRep, x = min(x, group), y = min(y, group);
        uint32_t r = x + y;
        if (r >= group) r -= group;
        out[i] = (x == group || y == group) ? group : r;
    }
    report_g(err, status);
}

// ------------------------------------------------------------- generators
__global__ void gen_draws_kernel(uint64_t seed, uint64_t start, uint64_t count, uint32_t bound, uint8_t* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint8_t>(splitmix_at(seed, start + i + 1) % bound);
}

__global__ void gen_words_kernel(uint64_t seed, uint64_t first, uint64_t n, uint64_t q, uint32_t d, double* out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t r = 0;
        for (uint32_t j = 0; j <= d; ++j) r = r * q + splitmix_at(seed, (first + i) * (d + 1) + j + 1) % q;
        out[i] = static_cast<double>(r);
    }
}

__global__ void gen_pairs_kernel(uint64_t seed, uint64_t n, uint32_t k, uint32_t bound, uint8_t* a, uint8_t* b) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * k;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t rec = i / k, c = i % k;
        a[i] = static_cast<uint8_t>(splitmix_at(seed, rec * 2 * k + c + 1) % bound);
        b[i] = static_cast<uint8_t>(splitmix_at(seed, rec * 2 * k + k + c + 1) % bound);
    }
}

unsigned grid_for(uint64_t n) {
    return static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
}

}  // namespace

int num_sms() {
    // per device ordinal (a process may drive several GPUs)
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

cudaError_t ensure_dyn_smem(const void* kernel, size_t bytes, size_t static_bytes) {
    // the 48 KB a launch gets without the attribute covers static + dynamic
    if (bytes + static_bytes <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[{kernel, dev}];
    if (bytes <= cur) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e == cudaSuccess) cur = bytes;
    return e;
}

cudaError_t launch_redq_f64(const RedqParams& P, const double* words, uint64_t n, uint8_t* out, uint32_t* status,
                            cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    switch (P.d + 1) {
        case 1: return redq_launch_nd1(P, words, n, out, status, s);
        case 2: return redq_launch_nd2(P, words, n, out, status, s);
        case 3: return redq_launch_nd3(P, words, n, out, status, s);
        case 4: return redq_launch_nd4(P, words, n, out, status, s);
        case 5: return redq_launch_nd5(P, words, n, out, status, s);
        case 6: return redq_launch_nd6(P, words, n, out, status, s);
        case 7: return redq_launch_nd7(P, words, n, out, status, s);
        case 8: return redq_launch_nd8(P, words, n, out, status, s);
        default:
            redq_generic_kernel<<<grid_for(n), 256, 0, s>>>(P, words, n, out, status);
            return cudaGetLastError();
    }
}

cudaError_t launch_redq_u64(const RedqParams& P, const uint64_t* words, uint64_t n, uint8_t* out, uint32_t* status,
                            cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (P.d + 1 > uint32_t(kMaxDigits)) return cudaErrorInvalidValue;
    redq_u64_kernel<<<grid_for(n), 256, 0, s>>>(P, words, n, out, status);
    return cudaGetLastError();
}

cudaError_t launch_gfq_rep_op(int op, uint32_t p, uint32_t group, const uint32_t* zech, const uint32_t* a,
                              const uint32_t* b, uint64_t n, uint32_t* out, uint32_t* status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (op < 0 || op > 3) return cudaErrorInvalidValue;
    return launch_pdl(gfq_rep_op_kernel, dim3(grid_for(n)), dim3(256), 0, s, op, p, group, zech, a, b, n, out, status);
}

cudaError_t launch_redq_u128(const RedqParams& P, const uint64_t* words, uint64_t n, uint8_t* out, uint32_t* status,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (P.d + 1 > uint32_t(kMaxDigits) || P.p > 256) return cudaErrorInvalidValue;
    // q^(d+1) as u128, 0 when it exceeds 2^128 (every u128 word then qualifies)
    unsigned __int128 limit = 1;
    for (uint32_t j = 0; j <= P.d && limit; ++j) {
        const unsigned __int128 next = limit * P.q;
        limit = (P.q != 0 && next / P.q == limit) ? next : 0;
    }
    return launch_pdl(redq_u128_kernel, dim3(grid_for(n)), dim3(256), 0, s, P,
                      reinterpret_cast<const unsigned __int128*>(words), n, limit, out, status);
}

cudaError_t launch_polymul(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                           uint32_t* status, cudaStream_t s) {
    switch (P.k) {
        case 1: return polymul_launch_k1(P, a, b, n, out, status, s);
        case 2: return polymul_launch_k2(P, a, b, n, out, status, s);
        case 3: return polymul_launch_k3(P, a, b, n, out, status, s);
        case 4: return polymul_launch_k4(P, a, b, n, out, status, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gfq_elem(const GfqElemParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                            cudaStream_t s) {
    switch (P.k) {
        case 1: return gfq_elem_launch_k1(P, a, b, n, out, s);
        case 2: return gfq_elem_launch_k2(P, a, b, n, out, s);
        case 3: return gfq_elem_launch_k3(P, a, b, n, out, s);
        case 4: return gfq_elem_launch_k4(P, a, b, n, out, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gfq_mul_rep(uint32_t group, const uint32_t* a, const uint32_t* b, uint64_t n, uint32_t* out,
                               uint32_t* status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    gfq_mul_rep_kernel<<<grid_for(n), 256, 0, s>>>(group, a, b, n, out, status);
    return cudaGetLastError();
}

cudaError_t launch_gen_draws(uint64_t seed, uint64_t start, uint64_t count, uint32_t bound, uint8_t* out,
                             cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    gen_draws_kernel<<<grid_for(count), 256, 0, s>>>(seed, start, count, bound, out);
    return cudaGetLastError();
}

cudaError_t launch_gen_words(uint64_t seed, uint64_t first, uint64_t n, uint64_t q, uint32_t d, double* out,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    gen_words_kernel<<<grid_for(n), 256, 0, s>>>(seed, first, n, q, d, out);
    return cudaGetLastError();
}

cudaError_t launch_gen_pairs(uint64_t seed, uint64_t n, uint32_t k, uint32_t bound, uint8_t* a, uint8_t* b,
                             cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    gen_pairs_kernel<<<grid_for(n * k), 256, 0, s>>>(seed, n, k, bound, a, b);
    return cudaGetLastError();
}

}  // namespace qpk
