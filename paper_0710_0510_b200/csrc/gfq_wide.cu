// GF(p^k) on the device for the fields outside the byte-packed fast form
// (k > 4 or p > 255: GF(2^5..2^8), GF(3^5), GF(3^6), GF(257^2), GF(p) with a
// large p, ... -- every field the reference builds at m = 53; SURVEY.md
// section 8(a) a15-a17).  Everything stays in the rep domain as the
// reference does: each REDQ group's raw digits index the low/high half
// tables (reps), the halves and the running sums are added through the Zech
// table (GfqField::add, gfq.cpp:266-275), field tables read through the
// read-only cache (they may exceed shared memory: up to 2^20 entries).
//
//   * elementwise product of coefficient records (p < 256: k bytes each),
//     dlog path (gfq.cpp:260-264) or DQT/REDQ/L-H path (gfq.cpp:353-384);
//   * GEMV / long dot on reps (fgdp_dot per row, gfq.cpp:335-387): one warp
//     per (row, K-split) task, a group closed every n_q products per lane,
//     lane sums combined by Zech additions; the product C = A*B of these
//     fields runs as GEMVs over B's columns (gpu_api.cpp gfq_matmul_by_columns).
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

namespace {

__device__ __forceinline__ uint32_t wide_add(const GfqWideParams& P, uint32_t a, uint32_t b) {
    const uint32_t g = P.group;
    if (a == g) return b;
    if (b == g) return a;
    const uint32_t t = __ldg(P.zech + (b + g - a) % g);
    return t == g ? g : static_cast<uint32_t>((static_cast<uint64_t>(a) + t) % g);
}

// REDQ of an exact integer word (< 2^53) and the two half-window lookups,
// added: the field element of one group (gfq.cpp:362-384)
__device__ __forceinline__ uint32_t wide_group(const GfqWideParams& P, uint64_t r) {
    const uint64_t rop = r / P.p;
    uint64_t il = 0, ih = 0;
    uint64_t u[2 * kMaxWideK - 1];
    const uint32_t nd = 2 * P.k - 1;
    for (uint32_t d = 0; d < nd; ++d) {
        const uint64_t x = P.qbits ? r >> (P.qbits * d) : r / P.qpow[d];
        const uint64_t y = P.qbits ? rop >> (P.qbits * d) : rop / P.qpow[d];
        u[d] = x - uint64_t(P.p) * y;
    }
    for (uint32_t t = P.k; t-- > 0;) {
        il = il * P.lh_radix + u[t];
        ih = ih * P.lh_radix + u[P.k - 1 + t];
    }
    return wide_add(P, __ldg(P.high + ih), __ldg(P.low + il));
}

// coefficient bytes of a rep (to_coeffs: base-p digits of its polynomial index)
__device__ __forceinline__ void wide_store(const GfqWideParams& P, uint32_t rep, uint8_t* dst) {
    uint32_t idx = rep == P.group ? 0u : __ldg(P.antilog + rep);
    for (uint32_t j = 0; j < P.k; ++j, idx /= P.p) dst[j] = static_cast<uint8_t>(idx % P.p);
}

__global__ void wide_mul_kernel(const GfqWideParams P, const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                uint64_t n, uint8_t* __restrict__ out, int path) {
    pdl_wait();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t ia = 0, ib = 0;
        double wa = 0.0, wb = 0.0;
        const double qd = static_cast<double>(P.qpow[1]);
        for (int j = static_cast<int>(P.k) - 1; j >= 0; --j) {
            const uint32_t ca = a[i * P.k + j] % P.p, cb = b[i * P.k + j] % P.p;  // from_coeffs reduces mod p
            ia = ia * P.p + ca;
            ib = ib * P.p + cb;
            wa = fma(wa, qd, static_cast<double>(ca));  // DQT pack (dqt.cpp:23-37), exact
            wb = fma(wb, qd, static_cast<double>(cb));
        }
        uint32_t rep;
        if (path == kGfqDlog) {
            const uint32_t ra = __ldg(P.log + ia), rb = __ldg(P.log + ib), g = P.group;
            rep = (ra == g || rb == g) ? g : static_cast<uint32_t>((uint64_t(ra) + rb) % g);
        } else {
            rep = wide_group(P, static_cast<uint64_t>(wa * wb));  // the fp64 product, exact below 2^53
        }
        wide_store(P, rep, out + i * P.k);
    }
}

__global__ void __launch_bounds__(256) wide_gemv_kernel(const GfqWideParams P, const uint32_t* __restrict__ A,
                                                        const uint32_t* __restrict__ x, uint64_t m, uint64_t K,
                                                        uint32_t splits, uint64_t ksplit, uint32_t* __restrict__ ws) {
    pdl_wait();
    const uint32_t lane = threadIdx.x & 31u, warps = blockDim.x >> 5;
    const uint32_t last = P.group;  // reps above it: read as zero, latched
    uint32_t err = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * warps + (threadIdx.x >> 5); t < m * splits;
         t += uint64_t(gridDim.x) * warps) {
        const uint64_t row = t / splits, s = t % splits;
        const uint64_t k0 = s * ksplit, k1 = k0 + ksplit < K ? k0 + ksplit : K;
        uint32_t sum = P.group, cnt = 0;
        double acc = 0.0;
        for (uint64_t j = k0 + lane; j < k1; j += 32) {
            uint32_t ea = __ldg(A + row * K + j), ex = __ldg(x + j);
            if (ea > last || ex > last) err |= kErrRep, ea = min(ea, last), ex = min(ex, last);
            acc = fma(__ldg(P.fval + ea), __ldg(P.fval + ex), acc);
            if (++cnt == P.chunk) {
                sum = wide_add(P, sum, wide_group(P, static_cast<uint64_t>(acc)));
                acc = 0.0;
                cnt = 0;
            }
        }
        if (cnt) sum = wide_add(P, sum, wide_group(P, static_cast<uint64_t>(acc)));
        for (int off = 16; off > 0; off >>= 1) sum = wide_add(P, sum, __shfl_xor_sync(0xffffffffu, sum, off));
        if (lane == 0) ws[s * m + row] = sum;
    }
    report_status(err, P.status);
}

__global__ void wide_finish_kernel(const GfqWideParams P, const uint32_t* __restrict__ ws, uint64_t m,
                                   uint32_t splits, uint32_t* __restrict__ out_rep, uint8_t* __restrict__ out_coeff) {
    pdl_wait();
    for (uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < m;
         row += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t sum = P.group;
        for (uint32_t s = 0; s < splits; ++s) sum = wide_add(P, sum, ws[s * m + row]);
        if (out_rep) out_rep[row] = sum;
        if (out_coeff) wide_store(P, sum, out_coeff + row * P.k);
    }
}

__global__ void wide_reps_to_coeffs_kernel(const GfqWideParams P, const uint32_t* __restrict__ reps, uint64_t n,
                                           uint8_t* __restrict__ out) {
    pdl_wait();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        wide_store(P, min(reps[i], P.group), out + i * P.k);
}

unsigned grid_of(uint64_t items, unsigned per_cta) {
    const uint64_t g = (items + per_cta - 1) / per_cta, cap = uint64_t(num_sms()) * 16;
    return static_cast<unsigned>(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

cudaError_t launch_gfq_wide_mul(const GfqWideParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                                int path, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    return launch_pdl(wide_mul_kernel, dim3(grid_of(n, 256)), dim3(256), 0, s, P, a, b, n, out, path);
}

uint64_t gfq_wide_workspace_bytes(uint64_t m, uint64_t K) {
    const uint64_t splits = K / 4096 + 1;
    return splits * m * 4 + 16;
}

cudaError_t launch_gfq_wide_gemv(const GfqWideParams& P, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t K,
                                 void* ws, uint32_t* out_rep, uint8_t* out_coeff, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    const uint32_t splits = static_cast<uint32_t>(K / 4096 + 1);  // 4096-term tasks: enough warps for long dots
    const uint64_t ksplit = (K + splits - 1) / splits;
    auto* part = static_cast<uint32_t*>(ws);
    if (cudaError_t e = launch_pdl(wide_gemv_kernel, dim3(grid_of(m * splits, 8)), dim3(256), 0, s, P, A, x, m, K,
                                   splits, ksplit, part);
        e != cudaSuccess)
        return e;
    return launch_pdl(wide_finish_kernel, dim3(grid_of(m, 256)), dim3(256), 0, s, P,
                      static_cast<const uint32_t*>(part), m, splits, out_rep, out_coeff);
}

cudaError_t launch_gfq_wide_reps_to_coeffs(const GfqWideParams& P, const uint32_t* reps, uint64_t n, uint8_t* out,
                                           cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    return launch_pdl(wide_reps_to_coeffs_kernel, dim3(grid_of(n, 256)), dim3(256), 0, s, P, reps, n, out);
}

}  // namespace qpk
