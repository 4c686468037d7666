// K7: the data-dependent part of gfq_matmul's table_accesses counter.
//
// The reference's gfq_matmul (gfq.cpp:389-404) runs fgdp_dot (gfq.cpp:335-387)
// per output: groups of n_q products, each closed by REDQ and two half-window
// lookups, then two Zech additions -- add(H, L) and add(result, group_sum) --
// each of which reads the Zech table only when both operands are nonzero
// (gfq.cpp:266-275).  Everything else in CostReport is closed form; this
// kernel replays the reference's grouping per output and counts those reads.
// It runs only when a caller asks for counters (the product itself comes
// from the DMMA kernel): one thread per output, A's row broadcast across the
// warp, B's row read coalesced, the field tables through the read-only cache.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

namespace {

// GfqField::add on reps (zero = g): one table read when both are nonzero
__device__ __forceinline__ uint32_t zech_add(const GfqCountParams& P, uint32_t a, uint32_t b, uint32_t& reads) {
    const uint32_t g = P.group;
    if (a == g) return b;
    if (b == g) return a;
    ++reads;
    const uint32_t t = __ldg(P.zech + (b + g - a) % g);
    return t == g ? g : static_cast<uint32_t>((static_cast<uint64_t>(a) + t) % g);
}

__global__ void __launch_bounds__(256) gfq_count_kernel(const GfqCountParams P, const uint32_t* __restrict__ A,
                                                        const uint32_t* __restrict__ B, uint64_t m, uint64_t K,
                                                        uint64_t n, unsigned long long* __restrict__ total) {
    pdl_wait();
    uint64_t mine = 0;
    const uint32_t nd = 2 * P.k - 1;
    for (uint64_t o = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < m * n; o += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = o / n, j = o % n;
        uint32_t result = P.group, reads = 0;
        for (uint64_t l0 = 0; l0 < K; l0 += P.n_q) {
            const uint64_t l1 = l0 + P.n_q < K ? l0 + P.n_q : K;
            double acc = 0.0;  // exact: the group's word stays below q^(2k-1) < 2^53
            for (uint64_t l = l0; l < l1; ++l)
                acc = fma(__ldg(P.fval + __ldg(A + i * K + l)), __ldg(P.fval + __ldg(B + l * n + j)), acc);
            const uint64_t r = static_cast<uint64_t>(acc), rop = r / P.p;
            uint64_t u[2 * kMaxCountK - 1];
            for (uint32_t d = 0; d < nd; ++d) {  // raw digits (redq.cpp:44-58)
                const uint64_t x = P.qbits ? r >> (P.qbits * d) : r / P.qpow[d];
                const uint64_t y = P.qbits ? rop >> (P.qbits * d) : rop / P.qpow[d];
                u[d] = x - static_cast<uint64_t>(P.p) * y;
            }
            // half-window indices over digits 0..k-1 and k-1..2k-2 (gfq.cpp:370-376)
            uint64_t il = 0, ih = 0;
            for (uint32_t t = P.k; t-- > 0;) {
                il = il * P.lh_radix + u[t];
                ih = ih * P.lh_radix + u[P.k - 1 + t];
            }
            const uint32_t h = __ldg(P.high + ih), lo = __ldg(P.low + il);
            const uint32_t gs = zech_add(P, h, lo, reads);
            result = zech_add(P, result, gs, reads);
        }
        mine += reads;
    }
    // one atomic per warp
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, static_cast<unsigned long long>(mine));
}

}  // namespace

cudaError_t launch_gfq_count(const GfqCountParams& P, const uint32_t* A, const uint32_t* B, uint64_t m, uint64_t K,
                             uint64_t n, unsigned long long* total, cudaStream_t s) {
    if (m == 0 || n == 0 || K == 0) return cudaSuccess;
    const uint64_t outs = m * n;
    const unsigned grid = static_cast<unsigned>((outs + 255) / 256 < uint64_t(num_sms()) * 16 ? (outs + 255) / 256
                                                                                               : uint64_t(num_sms()) * 16);
    return launch_pdl(gfq_count_kernel, dim3(grid), dim3(256), 0, s, P, A, B, m, K, n, total);
}

}  // namespace qpk
