// K6: chunked FQT product of two long polynomials over F_p (reference
// fqt_mul, polymul.cpp:81-147 = paper Sec. 5 d-FQT).
//
//  * pack: each operand is cut into chunks of k = d+1 coefficients and every
//    chunk packed into one q-adic word (fqt_encode, polymul.cpp:31-50), as an
//    exact double;
//  * product: output chunk t is sum_i pw[i] * qw[t-i] -- a 1-D convolution
//    of packed words, each fp64 product carrying a (d+1)x(d+1) block of
//    coefficient products.  A CTA sweeps i through shared-memory tiles (pw
//    broadcast, qw sliding window) for 2048 consecutive t, 8 per thread in
//    registers (n_q >= 8), or 256 t, one per thread, when a REDQ follows
//    nearly every product (n_q < 8); grid.y splits the i range;
//  * groups of at most n_q products are closed by REDQ (Alg. 2/3): the 2d+1
//    residues are added mod p into the thread's byte lanes, exactly as the
//    reference's per-group redq_residues_into + overlap-add;
//  * overlap-add: output coefficient c of chunk u is residue j of t = u plus
//    residue j+k of t = u-1, summed over the i splits, mod p.
// The result is the unique product mod p, so the grouping (which products
// share a REDQ) may differ from the reference's; the counters reported by
// the host are the reference's closed form.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"
#include "redq_core.cuh"

namespace qpk {

namespace {

constexpr int kFqtT = 256;  // output chunks per CTA (one per thread)
constexpr int kFqtI = 256;  // i-tile

__device__ __forceinline__ uint32_t add_mod_lanes(uint32_t x, uint32_t y, uint32_t p) {
    if (p < 128) {
        const uint32_t pp = p * 0x01010101u;
        const uint32_t s = __vadd4(x, y);
        return __vsub4(s, __vcmpgeu4(s, pp) & pp);
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t t = ((x >> (8 * i)) & 0xff) + ((y >> (8 * i)) & 0xff);
        if (t >= p) t -= p;
        r |= t << (8 * i);
    }
    return r;
}

// chunks of k coefficients (reduced mod p) -> q-adic words; chunk c of an
// operand of n coefficients, zero beyond n (fqt_encode, polymul.cpp:31-50)
__global__ void fqt_pack_kernel(uint32_t p, uint32_t k, double qd, const uint8_t* __restrict__ a, uint64_t n,
                                uint64_t chunks, double* __restrict__ w) {
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < chunks;
         c += uint64_t(gridDim.x) * blockDim.x) {
        double v = 0.0;
        for (int j = static_cast<int>(k) - 1; j >= 0; --j) {
            const uint64_t i = c * k + j;
            const uint32_t x = i < n ? a[i] % p : 0u;
            v = fma(v, qd, static_cast<double>(x));
        }
        w[c] = v;
    }
}

// n_q < 8 (e.g. C1's q = 2^5, d = 3, n_q = 1): one output chunk per thread,
// a REDQ after every group of at most n_q products; the register-blocked
// kernel would run 8 REDQs per step at a quarter of the occupancy.  SWAR3:
// p = 3 and q = 2^4..2^7 through Swar3 (about 20 instructions per REDQ
// instead of ~100 for the per-digit path).
template <int ND, int W, class K, int SWAR_B>
__global__ void __launch_bounds__(kFqtT) fqt_conv_step_kernel(const FqtParams P, const double* __restrict__ pw,
                                                         uint64_t L1, const double* __restrict__ qw, uint64_t L2,
                                                         uint64_t T, uint64_t isplit, uint32_t* __restrict__ res) {
    constexpr int NW = (ND + 3) / 4;
    __shared__ double pws[kFqtI];
    __shared__ double qws[kFqtT + kFqtI - 1];
    extern __shared__ __align__(16) uint32_t tab[];
    const int tid = threadIdx.x;
    if constexpr (W > 0)
        for (uint32_t i = tid; i < P.rq.n_entries; i += blockDim.x) tab[i] = P.rq.table[i];
    const K c{P.rq};
    const uint32_t tab_s = smem_addr(tab);

    const uint64_t t0 = uint64_t(blockIdx.x) * kFqtT, t = t0 + tid;
    const uint64_t s = blockIdx.y;
    // i with some t - i in [0, L2) for this tile, within split s
    // chunk s (isplit products long) of this tile's own i range: every
    // non-final chunk is the same work, empty chunks exit at once
    const uint64_t tlo = t0 + 1 > L2 ? t0 + 1 - L2 : 0, thi = std::min<uint64_t>(L1, t0 + kFqtT);
    const uint64_t lo = tlo + s * isplit, hi = std::min<uint64_t>(thi, lo + isplit);
    double acc = 0.0;
    uint32_t cnt = 0;
    uint32_t racc[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) racc[w] = 0;
    constexpr bool SWAR3 = SWAR_B > 0;
    using SW = Swar3<SWAR3 ? SWAR_B : 4, ND>;
    uint64_t lacc = 0;
    uint32_t ladds = 0;
    auto close_group = [&]() {
        if constexpr (SWAR3) {
            lacc += SW::mu(acc, P.rq.inv_p);
            if (++ladds == SW::adds) {
                lacc = SW::fold(lacc);
                ladds = 0;
            }
            acc = 0.0;
            cnt = 0;
            return;
        }
        uint32_t u[ND], mu[ND];
        redq_raw_digits<ND>(c, acc, u);
        redq_correct<ND, W>(c, u, mu, [&](uint32_t idx) { return lds_u32(tab_s + 4 * idx); });
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            uint32_t v = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (4 * w + j < ND) v |= mu[4 * w + j] << (8 * j);
            racc[w] = add_mod_lanes(racc[w], v, c.p());
        }
        acc = 0.0;
        cnt = 0;
    };
    for (uint64_t i0 = lo; i0 < hi; i0 += kFqtI) {
        const int n_i = static_cast<int>(std::min<uint64_t>(kFqtI, hi - i0));
        __syncthreads();
        pws[tid] = tid < n_i ? pw[i0 + tid] : 0.0;
        // qws[jj] = qw[t0 - i0 - (kFqtI-1) + jj]
        for (int jj = tid; jj < kFqtT + kFqtI - 1; jj += kFqtT) {
            const int64_t qi = static_cast<int64_t>(t0) - static_cast<int64_t>(i0) - (kFqtI - 1) + jj;
            qws[jj] = (qi >= 0 && qi < static_cast<int64_t>(L2)) ? qw[qi] : 0.0;
        }
        __syncthreads();
        // term ii: pws[ii] * qws[tid + kFqtI - 1 - ii]; every thread counts
        // the same terms (out-of-range products are zeros), so group closes
        // are CTA-uniform
        int ii = 0;
        if (P.nq == 1) {
            const double* pq = qws + tid + kFqtI - 1;
#pragma unroll 4
            for (; ii < n_i; ++ii) {
                acc = pws[ii] * pq[-ii];
                close_group();
            }
        }
        while (ii < n_i) {
            const int run = min(n_i - ii, static_cast<int>(P.nq - cnt));
            const double* pq = qws + tid + kFqtI - 1 - ii;
#pragma unroll 4
            for (int r = 0; r < run; ++r) acc = fma(pws[ii + r], pq[-r], acc);
            ii += run;
            cnt += run;
            if (cnt == P.nq) close_group();
        }
    }
    if (cnt) close_group();
    if constexpr (SWAR3) {
        lacc = SW::fold(lacc);
#pragma unroll
        for (int j = 0; j < ND; ++j)
            racc[j / 4] |= static_cast<uint32_t>((lacc >> (SWAR_B * j)) & 3u) << (8 * (j % 4));
    }
    if (t < T) {
#pragma unroll
        for (int w = 0; w < NW; ++w) res[(s * T + t) * NW + w] = racc[w];
    }
}

// Register-blocked convolution: thread `tid` of a CTA owns the RB = 8
// consecutive output chunks t0 + 8 tid + r.  Step i needs qw[t - i] for its
// eight t, the step after shifts that window down by one, so eight steps
// read 15 window values (7 carried over) and one broadcast pw each: 64 FMAs
// per 8 + 8 shared loads.  The qw tile is stored with one pad double per 8
// (element j at j + j/8): lanes 8 apart in j land 9 doubles apart, 16 lanes
// per 128-byte wavefront -- conflict-free.
// A group closes every G = n_q rounded down to 8 products (n_q >= 8),
// checked per 8-step block.
constexpr int kRB = 8;
constexpr int kFqtOut = kFqtT * kRB;       // output chunks per CTA
constexpr int kQw = kFqtOut + kFqtI - 1;   // window values per i-tile
constexpr int kQwPad = kQw + kQw / 8 + 1;  // padded smem doubles

__device__ __forceinline__ int qpad(int j) { return j + (j >> 3); }

template <int ND, int W, class K>
__global__ void __launch_bounds__(kFqtT) fqt_conv_kernel(const FqtParams P, const double* __restrict__ pw,
                                                         uint64_t L1, const double* __restrict__ qw, uint64_t L2,
                                                         uint64_t T, uint64_t isplit, uint32_t* __restrict__ res) {
    constexpr int NW = (ND + 3) / 4;
    __shared__ double pws[kFqtI];
    __shared__ double qws[kQwPad];
    extern __shared__ __align__(16) uint32_t tab[];
    const int tid = threadIdx.x;
    if constexpr (W > 0)
        for (uint32_t i = tid; i < P.rq.n_entries; i += blockDim.x) tab[i] = P.rq.table[i];
    const K c{P.rq};
    const uint32_t tab_s = smem_addr(tab);

    const uint64_t t0 = uint64_t(blockIdx.x) * kFqtOut;
    const uint64_t s = blockIdx.y;
    // i with some t - i in [0, L2) for this tile, within split s
    // chunk s (isplit products long) of this tile's own i range (see the
    // step kernel)
    const uint64_t tlo = t0 + 1 > L2 ? t0 + 1 - L2 : 0, thi = std::min<uint64_t>(L1, t0 + kFqtOut);
    const uint64_t lo = tlo + s * isplit, hi = std::min<uint64_t>(thi, lo + isplit);
    double acc[kRB];
    uint32_t racc[kRB][NW];
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
        acc[r] = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) racc[r][w] = 0;
    }
    uint32_t cnt = 0;
    const uint32_t G = P.nq - P.nq % 8;
    auto close_groups = [&]() {
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
            uint32_t u[ND], mu[ND];
            redq_raw_digits<ND>(c, acc[r], u);
            redq_correct<ND, W>(c, u, mu, [&](uint32_t idx) { return lds_u32(tab_s + 4 * idx); });
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint32_t v = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (4 * w + j < ND) v |= mu[4 * w + j] << (8 * j);
                racc[r][w] = add_mod_lanes(racc[r][w], v, c.p());
            }
            acc[r] = 0.0;
        }
        cnt = 0;
    };
    for (uint64_t i0 = lo; i0 < hi; i0 += kFqtI) {
        const int n_i = static_cast<int>(std::min<uint64_t>(kFqtI, hi - i0));
        __syncthreads();
        // zero past n_i: the unrolled 8-step blocks may run past the tile end
        pws[tid] = tid < n_i ? pw[i0 + tid] : 0.0;
        // Q(j) = qw[t0 - i0 - (kFqtI-1) + j], stored at qpad(j)
        for (int j = tid; j < kQw; j += kFqtT) {
            const int64_t qi = static_cast<int64_t>(t0) - static_cast<int64_t>(i0) - (kFqtI - 1) + j;
            qws[qpad(j)] = (qi >= 0 && qi < static_cast<int64_t>(L2)) ? qw[qi] : 0.0;
        }
        __syncthreads();
        // step ii, output r: Q(8 tid + r + kFqtI - 1 - ii).  Block of 8 steps
        // from ii0: X[m] = Q(8 tid + kFqtI - 8 - ii0 + m), m = 0..14, step s
        // output r uses X[7 - s + r]
        // two 8-value load sets alternate as the window's lower half; the
        // other set's first 7 values are the upper half -- no register moves
        double XA[8], XC[8];
        const int jb = kRB * tid + kFqtI - 8;
#pragma unroll
        for (int m = 0; m < 7; ++m) XC[m] = qws[qpad(jb + 8 + m)];
        auto block = [&](int ii0, double (&lo8)[8], const double (&hi8)[8]) {
#pragma unroll
            for (int m = 0; m < 8; ++m) lo8[m] = qws[qpad(jb - ii0 + m)];
            double pv[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) pv[m] = pws[ii0 + m];
            // zero-padded pws makes steps past n_i add nothing
#pragma unroll
            for (int st = 0; st < 8; ++st)
#pragma unroll
                for (int r = 0; r < kRB; ++r) {
                    const int m = 7 - st + r;
                    acc[r] = fma(pv[st], m < 8 ? lo8[m] : hi8[m - 8], acc[r]);
                }
            cnt += 8;
            if (cnt >= G) close_groups();
        };
        // n_i <= 256, so ii0 + 8 <= 248 keeps every window index >= 0
        for (int ii0 = 0; ii0 < n_i; ii0 += 16) {
            block(ii0, XA, XC);
            block(ii0 + 8, XC, XA);
        }
    }
    if (cnt) close_groups();
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
        const uint64_t t = t0 + kRB * tid + r;
        if (t < T) {
#pragma unroll
            for (int w = 0; w < NW; ++w) res[(s * T + t) * NW + w] = racc[r][w];
        }
    }
}

// Overlap-add: chunk u of the output is residues 0..k-1 of product chunk u
// plus residues k..2k-2 of chunk u-1, each summed over the splits.  A CTA
// owns 256 chunks: every thread sums its chunk's split partials lane-wise
// mod p (one coalesced word per split and lane word), the sums meet in
// shared memory, and each thread writes its k coefficients.
__global__ void __launch_bounds__(256) fqt_overlap_kernel(uint32_t p, uint32_t k, uint32_t nd,
                                                          const uint32_t* __restrict__ res, uint32_t splits,
                                                          uint64_t T, uint8_t* __restrict__ out, uint64_t nout) {
    __shared__ uint32_t sums[257][4];
    const uint32_t nw = (nd + 3) / 4;
    const uint64_t nchunks = (nout + k - 1) / k;
    for (uint64_t u0 = uint64_t(blockIdx.x) * 256; u0 < nchunks; u0 += uint64_t(gridDim.x) * 256) {
        // slot 0 holds chunk u0-1, slot i+1 chunk u0+i
        for (int slot = threadIdx.x; slot < 257; slot += blockDim.x) {
            const int64_t u = static_cast<int64_t>(u0) - 1 + slot;
            uint32_t acc[4] = {0, 0, 0, 0};
            if (u >= 0 && static_cast<uint64_t>(u) < T) {
                for (uint32_t w = 0; w < nw; ++w) {
                    const uint32_t* src = res + static_cast<uint64_t>(u) * nw + w;
                    const uint64_t stride = T * nw;
                    uint32_t sp = 0;
                    for (; sp + 8 <= splits; sp += 8) {  // 8 independent loads in flight
                        uint32_t v[8];
#pragma unroll
                        for (int x = 0; x < 8; ++x) v[x] = __ldg(src + (sp + x) * stride);
#pragma unroll
                        for (int x = 0; x < 8; ++x) acc[w] = add_mod_lanes(acc[w], v[x], p);
                    }
                    for (; sp < splits; ++sp) acc[w] = add_mod_lanes(acc[w], __ldg(src + sp * stride), p);
                }
            }
            for (uint32_t w = 0; w < 4; ++w) sums[slot][w] = acc[w];
        }
        __syncthreads();
        const uint64_t u = u0 + threadIdx.x;
        if (u < nchunks) {
            for (uint32_t j = 0; j < k; ++j) {
                const uint64_t ci = u * k + j;
                if (ci >= nout) break;
                uint32_t v = (sums[threadIdx.x + 1][j / 4] >> (8 * (j % 4))) & 0xffu;
                const uint32_t jh = j + k;
                if (jh < nd) v += (sums[threadIdx.x][jh / 4] >> (8 * (jh % 4))) & 0xffu;
                out[ci] = static_cast<uint8_t>(v >= p ? v - p : v);
            }
        }
        __syncthreads();
    }
}

template <int ND, int W, class K>
cudaError_t run_conv_k(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                       uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((T + kFqtOut - 1) / kFqtOut), splits);
    const size_t smem = W > 0 ? size_t(P.rq.n_entries) * 4 : 0;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    static size_t cur = 0;
    if (smem > 24 * 1024 && smem > cur) {
        if (cudaError_t e = cudaFuncSetAttribute(fqt_conv_kernel<ND, W, K>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            e != cudaSuccess)
            return e;
        cur = smem;
    }
    fqt_conv_kernel<ND, W, K><<<grid, kFqtT, smem, s>>>(P, pw, L1, qw, L2, T, isplit, res);
    return cudaGetLastError();
}

template <int ND, int W, class K, int SWAR_B = 0>
cudaError_t run_conv_step(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((T + kFqtT - 1) / kFqtT), splits);
    const size_t smem = W > 0 ? size_t(P.rq.n_entries) * 4 : 0;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    static size_t cur = 0;
    if (smem > 48 * 1024 && smem > cur) {
        if (cudaError_t e = cudaFuncSetAttribute(fqt_conv_step_kernel<ND, W, K, SWAR_B>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            e != cudaSuccess)
            return e;
        cur = smem;
    }
    fqt_conv_step_kernel<ND, W, K, SWAR_B><<<grid, kFqtT, smem, s>>>(P, pw, L1, qw, L2, T, isplit, res);
    return cudaGetLastError();
}

template <int ND, int W>
cudaError_t run_conv_w(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                       uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    // the SWAR path needs every group word below 2^52 and within r_max
    const bool swar3 = P.rq.p == 3 && P.rq.qbits >= 4 && P.rq.qbits <= 7 && P.rq.qbits * ND <= 52 &&
                       P.rq.limit <= P.rq.r_max + 1.0;
    if (P.nq < 8 && swar3) {
        switch (P.rq.qbits) {
            case 4: return run_conv_step<ND, 0, RtConst<true>, 4>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
            case 5: return run_conv_step<ND, 0, RtConst<true>, 5>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
            case 6: return run_conv_step<ND, 0, RtConst<true>, 6>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
            default: return run_conv_step<ND, 0, RtConst<true>, 7>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
        }
    }
    if (P.nq < 8)
        return P.rq.qbits ? run_conv_step<ND, W, RtConst<true>>(P, pw, L1, qw, L2, T, splits, isplit, res, s)
                          : run_conv_step<ND, W, RtConst<false>>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
    return P.rq.qbits ? run_conv_k<ND, W, RtConst<true>>(P, pw, L1, qw, L2, T, splits, isplit, res, s)
                      : run_conv_k<ND, W, RtConst<false>>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
}

template <int ND>
cudaError_t run_conv(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2, uint64_t T,
                     uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    switch (P.rq.neg_q ? P.rq.window : 0) {
        case 2: return run_conv_w<ND, 2>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
        case 3: return run_conv_w<ND, 3>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
        case 4: return run_conv_w<ND, 4>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
        default: return run_conv_w<ND, 0>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
    }
}

}  // namespace

int num_sms();

namespace {
uint64_t fqt_chunks(uint64_t n, uint32_t k) { return (n + k - 1) / k; }
// Work split: tile `x` (tw output chunks) has its own i range of len(x)
// products; it is cut into chunks of C, so all CTAs but each tile's last
// carry the same work (the convolution's triangle would leave fixed global
// splits badly unbalanced).  C targets ~12 CTAs per SM; returns the chunk
// count of the longest tile (grid.y) and C.
struct FqtSplit {
    uint32_t splits;
    uint64_t chunk;
};
FqtSplit fqt_split(uint64_t L1, uint64_t L2, uint32_t nq) {
    const uint64_t tw = nq < 8 ? kFqtT : kFqtOut, T = L1 + L2 - 1, tiles = (T + tw - 1) / tw;
    uint64_t total = 0, longest = 0;
    for (uint64_t x = 0; x < tiles; ++x) {
        const uint64_t t0 = x * tw, lo = t0 + 1 > L2 ? t0 + 1 - L2 : 0, hi = std::min<uint64_t>(L1, t0 + tw);
        const uint64_t len = hi > lo ? hi - lo : 0;
        total += len;
        longest = std::max(longest, len);
    }
    const uint64_t target = uint64_t(num_sms()) * 12;
    uint64_t C = std::max<uint64_t>((total + target - 1) / target, 256);
    C = (C + 255) / 256 * 256;
    const uint64_t splits = std::max<uint64_t>((longest + C - 1) / C, 1);
    return {static_cast<uint32_t>(std::min<uint64_t>(splits, 1u << 16)), std::max(C, (longest + 65535) / 65536)};
}
uint64_t align16(uint64_t b) { return (b + 15) / 16 * 16; }
}  // namespace

uint64_t fqt_workspace_bytes(uint32_t k, uint32_t nq, uint64_t na, uint64_t nb) {
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    const uint32_t nd = 2 * k - 1, nw = (nd + 3) / 4;
    return align16(L1 * 8) + align16(L2 * 8) + uint64_t(fqt_split(L1, L2, nq).splits) * T * nw * 4;
}

cudaError_t launch_fqt_mul(const FqtParams& P, const uint8_t* a, uint64_t na, const uint8_t* b, uint64_t nb,
                           uint8_t* out, void* ws, cudaStream_t s) {
    if (na == 0 || nb == 0) return cudaSuccess;
    const uint32_t k = P.k, nd = 2 * k - 1;
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    auto* base = static_cast<uint8_t*>(ws);
    auto* pw = reinterpret_cast<double*>(base);
    auto* qw = reinterpret_cast<double*>(base + align16(L1 * 8));
    auto* res = reinterpret_cast<uint32_t*>(base + align16(L1 * 8) + align16(L2 * 8));
    const double qd = static_cast<double>(P.rq.q);
    const int sms = num_sms();
    fqt_pack_kernel<<<static_cast<int>(std::min<uint64_t>((L1 + 255) / 256, sms * 8)), 256, 0, s>>>(P.rq.p, k, qd, a,
                                                                                                      na, L1, pw);
    fqt_pack_kernel<<<static_cast<int>(std::min<uint64_t>((L2 + 255) / 256, sms * 8)), 256, 0, s>>>(P.rq.p, k, qd, b,
                                                                                                      nb, L2, qw);
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
    const FqtSplit sp = fqt_split(L1, L2, P.nq);
    const uint32_t splits = sp.splits;
    const uint64_t isplit = sp.chunk;
    cudaError_t e;
    switch (nd) {
        case 1: e = run_conv<1>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 3: e = run_conv<3>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 5: e = run_conv<5>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 7: e = run_conv<7>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 9: e = run_conv<9>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 11: e = run_conv<11>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 13: e = run_conv<13>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 15: e = run_conv<15>(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const uint64_t nout = na + nb - 1;
    const uint64_t nchunks = (nout + k - 1) / k;
    fqt_overlap_kernel<<<static_cast<int>(std::min<uint64_t>((nchunks + 255) / 256, sms * 8)), 256, 0, s>>>(
        P.rq.p, k, nd, res, splits, T, out, nout);
    return cudaGetLastError();
}

}  // namespace qpk
