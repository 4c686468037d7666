// K6 kernels and launch templates, included by fqt_conv.cu (host launch) and
// fqt_conv_inst.cu (one object per chunk width).  Chunked FQT product of two
// long polynomials over F_p (reference fqt_mul, polymul.cpp:81-147 = paper
// Sec. 5 d-FQT).
//
//  * pack: each operand is cut into chunks of k = d+1 coefficients and every
//    chunk packed into one q-adic word (fqt_encode, polymul.cpp:31-50), as an
//    exact double;
//  * product: output chunk t is sum_i pw[i] * qw[t-i] -- a 1-D convolution
//    of packed words, each fp64 product carrying a (d+1)x(d+1) block of
//    coefficient products.  Three kernels by group size: n_q >= 16 on the
//    fp64 tensor cores (fqt_mma_kernel, a block-Toeplitz GEMM per block
//    shift); 8 <= n_q < 16 register-blocked FFMA (fqt_conv_kernel: a CTA
//    sweeps i through shared-memory tiles, pw broadcast, qw sliding window,
//    2048 consecutive t, 8 per thread); n_q < 8 one t per thread
//    (fqt_conv_step_kernel, a REDQ after nearly every product); grid.y
//    splits the i (or block-shift) range.  Words beyond fp64 (m > 53) run
//    fqt_wide_conv_kernel in fqt_conv.cu;
//  * groups of at most n_q products are closed by REDQ (Alg. 2/3): the 2d+1
//    residues are added mod p into the thread's byte lanes, exactly as the
//    reference's per-group redq_residues_into + overlap-add;
//  * overlap-add: output coefficient c of chunk u is residue j of t = u plus
//    residue j+k of t = u-1, summed over the i splits, mod p.
// The result is the unique product mod p, so the grouping (which products
// share a REDQ) may differ from the reference's; the counters reported by
// the host are the reference's closed form.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

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
    pdl_wait();  // pw / qw come from the preceding pack launch

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
    pdl_wait();  // pw / qw come from the preceding pack launch

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

// fp64 tensor-core (DMMA) formulation for n_q >= 16: the convolution as a
// sum of small GEMMs.  With blocks of 16 chunk words, output t = 16a + s and
// input i = 16b + u,
//     out[16a + s] = sum_d sum_u Q_d[s][u] * P[u][a - d],
//     Q_d[s][u] = qw[16d + s - u],  P[u][b] = pw[16b + u],
// so for a fixed block shift d the 16 x (a-range) output tile is the GEMM
// Q_d (16 x 16, Toeplitz, the same for every column) times the columns
// a - d of P -- mma.sync m8n8k4 f64 (DMMA) with M = s, N = a, K = u.  Every
// output gains 16 products per d, so a group closes every floor(n_q/16)
// d-steps (16 * that <= n_q products: the REDQ bound of Eq. (2)).
// A warp owns 16 consecutive a-blocks (two 8-column tiles) x 16 s, a CTA
// four warps (1024 output chunks) and one range [d_lo, d_hi) of block
// shifts: CTAs tile the (a, d) plane, so no product is computed twice and
// only the triangle's edges (b = a - d outside the operand) multiply zeros.
// P is staged u-major (row stride == 4 mod 16 doubles: conflict-free B
// fragments), the Q window linearly (A fragments read 7 consecutive doubles
// per half-warp).
constexpr int kMmaBs = 16;                      // chunk words per block
constexpr int kMmaWarps = 4;
constexpr int kMmaA = kMmaWarps * 16;           // a-blocks per CTA
constexpr int kMmaOut = kMmaA * kMmaBs;         // output chunks per CTA
constexpr int kMmaCD = 128;                     // max block shifts per CTA
constexpr int kMmaCtasPerSm = 4;                // resident CTAs per SM (launch bounds)
constexpr int kMmaPLD = kMmaCD + kMmaA + 4;     // P row stride (== 4 mod 16)
constexpr int kMmaQW = kMmaBs * kMmaCD + 31;    // Q window doubles (incl. the prefetched shift)
static_assert(kMmaPLD % 16 == 4, "conflict-free B fragments");

// valid block shifts [dmin, dmax] of the DMMA kernel's tile x (empty when
// dmax < dmin) -- shared by the kernel, the host split and the overlap-add
__host__ __device__ __forceinline__ void fqt_mma_tile_shifts(uint64_t x, uint64_t L1, uint64_t L2, int64_t& dmin,
                                                             int64_t& dmax) {
    const int64_t A0 = int64_t(x) * kMmaA;
    const int64_t nb1 = int64_t((L1 + kMmaBs - 1) / kMmaBs), dq = int64_t((L2 + kMmaBs - 2) / kMmaBs);
    dmin = A0 - nb1 + 1 > 0 ? A0 - nb1 + 1 : 0;
    dmax = dq < A0 + kMmaA - 1 ? dq : A0 + kMmaA - 1;
}

__host__ __device__ __forceinline__ uint32_t fqt_mma_tile_splits(uint64_t x, uint64_t L1, uint64_t L2, uint64_t cd) {
    int64_t dmin, dmax;
    fqt_mma_tile_shifts(x, L1, L2, dmin, dmax);
    return dmax >= dmin ? static_cast<uint32_t>((uint64_t(dmax - dmin) + cd) / cd) : 0u;
}

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int ND, int W, class K, bool INT>
__global__ void __launch_bounds__(kMmaWarps * 32, kMmaCtasPerSm)
    fqt_mma_kernel(const FqtParams P, const double* __restrict__ pw, uint64_t L1, const double* __restrict__ qw,
                   uint64_t L2, uint64_t T, uint64_t cd, uint32_t* __restrict__ res) {
    constexpr int NW = (ND + 3) / 4;
    extern __shared__ __align__(16) uint8_t fq_smem[];
    double* Ps = reinterpret_cast<double*>(fq_smem);     // [16][kMmaPLD]
    double* Qs = Ps + kMmaBs * kMmaPLD;                  // [kMmaQW]
    uint32_t* tab = reinterpret_cast<uint32_t*>(Qs + kMmaQW);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, c4 = lane & 3;
    if constexpr (W > 0)
        for (uint32_t i = tid; i < P.rq.n_entries; i += blockDim.x) tab[i] = P.rq.table[i];
    const K c{P.rq};
    const uint32_t tab_s = smem_addr(tab);
    pdl_wait();  // pw / qw come from the preceding pack launch

    // this CTA: a-blocks [A0, A0 + kMmaA) x shifts [d_lo, d_hi) (range
    // blockIdx.y of the tile's valid shifts: b = a - d inside pw's blocks,
    // Q_d not all zero)
    const int64_t A0 = int64_t(blockIdx.x) * kMmaA;
    int64_t dmin, dmax;
    fqt_mma_tile_shifts(blockIdx.x, L1, L2, dmin, dmax);
    const int64_t d_lo = dmin + int64_t(blockIdx.y) * int64_t(cd);
    const int64_t d_hi = std::min<int64_t>(dmax + 1, d_lo + int64_t(cd));
    const int64_t nd = d_hi > d_lo ? d_hi - d_lo : 0;
    const int64_t Pbase = A0 - d_hi;            // P column 0 is block Pbase (one spare column for the prefetch)
    const int64_t qbase = kMmaBs * d_lo - 15;   // Qs[x] = qw[qbase + x]

    // a split past the tile's shift range has no work and writes nothing
    // (the overlap-add reads only fqt_mma_tile_splits partials per tile)
    if (nd == 0) return;
    {
        // consecutive threads read consecutive pw words (coalesced)
        const int cols = static_cast<int>(nd) + kMmaA;
        for (int x = tid; x < kMmaBs * cols; x += blockDim.x) {
            const int u = x % kMmaBs, col = x / kMmaBs;
            const int64_t i = (Pbase + col) * kMmaBs + u;
            Ps[u * kMmaPLD + col] = (i >= 0 && i < static_cast<int64_t>(L1)) ? pw[i] : 0.0;
        }
        const int nq_w = static_cast<int>(kMmaBs * nd + 31);
        for (int x = tid; x < nq_w; x += blockDim.x) {
            const int64_t qi = qbase + x;
            Qs[x] = (qi >= 0 && qi < static_cast<int64_t>(L2)) ? qw[qi] : 0.0;
        }
    }
    __syncthreads();

    // accumulators: two sets (k-steps 0,1 and 2,3) x 2 m-tiles x 2 n-tiles
    // INT: both accumulator sets start at 2^52 (integers in [2^52, 2^53) are
    // exact with ulp 1), so a group sum is the integer sum of two mantissas
    // and the close issues no fp64 instruction (the fp64 floor and the set
    // sum competed with the other warps' DMMAs for the fp64 pipe)
    constexpr double kB = INT ? kTwo52 : 0.0;
    double acc[2][2][2][2];
    uint32_t racc[8][NW];
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int w = 0; w < NW; ++w) racc[x][w] = 0;
    auto zero_acc = [&]() {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[a][m][j][0] = acc[a][m][j][1] = kB;
    };
    zero_acc();
    auto close_groups = [&]() {
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t u[ND], mu[ND];
                    if constexpr (INT) {
                        // floor(r/p) = mulhi(r, ceil(2^64/p)): exact for r < 2^53, p < 2^11
                        const uint64_t r = (dbits(acc[0][m][j][h]) & kMask52) + (dbits(acc[1][m][j][h]) & kMask52);
                        const uint64_t rop = __umul64hi(r, P.p_magic);
#pragma unroll
                        for (int i = 0; i < ND; ++i) {
                            const uint32_t sh = c.qbits() * i;
                            u[i] = static_cast<uint32_t>(r >> sh) - c.p() * static_cast<uint32_t>(rop >> sh);
                        }
                    } else {
                        const double r = acc[0][m][j][h] + acc[1][m][j][h];  // exact: integers < 2^53
                        redq_raw_digits<ND>(c, r, u);
                    }
                    redq_correct<ND, W>(c, u, mu, [&](uint32_t idx) { return lds_u32(tab_s + 4 * idx); });
                    const int x = (m * 2 + j) * 2 + h;
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        uint32_t v = 0;
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            if (4 * w + jj < ND) v |= mu[4 * w + jj] << (8 * jj);
                        racc[x][w] = add_mod_lanes(racc[x][w], v, c.p());
                    }
                }
        zero_acc();
    };

    const int64_t aw = A0 + 16 * warp;
    {
        const int64_t Gd = P.nq / kMmaBs;
        // lane pointers: A fragment (m, kt) at Qs[16(d - d_lo) + 8m + g - 4kt - c4 + 15],
        // B fragment (j, kt) at Ps[(4kt + c4) * LD + (aw + 8j + g - d - Pbase)]
        const double* q = Qs + (g - c4 + 15);
        const double* pp = Ps + c4 * kMmaPLD + (aw + g - d_lo - Pbase);
        double af[2][2][4], bf[2][2][4];  // two fragment sets: step d+1 loads while d multiplies
        auto load = [&](int st) {
#pragma unroll
            for (int kt = 0; kt < 4; ++kt) {
                af[st][0][kt] = q[-4 * kt];
                af[st][1][kt] = q[8 - 4 * kt];
                bf[st][0][kt] = pp[4 * kt * kMmaPLD];
                bf[st][1][kt] = pp[4 * kt * kMmaPLD + 8];
            }
            q += kMmaBs;
            --pp;
        };
        // k-steps in the order 0, 2, 1, 3: consecutive DMMAs alternate
        // accumulator sets, 8 issues between dependent ones
        auto mma = [&](int st) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int kt = (kk & 1) * 2 + (kk >> 1);
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        dmma_f64(acc[kt >> 1][m][j][0], acc[kt >> 1][m][j][1], af[st][m][kt], bf[st][j][kt]);
            }
        };
        // groups of Gd shifts (16 Gd <= n_q products per output), branch-free
        // inside; the window always holds one spare shift (Qs/Ps margins)
        load(0);
        for (int64_t dd = 0; dd < nd;) {
            const int64_t run = std::min<int64_t>(nd - dd, Gd);
            int64_t r = 0;
            for (; r + 2 <= run; r += 2) {
                load(1);
                mma(0);
                load(0);
                mma(1);
            }
            if (r < run) {
                load(1);
                mma(0);
#pragma unroll
                for (int kt = 0; kt < 4; ++kt)
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        af[0][m][kt] = af[1][m][kt];
                        bf[0][m][kt] = bf[1][m][kt];
                    }
            }
            dd += run;
            close_groups();
        }
    }
    // output chunk t = 16a + s: s = 8m + g, a = aw + 8j + 2 c4 + h
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t t = uint64_t(aw + 8 * j + 2 * c4 + h) * kMmaBs + 8 * m + g;
                if (t < T) {
                    const int x = (m * 2 + j) * 2 + h;
#pragma unroll
                    for (int w = 0; w < NW; ++w) res[(uint64_t(blockIdx.y) * T + t) * NW + w] = racc[x][w];
                }
            }
}

// the DMMA kernel serves n_q >= 16 (a d-step adds 16 products per output);
// QPK_FQT_FFMA=1 forces the register-blocked FFMA kernel (A/B measurement)
inline bool fqt_use_mma(uint32_t nq) {
    static const bool ffma = [] {
        const char* e = std::getenv("QPK_FQT_FFMA");
        return e && e[0] == '1';
    }();
    return nq >= uint32_t(kMmaBs) && !ffma;
}

template <int ND, int W, class K>
cudaError_t run_conv_k(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                       uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((T + kFqtOut - 1) / kFqtOut), splits);
    const size_t smem = W > 0 ? size_t(P.rq.n_entries) * 4 : 0;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fqt_conv_kernel<ND, W, K>), smem); e != cudaSuccess)
        return e;
    return launch_pdl(fqt_conv_kernel<ND, W, K>, grid, dim3(kFqtT), smem, s, P, pw, L1, qw, L2, T, isplit, res);
}

template <int ND, int W, class K, bool INT = false>
cudaError_t run_conv_mma(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                         uint64_t T, uint32_t splits, uint64_t cd, uint32_t* res, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((T + kMmaOut - 1) / kMmaOut), splits);
    const size_t smem = (size_t(kMmaBs) * kMmaPLD + kMmaQW) * 8 + (W > 0 ? size_t(P.rq.n_entries) * 4 : 0);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fqt_mma_kernel<ND, W, K, INT>), smem); e != cudaSuccess)
        return e;
    return launch_pdl(fqt_mma_kernel<ND, W, K, INT>, grid, dim3(kMmaWarps * 32), smem, s, P, pw, L1, qw, L2, T, cd, res);
}

template <int ND, int W, class K, int SWAR_B = 0>
cudaError_t run_conv_step(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((T + kFqtT - 1) / kFqtT), splits);
    const size_t smem = W > 0 ? size_t(P.rq.n_entries) * 4 : 0;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fqt_conv_step_kernel<ND, W, K, SWAR_B>), smem); e != cudaSuccess)
        return e;
    return launch_pdl(fqt_conv_step_kernel<ND, W, K, SWAR_B>, grid, dim3(kFqtT), smem, s, P, pw, L1, qw, L2, T, isplit,
                      res);
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
    if (fqt_use_mma(P.nq)) {
        if (P.rq.qbits)
            return P.mma_int ? run_conv_mma<ND, W, RtConst<true>, true>(P, pw, L1, qw, L2, T, splits, isplit, res, s)
                             : run_conv_mma<ND, W, RtConst<true>>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
        return run_conv_mma<ND, W, RtConst<false>>(P, pw, L1, qw, L2, T, splits, isplit, res, s);
    }
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

}  // namespace qpk
