// K5: GF(p^k) matrix-vector products and long dot products on dlog reps
// (reference fgdp_dot, gfq.cpp:335-387 = paper Alg. 4, with the GfqElt
// output of Theorem 3's L/H epilogue).
//
// y_i = sum_j A_ij x_j for A m x K and x of length K, all as u32 dlog reps
// (GfqMatrix / GfqElt data).  A is streamed once (4 bytes per element, the
// HBM bound); x is converted once to packed values (gemv_prep_x_kernel) and
// then re-read from L1/L2 by every row.
//
//  * tabulated pack: rep -> q-adic evaluation (float_table_, gfq.cpp:194-207).
//    When every packed value fits 32 bits (all benchmark fields), the table
//    holds u32 values, replicated once per lane for small fields (entry e of
//    lane l at word 32e + l: each warp lookup is one conflict-free
//    wavefront), and the products accumulate exactly in u64 (one IMAD.WIDE
//    per term); otherwise fp64 values and fma, as the reference;
//  * one warp owns a (row, K-split) task; each lane closes a group every
//    `chunk` <= n_q products as the reference does (gfq.cpp:346-385):
//    word -> REDQ digits -> low/high half tables -> coefficient bytes, added
//    mod p into the lane's sum; a 5-step shuffle adds the 32 lane sums;
//  * split partials are combined by the finish kernels, which also map the
//    coefficient vector to its rep through the log table.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "gfq_matmul.cuh"
#include "kernels.hpp"
#include "redq_core.cuh"

namespace qpk {

namespace {

constexpr int kGemvThreads = 256;
#ifndef QPK_GEMV_UNROLL
#define QPK_GEMV_UNROLL 4
#endif
constexpr int kGemvUnroll = QPK_GEMV_UNROLL;  // 16-byte loads of A in flight per lane
#ifndef QPK_GEMV_UNROLL_X
#define QPK_GEMV_UNROLL_X 4
#endif
constexpr int kGemvUnrollX = QPK_GEMV_UNROLL_X;  // ... of A and of x each, when x is streamed too (few rows)
constexpr uint32_t kReplMax = 64;  // replicate the value table up to this order (8 KB)
#ifndef QPK_XREP_ROWS
#define QPK_XREP_ROWS 4
#endif
constexpr uint64_t kXrepRows = QPK_XREP_ROWS;  // up to this many rows x is looked up per use

__device__ __forceinline__ uint4 ldg_stream(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// packed values and their accumulator: exact u64 products of u32 values, or
// fp64 fma (the reference's float path, for fields with values >= 2^32)
template <bool INT>
struct Acc;
template <>
struct Acc<true> {
    using V = uint32_t;
    using T = uint64_t;
    __device__ __forceinline__ static void mac(T& a, V x, V y) { a += static_cast<uint64_t>(x) * y; }
    __device__ __forceinline__ static double word(T a) { return __ull2double_rn(a); }  // exact: a < 2^53
    __device__ __forceinline__ static V from(double v) { return static_cast<uint32_t>(v); }
};
template <>
struct Acc<false> {
    using V = double;
    using T = double;
    __device__ __forceinline__ static void mac(T& a, V x, V y) { a = fma(x, y, a); }
    __device__ __forceinline__ static double word(T a) { return a; }
    __device__ __forceinline__ static V from(double v) { return v; }
};

// x reps -> packed values (V), once per call
template <bool INT>
__global__ void gemv_prep_x_kernel(const double* __restrict__ fval, uint32_t order, const uint32_t* __restrict__ x,
                                   uint64_t K, typename Acc<INT>::V* __restrict__ xv, uint32_t* status) {
    pdl_wait();
    uint32_t err = 0;
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < K; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t e = x[j];
        if (e >= order) err |= kErrRep;
        xv[j] = Acc<INT>::from(fval[min(e, order - 1)]);  // order - 1: the zero element
    }
    report_status(err, status);
}

// XREP: x read as reps and looked up per use (few rows: no reuse to pay for
// the conversion pass); else x as packed values from gemv_prep_x_kernel
template <int KR, class K, bool VEC, bool INT, bool REPL, bool XREP>
__global__ void __launch_bounds__(kGemvThreads) gfq_gemv_kernel(const GfqGemvParams P, const uint32_t* __restrict__ A,
                                                                const void* __restrict__ xptr, uint64_t m,
                                                                uint64_t Kd, uint32_t splits, uint64_t ksplit,
                                                                uint32_t* __restrict__ ws) {
    using AC = Acc<INT>;
    using V = typename AC::V;
    const V* xv = static_cast<const V*>(xptr);
    const uint32_t* xr = static_cast<const uint32_t*>(xptr);
    extern __shared__ __align__(128) uint8_t smem[];
    V* tv = reinterpret_cast<V*>(smem);
    const uint32_t nval = REPL ? P.order * 32 : P.order;
    uint32_t* tabs = reinterpret_cast<uint32_t*>(tv + nval);
    uint32_t nlh = 1;
#pragma unroll
    for (int i = 0; i < KR; ++i) nlh *= P.lh_radix;
    for (uint32_t i = threadIdx.x; i < nval; i += blockDim.x) tv[i] = AC::from(P.fval[REPL ? i >> 5 : i]);
    for (uint32_t i = threadIdx.x; i < 2 * nlh; i += blockDim.x) tabs[i] = P.lc[i];
    // PDL: the field tables above are constant; A and x follow the previous launch
    pdl_wait();
    __syncthreads();
    const uint32_t lc_s = smem_addr(tabs), hc_s = lc_s + 4 * nlh;

    const K c{P.rq};
    const int lane = threadIdx.x & 31;
    const V* tl = REPL ? tv + lane : tv;  // this lane's copy: entry e at tl[32 e]
    // reps >= order read as the zero element (order - 1, one min per
    // lookup) and latch kErrRep (a running max: 3-input max per vector pair)
    uint32_t emax = 0;
    const uint32_t elast = P.order - 1;
    auto val = [&](uint32_t e) -> V {
        e = min(e, elast);
        return REPL ? tl[e << 5] : tl[e];
    };
    auto seen = [&](const uint4& v) { emax = __vimax3_u32(__vimax3_u32(emax, v.x, v.y), v.z, v.w); };
    // CTA-uniform rounds of 8 tasks; with many splits (a multiple of 8) the
    // 8 tasks of a round are 8 consecutive splits of one row and the CTA adds
    // them before writing one partial (slot split/8)
    __shared__ uint32_t red[kGemvThreads / 32];
    const bool cta_red = splits >= 64 && splits % 8 == 0;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t tasks = m * splits;
    for (uint64_t base = uint64_t(blockIdx.x) * 8; base < tasks; base += uint64_t(gridDim.x) * 8) {
        const uint64_t t = base + warp;
        const uint64_t row = t / splits, s = t % splits;
        uint32_t cf = 0;
        if (t < tasks) {
            const uint64_t k0 = s * ksplit, k1 = std::min<uint64_t>(Kd, k0 + ksplit);
            const uint32_t* arow = A + row * Kd;
            typename AC::T acc = 0;
            uint32_t cnt = 0, csum = 0;
            auto close_group = [&]() {
                csum = add_mod_bytes_mm(csum, acc_to_coeffs<KR>(c, P.lh_radix, AC::word(acc), lc_s, hc_s), P.p);
                acc = 0;
                cnt = 0;
            };
            // XREP: b = the x vector of the same position, streamed like A
            auto four = [&](const uint4& a, uint64_t j, const uint4& b) {
                V xs[4];
                if constexpr (XREP) {
                    seen(b);
                    xs[0] = val(b.x), xs[1] = val(b.y), xs[2] = val(b.z), xs[3] = val(b.w);
                } else if constexpr (INT) {
                    const V* xq = xv + j;
                    const uint4 b = __ldg(reinterpret_cast<const uint4*>(xq));
                    xs[0] = b.x, xs[1] = b.y, xs[2] = b.z, xs[3] = b.w;
                } else {
                    const V* xq = xv + j;
                    const double2 b0 = __ldg(reinterpret_cast<const double2*>(xq));
                    const double2 b1 = __ldg(reinterpret_cast<const double2*>(xq) + 1);
                    xs[0] = b0.x, xs[1] = b0.y, xs[2] = b1.x, xs[3] = b1.y;
                }
                seen(a);
                AC::mac(acc, val(a.x), xs[0]);
                AC::mac(acc, val(a.y), xs[1]);
                AC::mac(acc, val(a.z), xs[2]);
                AC::mac(acc, val(a.w), xs[3]);
                if (P.chunk) {
                    cnt += 4;
                    if (cnt >= P.chunk) close_group();
                }
            };
            if constexpr (VEC) {
                constexpr int U = XREP ? kGemvUnrollX : kGemvUnroll;
                // k0 and Kd are multiples of 4: every 16-byte vector is whole.
                // Software pipelined: the next U vectors of A are in
                // flight while the current ones are multiplied.
                constexpr uint64_t kStep = 128 * U;
                uint64_t j = k0 + 4 * lane;
                // (few rows: x is streamed too, one step ahead like A -- loaded at
                // its use, every step waited a full DRAM round trip for it)
                constexpr int XU = XREP ? U : 1;
                const uint4 none = make_uint4(0, 0, 0, 0);
                if (j + kStep - 128 < k1) {
                    uint4 cur[U], xcur[XU];
#pragma unroll
                    for (int u = 0; u < U; ++u) cur[u] = ldg_stream(arow + j + 128 * u);
                    if constexpr (XREP) {
#pragma unroll
                        for (int u = 0; u < U; ++u) xcur[u] = ldg_stream(xr + j + 128 * u);
                    }
                    for (; j + 2 * kStep - 128 < k1; j += kStep) {
                        uint4 nxt[U], xnxt[XU];
#pragma unroll
                        for (int u = 0; u < U; ++u) nxt[u] = ldg_stream(arow + j + kStep + 128 * u);
                        if constexpr (XREP) {
#pragma unroll
                            for (int u = 0; u < U; ++u) xnxt[u] = ldg_stream(xr + j + kStep + 128 * u);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) four(cur[u], j + 128 * u, XREP ? xcur[u] : none);
#pragma unroll
                        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
                        if constexpr (XREP) {
#pragma unroll
                            for (int u = 0; u < U; ++u) xcur[u] = xnxt[u];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) four(cur[u], j + 128 * u, XREP ? xcur[u] : none);
                    j += kStep;
                }
                for (; j < k1; j += 128) four(ldg_stream(arow + j), j, XREP ? ldg_stream(xr + j) : none);
            } else {
                for (uint64_t j = k0 + lane; j < k1; j += 32) {
                    emax = max(emax, arow[j]);
                    if constexpr (XREP) emax = max(emax, xr[j]);
                    AC::mac(acc, val(arow[j]), XREP ? val(xr[j]) : xv[j]);
                    if (P.chunk && ++cnt >= P.chunk) close_group();
                }
            }
            cf = add_mod_bytes_mm(csum, acc_to_coeffs<KR>(c, P.lh_radix, AC::word(acc), lc_s, hc_s), P.p);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1)
                cf = add_mod_bytes_mm(cf, __shfl_xor_sync(0xffffffffu, cf, off), P.p);
        }
        if (cta_red) {
            if (lane == 0) red[warp] = cf;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t v = red[0];
#pragma unroll
                for (int w = 1; w < kGemvThreads / 32; ++w) v = add_mod_bytes_mm(v, red[w], P.p);
                ws[(base % splits) / 8 * m + base / splits] = v;
            }
            __syncthreads();
        } else if (t < tasks && lane == 0) {
            ws[s * m + row] = cf;
        }
    }
    report_status(emax > elast ? kErrRep : 0u, P.status);
}

__device__ __forceinline__ void gemv_emit(uint32_t p, uint32_t k, const uint32_t* log, uint64_t row, uint32_t cf,
                                          uint32_t* out_rep, uint8_t* out_coeff) {
    if (out_coeff)
        for (uint32_t t = 0; t < k; ++t) out_coeff[row * k + t] = static_cast<uint8_t>(cf >> (8 * t));
    if (out_rep) {
        uint32_t idx = 0;
        for (int t = static_cast<int>(k) - 1; t >= 0; --t) idx = idx * p + ((cf >> (8 * t)) & 0xffu);
        out_rep[row] = log[idx];
    }
}

// few splits: one thread per row sums them
__global__ void gemv_finish_rows_kernel(uint32_t p, uint32_t k, const uint32_t* __restrict__ log,
                                        const uint32_t* __restrict__ ws, uint64_t m, uint32_t splits,
                                        uint32_t* __restrict__ out_rep, uint8_t* __restrict__ out_coeff) {
    pdl_wait();
    for (uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < m;
         row += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t cf = ws[row];
        for (uint32_t s = 1; s < splits; ++s) cf = add_mod_bytes_mm(cf, ws[s * m + row], p);
        gemv_emit(p, k, log, row, cf, out_rep, out_coeff);
    }
}

// many splits (long dot products): one CTA per row reduces them
__global__ void __launch_bounds__(256) gemv_finish_cta_kernel(uint32_t p, uint32_t k, const uint32_t* __restrict__ log,
                                                              const uint32_t* __restrict__ ws, uint64_t m,
                                                              uint32_t splits, uint32_t* __restrict__ out_rep,
                                                              uint8_t* __restrict__ out_coeff) {
    __shared__ uint32_t part[8];
    pdl_wait();
    for (uint64_t row = blockIdx.x; row < m; row += gridDim.x) {
        uint32_t cf = 0;
        for (uint32_t s = threadIdx.x; s < splits; s += blockDim.x) cf = add_mod_bytes_mm(cf, ws[s * m + row], p);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) cf = add_mod_bytes_mm(cf, __shfl_xor_sync(0xffffffffu, cf, off), p);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cf;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) cf = add_mod_bytes_mm(cf, part[w], p);
            gemv_emit(p, k, log, row, cf, out_rep, out_coeff);
        }
        __syncthreads();
    }
}

template <int KR, class K, bool INT, bool REPL, bool XREP>
cudaError_t run_gemv_v(const GfqGemvParams& P, const uint32_t* A, const void* xv, uint64_t m, uint64_t Kd,
                       uint32_t splits, uint64_t ksplit, uint32_t* ws, int grid, cudaStream_t s) {
    using V = typename Acc<INT>::V;
    (void)m;
    uint32_t nlh = 1;
    for (int i = 0; i < KR; ++i) nlh *= P.lh_radix;
    const size_t smem = size_t(REPL ? P.order * 32 : P.order) * sizeof(V) + size_t(2 * nlh) * 4;
    if (smem > 226 * 1024) return cudaErrorInvalidValue;  // + the static reduction slots
    const bool vec = Kd % 4 == 0 && ksplit % 128 == 0 && P.chunk % 4 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(xv) % 16 == 0;
    if (vec) {
        if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(gfq_gemv_kernel<KR, K, true, INT, REPL, XREP>), smem); e != cudaSuccess)
            return e;
        return launch_pdl(gfq_gemv_kernel<KR, K, true, INT, REPL, XREP>, dim3(grid), dim3(kGemvThreads), smem, s, P,
                          A, xv, m, Kd, splits, ksplit, ws);
    } else {
        if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(gfq_gemv_kernel<KR, K, false, INT, REPL, XREP>), smem); e != cudaSuccess)
            return e;
        return launch_pdl(gfq_gemv_kernel<KR, K, false, INT, REPL, XREP>, dim3(grid), dim3(kGemvThreads), smem, s, P,
                          A, xv, m, Kd, splits, ksplit, ws);
    }
}

template <int KR, class K>
cudaError_t run_gemv_t(const GfqGemvParams& P, const uint32_t* A, const void* xv, uint64_t m, uint64_t Kd,
                       uint32_t splits, uint64_t ksplit, uint32_t* ws, int grid, cudaStream_t s) {
    const bool xrep = m <= kXrepRows;
    if (!P.vals32)
        return xrep ? run_gemv_v<KR, K, false, false, true>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s)
                    : run_gemv_v<KR, K, false, false, false>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
    if (P.order <= kReplMax)
        return xrep ? run_gemv_v<KR, K, true, true, true>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s)
                    : run_gemv_v<KR, K, true, true, false>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
    return xrep ? run_gemv_v<KR, K, true, false, true>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s)
                : run_gemv_v<KR, K, true, false, false>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
}

template <int KR>
cudaError_t run_gemv(const GfqGemvParams& P, const uint32_t* A, const void* xv, uint64_t m, uint64_t Kd,
                     uint32_t splits, uint64_t ksplit, uint32_t* ws, int grid, cudaStream_t s) {
    // compile-time fast paths for the benchmark fields (C4 GF(3^2) at 2^16,
    // C5 GF(3^3) at 2^10); runtime parameters otherwise
    if constexpr (KR == 2) {
        if (P.p == 3 && P.rq.qbits == 16 && mm_plan_safe(P.rq))
            return run_gemv_t<2, CtConst<3, 16>>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
    }
    if constexpr (KR == 3) {
        if (P.p == 3 && P.rq.qbits == 10 && mm_plan_safe(P.rq))
            return run_gemv_t<3, CtConst<3, 10>>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
    }
    return P.rq.qbits ? run_gemv_t<KR, RtConst<true>>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s)
                      : run_gemv_t<KR, RtConst<false>>(P, A, xv, m, Kd, splits, ksplit, ws, grid, s);
}

}  // namespace

int num_sms();

uint32_t gemv_splits(uint64_t m, uint64_t Kd) {
    // Measured on B200 (scripts/gemv_sweep*.py, 2^26-element shapes): a round
    // of tasks just above the resident warp count W (4 CTAs x 8 warps per
    // SM) costs a second round, so either every task fits one round (few
    // rows: long tasks) or there are ~7 rounds (many rows: the tail is
    // small); tasks stay >= 2048 elements.
    const uint64_t W = uint64_t(num_sms()) * 32;
    const uint64_t cap = std::max<uint64_t>(Kd / 2048, 1);
    uint64_t s = m <= W / 2 ? std::max<uint64_t>(W * 9 / 10 / m, 1) : (7 * W + m - 1) / m;
    s = std::min(s, cap);
    if (s >= 64) s = s / 8 * 8;  // the kernel adds the 8 splits of a CTA round
    return static_cast<uint32_t>(std::clamp<uint64_t>(s, 1, 1u << 20));
}

uint64_t gemv_workspace_bytes(uint64_t m, uint64_t Kd, uint32_t splits) {
    return (Kd * 8 + 15) / 16 * 16 + uint64_t(splits) * m * 4;
}

cudaError_t launch_gfq_gemv(const GfqGemvParams& P, const uint32_t* A, const uint32_t* x, uint64_t m, uint64_t Kd,
                            uint32_t splits, void* ws, uint32_t* out_rep, uint8_t* out_coeff, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    if (splits == 0) splits = 1;
    auto* xv = static_cast<uint8_t*>(ws);
    auto* part = reinterpret_cast<uint32_t*>(xv + (Kd * 8 + 15) / 16 * 16);
    const bool xrep = m <= kXrepRows;
    if (Kd && !xrep) {
        const int g = static_cast<int>(std::min<uint64_t>((Kd + 255) / 256, uint64_t(num_sms()) * 8));
        const cudaError_t e =
            P.vals32 ? launch_pdl(gemv_prep_x_kernel<true>, dim3(g), dim3(256), 0, s, P.fval, P.order, x, Kd,
                                  reinterpret_cast<uint32_t*>(xv), P.status)
                     : launch_pdl(gemv_prep_x_kernel<false>, dim3(g), dim3(256), 0, s, P.fval, P.order, x, Kd,
                                  reinterpret_cast<double*>(xv), P.status);
        if (e != cudaSuccess) return e;
    }
    // split length: a multiple of 128 (one warp-wide 16-byte vector row)
    uint64_t ksplit = (Kd + splits - 1) / splits;
    ksplit = std::max<uint64_t>((ksplit + 127) / 128 * 128, 128);
    const uint64_t tasks = m * splits;
    const int grid = static_cast<int>(std::min<uint64_t>((tasks + 7) / 8, uint64_t(num_sms()) * 8));
    const void* xa = xrep ? static_cast<const void*>(x) : xv;
    cudaError_t e;
    switch (P.k) {
        case 1: e = run_gemv<1>(P, A, xa, m, Kd, splits, ksplit, part, grid, s); break;
        case 2: e = run_gemv<2>(P, A, xa, m, Kd, splits, ksplit, part, grid, s); break;
        case 3: e = run_gemv<3>(P, A, xa, m, Kd, splits, ksplit, part, grid, s); break;
        case 4: e = run_gemv<4>(P, A, xa, m, Kd, splits, ksplit, part, grid, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const uint32_t parts = splits >= 64 && splits % 8 == 0 ? splits / 8 : splits;  // the kernel's CTA reduction
    if (parts >= 64) {
        const int fgrid = static_cast<int>(std::min<uint64_t>(m, uint64_t(num_sms()) * 8));
        return launch_pdl(gemv_finish_cta_kernel, dim3(fgrid), dim3(256), 0, s, P.p, P.k, P.log,
                          static_cast<const uint32_t*>(part), m, parts, out_rep, out_coeff);
    }
    const int fgrid = static_cast<int>(std::min<uint64_t>((m + 255) / 256, uint64_t(num_sms()) * 4));
    return launch_pdl(gemv_finish_rows_kernel, dim3(fgrid), dim3(256), 0, s, P.p, P.k, P.log,
                      static_cast<const uint32_t*>(part), m, parts, out_rep, out_coeff);
}

}  // namespace qpk
