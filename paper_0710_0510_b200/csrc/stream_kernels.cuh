// HBM-streaming kernels of the q-adic pipeline on sm_100a:
//
//   K2  batched REDQ / FQT-inverse      fp64 words -> d+1 residues (uint8)
//   C1  fused DQT pack + fp64 product + REDQ (batched small polymul)
//   K3  GF(p^k) elementwise product, DQT/REDQ/L-H path or dlog/Zech path
//
// All three share one persistent TMA pipeline (stream_tma_kernel): a CTA
// owns tiles of THREADS*R records; one elected thread moves each input tile
// global->shared with cp.async.bulk (completion on an mbarrier, STAGES deep)
// and each finished output tile shared->global with a bulk store, so every
// HBM transfer is a long contiguous burst regardless of the awkward 7- or
// 3-byte record sizes.  Threads only touch shared memory, each one a run of R
// consecutive records, and all lookup tables (REDQ correction windows, L/H
// half tables, log/antilog) are staged in shared memory per CTA.
//
// (templates only: instantiated per digit count / record width in
// stream_inst.cu, compiled once per -DQPK_INST value so nvcc runs in parallel)
//
// Records that do not fill a whole tile, or buffers that are not 16-byte
// aligned, go through stream_tail_kernel (plain byte loads, same op).

#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

namespace {

constexpr uint64_t kMask52 = (uint64_t(1) << 52) - 1;

// ------------------------------------------------------------------ REDQ core
// Raw REDQ digits of one word (redq.cpp:31-59): rop = floor(r/p) with one
// premultiplied fp64 floor, u_i = floor(r/q^i) - p*floor(rop/q^i).  Every
// u_i is in [0, p-1] (paper Theorem 2), so it is formed in wrapping 32-bit
// arithmetic from the low 32 bits of the two shifted quotients.
//
// `w` follows packed_from_double (dqt.cpp:96-100): truncated toward zero,
// rejected when negative, NaN or not below min(q^(d+1), 2^53) (the latter is
// check_input, redq.cpp:22-29).
template <int ND, bool POW2>
__device__ __forceinline__ void redq_digits(const RedqParams& P, double w, uint32_t (&u)[ND], uint32_t& err) {
    double r = trunc(w);
    if (!(w >= 0.0 && r < P.limit)) {
        err |= kErrDomain;
        r = 0.0;
    }
    const bool premul = r <= P.r_max;
    const uint64_t rb = r < kTwo52 ? (dbits(r + kTwo52) & kMask52) : __double2ull_rz(r);
    const uint64_t rop = premul ? floor_div_premul(r, P.inv_p) : rb / P.p;
    if constexpr (POW2) {
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            const uint32_t sh = P.qbits * i;
            u[i] = static_cast<uint32_t>(rb >> sh) - P.p * static_cast<uint32_t>(rop >> sh);
        }
    } else {
        const double ropd = static_cast<double>(rop);
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            uint64_t x, y;
            if (premul) {
                x = floor_div_premul(r, P.inv_q[i]);
                y = floor_div_premul(ropd, P.inv_q[i]);
            } else {
                x = rb / P.qpow[i];
                y = rop / P.qpow[i];
            }
            u[i] = static_cast<uint32_t>(x) - P.p * static_cast<uint32_t>(y);
        }
    }
}

// (u_i + neg_q * u_{i+1}) mod p for t < 2^16, p <= 256: floor(t/p) from a
// 32-bit multiply-high by ceil(2^32/p) is exact in that range.
__device__ __forceinline__ uint32_t mod_small(uint32_t t, uint32_t p, uint32_t magic) {
    return t - p * __umulhi(t, magic);
}

// Correction mu from u (redq.cpp:61-100).  W = 0: direct formula (or the
// identity when p | q); W = 2..4: the windowed table of Alg. 3, windows of
// W digits starting at a*(W-1), zero padded past the top digit, a window's
// last slot kept only at the top digit.  The device table stores each
// window's residues one per byte so decoding is a byte extract.
template <int ND, int W>
__device__ __forceinline__ void redq_correct(const RedqParams& P, const uint32_t (&u)[ND], uint32_t (&mu)[ND],
                                             const uint32_t* tab) {
    constexpr int D = ND - 1;
    if constexpr (W == 0 || D == 0) {
        if (W == 0 && D > 0 && P.neg_q != 0) {
#pragma unroll
            for (int i = 0; i < D; ++i) mu[i] = mod_small(u[i] + P.neg_q * u[i + 1], P.p, P.mod_magic);
            mu[D] = u[D];
        } else {
#pragma unroll
            for (int i = 0; i < ND; ++i) mu[i] = u[i];
        }
    } else {
        constexpr int A = (D + W - 2) / (W - 1);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int s = a * (W - 1);
            uint32_t idx = 0;
#pragma unroll
            for (int j = W - 1; j >= 0; --j) idx = idx * P.radix + (s + j <= D ? u[s + j] : 0u);
            const uint32_t e = tab[idx];
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (s + j <= D && (j + 1 < W || s + j == D)) mu[s + j] = byte_of(e, j);
        }
    }
}

// --------------------------------------------------------------------- ops
// An op maps R consecutive records (IN0 + IN1 bytes each, given as packed
// little-endian u32 words) to R output records of OUT bytes.

template <int ND, bool POW2, int W>
struct RedqOp {
    static constexpr int IN0 = 8, IN1 = 0, OUT = ND, R = 4;
    RedqParams P;
    __host__ __device__ uint32_t tables_words() const { return W ? P.n_entries : 0u; }
    __host__ __device__ const uint32_t* tables_src() const { return P.table; }
    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t*, uint8_t (&o)[R * OUT],
                                          const uint32_t* tab, uint32_t& err) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double w = __hiloint2double(static_cast<int>(a[2 * r + 1]), static_cast<int>(a[2 * r]));
            uint32_t u[ND], mu[ND];
            redq_digits<ND, POW2>(P, w, u, err);
            redq_correct<ND, W>(P, u, mu, tab);
#pragma unroll
            for (int j = 0; j < ND; ++j) o[r * OUT + j] = static_cast<uint8_t>(mu[j]);
        }
    }
};

// byte `i` of a run of packed u32 words
__device__ __forceinline__ uint32_t run_byte(const uint32_t* w, int i) { return byte_of(w[i >> 2], i & 3); }

template <int K, bool POW2, int W>
struct PolymulOp {
    static constexpr int ND = 2 * K - 1;
    static constexpr int IN0 = K, IN1 = K, OUT = ND, R = 4;
    PolymulParams P;
    __host__ __device__ uint32_t tables_words() const { return W ? P.rq.n_entries : 0u; }
    __host__ __device__ const uint32_t* tables_src() const { return P.rq.table; }

    // DQT pack (dqt.cpp:23-37) of one record, coefficients reduced mod p first
    // as DensePoly's constructor does (poly.hpp:19-21)
    __device__ __forceinline__ double pack(const uint32_t* w, int rec) const {
        const RedqParams& Q = P.rq;
        uint64_t v = 0;
        double vd = 0.0;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            const uint32_t c = mod_small(run_byte(w, rec * K + i), Q.p, Q.mod_magic);
            if constexpr (POW2)
                v = (v << Q.qbits) | c;
            else
                vd = fma(vd, static_cast<double>(Q.q), static_cast<double>(c));
        }
        return POW2 ? static_cast<double>(v) : vd;
    }

    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t* b, uint8_t (&o)[R * OUT],
                                          const uint32_t* tab, uint32_t& err) const {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double prod = pack(a, r) * pack(b, r);  // exact: q^(2k-1) < 2^53
            uint32_t u[ND], mu[ND];
            redq_digits<ND, POW2>(P.rq, prod, u, err);
            redq_correct<ND, W>(P.rq, u, mu, tab);
#pragma unroll
            for (int j = 0; j < ND; ++j) o[r * OUT + j] = static_cast<uint8_t>(mu[j]);
        }
    }
};

// bytewise (x + y) mod p for packed coefficient bytes, each < p
__device__ __forceinline__ uint32_t add_mod_bytes(uint32_t x, uint32_t y, uint32_t p, uint32_t k) {
    if (p < 128) {
        const uint32_t pp = p * 0x01010101u;
        const uint32_t s = __vadd4(x, y);
        return __vsub4(s, __vcmpgeu4(s, pp) & pp);
    }
    uint32_t r = 0;
    for (uint32_t i = 0; i < k; ++i) {
        uint32_t t = byte_of(x, i) + byte_of(y, i);
        if (t >= p) t -= p;
        r |= t << (8 * i);
    }
    return r;
}

template <int K, bool POW2>
struct GfqElemOp {
    static constexpr int ND = 2 * K - 1;
    static constexpr int IN0 = K, IN1 = K, OUT = K, R = 4;
    GfqElemParams P;
    __host__ __device__ uint32_t tables_words() const { return P.tables_words; }
    __host__ __device__ const uint32_t* tables_src() const { return P.lc; }  // lc|hc|log|alog contiguous

    __device__ __forceinline__ void apply(const uint32_t* a, const uint32_t* b, uint8_t (&o)[R * OUT],
                                          const uint32_t* tab, uint32_t& err) const {
        const uint32_t p = P.p, magic = P.rq.mod_magic;
        uint32_t nlh = 1;
#pragma unroll
        for (int i = 0; i < K; ++i) nlh *= P.lh_radix;
        const uint32_t* lc = tab;
        const uint32_t* hc = tab + nlh;
        const uint32_t* lg = tab + 2 * nlh;
        const uint32_t* al = tab + 2 * nlh + P.order;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t ca[K], cb[K];
#pragma unroll
            for (int i = 0; i < K; ++i) {
                ca[i] = mod_small(run_byte(a, r * K + i), p, magic);
                cb[i] = mod_small(run_byte(b, r * K + i), p, magic);
            }
            uint32_t res;
            if (P.mode == 0) {
                // paper Alg. 4 with one term: pack, fp64 product, REDQ digits,
                // low/high half tables (gfq.cpp:353-381) -- here the tables give
                // coefficient vectors and the two halves add coefficient-wise
                double va = 0.0, vb = 0.0;
                if constexpr (POW2) {
                    uint64_t ia = 0, ib = 0;
#pragma unroll
                    for (int i = K - 1; i >= 0; --i) {
                        ia = (ia << P.rq.qbits) | ca[i];
                        ib = (ib << P.rq.qbits) | cb[i];
                    }
                    va = static_cast<double>(ia);
                    vb = static_cast<double>(ib);
                } else {
#pragma unroll
                    for (int i = K - 1; i >= 0; --i) {
                        va = fma(va, P.qd, static_cast<double>(ca[i]));
                        vb = fma(vb, P.qd, static_cast<double>(cb[i]));
                    }
                }
                uint32_t u[ND];
                redq_digits<ND, POW2>(P.rq, va * vb, u, err);
                uint32_t il = 0, ih = 0;
#pragma unroll
                for (int i = K - 1; i >= 0; --i) {
                    il = il * P.lh_radix + u[i];
                    ih = ih * P.lh_radix + u[K - 1 + i];
                }
                res = add_mod_bytes(lc[il], hc[ih], p, K);
            } else {
                // dlog representation: rep(a*b) = rep(a) + rep(b) mod p^k-1 with
                // the zero sentinel (gfq.cpp:260-264), then back to coefficients
                uint32_t ia = 0, ib = 0;
#pragma unroll
                for (int i = K - 1; i >= 0; --i) {
                    ia = ia * p + ca[i];
                    ib = ib * p + cb[i];
                }
                const uint32_t ra = lg[ia], rb = lg[ib];
                uint32_t rc = ra + rb;
                if (rc >= P.group) rc -= P.group;
                if (ra == P.group || rb == P.group) rc = P.group;
                res = al[rc];
            }
#pragma unroll
            for (int j = 0; j < K; ++j) o[r * OUT + j] = static_cast<uint8_t>(byte_of(res, j));
        }
    }
};

// ------------------------------------------------------------- the pipeline
constexpr int kThreads = 256;
constexpr int kStages = 4;
constexpr int kOutStages = 2;

template <class Op>
struct Geometry {
    static constexpr int R = Op::R;
    static constexpr int TILE = kThreads * R;  // records per tile
    static constexpr uint32_t B0 = Op::IN0 * TILE, B1 = Op::IN1 * TILE, BO = Op::OUT * TILE;
    static constexpr int W0 = R * Op::IN0 / 4, W1 = R * Op::IN1 / 4, WO = R * Op::OUT / 4;
    static_assert((R * Op::IN0) % 4 == 0 && (R * Op::IN1) % 4 == 0 && (R * Op::OUT) % 4 == 0, "u32 runs");
    static_assert(B0 % 16 == 0 && B1 % 16 == 0 && BO % 16 == 0, "bulk copies move multiples of 16 bytes");
    static constexpr size_t smem_fixed = size_t(kStages) * (B0 + B1) + size_t(kOutStages) * BO + kStages * 8;
};

// load `N` u32 words at smem+off with the widest conflict-light vector
template <int N>
__device__ __forceinline__ void lds_run(const uint8_t* base, uint32_t (&w)[N > 0 ? N : 1]) {
    if constexpr (N == 0) {
        w[0] = 0;
    } else if constexpr (N % 4 == 0) {
#pragma unroll
        for (int i = 0; i < N / 4; ++i) {
            const uint4 v = reinterpret_cast<const uint4*>(base)[i];
            w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = reinterpret_cast<const uint32_t*>(base)[i];
    }
}

template <int N>
__device__ __forceinline__ void pack_out(const uint8_t (&o)[4 * N], uint32_t (&w)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i)
        w[i] = uint32_t(o[4 * i]) | (uint32_t(o[4 * i + 1]) << 8) | (uint32_t(o[4 * i + 2]) << 16) |
               (uint32_t(o[4 * i + 3]) << 24);
}

__device__ __forceinline__ void report(uint32_t err, uint32_t* status) {
    err = __reduce_or_sync(0xffffffffu, err);
    if (err && (threadIdx.x & 31) == 0 && status) atomicOr(status, err);
}

template <class Op>
__device__ __forceinline__ void stage_tables(const Op& op, uint32_t* dst) {
    const uint32_t nt = op.tables_words();
    const uint32_t* src = op.tables_src();
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) dst[i] = src[i];
}

template <class Op>
__global__ void __launch_bounds__(kThreads) stream_tma_kernel(const Op op, const uint8_t* __restrict__ in0,
                                                              const uint8_t* __restrict__ in1,
                                                              uint8_t* __restrict__ out, uint64_t n_tiles,
                                                              uint32_t* status) {
    using G = Geometry<Op>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* s_in = smem;
    uint8_t* s_out = smem + size_t(kStages) * (G::B0 + G::B1);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_out + size_t(kOutStages) * G::BO);
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(bars + kStages);
    const int tid = threadIdx.x;

    stage_tables(op, s_tab);
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    uint64_t policy = 0;
    auto issue = [&](int s, uint64_t tile) {
        uint8_t* dst = s_in + size_t(s) * (G::B0 + G::B1);
        mbar_expect_tx(&bars[s], G::B0 + G::B1);
        bulk_g2s_stream(dst, in0 + tile * G::B0, G::B0, &bars[s], policy);
        if constexpr (G::B1 > 0) bulk_g2s_stream(dst + G::B0, in1 + tile * G::B1, G::B1, &bars[s], policy);
    };
    if (tid == 0) {
        policy = policy_evict_first();
        for (int s = 0; s < kStages; ++s) {
            const uint64_t t = blockIdx.x + uint64_t(s) * gridDim.x;
            if (t < n_tiles) issue(s, t);
        }
    }

    uint32_t err = 0;
    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const int s = it % kStages;
        const int os = it % kOutStages;
        if (tid == 0) bulk_wait_read<kOutStages - 1>();  // output buffer `os` drained
        mbar_wait(&bars[s], (it / kStages) & 1);
        __syncthreads();

        const uint8_t* src = s_in + size_t(s) * (G::B0 + G::B1);
        uint32_t a[G::W0 > 0 ? G::W0 : 1], b[G::W1 > 0 ? G::W1 : 1];
        lds_run<G::W0>(src + tid * (G::R * Op::IN0), a);
        lds_run<G::W1>(src + G::B0 + tid * (G::R * Op::IN1), b);
        uint8_t o[G::R * Op::OUT];
        op.apply(a, b, o, s_tab, err);
        uint32_t ow[G::WO];
        pack_out<G::WO>(o, ow);
        uint32_t* dst = reinterpret_cast<uint32_t*>(s_out + size_t(os) * G::BO) + tid * G::WO;
#pragma unroll
        for (int i = 0; i < G::WO; ++i) dst[i] = ow[i];
        fence_proxy_async_smem();
        __syncthreads();

        if (tid == 0) {
            bulk_s2g(out + tile * G::BO, s_out + size_t(os) * G::BO, G::BO);
            bulk_commit();
            const uint64_t next = tile + uint64_t(kStages) * gridDim.x;
            if (next < n_tiles) issue(s, next);
        }
    }
    if (tid == 0) bulk_wait_all<0>();
    report(err, status);
}

// Records [first, n) with byte-granular global loads (tails, unaligned buffers).
template <class Op>
__global__ void __launch_bounds__(kThreads) stream_tail_kernel(const Op op, const uint8_t* __restrict__ in0,
                                                               const uint8_t* __restrict__ in1,
                                                               uint8_t* __restrict__ out, uint64_t first,
                                                               uint64_t n, uint32_t* status) {
    using G = Geometry<Op>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* s_tab = reinterpret_cast<uint32_t*>(smem);
    stage_tables(op, s_tab);
    __syncthreads();
    uint32_t err = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * G::R;
    for (uint64_t base = first + (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * G::R; base < n;
         base += stride) {
        const int cnt = n - base < uint64_t(G::R) ? static_cast<int>(n - base) : G::R;
        uint32_t a[G::W0 > 0 ? G::W0 : 1] = {}, b[G::W1 > 0 ? G::W1 : 1] = {};
        for (int i = 0; i < cnt * Op::IN0; ++i) a[i >> 2] |= uint32_t(in0[base * Op::IN0 + i]) << (8 * (i & 3));
        for (int i = 0; i < cnt * Op::IN1; ++i) b[i >> 2] |= uint32_t(in1[base * Op::IN1 + i]) << (8 * (i & 3));
        uint8_t o[G::R * Op::OUT];
        // zero padding is a valid input for every op, so it never raises
        op.apply(a, b, o, s_tab, err);
        for (int i = 0; i < cnt * Op::OUT; ++i) out[base * Op::OUT + i] = o[i];
    }
    report(err, status);
}

template <class Op>
cudaError_t run_stream(const Op& op, const uint8_t* in0, const uint8_t* in1, uint8_t* out, uint64_t n,
                       uint32_t* status, cudaStream_t s) {
    using G = Geometry<Op>;
    if (n == 0) return cudaSuccess;
    const size_t tab_bytes = size_t(op.tables_words()) * 4;
    const bool aligned = (reinterpret_cast<uintptr_t>(in0) % 16 == 0) &&
                         (G::B1 == 0 || reinterpret_cast<uintptr_t>(in1) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    const uint64_t n_tiles = aligned ? n / G::TILE : 0;
    const int sms = num_sms();
    if (n_tiles > 0) {
        const size_t smem = G::smem_fixed + tab_bytes;
        static bool attr_done = false;  // per instantiation
        if (!attr_done) {
            cudaError_t e = cudaFuncSetAttribute(stream_tma_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 227 * 1024);
            if (e != cudaSuccess) return e;
            attr_done = true;
        }
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stream_tma_kernel<Op>, kThreads, smem);
        if (e != cudaSuccess) return e;
        per_sm = std::max(per_sm, 1);
        const uint64_t grid = std::min<uint64_t>(n_tiles, uint64_t(sms) * per_sm);
        stream_tma_kernel<Op><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(op, in0, in1, out, n_tiles, status);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint64_t first = n_tiles * G::TILE;
    if (first < n) {
        static bool attr_done = false;
        if (!attr_done) {
            cudaError_t e = cudaFuncSetAttribute(stream_tail_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 227 * 1024);
            if (e != cudaSuccess) return e;
            attr_done = true;
        }
        const uint64_t groups = (n - first + G::R - 1) / G::R;
        const uint64_t grid = std::min<uint64_t>((groups + kThreads - 1) / kThreads, uint64_t(sms) * 8);
        stream_tail_kernel<Op><<<static_cast<unsigned>(grid), kThreads, tab_bytes, s>>>(op, in0, in1, out, first, n,
                                                                                        status);
        return cudaGetLastError();
    }
    return cudaSuccess;
}

template <int ND, bool POW2>
cudaError_t redq_dispatch_w(const RedqParams& P, const double* w, uint64_t n, uint8_t* out, uint32_t* st,
                            cudaStream_t s) {
    const auto* in = reinterpret_cast<const uint8_t*>(w);
    switch (P.window) {
        case 2: return run_stream(RedqOp<ND, POW2, 2>{P}, in, nullptr, out, n, st, s);
        case 3: return run_stream(RedqOp<ND, POW2, 3>{P}, in, nullptr, out, n, st, s);
        case 4: return run_stream(RedqOp<ND, POW2, 4>{P}, in, nullptr, out, n, st, s);
        default: return run_stream(RedqOp<ND, POW2, 0>{P}, in, nullptr, out, n, st, s);
    }
}

template <int ND>
cudaError_t redq_dispatch_q(const RedqParams& P, const double* w, uint64_t n, uint8_t* out, uint32_t* st,
                            cudaStream_t s) {
    return P.qbits ? redq_dispatch_w<ND, true>(P, w, n, out, st, s) : redq_dispatch_w<ND, false>(P, w, n, out, st, s);
}

template <int K, bool POW2>
cudaError_t polymul_dispatch_w(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out,
                               uint32_t* st, cudaStream_t s) {
    switch (P.rq.window) {
        case 2: return run_stream(PolymulOp<K, POW2, 2>{P}, a, b, out, n, st, s);
        case 3: return run_stream(PolymulOp<K, POW2, 3>{P}, a, b, out, n, st, s);
        case 4: return run_stream(PolymulOp<K, POW2, 4>{P}, a, b, out, n, st, s);
        default: return run_stream(PolymulOp<K, POW2, 0>{P}, a, b, out, n, st, s);
    }
}

template <int K>
cudaError_t polymul_dispatch_q(const PolymulParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                               uint8_t* out, uint32_t* st, cudaStream_t s) {
    return P.rq.qbits ? polymul_dispatch_w<K, true>(P, a, b, n, out, st, s)
                      : polymul_dispatch_w<K, false>(P, a, b, n, out, st, s);
}

template <int K>
cudaError_t gfq_elem_dispatch(const GfqElemParams& P, const uint8_t* a, const uint8_t* b, uint64_t n,
                              uint8_t* out, cudaStream_t s) {
    return P.rq.qbits ? run_stream(GfqElemOp<K, true>{P}, a, b, out, n, nullptr, s)
                      : run_stream(GfqElemOp<K, false>{P}, a, b, out, n, nullptr, s);
}

}  // namespace

}  // namespace qpk
