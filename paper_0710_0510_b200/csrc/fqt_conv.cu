// K6 host launch: pack kernels, the per-chunk-width convolution kernels
// (instantiated in fqt_conv_inst.cu, one object per width), overlap-add.
#include "fqt_conv.cuh"

namespace qpk {

// fqt_conv_inst.cu, -DQPK_INST=ND
cudaError_t fqt_conv_nd1(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd3(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd5(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd7(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd9(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd11(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd13(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);
cudaError_t fqt_conv_nd15(const FqtParams& P, const double* pw, uint64_t L1, const double* qw, uint64_t L2,
                          uint64_t T, uint32_t splits, uint64_t isplit, uint32_t* res, cudaStream_t s);

namespace {

// Overlap-add: chunk u of the output is residues 0..k-1 of product chunk u
// plus residues k..2k-2 of chunk u-1, each summed over the splits.  A CTA
// owns 256 chunks: thread i sums chunk u0+i's split partials lane-wise mod
// p (one coalesced word per split and lane word, up to 16 loads in flight),
// a 257th thread (warp 8) chunk u0-1; the sums meet in shared memory and
// each thread writes its k coefficients.  The DMMA kernel writes only the
// valid splits of its tile (fqt_mma_tile_splits, mma_cd != 0).
constexpr int kOvThreads = 256 + 32;

__global__ void __launch_bounds__(kOvThreads) fqt_overlap_kernel(uint32_t p, uint32_t k, uint32_t nd,
                                                                 const uint32_t* __restrict__ res, uint32_t splits,
                                                                 uint64_t T, uint8_t* __restrict__ out,
                                                                 uint64_t nout, uint64_t mma_cd, uint64_t L1,
                                                                 uint64_t L2) {
    __shared__ uint32_t sums[257][4];
    pdl_wait();
    const uint32_t nw = (nd + 3) / 4;
    const uint64_t nchunks = (nout + k - 1) / k;
    const int tid = threadIdx.x;
    // slot 0 holds chunk u0-1, slot i+1 chunk u0+i
    const int slot = tid < 256 ? tid + 1 : (tid == 256 ? 0 : -1);
    for (uint64_t u0 = uint64_t(blockIdx.x) * 256; u0 < nchunks; u0 += uint64_t(gridDim.x) * 256) {
        if (slot >= 0) {
            const int64_t u = static_cast<int64_t>(u0) - 1 + slot;
            uint32_t acc[4] = {0, 0, 0, 0};
            if (u >= 0 && static_cast<uint64_t>(u) < T) {
                const uint32_t splits_u =
                    mma_cd ? fqt_mma_tile_splits(static_cast<uint64_t>(u) / kMmaOut, L1, L2, mma_cd) : splits;
                const uint64_t stride = T * nw;
                for (uint32_t w = 0; w < nw; ++w) {
                    const uint32_t* src = res + static_cast<uint64_t>(u) * nw + w;
                    uint32_t sp = 0;
                    for (; sp + 16 <= splits_u; sp += 16) {
                        uint32_t v[16];
#pragma unroll
                        for (int x = 0; x < 16; ++x) v[x] = __ldg(src + (sp + x) * stride);
#pragma unroll
                        for (int x = 0; x < 16; ++x) acc[w] = add_mod_lanes(acc[w], v[x], p);
                    }
                    if (sp < splits_u) {
                        uint32_t v[16];
#pragma unroll
                        for (int x = 0; x < 16; ++x) v[x] = sp + x < splits_u ? __ldg(src + (sp + x) * stride) : 0u;
#pragma unroll
                        for (int x = 0; x < 16; ++x) acc[w] = add_mod_lanes(acc[w], v[x], p);
                    }
                }
            }
            for (uint32_t w = 0; w < 4; ++w) sums[slot][w] = acc[w];
        }
        __syncthreads();
        const uint64_t u = u0 + tid;
        if (tid < 256 && u < nchunks) {
            for (uint32_t j = 0; j < k; ++j) {
                const uint64_t ci = u * k + j;
                if (ci >= nout) break;
                uint32_t v = (sums[tid + 1][j / 4] >> (8 * (j % 4))) & 0xffu;
                const uint32_t jh = j + k;
                if (jh < nd) v += (sums[tid][jh / 4] >> (8 * (jh % 4))) & 0xffu;
                out[ci] = static_cast<uint8_t>(v >= p ? v - p : v);
            }
        }
        __syncthreads();
    }
}

// both operands packed by one launch: chunks [0, L1) of a, then [0, L2) of b
__global__ void fqt_pack2_kernel(uint32_t p, uint32_t k, double qd, const uint8_t* __restrict__ a, uint64_t na,
                                 uint64_t L1, double* __restrict__ wa, const uint8_t* __restrict__ b, uint64_t nb,
                                 uint64_t L2, double* __restrict__ wb) {
    pdl_wait();
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < L1 + L2;
         x += uint64_t(gridDim.x) * blockDim.x) {
        const bool first = x < L1;
        const uint64_t c = first ? x : x - L1, n = first ? na : nb;
        const uint8_t* src = first ? a : b;
        double v = 0.0;
        for (int j = static_cast<int>(k) - 1; j >= 0; --j) {
            const uint64_t i = c * k + j;
            const uint32_t xv = i < n ? src[i] % p : 0u;
            v = fma(v, qd, static_cast<double>(xv));
        }
        (first ? wa : wb)[c] = v;
    }
}

// ---- wide words (m > 53): u128 packed words, one thread per output chunk ----
using u128d = unsigned __int128;

struct FqtWideParams {
    uint32_t p, k, nq, nd, neg_q, qbits;  // qbits: log2 q when q is a power of two, else 0
    uint64_t q;
    u128d qpow[15];                       // q^i, i < nd
};

__global__ void fqt_wide_pack_kernel(uint32_t p, uint32_t k, uint64_t q, const uint8_t* __restrict__ a, uint64_t na,
                                     uint64_t L1, u128d* __restrict__ wa, const uint8_t* __restrict__ b, uint64_t nb,
                                     uint64_t L2, u128d* __restrict__ wb) {
    pdl_wait();
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < L1 + L2;
         x += uint64_t(gridDim.x) * blockDim.x) {
        const bool first = x < L1;
        const uint64_t c = first ? x : x - L1, n = first ? na : nb;
        const uint8_t* src = first ? a : b;
        u128d v = 0;  // Horner (pack, dqt.cpp:23-37)
        for (int j = static_cast<int>(k) - 1; j >= 0; --j) {
            const uint64_t i = c * k + j;
            v = v * q + (i < n ? src[i] % p : 0u);
        }
        (first ? wa : wb)[c] = v;
    }
}

// integer-mode REDQ of one group sum (redq.cpp:44-58): rop = r / p,
// u_i = r / q^i - p (rop / q^i), then mu_d = u_d, mu_i = (u_i + neg_q u_{i+1})
// mod p (redq.cpp:63-65); the residues are added mod p into byte lanes
__device__ __forceinline__ void fqt_wide_close(const FqtWideParams& P, u128d r, uint32_t (&racc)[4]) {
    const u128d rop = r / P.p;
    uint32_t u[15];
    for (uint32_t i = 0; i < P.nd; ++i) {
        u128d x, y;
        if (P.qbits) {
            x = r >> (P.qbits * i);
            y = rop >> (P.qbits * i);
        } else {
            x = r / P.qpow[i];
            y = rop / P.qpow[i];
        }
        u[i] = static_cast<uint32_t>(static_cast<uint64_t>(x) - P.p * static_cast<uint64_t>(y));
    }
    for (uint32_t i = 0; i < P.nd; ++i) {
        const uint32_t mu = i + 1 < P.nd ? (u[i] + P.neg_q * u[i + 1]) % P.p : u[i];
        const uint32_t w = i / 4, sh = 8 * (i % 4);
        uint32_t lane = ((racc[w] >> sh) & 0xffu) + mu;
        if (lane >= P.p) lane -= P.p;
        racc[w] = (racc[w] & ~(0xffu << sh)) | (lane << sh);
    }
}

// output chunk t = sum_i pw[i] qw[t-i] in u128, a REDQ every n_q products
__global__ void __launch_bounds__(256) fqt_wide_conv_kernel(const FqtWideParams P, const u128d* __restrict__ pw,
                                                            uint64_t L1, const u128d* __restrict__ qw, uint64_t L2,
                                                            uint64_t T, uint32_t* __restrict__ res) {
    pdl_wait();
    const uint32_t nw = (P.nd + 3) / 4;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < T; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t lo = t + 1 > L2 ? t + 1 - L2 : 0, hi = t < L1 - 1 ? t : L1 - 1;
        uint32_t racc[4] = {0, 0, 0, 0};
        u128d acc = 0;
        uint32_t cnt = 0;
        for (uint64_t i = lo; i <= hi; ++i) {
            acc += pw[i] * qw[t - i];  // exact: a group sum stays below q^(2k-1) < 2^m <= 2^128
            if (++cnt == P.nq) {
                fqt_wide_close(P, acc, racc);
                acc = 0;
                cnt = 0;
            }
        }
        if (cnt) fqt_wide_close(P, acc, racc);
        for (uint32_t w = 0; w < nw; ++w) res[t * nw + w] = racc[w];
    }
}

// ---- large p (p > 256, u64 coefficients): u128 words and group sums, one
// thread per output chunk; residues kept per coefficient as u64 ----
struct FqtWidePParams {
    uint64_t p, neg_q, q;
    uint32_t k, nq, nd, qbits;  // qbits: log2 q when q is a power of two, else 0
    u128d qpow[15];             // q^i, i < nd
};

__global__ void fqt_widep_pack_kernel(uint64_t p, uint32_t k, uint64_t q, const uint64_t* __restrict__ a,
                                      uint64_t na, uint64_t L1, u128d* __restrict__ wa,
                                      const uint64_t* __restrict__ b, uint64_t nb, uint64_t L2,
                                      u128d* __restrict__ wb) {
    pdl_wait();
    for (uint64_t x = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < L1 + L2;
         x += uint64_t(gridDim.x) * blockDim.x) {
        const bool first = x < L1;
        const uint64_t c = first ? x : x - L1, n = first ? na : nb;
        const uint64_t* src = first ? a : b;
        u128d v = 0;  // Horner (pack, dqt.cpp:23-37), coefficients reduced mod p (DensePoly)
        for (int j = static_cast<int>(k) - 1; j >= 0; --j) {
            const uint64_t i = c * k + j;
            v = v * q + (i < n ? src[i] % p : 0u);
        }
        (first ? wa : wb)[c] = v;
    }
}

// integer-mode REDQ of one group sum (redq.cpp:44-65) added mod p into the
// chunk's residues
__device__ __forceinline__ void fqt_widep_close(const FqtWidePParams& P, u128d r, uint64_t (&racc)[15]) {
    const u128d rop = r / P.p;
    uint64_t u[15];
    for (uint32_t i = 0; i < P.nd; ++i) {
        const u128d x = P.qbits ? r >> (P.qbits * i) : r / P.qpow[i];
        const u128d y = P.qbits ? rop >> (P.qbits * i) : rop / P.qpow[i];
        u[i] = static_cast<uint64_t>(x - static_cast<u128d>(P.p) * y);  // in [0, p)
    }
    for (uint32_t i = 0; i < P.nd; ++i) {
        const uint64_t mu =
            i + 1 < P.nd ? static_cast<uint64_t>((u[i] + static_cast<u128d>(P.neg_q) * u[i + 1]) % P.p) : u[i];
        const uint64_t s = racc[i] + mu;  // both < p < 2^63: no wrap
        racc[i] = s >= P.p ? s - P.p : s;
    }
}

__global__ void __launch_bounds__(256) fqt_widep_conv_kernel(const FqtWidePParams P, const u128d* __restrict__ pw,
                                                             uint64_t L1, const u128d* __restrict__ qw, uint64_t L2,
                                                             uint64_t T, uint64_t* __restrict__ res) {
    pdl_wait();
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < T; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t lo = t + 1 > L2 ? t + 1 - L2 : 0, hi = t < L1 - 1 ? t : L1 - 1;
        uint64_t racc[15] = {};
        u128d acc = 0;
        uint32_t cnt = 0;
        for (uint64_t i = lo; i <= hi; ++i) {
            acc += pw[i] * qw[t - i];  // exact: a group sum stays below q^(2k-1) <= 2^m <= 2^128
            if (++cnt == P.nq) {
                fqt_widep_close(P, acc, racc);
                acc = 0;
                cnt = 0;
            }
        }
        if (cnt) fqt_widep_close(P, acc, racc);
        for (uint32_t i = 0; i < P.nd; ++i) res[t * P.nd + i] = racc[i];
    }
}

// out coefficient c of chunk u = c / k, j = c % k: residue j of chunk u plus
// residue j + k of chunk u - 1 (fqt_decode's overlap, polymul.cpp:52-79)
__global__ void fqt_widep_overlap_kernel(uint64_t p, uint32_t k, uint32_t nd, const uint64_t* __restrict__ res,
                                         uint64_t T, uint64_t* __restrict__ out, uint64_t nout) {
    pdl_wait();
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < nout;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t u = c / k;
        const uint32_t j = static_cast<uint32_t>(c % k);
        uint64_t v = u < T ? res[u * nd + j] : 0;
        if (u >= 1 && j + k < nd) {
            const uint64_t w = res[(u - 1) * nd + j + k];
            v = v + w >= p ? v + w - p : v + w;
        }
        out[c] = v;
    }
}

}  // namespace


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
// DMMA kernel: each 1024-output tile's valid block shifts d cut into equal
// ranges of at most kMmaCD, ~8 CTAs per SM (chunk = the range length)
FqtSplit fqt_split_mma_uncached(uint64_t L1, uint64_t L2) {
    const uint64_t T = L1 + L2 - 1, tiles = (T + kMmaOut - 1) / kMmaOut;
    uint64_t total = 0, longest = 0;
    for (uint64_t x = 0; x < tiles; ++x) {
        int64_t dmin, dmax;
        fqt_mma_tile_shifts(x, L1, L2, dmin, dmax);
        const uint64_t len = dmax >= dmin ? uint64_t(dmax - dmin + 1) : 0;
        total += len;
        longest = std::max(longest, len);
    }
    // CTAs run in waves of kMmaCtasPerSm per SM over (nearly) equal shift
    // ranges: pick cd minimising waves * (cd + per-CTA overhead) so the last
    // wave is nearly full (a 2.06-wave split left the DMMA pipe 22% idle)
    (void)total;
    const uint64_t resident = uint64_t(num_sms()) * kMmaCtasPerSm;
    uint64_t best_cd = kMmaCD;
    double best = -1.0;
    // (large products: many waves, the search is not worth its host time)
    for (uint64_t cd = tiles > 4096 ? uint64_t(kMmaCD) : 16; cd <= uint64_t(kMmaCD); ++cd) {
        uint64_t items = 0;
        for (uint64_t x = 0; x < tiles; ++x) items += fqt_mma_tile_splits(x, L1, L2, cd);
        const double cost = double((items + resident - 1) / resident) * double(cd + 6);
        if (best < 0 || cost < best) {
            best = cost;
            best_cd = cd;
        }
    }
    return {static_cast<uint32_t>(std::max<uint64_t>((longest + best_cd - 1) / best_cd, 1)), best_cd};
}
// the search above costs host microseconds: remember the last shapes
FqtSplit fqt_split_mma(uint64_t L1, uint64_t L2) {
    struct Entry {
        uint64_t L1 = 0, L2 = 0;
        FqtSplit sp{};
    };
    static thread_local Entry cache[4];
    static thread_local unsigned next = 0;
    for (const Entry& e : cache)
        if (e.L1 == L1 && e.L2 == L2 && e.sp.splits) return e.sp;
    Entry& e = cache[next++ % 4];
    e = {L1, L2, fqt_split_mma_uncached(L1, L2)};
    return e.sp;
}
FqtSplit fqt_split(uint64_t L1, uint64_t L2, uint32_t nq) {
    if (fqt_use_mma(nq)) return fqt_split_mma(L1, L2);
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

uint64_t fqt_wide_workspace_bytes(uint32_t k, uint64_t na, uint64_t nb) {
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    const uint32_t nw = (2 * k - 1 + 3) / 4;
    return align16(L1 * 16) + align16(L2 * 16) + T * nw * 4;
}

cudaError_t launch_fqt_mul_wide(uint32_t p, uint64_t q, uint32_t k, uint32_t nq, const uint8_t* a, uint64_t na,
                                const uint8_t* b, uint64_t nb, uint8_t* out, void* ws, cudaStream_t s) {
    if (na == 0 || nb == 0) return cudaSuccess;
    if (k < 1 || k > 8 || p < 2 || p > 256 || nq == 0) return cudaErrorInvalidValue;
    FqtWideParams P{};
    P.p = p;
    P.k = k;
    P.nq = nq;
    P.nd = 2 * k - 1;
    P.q = q;
    P.neg_q = static_cast<uint32_t>((p - q % p) % p);
    P.qbits = (q & (q - 1)) == 0 ? static_cast<uint32_t>(__builtin_ctzll(q)) : 0u;
    u128d qp = 1;
    for (uint32_t i = 0; i < P.nd; ++i, qp *= q) P.qpow[i] = qp;
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    auto* base = static_cast<uint8_t*>(ws);
    auto* pw = reinterpret_cast<u128d*>(base);
    auto* qw = reinterpret_cast<u128d*>(base + align16(L1 * 16));
    auto* res = reinterpret_cast<uint32_t*>(base + align16(L1 * 16) + align16(L2 * 16));
    const int sms = num_sms();
    if (cudaError_t e = launch_pdl(fqt_wide_pack_kernel,
                                   dim3(static_cast<unsigned>(std::min<uint64_t>((L1 + L2 + 255) / 256, sms * 8))),
                                   dim3(256), 0, s, p, k, q, a, na, L1, pw, b, nb, L2, qw);
        e != cudaSuccess)
        return e;
    if (cudaError_t e = launch_pdl(fqt_wide_conv_kernel,
                                   dim3(static_cast<unsigned>(std::min<uint64_t>((T + 255) / 256, sms * 16))),
                                   dim3(256), 0, s, P, static_cast<const u128d*>(pw), L1, static_cast<const u128d*>(qw),
                                   L2, T, res);
        e != cudaSuccess)
        return e;
    const uint64_t nout = na + nb - 1, nchunks = (nout + k - 1) / k;
    return launch_pdl(fqt_overlap_kernel, dim3(static_cast<unsigned>(std::min<uint64_t>((nchunks + 255) / 256, sms * 8))),
                      dim3(kOvThreads), 0, s, p, k, 2 * k - 1, static_cast<const uint32_t*>(res), 1u, T, out, nout,
                      uint64_t(0), L1, L2);
}

uint64_t fqt_widep_workspace_bytes(uint32_t k, uint64_t na, uint64_t nb) {
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    return align16(L1 * 16) + align16(L2 * 16) + T * (2 * k - 1) * 8 + 16;
}

cudaError_t launch_fqt_mul_widep(uint64_t p, uint64_t q, uint32_t k, uint32_t nq, const uint64_t* a, uint64_t na,
                                 const uint64_t* b, uint64_t nb, uint64_t* out, void* ws, cudaStream_t s) {
    if (na == 0 || nb == 0) return cudaSuccess;
    if (k < 1 || k > 8 || p < 2 || p >= (uint64_t(1) << 63) || nq == 0) return cudaErrorInvalidValue;
    FqtWidePParams P{};
    P.p = p;
    P.k = k;
    P.nq = nq;
    P.nd = 2 * k - 1;
    P.q = q;
    P.neg_q = (p - q % p) % p;
    P.qbits = (q & (q - 1)) == 0 ? static_cast<uint32_t>(__builtin_ctzll(q)) : 0u;
    u128d qp = 1;
    for (uint32_t i = 0; i < P.nd; ++i, qp *= q) P.qpow[i] = qp;
    const uint64_t L1 = fqt_chunks(na, k), L2 = fqt_chunks(nb, k), T = L1 + L2 - 1;
    auto* base = static_cast<uint8_t*>(ws);
    auto* pw = reinterpret_cast<u128d*>(base);
    auto* qw = reinterpret_cast<u128d*>(base + align16(L1 * 16));
    auto* res = reinterpret_cast<uint64_t*>(base + align16(L1 * 16) + align16(L2 * 16));
    const int sms = num_sms();
    if (cudaError_t e = launch_pdl(fqt_widep_pack_kernel,
                                   dim3(static_cast<unsigned>(std::min<uint64_t>((L1 + L2 + 255) / 256, sms * 8))),
                                   dim3(256), 0, s, p, k, q, a, na, L1, pw, b, nb, L2, qw);
        e != cudaSuccess)
        return e;
    if (cudaError_t e = launch_pdl(fqt_widep_conv_kernel,
                                   dim3(static_cast<unsigned>(std::min<uint64_t>((T + 255) / 256, sms * 16))),
                                   dim3(256), 0, s, P, static_cast<const u128d*>(pw), L1, static_cast<const u128d*>(qw),
                                   L2, T, res);
        e != cudaSuccess)
        return e;
    const uint64_t nout = na + nb - 1;
    return launch_pdl(fqt_widep_overlap_kernel,
                      dim3(static_cast<unsigned>(std::min<uint64_t>((nout + 255) / 256, sms * 8))), dim3(256), 0, s,
                      p, k, 2 * k - 1, static_cast<const uint64_t*>(res), T, out, nout);
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
    // chunks of k coefficients (reduced mod p) -> q-adic words (fqt_encode,
    // polymul.cpp:31-50), zero beyond n
    if (cudaError_t e = launch_pdl(fqt_pack2_kernel,
                                   dim3(static_cast<unsigned>(std::min<uint64_t>((L1 + L2 + 255) / 256, sms * 8))),
                                   dim3(256), 0, s, P.rq.p, k, qd, a, na, L1, pw, b, nb, L2, qw);
        e != cudaSuccess)
        return e;
    const FqtSplit sp = fqt_split(L1, L2, P.nq);
    const uint32_t splits = sp.splits;
    const uint64_t isplit = sp.chunk;
    cudaError_t e;
    switch (nd) {
        case 1: e = fqt_conv_nd1(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 3: e = fqt_conv_nd3(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 5: e = fqt_conv_nd5(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 7: e = fqt_conv_nd7(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 9: e = fqt_conv_nd9(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 11: e = fqt_conv_nd11(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 13: e = fqt_conv_nd13(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        case 15: e = fqt_conv_nd15(P, pw, L1, qw, L2, T, splits, isplit, res, s); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const uint64_t nout = na + nb - 1;
    const uint64_t nchunks = (nout + k - 1) / k;
    return launch_pdl(fqt_overlap_kernel, dim3(static_cast<unsigned>(std::min<uint64_t>((nchunks + 255) / 256, sms * 8))),
                      dim3(kOvThreads), 0, s, P.rq.p, k, nd, static_cast<const uint32_t*>(res), splits, T, out, nout,
                      fqt_use_mma(P.nq) ? isplit : uint64_t(0), L1, L2);
}

}  // namespace qpk
