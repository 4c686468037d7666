// K1 pack kernels (coefficient records and dlog reps -> q-adic doubles) and
// the K4 launch dispatcher; the K4 kernel templates are in gfq_matmul.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"

namespace qpk {

// gfq_matmul_inst.cu, one per (k, variant): variant 1 = compile-time fast
// path (cudaErrorNotSupported when the field is not one it covers)
#define QPK_DECL_MM(K, V)                                                                                     \
    cudaError_t matmul_launch_k##K##_v##V(const GfqMatmulParams&, const double*, const double*, uint64_t,     \
                                          uint64_t, uint64_t, uint64_t, uint64_t, uint8_t*, uint32_t*,         \
                                          cudaStream_t);
QPK_DECL_MM(1, 0)
QPK_DECL_MM(2, 0)
QPK_DECL_MM(3, 0)
QPK_DECL_MM(4, 0)
QPK_DECL_MM(2, 1)
QPK_DECL_MM(3, 1)
#undef QPK_DECL_MM

namespace {

// 32x32 shared-memory tile transpose of u32 (coalesced both ways)
__global__ void transpose_u32_kernel(const uint32_t* __restrict__ src, uint64_t rows, uint64_t cols,
                                     uint32_t* __restrict__ dst) {
    __shared__ uint32_t tile[32][33];
    const uint64_t r0 = uint64_t(blockIdx.y) * 32, c0 = uint64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int i = ty; i < 32; i += 8)
        if (r0 + i < rows && c0 + tx < cols) tile[i][tx] = src[(r0 + i) * cols + c0 + tx];
    __syncthreads();
    for (int i = ty; i < 32; i += 8)
        if (c0 + i < cols && r0 + tx < rows) dst[(c0 + i) * rows + r0 + tx] = tile[tx][i];
}

// coefficient record (k bytes, reduced mod p as from_coeffs) -> rep
// (gfq.cpp:296-314: index sum c_i p^i, then the log table)
__global__ void coeffs_to_reps_kernel(uint32_t p, uint32_t k, const uint32_t* __restrict__ log,
                                      const uint8_t* __restrict__ src, uint64_t n, uint32_t* __restrict__ dst) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t idx = 0;
        for (int j = static_cast<int>(k) - 1; j >= 0; --j) idx = idx * p + src[i * k + j] % p;
        dst[i] = log[idx];
    }
}

// rep -> coefficient bytes (to_coeffs; the zero sentinel maps to 0)
__global__ void reps_to_coeffs_kernel(uint32_t k, const uint32_t* __restrict__ alog, const uint32_t* __restrict__ src,
                                      uint64_t n, uint8_t* __restrict__ dst) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t w = alog[src[i]];
        for (uint32_t j = 0; j < k; ++j) dst[i * k + j] = static_cast<uint8_t>(w >> (8 * j));
    }
}

// ---------------------------------------------------------------- K1 packs
// 32x32 tiles through shared memory so both the record reads and the
// (possibly transposed) double writes are coalesced.  KR (record width) is a
// template parameter; a thread reads 4 records with one vector load and the
// runtime reduction mod p runs only for bytes >= p (ncu: a runtime-k byte
// loop with an unconditional `% p` spent ~110 instructions per element at
// 2.5 TB/s: 68 -> 55 us per C4 operand with the template, less with the
// vector loads).
template <int KR>
__global__ void pack_coeffs_kernel(uint32_t p, double qd, const uint8_t* __restrict__ src, uint64_t rows,
                                   uint64_t cols, double* __restrict__ dst, uint64_t ld, bool transpose, bool pair) {
    __shared__ double tile[32][33];
    const uint64_t r0 = uint64_t(blockIdx.y) * 32, c0 = uint64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    // reads: each thread takes 4 consecutive records of one row (4 KR bytes,
    // one vector load when aligned): 8 threads per row, 32 rows
    {
        const int lin = ty * 32 + tx, rr = lin >> 3, cc = (lin & 7) * 4;
        const uint64_t r = r0 + rr, c = c0 + cc;
        uint32_t x[4][KR];
        const uint8_t* e = src + (r * cols + c) * KR;
        const bool full = r < rows && c + 4 <= cols;
        if (full && (reinterpret_cast<uintptr_t>(e) % (KR == 3 ? 4 : 4 * KR)) == 0) {
            uint32_t w[KR];  // 4 KR bytes as KR words
            if constexpr (KR == 1) {
                w[0] = *reinterpret_cast<const uint32_t*>(e);
            } else if constexpr (KR == 2) {
                const uint2 v = *reinterpret_cast<const uint2*>(e);
                w[0] = v.x, w[1] = v.y;
            } else if constexpr (KR == 3) {
#pragma unroll
                for (int t = 0; t < 3; ++t) w[t] = reinterpret_cast<const uint32_t*>(e)[t];
            } else {
                const uint4 v = *reinterpret_cast<const uint4*>(e);
                w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int t = 0; t < KR; ++t) {
                    const int byte = j * KR + t;
                    x[j][t] = (w[byte >> 2] >> (8 * (byte & 3))) & 0xffu;
                }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int t = 0; t < KR; ++t) x[j][t] = (r < rows && c + j < cols) ? e[j * KR + t] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double v = 0.0;
#pragma unroll
            for (int t = KR - 1; t >= 0; --t) {
                uint32_t xt = x[j][t];
                if (xt >= p) xt %= p;  // unreduced bytes are reduced as from_coeffs does
                v = fma(v, qd, static_cast<double>(xt));
            }
            tile[rr][cc + j] = v;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = ty; i < 32; i += 8) {
        if (transpose) {
            const uint64_t c = c0 + i, r = r0 + tx;
            if (r < rows && c < cols) dst[c * ld + (pair ? mm_col_a(r) : r)] = tile[tx][i];
        } else {
            const uint64_t r = r0 + i, c = c0 + tx;
            if (r < rows && c < cols) dst[r * ld + (pair ? mm_col_b(c) : c)] = tile[i][tx];
        }
    }
}

__global__ void pack_reps_kernel(const double* __restrict__ fval, uint32_t order, const uint32_t* __restrict__ src,
                                 uint64_t rows, uint64_t cols, double* __restrict__ dst, uint64_t ld, bool transpose,
                                 bool pair, uint32_t* status) {
    extern __shared__ double s_fval[];
    __shared__ double tile[32][33];
    for (uint32_t i = threadIdx.y * 32 + threadIdx.x; i < order; i += 256) s_fval[i] = fval[i];
    __syncthreads();
    const uint64_t r0 = uint64_t(blockIdx.y) * 32, c0 = uint64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    uint32_t err = 0;
    for (int i = ty; i < 32; i += 8) {
        const uint64_t r = r0 + i, c = c0 + tx;
        double v = 0.0;
        if (r < rows && c < cols) {
            const uint32_t rep = src[r * cols + c];
            if (rep < order) v = s_fval[rep];
            else err |= kErrRep;  // read as the zero element
        }
        tile[i][tx] = v;
    }
    report_status(err, status);
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        if (transpose) {
            const uint64_t c = c0 + i, r = r0 + tx;
            if (r < rows && c < cols) dst[c * ld + (pair ? mm_col_a(r) : r)] = tile[tx][i];
        } else {
            const uint64_t r = r0 + i, c = c0 + tx;
            if (r < rows && c < cols) dst[r * ld + (pair ? mm_col_b(c) : c)] = tile[i][tx];
        }
    }
}

}  // namespace

cudaError_t launch_gfq_matmul(const GfqMatmulParams& P, const double* at, const double* b, uint64_t m, uint64_t n,
                              uint64_t K_pad, uint64_t m_pad, uint64_t n_pad, uint8_t* out_coeffs,
                              uint32_t* out_reps, cudaStream_t s) {
    if (m == 0 || n == 0) return cudaSuccess;
    if (m_pad % 128 || n_pad % 128 || K_pad % 16) return cudaErrorInvalidValue;
    cudaError_t e = cudaErrorNotSupported;
    if (P.k == 2) e = matmul_launch_k2_v1(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
    if (P.k == 3) e = matmul_launch_k3_v1(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
    if (e != cudaErrorNotSupported) return e;
    switch (P.k) {
        case 1: return matmul_launch_k1_v0(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
        case 2: return matmul_launch_k2_v0(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
        case 3: return matmul_launch_k3_v0(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
        case 4: return matmul_launch_k4_v0(P, at, b, m, n, K_pad, m_pad, n_pad, out_coeffs, out_reps, s);
        default: return cudaErrorInvalidValue;
    }
}

int num_sms();

cudaError_t launch_transpose_u32(const uint32_t* src, uint64_t rows, uint64_t cols, uint32_t* dst, cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    transpose_u32_kernel<<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, dst);
    return cudaGetLastError();
}

cudaError_t launch_coeffs_to_reps(uint32_t p, uint32_t k, const uint32_t* log, const uint8_t* src, uint64_t n,
                                  uint32_t* dst, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8));
    coeffs_to_reps_kernel<<<grid, 256, 0, s>>>(p, k, log, src, n, dst);
    return cudaGetLastError();
}

cudaError_t launch_reps_to_coeffs(uint32_t k, const uint32_t* alog, const uint32_t* src, uint64_t n, uint8_t* dst,
                                  cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8));
    reps_to_coeffs_kernel<<<grid, 256, 0, s>>>(k, alog, src, n, dst);
    return cudaGetLastError();
}

cudaError_t launch_pack_coeffs(uint32_t p, uint32_t k, double qd, const uint8_t* src, uint64_t rows, uint64_t cols,
                               double* dst, uint64_t ld, bool transpose, bool pair_layout, cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    switch (k) {
        case 1: pack_coeffs_kernel<1><<<grid, dim3(32, 8), 0, s>>>(p, qd, src, rows, cols, dst, ld, transpose, pair_layout); break;
        case 2: pack_coeffs_kernel<2><<<grid, dim3(32, 8), 0, s>>>(p, qd, src, rows, cols, dst, ld, transpose, pair_layout); break;
        case 3: pack_coeffs_kernel<3><<<grid, dim3(32, 8), 0, s>>>(p, qd, src, rows, cols, dst, ld, transpose, pair_layout); break;
        case 4: pack_coeffs_kernel<4><<<grid, dim3(32, 8), 0, s>>>(p, qd, src, rows, cols, dst, ld, transpose, pair_layout); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_pack_reps(const double* fval, uint32_t order, const uint32_t* src, uint64_t rows, uint64_t cols,
                             double* dst, uint64_t ld, bool transpose, bool pair_layout, uint32_t* status,
                             cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
    const size_t smem = size_t(order) * 8;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(pack_reps_kernel), smem); e != cudaSuccess)
        return e;
    pack_reps_kernel<<<grid, dim3(32, 8), smem, s>>>(fval, order, src, rows, cols, dst, ld, transpose, pair_layout, status);
    return cudaGetLastError();
}

}  // namespace qpk
