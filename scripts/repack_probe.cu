// Delayed-REDQ re-pack for C5 (GF(3^3), q = 2^10): generic REDQ vs the SWAR
// formulation -- exhaustive agreement on random words and cycles per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_0710_0510_b200/csrc \
//        scripts/repack_probe.cu -o scripts/rp_bin
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "gfq_matmul.cuh"

using namespace qpk;

__global__ void check(RedqParams P, unsigned long long n, unsigned long long* bad) {
    const CtConst<3, 10> c{P};
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) {
        const unsigned long long x = splitmix_at(99, i) >> 14;  // < 2^50
        const double r = static_cast<double>(x);
        if (redq_repack<5>(c, r) != redq_repack_swar3<5, 10>(P, r)) atomicAdd(bad, 1ull);
    }
}

template <bool SWAR>
__global__ void __launch_bounds__(128, 1) timing(RedqParams P, double* sink, int iters, long long* cyc) {
    const CtConst<3, 10> c{P};
    double acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = double((threadIdx.x * 64 + i) * 1234567ull % (1ull << 49));
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
            acc[i] = SWAR ? redq_repack_swar3<5, 10>(P, acc[i] + 700.0) : redq_repack<5>(c, acc[i] + 700.0);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s += acc[i];
    if (s == 1.5) sink[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / iters;
}

int main() {
    RedqParams P{};
    P.p = 3, P.d = 4, P.qbits = 10, P.neg_q = 2, P.q = 1024;
    P.mod_magic = uint32_t(((1ull << 32) + 2) / 3);
    P.inv_p = std::nextafter(1.0 / 3.0, 1.0);  // ReciprocalDivisor::make(3).inv_up
    P.r_max = 1501199875790165.0;
    P.limit = double(1ull << 50);
    double* s;
    long long* cyc;
    unsigned long long* bad;
    cudaMalloc(&s, 64);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    const unsigned long long n = 1ull << 30;
    check<<<148 * 8, 256>>>(P, n, bad);
    unsigned long long hb = 0;
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    printf("SWAR vs generic re-pack: %llu mismatches in %llu words\n", hb, n);
    for (int sw = 0; sw < 2; ++sw) {
        if (sw) timing<true><<<148, 128>>>(P, s, 100, cyc);
        else timing<false><<<148, 128>>>(P, s, 100, cyc);
        long long h = 0;
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%s: %lld cycles per re-pack of 64 accumulators (one warp per SMSP)\n", sw ? "swar   " : "generic", h);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
