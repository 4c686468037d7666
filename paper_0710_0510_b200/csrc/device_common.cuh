// Device-side building blocks shared by the qpack B200 kernels (sm_100a).
//
//  * exact-integer fp64 helpers (the "floating-point floor" of paper Lemma 1)
//  * SplitMix64 at a counter (rng.hpp:17-22 restated for parallel generation)
//  * TMA bulk-copy (cp.async.bulk) + mbarrier wrappers, inline PTX
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

namespace qpk {

// ---------------------------------------------------------------- fp64 ints
constexpr double kTwo52 = 4503599627370496.0;  // 2^52
constexpr double kTwo53 = 9007199254740992.0;  // 2^53

// low 52 bits of a double in [2^52, 2^53) are the integer it holds minus 2^52
__device__ __forceinline__ uint64_t dbits(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }

// floor(x) as an exact 52-bit integer for 0 <= x < 2^52: x + 2^52 rounded
// toward zero lands on an integer of the [2^52, 2^53) binade (ulp = 1).
__device__ __forceinline__ uint64_t floor_u52(double x) {
    return dbits(__dadd_rz(x, kTwo52)) & ((uint64_t(1) << 52) - 1);
}

// floor(r / divisor) for an exact integer r <= r_max (paper Lemma 1,
// fpdiv.cpp:132-139).  The reference rounds the product to nearest and then
// steps one ulp up; rounding the product upward directly lands between
// r/divisor and that value, so for every r <= r_max both floor to the same
// integer floor(r/divisor).
__device__ __forceinline__ uint64_t floor_div_premul(double r, double inv_up) {
    return floor_u52(__dmul_ru(r, inv_up));
}

// OR a thread's error bits into *status once per warp (every lane of the
// warp must arrive)
__device__ __forceinline__ void report_status(uint32_t err, uint32_t* status) {
    err = __reduce_or_sync(0xffffffffu, err);
    if (err && (threadIdx.x & 31) == 0 && status) atomicOr(status, err);
}

// ----------------------------------------------------------------- SplitMix64
__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + j * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// --------------------------------------------------------- TMA bulk + mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared, completion counted on the mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// same, with an L2 evict-first hint for data read exactly once
__device__ __forceinline__ void bulk_g2s_stream(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                                uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// shared -> global bulk store, tracked by the bulk async-group
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// wait until at most N bulk groups still READ their shared source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// make generic-proxy shared-memory writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------- misc
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) { return (w >> (8 * i)) & 0xffu; }

// Programmatic dependent launch (kernels launched with launch_pdl below):
// pdl_wait blocks until every prerequisite grid has completed and its
// memory is visible; the launch itself, the CTA rasterisation and anything
// before pdl_wait (barrier setup, constant plan tables uploaded before the
// predecessor ran) overlap the previous kernel's tail.  A PDL kernel touches
// no data buffer before pdl_wait.  No kernel triggers its dependents early
// (griddepcontrol.launch_dependents) except the producer-warp stream
// pipeline at its CTAs' last tile (stream_kernels.cuh, one CTA per SM whose
// shared memory leaves no room for a waiting dependent): measured, an early
// trigger cost C2 0.1588 -> 0.1604 ms per step, C1 6.8 -> 7.3 us and K5
// 48.0 -> 50.2 us -- the dependents' waiting CTAs take SM slots (and
// launch work) while the primary still runs; the implicit trigger at exit
// keeps the overlap without that.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// host: launch with programmatic stream serialization (the kernel's prologue
// overlaps the previous kernel's tail; its data accesses follow pdl_wait)
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace qpk
