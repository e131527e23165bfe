// hdf_common.cuh -- shared device/host helpers of the CUDA path (sm_100a).
// Product code; shares nothing with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hdf.h"

#define HDF_DEV __device__ __forceinline__

namespace hdf {

constexpr int kMaxTaps = 2 * HDF_MAX_RADIUS + 1;

// ---------------------------------------------------------------------------------------------
// mbarrier / TMA (cp.async.bulk.tensor) wrappers -- inline PTX for sm_100a.
// ---------------------------------------------------------------------------------------------
HDF_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

HDF_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
HDF_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
HDF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

HDF_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
HDF_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
HDF_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
#ifndef HDF_MBAR_SLEEP_NS
#define HDF_MBAR_SLEEP_NS 0
#endif
HDF_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
#if HDF_MBAR_SLEEP_NS > 0
        __nanosleep(HDF_MBAR_SLEEP_NS);   // back off: a waiting warp leaves the issue slots to the others
#endif
    }
}

// The same with a run-time back-off (ns; 0 = plain spinning): for the roles that are not on the critical path, whose
// spinning would take issue slots from the ones that are.
HDF_DEV void mbar_wait_backoff(uint64_t* bar, uint32_t parity, int ns) {
    while (!mbar_try_wait(bar, parity)) {
        if (ns > 0) __nanosleep((unsigned)ns);
    }
}

// 3-D tiled TMA load global -> shared, completion signalled on `bar` (complete_tx::bytes).
HDF_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
HDF_DEV void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Named barrier among `nthreads` threads (id 1..15; id 0 is __syncthreads).
HDF_DEV void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

HDF_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
HDF_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exactly rounded fp64 squared distance accumulated in dimension order with no FMA contraction
// (so comparisons are reproducible, clustering).
HDF_DEV double d2_rn(double acc, double a, double b) {
    double t = __dsub_rn(a, b);
    return __dadd_rn(acc, __dmul_rn(t, t));
}

// packed f32x2 arithmetic (sm_100a): one FP32-pipe instruction per 64-bit register pair
HDF_DEV unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
HDF_DEV unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
HDF_DEV unsigned long long fsub2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
HDF_DEV unsigned long long fmul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
HDF_DEV unsigned long long pack2(float lo, float hi) {
    unsigned long long d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}
HDF_DEV void unpack2(unsigned long long v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }

}  // namespace hdf
