// Micro-benchmark (design calibration, not product code): aggregate HBM -> shared-memory bandwidth of
// 1-D bulk copies (cp.async.bulk + mbarrier complete_tx) issued by one thread per CTA, as the
// clustering's streamed tiles do, against the same data read with 16-byte vector loads by all
// threads.  Each CTA streams its contiguous share of a 1 GiB buffer through a `tile`-byte buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1811_02363_b200/csrc microbench/mb_tma.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "hdf_common.cuh"
using namespace hdf;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// mode 0: bulk copies of `chunk` bytes (thread 0), one tile at a time; mode 1: double-buffered
// half tiles; mode 2: all threads, LDG.128 into shared memory
__global__ void __launch_bounds__(512, 1) stream(const char* src, size_t per_cta, int tile, int chunk, int mode,
                                                 float* sink) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t ph;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
        ph = 0;
    }
    __syncthreads();
    const char* base = src + per_cta * blockIdx.x;
    float acc = 0.f;
    if (mode == 0) {
        for (size_t off = 0; off < per_cta; off += tile) {
            const uint32_t n = (uint32_t)min((size_t)tile, per_cta - off);
            __syncthreads();
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&bar[0], n);
                for (uint32_t c = 0; c < n; c += chunk) bulk(sm + c, base + off + c, min((uint32_t)chunk, n - c), &bar[0]);
            }
            mbar_wait(&bar[0], ph & 1u);
            __syncthreads();
            if (threadIdx.x == 0) ph ^= 1u;
            acc += reinterpret_cast<const float*>(sm)[threadIdx.x];
        }
    } else if (mode == 1) {
        const int half = tile / 2;
        int k = 0;
        auto issue = [&](size_t off, int b) {
            const uint32_t n = (uint32_t)min((size_t)half, per_cta - off);
            mbar_arrive_expect_tx(&bar[b], n);
            for (uint32_t c = 0; c < n; c += chunk) bulk(sm + b * half + c, base + off + c, min((uint32_t)chunk, n - c), &bar[b]);
        };
        if (threadIdx.x == 0) issue(0, 0);
        uint32_t phs = 0;
        for (size_t off = 0; off < per_cta; off += half, k++) {
            __syncthreads();
            if (threadIdx.x == 0 && off + half < per_cta) issue(off + half, (k + 1) & 1);
            mbar_wait(&bar[k & 1], (phs >> (k & 1)) & 1u);
            phs ^= 1u << (k & 1);
            acc += reinterpret_cast<const float*>(sm + (k & 1) * half)[threadIdx.x];
        }
    } else {
        for (size_t off = 0; off < per_cta; off += tile) {
            const uint32_t n = (uint32_t)min((size_t)tile, per_cta - off);
            __syncthreads();
            for (uint32_t c = threadIdx.x * 16; c < n; c += 512 * 16)
                *reinterpret_cast<float4*>(sm + c) = __ldcs(reinterpret_cast<const float4*>(base + off + c));
            __syncthreads();
            acc += reinterpret_cast<const float*>(sm)[threadIdx.x];
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main() {
    const size_t total = 1ull << 30;
    char* src;
    float* sink;
    CK(cudaMalloc(&src, total));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(src, 1, total));
    const int tile = 190 * 1024;
    CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, tile));
    for (int ncta : {112, 148}) {
        const size_t per = (total / ncta) & ~(size_t)255;
        for (int mode = 0; mode < 3; mode++)
            for (int chunk : {16384, 32768, 65536}) {
                if (mode == 2 && chunk != 32768) continue;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                stream<<<ncta, 512, tile>>>(src, per, tile, chunk, mode, sink);
                cudaEventRecord(a);
                for (int r = 0; r < 5; r++) stream<<<ncta, 512, tile>>>(src, per, tile, chunk, mode, sink);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("ctas %d mode %d chunk %6d: %.1f GB/s\n", ncta, mode, chunk, 5.0 * per * ncta / (ms * 1e-3) / 1e9);
            }
    }
    return 0;
}
