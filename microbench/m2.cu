// m2.cu -- latency micro-benchmarks that decide the clustering kernel's synchronisation design.
//   (a) cooperative grid.sync with 1 fat CTA per SM
//   (b) grid.sync + every CTA re-reading all CTAs' 8-double records (publish / reduce round trip)
//   (c) thread-block-cluster barrier (barrier.cluster) and a DSMEM read round trip
//   (d) whether a cooperative launch accepts a cluster dimension
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o m2 m2.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); } } while (0)

__global__ void k_sync(int iters, long long* out) {
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

__global__ void k_sync_reduce(int iters, double* rec, double* sink, long long* out) {
    cg::grid_group g = cg::this_grid();
    extern __shared__ double sm[];
    const int G = gridDim.x;
    long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < iters; i++) {
        double* r = rec + (size_t)(i & 1) * G * 8;
        if (threadIdx.x < 8) r[blockIdx.x * 8 + threadIdx.x] = i + blockIdx.x + threadIdx.x;
        g.sync();
        for (int f = threadIdx.x; f < G * 8; f += blockDim.x) sm[f] = __ldcg(r + f);
        __syncthreads();
        if (threadIdx.x < 8) {
            double s = 0;
            for (int b = 0; b < G; b++) s += sm[b * 8 + threadIdx.x];
            acc += s;
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { *out = clock64() - t0; *sink = acc; }
}

__global__ void k_l2_rtt(const double* p, int iters, long long* out, double* sink) {
    // dependent pointer-chase-like chain through L2 (cg loads) from one thread
    long long t0 = clock64();
    double s = 0;
    int idx = 0;
    for (int i = 0; i < iters; i++) {
        double v = __ldcg(p + idx);
        s += v;
        idx = ((int)v + i * 97) & 1023;
    }
    *out = clock64() - t0;
    *sink = s;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster_bar(int iters, long long* out, double* sink) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double v[16];
    long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < iters; i++) {
        if (threadIdx.x < 16) v[threadIdx.x] = i + threadIdx.x;
        cl.sync();
        if (threadIdx.x < 16) {
            double* rv = cl.map_shared_rank(v, threadIdx.x);
            acc += rv[cl.block_rank()];
        }
        cl.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { *out = clock64() - t0; *sink = acc; }
}

__global__ void k_coop_cluster(int* ok) {
    cg::grid_group g = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *ok = 1 + (int)cl.num_blocks();
}

__global__ void k_fp64(int iters, double* out) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; i++) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    }
    if (a0 + a1 + a2 + a3 == 12345.0) *out = a0;
}
__global__ void k_fp64_addmul(int iters, double* out) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; i++) {
        a0 = __dadd_rn(__dmul_rn(a0, b), c); a1 = __dadd_rn(__dmul_rn(a1, b), c);
        a2 = __dadd_rn(__dmul_rn(a2, b), c); a3 = __dadd_rn(__dmul_rn(a3, b), c);
    }
    if (a0 + a1 + a2 + a3 == 12345.0) *out = a0;
}
__global__ void k_fp32(int iters, float* out) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = 1.0000001f, c = 1e-9f;
    for (int i = 0; i < iters; i++) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
    }
    if (a0 + a1 + a2 + a3 == 12345.0f) *out = a0;
}

__global__ void k_lat(int iters, long long* out, double* sink) {
    double a = threadIdx.x * 1e-3 + 1.0, b = 1.0000001, c = 1e-9;
    float fa = threadIdx.x * 1e-3f + 1.0f, fb = 1.0000001f, fc = 1e-9f;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < iters; i++) a = __dadd_rn(__dmul_rn(a, b), c);
    long long t2 = clock64();
    for (int i = 0; i < iters; i++) fa = fmaf(fa, fb, fc);
    long long t3 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; }
    sink[threadIdx.x] = a + fa;
}

// (g) generic vs explicit shared loads: pair loop like the farthest-pair seed (fp64 distance of
// 1024 fp32 points of dim 3 held in shared memory), one CTA of 512 threads.
__global__ void k_pairs(const float* src, int generic_ptr, long long* out, double* sink) {
    __shared__ float pts[1024 * 3];
    for (int i = threadIdx.x; i < 3072; i += blockDim.x) pts[i] = src[i];
    __syncthreads();
    const float* P = generic_ptr ? (const float*)((volatile const float*)pts) : pts;
    long long t0 = clock64();
    double best = -1; int arg = -1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int a = warp; a < 1024; a += 16) {
        const float* xa = P + a * 3;
        for (int b = a + 1 + lane; b < 1024; b += 32) {
            const float* xb = P + b * 3;
            double dd = 0.0;
            for (int d = 0; d < 3; d++) {
                double t = __dsub_rn((double)xa[d], (double)xb[d]);
                dd = __dadd_rn(dd, __dmul_rn(t, t));
            }
            if (dd > best) { best = dd; arg = b; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = clock64() - t0;
    sink[threadIdx.x] = best + arg;
}

__device__ __forceinline__ double d2_rn(double acc, double a, double b) {
    double t = __dsub_rn(a, b);
    return __dadd_rn(acc, __dmul_rn(t, t));
}
template <class Base>
__device__ __forceinline__ void row_farthest(int a, int sN, int rho, Base base, double& best, int& arg) {
    const int lane = threadIdx.x & 31;
    constexpr float u = 5.9604644775390625e-08f;
    const float* xa = base(a);
    float m = 0.f;
    for (int q = a + 1 + lane; q < sN; q += 32) {
        const float* xb = base(q);
        float acc = 0.f;
        for (int d = 0; d < rho; d++) { const float t = xa[d] - xb[d]; acc = fmaf(t, t, acc); }
        m = fmaxf(m, acc);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float thr = m * (1.0f - 8.0f * (float)(rho + 3) * u);
    best = -1.0; arg = -1;
    for (int q = a + 1 + lane; q < sN; q += 32) {
        const float* xb = base(q);
        float acc = 0.f;
        for (int d = 0; d < rho; d++) { const float t = xa[d] - xb[d]; acc = fmaf(t, t, acc); }
        if (acc >= thr) {
            double dd = 0.0;
            for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)xa[d], (double)xb[d]);
            if (dd > best) { best = dd; arg = q; }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (oa >= 0 && (arg < 0 || ob > best || (ob == best && oa < arg))) { best = ob; arg = oa; }
    }
}
__global__ void k_rowfar(const float* src, int rho, long long* out, double* sink) {
    extern __shared__ float tp[];
    for (int i = threadIdx.x; i < 1024 * rho; i += blockDim.x) tp[i] = src[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    double bv = -1; int ba = -1;
    for (int ra = 16 * warp; ra < 1024; ra += 16 * 16) {
        double best; int arg;
        const float* tpc = tp;
        row_farthest(ra, 1024, rho, [&](int q) { return tpc + (size_t)q * rho; }, best, arg);
        if (arg >= 0 && (ba < 0 || best > bv)) { bv = best; ba = ra; }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = clock64() - t0;
    sink[threadIdx.x] = bv + ba;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double ghz = clk * 1e-6;
    long long* dout;
    double *drec, *dsink;
    int* dok;
    CK(cudaMalloc(&dout, 8));
    CK(cudaMalloc(&drec, 1 << 20));
    CK(cudaMalloc(&dsink, 8));
    CK(cudaMalloc(&dok, 4));
    CK(cudaMemset(drec, 0, 1 << 20));
    long long h;
    const int iters = 2000;
    for (int bs : {128, 512}) {
        for (size_t smem : {(size_t)0, (size_t)180 * 1024}) {
            CK(cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int it = iters;
            void* args[] = {&it, &dout};
            for (int rep = 0; rep < 2; rep++)
                CK(cudaLaunchCooperativeKernel((void*)k_sync, nsm, bs, args, smem, 0));
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost));
            printf("(a) grid.sync  G=%d bs=%d smem=%zuK: %.3f us/sync\n", nsm, bs, smem / 1024, h / ghz / 1e3 / iters);
        }
    }
    {
        size_t smem = 180 * 1024;
        CK(cudaFuncSetAttribute(k_sync_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int it = iters;
        void* args[] = {&it, &drec, &dsink, &dout};
        for (int rep = 0; rep < 2; rep++)
            CK(cudaLaunchCooperativeKernel((void*)k_sync_reduce, nsm, 512, args, smem, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost));
        printf("(b) publish + grid.sync + read all records: %.3f us/iter\n", h / ghz / 1e3 / iters);
    }
    {
        int it = 4000;
        for (int rep = 0; rep < 2; rep++) k_l2_rtt<<<1, 1>>>(drec, it, dout, dsink);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost));
        printf("(L2) dependent __ldcg chain: %.1f ns/load\n", h / ghz / it);
    }
    {
        CK(cudaFuncSetAttribute(k_cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int it = iters;
        for (int rep = 0; rep < 2; rep++) k_cluster_bar<<<144, 256>>>(it, dout, dsink);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&h, dout, 8, cudaMemcpyDeviceToHost));
        printf("(c) cluster16: 2x barrier.cluster + DSMEM read: %.3f us/iter\n", h / ghz / 1e3 / it);
    }
    {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = 8;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(144);
        cfg.blockDim = dim3(256);
        cfg.attrs = at;
        cfg.numAttrs = 2;
        CK(cudaMemset(dok, 0, 4));
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_coop_cluster, dok);
        cudaError_t e2 = cudaDeviceSynchronize();
        int ok = 0;
        cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
        printf("(d) cooperative + cluster8 launch: launch=%s sync=%s result=%d\n", cudaGetErrorString(e),
               cudaGetErrorString(e2), ok);
        int ncl = 0;
        cudaLaunchConfig_t c2 = cfg;
        c2.numAttrs = 2;
        CK(cudaOccupancyMaxActiveClusters(&ncl, (void*)k_coop_cluster, &c2));
        printf("    max active clusters of 8: %d\n", ncl);
    }
    {
        int it = 100000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        float ms;
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            k_fp64<<<nsm * 4, 256>>>(it, (double*)dsink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)nsm * 4 * 256 * it * 4;
        printf("(e) DFMA: %.2f TFMA/s = %.1f per clk per SM\n", ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3));
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            k_fp64_addmul<<<nsm * 4, 256>>>(it, (double*)dsink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        ops = (double)nsm * 4 * 256 * it * 8;
        printf("(e) DADD+DMUL: %.2f Tops/s = %.1f per clk per SM\n", ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3));
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            k_fp32<<<nsm * 4, 256>>>(it, (float*)dsink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        ops = (double)nsm * 4 * 256 * it * 4;
        printf("(e) FFMA (4 chains/thread): %.2f TFMA/s = %.1f per clk per SM\n", ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3));
    }
    {
        long long* dl;
        double* ds;
        cudaMalloc(&dl, 64);
        cudaMalloc(&ds, 8 * 1024);
        long long hl[3];
        for (int nthr : {32, 512}) {
            for (int rep = 0; rep < 2; rep++) k_lat<<<1, nthr>>>(10000, dl, ds);
            cudaDeviceSynchronize();
            cudaMemcpy(hl, dl, 24, cudaMemcpyDeviceToHost);
            printf("(f) dependent latency, %d threads in 1 CTA: DFMA %.1f clk, DMUL+DADD %.1f clk, FFMA %.1f clk\n", nthr,
                   hl[0] / 10000.0, hl[1] / 10000.0, hl[2] / 10000.0);
        }
    }
    {
        float* dsrc;
        cudaMalloc(&dsrc, 3072 * 4);
        cudaMemset(dsrc, 0, 3072 * 4);
        long long* dl;
        double* ds;
        cudaMalloc(&dl, 64);
        cudaMalloc(&ds, 8 * 1024);
        for (int g = 0; g < 2; g++) {
            long long hl = 0;
            for (int rep = 0; rep < 2; rep++) k_pairs<<<1, 512>>>(dsrc, g, dl, ds);
            cudaDeviceSynchronize();
            cudaMemcpy(&hl, dl, 8, cudaMemcpyDeviceToHost);
            printf("(g) 1024-point farthest pair, 1 CTA x 512 threads, %s: %lld clk = %.1f clk per pair per thread\n",
                   g ? "volatile-generic" : "plain", hl, hl / (523776.0 / 512));
        }
    }
    {
        float* dsrc;
        cudaMalloc(&dsrc, 1024 * 64 * 4);
        std::vector<float> h(1024 * 64);
        for (size_t i = 0; i < h.size(); i++) h[i] = (float)((i * 2654435761u) % 1000) * 0.255f;
        cudaMemcpy(dsrc, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        long long* dl; double* ds;
        cudaMalloc(&dl, 64); cudaMalloc(&ds, 8 * 1024);
        for (int rho : {3, 31}) {
            long long hl = 0;
            cudaFuncSetAttribute(k_rowfar, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * rho * 4);
            for (int rep = 0; rep < 2; rep++) k_rowfar<<<1, 512, 1024 * rho * 4>>>(dsrc, rho, dl, ds);
            cudaDeviceSynchronize();
            cudaMemcpy(&hl, dl, 8, cudaMemcpyDeviceToHost);
            printf("(h) row_farthest, 64 rows of a 1024 sample, rho=%d, 1 CTA x 512: %lld clk = %.2f us\n", rho, hl, hl / ghz / 1e3);
        }
    }
    return 0;
}
