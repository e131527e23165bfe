// Micro-benchmark (design calibration, not product code): cost of one Lloyd pass of k_bisect
// (pass_small<3>) over a resident shared-memory tile of T points in one 512-thread CTA, and of the
// per-iteration block reduction that follows it.  Late-iteration regime (no point moves) and
// first-iteration regime (every point "moves").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1811_02363_b200/csrc \
//      microbench/mb_pass.cu -o /tmp/mb_pass
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <cuda_runtime.h>
#include "k_bisect.cuh"
using namespace hdf;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

constexpr int REPS = 64;

// Variants of pass_small for timing (ONE1: one FMA per dimension, D = sum (2w) x - C; U points per step)
template <int RHO, int U, bool ONE1>
__device__ void pass_var(const float* X, int tn, const uint32_t* prevW, uint32_t* curW, bool cmp, bool full,
                         const SplitSm& S, double (&s1)[RHO], int& n1, int& chg) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float wt[RHO], mt[RHO], bound;
    lin_consts<RHO>(S, wt, mt, bound);
    float w2[RHO], C = 0.f;
#pragma unroll
    for (int d = 0; d < RHO; d++) { w2[d] = 2.f * wt[d]; C = fmaf(wt[d], mt[d], C); }
    for (int j0 = 0; j0 < tn; j0 += U * kBT) {
        float x[U][RHO];
        bool sd[U], cert[U];
        uint32_t pw[U];
        bool allc = true;
#pragma unroll
        for (int h = 0; h < U; h++) {
            const int wi = (j0 >> 5) + h * kBW + warp;
            const bool has = j0 + h * kBT < tn;
            pw[h] = (cmp && has) ? prevW[wi] : 0u;
            const int j = j0 + h * kBT + tid;
            const bool ok = j < tn;
            float D = ONE1 ? -C : 0.f;
#pragma unroll
            for (int d = 0; d < RHO; d++) {
                x[h][d] = ok ? lds_f(X + (size_t)j * RHO + d) : 0.f;
                if (ONE1) D = fmaf(w2[d], x[h][d], D);
                else D = fmaf(wt[d], fmaf(2.0f, x[h][d], -mt[d]), D);
            }
            cert[h] = !ok || fabsf(D) > bound;
            sd[h] = ok && D > 0.f;
            allc = allc && cert[h];
        }
        if (__ballot_sync(0xffffffffu, !allc)) {
#pragma unroll
            for (int h = 0; h < U; h++) {
                if (!cert[h]) {
                    double dd0 = 0.0, dd1 = 0.0;
#pragma unroll
                    for (int d = 0; d < RHO; d++) {
                        const double v = (double)x[h][d];
                        dd0 = d2_rn(dd0, v, S.c0[d]);
                        dd1 = d2_rn(dd1, v, S.c1[d]);
                    }
                    sd[h] = !(dd0 <= dd1);
                }
            }
        }
        uint32_t anym = 0;
        uint32_t mk[U];
#pragma unroll
        for (int h = 0; h < U; h++) {
            const uint32_t w = __ballot_sync(0xffffffffu, sd[h]);
            const bool has = j0 + h * kBT < tn;
            if (lane == 0 && has) curW[(j0 >> 5) + h * kBW + warp] = w;
            if (cmp) chg += __popc(w ^ pw[h]);
            n1 += __popc(w);
            mk[h] = full ? w : (w ^ pw[h]);
            anym |= mk[h];
        }
        if (anym) {
#pragma unroll
            for (int h = 0; h < U; h++) {
                const double k = ((mk[h] >> lane) & 1u) ? (sd[h] ? 1.0 : -1.0) : 0.0;
#pragma unroll
                for (int d = 0; d < RHO; d++) s1[d] = fma(k, (double)x[h][d], s1[d]);
            }
        }
    }
}

template <int VARIANT>
__global__ void __launch_bounds__(kBT, 1) mb(const float* P, int T, long long* out, double* sink, int moving) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ SplitSm S;
    float* X = reinterpret_cast<float*>(dyn);
    uint32_t* W0 = reinterpret_cast<uint32_t*>(X + T * 3);
    uint32_t* W1 = W0 + T / 32 + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < T * 3; i += kBT) X[i] = P[i];
    for (int i = tid; i < T / 32 + 2; i += kBT) { W0[i] = 0; W1[i] = 0; }
    if (tid < 3) {
        S.c0[tid] = 60.0 + 10 * tid;
        S.c1[tid] = 190.0 - 5 * tid;
        S.xmax[tid] = 255.f;
    }
    __syncthreads();
    set_lin(S, 3);
    __syncthreads();
    double s1p[3] = {0, 0, 0}, stp[3] = {0, 0, 0};
    long long tp = 0, tr = 0;
    for (int rep = 0; rep < REPS; rep++) {
        uint32_t* curW = (rep & 1) ? W1 : W0;
        const uint32_t* prevW = (rep & 1) ? W0 : W1;
        int n1 = 0, chg = 0;
        __syncthreads();
        const long long t0 = clock64();
        if (VARIANT == 0) pass_small<3, false>(X, T, WordsSm{smem_pin(prevW), smem_pin(curW)}, rep > 0, moving != 0, S, s1p, stp, n1, chg);
        if (VARIANT == 1) pass_var<3, 4, true>(X, T, prevW, curW, rep > 0, moving != 0, S, s1p, n1, chg);
        if (VARIANT == 2) pass_var<3, 8, false>(X, T, prevW, curW, rep > 0, moving != 0, S, s1p, n1, chg);
        if (VARIANT == 3) pass_var<3, 8, true>(X, T, prevW, curW, rep > 0, moving != 0, S, s1p, n1, chg);
        if (VARIANT == 4) pass_var<3, 2, false>(X, T, prevW, curW, rep > 0, moving != 0, S, s1p, n1, chg);
        __syncthreads();
        const long long t1 = clock64();
        double vv[16];
#pragma unroll
        for (int q = 0; q < 16; q++) vv[q] = 0.0;
#pragma unroll
        for (int q = 0; q < 3; q++) vv[3 + q] = s1p[q];
        vv[6] = (lane == 0) ? (double)n1 : 0.0;
        vv[7] = (lane == 0) ? (double)chg : 0.0;
        const int vi = warp_reduce_scatter16(vv);
        if ((lane & 1) == 0) S.red[warp * 16 + vi] = vv[0];
        __syncthreads();
        if (warp == 0 && lane < 8) {
            double ts = 0.0;
            for (int w = 0; w < kBW; w++) ts += S.red[w * 16 + lane];
            S.tot[lane] = ts;
        }
        __syncthreads();
        const long long t2 = clock64();
        tp += t1 - t0;
        tr += t2 - t1;
    }
    if (tid == 0) { out[0] = tp / REPS; out[1] = tr / REPS; }
    if (tid < 8) sink[tid] = S.tot[tid];
}

int main(int argc, char** argv) {
    const int only_var = argc > 1 ? atoi(argv[1]) : -1, only_T = argc > 2 ? atoi(argv[2]) : -1;
    const int Ts[] = {512, 1024, 2048, 4096, 8192, 16384};
    std::vector<float> h(16384 * 3);
    unsigned s = 12345;
    for (auto& v : h) { s = s * 1664525u + 1013904223u; v = (float)((s >> 8) % 25500) / 100.f; }
    float* dP;
    long long* dO;
    double* dS;
    CK(cudaMalloc(&dP, h.size() * 4));
    CK(cudaMalloc(&dO, 16));
    CK(cudaMalloc(&dS, 64));
    CK(cudaMemcpy(dP, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    void (*ks[5])(const float*, int, long long*, double*, int) = {mb<0>, mb<1>, mb<2>, mb<3>, mb<4>};
    for (int var = 0; var < 5; var++)
    for (int moving = 0; moving < 2; moving++)
        for (int T : Ts) {
            if ((only_var >= 0 && var != only_var) || (only_T >= 0 && T != only_T)) continue;
            const size_t smem = (size_t)T * 12 + (T / 32 + 2) * 8;
            CK(cudaFuncSetAttribute(ks[var], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            ks[var]<<<1, kBT, smem>>>(dP, T, dO, dS, moving);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            long long o[2];
            CK(cudaMemcpy(o, dO, 16, cudaMemcpyDeviceToHost));
            printf("var=%d moving=%d T=%5d pass %6lld cyc (%.2f cyc/pt/warp-slot)  reduce %5lld cyc\n", var, moving, T, o[0],
                   (double)o[0] * 4 / T, o[1]);
        }
    return 0;
}
