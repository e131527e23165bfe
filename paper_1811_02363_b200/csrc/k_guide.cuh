// k_guide.cuh -- on-GPU PCA-NLM guide (reading R11).
//
// p(i) = the m x m patch of f around i (all n channels, D = n m^2 values in (channel, dy, dx) order,
// replicate borders), centred on the mean patch and projected on the `dim` leading eigenvectors of
// the patch covariance (PCA-NLM).  Eigenvectors in descending eigenvalue order, each signed so
// that its entry of largest magnitude is positive (the oracle's convention, oracle.pca_guide).
//
//   k_pca_moments   per-CTA fp64 sums of x and of the upper triangle of x x^T over a contiguous
//                   pixel range (patches staged in shared memory, products exact in fp64)
//   k_pca_eig       one CTA: the partial sums in a fixed order, C = S2 / N - mean mean^T, cyclic
//                   Jacobi (one warp, fp64), sort, sign, basis (fp32) and mean
//   k_pca_project   one thread per pixel: (patch - mean) . basis_j, j < dim
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hdf_common.cuh"

namespace hdf {

constexpr int kPcaMaxD = 64;        // n m^2 <= 64
constexpr int kPcaMaxDim = 32;      // projected dimensions
constexpr int kPcaThreads = 256;
constexpr int kPcaTile = 128;       // pixels staged per step of k_pca_moments
constexpr int kPcaGrid = 296;       // CTAs of k_pca_moments (fixed: the partial-sum buffer)

HDF_DEV int pca_nent(int D) { return D + D * (D + 1) / 2; }   // sums of x, then x_a x_b (a <= b)

// patch value d of pixel (y, x): channel c, offset (dy, dx), replicate borders
HDF_DEV float pca_patch(const float* f, int H, int W, int n, int m, int y, int x, int d) {
    const int mm = m * m, r = m / 2;
    const int c = d / mm, o = d - c * mm, dy = o / m - r, dx = o % m - r;
    const int yy = min(max(y + dy, 0), H - 1), xx = min(max(x + dx, 0), W - 1);
    return __ldg(f + ((long long)yy * W + xx) * n + c);
}

__global__ void __launch_bounds__(kPcaThreads) k_pca_moments(const float* f, int H, int W, int n, int m,
                                                             double* part) {
    __shared__ float X[kPcaTile * kPcaMaxD];
    const int D = n * m * m, E = pca_nent(D);
    const long long N = (long long)H * W;
    const long long per = (N + gridDim.x - 1) / gridDim.x;
    const long long b0 = min(N, (long long)blockIdx.x * per), b1 = min(N, b0 + per);
    constexpr int NQ = (kPcaMaxD + kPcaMaxD * (kPcaMaxD + 1) / 2 + kPcaThreads - 1) / kPcaThreads;
    double acc[NQ];   // entries tid + kPcaThreads * q
    int ea[NQ], eb[NQ];
#pragma unroll
    for (int q = 0; q < NQ; q++) {
        acc[q] = 0.0;
        int e = threadIdx.x + kPcaThreads * q, a = -1, b = -1;
        if (e < D) {
            a = e;   // sum of x_a (b = -1)
        } else if (e < E) {
            e -= D;   // (a, b), a <= b, row-major upper triangle
            a = 0;
            while (e >= D - a) { e -= D - a; a++; }
            b = a + e;
        } else {
            a = -2;
        }
        ea[q] = a;
        eb[q] = b;
    }
    for (long long t0 = b0; t0 < b1; t0 += kPcaTile) {
        const int tn = (int)min((long long)kPcaTile, b1 - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < tn * D; e += kPcaThreads) {
            const int p = e / D, d = e - p * D;
            const long long i = t0 + p;
            const int y = (int)(i / W), x = (int)(i - (long long)y * W);
            X[p * kPcaMaxD + d] = pca_patch(f, H, W, n, m, y, x, d);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            const int a = ea[q], b = eb[q];
            if (a < 0) continue;
            double s0 = 0.0, s1 = 0.0;   // two chains
            if (b < 0) {
                for (int p = 0; p < tn; p += 2) {
                    s0 += (double)X[p * kPcaMaxD + a];
                    if (p + 1 < tn) s1 += (double)X[(p + 1) * kPcaMaxD + a];
                }
            } else {
                for (int p = 0; p < tn; p += 2) {
                    s0 = fma((double)X[p * kPcaMaxD + a], (double)X[p * kPcaMaxD + b], s0);
                    if (p + 1 < tn) s1 = fma((double)X[(p + 1) * kPcaMaxD + a], (double)X[(p + 1) * kPcaMaxD + b], s1);
                }
            }
            acc[q] += s0 + s1;
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; q++) {
        const int e = threadIdx.x + kPcaThreads * q;
        if (e < E) part[(size_t)blockIdx.x * E + e] = acc[q];
    }
}

struct PcaOut {
    float* basis;    // [dim][D]
    float* mean;     // [D]
    double* evals;   // [dim]
};

// One CTA of kPcaThreads threads.  Dynamic shared memory (pca_eig_smem): C [D][D], V [D][D], mean (fp64).
constexpr int kPcaLd = kPcaMaxD + 1;   // row stride of C and V (odd: column walks hit distinct banks)
constexpr size_t pca_eig_smem() { return sizeof(double) * (2 * kPcaMaxD * kPcaLd + kPcaMaxD); }
__global__ void __launch_bounds__(kPcaThreads) k_pca_eig(const double* part, int G, int D, int dim, long long N,
                                                         PcaOut out) {
    extern __shared__ __align__(16) double pca_sm[];
    double* C = pca_sm;
    double* V = C + kPcaMaxD * kPcaLd;
    double* mu = V + kPcaMaxD * kPcaLd;
    __shared__ int sel[kPcaMaxDim];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int E = pca_nent(D);
    // partial sums of the CTAs: one warp per entry, lanes over CTAs (all loads in flight), then a
    // fixed butterfly (the same order in every run)
    for (int e = warp; e < E; e += kPcaThreads / 32) {
        double s = 0.0;
        for (int g = lane; g < G; g += 32) s += part[(size_t)g * E + e];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane != 0) continue;
        if (e < D) {
            mu[e] = s / (double)N;
        } else {
            int r = e - D, a = 0;
            while (r >= D - a) { r -= D - a; a++; }
            C[a * kPcaLd + a + r] = s / (double)N;   // E[x_a x_b], b = a + r
        }
    }
    __syncthreads();
    for (int e = tid; e < D * D; e += kPcaThreads) {
        const int a = e / D, b = e - a * D;
        if (a <= b) {
            const double c = C[a * kPcaLd + b] - mu[a] * mu[b];
            C[a * kPcaLd + b] = c;
            if (a != b) C[b * kPcaLd + a] = c;
        }
        V[a * kPcaLd + b] = (a == b) ? 1.0 : 0.0;
    }
    __syncthreads();
    // Parallel (round-robin) Jacobi: each step rotates D'/2 disjoint pairs at once (D' = D rounded up
    // to even; index D' - 1 >= D is a dummy): column rotations for all pairs, then row rotations,
    // then the next pairing; D' - 1 steps per sweep.  The pairings are tabulated once, and in the update
    // phases warp w takes the pairs w, w + 8, .. with lane = matrix row (or column): no integer division
    // or modulo per element (they were most of the ~3.3 us per step of the first version).
    __shared__ double rc[kPcaMaxD / 2], rs[kPcaMaxD / 2];
    __shared__ unsigned char pp[kPcaMaxD - 1][kPcaMaxD / 2], pq[kPcaMaxD - 1][kPcaMaxD / 2];
    __shared__ int done;
    const int Dp = (D + 1) & ~1, np = Dp / 2;
    constexpr int NW = kPcaThreads / 32;
    for (int e = tid; e < (Dp - 1) * np; e += kPcaThreads) {
        const int step = e / np, i = e - step * np;
        // round robin: position 0 holds index 0, position k >= 1 holds 1 + (k - 1 + step) mod (Dp - 1);
        // pair i = (positions i, Dp - 1 - i)
        auto ring = [&](int k) { return k == 0 ? 0 : 1 + (k - 1 + step) % (Dp - 1); };
        int p = ring(i), q = ring(Dp - 1 - i);
        if (p > q) { const int t = p; p = q; q = t; }
        pp[step][i] = (unsigned char)p;
        pq[step][i] = (unsigned char)q;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 60; sweep++) {
        if (warp == 0) {
            double off = 0.0, fro = 0.0;
            for (int a = 0; a < D; a++)
                for (int b = lane; b < D; b += 32) {
                    const double v = C[a * kPcaLd + b];
                    fro += v * v;
                    if (a != b) off += v * v;
                }
            for (int o = 16; o > 0; o >>= 1) {
                off += __shfl_xor_sync(0xffffffffu, off, o);
                fro += __shfl_xor_sync(0xffffffffu, fro, o);
            }
            // converged when the off-diagonal part is ~1e-13 of the whole (fp64 cannot go much lower
            // than D eps; the fp32 guide needs far less)
            if (lane == 0) done = !(off > 1e-26 * fro);
        }
        __syncthreads();
        if (done) break;
        for (int step = 0; step < Dp - 1; step++) {
            for (int i = tid; i < np; i += kPcaThreads) {   // the step's rotation angles
                const int p = pp[step][i], q = pq[step][i];
                double c = 1.0, sn = 0.0;
                if (q < D) {
                    const double apq = C[p * kPcaLd + q];
                    if (apq != 0.0) {
                        // the angle in fp32 (an inexact angle only slows the last sweeps down), the
                        // rotation itself in fp64 and exactly orthogonal to rounding: c from one Newton
                        // step of 1/sqrt(1 + t^2) seeded in fp32, s = t c
                        // (tau itself in fp32 too: an fp64 division is a long dependent chain per step)
                        const float tau = (float)(C[q * kPcaLd + q] - C[p * kPcaLd + p]) / (2.0f * (float)apq);
                        const float tf = copysignf(1.0f, tau) / (fabsf(tau) + sqrtf(fmaf(tau, tau, 1.0f)));
                        const double t = (double)tf, u = fma(t, t, 1.0);
                        double r = (double)rsqrtf((float)u);
                        r = r * fma(-0.5 * u, r * r, 1.5);
                        r = r * fma(-0.5 * u, r * r, 1.5);
                        c = r;
                        sn = t * r;
                    }
                }
                rc[i] = c;
                rs[i] = sn;
            }
            __syncthreads();
            for (int i = warp; i < np; i += NW) {   // columns p, q of C and V: lane = row k
                const double sn = rs[i];
                const int p = pp[step][i], q = pq[step][i];
                if (q >= D || sn == 0.0) continue;
                const double c = rc[i];
                for (int k = lane; k < D; k += 32) {
                    const double akp = C[k * kPcaLd + p], akq = C[k * kPcaLd + q];
                    C[k * kPcaLd + p] = c * akp - sn * akq;
                    C[k * kPcaLd + q] = sn * akp + c * akq;
                    const double vkp = V[k * kPcaLd + p], vkq = V[k * kPcaLd + q];
                    V[k * kPcaLd + p] = c * vkp - sn * vkq;
                    V[k * kPcaLd + q] = sn * vkp + c * vkq;
                }
            }
            __syncthreads();
            for (int i = warp; i < np; i += NW) {   // rows p, q (all columns k): lane = column k
                const double sn = rs[i];
                const int p = pp[step][i], q = pq[step][i];
                if (q >= D || sn == 0.0) continue;
                const double c = rc[i];
                for (int k = lane; k < D; k += 32) {
                    const double apk = C[p * kPcaLd + k], aqk = C[q * kPcaLd + k];
                    C[p * kPcaLd + k] = c * apk - sn * aqk;
                    C[q * kPcaLd + k] = sn * apk + c * aqk;
                }
            }
            __syncthreads();
        }
    }
    if (warp == 0) {
        // the dim largest eigenvalues, descending (ties -> lower index)
        if (lane == 0) {
            unsigned long long used = 0ull;
            for (int j = 0; j < dim; j++) {
                int bi = -1;
                for (int k = 0; k < D; k++)
                    if (!((used >> k) & 1ull) && (bi < 0 || C[k * kPcaLd + k] > C[bi * kPcaLd + bi])) bi = k;
                used |= 1ull << bi;
                sel[j] = bi;
            }
        }
        __syncwarp();
    }
    __syncthreads();
    for (int j = warp; j < dim; j += kPcaThreads / 32) {
        const int col = sel[j];
        // sign: entry of largest magnitude positive (ties -> first)
        double best = -1.0, val = 0.0;
        int bk = D;
        for (int k = lane; k < D; k += 32) {
            const double v = V[k * kPcaLd + col];
            if (fabs(v) > best) { best = fabs(v); val = v; bk = k; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const double ov = __shfl_xor_sync(0xffffffffu, val, o);
            const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            if (ob > best || (ob == best && ok < bk)) { best = ob; val = ov; bk = ok; }
        }
        const double sg = val < 0.0 ? -1.0 : 1.0;
        for (int k = lane; k < D; k += 32) out.basis[j * D + k] = (float)(sg * V[k * kPcaLd + col]);
        if (lane == 0) out.evals[j] = C[col * kPcaLd + col];
    }
    for (int d = tid; d < D; d += kPcaThreads) out.mean[d] = (float)mu[d];
}

template <int DIMT>
__global__ void __launch_bounds__(kPcaThreads) k_pca_project(const float* f, int H, int W, int n, int m, int dim,
                                                             const float* basis, const float* mean, float* p) {
    __shared__ float Bs[kPcaMaxDim * kPcaMaxD];
    __shared__ float Ms[kPcaMaxD];
    const int D = n * m * m;
    for (int e = threadIdx.x; e < dim * D; e += kPcaThreads) Bs[e] = basis[e];
    for (int e = threadIdx.x; e < D; e += kPcaThreads) Ms[e] = mean[e];
    __syncthreads();
    const long long N = (long long)H * W;
    for (long long i = (long long)blockIdx.x * kPcaThreads + threadIdx.x; i < N;
         i += (long long)gridDim.x * kPcaThreads) {
        const int y = (int)(i / W), x = (int)(i - (long long)y * W);
        float acc[DIMT];
#pragma unroll
        for (int j = 0; j < DIMT; j++) acc[j] = 0.f;
        for (int d = 0; d < D; d++) {
            const float v = pca_patch(f, H, W, n, m, y, x, d) - Ms[d];
#pragma unroll
            for (int j = 0; j < DIMT; j++)
                if (j < dim) acc[j] = fmaf(v, Bs[j * D + d], acc[j]);
        }
        float* o = p + i * dim;
#pragma unroll
        for (int j = 0; j < DIMT; j++)
            if (j < dim) o[j] = acc[j];
    }
}

// ---------------------------------------------------------------------------------------------
// Anisotropic / augmented guides: the diagonal range kernel
// phi(x) = exp(-sum_d x_d^2 / 2 sigma_d^2) equals the isotropic kernel with sigma_r = 1 on the guide
// scaled per channel by s_d = 1 / sigma_d, and an extra guide channel (e.g. an infrared band, P:672-
// 679) is appended with its own scale.  out(i) = (p(i)_d s_d)_{d < rho} ++ (extra(i)_j t_j)_{j < e}.
// One thread per output element, coalesced over the flat [H*W][rho + e] output.
struct ScaleParams {
    const float* p;        // [N][rho]
    const float* extra;    // [N][e] or NULL
    float* out;            // [N][rho + e]
    long long N;
    int rho, e;
    float s[HDF_MAX_RHO];  // per-channel scales: s_0..s_{rho-1}, then t_0..t_{e-1}
};

__global__ void __launch_bounds__(256) k_scale_guide(const __grid_constant__ ScaleParams P) {
    const int D = P.rho + P.e;
    const long long tot = P.N * D;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const long long i = t / D;
        const int d = (int)(t - i * D);
        const float v = d < P.rho ? __ldg(P.p + i * P.rho + d) : __ldg(P.extra + i * P.e + (d - P.rho));
        P.out[t] = v * P.s[d];
    }
}

// ---------------------------------------------------------------------------------------------
// Stride sample of the guide for the sampled clustering mode ("any efficient clustering
// method" may replace the exact procedure): out[j] = p[i0 + j * stride], j < M (rho floats each).
__global__ void __launch_bounds__(256) k_sample_guide(const float* __restrict__ p, int rho, long long i0,
                                                      long long stride, float* __restrict__ out, long long M) {
    const long long tot = M * rho;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const long long j = t / rho;
        const int d = (int)(t - j * rho);
        out[t] = __ldg(p + (i0 + j * stride) * rho + d);
    }
}

}  // namespace hdf
