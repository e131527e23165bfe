// k_vpass.cuh -- F1: fused range weights + vertical pass of the K(n+1) convolutions.
//
// Algorithm 1 loop for1 fused with the column half of the separable convolutions
// v_k = omega * u_k, r_k = omega * b_k:
//   b_k(j) = phi(p(j) - mu_k) = exp(-||p(j) - mu_k||^2 / 2 sigma_r^2),  u_k(j) = b_k(j) f(j),
//   t_q(y, x) = sum_{t=-R}^{R} w_t z_q(y - t, x),  z_q in {u_k channels, b_k}, plane q = k(n+1)+c,
// with rows outside [0, H) contributing zero (window clipped to Omega, R8).
//
// Layout: one CTA owns a 32-column strip x0..x0+31, a row segment [y0, y1) and a group of Pg
// consecutive planes.  It marches down the rows in steps of J rows:
//   phase A (all threads): the J new rows of b/u for the CTA's clusters -> shared staging
//            (double buffered, one barrier per step);
//   phase B (thread = (column, plane)): the J new values enter a register window of S = 2R+J rows
//            that rotates by position (the step loop is unrolled S/J times so every window index is a
//            compile-time register), then J outputs are computed with 2R+1 FFMAs each (taps from the
//            kernel-parameter constant bank) and stored coalesced (32 columns = 128 B per warp).
// Each input value is read from shared memory exactly once; the window never spills.
#pragma once
#include "hdf_common.cuh"

namespace hdf {

constexpr int kVTX = 32;  // columns per CTA (one warp-width)

struct VParams {
    const float* f;        // [H][W][n]
    const float* p;        // [H][W][rho]
    const float* centres;  // [K][rho]
    float* planes;         // [P][H][Wp]
    long long pstride;     // H * Wp
    int n, rho, H, W, Wp, K, NP, P;  // NP = n + 1 planes per cluster, P = K * NP
    int Pg;                // planes per CTA (blockDim.x = 32 * Pg)
    int TY;                // rows per CTA
    float neg_inv2sr2;     // -1 / (2 sigma_r^2)
    float taps[kMaxTaps];  // w_{-R..R} (box: ones)
};

// Phase A: rows [ybase, ybase + J) of b/u for the CTA's planes [q0, q0 + Pg) -> stage[Pg][J][32].
template <int J>
HDF_DEV void vpass_phase_a(const VParams& P, float* __restrict__ stage, const float* __restrict__ mus, int ybase,
                           int x0, int q0, int kA, int nk) {
    const int nitems = nk * J * kVTX;
    for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
        const int tx = it % kVTX;
        const int ri = (it / kVTX) % J;
        const int kl = it / (kVTX * J);
        const int k = kA + kl;
        const int y = ybase + ri, x = x0 + tx;
        const bool valid = (y >= 0) && (y < P.H) && (x < P.W);
        const long long pix = (long long)y * P.W + x;
        float b = 0.f;
        if (valid) {
            const float* pp = P.p + pix * P.rho;
            const float* mu = mus + kl * P.rho;
            float d2 = 0.f;
            for (int d = 0; d < P.rho; d++) {
                float t = __ldg(pp + d) - mu[d];
                d2 = fmaf(t, t, d2);
            }
            b = expf(d2 * P.neg_inv2sr2);
        }
        // planes of cluster k inside [q0, q0 + Pg)
        const int qa = max(k * P.NP, q0), qb = min((k + 1) * P.NP, q0 + P.Pg);
        for (int q = qa; q < qb; q++) {
            const int c = q - k * P.NP;
            float v;
            if (c < P.n) v = valid ? b * __ldg(P.f + pix * P.n + c) : 0.f;
            else v = b;
            stage[((q - q0) * J + ri) * kVTX + tx] = v;
        }
    }
}

template <int R, int J, bool BOX, int NT>
__global__ void __launch_bounds__(NT, 1) k_range_vpass(const __grid_constant__ VParams P) {
    constexpr int S = 2 * R + J;
    constexpr int NSTEP = S / J;
    static_assert(S % J == 0, "J must divide 2R");
    extern __shared__ float sm_v[];
    const int q0 = blockIdx.z * P.Pg;
    const int kA = q0 / P.NP;
    const int kB = min(P.K - 1, (q0 + P.Pg - 1) / P.NP);
    const int nk = kB - kA + 1;
    float* mus = sm_v;                                   // [nk][rho]
    const int mus_len = ((nk * P.rho) + 3) & ~3;
    float* stage0 = sm_v + mus_len;                      // [2][Pg][J][32]
    const int stage_len = P.Pg * J * kVTX;
    for (int e = threadIdx.x; e < nk * P.rho; e += blockDim.x) mus[e] = P.centres[kA * P.rho + e];
    __syncthreads();

    const int tx = threadIdx.x % kVTX;
    const int qi = threadIdx.x / kVTX;
    const int x0 = blockIdx.x * kVTX;
    const int x = x0 + tx;
    const int q = q0 + qi;
    const bool active = (q < P.P) && (x < P.W);
    const int y0 = blockIdx.y * P.TY;
    const int y1 = min(P.H, y0 + P.TY);
    const int ystart = y0 - R;
    const int nsteps = NSTEP - 1 + (y1 - y0 + J - 1) / J;
    float* outp = P.planes + (long long)q * P.pstride + x;

    float win[S];
#pragma unroll
    for (int i = 0; i < S; i++) win[i] = 0.f;

    vpass_phase_a<J>(P, stage0, mus, ystart, x0, q0, kA, nk);
    __syncthreads();
    int g = 0;
    while (true) {
#pragma unroll
        for (int u = 0; u < NSTEP; u++) {
            if (g + 1 < nsteps)
                vpass_phase_a<J>(P, stage0 + ((g + 1) & 1) * stage_len, mus, ystart + (g + 1) * J, x0, q0, kA, nk);
            const float* st = stage0 + (g & 1) * stage_len + qi * J * kVTX + tx;
#pragma unroll
            for (int i = 0; i < J; i++) win[u * J + i] = st[i * kVTX];
            if (g >= NSTEP - 1 && active) {
                const int yb = y0 + (g - NSTEP + 1) * J;
                const int oldest = ((u + 1) % NSTEP) * J;   // window position of logical row 0
                if (BOX) {
                    float acc = 0.f;
#pragma unroll
                    for (int s = 0; s <= 2 * R; s++) acc += win[(oldest + s) % S];
#pragma unroll
                    for (int j = 0; j < J; j++) {
                        if (j > 0) acc = acc + win[(oldest + j + 2 * R) % S] - win[(oldest + j - 1) % S];
                        if (yb + j < y1) outp[(long long)(yb + j) * P.Wp] = acc;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < J; j++) {
                        float acc = 0.f;
#pragma unroll
                        for (int t = -R; t <= R; t++) acc = fmaf(P.taps[t + R], win[(oldest + j + R - t) % S], acc);
                        if (yb + j < y1) outp[(long long)(yb + j) * P.Wp] = acc;
                    }
                }
            }
            __syncthreads();
            g++;
            if (g >= nsteps) return;
        }
    }
}

}  // namespace hdf
