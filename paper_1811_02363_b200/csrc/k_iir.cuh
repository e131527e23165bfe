// Young's recursive Gaussian for the plane convolutions (NEXT #1, the paper's own O(1)
// implementation of the Gaussian steps conv1/conv2).  Readings R17:
//   causal      w[t] = gB x[t] + a1 w[t-1] + a2 w[t-2] + a3 w[t-3], from rest before the first sample;
//   anti-causal y[t] = B w[t] + a1 y[t+1] + a2 y[t+2] + a3 y[t+3], started from the state the
//               zero-input continuation of the causal pass past the last sample gives it:
//               (y[N], y[N+1], y[N+2]) = M (w[N-1], w[N-2], w[N-3]) with M (3x3) computed on the host;
// i.e. the signal is zero outside the image, as under the FIR's clipped window.  gB = G B, with
// G = sqrt(2 pi) sigma so that omega(0) ~ 1 like the FIR's unnormalised taps (rule R9's floor).
// Both kernels work in place on the column pass's plane buffer [P][H][Wp] (the range-weighted planes,
// written unfiltered by k_range_vpass with identity taps), columns first, then rows; the row pass +
// combine kernel then runs with identity taps.  The recursion runs in fp64 (planes stored fp32):
// memory-bound either way, and an fp32 state loses ~sigma^3 x 1e-7 with the poles near 1.
#pragma once
#include "hdf_common.cuh"

namespace hdf {

struct IIRParams {
    float* planes;
    long long pstride;   // H * Wp
    int P, H, W, Wp;
    double gB, B, a1, a2, a3;   // fp64 recursion (the planes stay fp32): with poles near 1 at large
    double M[9];                // sigma an fp32 state loses ~sigma^3 x 1e-7 (measured)
                                // M row-major: y[N + r] = sum_c M[3 r + c] w[N - 1 - c]
};

constexpr int kIirColThreads = 128;
constexpr int kIirBatch = 8;

// one thread per (plane, column): coalesced rows of 128 columns; batches of 8 rows loaded ahead
static __global__ void __launch_bounds__(kIirColThreads) k_iir_cols(const __grid_constant__ IIRParams P) {
    const int x = blockIdx.x * kIirColThreads + threadIdx.x;
    const int q = blockIdx.y;
    if (x >= P.W || q >= P.P) return;
    float* col = P.planes + (long long)q * P.pstride + x;
    const long long s = P.Wp;
    double w1 = 0.0, w2 = 0.0, w3 = 0.0;
    int y = 0;
    for (; y + kIirBatch <= P.H; y += kIirBatch) {
        float v[kIirBatch];
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) v[i] = col[(y + i) * s];
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) {
            const double w = fma(P.gB, (double)v[i], fma(P.a1, w1, fma(P.a2, w2, P.a3 * w3)));
            w3 = w2; w2 = w1; w1 = w;
            v[i] = (float)w;
        }
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) col[(y + i) * s] = v[i];
    }
    for (; y < P.H; y++) {
        const double w = fma(P.gB, (double)col[y * s], fma(P.a1, w1, fma(P.a2, w2, P.a3 * w3)));
        w3 = w2; w2 = w1; w1 = w;
        col[y * s] = (float)w;
    }
    double y1 = P.M[0] * w1 + P.M[1] * w2 + P.M[2] * w3;   // y[N]
    double y2 = P.M[3] * w1 + P.M[4] * w2 + P.M[5] * w3;   // y[N+1]
    double y3 = P.M[6] * w1 + P.M[7] * w2 + P.M[8] * w3;   // y[N+2]
    y = P.H - 1;
    for (; y + 1 - kIirBatch >= 0; y -= kIirBatch) {
        float v[kIirBatch];
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) v[i] = col[(y - i) * s];
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) {
            const double o = fma(P.B, (double)v[i], fma(P.a1, y1, fma(P.a2, y2, P.a3 * y3)));
            y3 = y2; y2 = y1; y1 = o;
            v[i] = (float)o;
        }
#pragma unroll
        for (int i = 0; i < kIirBatch; i++) col[(y - i) * s] = v[i];
    }
    for (; y >= 0; y--) {
        const double o = fma(P.B, (double)col[y * s], fma(P.a1, y1, fma(P.a2, y2, P.a3 * y3)));
        y3 = y2; y2 = y1; y1 = o;
        col[y * s] = (float)o;
    }
}

// one warp per (plane, 32 rows): 32 x 32 tiles staged through shared memory (coalesced row loads and
// stores), lane r runs the recursion along row r of the tile
static __global__ void __launch_bounds__(32) k_iir_rows(const __grid_constant__ IIRParams P) {
    __shared__ float t[32][33];
    const int lane = threadIdx.x;
    const int r0 = blockIdx.x * 32, q = blockIdx.y;
    float* base = P.planes + (long long)q * P.pstride;
    const int nr = min(32, P.H - r0);
    auto load = [&](int c0, int nc) {
        for (int r = 0; r < nr; r++) t[r][lane] = lane < nc ? base[(long long)(r0 + r) * P.Wp + c0 + lane] : 0.f;
        __syncwarp();
    };
    auto store = [&](int c0, int nc) {
        __syncwarp();
        for (int r = 0; r < nr; r++)
            if (lane < nc) base[(long long)(r0 + r) * P.Wp + c0 + lane] = t[r][lane];
        __syncwarp();
    };
    double w1 = 0.0, w2 = 0.0, w3 = 0.0;
    for (int c0 = 0; c0 < P.W; c0 += 32) {
        const int nc = min(32, P.W - c0);
        load(c0, nc);
        for (int c = 0; c < nc; c++) {
            const double w = fma(P.gB, (double)t[lane][c], fma(P.a1, w1, fma(P.a2, w2, P.a3 * w3)));
            w3 = w2; w2 = w1; w1 = w;
            t[lane][c] = (float)w;
        }
        store(c0, nc);
    }
    double y1 = P.M[0] * w1 + P.M[1] * w2 + P.M[2] * w3;
    double y2 = P.M[3] * w1 + P.M[4] * w2 + P.M[5] * w3;
    double y3 = P.M[6] * w1 + P.M[7] * w2 + P.M[8] * w3;
    for (int c0 = ((P.W - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
        const int nc = min(32, P.W - c0);
        load(c0, nc);
        for (int c = nc - 1; c >= 0; c--) {
            const double o = fma(P.B, (double)t[lane][c], fma(P.a1, y1, fma(P.a2, y2, P.a3 * y3)));
            y3 = y2; y2 = y1; y1 = o;
            t[lane][c] = (float)o;
        }
        store(c0, nc);
    }
}

}  // namespace hdf
