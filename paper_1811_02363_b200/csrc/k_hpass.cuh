// k_hpass.cuh -- F2: row half of the separable convolutions fused with the combine and normalise.
//
// For every cluster k (Algorithm 1 loop for3) and plane q = k(n+1)+c of the
// column-filtered planes t_q produced by F1:
//   v_{k,c}(i) = sum_{t=-R}^{R} w_t t_q(y, x - t)   (row half of omega * u_k),
//   r_k(i)     = same for the b_k plane,
// then  num_c(i) += c_k(i) v_{k,c}(i),  den(i) += c_k(i) r_k(i)  (HDapprox/approxDen)
// and finally g(i) = num(i) / den(i).  Columns outside [0, W) contribute zero (R8).
// Pixels with den < tau omega(0) phi(0) are appended to a list for the direct fallback (R9).
//
// Data movement: one producer lane issues, per cluster k, one 3-D TMA (cp.async.bulk.tensor) of the
// (n+1) planes' tile [n+1][RR][Lbox] (Lbox = 128 + 2 R4 (+4), halo zero-filled by TMA out of bounds)
// and one of the coefficient tile c_k [RR][132] into a multi-stage shared-memory ring guarded by
// full/empty mbarriers.  Consumer warps own (row pair, plane set); a lane owns 8 consecutive pixels
// of one row.  Lbox == 4 (mod 8) floats makes the float4 window loads bank-conflict free
// (a quarter-warp covers 2 rows x 4 chunks).
#pragma once
#include "hdf_common.cuh"

namespace hdf {

constexpr int kHTW = 128;   // columns per CTA tile
constexpr int kHPix = 8;    // consecutive pixels per lane
constexpr int kCoefBox = kHTW + 4;

struct HParams {
    float* g;              // [H][W][n]
    int* flag_count;       // device counter
    int* flag_list;        // [H*W] flagged pixel indices
    int n, NP, H, W, K;
    int RR;                // rows per CTA (even)
    int NJW;               // plane-warps per row pair
    int NWC;               // consumer warps = (RR/2) * NJW
    int NS;                // pipeline stages
    int Lbox;              // inner box length (floats)
    int stage_bytes;       // bytes per stage (planes + coef, 128-aligned parts)
    int planes_bytes;      // bytes of the plane part of a stage
    float tau_floor;       // tau * omega(0) * phi(0); <= 0 disables flagging
    int ytile0;            // first row tile of this launch (the host path launches row chunks)
    float taps[kMaxTaps];
};

template <int R>
constexpr int h_r4() { return (R + 3) & ~3; }

template <int R, int MAXJP, bool BOX>
__global__ void __launch_bounds__(1024, 1)
    k_hpass_combine(const __grid_constant__ CUtensorMap tm_planes, const __grid_constant__ CUtensorMap tm_coef,
                    const __grid_constant__ HParams P) {
    constexpr int R4 = (R + 3) & ~3;
    constexpr int WIN = kHPix + 2 * R4;   // window floats per lane (multiple of 4)
    extern __shared__ __align__(128) unsigned char sm_raw[];
    // 128-byte aligned base (TMA destinations); the launcher adds 128 bytes of slack
    unsigned char* sm_h = sm_raw + ((128u - (smem_u32(sm_raw) & 127u)) & 127u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm_h);
    uint64_t* empty = full + 8;
    float* den_s = reinterpret_cast<float*>(sm_h + 128);          // [RR][128]
    unsigned char* stages = sm_h + 128 + ((P.RR * kHTW * 4 + 127) & ~127);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = blockIdx.x * kHTW, y0 = (blockIdx.y + P.ytile0) * P.RR;

    if (threadIdx.x == 0) {
        prefetch_tmap(&tm_planes);
        prefetch_tmap(&tm_coef);
        for (int s = 0; s < P.NS; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], P.NWC);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == P.NWC) {   // ---------------- producer warp ----------------
        if (lane == 0) {
            for (int k = 0; k < P.K; k++) {
                const int s = k % P.NS, r = k / P.NS;
                if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
                unsigned char* st = stages + (size_t)s * P.stage_bytes;
                mbar_arrive_expect_tx(&full[s], (uint32_t)(P.Lbox * P.RR * P.NP * 4 + kCoefBox * P.RR * 4));
                tma_load_3d(st, &tm_planes, &full[s], x0 - R4, y0, k * P.NP);
                tma_load_3d(st + P.planes_bytes, &tm_coef, &full[s], x0, y0, k);
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    const int npairs = P.RR >> 1;
    const int rp = warp % npairs, jw = warp / npairs;
    const int row = 2 * rp + (lane & 1);
    const int xl = (lane >> 1) * kHPix;
    float acc[MAXJP][kHPix];
#pragma unroll
    for (int a = 0; a < MAXJP; a++)
#pragma unroll
        for (int i = 0; i < kHPix; i++) acc[a][i] = 0.f;

    for (int k = 0; k < P.K; k++) {
        const int s = k % P.NS, r = k / P.NS;
        mbar_wait(&full[s], r & 1);
        const unsigned char* st = stages + (size_t)s * P.stage_bytes;
        const float* cf = reinterpret_cast<const float*>(st + P.planes_bytes) + row * kCoefBox + xl;
        float c[kHPix];
        {
            const float4 c0 = *reinterpret_cast<const float4*>(cf);
            const float4 c1 = *reinterpret_cast<const float4*>(cf + 4);
            c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w;
            c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
        }
#pragma unroll
        for (int a = 0; a < MAXJP; a++) {
            const int j = jw + a * P.NJW;
            if (j < P.NP) {
                const float* base = reinterpret_cast<const float*>(st) + (j * P.RR + row) * P.Lbox + xl;
                float h[kHPix];
                if (BOX) {
                    float w[WIN];
#pragma unroll
                    for (int s4 = 0; s4 < WIN / 4; s4++) {
                        const float4 v = *reinterpret_cast<const float4*>(base + 4 * s4);
                        w[4 * s4] = v.x; w[4 * s4 + 1] = v.y; w[4 * s4 + 2] = v.z; w[4 * s4 + 3] = v.w;
                    }
                    float run = 0.f;
#pragma unroll
                    for (int d = -R; d <= R; d++) run += w[R4 + d];
                    h[0] = run;
#pragma unroll
                    for (int i = 1; i < kHPix; i++) {
                        run = run + w[i + R4 + R] - w[i - 1 + R4 - R];
                        h[i] = run;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < kHPix; i++) h[i] = 0.f;
#pragma unroll
                    for (int s4 = 0; s4 < WIN / 4; s4++) {
                        const float4 v = *reinterpret_cast<const float4*>(base + 4 * s4);
                        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int sidx = 4 * s4 + e;
#pragma unroll
                            for (int i = 0; i < kHPix; i++) {
                                const int d = sidx - i - R4;   // column offset of this value from pixel i
                                if (d >= -R && d <= R) h[i] = fmaf(P.taps[R - d], vv[e], h[i]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < kHPix; i++) acc[a][i] = fmaf(c[i], h[i], acc[a][i]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---------------- epilogue: normalise, flag, store ----------------
    const int nc = P.NWC * 32;
    const int y = y0 + row;
#pragma unroll
    for (int a = 0; a < MAXJP; a++) {
        const int j = jw + a * P.NJW;
        if (j == P.n) {
#pragma unroll
            for (int i = 0; i < kHPix; i++) {
                den_s[row * kHTW + xl + i] = acc[a][i];
                const int x = x0 + xl + i;
                const bool flag = (P.tau_floor > 0.f) && (acc[a][i] < P.tau_floor) && (x < P.W) && (y < P.H);
                const unsigned m = __ballot_sync(__activemask(), flag);
                if (m) {
                    int basei = 0;
                    const int leader = __ffs(m) - 1;
                    if (lane == leader) basei = atomicAdd(P.flag_count, __popc(m));
                    basei = __shfl_sync(__activemask(), basei, leader);
                    if (flag) P.flag_list[basei + __popc(m & ((1u << lane) - 1))] = y * P.W + x;
                }
            }
        }
    }
    named_sync(1, nc);
    // stage g tile [RR][128][n] in the (now idle) ring and write it out coalesced
    float* gst = reinterpret_cast<float*>(stages);
#pragma unroll
    for (int a = 0; a < MAXJP; a++) {
        const int j = jw + a * P.NJW;
        if (j < P.n) {
#pragma unroll
            for (int i = 0; i < kHPix; i++)
                gst[(row * kHTW + xl + i) * P.n + j] = acc[a][i] / den_s[row * kHTW + xl + i];
        }
    }
    named_sync(1, nc);
    const int ncols = min(kHTW, P.W - x0);
    const int seg = ncols * P.n;
    for (int rr = 0; rr < P.RR; rr++) {
        const int yy = y0 + rr;
        if (yy >= P.H) break;
        float* dst = P.g + ((long long)yy * P.W + x0) * P.n;
        const float* src = gst + rr * kHTW * P.n;
        for (int e = threadIdx.x; e < seg; e += nc) dst[e] = src[e];
    }
}

// ---------------------------------------------------------------------------------------------
// F3: direct (num)/(den) for the pixels flagged by rule R9.  One warp per flagged pixel
// (grid-stride over the list, a grid of many warps so that each takes about one pixel): every lane
// takes window taps j, evaluates the weight omega(j) phi(p(i - j) - p(i)) once and accumulates it times
// all n <= NC channels of f(i - j) in registers; warp shuffles reduce den and num; fp32 throughout.
// ---------------------------------------------------------------------------------------------
constexpr int kFbThreads = 256;

struct FBParams {
    const float* f;
    const float* p;
    float* g;
    const int* flag_count;
    const int* flag_list;
    const int* flag_start;     // first list entry to evaluate (device; NULL: 0) -- row chunks of the host path
    int n, rho, H, W, R;
    float neg_inv2sr2;
    float taps[kMaxTaps];
    float neg_inv2ss2;         // != 0: Gaussian spatial weights exp(t^2 neg_inv2ss2) computed in place of
                               // the table (the recursive Gaussian's fallback window beyond kMaxTaps)
    const float* mu;           // hard variant: centres [K][rho] and labels [H*W]: the range kernel is
    const int32_t* labels;     // phi(p(j) - mu_{label(i)}); NULL: phi(p(j) - p(i))
};

template <int NC>   // channels held in registers (n <= NC)
__global__ void __launch_bounds__(kFbThreads) k_fallback(const __grid_constant__ FBParams P) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int cnt = *P.flag_count;
    const int t0 = P.flag_start ? *P.flag_start : 0;
    const int side = 2 * P.R + 1, win = side * side;
    for (int t = t0 + gw; t < cnt; t += nw) {
        const int i = P.flag_list[t];
        const int y = i / P.W, x = i % P.W;
        const float* pi = P.labels ? P.mu + (long long)__ldg(P.labels + i) * P.rho : P.p + (long long)i * P.rho;
        // hard variant: the window's weights are scaled by exp(-d2min / (2 sr^2)) (the ratio is
        // unchanged) so that a window far from its centre does not underflow
        float dmin = 0.f;
        if (P.labels) {
            dmin = INFINITY;
            for (int e = lane; e < win; e += 32) {
                const int ty = e / side - P.R, tx = e % side - P.R;
                const int yy = y - ty, xx = x - tx;
                if (yy < 0 || yy >= P.H || xx < 0 || xx >= P.W) continue;
                const float* pj = P.p + ((long long)yy * P.W + xx) * P.rho;
                float d2 = 0.f;
                for (int d = 0; d < P.rho; d++) {
                    const float dd = __ldg(pj + d) - __ldg(pi + d);
                    d2 = fmaf(dd, dd, d2);
                }
                dmin = fminf(dmin, d2);
            }
            for (int o = 16; o > 0; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        }
        float num[NC];
#pragma unroll
        for (int c = 0; c < NC; c++) num[c] = 0.f;
        float den = 0.f;
        for (int e = lane; e < win; e += 32) {
            const int ty = e / side - P.R, tx = e % side - P.R;
            const int yy = y - ty, xx = x - tx;
            if (yy < 0 || yy >= P.H || xx < 0 || xx >= P.W) continue;
            const long long jj = (long long)yy * P.W + xx;
            const float* pj = P.p + jj * P.rho;
            float d2 = 0.f;
            for (int d = 0; d < P.rho; d++) {
                const float dd = __ldg(pj + d) - __ldg(pi + d);
                d2 = fmaf(dd, dd, d2);
            }
            const float sy = P.neg_inv2ss2 != 0.f ? expf((float)(ty * ty) * P.neg_inv2ss2) : P.taps[ty + P.R];
            const float sx = P.neg_inv2ss2 != 0.f ? expf((float)(tx * tx) * P.neg_inv2ss2) : P.taps[tx + P.R];
            const float wt = sy * sx * expf((d2 - dmin) * P.neg_inv2sr2);
            den += wt;
            const float* fj = P.f + jj * P.n;
#pragma unroll
            for (int c = 0; c < NC; c++)
                if (c < P.n) num[c] = fmaf(wt, __ldg(fj + c), num[c]);
        }
        den = warp_sum(den);
#pragma unroll
        for (int c = 0; c < NC; c++) {
            if (c < P.n) {
                const float v = warp_sum(num[c]);
                if (lane == 0) P.g[(long long)i * P.n + c] = v / den;
            }
        }
    }
}

// Wide images (n > 16 channels, e.g. the 31-band config): one CTA of kFbCtaThreads per flagged pixel
// instead of one warp, the taps spread over the CTA, warp shuffles then one shared-memory pass.
constexpr int kFbCtaThreads = 128;
static __global__ void __launch_bounds__(kFbCtaThreads) k_fallback_cta(const __grid_constant__ FBParams P) {
    __shared__ float red[kFbCtaThreads / 32][HDF_MAX_N + 1];
    __shared__ float pi_s[HDF_MAX_RHO];
    __shared__ float dmin_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cnt = *P.flag_count;
    const int t0 = P.flag_start ? *P.flag_start : 0;
    const int side = 2 * P.R + 1, win = side * side;
    for (int t = t0 + blockIdx.x; t < cnt; t += gridDim.x) {
        const int i = P.flag_list[t];
        const int y = i / P.W, x = i % P.W;
        const float* pi = P.labels ? P.mu + (long long)__ldg(P.labels + i) * P.rho : P.p + (long long)i * P.rho;
        __syncthreads();   // the previous pixel is done with the shared buffers
        for (int d = tid; d < P.rho; d += kFbCtaThreads) pi_s[d] = pi[d];
        __syncthreads();
        // hard variant: the window's weights are scaled by exp(-d2min / (2 sr^2)) (the ratio is
        // unchanged) so that a window far from its centre does not underflow
        float dmin = 0.f;
        if (P.labels) {
            float m = INFINITY;
            for (int e = tid; e < win; e += kFbCtaThreads) {
                const int ty = e / side - P.R, tx = e % side - P.R;
                const int yy = y - ty, xx = x - tx;
                if (yy < 0 || yy >= P.H || xx < 0 || xx >= P.W) continue;
                const float* pj = P.p + ((long long)yy * P.W + xx) * P.rho;
                float d2 = 0.f;
                for (int d = 0; d < P.rho; d++) {
                    const float dd = __ldg(pj + d) - pi_s[d];
                    d2 = fmaf(dd, dd, d2);
                }
                m = fminf(m, d2);
            }
            for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[warp][0] = m;
            __syncthreads();
            if (tid == 0) {
                float mm = red[0][0];
                for (int w = 1; w < kFbCtaThreads / 32; w++) mm = fminf(mm, red[w][0]);
                dmin_s = mm;
            }
            __syncthreads();
            dmin = dmin_s;
        }
        float num[HDF_MAX_N];
#pragma unroll
        for (int c = 0; c < HDF_MAX_N; c++) num[c] = 0.f;
        float den = 0.f;
        for (int e = tid; e < win; e += kFbCtaThreads) {
            const int ty = e / side - P.R, tx = e % side - P.R;
            const int yy = y - ty, xx = x - tx;
            if (yy < 0 || yy >= P.H || xx < 0 || xx >= P.W) continue;
            const long long jj = (long long)yy * P.W + xx;
            const float* pj = P.p + jj * P.rho;
            float d2 = 0.f;
            for (int d = 0; d < P.rho; d++) {
                const float dd = __ldg(pj + d) - pi_s[d];
                d2 = fmaf(dd, dd, d2);
            }
            const float sy = P.neg_inv2ss2 != 0.f ? expf((float)(ty * ty) * P.neg_inv2ss2) : P.taps[ty + P.R];
            const float sx = P.neg_inv2ss2 != 0.f ? expf((float)(tx * tx) * P.neg_inv2ss2) : P.taps[tx + P.R];
            const float wt = sy * sx * expf((d2 - dmin) * P.neg_inv2sr2);
            den += wt;
            const float* fj = P.f + jj * P.n;
#pragma unroll
            for (int c = 0; c < HDF_MAX_N; c++)
                if (c < P.n) num[c] = fmaf(wt, __ldg(fj + c), num[c]);
        }
        // reduce: warps by shuffles, then across warps through shared memory
        den = warp_sum(den);
        if (lane == 0) red[warp][HDF_MAX_N] = den;
#pragma unroll
        for (int c = 0; c < HDF_MAX_N; c++) {
            if (c < P.n) {
                const float v = warp_sum(num[c]);
                if (lane == 0) red[warp][c] = v;
            }
        }
        __syncthreads();
        if (tid < P.n) {
            float a = 0.f, b = 0.f;
            for (int w = 0; w < kFbCtaThreads / 32; w++) {
                a += red[w][tid];
                b += red[w][HDF_MAX_N];
            }
            P.g[(long long)i * P.n + tid] = a / b;
        }
    }
}

}  // namespace hdf
