// k_vpass_tc.cuh -- F1 on the 5th-generation tensor cores: range weights + the column half of the
// Gaussian convolutions (Algorithm 1 loop for1 + the column pass of loop for3, P:281-288, P:297-302,
// P:309-312) for colour images (n + 1 = 4 planes per cluster), as a banded (Toeplitz) product:
//
//   t_q(y0 + j, x) = sum_{i=0}^{Kp-1} T[j][i] z_q(y0 - R + i, x),   T[j][i] = w_{i - j - R} (0 outside [-R, R]),
//
// for a tile of 64 output rows j and M = 128 (plane, column) pairs: D[M x 64] = Z[M x Kp] . T^T[Kp x 64]
// with tcgen05.mma kind::f16 (fp32 accumulation in TMEM), Kp = round_up(64 + 2R, 16) input rows.  The
// rows outside [0, H) contribute zero (R8).
//
// Precision (fp32-level): fp16 operands split in two, x = hi + lo (hi = fp16(x), lo = fp16(x - hi),
// ~22 significant bits together), D = z_lo T_hi + z_hi T_lo + z_hi T_hi.  The planes are scaled by
// powers of two into fp16's normal range before the split and scaled back exactly in the epilogue:
// the b planes by 2^14 (b <= 1), the b f planes by 2^(14 - e) with 2^e >= max |f| (a device-side
// reduction, k_absmax, so any finite image works).
//
// One CTA per SM (persistent over (32-column strip, cluster) columns x row segments, in tiles of 64
// output rows), warp-specialised and double-buffered:
//   * producers (warpgroup 0): per tile, z for the Kp input rows of the strip's 32 columns and the
//     cluster's 4 planes (b_k = exp2(-|p - mu_k|^2 log2(e) / 2 sigma_r^2), u_k = b_k f), split, stored
//     into the A stage in the canonical K-major no-swizzle layout (8 x 16-byte core matrices; one
//     16-byte store = 8 consecutive rows of one (plane, column)); arrive on "A full";
//   * MMA warp (one thread): waits "A full" and "D free", issues 3 Kp/16 MMAs (M = 128, N = 64, K = 16),
//     commits to "A free" and "D full";
//   * consumers (warpgroup 1, TMEM lane quarter = plane): load the 64 output rows of their (plane,
//     column) from TMEM, release the stage, scale back and store (coalesced over the 32 columns).
// The Toeplitz operand T (hi, lo) is staged once per CTA.
#pragma once
#include <cuda_fp16.h>

#include "hdf_common.cuh"
#include "k_coeffs_tc.cuh"
#include "k_vpass.cuh"

namespace hdf {

constexpr int kVtcRows = 64;       // output rows per tile (UMMA N)
constexpr int kVtcM = 128;         // (plane, column) pairs per tile (UMMA M): 4 planes x 32 columns
constexpr int kVtcThreads = 288;   // producers 128 + consumers 128 + MMA warp 32

inline __host__ __device__ int vtc_kp(int R) { return ((kVtcRows + 2 * R) + 15) & ~15; }
// Dynamic shared memory: T_hi, T_lo [64][Kp] and two stages of Z_hi, Z_lo [128][Kp] (fp16)
inline __host__ __device__ size_t vpass_tc_smem(int R) {
    const int Kp = vtc_kp(R);
    return (size_t)2 * kVtcRows * Kp * 2 + (size_t)4 * kVtcM * Kp * 2 + 64;
}

struct VtcParams {
    const float* f;        // [H][W][3]
    const float* p;        // [H][W][RHO]
    const float* centres;  // [K][RHO]
    float* planes;         // [4K][H][Wp]
    const int* absmax;     // max |f| as float bits (k_absmax)
    long long pstride;     // H * Wp
    int H, W, Wp, K, R;
    int nstrip, nseg, seglen;   // 32-column strips, row segments per column and their length
    float neg_inv2sr2;     // -1 / (2 sigma_r^2)
    float taps[kMaxTaps];  // w_{-R..R}
};

// max |x| over count floats -> *out (float bits, non-negative floats order as integers); *out = 0 first
__global__ void __launch_bounds__(256) k_absmax(const float* __restrict__ x, long long count, int* out) {
    float m = 0.f;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(__ldg(x + i)));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_int(m));
}

HDF_DEV uint32_t umma_idesc_f16(int M, int N) {   // kind::f16: D fp32, A and B fp16, K-major
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
HDF_DEV void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// fp16 hi/lo split of x: hi = fp16(x), lo = fp16(x - hi)
HDF_DEV void split_f16(float x, unsigned short& hi, unsigned short& lo) {
    const __half h = __float2half_rn(x);
    hi = __half_as_ushort(h);
    lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
}

// Byte offset of (row r, k) in an operand of nrow rows (multiple of 8) and Kp columns, K-major, no
// swizzle, layout "m-groups adjacent": core matrix (r / 8, k / 8) at (k / 8) * (nrow * 16) + (r / 8) * 128.
HDF_DEV uint32_t vtc_off(int r, int k, int nrow) {
    return (uint32_t)((k >> 3) * (nrow * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

template <int RHO>
__global__ void __launch_bounds__(kVtcThreads, 1) k_range_vpass_tc(const __grid_constant__ VtcParams P) {
    extern __shared__ __align__(128) unsigned char sm_vt[];
    __shared__ uint64_t a_full[2], a_free[2], d_full[2], d_free[2];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = P.R, Kp = vtc_kp(R);
    const size_t tbytes = (size_t)kVtcRows * Kp * 2, zbytes = (size_t)kVtcM * Kp * 2;
    unsigned char* Th = sm_vt;
    unsigned char* Tl = Th + tbytes;
    unsigned char* Z0 = Tl + tbytes;   // stage s: Z_hi at Z0 + 2 s zbytes, Z_lo after it

    // the Toeplitz operand: row j (output row), column i (input row): w_{i - j - R}
    for (int e = tid; e < kVtcRows * Kp; e += kVtcThreads) {
        const int j = e / Kp, i = e - j * Kp;
        const int t = i - j - R;
        const float w = (t >= -R && t <= R) ? P.taps[t + R] : 0.f;
        unsigned short h, l;
        split_f16(w, h, l);
        *reinterpret_cast<unsigned short*>(Th + vtc_off(j, i, kVtcRows)) = h;
        *reinterpret_cast<unsigned short*>(Tl + vtc_off(j, i, kVtcRows)) = l;
    }
    if (tid == 0) {
        for (int s = 0; s < 2; s++) {
            mbar_init(&a_full[s], 128);
            mbar_init(&a_free[s], 1);
            mbar_init(&d_full[s], 1);
            mbar_init(&d_free[s], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(128)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_sh;

    // the scales that keep the fp16 operands in their normal range (powers of two: exact)
    int e2;
    frexpf(fmaxf(__int_as_float(*P.absmax), 1e-30f), &e2);   // max |f| <= 2^e2
    const float su = ldexpf(1.f, 14 - e2), sr = 16384.f;
    const long long ncol = (long long)P.nstrip * P.K;
    const long long nunit = ncol * P.nseg;
    // the tile sequence (identical in every role): units u = blockIdx.x + i gridDim.x, each the row segment
    // [ys, ye) of column (strip, cluster), in tiles of 64 output rows
    auto unit_rows = [&](long long u, int& strip, int& k, int& ys, int& ye) {
        const long long col = u / P.nseg;
        const int seg = (int)(u - col * P.nseg);
        strip = (int)(col % P.nstrip);
        k = (int)(col / P.nstrip);
        ys = seg * P.seglen;
        ye = min(P.H, ys + P.seglen);
    };

    if (warp < 4) {   // ---------------------------------------------------------- producers ----------
        const int col = tid & 31, cg = tid >> 5;   // this thread's column and first 8-row chunk
        const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;
        int it = 0;
        for (long long u = blockIdx.x; u < nunit; u += gridDim.x) {
            int strip, k, ys, ye;
            unit_rows(u, strip, k, ys, ye);
            const int x = strip * 32 + col;
            const bool xok = x < P.W;
            float mu[RHO];
#pragma unroll
            for (int d = 0; d < RHO; d++) mu[d] = __ldg(P.centres + k * RHO + d);
            for (int yt = ys; yt < ye; yt += kVtcRows, it++) {
                const int s = it & 1;
                const uint32_t ph = (uint32_t)(it >> 1) & 1u;
                mbar_wait(&a_free[s], ph ^ 1u);   // the MMAs of tile it - 2 have read Z[s]
                unsigned char* Zh = Z0 + 2 * s * zbytes;
                unsigned char* Zl = Zh + zbytes;
                for (int ch = cg; ch < Kp / 8; ch += 4) {
                    unsigned short hv[4][8], lv[4][8];
#pragma unroll
                    for (int r = 0; r < 8; r++) {
                        const int i = ch * 8 + r;             // input row index within the tile
                        const int yy = yt - R + i;
                        const bool ok = xok && i < kVtcRows + 2 * R && yy >= 0 && yy < P.H;
                        float pv[RHO], fv[3];
                        const long long pix = ok ? (long long)yy * P.W + x : 0;
#pragma unroll
                        for (int d = 0; d < RHO; d++) pv[d] = ok ? __ldg(P.p + pix * RHO + d) : 0.f;
#pragma unroll
                        for (int c = 0; c < 3; c++) fv[c] = (RHO == 3 && P.f == P.p) ? pv[c] : (ok ? __ldg(P.f + pix * 3 + c) : 0.f);
                        float d2 = 0.f;
#pragma unroll
                        for (int d = 0; d < RHO; d++) {
                            const float t = pv[d] - mu[d];
                            d2 = fmaf(t, t, d2);
                        }
                        float b;
                        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(d2 * c2));
                        b = ok ? b : 0.f;
                        const float bu = b * su;
#pragma unroll
                        for (int c = 0; c < 3; c++) split_f16(bu * fv[c], hv[c][r], lv[c][r]);
                        split_f16(b * sr, hv[3][r], lv[3][r]);
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t off = vtc_off(q * 32 + col, ch * 8, kVtcM);
                        uint4 h4, l4;
                        h4.x = hv[q][0] | ((uint32_t)hv[q][1] << 16);
                        h4.y = hv[q][2] | ((uint32_t)hv[q][3] << 16);
                        h4.z = hv[q][4] | ((uint32_t)hv[q][5] << 16);
                        h4.w = hv[q][6] | ((uint32_t)hv[q][7] << 16);
                        l4.x = lv[q][0] | ((uint32_t)lv[q][1] << 16);
                        l4.y = lv[q][2] | ((uint32_t)lv[q][3] << 16);
                        l4.z = lv[q][4] | ((uint32_t)lv[q][5] << 16);
                        l4.w = lv[q][6] | ((uint32_t)lv[q][7] << 16);
                        *reinterpret_cast<uint4*>(Zh + off) = h4;
                        *reinterpret_cast<uint4*>(Zl + off) = l4;
                    }
                }
                fence_proxy_async();   // generic-proxy writes of Z[s] -> visible to the tensor core
                mbar_arrive(&a_full[s]);
            }
        }
    } else if (warp < 8) {   // ---------------------------------------------------- consumers ------
        const int q = warp & 3, col = lane;   // TMEM lane quarter q = plane q, lane = column
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const float inv = (q < 3) ? 1.f / su : 1.f / sr;   // exact (powers of two)
        int it = 0;
        for (long long u = blockIdx.x; u < nunit; u += gridDim.x) {
            int strip, k, ys, ye;
            unit_rows(u, strip, k, ys, ye);
            const int x = strip * 32 + col;
            float* out = P.planes + (long long)(4 * k + q) * P.pstride + x;
            for (int yt = ys; yt < ye; yt += kVtcRows, it++) {
                const int s = it & 1;
                const uint32_t ph = (uint32_t)(it >> 1) & 1u;
                mbar_wait(&d_full[s], ph);
                tc_fence_after();
                float v[kVtcRows];
#pragma unroll
                for (int n0 = 0; n0 < kVtcRows; n0 += 16) {
                    float t16[16];
                    tmem_ld16(tbase + lane_base + (uint32_t)(s * kVtcRows + n0), t16);
#pragma unroll
                    for (int j = 0; j < 16; j++) v[n0 + j] = t16[j];
                }
                tc_fence_before();
                mbar_arrive(&d_free[s]);
                if (x < P.W) {
                    const int nr = min(kVtcRows, ye - yt);
#pragma unroll
                    for (int j = 0; j < kVtcRows; j++)
                        if (j < nr) out[(long long)(yt + j) * P.Wp] = v[j] * inv;
                }
            }
        }
    } else if (lane == 0) {   // -------------------------------------------------- MMA warp ------
        const uint32_t idesc = umma_idesc_f16(kVtcM, kVtcRows);
        const uint32_t tH = smem_u32(Th), tL = smem_u32(Tl);
        const uint32_t lboZ = kVtcM * 16, lboT = kVtcRows * 16, sbo = 128;
        int it = 0;
        for (long long u = blockIdx.x; u < nunit; u += gridDim.x) {
            int strip, k, ys, ye;
            unit_rows(u, strip, k, ys, ye);
            for (int yt = ys; yt < ye; yt += kVtcRows, it++) {
                const int s = it & 1;
                const uint32_t ph = (uint32_t)(it >> 1) & 1u;
                mbar_wait(&a_full[s], ph);
                mbar_wait(&d_free[s], ph ^ 1u);
                tc_fence_after();
                const uint32_t zH = smem_u32(Z0 + 2 * s * zbytes), zL = zH + (uint32_t)zbytes;
                const uint32_t td = tbase + (uint32_t)(s * kVtcRows);
                for (int ks = 0; ks < Kp / 16; ks++) {
                    const uint32_t oz = (uint32_t)ks * 2u * lboZ, ot = (uint32_t)ks * 2u * lboT;
                    umma_f16(td, umma_desc(zL + oz, lboZ, sbo), umma_desc(tH + ot, lboT, sbo), idesc, ks > 0 ? 1u : 0u);
                    umma_f16(td, umma_desc(zH + oz, lboZ, sbo), umma_desc(tL + ot, lboT, sbo), idesc, 1u);
                    umma_f16(td, umma_desc(zH + oz, lboZ, sbo), umma_desc(tH + ot, lboT, sbo), idesc, 1u);
                }
                umma_commit(&a_free[s]);
                umma_commit(&d_full[s]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128) : "memory");
    }
}

}  // namespace hdf
