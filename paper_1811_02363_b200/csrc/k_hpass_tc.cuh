// k_hpass_tc.cuh -- F2 on the 5th-generation tensor cores: the row half of the Gaussian convolutions
// fused with the combine and normalise (Algorithm 1 loop for3; HDapprox / approxDen,
// P:272-279) for colour images (n + 1 = 4 planes per cluster), fed by the fp16 hi/lo planes that
// k_range_vpass_tc writes.
//
// The row FIR of a tile of 64 output columns is a banded (Toeplitz) product
//   v_q(y, x0 + j) = sum_{i=0}^{127} T[j][i] t_q(y, x0 - 32 + i),   T[j][i] = w_{i - 32 - j} (0 outside [-R, R]),
// for M = 128 (plane, row) pairs (4 planes x 32 rows):
//   D[M x 64] = Z[M x 128] . T^T[128 x 64]   with tcgen05.mma kind::f16, fp32 accumulation in TMEM.
// Z comes straight from HBM: the planes are stored as t = hi + lo (scaled by a power of two), hi = fp16(t)
// in a strip-major layout [plane][x / 32][y][32] (64-byte rows) and the residual lo as e4m3(lo) in the same
// layout with 32-byte rows (3 bytes per value; k_vpass_tc.cuh writes them), so one TMA box [4 planes][32 rows]
// [one strip] of hi (SWIZZLE_64B) is a canonical K-major SW64 fp16 operand block of K = 32 and one of lo
// (SWIZZLE_32B) a canonical K-major SW32 e4m3 block of K = 32: no conversion on the SMs.  Strips outside the
// image are zero-filled by the TMA and columns past W are exact zeros (R8).
// Precision: D = z_hi T_lo + z_hi T_hi (kind::f16, T = T_hi + T_lo its fp16 split) + z_lo T_e4m3 (kind::f8f6f4,
// the same accumulator): t to ~2^-15 relative.
//
// A CTA is persistent over units (32-row block, 128-column strip of output).  For each cluster k (in
// order) the TMA warp loads the 6 input strips x0 - 32 .. x0 + 159 (tile t reads strips 2t .. 2t + 3, so
// the middle two are shared) and the two tiles' coefficient blocks c_k [32 rows][64 columns] fp32; the MMA
// warp issues each tile's MMAs into a TMEM stage (per K step of 16 columns z_hi against the stacked operand
// [T_hi; T_lo], N = 128, and per strip one kind::f8f6f4 MMA z_lo T_e4m3, N = 64; NS = false: two N = 64 fp16
// MMAs per K step); consumer warpgroup t (TMEM lane quarter = plane q, lane = row) reads tile t's 64 filtered
// values per (plane, row) (the sum of the stage's two halves) and accumulates
//   num_q(y, x) += c_k(y, x) v_{k,q}(y, x)    (q < 3),     den(y, x) += c_k(y, x) r_k(y, x)    (q = 3)
// in registers over all k.  The epilogue exchanges den through shared memory, writes g = num / den
// (coalesced, [H][W][3]) and appends the pixels with den < tau omega(0) phi(0) to the R9 list.
#pragma once
#include <cuda_fp16.h>

#include "hdf_common.cuh"
#include "k_coeffs_tc.cuh"
#include "k_vpass_tc.cuh"

namespace hdf {

constexpr int kHtcRows = 32;                       // rows per tile (x 4 planes = UMMA M = 128)
constexpr int kHtcN = 64;                          // output columns per tile (UMMA N)
constexpr int kHtcS = 2;                           // tiles per unit (one consumer warpgroup each)
constexpr int kHtcRB = 32;                         // input halo each side (one strip): R <= 32
constexpr int kHtcKp = kHtcN + 2 * kHtcRB;         // input columns per tile (8 K steps of 16)
constexpr int kHtcBoxes = 2 * kHtcS + 2;           // 32-column strips per (unit, cluster)
#ifndef HDF_HTC_NB
#define HDF_HTC_NB 11
#endif
constexpr int kHtcNB = HDF_HTC_NB;                 // strip ring slots (hi + lo each; 9 = 225 KB with the rest)
static_assert(kHtcNB > 2 * kHtcS + 2, "a step's strips must wrap the ring at most once");
constexpr int kHtcNC = 4;                          // coefficient ring slots
constexpr int kHtcThreads = 128 * kHtcS + 64;      // consumers + MMA warp + TMA warp
constexpr int kHtcMaxR = kHtcRB;
constexpr uint32_t kHtcBoxBytes = 4 * kHtcRows * 32 * 2;    // hi part (fp16): 8 KB
constexpr uint32_t kHtcLoBytes = 4 * kHtcRows * 32;         // lo part (e4m3): 4 KB
constexpr uint32_t kHtcSlotBytes = kHtcBoxBytes + kHtcLoBytes;
constexpr uint32_t kHtcCBytes = kHtcRows * kHtcN * 4;       // 8 KB: two SW128 halves of [32][32] fp32
#ifndef HDF_HTC_EPI
#define HDF_HTC_EPI 16
#endif
constexpr int kHtcEpiCols = HDF_HTC_EPI;                    // epilogue column chunk (8 frees 8 KB: a 12th ring slot fits)

inline __host__ __device__ size_t hpass_tc_smem() {
    return (size_t)kHtcNB * kHtcSlotBytes + (size_t)kHtcNC * kHtcCBytes + (size_t)2 * kHtcN * kHtcKp * 2 +
           (size_t)kHtcN * kHtcKp +
           (size_t)kHtcS * kHtcRows * kHtcEpiCols * 4 * 4 + 1024;
}

struct HtcParams {
    float* g;              // [H][W][3]
    int* flag_count;
    int* flag_list;
    const int* absmax;     // max |f| as float bits (k_absmax): the u planes' scale, one entry per band of band_rows rows
    int band_rows;         // rows per band of the column pass (multiple of 64; >= H: one band)
    int H, W, K, R;
    int nstrip;            // 128-column output strips
    int yb0, yb1;          // 32-row blocks [yb0, yb1) of this launch (the host path launches row chunks)
    int csleep;            // back-off (ns) of the consumers' mbarrier waits (HDF_HTC_CSLEEP)
    int wexp;              // the planes are stored as t 2^(14 - e2 - wexp) (u) and t 2^(14 - wexp) (b)
    float tau_floor;       // tau omega(0) phi(0); <= 0 disables flagging
    float taps[kMaxTaps];  // w_{-R..R} at [t + R]
};

// Shared-memory descriptor of a K-major SWIZZLE_64B operand (8-row atoms of 64-byte rows, 512 B apart):
// the start address advances by 32 B for the second 16-element K step inside the atom.
HDF_DEV uint64_t umma_desc_sw64(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) |
           (4ull << 61);
}

// The same for a K-major SWIZZLE_32B operand (8-row atoms of 32-byte rows, 256 B apart): one e4m3 K block of 32.
HDF_DEV uint64_t umma_desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) |
           (6ull << 61);
}
// kind::f8f6f4 (A, B e4m3 with format code 0, so the instruction descriptor is umma_idesc_f16's)
HDF_DEV void umma_f8_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
HDF_DEV void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

HDF_DEV void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane (no wait)
HDF_DEV void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
HDF_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// One half (32 columns) of a consumer's combine step: acc[32 HALF + j] += c(r, 32 HALF + j) (da[j] + db[j]).
// The coefficient block of the (tile, cluster) sits in its ring slot `cb` either as fp32 (two SWIZZLE_128B [32][32]
// halves, 4 KB each) or in 24 bits (C24; CoefParams in k_coeffs.cuh): the upper 16 bits as one SWIZZLE_128B box
// [32 rows][64 columns] of 16-bit words and, 4 KB further, the byte m as one SWIZZLE_64B box [32][64]; a value is
// rebuilt with one PRMT as bits (hi16, m, m).  Every lane reads its own row r: the swizzles make the 16-byte
// chunks of 8 consecutive rows fall into distinct banks.
template <bool C24, int HALF>
HDF_DEV void htc_fma_half(float (&acc)[kHtcN], const uint32_t (&da)[32], const uint32_t (&db)[32],
                          const unsigned char* cb, int r) {
    if (C24) {
        const unsigned char* ch = cb + r * 128;
        const unsigned char* cm = cb + 4096 + r * 64;
        uint4 mv = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c8l = 0; c8l < 4; c8l++) {
            const int c8 = 4 * HALF + c8l;   // 16-byte chunk of the hi row: columns 8 c8 .. 8 c8 + 7
            const uint4 hv = *reinterpret_cast<const uint4*>(ch + ((c8 ^ (r & 7)) << 4));
            if ((c8l & 1) == 0) mv = *reinterpret_cast<const uint4*>(cm + (((c8 >> 1) ^ ((r >> 1) & 3)) << 4));
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, mw[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
            for (int e = 0; e < 8; e++) {
                const int j = 8 * c8l + e;
                const uint32_t sel = (uint32_t)(((2 * (e & 1) + 1) << 12) | ((2 * (e & 1)) << 8) | ((4 + (e & 3)) << 4) |
                                                (4 + (e & 3)));
                const float cv = __uint_as_float(__byte_perm(hw[e >> 1], mw[((c8l & 1) * 8 + e) >> 2], sel));
                acc[32 * HALF + j] = fmaf(cv, __uint_as_float(da[j]) + __uint_as_float(db[j]), acc[32 * HALF + j]);
            }
        }
    } else {
        const unsigned char* cr = cb + r * 128 + HALF * 4096;
#pragma unroll
        for (int c4 = 0; c4 < 8; c4++) {   // 16-byte chunks swizzled by r & 7
            const float4 cv = *reinterpret_cast<const float4*>(cr + ((c4 ^ (r & 7)) << 4));
            const int j = 4 * c4;
            acc[32 * HALF + j + 0] = fmaf(cv.x, __uint_as_float(da[j + 0]) + __uint_as_float(db[j + 0]), acc[32 * HALF + j + 0]);
            acc[32 * HALF + j + 1] = fmaf(cv.y, __uint_as_float(da[j + 1]) + __uint_as_float(db[j + 1]), acc[32 * HALF + j + 1]);
            acc[32 * HALF + j + 2] = fmaf(cv.z, __uint_as_float(da[j + 2]) + __uint_as_float(db[j + 2]), acc[32 * HALF + j + 2]);
            acc[32 * HALF + j + 3] = fmaf(cv.w, __uint_as_float(da[j + 3]) + __uint_as_float(db[j + 3]), acc[32 * HALF + j + 3]);
        }
    }
}

// NS (the default): the two fp16 MMAs of a K step that share the operand z_hi run as ONE MMA of N = 128 against
// the stacked Toeplitz operand [T_hi; T_lo] (z_hi is read from shared memory once instead of twice: the kernel is
// bound by shared-memory bandwidth); the accumulator stage is then 128 columns (z_hi T_hi +
// z_lo T_8 in columns 0..63, z_hi T_lo in 64..127: all 512 TMEM columns) and the consumers add the halves.
// C24 (with NS only): the coefficient planes in 24 bits (tm_c: the 16-bit part, tm_cm: the byte), see htc_fma_half.
template <bool NS, bool C24>
__global__ void __launch_bounds__(kHtcThreads, 1) k_hpass_combine_tc(const __grid_constant__ CUtensorMap tm_zh,
                                                                     const __grid_constant__ CUtensorMap tm_zl,
                                                                     const __grid_constant__ CUtensorMap tm_c,
                                                                     const __grid_constant__ CUtensorMap tm_cm,
                                                                     const __grid_constant__ HtcParams P) {
    static_assert(NS || !C24, "the 24-bit coefficient planes are read by the stacked-operand consumers only");
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
    __shared__ uint64_t box_full[kHtcNB], box_free[kHtcNB], c_full[kHtcNC], c_free[kHtcNC], d_full[2 * kHtcS],
        d_free[2 * kHtcS];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = P.R, Kp = kHtcKp;
    constexpr uint32_t kStageCols = NS ? 2 * kHtcN : kHtcN;          // TMEM columns per accumulator stage
    constexpr uint32_t kTmemCols = 2 * kHtcS * kStageCols;           // 256, or all 512
    unsigned char* ring = sm;                                              // [NB][hi 8 KB | lo 4 KB]
    unsigned char* cring = ring + (size_t)kHtcNB * kHtcSlotBytes;          // [NC][2][32][32] fp32, SW128
    unsigned char* Th = cring + (size_t)kHtcNC * kHtcCBytes;
    unsigned char* Tl = Th + (size_t)kHtcN * Kp * 2;
    unsigned char* T8 = Tl + (size_t)kHtcN * Kp * 2;                     // T in e4m3 [64][128]
    float* epi = reinterpret_cast<float*>(T8 + (size_t)kHtcN * Kp);      // [S][den 32 x 16 | g 32 x 16 x 3]

    // the Toeplitz operand: row j (output column), column i (input column x0 - 32 + i): w_{i - 32 - j}
    for (int e = tid; e < kHtcN * Kp; e += kHtcThreads) {
        const int j = e / Kp, i = e - j * Kp;
        const int t = i - kHtcRB - j;
        const float w = (t >= -R && t <= R) ? P.taps[t + R] : 0.f;
        unsigned short h, l;
        split_f16(w, h, l);
        if (NS) {   // one operand of 128 rows: T_hi in rows 0..63, T_lo in rows 64..127 (Th and Tl are contiguous)
            *reinterpret_cast<unsigned short*>(Th + vtc_off(j, i, 2 * kHtcN)) = h;
            *reinterpret_cast<unsigned short*>(Th + vtc_off(kHtcN + j, i, 2 * kHtcN)) = l;
        } else {
            *reinterpret_cast<unsigned short*>(Th + vtc_off(j, i, kHtcN)) = h;
            *reinterpret_cast<unsigned short*>(Tl + vtc_off(j, i, kHtcN)) = l;
        }
        // e4m3 operand, K-major no swizzle: core matrix (j / 8, i / 16) of 8 rows x 16 bytes
        T8[(i >> 4) * (kHtcN * 16) + (j >> 3) * 128 + (j & 7) * 16 + (i & 15)] =
            (unsigned char)(cvt_e4m3x2(0.f, w * (1.f / kLoScale)) & 0xFFu);
    }
    if (tid == 0) {
        prefetch_tmap(&tm_zh);
        prefetch_tmap(&tm_zl);
        prefetch_tmap(&tm_c);
        if (C24) prefetch_tmap(&tm_cm);
        for (int s = 0; s < kHtcNB; s++) {
            mbar_init(&box_full[s], 1);
            mbar_init(&box_free[s], 1);
        }
        for (int s = 0; s < kHtcNC; s++) {
            mbar_init(&c_full[s], 1);
            mbar_init(&c_free[s], 4);
        }
        for (int s = 0; s < 2 * kHtcS; s++) {
            mbar_init(&d_full[s], 1);
            mbar_init(&d_free[s], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_sh;

    // units u = blockIdx.x + ui gridDim.x (strip-fastest: concurrent CTAs share the boundary strips
    // through L2); step kk = ui K + k; input strip g = 6 kk + b (ring slot g % NB); coefficient block
    // h = 2 kk + t (slot h % NC); TMEM stage of (kk, t): 2 t + (kk & 1)
    const int nrb = P.yb1 - P.yb0;
    const long long nunit = (long long)nrb * P.nstrip;
    const long long nui = nunit > blockIdx.x ? (nunit - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int K = P.K;

    if (warp < 4 * kHtcS) {   // ---------------------------------------------------- consumers -------
        const int t = warp >> 2, q = warp & 3, r = lane;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        float* den_s = epi + (size_t)t * (kHtcRows * kHtcEpiCols * 4);   // [32][16]
        float* g_s = den_s + kHtcRows * kHtcEpiCols;                     // [32][16][3]
        const float inv_sb = ldexpf(1.f, P.wexp - 14);
        for (long long ui = 0; ui < nui; ui++) {
            const long long u = blockIdx.x + ui * (long long)gridDim.x;
            const int ry = P.yb0 + (int)(u / P.nstrip), sx = (int)(u % P.nstrip);
            // the u planes' scale of this row block's band (the column pass ran in bands when the input arrived in
            // row chunks: hdf_filter_host)
            int e2;
            frexpf(fmaxf(__int_as_float(P.absmax[(ry * kHtcRows) / P.band_rows]), 1e-30f), &e2);
            const float inv_su = ldexpf(1.f, e2 + P.wexp - 14);
            float acc[kHtcN];
#pragma unroll
            for (int j = 0; j < kHtcN; j++) acc[j] = 0.f;
            for (int k = 0; k < K; k++) {
                const long long kk = ui * K + k;
                const long long h = 2 * kk + t;
                const int cs = (int)(h % kHtcNC);
                const int s = 2 * t + (int)(kk & 1);
                mbar_wait_backoff(&c_full[cs], (uint32_t)(h / kHtcNC) & 1u, P.csleep);
                mbar_wait_backoff(&d_full[s], (uint32_t)(kk >> 1) & 1u, P.csleep);
                tc_fence_after();
                uint32_t d0[32], d1[32];
                const unsigned char* cslot = cring + (size_t)cs * kHtcCBytes;
                const unsigned char* cb = cslot + r * 128;
                if (NS) {   // columns j and 64 + j of the stage: (z_hi T_hi + z_lo T_8) + z_hi T_lo
                    const uint32_t ta = tbase + lane_base + (uint32_t)s * kStageCols;
                    tmem_ld32_nw(ta, d0);
                    tmem_ld32_nw(ta + 64, d1);
                    tmem_wait_ld();
                    htc_fma_half<C24, 0>(acc, d0, d1, cslot, r);
                    tmem_ld32_nw(ta + 32, d0);
                    tmem_ld32_nw(ta + 96, d1);
                    tmem_wait_ld();
                    tc_fence_before();
                    mbar_arrive(&d_free[s]);
                    htc_fma_half<C24, 1>(acc, d0, d1, cslot, r);
                } else {
                tmem_ld32_nw(tbase + lane_base + (uint32_t)(s * kHtcN), d0);
                tmem_ld32_nw(tbase + lane_base + (uint32_t)(s * kHtcN + 32), d1);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&d_free[s]);
#pragma unroll
                for (int c4 = 0; c4 < 8; c4++) {   // half 0: columns 0..31 (16-byte chunks swizzled by r & 7)
                    const float4 cv = *reinterpret_cast<const float4*>(cb + ((c4 ^ (r & 7)) << 4));
                    acc[4 * c4 + 0] = fmaf(cv.x, __uint_as_float(d0[4 * c4 + 0]), acc[4 * c4 + 0]);
                    acc[4 * c4 + 1] = fmaf(cv.y, __uint_as_float(d0[4 * c4 + 1]), acc[4 * c4 + 1]);
                    acc[4 * c4 + 2] = fmaf(cv.z, __uint_as_float(d0[4 * c4 + 2]), acc[4 * c4 + 2]);
                    acc[4 * c4 + 3] = fmaf(cv.w, __uint_as_float(d0[4 * c4 + 3]), acc[4 * c4 + 3]);
                }
#pragma unroll
                for (int c4 = 0; c4 < 8; c4++) {   // half 1: columns 32..63
                    const float4 cv = *reinterpret_cast<const float4*>(cb + 4096 + ((c4 ^ (r & 7)) << 4));
                    acc[32 + 4 * c4 + 0] = fmaf(cv.x, __uint_as_float(d1[4 * c4 + 0]), acc[32 + 4 * c4 + 0]);
                    acc[32 + 4 * c4 + 1] = fmaf(cv.y, __uint_as_float(d1[4 * c4 + 1]), acc[32 + 4 * c4 + 1]);
                    acc[32 + 4 * c4 + 2] = fmaf(cv.z, __uint_as_float(d1[4 * c4 + 2]), acc[32 + 4 * c4 + 2]);
                    acc[32 + 4 * c4 + 3] = fmaf(cv.w, __uint_as_float(d1[4 * c4 + 3]), acc[32 + 4 * c4 + 3]);
                }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&c_free[cs]);
            }
            // ---- epilogue: den through shared memory, g = num / den, R9 flags, coalesced stores ----
            const int y = ry * kHtcRows + r;
            const int xt = sx * (kHtcS * kHtcN) + t * kHtcN;   // first column of this tile
#pragma unroll
            for (int ch = 0; ch < kHtcN / kHtcEpiCols; ch++) {
                if (q == 3) {
#pragma unroll
                    for (int j = 0; j < kHtcEpiCols; j++) {
                        const float den = acc[ch * kHtcEpiCols + j] * inv_sb;
                        den_s[r * kHtcEpiCols + j] = den;
                        const int x = xt + ch * kHtcEpiCols + j;
                        const bool flag = (P.tau_floor > 0.f) && (den < P.tau_floor) && (x < P.W) && (y < P.H);
                        const unsigned m = __ballot_sync(0xffffffffu, flag);
                        if (m) {
                            int basei = 0;
                            if (lane == 0) basei = atomicAdd(P.flag_count, __popc(m));
                            basei = __shfl_sync(0xffffffffu, basei, 0);
                            if (flag) P.flag_list[basei + __popc(m & ((1u << lane) - 1))] = y * P.W + x;
                        }
                    }
                }
                named_sync(1 + t, 128);
                if (q < 3) {
#pragma unroll
                    for (int j = 0; j < kHtcEpiCols; j++)
                        g_s[(r * kHtcEpiCols + j) * 3 + q] = acc[ch * kHtcEpiCols + j] * inv_su / den_s[r * kHtcEpiCols + j];
                }
                named_sync(1 + t, 128);
                {
                    const int xc = xt + ch * kHtcEpiCols;
                    const int ncol = min(kHtcEpiCols, P.W - xc);
                    const int seg = ncol * 3;
                    const int tl = warp * 32 + lane - t * 128;
                    for (int e = tl; e < kHtcRows * kHtcEpiCols * 3; e += 128) {
                        const int rr = e / (kHtcEpiCols * 3), o = e - rr * (kHtcEpiCols * 3);
                        const int yy = ry * kHtcRows + rr;
                        if (o < seg && yy < P.H) P.g[((long long)yy * P.W + xc) * 3 + o] = g_s[e];
                    }
                }
                named_sync(1 + t, 128);
            }
        }
    } else if (warp == 4 * kHtcS) {   // ------------------------------------------------ MMA warp -------
        const uint32_t idesc = umma_idesc_f16(128, kHtcN), idesc_s = umma_idesc_f16(128, 2 * kHtcN);
        const uint64_t dt = umma_desc(0, kHtcN * 16, 128), dts = umma_desc(0, 2 * kHtcN * 16, 128);
        const uint32_t tH = smem_u32(Th), tL = smem_u32(Tl), t8 = smem_u32(T8), rb = smem_u32(ring);
        // ring slot and phase of the step's first strip g0 = 6 kk, kept in 32-bit incremental form (a step's
        // strips g0 .. g0 + 5 wrap the ring at most once)
        int bslot = 0, bph = 0;
        for (long long ui = 0; ui < nui; ui++) {
            for (int k = 0; k < K; k++) {
                const long long kk = ui * K + k;
#pragma unroll 1
                for (int t = 0; t < kHtcS; t++) {
                    const int s = 2 * t + (int)(kk & 1);
                    // tile t reads input strips 2t .. 2t + 3
                    for (int b = 0; b < 4; b++) {
                        int sl = bslot + 2 * t + b, ph = bph;
                        if (sl >= kHtcNB) {
                            sl -= kHtcNB;
                            ph ^= 1;
                        }
                        mbar_wait(&box_full[sl], (uint32_t)ph);
                    }
                    if (kk >= 2) mbar_wait(&d_free[s], (uint32_t)((kk >> 1) - 1) & 1u);
                    tc_fence_after();
                    const uint32_t td = tbase + (uint32_t)s * kStageCols;
#pragma unroll
                    for (int ks = 0; ks < kHtcKp / 16; ks++) {
                        int sl = bslot + 2 * t + (ks >> 1);
                        if (sl >= kHtcNB) sl -= kHtcNB;
                        const uint32_t za = rb + (uint32_t)sl * kHtcSlotBytes + (uint32_t)((ks & 1) * 32);
                        const uint64_t aH = umma_desc_sw64(za);
                        if (NS) {   // z_hi [T_hi; T_lo]^T: 128 accumulator columns
                            const uint32_t ot = (uint32_t)ks * (2u * 2u * kHtcN * 16u);
                            const uint64_t bS = dts | (uint64_t)(((tH + ot) >> 4) & 0x3FFFu);
                            umma_f16_warp(td, aH, bS, idesc_s, ks > 0 ? 1u : 0u);
                        } else {
                            const uint32_t ot = (uint32_t)ks * (2u * kHtcN * 16u);
                            const uint64_t bH = dt | (uint64_t)(((tH + ot) >> 4) & 0x3FFFu);
                            const uint64_t bL = dt | (uint64_t)(((tL + ot) >> 4) & 0x3FFFu);
                            umma_f16_warp(td, aH, bL, idesc, ks > 0 ? 1u : 0u);
                            umma_f16_warp(td, aH, bH, idesc, 1u);
                        }
                    }
#pragma unroll
                    for (int b = 0; b < 4; b++) {   // the residuals: one e4m3 MMA (K = 32) per strip
                        int sl = bslot + 2 * t + b;
                        if (sl >= kHtcNB) sl -= kHtcNB;
                        const uint64_t aL = umma_desc_sw32(rb + (uint32_t)sl * kHtcSlotBytes + kHtcBoxBytes);
                        const uint64_t b8 = dt | (uint64_t)(((t8 + (uint32_t)b * (2u * kHtcN * 16u)) >> 4) & 0x3FFFu);
                        umma_f8_warp(td, aL, b8, idesc, 1u);
                    }
                    umma_commit_warp(&d_full[s]);
                    // strips 2t, 2t + 1 are read by no later tile of this step; the last tile releases all four
                    const int nrel = (t == kHtcS - 1) ? 4 : 2;
                    for (int b = 0; b < nrel; b++) {
                        int sl = bslot + 2 * t + b;
                        if (sl >= kHtcNB) sl -= kHtcNB;
                        umma_commit_warp(&box_free[sl]);
                    }
                }
                bslot += kHtcBoxes;
                if (bslot >= kHtcNB) {
                    bslot -= kHtcNB;
                    bph ^= 1;
                }
            }
        }
    } else if (lane == 0) {   // ------------------------------------------------------- TMA warp -------
        int tslot = 0, tph = 0, tfilled = 0;
        for (long long ui = 0; ui < nui; ui++) {
            const long long u = blockIdx.x + ui * (long long)gridDim.x;
            const int ry = P.yb0 + (int)(u / P.nstrip), sx = (int)(u % P.nstrip);
            const int s0 = sx * (2 * kHtcS) - 1, y0 = ry * kHtcRows;   // first input strip (x0 - 32)
            for (int k = 0; k < K; k++) {
                const long long kk = ui * K + k;
                for (int b = 0; b < kHtcBoxes; b++) {
                    // strip g = 6 kk + b: ring slot sl = g % NB, phase (g / NB) & 1 (incremental, 32-bit)
                    const int sl = tslot;
                    if (tfilled >= kHtcNB) mbar_wait(&box_free[sl], (uint32_t)(tph ^ 1));
                    else tfilled++;
                    if (++tslot == kHtcNB) {
                        tslot = 0;
                        tph ^= 1;
                    }
                    mbar_arrive_expect_tx(&box_full[sl], kHtcSlotBytes);
                    unsigned char* dst = ring + (size_t)sl * kHtcSlotBytes;
                    tma_load_4d(dst, &tm_zh, &box_full[sl], 0, y0, s0 + b, 4 * k);                  // hi (fp16)
                    tma_load_4d(dst + kHtcBoxBytes, &tm_zl, &box_full[sl], 0, y0, s0 + b, 4 * k);   // lo (e4m3)
                    if (b == 3 || b == 5) {   // tile (b - 3) / 2's coefficients
                        const int t = (b - 3) / 2;
                        const long long h = 2 * kk + t;
                        const int cs = (int)(h % kHtcNC);
                        if (h >= kHtcNC) mbar_wait(&c_free[cs], (uint32_t)((h / kHtcNC) - 1) & 1u);
                        mbar_arrive_expect_tx(&c_full[cs], C24 ? 4096u + 2048u : kHtcCBytes);
                        unsigned char* cd = cring + (size_t)cs * kHtcCBytes;
                        const int xt = sx * (kHtcS * kHtcN) + kHtcN * t;
                        if (C24) {   // [32 rows][64 columns]: 16-bit words (4 KB), bytes (2 KB)
                            tma_load_3d(cd, &tm_c, &c_full[cs], xt, y0, k);
                            tma_load_3d(cd + 4096, &tm_cm, &c_full[cs], xt, y0, k);
                        } else {
                            tma_load_3d(cd, &tm_c, &c_full[cs], xt, y0, k);
                            tma_load_3d(cd + 4096, &tm_c, &c_full[cs], xt + 32, y0, k);
                        }
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kTmemCols) : "memory");
    }
}

}  // namespace hdf
