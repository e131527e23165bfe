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
// output rows; every unit has the same number of tiles), warp-specialised:
//   * a TMA warp streams the raw guide rows of the strip, [64 rows x 32 pixels x 3] per TMA box (rows outside the
//     image zero-filled), into a ring of kVtcRaw slots: a tile reads 2 consecutive slots (Kp <= 128 rows), the next
//     ones load while it computes, and each slot is released by the last tile that reads it;
//   * producers (8 warps): z for the new 8-row chunks of the strip's 32 columns and the cluster's 4 planes
//     (b_k = exp2(-|p - mu_k|^2 log2(e) / 2 sigma_r^2), u_k = b_k f, f = p; packed f32x2 arithmetic on row pairs)
//     from the raw stage, split, stored into the Z ring in the canonical K-major no-swizzle layout (8 x 16-byte
//     core matrices; one 16-byte store = 8 consecutive rows of one (plane, column)); arrive on "Z full";
//   * MMA warp: waits "Z full" and "D free", issues the tile's MMAs (M = 128, K = 16 per step: with the stacked
//     operand z_hi [T_hi; T_lo]^T, N = 128, and z_lo T_hi^T, N = 64; else the three N = 64 products) and commits
//     them to "Z free" and "D full" (kVtcStages tiles in flight, D in TMEM);
//   * consumers (8 warps of 32 rows each, TMEM lane quarter = plane; HDF_VTC_CONS=4: 4 warps of 64 rows): load
//     the output rows of their (plane, column), release the stage and store them: fp32 planes (scaled back,
//     coalesced over the 32 columns), or -- for the tensor-core row pass -- 3 bytes per value in the strip-major
//     layout: hi = fp16 [plane][strip][y][32] (two rows' 64-byte lines per warp store after a lane-pair exchange)
//     and the residual as e4m3 in the same order (four rows' 32-byte lines per warp store after a 4 x 4 byte
//     transpose over lane quads) (k_hpass_tc.cuh).
// The Toeplitz operand T (hi, lo) is staged once per CTA.
#pragma once
#include <cuda_fp16.h>

#include "hdf_common.cuh"
#include "k_coeffs_tc.cuh"
#include "k_vpass.cuh"

namespace hdf {

constexpr int kVtcRows = 64;       // output rows per tile (UMMA N)
constexpr int kVtcM = 128;         // (plane, column) pairs per tile (UMMA M): 4 planes x 32 columns
constexpr int kVtcProd = 256;      // producer threads (8 warps)
// consumer warps CONS (a template parameter: 4 take 64 rows each, 8 take 32 rows each)
constexpr int vtc_threads(int cons) { return kVtcProd + 32 * cons + 64; }   // + consumers + MMA warp + TMA warp

inline __host__ __device__ int vtc_kp(int R) { return ((kVtcRows + 2 * R) + 15) & ~15; }
constexpr int kVtcMaxR = 24;       // Kp <= 112: the shared-memory budget below
#ifndef HDF_VTC_STAGES
#define HDF_VTC_STAGES 2
#endif
#ifndef HDF_VTC_RAW
#define HDF_VTC_RAW 4
#endif
constexpr int kVtcStages = HDF_VTC_STAGES;   // tiles in flight between the producers, the MMA warp and the consumers
constexpr int kVtcRaw = HDF_VTC_RAW;         // raw guide chunks (64 rows) in the TMA ring: a tile reads 2, the
                                             // rest load ahead (the ring depth hides the L2 latency of the
                                             // raw rows, which every cluster's unit of a strip re-reads)
constexpr int kVtcZChunks = 6 + 8 * kVtcStages;   // Z ring: 8-row chunks (a tile reads Kp / 8 <= 14; the producers write up
                                   // to two further tiles' 8 new chunks meanwhile; even, so a 16-row K step
                                   // never wraps)
constexpr int kVtcZChunkBytes = kVtcM * 8 * 2;
// Dynamic shared memory: T_hi, T_lo [64][Kp], the Z ring hi and lo [22 chunks][128][8] (fp16), the raw
// ring [3][64][96] fp32
inline __host__ __device__ size_t vpass_tc_smem(int R) {
    const int Kp = vtc_kp(R);
    return (size_t)2 * kVtcRows * Kp * 2 + (size_t)2 * kVtcZChunks * kVtcZChunkBytes + (size_t)kVtcRaw * 64 * 96 * 4 +
           128;
}

struct VtcParams {
    const float* centres;  // [K][3]
    float* planes;         // [4K][H][Wp] fp32 (ph == NULL)
    unsigned short* ph;    // else fp16 hi parts, strip-major: ph [4K][Wp / 32][H][32] (64-byte rows), and
    unsigned char* pl;     // the residuals as e4m3(lo): pl [4K][Wp / 32][H][32] (32-byte rows)
                           // (k_hpass_tc.cuh); Wp a multiple of 32
    int wexp;              // ph: stored value = t 2^(14 - e2 - wexp) (u planes), t 2^(14 - wexp) (b planes)
    const int* absmax;     // max |f| as float bits (k_absmax)
    long long pstride;     // H * Wp
    int H, W, Wp, K, R;
    int nstrip, nseg, seglen;   // 32-column strips, row segments per column and their length (multiple of 64)
    int y0;                     // first output row of this launch (row bands of the pipelined filter)
    int csleep;                 // back-off (ns) of the consumers' and the TMA warp's mbarrier waits (HDF_VTC_CSLEEP)
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
// Whole-warp forms: every lane of the warp executes them (warp-uniform operands, so the descriptors stay
// in uniform registers) and elect.sync picks the one lane that issues (always the same: the lowest).
HDF_DEV void umma_f16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
HDF_DEV void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// fp16 hi/lo split of x: hi = fp16(x), lo = fp16(x - hi)
HDF_DEV void split_f16(float x, unsigned short& hi, unsigned short& lo) {
    const __half h = __float2half_rn(x);
    hi = __half_as_ushort(h);
    lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
}

// packed split of two values (rows r, r + 1 of one operand column): the 32-bit words of hi and lo
// (one cvt.rn.f16x2.f32 each; the conversions stay off the transcendental pipe)
HDF_DEV void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// fp16 rounding of two values (rows r, r + 1 of one column): the 32-bit hi word and the fp32 residuals
HDF_DEV uint32_t split_f16x2_res(float a, float b, float& ra, float& rb) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    ra = a - hf.x;
    rb = b - hf.y;
    return *reinterpret_cast<const uint32_t*>(&h);
}
// fp16 rounding of a packed pair: the 32-bit hi word and the packed fp32 residuals (one packed subtraction)
HDF_DEV uint32_t split_f16x2_res2(unsigned long long ab, unsigned long long& res) {
    float a, b;
    unpack2(ab, a, b);
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    res = fsub2(ab, pack2(hf.x, hf.y));
    return *reinterpret_cast<const uint32_t*>(&h);
}
// hi and lo words of a packed pair
HDF_DEV void split_f16x2p(unsigned long long ab, uint32_t& hi, uint32_t& lo) {
    unsigned long long res;
    hi = split_f16x2_res2(ab, res);
    float ra, rb;
    unpack2(res, ra, rb);
    const __half2 l = __floats2half2_rn(ra, rb);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
// two fp32 -> e4m3 (saturating, round to nearest even): hi_val in the upper byte, lo_val in the lower
HDF_DEV uint32_t cvt_e4m3x2(float hi_val, float lo_val) {
    unsigned short r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi_val), "f"(lo_val));
    return r;
}
// The stored planes of the tensor-core row pass: t = hi + lo with hi = fp16(t) and the residual lo kept
// as e4m3(kLoScale lo) (3 bytes per value; k_hpass_tc.cuh multiplies it by the taps / kLoScale).  With
// |t| <= 2^14, |lo| <= 4 sits well inside e4m3's range unscaled; its subnormal floor (2^-10 absolute) is
// 2^-24 of the largest value.
constexpr float kLoScale = 1.f;
static_assert(kLoScale == 1.f, "the whole-tile store path of k_range_vpass_tc stores the residuals unscaled");

// Byte offset of (row r, k) in an operand of nrow rows (multiple of 8) and Kp columns, K-major, no
// swizzle, layout "m-groups adjacent": core matrix (r / 8, k / 8) at (k / 8) * (nrow * 16) + (r / 8) * 128.
HDF_DEV uint32_t vtc_off(int r, int k, int nrow) {
    return (uint32_t)((k >> 3) * (nrow * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// f = p, rho = n = 3 (the colour bilateral filter); tm_p: p as [H][3W] fp32, box [96][64]
// NS: the two MMAs of a K step that share the operand z_hi run as one MMA of N = 128 against the stacked Toeplitz
// operand [T_hi; T_lo] (z_hi is read from shared memory once; an accumulator stage is then 128 TMEM columns:
// z_hi T_hi + z_lo T_hi in columns 0..63, z_hi T_lo in 64..127, added by the consumers)
template <int kVtcCons, bool NS>
__global__ void __launch_bounds__(vtc_threads(kVtcCons), 1) k_range_vpass_tc(const __grid_constant__ CUtensorMap tm_p,
                                                                             const __grid_constant__ VtcParams P) {
    constexpr int kVtcNRW = kVtcRows / (kVtcCons / 4);           // output rows per consumer thread
    constexpr int kVtcThreads = vtc_threads(kVtcCons);
    extern __shared__ __align__(128) unsigned char sm_raw[];
    unsigned char* sm_vt = sm_raw + ((128u - (smem_u32(sm_raw) & 127u)) & 127u);
    __shared__ uint64_t c_full[kVtcRaw], c_free[kVtcRaw], z_full[kVtcStages], z_free[kVtcStages], d_full[kVtcStages],
        d_free[kVtcStages];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = P.R, Kp = vtc_kp(R);
    const size_t tbytes = (size_t)kVtcRows * Kp * 2, zbytes = (size_t)kVtcM * Kp * 2;
    constexpr uint32_t kSlotBytes = 64 * 96 * 4;
    constexpr uint32_t kStageCols = NS ? 2 * kVtcRows : kVtcRows;   // TMEM columns per accumulator stage
    constexpr uint32_t kTmemCols = kVtcStages * kStageCols <= 256 ? 256 : 512;
    unsigned char* Th = sm_vt;
    unsigned char* Tl = Th + tbytes;
    unsigned char* ZH = Tl + tbytes;                                          // Z ring, hi
    unsigned char* ZL = ZH + (size_t)kVtcZChunks * kVtcZChunkBytes;            // Z ring, lo
    float* ring = reinterpret_cast<float*>(ZL + (size_t)kVtcZChunks * kVtcZChunkBytes);   // [kVtcRaw][64][96]
    (void)zbytes;

    // the Toeplitz operand: row j (output row), column i (input row): w_{i - j - R}
    for (int e = tid; e < kVtcRows * Kp; e += kVtcThreads) {
        const int j = e / Kp, i = e - j * Kp;
        const int t = i - j - R;
        const float w = (t >= -R && t <= R) ? P.taps[t + R] : 0.f;
        unsigned short h, l;
        split_f16(w, h, l);
        if (NS) {   // one operand of 128 rows: T_hi in rows 0..63, T_lo in rows 64..127 (Th and Tl are contiguous)
            *reinterpret_cast<unsigned short*>(Th + vtc_off(j, i, 2 * kVtcRows)) = h;
            *reinterpret_cast<unsigned short*>(Th + vtc_off(kVtcRows + j, i, 2 * kVtcRows)) = l;
        } else {
            *reinterpret_cast<unsigned short*>(Th + vtc_off(j, i, kVtcRows)) = h;
            *reinterpret_cast<unsigned short*>(Tl + vtc_off(j, i, kVtcRows)) = l;
        }
    }
    if (tid == 0) {
        prefetch_tmap(&tm_p);
        for (int s = 0; s < kVtcRaw; s++) {
            mbar_init(&c_full[s], 1);
            mbar_init(&c_free[s], kVtcProd);
        }
        for (int s = 0; s < kVtcStages; s++) {
            mbar_init(&z_full[s], kVtcProd);
            mbar_init(&z_free[s], 1);
            mbar_init(&d_full[s], 1);
            mbar_init(&d_free[s], 32 * kVtcCons);
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

    // the scales that keep the fp16 operands in their normal range (powers of two: exact)
    int e2;
    frexpf(fmaxf(__int_as_float(*P.absmax), 1e-30f), &e2);   // max |f| <= 2^e2
    const float su = ldexpf(1.f, 14 - e2), sr = 16384.f;
    // the tile sequence (identical in every role): tile `it` of this CTA is tile j = it % TU of its
    // unit number ui = it / TU, unit u = blockIdx.x + ui gridDim.x = the row segment of column (strip,
    // cluster).  The raw rows of a unit are its chunks c = 0 .. TU (64 rows each, from ys - R); the
    // CTA's chunk sequence number is g = ui (TU + 1) + c, ring slot g % kVtcRaw, and tile j reads chunks j, j+1.
    const long long nunit = (long long)P.nstrip * P.K * P.nseg;
    const int TU = P.seglen / kVtcRows;
    const long long nui = nunit > blockIdx.x ? (nunit - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long nit = nui * TU;
    auto unit_of = [&](long long ui, int& strip, int& k, int& ys) {
        const long long u = blockIdx.x + ui * (long long)gridDim.x;
        const long long col = u / P.nseg;
        const int seg = (int)(u - col * P.nseg);
        // cluster-fastest: the CTAs running at the same time cover all clusters of a few strips, so a
        // strip's raw rows come from L2 for all but the first of them (strip-fastest re-read the whole
        // guide from DRAM once per cluster: 10.9 GB at config 5)
        k = (int)(col % P.K);
        strip = (int)(col / P.K);
        ys = P.y0 + seg * P.seglen;
    };

    if (warp < kVtcProd / 32) {   // ------------------------------------------------ producers -------
        const int col = tid & 31, cg = tid >> 5;   // this thread's column and first 8-row chunk
        const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;
        // b su = 2^(d2 c2 + 14 - e2) (the u planes' scale folded into the exponent: exact), b sr = (b su) 2^e2
        // (the fp16 planes' output scale 2^-wexp folded in as well: the MMA then yields the stored value)
        const float lsu = (float)(14 - e2 - (P.ph ? P.wexp : 0)), sbu = ldexpf(1.f, e2);
        // per-tile bookkeeping in 32-bit incremental form: raw chunk ga = ui (TU + 1) + j (ring slot ga %
        // kVtcRaw, phase ga / kVtcRaw), the unit's first Z slot zs0 = ui (8 TU + 6) % kVtcZChunks
        const unsigned long long c2p = pack2(c2, c2), lsup = pack2(lsu, lsu), sbup = pack2(sbu, sbu);
        // this thread's 16-byte slot inside a Z chunk: (plane 0, col) at ((col >> 3) * 128 + (col & 7) * 16); plane q is
        // 4 row groups (512 bytes) further
        const uint32_t zcol = (uint32_t)((col >> 3) * 128 + (col & 7) * 16);
        const int U = 8 * TU + 6;
        int ga_slot = 0, ga_ph = 0, zs0 = 0;
        long long it = 0;
        for (long long ui = 0; ui < nui; ui++) {
            int strip, k, ys;
            unit_of(ui, strip, k, ys);
            const bool xok = strip * 32 + col < P.W;
            const float m0 = __ldg(P.centres + k * 3), m1 = __ldg(P.centres + k * 3 + 1),
                        m2 = __ldg(P.centres + k * 3 + 2);
            const unsigned long long m0p = pack2(m0, m0), m1p = pack2(m1, m1), m2p = pack2(m2, m2);
            for (int j = 0; j < TU; j++, it++) {
                const int yt = ys + j * kVtcRows;
                const int gb_slot = ga_slot + 1 == kVtcRaw ? 0 : ga_slot + 1;
                const int gb_ph = ga_slot + 1 == kVtcRaw ? ga_ph ^ 1 : ga_ph;
                mbar_wait(&c_full[ga_slot], (uint32_t)ga_ph);
                mbar_wait(&c_full[gb_slot], (uint32_t)gb_ph);
                // Z chunks of this unit: c = 0 .. U - 1, U = 8 TU + 6 (tile j reads 8j .. 8j + Kp/8 - 1).  Tile j
                // writes the chunks no earlier tile wrote: all Kp/8 for j = 0, else 8j + Kp/8 - 8 .. 8j + Kp/8 - 1.
                const int c0 = (j == 0) ? 0 : 8 * j + Kp / 8 - 8, c1 = 8 * j + Kp / 8;
                {
                    // Their ring slots held the chunk kVtcZChunks back in the CTA's chunk sequence (S = ui U + c).
                    // The last reader of that chunk is tile min(TU - 1, c' / 8) of its unit (chunks past the last
                    // tile's reads have none: the clamp is conservative); readers are monotonic in S, so the
                    // highest chunk written decides, and the MMAs complete in order.  (A fixed "it - 3" let the
                    // producers overwrite the first input rows of a unit's last tile while its MMAs were pending.)
                    int up = 0, cp = c1 - 1 - kVtcZChunks;   // (unit offset, chunk) of S - kVtcZChunks
                    while (cp < 0) {
                        cp += U;
                        up++;
                    }
                    const long long tw = (ui - up) * TU + min(TU - 1, cp / 8);
                    if (ui - up >= 0 && tw >= 0) mbar_wait(&z_free[tw % kVtcStages], (uint32_t)(tw / kVtcStages) & 1u);
                }
                const float* slot_a = ring + (size_t)ga_slot * (64 * 96) + col * 3;
                const float* slot_b = ring + (size_t)gb_slot * (64 * 96) + col * 3;
                for (int cc = c0 + cg; cc < c1; cc += kVtcProd / 32) {
                    const int ch = cc - 8 * j;   // 8-row chunk within the tile
                    unsigned long long zv[4][4];   // [plane][row pair] packed (rows 2i, 2i + 1)
                    const float* px = ((ch < 8) ? slot_a : slot_b) + (ch & 7) * (8 * 96);
                    const int y8 = yt - R + ch * 8;   // image row of the chunk's first input row
                    if (xok && y8 >= 0 && y8 + 8 <= P.H) {   // the whole chunk inside the image: packed, no row tests
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            const unsigned long long p0 = pack2(px[(2 * i) * 96], px[(2 * i + 1) * 96]);
                            const unsigned long long p1 = pack2(px[(2 * i) * 96 + 1], px[(2 * i + 1) * 96 + 1]);
                            const unsigned long long p2 = pack2(px[(2 * i) * 96 + 2], px[(2 * i + 1) * 96 + 2]);
                            const unsigned long long t0 = fsub2(p0, m0p), t1 = fsub2(p1, m1p), t2 = fsub2(p2, m2p);
                            const unsigned long long d2 = ffma2(t2, t2, ffma2(t1, t1, fmul2(t0, t0)));
                            float a0, a1, b0, b1;
                            unpack2(ffma2(d2, c2p, lsup), a0, a1);
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b0) : "f"(a0));
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b1) : "f"(a1));
                            const unsigned long long bu = pack2(b0, b1);
                            zv[0][i] = fmul2(bu, p0);
                            zv[1][i] = fmul2(bu, p1);
                            zv[2][i] = fmul2(bu, p2);
                            zv[3][i] = fmul2(bu, sbup);
                        }
                    } else {
                        float zs[4][8];
#pragma unroll
                        for (int r = 0; r < 8; r++) {
                            const float p0 = px[r * 96], p1 = px[r * 96 + 1], p2 = px[r * 96 + 2];
                            const float t0 = p0 - m0, t1 = p1 - m1, t2 = p2 - m2;
                            const float d2 = fmaf(t2, t2, fmaf(t1, t1, t0 * t0));
                            float bu;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(bu) : "f"(fmaf(d2, c2, lsu)));
                            // rows outside [0, H) and columns past W contribute zero (R8); rows past 64 + 2R meet zero
                            // taps (a chunk may be shared with the next tile)
                            bu = (xok && (unsigned)(y8 + r) < (unsigned)P.H) ? bu : 0.f;
                            zs[0][r] = bu * p0;
                            zs[1][r] = bu * p1;
                            zs[2][r] = bu * p2;
                            zs[3][r] = bu * sbu;
                        }
#pragma unroll
                        for (int q = 0; q < 4; q++)
#pragma unroll
                            for (int i = 0; i < 4; i++) zv[q][i] = pack2(zs[q][2 * i], zs[q][2 * i + 1]);
                    }
                    int zslot = zs0 + cc;
                    while (zslot >= kVtcZChunks) zslot -= kVtcZChunks;
                    const uint32_t zoff = (uint32_t)zslot * (uint32_t)kVtcZChunkBytes + zcol;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        uint4 h4, l4;
                        split_f16x2p(zv[q][0], h4.x, l4.x);
                        split_f16x2p(zv[q][1], h4.y, l4.y);
                        split_f16x2p(zv[q][2], h4.z, l4.z);
                        split_f16x2p(zv[q][3], h4.w, l4.w);
                        *reinterpret_cast<uint4*>(ZH + zoff + q * 512) = h4;
                        *reinterpret_cast<uint4*>(ZL + zoff + q * 512) = l4;
                    }
                }
                // raw chunk j has no later reader in this unit (tile j + 1 reads j + 1, j + 2); the last tile
                // also releases chunk j + 1
                mbar_arrive(&c_free[ga_slot]);
                if (j == TU - 1) mbar_arrive(&c_free[gb_slot]);
                fence_proxy_async();   // generic-proxy writes of Z -> visible to the tensor core
                mbar_arrive(&z_full[it % kVtcStages]);
                // the next tile's first raw chunk is this tile's second; a unit's last tile also consumed the
                // unit's extra chunk (TU + 1 chunks per unit)
                ga_slot = gb_slot;
                ga_ph = gb_ph;
                if (j == TU - 1) {
                    ga_ph = ga_slot + 1 == kVtcRaw ? ga_ph ^ 1 : ga_ph;
                    ga_slot = ga_slot + 1 == kVtcRaw ? 0 : ga_slot + 1;
                }
            }
            zs0 = (zs0 + U) % kVtcZChunks;
        }
    } else if (warp < kVtcProd / 32 + kVtcCons) {   // ------------------------------- consumers -------
        // TMEM lane quarter q = plane q, lane = column; consumer warp group h takes rows r0 .. r0 + NRW - 1
        const int q = warp & 3, col = lane, r0 = ((warp - kVtcProd / 32) >> 2) * kVtcNRW;
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        // fp32 output: t = D / su (u planes), D / sr (b planes); fp16 output: D itself, already t 2^(14 - e2 - wexp)
        // (u) or t 2^(14 - wexp) (b) by the producers' scale, |value| <= 2^14 since the taps sum to at most 2^wexp
        const float inv = (q < 3) ? 1.f / su : 1.f / sr;   // exact (powers of two); unused for the fp16 planes
        const int step = P.Wp;
        long long it = 0;
        for (long long ui = 0; ui < nui; ui++) {
            int strip, k, ys;
            unit_of(ui, strip, k, ys);
            const int x = strip * 32 + col;
            float* base = P.planes + (long long)(4 * k + q) * P.pstride + x;
            for (int j = 0; j < TU; j++, it++) {
                const int yt = ys + j * kVtcRows;
                const int s = (int)(it % kVtcStages);
                mbar_wait_backoff(&d_full[s], (uint32_t)(it / kVtcStages) & 1u, P.csleep);
                tc_fence_after();
                float v[kVtcNRW];
#pragma unroll
                for (int n0 = 0; n0 < kVtcNRW; n0 += 16) {
                    float t16[16];
                    tmem_ld16(tbase + lane_base + (uint32_t)s * kStageCols + (uint32_t)(r0 + n0), t16);
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) v[n0 + jj] = t16[jj];
                    if (NS) {
                        tmem_ld16(tbase + lane_base + (uint32_t)s * kStageCols + (uint32_t)(kVtcRows + r0 + n0), t16);
#pragma unroll
                        for (int jj = 0; jj < 16; jj++) v[n0 + jj] += t16[jj];
                    }
                }
                tc_fence_before();
                mbar_arrive(&d_free[s]);
                if (P.ph) {   // strip-major planes: hi [plane][strip][H][32] fp16, lo [plane][strip][H][32] e4m3
                    if (yt + r0 < P.H) {   // (columns past W hold exact zeros: b = 0 there)
                        // hi: rows r, r + 1 at a time: after one exchange with the partner lane (col ^ 1) an even
                        // lane holds row r's words of columns col, col + 1 and an odd lane row r + 1's of columns
                        // col - 1, col, so one warp store writes the two rows' 64-byte lines (128 contiguous bytes).
                        // lo: rows r .. r + 3 at a time: each lane packs its column's 4 bytes, a 4 x 4 byte transpose
                        // over lane groups of 4 leaves lane 4m + i with row r + i of columns 4m .. 4m + 3, so one
                        // warp store writes the four rows' 32-byte lines.
                        const int odd = col & 1;
                        const uint32_t sel = odd ? 0x3276u : 0x5410u;
                        const uint32_t sel1 = odd ? 0x3715u : 0x6240u, sel2 = (lane & 2) ? 0x3276u : 0x5410u;
                        const int nr = min(kVtcNRW, P.H - yt - r0);
                        const long long row0 = ((long long)(4 * k + q) * (P.Wp >> 5) + strip) * P.H + (yt + r0);
                        uint32_t* oh = reinterpret_cast<uint32_t*>(P.ph) + row0 * 16 + odd * 16 + (col >> 1);
                        uint32_t* ol = reinterpret_cast<uint32_t*>(P.pl) + row0 * 8 + (lane & 3) * 8 + (lane >> 2);
                        if (nr == kVtcNRW) {   // whole tile: packed residuals, no row tests, fixed store offsets
#pragma unroll
                            for (int jj = 0; jj < kVtcNRW; jj += 4) {
                                unsigned long long q01, q23;
                                const uint32_t h01 = split_f16x2_res2(pack2(v[jj], v[jj + 1]), q01);
                                const uint32_t h23 = split_f16x2_res2(pack2(v[jj + 2], v[jj + 3]), q23);
                                float l0, l1, l2, l3;
                                unpack2(q01, l0, l1);
                                unpack2(q23, l2, l3);
                                const uint32_t p01 = __shfl_xor_sync(0xffffffffu, h01, 1);
                                const uint32_t p23 = __shfl_xor_sync(0xffffffffu, h23, 1);
                                const uint32_t lw = cvt_e4m3x2(l1, l0) | (cvt_e4m3x2(l3, l2) << 16);
                                const uint32_t a = __byte_perm(lw, __shfl_xor_sync(0xffffffffu, lw, 1), sel1);
                                const uint32_t b = __byte_perm(a, __shfl_xor_sync(0xffffffffu, a, 2), sel2);
                                oh[jj * 16] = __byte_perm(h01, p01, sel);
                                oh[(jj + 2) * 16] = __byte_perm(h23, p23, sel);
                                ol[jj * 8] = b;
                            }
                        } else {
#pragma unroll
                            for (int jj = 0; jj < kVtcNRW; jj += 4) {
                                float l0, l1, l2, l3;
                                const uint32_t h01 = split_f16x2_res(v[jj], v[jj + 1], l0, l1);
                                const uint32_t h23 = split_f16x2_res(v[jj + 2], v[jj + 3], l2, l3);
                                const uint32_t p01 = __shfl_xor_sync(0xffffffffu, h01, 1);
                                const uint32_t p23 = __shfl_xor_sync(0xffffffffu, h23, 1);
                                const uint32_t lw = cvt_e4m3x2(l1 * kLoScale, l0 * kLoScale) |
                                                    (cvt_e4m3x2(l3 * kLoScale, l2 * kLoScale) << 16);
                                const uint32_t a = __byte_perm(lw, __shfl_xor_sync(0xffffffffu, lw, 1), sel1);
                                const uint32_t b = __byte_perm(a, __shfl_xor_sync(0xffffffffu, a, 2), sel2);
                                if (jj + odd < nr) oh[jj * 16] = __byte_perm(h01, p01, sel);
                                if (jj + 2 + odd < nr) oh[(jj + 2) * 16] = __byte_perm(h23, p23, sel);
                                if (jj + (lane & 3) < nr) ol[jj * 8] = b;
                            }
                        }
                    }
                } else if (x < P.W && yt + r0 < P.H) {
                    const int nr = min(kVtcNRW, P.H - yt - r0);
                    float* o = base + (long long)(yt + r0) * step;
                    if (nr == kVtcNRW) {   // whole tile: a running pointer, no per-row predicate
#pragma unroll
                        for (int jj = 0; jj < kVtcNRW; jj++) {
                            o[0] = v[jj] * inv;
                            o += step;
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < kVtcNRW; jj++) {
                            if (jj < nr) o[0] = v[jj] * inv;
                            o += step;
                        }
                    }
                }
            }
        }
    } else if (warp == kVtcProd / 32 + kVtcCons) {   // ------------------------------ MMA warp ---------
        {
            // the whole warp runs the loop (warp-uniform values in uniform registers) and one elected lane
            // issues: 32-bit incremental index math only (the ring slot of the tile's first chunk advances by
            // 8 per tile and by 8 TU + 6 per unit, modulo the ring)
            const uint32_t idesc = umma_idesc_f16(kVtcM, kVtcRows), idesc_s = umma_idesc_f16(kVtcM, 2 * kVtcRows);
            const uint64_t dz = umma_desc(0, kVtcZChunkBytes, 128),
                           dt = umma_desc(0, (NS ? 2 : 1) * kVtcRows * 16, 128);
            const uint32_t tH = smem_u32(Th), tL = smem_u32(Tl), zH = smem_u32(ZH), zL = smem_u32(ZL);
            const int per_unit = (8 * TU + 6) % kVtcZChunks;
            int ubase = (int)((long long)0 % kVtcZChunks);
            int s = 0, wrap = 0;   // stage = it % kVtcStages, phase parity = (it / kVtcStages) & 1
            long long it = 0;
            for (long long ui = 0; ui < nui; ui++) {
                int base = ubase;
                for (int j = 0; j < TU; j++, it++) {
                    mbar_wait(&z_full[s], (uint32_t)wrap);
                    if (it >= kVtcStages) mbar_wait(&d_free[s], (uint32_t)(wrap ^ 1));
                    tc_fence_after();
                    const uint32_t td = tbase + (uint32_t)s * kStageCols;
                    int slot = base;
                    for (int ks = 0; ks < Kp / 16; ks++) {
                        const uint32_t oz = (uint32_t)slot * (uint32_t)kVtcZChunkBytes;
                        const uint32_t ot = (uint32_t)ks * ((NS ? 4u : 2u) * kVtcRows * 16u);
                        const uint64_t aL = dz | (uint64_t)(((zL + oz) >> 4) & 0x3FFFu);
                        const uint64_t aH = dz | (uint64_t)(((zH + oz) >> 4) & 0x3FFFu);
                        const uint64_t bH = dt | (uint64_t)(((tH + ot) >> 4) & 0x3FFFu);   // NS: rows 0..63 of the stack
                        if (NS) {
                            umma_f16_warp(td, aH, bH, idesc_s, ks > 0 ? 1u : 0u);   // z_hi [T_hi; T_lo]^T
                            umma_f16_warp(td, aL, bH, idesc, 1u);                   // z_lo T_hi^T
                        } else {
                            const uint64_t bL = dt | (uint64_t)(((tL + ot) >> 4) & 0x3FFFu);
                            umma_f16_warp(td, aL, bH, idesc, ks > 0 ? 1u : 0u);
                            umma_f16_warp(td, aH, bL, idesc, 1u);
                            umma_f16_warp(td, aH, bH, idesc, 1u);
                        }
                        slot += 2;
                        if (slot >= kVtcZChunks) slot -= kVtcZChunks;
                    }
                    umma_commit_warp(&z_free[s]);
                    umma_commit_warp(&d_full[s]);
                    base += 8;
                    if (base >= kVtcZChunks) base -= kVtcZChunks;
                    if (++s == kVtcStages) {
                        s = 0;
                        wrap ^= 1;
                    }
                }
                ubase += per_unit;
                if (ubase >= kVtcZChunks) ubase -= kVtcZChunks;
            }
        }
    } else if (lane == 0) {   // ------------------------------------------------------- TMA warp -----
        // the CTA's raw chunks in order; chunk g waits for the release of chunk g - kVtcRaw (its ring slot)
        const long long nchunk = nui * (TU + 1);
        for (long long g = 0; g < nchunk; g++) {
            const long long ui = g / (TU + 1);
            const int c = (int)(g - ui * (TU + 1));
            int strip, k, ys;
            unit_of(ui, strip, k, ys);
            const int sl = (int)(g % kVtcRaw);
            if (g >= kVtcRaw) mbar_wait_backoff(&c_free[sl], (uint32_t)((g / kVtcRaw) - 1) & 1u, P.csleep);
            mbar_arrive_expect_tx(&c_full[sl], kSlotBytes);
            tma_load_3d(ring + (size_t)sl * (64 * 96), &tm_p, &c_full[sl], strip * 96, ys - R + 64 * c, 0);
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
