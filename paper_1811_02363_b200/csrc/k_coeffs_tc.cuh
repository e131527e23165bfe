// k_coeffs_tc.cuh -- Algorithm 1 loop for2 on the 5th-generation tensor cores:
//   c(i) = A^+ b(i),  b_l(i) = phi(p(i) - mu_l) (defAb),
// for all pixels as one contraction C[pixels x K] = Bm[pixels x K] . (A^+)^T, issued with tcgen05.mma
// (kind::tf32) from shared-memory operands into a TMEM accumulator and read back with tcgen05.ld.
//
// Accuracy (fp32-level, as the CUDA-core and mma.sync kernels it replaces): every operand x is split
// x = hi + lo, hi = x with the low 13 mantissa bits cleared (exact in TF32), lo = x - hi (exact in fp32;
// the tensor core reads its top 19 bits, so hi + lo carries x to ~2^-21 relative), and
//   C = b_lo A_hi^T + b_hi A_lo^T + b_hi A_hi^T   (fp32 accumulation in TMEM, small terms first).
//
// Warp-specialised, double-buffered pipeline, one CTA of three warpgroups per SM (persistent over tiles
// of 128 consecutive pixels; tile t uses stage s = t % 2 of the A operands and of the TMEM accumulator):
//   * producers (warpgroups 0 and 1): thread (h, m) evaluates b_l(i) for pixel i = 128 t + m and the
//     half h of l (exp2; for rho = 3 its 32 centres live in registers and the 32 evaluations are
//     independent), splits it, writes row m of A_hi[s], A_lo[s] (canonical K-major no-swizzle layout:
//     8 x 16-byte core matrices) and arrives on the mbarrier A[s] full;
//   * the MMA warp (one elected thread): waits for A[s] full and D[s] free, issues the 3 (K/8) MMAs of
//     M = 128, N = round_up(K, 16), K-step 8 into D[s] and commits them to two mbarriers (A[s] free,
//     D[s] full);
//   * consumers (warpgroups 2 and 3, coefficients 0..31 and 32..63): warp w reads TMEM lanes
//     32 (w % 4) .. + 31 of D[s] (its pixels' rows) with tcgen05.ld, releases D[s] (mbarrier) and stores
//     c_k(i) to the coefficient planes (coalesced over m) while the producers already compute tile t + 1
//     (one consumer warpgroup was the bottleneck: 64 stores per pixel).
// A^+ (hi, lo) is staged once per CTA as the B operands.
#pragma once
#include "hdf_common.cuh"
#include "k_coeffs.cuh"

namespace hdf {

constexpr int kTcProd = 256;      // producer threads: (half h, pixel row m)
constexpr int kTcThreads = 544;   // + two consumer warpgroups (columns 0..31, 32..63) + one MMA-issuing warp
constexpr int kTcM = 128;         // pixels per MMA tile (UMMA M)
constexpr int kTcMaxK = 64;       // N = round_up(K, 16) <= 64 (larger K: the CUDA-core kernels)

// Shared-memory descriptor of a K-major, no-swizzle operand (canonical layout ((8, m), 2) :
// ((16 B, SBO), LBO)): start address, leading byte offset (between the two 16-byte core matrices
// of one 8-element K step), stride byte offset (between 8-row groups); version 1 (sm_100).
HDF_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Instruction descriptor: kind::tf32, D fp32, A and B TF32 K-major, shape M x N.
HDF_DEV uint32_t umma_idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
HDF_DEV void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
HDF_DEV void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
HDF_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
HDF_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 16 consecutive fp32 columns of this thread's TMEM lane
HDF_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] = __uint_as_float(r[j]);
}

// Byte offset of element (row, k) in a K-major no-swizzle operand with Kr (multiple of 8) columns:
// core matrix (row / 8, k / 4) of 8 rows x 16 bytes, K-adjacent core matrices 128 B apart (LBO),
// 8-row groups Kr * 32 B apart (SBO).
HDF_DEV uint32_t tc_off(int row, int k, int Kr) {
    return (uint32_t)((row >> 3) * (Kr * 32) + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

// Dynamic shared memory: B_hi, B_lo [N][Kr], 2 stages of A_hi, A_lo [128][Kr], centres [N][rho].
inline __host__ __device__ size_t coeffs_tc_smem(int K, int rho) {
    const int Kr = (K + 7) & ~7, N = (K + 15) & ~15;
    // (+ the tile's guide rows [128][rho] for a runtime rho: read once per tile instead of once per centre)
    // (+ the centres once more, pair-interleaved, for the packed rho = 3 evaluations)
    return (size_t)(2 * N + 4 * kTcM) * Kr * 4 + (size_t)2 * N * rho * 4 + (size_t)kTcM * rho * 4 + 64;
}

template <int RHO>   // RHO > 0: compile-time guide dimension, 0: runtime
__global__ void __launch_bounds__(kTcThreads, 1) k_coeffs_tc(const __grid_constant__ CoefParams P) {
    extern __shared__ __align__(128) unsigned char sm_tc[];
    __shared__ uint64_t a_full[2], a_free[2], d_full[2], d_free[2];
    __shared__ uint32_t tmem_base_sh;
    constexpr int RR = RHO > 0 ? RHO : 1;
    const int K = P.K, rho = RHO > 0 ? RHO : P.rho;
    const int Kr = (K + 7) & ~7, N = (K + 15) & ~15;
    const int tid = threadIdx.x, warp = tid >> 5;
    const size_t abytes = (size_t)kTcM * Kr * 4;
    unsigned char* Bh = sm_tc;
    unsigned char* Bl = Bh + (size_t)N * Kr * 4;
    unsigned char* A0 = Bl + (size_t)N * Kr * 4;   // stage s: A_hi at A0 + 2 s abytes, A_lo after it
    float* mus = reinterpret_cast<float*>(A0 + 4 * abytes);
    float* mup = mus + (size_t)N * rho;  // centre pairs [N / 2][rho][2]: (mu_{2i}[d], mu_{2i+1}[d]) adjacent (one LDS.64)
    float* xs = mup + (size_t)N * rho;   // runtime rho: the tile's guide rows [128][rho]
    const uint32_t ncols = N <= 32 ? 64u : 128u;   // two accumulator stages of N (<= 64) columns

    // A^+ (hi, lo) as the B operands: row n = output coefficient n, K index l; zero-padded
    for (int e = tid; e < N * Kr; e += kTcThreads) {
        const int nn = e / Kr, l = e - nn * Kr;
        const float a = (nn < K && l < K) ? P.Ap32[nn * K + l] : 0.f;
        const uint32_t h = tf32_hi(a);
        *reinterpret_cast<uint32_t*>(Bh + tc_off(nn, l, Kr)) = h;
        *reinterpret_cast<uint32_t*>(Bl + tc_off(nn, l, Kr)) = tf32_lo(a, h);
    }
    for (int e = tid; e < N * rho; e += kTcThreads) {
        const float m = (e < K * rho) ? P.centres[e] : 0.f;
        const int l = e / rho, d = e - l * rho;
        mus[e] = m;
        mup[((l >> 1) * rho + d) * 2 + (l & 1)] = m;
    }
    if (tid == 0) {
        for (int s = 0; s < 2; s++) {
            mbar_init(&a_full[s], kTcProd);
            mbar_init(&a_free[s], 1);
            mbar_init(&d_full[s], 1);
            mbar_init(&d_free[s], 2 * kTcM);
        }
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();   // the B operands are read by the tensor core (async proxy)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_sh;
    const long long npix = (long long)P.H * P.W;
    const long long ntile = (npix + kTcM - 1) / kTcM;
    const uint32_t dcols = ncols / 2;

    if (tid < kTcProd) {   // ------------------------------------------------ producers --------
        const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;
        const int m = tid & (kTcM - 1), half = tid >> 7;
        const int lh = ((Kr / 4 + 1) / 2) * 4;   // the first half's columns (a multiple of 4, <= 32)
        const int la = half ? lh : 0, lb = half ? Kr : lh;
        // rho = 3: the half's 32 evaluations fully unrolled (independent; centre loads at fixed offsets)
        constexpr bool MUREG = (RHO == 3);
        // compile-time rho: the guide values of the next tile are loaded one tile ahead
        float xn[RR];
        auto load_x = [&](long long tile) {
            const long long ii = tile * kTcM + m;
#pragma unroll
            for (int d = 0; d < RR; d++) xn[d] = (ii < npix) ? __ldg(P.p + ii * RR + d) : 0.f;
        };
        if (RHO > 0) load_x(blockIdx.x);
        int it = 0;
        for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x, it++) {
            const int s = it & 1;
            const uint32_t ph = (uint32_t)(it >> 1) & 1u;
            const long long i = tile * kTcM + m;
            const bool valid = i < npix;
            float x[RR];
            if (RHO > 0) {
#pragma unroll
                for (int d = 0; d < RR; d++) x[d] = xn[d];
                if (tile + gridDim.x < ntile) load_x(tile + gridDim.x);
            }
            if (RHO == 0) {   // runtime rho: the tile's guide rows staged once, coalesced (they are contiguous)
                named_sync(2, kTcProd);   // the previous tile's rows have been read by both halves
                const long long t0 = tile * kTcM;
                const int nf = (int)(min((long long)kTcM, npix - t0) * rho);
                for (int e = tid; e < nf; e += kTcProd) xs[e] = __ldg(P.p + t0 * rho + e);
                named_sync(2, kTcProd);
            }
            mbar_wait(&a_free[s], ph ^ 1u);   // the MMAs of tile it - 2 have read A[s]
            const uint32_t aH = smem_u32(A0 + 2 * s * abytes), aL = aH + (uint32_t)abytes;
            if (MUREG) {   // packed f32x2 arithmetic on centre pairs (l, l + 1): la and lb are multiples of 4
                const unsigned long long xp0 = pack2(x[0], x[0]), xp1 = pack2(x[1 % RR], x[1 % RR]),
                                         xp2 = pack2(x[2 % RR], x[2 % RR]), c2p = pack2(c2, c2);
                const float* mq = mup + la * RR;
#pragma unroll
                for (int j0 = 0; j0 < 32; j0 += 4) {
                    if (la + j0 < lb) {
                        uint32_t h[4], q[4];
#pragma unroll
                        for (int u = 0; u < 4; u += 2) {
                            const int j = j0 + u;
                            const float* mp = mq + j * RR;   // pair (la + j) / 2: [d][2]
                            const unsigned long long t0 = fsub2(xp0, *reinterpret_cast<const unsigned long long*>(mp));
                            const unsigned long long t1 = fsub2(xp1, *reinterpret_cast<const unsigned long long*>(mp + 2));
                            const unsigned long long t2 = fsub2(xp2, *reinterpret_cast<const unsigned long long*>(mp + 4));
                            const unsigned long long d2 = ffma2(t2, t2, ffma2(t1, t1, fmul2(t0, t0)));
                            float a0, a1, b0, b1;
                            unpack2(fmul2(d2, c2p), a0, a1);
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b0) : "f"(a0));
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b1) : "f"(a1));
                            b0 = (valid && la + j < K) ? b0 : 0.f;
                            b1 = (valid && la + j + 1 < K) ? b1 : 0.f;
                            h[u] = tf32_hi(b0);
                            h[u + 1] = tf32_hi(b1);
                            float l0, l1;
                            unpack2(fsub2(pack2(b0, b1), pack2(__uint_as_float(h[u]), __uint_as_float(h[u + 1]))), l0, l1);
                            q[u] = __float_as_uint(l0);
                            q[u + 1] = __float_as_uint(l1);
                        }
                        const uint32_t off = tc_off(m, la + j0, Kr);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aH + off), "r"(h[0]), "r"(h[1]),
                                     "r"(h[2]), "r"(h[3])
                                     : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aL + off), "r"(q[0]), "r"(q[1]),
                                     "r"(q[2]), "r"(q[3])
                                     : "memory");
                    }
                }
            } else {
#pragma unroll 2
                for (int l0 = la; l0 < lb; l0 += 4) {
                    uint32_t h[4], q[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int l = l0 + u;
                        float b = 0.f;
                        if (valid && l < K) {
                            const float* mu = mus + l * rho;
                            float d2 = 0.f;
                            if (RHO > 0) {
#pragma unroll
                                for (int d = 0; d < RR; d++) {
                                    const float t = x[d] - mu[d];
                                    d2 = fmaf(t, t, d2);
                                }
                            } else {
                                const float* xr = xs + m * rho;
                                for (int d = 0; d < rho; d++) {
                                    const float t = xr[d] - mu[d];
                                    d2 = fmaf(t, t, d2);
                                }
                            }
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(d2 * c2));
                        }
                        h[u] = tf32_hi(b);
                        q[u] = tf32_lo(b, h[u]);
                    }
                    const uint32_t off = tc_off(m, l0, Kr);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aH + off), "r"(h[0]), "r"(h[1]),
                                 "r"(h[2]), "r"(h[3])
                                 : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aL + off), "r"(q[0]), "r"(q[1]),
                                 "r"(q[2]), "r"(q[3])
                                 : "memory");
                }
            }
            fence_proxy_async();   // generic-proxy writes of A[s] -> visible to the tensor core
            mbar_arrive(&a_full[s]);
        }
    } else if (warp == (kTcProd + 2 * kTcM) / 32) {   // ------------------------ MMA warp ----------
        if ((tid & 31) == 0) {    // D = b_lo A_hi^T + b_hi A_lo^T + b_hi A_hi^T into D[s]
            const uint32_t idesc = umma_idesc_tf32(kTcM, N);
            const uint32_t sbo = (uint32_t)Kr * 32u, lbo = 128u;
            const uint32_t bH = smem_u32(Bh), bL = smem_u32(Bl);
            int it = 0;
            for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x, it++) {
                const int s = it & 1;
                const uint32_t ph = (uint32_t)(it >> 1) & 1u;
                mbar_wait(&a_full[s], ph);          // the producers wrote A[s]
                mbar_wait(&d_free[s], ph ^ 1u);     // the consumer has read D[s] of tile it - 2
                tc_fence_after();
                const uint32_t aH = smem_u32(A0 + 2 * s * abytes), aL = aH + (uint32_t)abytes;
                const uint32_t td = tbase + (uint32_t)s * dcols;
                for (int k8 = 0; k8 < Kr / 8; k8++) {
                    const uint32_t ko = (uint32_t)k8 * 256u;   // two 16-byte core matrices per K step of 8
                    umma_tf32(td, umma_desc(aL + ko, lbo, sbo), umma_desc(bH + ko, lbo, sbo), idesc, k8 > 0 ? 1u : 0u);
                    umma_tf32(td, umma_desc(aH + ko, lbo, sbo), umma_desc(bL + ko, lbo, sbo), idesc, 1u);
                    umma_tf32(td, umma_desc(aH + ko, lbo, sbo), umma_desc(bH + ko, lbo, sbo), idesc, 1u);
                }
                umma_commit(&a_free[s]);
                umma_commit(&d_full[s]);
            }
        }
    } else {               // ------------------------------------------------ consumer ---------
        // warpgroup cw (warps 8..11, 12..15) stores the coefficients n = 32 cw .. 32 cw + 31; warp & 3 is
        // the TMEM lane quarter (pixel m)
        const int cw = (tid - kTcProd) >> 7, m = (tid - kTcProd) & (kTcM - 1);
        const int n0 = 32 * cw;
        const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
        int it = 0;
        for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x, it++) {
            const int s = it & 1;
            const uint32_t ph = (uint32_t)(it >> 1) & 1u;
            const long long i = tile * kTcM + m;
            const bool valid = i < npix;
            long long y = 0, xx = 0;
            if (valid) {
                if (npix <= 0x7fffffffLL) {   // 32-bit division (the 64-bit one was 5% of this kernel's stall samples)
                    const unsigned yi = (unsigned)i / (unsigned)P.W;
                    y = yi;
                    xx = (unsigned)i - yi * (unsigned)P.W;
                } else {
                    y = i / P.W;
                    xx = i - y * P.W;
                }
            }
            float* o = P.cpl + (long long)n0 * P.cstride + y * P.Wp + xx;
            mbar_wait(&d_full[s], ph);
            tc_fence_after();
            float v[32];
            if (n0 < N) {
                float t16[16];
                tmem_ld16(tbase + lane_base + (uint32_t)s * dcols + (uint32_t)n0, t16);
#pragma unroll
                for (int j = 0; j < 16; j++) v[j] = t16[j];
                if (n0 + 16 < N) {
                    tmem_ld16(tbase + lane_base + (uint32_t)s * dcols + (uint32_t)(n0 + 16), t16);
#pragma unroll
                    for (int j = 0; j < 16; j++) v[16 + j] = t16[j];
                }
            }
            tc_fence_before();
            mbar_arrive(&d_free[s]);
            if (P.ch) {   // 24-bit planes (CoefParams): packed over lane pairs (hi 16 bits) and lane quads (the byte)
                // the lane's pixel i has x = lane (mod 4) (W % 4 == 0, tiles of 128 pixels), so a lane pair / quad is a
                // pixel pair / quad of one row, all valid or all invalid; every lane runs the shuffles
                const int lane = tid & 31, odd = lane & 1, l3 = lane & 3;
                const int nn = min(32, K - n0);
                const long long pb = y * P.Wp + xx;
                // plane n0 + odd, pixels (x - odd, x - odd + 1): one 32-bit word; two planes further per pair
                uint32_t* oh = reinterpret_cast<uint32_t*>(P.ch + (long long)(n0 + odd) * P.cstride + (pb - odd));
                // plane n0 + l3, pixels x - l3 .. x - l3 + 3: one 32-bit word; four planes further per group
                uint32_t* om = reinterpret_cast<uint32_t*>(P.cm + (long long)(n0 + l3) * P.cstride + (pb - l3));
                const uint32_t sel1 = odd ? 0x3715u : 0x6240u, sel2 = (lane & 2) ? 0x3276u : 0x5410u;
#pragma unroll
                for (int n = 0; n < 32; n += 4) {
                    uint32_t e[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const uint32_t w = __float_as_uint(v[n + u]);
                        const uint32_t m = ((w & 0xFFFFu) * 255u + 32768u) >> 16;
                        e[u] = __byte_perm(w, m, 0x3244);   // the stored value's bits: (hi16, m, m)
                    }
                    const uint32_t r01 = __shfl_xor_sync(0xffffffffu, odd ? e[0] : e[1], 1);
                    const uint32_t r23 = __shfl_xor_sync(0xffffffffu, odd ? e[2] : e[3], 1);
                    // even lane: (own coefficient n, partner's n) of pixels (x, x + 1); odd lane: (partner's n + 1, own)
                    const uint32_t h01 = __byte_perm(odd ? r01 : e[0], odd ? e[1] : r01, 0x7632);
                    const uint32_t h23 = __byte_perm(odd ? r23 : e[2], odd ? e[3] : r23, 0x7632);
                    // the bytes of coefficients n .. n + 3, then a 4 x 4 byte transpose over the lane quad: lane l3 ends
                    // with coefficient n + l3 of the quad's four pixels
                    const uint32_t lw = __byte_perm(__byte_perm(e[0], e[1], 0x0051), __byte_perm(e[2], e[3], 0x0051), 0x5410);
                    const uint32_t ta = __byte_perm(lw, __shfl_xor_sync(0xffffffffu, lw, 1), sel1);
                    const uint32_t tb = __byte_perm(ta, __shfl_xor_sync(0xffffffffu, ta, 2), sel2);
                    if (valid && n < nn) {
                        oh[0] = h01;
                        oh[P.cstride] = h23;   // (32-bit words: two planes of 16-bit values further)
                        om[0] = tb;
                    }
                    oh += 2 * P.cstride;
                    om += P.cstride;
                }
            } else if (valid) {
                const int nn = min(32, K - n0);
                if (nn == 32) {   // all 32 planes: no per-plane test
#pragma unroll
                    for (int n = 0; n < 32; n++) {
                        o[0] = v[n];
                        o += P.cstride;
                    }
                } else {
#pragma unroll
                    for (int n = 0; n < 32; n++) {
                        if (n < nn) o[0] = v[n];
                        o += P.cstride;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols) : "memory");
    }
}

}  // namespace hdf
