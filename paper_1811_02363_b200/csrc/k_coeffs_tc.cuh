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
// One CTA = two warpgroups (256 threads), persistent over tiles of 128 consecutive pixels; thread
// (h, m) = (tid / 128, tid % 128) serves pixel row m and half h of the K coefficients:
//   1. it evaluates b_l(i), l in its half, for pixel i = 128 t + m (exp2) and writes b_hi, b_lo into row
//      m of the A operands (canonical K-major no-swizzle layout: 8 x 16-byte core matrices);
//   2. one thread issues 3 (K/8) MMAs of M = 128, N = round_up(K, 16), K-step 8 and commits them to an
//      mbarrier;
//   3. warp w reads TMEM lanes 32 (w % 4) .. + 31 (its quarter), columns of its half, with tcgen05.ld
//      (16 at a time) and stores c_k(i) to the coefficient planes (coalesced over m).
// A^+ (hi, lo) is staged once per CTA as the B operands.  Two CTAs per SM (16 warps) hide the exp2 /
// shared-memory latency of step 1 and the stores of step 3.
#pragma once
#include "hdf_common.cuh"
#include "k_coeffs.cuh"

namespace hdf {

constexpr int kTcThreads = 256;   // two warpgroups: thread (h, m) <-> accumulator row / TMEM lane m, half h
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

// Dynamic shared memory: B_hi, B_lo [N][Kr], A_hi, A_lo [128][Kr], centres [N][rho].
inline __host__ __device__ size_t coeffs_tc_smem(int K, int rho) {
    const int Kr = (K + 7) & ~7, N = (K + 15) & ~15;
    return (size_t)(2 * N + 2 * kTcM) * Kr * 4 + (size_t)N * rho * 4 + 64;
}

template <int RHO>   // RHO > 0: compile-time guide dimension, 0: runtime
__global__ void __launch_bounds__(kTcThreads, 2) k_coeffs_tc(const __grid_constant__ CoefParams P) {
    extern __shared__ __align__(128) unsigned char sm_tc[];
    __shared__ uint64_t mma_done;
    __shared__ uint32_t tmem_base_sh;
    constexpr int RR = RHO > 0 ? RHO : 1;
    const int K = P.K, rho = RHO > 0 ? RHO : P.rho;
    const int Kr = (K + 7) & ~7, N = (K + 15) & ~15;
    const int tid = threadIdx.x, warp = tid >> 5;
    unsigned char* Bh = sm_tc;
    unsigned char* Bl = Bh + (size_t)N * Kr * 4;
    unsigned char* Ah = Bl + (size_t)N * Kr * 4;
    unsigned char* Al = Ah + (size_t)kTcM * Kr * 4;
    float* mus = reinterpret_cast<float*>(Al + (size_t)kTcM * Kr * 4);
    const uint32_t ncols = N <= 32 ? 32u : 64u;

    // A^+ (hi, lo) as the B operands: row n = output coefficient n, K index l; zero-padded
    for (int e = tid; e < N * Kr; e += kTcThreads) {
        const int nn = e / Kr, l = e - nn * Kr;
        const float a = (nn < K && l < K) ? P.Ap32[nn * K + l] : 0.f;
        const uint32_t h = tf32_hi(a);
        *reinterpret_cast<uint32_t*>(Bh + tc_off(nn, l, Kr)) = h;
        *reinterpret_cast<uint32_t*>(Bl + tc_off(nn, l, Kr)) = tf32_lo(a, h);
    }
    for (int e = tid; e < N * rho; e += kTcThreads) mus[e] = (e < K * rho) ? P.centres[e] : 0.f;
    if (tid == 0) {
        mbar_init(&mma_done, 1);
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
    const uint32_t idesc = umma_idesc_tf32(kTcM, N);
    const uint32_t sbo = (uint32_t)Kr * 32u, lbo = 128u;
    const uint32_t aH = smem_u32(Ah), aL = smem_u32(Al), bH = smem_u32(Bh), bL = smem_u32(Bl);

    const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;
    const long long npix = (long long)P.H * P.W;
    const long long ntile = (npix + kTcM - 1) / kTcM;
    uint32_t phase = 0;
    const int m = tid & (kTcM - 1), half = tid >> 7;
    // compile-time rho: the guide values of the CTA's next tile are loaded while this tile's MMAs run
    float xn[RR];
    auto load_x = [&](long long tile) {
        const long long ii = tile * kTcM + m;
#pragma unroll
        for (int d = 0; d < RR; d++) xn[d] = (ii < npix) ? __ldg(P.p + ii * RR + d) : 0.f;
    };
    if (RHO > 0) load_x(blockIdx.x);
    for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        // 1. b(i) for this thread's pixel and half, split into the A operands' row m
        const long long i = tile * kTcM + m;
        const bool valid = i < npix;
        float x[RR];
        if (RHO > 0) {
#pragma unroll
            for (int d = 0; d < RR; d++) x[d] = xn[d];
        }
        const int lh = ((Kr / 4 + 1) / 2) * 4;   // the first half's columns (a multiple of 4)
        const int la = half ? lh : 0, lb = half ? Kr : lh;
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
                        for (int d = 0; d < rho; d++) {
                            const float t = __ldg(P.p + i * rho + d) - mu[d];
                            d2 = fmaf(t, t, d2);
                        }
                    }
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(d2 * c2));
                }
                h[u] = tf32_hi(b);
                q[u] = tf32_lo(b, h[u]);
            }
            const uint32_t off = tc_off(m, l0, Kr);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aH + off), "r"(h[0]), "r"(h[1]), "r"(h[2]),
                         "r"(h[3])
                         : "memory");
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(aL + off), "r"(q[0]), "r"(q[1]), "r"(q[2]),
                         "r"(q[3])
                         : "memory");
        }
        fence_proxy_async();   // generic-proxy writes of A -> visible to the tensor core
        tc_fence_before();     // (the previous tile's tcgen05.ld are complete: wait::ld in tmem_ld16)
        __syncthreads();
        // 2. one thread issues the MMAs: D = b_lo A_hi^T + b_hi A_lo^T + b_hi A_hi^T
        if (tid == 0) {
            tc_fence_after();
            for (int s = 0; s < Kr / 8; s++) {
                const uint32_t ko = (uint32_t)s * 256u;   // two 16-byte core matrices per K step of 8
                umma_tf32(tbase, umma_desc(aL + ko, lbo, sbo), umma_desc(bH + ko, lbo, sbo), idesc, s > 0 ? 1u : 0u);
                umma_tf32(tbase, umma_desc(aH + ko, lbo, sbo), umma_desc(bL + ko, lbo, sbo), idesc, 1u);
                umma_tf32(tbase, umma_desc(aH + ko, lbo, sbo), umma_desc(bH + ko, lbo, sbo), idesc, 1u);
            }
            umma_commit(&mma_done);
        }
        if (RHO > 0 && tile + gridDim.x < ntile) load_x(tile + gridDim.x);
        // 3. the accumulator row of this thread's pixel -> coefficient planes
        mbar_wait(&mma_done, phase);
        phase ^= 1u;
        tc_fence_after();
        const uint32_t trow = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
        long long y = 0, xx = 0;
        if (valid) {
            y = i / P.W;
            xx = i - y * P.W;
        }
        float* o = P.cpl + y * P.Wp + xx;
        const int nh = ((N / 16 + 1) / 2) * 16;   // the first half's columns (a multiple of 16)
        for (int n0 = half ? nh : 0; n0 < (half ? N : nh); n0 += 16) {
            float v[16];
            tmem_ld16(trow + (uint32_t)n0, v);
            if (valid) {
#pragma unroll
                for (int j = 0; j < 16; j++)
                    if (n0 + j < K) o[(long long)(n0 + j) * P.cstride] = v[j];
            }
        }
        tc_fence_before();
        __syncthreads();   // every lane's tcgen05.ld is done before the next tile's MMAs overwrite D,
                           // and the A operands are no longer read
    }
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols) : "memory");
    }
}

}  // namespace hdf
