// k_vpass.cuh -- F1: fused range weights + vertical pass of the K(n+1) convolutions.
//
// Algorithm 1 loop for1 fused with the column half of the separable convolutions
// v_k = omega * u_k, r_k = omega * b_k:
//   b_k(j) = phi(p(j) - mu_k) = exp(-||p(j) - mu_k||^2 / 2 sigma_r^2),  u_k(j) = b_k(j) f(j),
//   t_q(y, x) = sum_{t=-R}^{R} w_t z_q(y - t, x),  z_q in {u_k channels, b_k}, plane q = k(n+1)+c,
// with rows outside [0, H) contributing zero (window clipped to Omega, R8).
//
// Layout: a CTA (512 threads) owns a 32-column strip, a row segment [y0, y1) and a group of NPL
// consecutive planes q.  PACK (2R + J <= 52): NPL = 32, thread (cp, pq) = (tid & 15, tid >> 4) owns
// columns x0 + 2cp, x0 + 2cp + 1 of plane q0 + pq and the FIR runs on packed column pairs (FFMA2 /
// FADD2, sm_100a) with the symmetric taps folded, out = w0 z_c + sum_{t=1..R} w_t (z_{c-t} + z_{c+t});
// otherwise (large R) NPL = 16, one column per thread, scalar FFMA.  Taps live in uniform registers.
// The CTA marches down the rows in steps of J rows:
//   * raw guide / image rows for step g + 2 are copied global -> shared with cp.async (no register
//     staging, latency hidden behind two steps of work);
//   * stage A: the J rows of b_k and u_k for step g + 1 from the raw rows -> shared (double buffered);
//   * stage B: the J rows of step g enter a register window of S = 2R + J rows that rotates by
//     position (the step loop is unrolled S/J times so every window index is a compile-time
//     register), and J outputs per column pair are written (coalesced float2 stores).
// One __syncthreads per step.
#pragma once
#include <type_traits>

#include "hdf_common.cuh"

namespace hdf {

constexpr int kVTX = 32;   // columns per CTA
constexpr int kVNT = 512;  // threads per CTA (256 for the packed large-radius kernels, vpass_nt)
// planes per CTA: 16 column pairs (packed) or 32 columns per plane
__host__ __device__ constexpr int vfir_npl(bool pack, int nt = kVNT) { return pack ? nt / 16 : nt / 32; }

struct VParams {
    const float* f;        // [H][W][n]
    const float* p;        // [H][W][rho]
    const float* centres;  // [K][rho]
    float* planes;         // [P][H][Wp]
    long long pstride;     // H * Wp
    int n, rho, H, W, Wp, K, NP, P;  // NP = n + 1 planes per cluster, P = K * NP
    int nstrip, ncol;      // 32-column strips; strips * plane groups
    int f_is_p;            // f aliases p (bilateral): the raw rows hold p only
    float neg_inv2sr2;     // -1 / (2 sigma_r^2)
    unsigned long long tw[HDF_MAX_RADIUS + 1];   // {w_t, w_t} packed, t = 0..R (box: ones)
    float tws[2 * HDF_MAX_RADIUS + 1];           // w_{-R..R} (scalar path)
};

// (packed f32x2 arithmetic: ffma2 / fadd2 / fsub2 / fmul2 / pack2 / unpack2 in hdf_common.cuh)
HDF_DEV unsigned long long lds_u64(const void* p) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)));
    return v;
}
HDF_DEV float lds_f32(const float* p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}
HDF_DEV void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
HDF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
HDF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Shared-memory layout (floats): mus [nkmax * rho, rounded to 4] | raw [2][J][32][RW] | zs [2][J][NPL][32]
inline __host__ __device__ int vfir_nkmax(int NP, int npl) { return (npl + NP - 1) / NP + 1; }

// J rows (from row y0) of a 32-pixel segment [x0, x0 + nx) of an [H][W][c] image -> dst [J][32][c]:
// 16-byte cp.async chunks when the segment is whole and rows are 16-byte aligned, else 4-byte ones.
template <int J, int NT>
HDF_DEV void vfir_copy_rows(float* dst, const float* src, int c, int W, int H, int y0, int x0, int nx) {
    if (nx == kVTX && (W * c) % 4 == 0) {
        const int cpr = 8 * c;   // 16-byte chunks per row (32 c floats)
        for (int e = threadIdx.x; e < J * cpr; e += NT) {
            const int r = e / cpr, w = e - r * cpr;
            const int y = y0 + r;
            if (y < 0 || y >= H) continue;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + r * kVTX * c + 4 * w)),
                         "l"(src + ((long long)y * W + x0) * c + 4 * w)
                         : "memory");
        }
    } else {
        const int per_row = nx * c;
        for (int e = threadIdx.x; e < J * per_row; e += NT) {
            const int r = e / per_row, w = e - r * per_row;
            const int y = y0 + r;
            if (y < 0 || y >= H) continue;
            cp_async4(dst + r * kVTX * c + w, src + ((long long)y * W + x0) * c + w);
        }
    }
}

// raw rows of step `step` (input rows ystart + step*J + r) -> raw buffer: [J][32][rho] when f is p,
// else [J][32][rho] guide rows followed by [J][32][n] image rows.
// When f aliases p the 32 pixels of a row are one contiguous run of 32*rho floats (16-byte copies when
// aligned); otherwise p and f are interleaved per pixel with 4-byte copies.
template <int J, int RHO, int NT>
HDF_DEV void vfir_issue_raw(const VParams& P, float* raw, int ystart, int step, int x0, int nx, int RW, bool vec) {
    const int rho = RHO > 0 ? RHO : P.rho;
    if (P.f_is_p) {
        const int per_row = nx * rho;
        if (vec) {   // nx == 32, W * rho % 4 == 0: rows of 8 rho 16-byte chunks
            const int cpr = 8 * rho;
            // (row, chunk) walked with a running pair instead of a division per element (rho = 31: an
            // integer division by 248 per 16-byte copy was 9% of the kernel's stall samples)
            int r = threadIdx.x / cpr, w = threadIdx.x - r * cpr;
            const int dr = NT / cpr, dw = NT - dr * cpr;
            for (int e = threadIdx.x; e < J * cpr; e += NT) {
                const int y = ystart + step * J + r;
                if (y >= 0 && y < P.H) {
                    const float* src = P.p + ((long long)y * P.W + x0) * rho + 4 * w;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     smem_u32(raw + r * kVTX * rho + 4 * w)),
                                 "l"(src)
                                 : "memory");
                }
                r += dr;
                w += dw;
                if (w >= cpr) {
                    w -= cpr;
                    r++;
                }
            }
        } else {
            for (int e = threadIdx.x; e < J * per_row; e += NT) {
                const int r = e / per_row, w = e - r * per_row;
                const int y = ystart + step * J + r;
                if (y < 0 || y >= P.H) continue;
                cp_async4(raw + r * kVTX * rho + w, P.p + ((long long)y * P.W + x0) * rho + w);
            }
        }
    } else {
        // f is not p: the guide rows [J][32][rho] and the image rows [J][32][n] in two arrays, each row
        // segment one contiguous run (16-byte copies when aligned)
        (void)RW;
        float* rawf = raw + J * kVTX * rho;
        vfir_copy_rows<J, NT>(raw, P.p, rho, P.W, P.H, ystart + step * J, x0, nx);
        vfir_copy_rows<J, NT>(rawf, P.f, P.n, P.W, P.H, ystart + step * J, x0, nx);
    }
    cp_async_commit();
}

// stage A: z rows of step `step` for planes [q0, q0 + NPL) -> zs[J][NPL planes][32 cols].
// Thread -> (column x, cluster kl, row phase h): it handles rows h, h + HS, ... of the step for one
// column and one cluster, with the cluster's centre in registers.  b = 2^(d2 * log2(e) * -1/2sr^2)
// (ex2.approx, relative error < 2^-21 over the range that matters).  RHO / NPC compile-time when > 0.
HDF_DEV float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Raw rows for the specialised path: [J][32][RHO] (pixel-major, as in memory).  A full strip whose rows
// are 16-byte aligned is copied in 16-byte chunks; rows / columns off the image are zero-filled (their
// b is 0, but 0 * garbage could be NaN).
template <int J, int RHO, int NT>
HDF_DEV void vfir_issue_raw_aos(const VParams& P, float* raw, int ystart, int step, int x0, int nx, bool vec) {
    constexpr int PR = kVTX * RHO;   // floats per row
    if (vec) {
        constexpr int CR = PR / 4;   // 16-byte chunks per row (RHO * 8)
        for (int e = threadIdx.x; e < J * CR; e += NT) {
            const int r = e / CR, c = e - r * CR;
            const int y = ystart + step * J + r;
            float* dst = raw + r * PR + 4 * c;
            if (y < 0 || y >= P.H) {
                asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(dst)), "f"(0.f) : "memory");
            } else {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
                             "l"(P.p + ((long long)y * P.W + x0) * RHO + 4 * c)
                             : "memory");
            }
        }
    } else {
        for (int e = threadIdx.x; e < J * PR; e += NT) {
            const int r = e / PR, w = e - r * PR;
            const int y = ystart + step * J + r;
            float* dst = raw + r * PR + w;
            if (y < 0 || y >= P.H || w >= nx * RHO) *dst = 0.f;
            else cp_async4(dst, P.p + ((long long)y * P.W + x0) * RHO + w);
        }
    }
    cp_async_commit();
}

// Specialised stage A: RHO, NPC compile-time and plane groups aligned to clusters (NPL % NPC == 0).
template <int J, int NPL, int RHO, int NPC, int NT>
HDF_DEV void vfir_stage_a_fast(const VParams& P, const float* raw, float* zs, const float* mus, int ystart, int step,
                               int x0, int nk) {
    // thread -> (column pair xp, cluster kl, row phase h); packed f32x2 arithmetic on the column pair
    constexpr int NK = NPL / NPC;                 // clusters per group
    constexpr int NW = NT / 16;                   // NT threads = 16 pairs x NK x HS
    constexpr int HS = (NW / NK) > 0 ? (NW / NK) : 1;
    constexpr int RPT = (J + HS - 1) / HS;
    const int xp = threadIdx.x & 15;
    const int w = threadIdx.x >> 4;               // 0..NW-1
    const int kl = w / HS, h = w - kl * HS;
    if (kl >= nk) return;
    const int xa = x0 + 2 * xp;
    const bool ok0 = xa < P.W, ok1 = xa + 1 < P.W;
    const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;
    unsigned long long mu2[RHO];
#pragma unroll
    for (int d = 0; d < RHO; d++) {
        const float m = lds_f32(mus + kl * RHO + d);
        uint32_t bits = __float_as_uint(m);
        mu2[d] = ((unsigned long long)bits << 32) | bits;
    }
    uint32_t cb = __float_as_uint(c2);
    const unsigned long long c22 = ((unsigned long long)cb << 32) | cb;
    const int ybase = ystart + step * J;
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        const int r = h + i * HS;
        if (RPT * HS != J && r >= J) break;
        const int y = ybase + r;
        const bool rowok = (y >= 0) && (y < P.H);
        const float* pp = raw + r * RHO * kVTX + 2 * xp * RHO;   // pixels 2xp, 2xp + 1: 2 RHO floats, 8-byte aligned
        float fv[2 * RHO];
#pragma unroll
        for (int e = 0; e < RHO; e++) {
            const unsigned long long v = lds_u64(pp + 2 * e);
            fv[2 * e] = __uint_as_float((uint32_t)v);
            fv[2 * e + 1] = __uint_as_float((uint32_t)(v >> 32));
        }
        unsigned long long xv[RHO];
        unsigned long long d2 = 0ull;
#pragma unroll
        for (int d = 0; d < RHO; d++) {
            xv[d] = ((unsigned long long)__float_as_uint(fv[RHO + d]) << 32) | __float_as_uint(fv[d]);
            const unsigned long long t = fsub2(xv[d], mu2[d]);
            d2 = ffma2(t, t, d2);
        }
        const unsigned long long e2 = ffma2(d2, c22, 0ull);
        const float b0 = (rowok && ok0) ? ex2_approx(__uint_as_float((uint32_t)e2)) : 0.f;
        const float b1 = (rowok && ok1) ? ex2_approx(__uint_as_float((uint32_t)(e2 >> 32))) : 0.f;
        const unsigned long long bb = ((unsigned long long)__float_as_uint(b1) << 32) | __float_as_uint(b0);
        float* zo = zs + (r * NPL + kl * NPC) * kVTX + 2 * xp;
#pragma unroll
        for (int c = 0; c < NPC; c++) {
            const unsigned long long z = (c < NPC - 1) ? ffma2(bb, xv[c], 0ull) : bb;   // b = 0 off the image
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(smem_u32(zo + c * kVTX)), "l"(z) : "memory");
        }
    }
}

template <int J, int NPL, int RHO, int NPC, int NT>
HDF_DEV void vfir_stage_a(const VParams& P, const float* raw, float* zs, const float* mus, int ystart, int step,
                          int x0, int q0, int kA, int nk, int RW) {
    const int rho = RHO > 0 ? RHO : P.rho;
    const int NP = NPC > 0 ? NPC : P.NP;
    const int n = NP - 1;
    const int x = threadIdx.x & (kVTX - 1);
    const int w = threadIdx.x >> 5;                 // 0..NT/32-1
    const int HS = max(1, (NT / 32) / nk);          // row phases per (column, cluster)
    const int kl = w / HS, h = w - kl * HS;
    if (kl >= nk) return;
    const int k = kA + kl;
    const bool xok = x0 + x < P.W;
    const float c2 = P.neg_inv2sr2 * 1.4426950408889634f;   // -log2(e) / 2 sigma_r^2
    constexpr int RR = RHO > 0 ? RHO : 1;
    float mu[RR];
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) mu[d] = lds_f32(mus + kl * rho + d);
    }
    const bool whole = NPC > 0 && q0 <= k * NPC && (k + 1) * NPC <= q0 + NPL;
    const int qa = max(k * NP, q0), qb = min((k + 1) * NP, q0 + NPL);
    for (int r = h; r < J; r += HS) {
        const int y = ystart + step * J + r;
        const bool valid = xok && (y >= 0) && (y < P.H);
        const float* pp = raw + (r * kVTX + x) * rho;
        float d2 = 0.f;
        if (RHO > 0) {
#pragma unroll
            for (int d = 0; d < RR; d++) {
                const float t = lds_f32(pp + d) - mu[d];
                d2 = fmaf(t, t, d2);
            }
        } else {   // runtime rho (large: 31 at config 3): four independent partial sums
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
            const float* mk = mus + kl * rho;
            int d = 0;
            for (; d + 4 <= rho; d += 4) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const float t = lds_f32(pp + d + u) - lds_f32(mk + d + u);
                    s4[u] = fmaf(t, t, s4[u]);
                }
            }
            for (; d < rho; d++) {
                const float t = lds_f32(pp + d) - lds_f32(mk + d);
                s4[0] = fmaf(t, t, s4[0]);
            }
            d2 = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        }
        const float b = valid ? ex2_approx(d2 * c2) : 0.f;
        const float* fp = P.f_is_p ? pp : raw + J * kVTX * rho + (r * kVTX + x) * n;
        float* zo = zs + (r * NPL - q0) * kVTX + x;
        if (whole) {
#pragma unroll
            for (int c = 0; c < (NPC > 0 ? NPC : 1); c++) {
                const float z = (c < NPC - 1) ? (valid ? b * lds_f32(fp + c) : 0.f) : b;
                zo[(k * NPC + c) * kVTX] = z;
            }
        } else {
            for (int q = qa; q < qb; q++) {
                const int c = q - k * NP;
                zo[q * kVTX] = (c < n) ? (valid ? b * lds_f32(fp + c) : 0.f) : b;
            }
        }
    }
}

// window element: a packed column pair (u64) or one column (float)
HDF_DEV unsigned long long wmul0(unsigned long long w, unsigned long long a) { return ffma2(w, a, 0ull); }
HDF_DEV float wmul0(float w, float a) { return w * a; }
HDF_DEV unsigned long long wfma(unsigned long long w, unsigned long long a, unsigned long long c) { return ffma2(w, a, c); }
HDF_DEV float wfma(float w, float a, float c) { return fmaf(w, a, c); }
HDF_DEV unsigned long long wadd(unsigned long long a, unsigned long long b) { return fadd2(a, b); }
HDF_DEV float wadd(float a, float b) { return a + b; }
HDF_DEV unsigned long long wsub(unsigned long long a, unsigned long long b) { return fsub2(a, b); }
HDF_DEV float wsub(float a, float b) { return a - b; }
HDF_DEV void wload(unsigned long long& v, const float* p) { v = lds_u64(p); }
HDF_DEV void wload(float& v, const float* p) { v = lds_f32(p); }
HDF_DEV void wstore(float* p, unsigned long long v) { *reinterpret_cast<unsigned long long*>(p) = v; }
HDF_DEV void wstore(float* p, float v) { *p = v; }

template <int R, int J, bool BOX, bool PACK, int RHO, int NPC, int NT>
HDF_DEV void vfir_segment(const VParams& P, float* sm_v, int strip, int group, int y0, int y1) {
    using WT = typename std::conditional<PACK, unsigned long long, float>::type;
    constexpr int NPL = vfir_npl(PACK, NT);
    constexpr int NCW = NT / NPL;            // column workers per plane (16 pairs or 32 columns)
    constexpr int CPW = kVTX / NCW;          // columns per worker (2 or 1)
    constexpr int S = 2 * R + J;
    constexpr int NSTEP = S / J;
    static_assert(S % J == 0, "J must divide 2R");
    const int q0 = group * NPL;
    const int kA = q0 / P.NP;
    const int kB = min(P.K - 1, (q0 + NPL - 1) / P.NP);
    const int nk = kB - kA + 1;
    const int rho = RHO > 0 ? RHO : P.rho;
    const int RW = P.f_is_p ? rho : rho + P.n;
    float* mus = sm_v;
    const int mus_len = (vfir_nkmax(P.NP, NPL) * rho + 3) & ~3;
    float* raw0 = sm_v + mus_len;
    const int raw_len = (J * kVTX * RW + 3) & ~3;
    float* zs0 = raw0 + 2 * raw_len;
    constexpr int zs_len = J * NPL * kVTX;
    __syncthreads();   // the previous segment is done with the shared buffers
    for (int e = threadIdx.x; e < nk * rho; e += NT) mus[e] = P.centres[kA * rho + e];

    const int tid = threadIdx.x;
    const int cw = tid % NCW, pq = tid / NCW;
    const int x0 = strip * kVTX;
    const int nx = min(kVTX, P.W - x0);
    const int xo = x0 + CPW * cw;
    const int q = q0 + pq;
    const bool active = (q < P.P) && (xo < P.Wp);
    const int ystart = y0 - R;
    const int nsteps = NSTEP - 1 + (y1 - y0 + J - 1) / J;
    float* outp = P.planes + (long long)q * P.pstride + xo;
    const bool vec = (nx == kVTX) && ((P.W * rho) % 4 == 0);

    WT win[S];
#pragma unroll
    for (int i = 0; i < S; i++) win[i] = WT(0);

    // prologue: raw rows of steps 0 and 1, z rows of step 0
    constexpr bool FAST = (RHO > 0) && (NPC > 0) && (NPL % (NPC > 0 ? NPC : 1) == 0) && (RHO == NPC - 1);
    const bool fast = FAST && P.f_is_p;
    auto issue = [&](float* dst, int step) {
        if (fast) vfir_issue_raw_aos<J, (RHO > 0 ? RHO : 1), NT>(P, dst, ystart, step, x0, nx, vec);
        else vfir_issue_raw<J, RHO, NT>(P, dst, ystart, step, x0, nx, RW, vec);
    };
    issue(raw0, 0);
    if (nsteps > 1) issue(raw0 + raw_len, 1);
    cp_async_wait_all();
    __syncthreads();
    if (fast) vfir_stage_a_fast<J, NPL, (RHO > 0 ? RHO : 1), (FAST ? NPC : 1), NT>(P, raw0, zs0, mus, ystart, 0, x0, nk);
    else vfir_stage_a<J, NPL, RHO, NPC, NT>(P, raw0, zs0, mus, ystart, 0, x0, q0, kA, nk, RW);
    __syncthreads();
    int g = 0;
    while (true) {
#pragma unroll
        for (int u = 0; u < NSTEP; u++) {
            if (g + 2 < nsteps) issue(raw0 + (g & 1) * raw_len, g + 2);
            if (g + 1 < nsteps) {
                if (fast)
                    vfir_stage_a_fast<J, NPL, (RHO > 0 ? RHO : 1), (FAST ? NPC : 1), NT>(
                        P, raw0 + ((g + 1) & 1) * raw_len, zs0 + ((g + 1) & 1) * zs_len, mus, ystart, g + 1, x0, nk);
                else
                    vfir_stage_a<J, NPL, RHO, NPC, NT>(P, raw0 + ((g + 1) & 1) * raw_len, zs0 + ((g + 1) & 1) * zs_len,
                                                       mus, ystart, g + 1, x0, q0, kA, nk, RW);
            }
            const float* st = zs0 + (g & 1) * zs_len + pq * kVTX + CPW * cw;
#pragma unroll
            for (int i = 0; i < J; i++) wload(win[u * J + i], st + i * NPL * kVTX);
            if (g >= NSTEP - 1 && active) {
                const int yb = y0 + (g - NSTEP + 1) * J;
                float* orow = outp + (size_t)yb * P.Wp;
                const int oldest = ((u + 1) % NSTEP) * J;   // window position of logical row 0
                if (BOX) {
                    WT acc = win[oldest % S];
#pragma unroll
                    for (int s = 1; s <= 2 * R; s++) acc = wadd(acc, win[(oldest + s) % S]);
#pragma unroll
                    for (int j = 0; j < J; j++) {
                        if (j > 0) acc = wsub(wadd(acc, win[(oldest + j + 2 * R) % S]), win[(oldest + j - 1) % S]);
                        if (yb + j < y1) wstore(orow + (size_t)j * P.Wp, acc);
                    }
                } else {
                    const bool full = yb + J <= y1;
                    // Every output accumulates its taps in four independent partial sums (taps t mod 4),
                    // added at the end: the scheduler tends to run one output's taps back to back (to
                    // save registers), so the ILP has to be inside one output's chain (measured: with a
                    // single chain per output the FP32 pipe waited on the FMA latency, ~55% busy).
                    WT acc[J];
#pragma unroll
                    for (int j = 0; j < J; j++) {
                        const int c = oldest + j + R;
                        constexpr int NC = 4;   // partial sums per output (8 measured slower at R = 24: 11.7 vs 10.1 ms)
                        WT a4[NC];
                        if constexpr (PACK) a4[0] = wmul0((WT)P.tw[0], win[c % S]);
                        else a4[0] = wmul0((WT)P.tws[R], win[c % S]);
#pragma unroll
                        for (int u = 1; u < NC; u++) a4[u] = WT(0);
#pragma unroll
                        for (int t = 1; t <= R; t++) {
                            if constexpr (PACK) {
                                a4[t % NC] = wfma((WT)P.tw[t], wadd(win[(c - t) % S], win[(c + t) % S]), a4[t % NC]);
                            } else {
                                a4[t % NC] = wfma((WT)P.tws[R - t], win[(c + t) % S], a4[t % NC]);
                                a4[t % NC] = wfma((WT)P.tws[R + t], win[(c - t) % S], a4[t % NC]);
                            }
                        }
#pragma unroll
                        for (int h = NC / 2; h >= 1; h /= 2)
#pragma unroll
                            for (int u = 0; u < h; u++) a4[u] = wadd(a4[u], a4[u + h]);
                        acc[j] = a4[0];
                    }
#pragma unroll
                    for (int j = 0; j < J; j++) {
                        if (full || yb + j < y1) wstore(orow, acc[j]);
                        orow += P.Wp;
                    }
                }
            }
            cp_async_wait_all();
            __syncthreads();
            g++;
            if (g >= nsteps) return;
        }
    }
}

// Persistent schedule: the (strip, plane group) columns x H rows are linearised column by column and
// CTA b takes the contiguous share [T b / G, T (b + 1) / G) (T = columns * H): every CTA gets the same
// number of output rows (no wave quantisation) and a window is primed at most once per column
// touched.
template <int R, int J, bool BOX, bool PACK, int RHO, int NPC, int NT>
__global__ void __launch_bounds__(NT, 1) k_range_vpass(const __grid_constant__ VParams P) {
    extern __shared__ __align__(16) float sm_v[];
    const long long T = (long long)P.ncol * P.H;
    const long long u0 = T * blockIdx.x / gridDim.x, u1 = T * (blockIdx.x + 1) / gridDim.x;
    long long u = u0;
    while (u < u1) {
        const int col = (int)(u / P.H);
        const int ya = (int)(u - (long long)col * P.H);
        const int yb = (int)((u1 - u < (long long)(P.H - ya)) ? ya + (u1 - u) : P.H);
        vfir_segment<R, J, BOX, PACK, RHO, NPC, NT>(P, sm_v, col % P.nstrip, col / P.nstrip, ya, yb);
        u += yb - ya;
    }
}

}  // namespace hdf
