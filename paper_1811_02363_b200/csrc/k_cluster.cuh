// k_cluster.cuh -- step 1: bisecting K-means of Theta = {p(i)}.
//
// One cooperative persistent kernel runs the whole procedure (no host round trips):
//   * Theta is copied once into leaf-contiguous storage (pts, idx); every leaf is a segment whose
//     members stay in ascending pixel order ("member order", R3) because splits are stable
//     partitions.
//   * The leaf of largest SSE (R2; ties -> lowest id) is split by 2-means seeded with the farthest
//     pair of the stride sample members[0::ceil(m/1024)] (R3), Lloyd iterations until no
//     assignment changes or 50 iterations (R4, ties -> first centre, empty side reseeded at the
//     farthest member).  The parent id keeps child 0, child 1 takes id = #leaves.
//   * Concurrency without changing the result: the set of current leaves that the sequential
//     procedure will split in its remaining K - L steps is a prefix of the leaves ordered by
//     (SSE desc, id asc).  Each round therefore computes the splits of all not-yet-split leaves in
//     the top (K - L) concurrently (lock-step Lloyd, one grid barrier per iteration), then commits
//     splits in the sequential order for as long as the current maximum leaf has a computed split.
//   * Distances are fp64 with explicit round-to-nearest operations in dimension order (the exact
//     operation sequence of a plain loop), so assignment and farthest-pair decisions are
//     reproducible; sums are fp64 with a fixed reduction tree (deterministic run to run).
#pragma once
#include <cooperative_groups.h>

#include "hdf_common.cuh"

namespace hdf {
namespace cg = cooperative_groups;

constexpr int kClThreads = 512;
constexpr int kClWarps = kClThreads / 32;
constexpr int kFpCap = 1024;      // farthest-pair stride-sample cap (R3)
constexpr int kMaxIter = 50;      // Lloyd cap (R4)

struct CLeaf {
    int start, m, state, m0;     // state 1 = split computed (children ready, segment partitioned)
    double sse, csse0, csse1;
};
struct CSlot {
    int leaf, conv, reseed, stride, s, fa, fb, fbuf, cbeg, cend;   // chunk range [cbeg, cend)
};
struct CChunk {
    int slot, begin, end;
};

// control words
enum { C_NLEAVES = 0, C_NSLOTS, C_NCHUNKS, C_STATUS, C_ROUNDS, C_ITERS, C_DONE, C_NUM };

struct ClusterArgs {
    const float* p;
    int N, rho, K, CH, maxch, slotmax;
    float* pts[2];
    int* idx[2];
    unsigned char* side[2];
    CLeaf* leaves;
    double* lmean;     // [K][rho]
    double* cmean0;    // [K][rho]  child means of a computed split (by leaf id)
    double* cmean1;
    CSlot* slots;      // [slotmax]
    double* c0g;       // [slotmax][rho] centres (written by the finalising block)
    double* c1g;
    CChunk* chunks;    // [maxch]
    double* part;      // [maxch][pstride]
    int pstride;
    double* fpd;       // [slotmax * kFpCap] farthest-pair row maxima
    int* fpi;          // [slotmax * kFpCap]
    int* ctrl;         // [C_NUM]
    float* centres;    // [K][rho] out
    int* labels;       // [N] out (may be null)
    double* ek;        // out
};

// ---------------------------------------------------------------------------- small helpers ---
HDF_DEV double ldd(const double* p) { return __ldcg(p); }
HDF_DEV int ldi(const int* p) { return __ldcg(p); }

HDF_DEV CChunk ld_chunk(const CChunk* c) {
    CChunk r;
    r.slot = __ldcg(&c->slot);
    r.begin = __ldcg(&c->begin);
    r.end = __ldcg(&c->end);
    return r;
}
HDF_DEV CLeaf ld_leaf(const CLeaf* l) {
    CLeaf r;
    r.start = __ldcg(&l->start);
    r.m = __ldcg(&l->m);
    r.state = __ldcg(&l->state);
    r.m0 = __ldcg(&l->m0);
    r.sse = __ldcg(&l->sse);
    r.csse0 = __ldcg(&l->csse0);
    r.csse1 = __ldcg(&l->csse1);
    return r;
}

HDF_DEV double dist_pt(const float* x, const double* c, int rho) {
    double s = 0.0;
    for (int d = 0; d < rho; d++) s = d2_rn(s, (double)__ldcg(x + d), c[d]);
    return s;
}

// Block-wide deterministic reduction of `nv` doubles laid out as red[warp * ld + v] -> out[nv].
HDF_DEV void block_reduce_rows(const double* red, int nv, int ld, double* out) {
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < kClWarps; w++) s += red[w * ld + v];
        out[v] = s;
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------ plan (serial) --
// Commit computed splits in sequential order; select the next batch; build the chunk table.
HDF_DEV void cl_plan(const ClusterArgs& A) {
    int L = ldi(&A.ctrl[C_NLEAVES]);
    const int K = A.K, rho = A.rho;
    int status = ldi(&A.ctrl[C_STATUS]);
    while (L < K) {
        int s = 0;
        double best = ldd(&A.leaves[0].sse);
        for (int l = 1; l < L; l++) {
            double v = ldd(&A.leaves[l].sse);
            if (v > best) { best = v; s = l; }
        }
        if (!(best > 0.0)) { status = HDF_ERR_K; break; }
        if (ldi(&A.leaves[s].state) != 1) break;
        // commit: parent keeps child 0, child 1 gets id L
        const CLeaf P = ld_leaf(&A.leaves[s]);
        CLeaf c0, c1;
        c0.start = P.start; c0.m = P.m0; c0.state = 0; c0.m0 = 0; c0.sse = P.csse0; c0.csse0 = c0.csse1 = 0.0;
        c1.start = P.start + P.m0; c1.m = P.m - P.m0; c1.state = 0; c1.m0 = 0; c1.sse = P.csse1; c1.csse0 = c1.csse1 = 0.0;
        for (int d = 0; d < rho; d++) {
            A.lmean[s * rho + d] = ldd(&A.cmean0[s * rho + d]);
            A.lmean[L * rho + d] = ldd(&A.cmean1[s * rho + d]);
        }
        A.leaves[s] = c0;
        A.leaves[L] = c1;
        L++;
    }
    A.ctrl[C_NLEAVES] = L;
    A.ctrl[C_STATUS] = status;
    if (L >= K || status != HDF_OK) {
        A.ctrl[C_DONE] = 1;
        A.ctrl[C_NSLOTS] = 0;
        return;
    }
    // batch: leaves among the top (K - L) by (sse desc, id asc) without a computed split
    const int need = K - L;
    int nslots = 0, nch = 0;
    unsigned char taken[HDF_MAX_K];
    for (int l = 0; l < L; l++) taken[l] = 0;
    for (int r = 0; r < need && r < L; r++) {
        int s = -1;
        double best = -1.0;
        for (int l = 0; l < L; l++) {
            if (taken[l]) continue;
            double v = ldd(&A.leaves[l].sse);
            if (s < 0 || v > best) { best = v; s = l; }
        }
        taken[s] = 1;
        if (!(best > 0.0)) break;
        if (ldi(&A.leaves[s].state) == 1) continue;
        const int start = ldi(&A.leaves[s].start), m = ldi(&A.leaves[s].m);
        CSlot sl;
        sl.leaf = s;
        sl.conv = 0;
        sl.reseed = 0;
        sl.stride = (m + kFpCap - 1) / kFpCap;
        sl.s = (m + sl.stride - 1) / sl.stride;
        sl.fa = 0;
        sl.fb = 0;
        sl.fbuf = 0;
        sl.cbeg = nch;
        for (int b = start; b < start + m; b += A.CH) {
            CChunk c;
            c.slot = nslots;
            c.begin = b;
            c.end = min(start + m, b + A.CH);
            A.chunks[nch++] = c;
        }
        sl.cend = nch;
        A.slots[nslots++] = sl;
    }
    A.ctrl[C_NSLOTS] = nslots;
    A.ctrl[C_NCHUNKS] = nch;
    A.ctrl[C_ROUNDS] = ldi(&A.ctrl[C_ROUNDS]) + 1;
}


// One lock-step Lloyd pass: for every chunk of an active slot, assign each member to the nearer
// centre (ties -> first), count changes against the previous assignment, and write per-chunk
// partial sums (sum0[rho], sum1[rho], n1, changed).  `only` (optional) restricts to slots with
// only[sl] != 0 (the reseed redo pass).
HDF_DEV void cl_pass(const ClusterArgs& A, const float* P, int nch, const double* cen0, const double* cen1,
                     const int* s_conv, const int* only, int it, int wb, double* red, double* tmpv) {
    const int rho = A.rho, nvL = 2 * rho + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned char* sw = A.side[wb];
    const unsigned char* sp = A.side[wb ^ 1];
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
        const CChunk ch = ld_chunk(&A.chunks[c]);
        if (s_conv[ch.slot]) continue;
        if (only && !only[ch.slot]) continue;
        const double* c0 = cen0 + ch.slot * rho;
        const double* c1 = cen1 + ch.slot * rho;
        double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0};
        int cnt1 = 0, changed = 0;
        for (int t0 = ch.begin; t0 < ch.end; t0 += blockDim.x) {
            const int t = t0 + tid;
            const bool ok = t < ch.end;
            int sd = 0;
            if (ok) {
                const float* x = P + (size_t)t * rho;
                const double d0 = dist_pt(x, c0, rho), d1 = dist_pt(x, c1, rho);
                sd = (d0 <= d1) ? 0 : 1;
                if (it > 0 && sd != (int)__ldcg(sp + t)) changed++;
                sw[t] = (unsigned char)sd;
                cnt1 += sd;
            }
            // lane-distributed per-dimension sums (lane d % 32 owns dimension d)
            for (int d = 0; d < rho; d++) {
                const double v = ok ? (double)__ldcg(P + (size_t)t * rho + d) : 0.0;
                const double s0 = warp_sum(sd == 0 ? v : 0.0);
                const double s1 = warp_sum(sd == 1 ? v : 0.0);
                if (lane == (d & 31)) { a0[d >> 5] += s0; a1[d >> 5] += s1; }
            }
        }
        for (int d = lane; d < rho; d += 32) {
            red[warp * nvL + d] = a0[d >> 5];
            red[warp * nvL + rho + d] = a1[d >> 5];
        }
        const double cn = warp_sum((double)cnt1), chg = warp_sum((double)changed);
        if (lane == 0) { red[warp * nvL + 2 * rho] = cn; red[warp * nvL + 2 * rho + 1] = chg; }
        block_reduce_rows(red, 2 * rho + 2, nvL, tmpv);
        for (int v = tid; v < 2 * rho + 2; v += blockDim.x) A.part[(size_t)c * A.pstride + v] = tmpv[v];
        __syncthreads();
    }
}

// Finalise one iteration for every active slot, redundantly in every block (identical inputs,
// identical fixed-order arithmetic -> identical results everywhere).  Returns 1 if some slot came
// out with an empty side (s_rs[sl] = 1: side 1 empty, 2: side 0 empty).
HDF_DEV int cl_finalize(const ClusterArgs& A, int nslots, int it, int wb, double* cen0, double* cen1, int* s_conv,
                        int* s_rs, int* s_fbuf, bool redo, double* tmpv) {
    const int rho = A.rho;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int any = 0;
    for (int sl = 0; sl < nslots; sl++) {
        if (s_conv[sl]) continue;
        if (redo && !s_rs[sl]) continue;
        const int cb = ldi(&A.slots[sl].cbeg), ce = ldi(&A.slots[sl].cend);
        const int leaf = ldi(&A.slots[sl].leaf);
        const long long m = ldi(&A.leaves[leaf].m);
        __syncthreads();
        for (int v = warp; v < 2 * rho + 2; v += kClWarps) {
            double s = 0.0;
            for (int c = cb + lane; c < ce; c += 32) s += ldd(&A.part[(size_t)c * A.pstride + v]);
            s = warp_sum(s);
            if (lane == 0) tmpv[v] = s;
        }
        __syncthreads();
        const long long n1 = (long long)tmpv[2 * rho];
        const long long chg = (long long)tmpv[2 * rho + 1];
        if (!redo && (n1 == 0 || n1 == m)) {
            any = 1;
            if (tid == 0) s_rs[sl] = (n1 == 0) ? 1 : 2;
        } else if (it > 0 && chg == 0) {
            if (tid == 0) { s_conv[sl] = 1; s_fbuf[sl] = wb; }
        } else {
            for (int d = tid; d < rho; d += blockDim.x) {
                cen0[sl * rho + d] = tmpv[d] / (double)(m - n1);
                cen1[sl * rho + d] = tmpv[rho + d] / (double)n1;
            }
            if (tid == 0) s_fbuf[sl] = wb;
        }
        __syncthreads();
    }
    if (redo) {
        __syncthreads();
        for (int sl = tid; sl < nslots; sl += blockDim.x) s_rs[sl] = 0;
        __syncthreads();
    }
    return any;
}

// Farthest member of a reseed slot's leaf from the non-empty side's centre (ties -> first in
// member order); the block owning the slot writes the new centre to c0g / c1g.
HDF_DEV void cl_reseed(const ClusterArgs& A, const float* P, int nslots, const double* cen0, const double* cen1,
                       const int* s_rs, double* red) {
    const int rho = A.rho;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int sl = blockIdx.x; sl < nslots; sl += gridDim.x) {
        const int rs = s_rs[sl];
        if (!rs) continue;
        const int leaf = ldi(&A.slots[sl].leaf);
        const int start = ldi(&A.leaves[leaf].start), m = ldi(&A.leaves[leaf].m);
        const double* cref = (rs == 1) ? cen0 + sl * rho : cen1 + sl * rho;
        double best = -1.0;
        int arg = -1;
        for (int t = start + tid; t < start + m; t += blockDim.x) {
            const double d = dist_pt(P + (size_t)t * rho, cref, rho);
            if (d > best) { best = d; arg = t; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (oa >= 0 && (arg < 0 || ob > best || (ob == best && oa < arg))) { best = ob; arg = oa; }
        }
        __syncthreads();
        if (lane == 0) { red[warp * 2] = best; red[warp * 2 + 1] = (double)arg; }
        __syncthreads();
        if (tid == 0) {
            double bb = -1.0;
            int aa = -1;
            for (int w = 0; w < kClWarps; w++) {
                const int oa = (int)red[w * 2 + 1];
                const double ob = red[w * 2];
                if (oa >= 0 && (aa < 0 || ob > bb || (ob == bb && oa < aa))) { bb = ob; aa = oa; }
            }
            double* dst = (rs == 1) ? A.c1g + sl * rho : A.c0g + sl * rho;
            for (int d = 0; d < rho; d++) dst[d] = (double)__ldcg(P + (size_t)aa * rho + d);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------- the kernel ---
__global__ void __launch_bounds__(kClThreads) k_bisect_kmeans(const ClusterArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm_cl[];
    const int rho = A.rho, K = A.K;
    const int nvL = 2 * rho + 4;                    // per-chunk partial: sum0[rho], sum1[rho], cnt1, changed, sse0, sse1
    double* red = sm_cl;                            // [kClWarps][nvL]
    double* cen0 = red + kClWarps * nvL;            // [slotmax][rho] block-local centres
    double* cen1 = cen0 + A.slotmax * rho;
    double* tmpv = cen1 + A.slotmax * rho;          // [nvL]
    __shared__ int s_conv[HDF_MAX_K];
    __shared__ int s_rs[HDF_MAX_K];
    __shared__ int s_fbuf[HDF_MAX_K];
    __shared__ int s_scan[kClWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const long long gtid = (long long)blockIdx.x * blockDim.x + tid;
    const long long gthreads = (long long)G * blockDim.x;

    // ---- init: copy Theta into leaf storage, root leaf = all pixels in pixel order -----------
    for (long long e = gtid; e < (long long)A.N * rho; e += gthreads) A.pts[0][e] = A.p[e];
    for (long long e = gtid; e < A.N; e += gthreads) A.idx[0][e] = (int)e;
    if (gtid == 0) {
        for (int c = 0; c < C_NUM; c++) A.ctrl[c] = 0;
        A.ctrl[C_NLEAVES] = 1;
    }
    // root mean: per-block partial sums over a fixed contiguous range, then block 0 totals them
    {
        const long long per = ((long long)A.N + G - 1) / G;
        const long long b = (long long)blockIdx.x * per, e = min((long long)A.N, b + per);
        for (int d = 0; d < rho; d++) {
            double s = 0.0;
            for (long long t = b + tid; t < e; t += blockDim.x) s += (double)A.p[t * rho + d];
            s = warp_sum(s);
            if (lane == 0) red[warp * nvL + d] = s;
        }
        block_reduce_rows(red, rho, nvL, tmpv);
        if (tid < rho) A.part[(size_t)blockIdx.x * A.pstride + tid] = tmpv[tid];
    }
    grid.sync();
    if (tid < rho) {
        double s = 0.0;
        for (int bI = 0; bI < G; bI++) s += ldd(&A.part[(size_t)bI * A.pstride + tid]);
        tmpv[tid] = s / (double)A.N;
    }
    __syncthreads();
    {
        const long long per = ((long long)A.N + G - 1) / G;
        const long long b = (long long)blockIdx.x * per, e = min((long long)A.N, b + per);
        double s = 0.0;
        for (long long t = b + tid; t < e; t += blockDim.x) {
            double dd = 0.0;
            for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)A.p[t * rho + d], tmpv[d]);
            s += dd;
        }
        s = warp_sum(s);
        if (lane == 0) red[warp * nvL] = s;
        block_reduce_rows(red, 1, nvL, tmpv + rho);
        if (tid == 0) A.part[(size_t)blockIdx.x * A.pstride + rho] = tmpv[rho];
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {
        double s = 0.0;
        for (int bI = 0; bI < G; bI++) s += ldd(&A.part[(size_t)bI * A.pstride + rho]);
        CLeaf r;
        r.start = 0; r.m = A.N; r.state = 0; r.m0 = 0; r.sse = s; r.csse0 = r.csse1 = 0.0;
        A.leaves[0] = r;
        for (int d = 0; d < rho; d++) A.lmean[d] = tmpv[d];
    }
    grid.sync();

    int cur = 0;   // which pts/idx buffer holds the leaf storage
    while (true) {
        // ---------------- plan ----------------
        if (blockIdx.x == 0 && tid == 0) cl_plan(A);
        grid.sync();
        if (ldi(&A.ctrl[C_DONE])) break;
        const int nslots = ldi(&A.ctrl[C_NSLOTS]);
        const int nch = ldi(&A.ctrl[C_NCHUNKS]);
        const float* P = A.pts[cur];

        // ---------------- farthest pair rows: warp per (slot, row a) ----------------
        {
            int rows_total = 0;
            for (int sl = 0; sl < nslots; sl++) rows_total += ldi(&A.slots[sl].s);
            const int gw = (int)(gtid >> 5), nw = (int)(gthreads >> 5);
            for (int r = gw; r < rows_total; r += nw) {
                int sl = 0, base = 0;
                while (r >= base + ldi(&A.slots[sl].s)) { base += ldi(&A.slots[sl].s); sl++; }
                const int a = r - base;
                const int leaf = ldi(&A.slots[sl].leaf);
                const int start = ldi(&A.leaves[leaf].start);
                const int stride = ldi(&A.slots[sl].stride), s = ldi(&A.slots[sl].s);
                const float* xa = P + (size_t)(start + (long long)a * stride) * rho;
                double best = -1.0;
                int arg = -1;
                for (int b = a + 1 + lane; b < s; b += 32) {
                    const float* xb = P + (size_t)(start + (long long)b * stride) * rho;
                    double dd = 0.0;
                    for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)__ldcg(xa + d), (double)__ldcg(xb + d));
                    if (dd > best) { best = dd; arg = b; }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    int oa = __shfl_xor_sync(0xffffffffu, arg, o);
                    if (oa >= 0 && (arg < 0 || ob > best || (ob == best && oa < arg))) { best = ob; arg = oa; }
                }
                if (lane == 0) {
                    A.fpd[(size_t)sl * kFpCap + a] = best;
                    A.fpi[(size_t)sl * kFpCap + a] = arg;
                }
            }
        }
        grid.sync();
        // argmax over rows (ties -> first row), one block per slot; centres from the pair
        for (int sl = blockIdx.x; sl < nslots; sl += G) {
            const int s = ldi(&A.slots[sl].s);
            double best = -1.0;
            int ra = -1;
            for (int a = tid; a < s; a += blockDim.x) {
                const int arg = ldi(&A.fpi[(size_t)sl * kFpCap + a]);
                const double v = ldd(&A.fpd[(size_t)sl * kFpCap + a]);
                if (arg >= 0 && (ra < 0 || v > best)) { best = v; ra = a; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(0xffffffffu, best, o);
                int oa = __shfl_xor_sync(0xffffffffu, ra, o);
                if (oa >= 0 && (ra < 0 || ob > best || (ob == best && oa < ra))) { best = ob; ra = oa; }
            }
            if (lane == 0) { red[warp * 2] = best; red[warp * 2 + 1] = (double)ra; }
            __syncthreads();
            if (tid == 0) {
                double bb = -1.0;
                int rr = -1;
                for (int w = 0; w < kClWarps; w++) {
                    const int oa = (int)red[w * 2 + 1];
                    const double ob = red[w * 2];
                    if (oa >= 0 && (rr < 0 || ob > bb || (ob == bb && oa < rr))) { bb = ob; rr = oa; }
                }
                int fa = 0, fb = 0;
                if (rr >= 0) { fa = rr; fb = ldi(&A.fpi[(size_t)sl * kFpCap + rr]); }
                A.slots[sl].fa = fa;
                A.slots[sl].fb = fb;
                const int leaf = ldi(&A.slots[sl].leaf);
                const int start = ldi(&A.leaves[leaf].start), stride = ldi(&A.slots[sl].stride);
                for (int d = 0; d < rho; d++) {
                    A.c0g[sl * rho + d] = (double)__ldcg(P + (size_t)(start + (long long)fa * stride) * rho + d);
                    A.c1g[sl * rho + d] = (double)__ldcg(P + (size_t)(start + (long long)fb * stride) * rho + d);
                }
            }
            __syncthreads();
        }
        grid.sync();
        for (int e = tid; e < nslots * rho; e += blockDim.x) {
            cen0[e] = ldd(&A.c0g[e]);
            cen1[e] = ldd(&A.c1g[e]);
        }
        for (int sl = tid; sl < nslots; sl += blockDim.x) { s_conv[sl] = 0; s_rs[sl] = 0; s_fbuf[sl] = (kMaxIter - 1) & 1; }
        __syncthreads();

        // ---------------- lock-step Lloyd iterations ----------------
        int it = 0;
        for (; it < kMaxIter; it++) {
            const int wb = it & 1;
            cl_pass(A, P, nch, cen0, cen1, s_conv, nullptr, it, wb, red, tmpv);
            grid.sync();
            const int any = cl_finalize(A, nslots, it, wb, cen0, cen1, s_conv, s_rs, s_fbuf, false, tmpv);
            if (any) {
                // Rare path (R4): a side came out empty.  Move that side's centre to the member
                // farthest from the other centre (ties -> first), redo this iteration's assignment.
                cl_reseed(A, P, nslots, cen0, cen1, s_rs, red);
                grid.sync();
                for (int sl = 0; sl < nslots; sl++) {
                    if (!s_rs[sl]) continue;
                    for (int d = tid; d < rho; d += blockDim.x) {
                        if (s_rs[sl] == 1) cen1[sl * rho + d] = ldd(&A.c1g[sl * rho + d]);
                        else cen0[sl * rho + d] = ldd(&A.c0g[sl * rho + d]);
                    }
                }
                __syncthreads();
                cl_pass(A, P, nch, cen0, cen1, s_conv, s_rs, it, wb, red, tmpv);
                grid.sync();
                cl_finalize(A, nslots, it, wb, cen0, cen1, s_conv, s_rs, s_fbuf, true, tmpv);
            }
            bool all = true;
            for (int sl = 0; sl < nslots; sl++) all = all && s_conv[sl];
            if (all) break;
        }
        if (it == kMaxIter) it = kMaxIter - 1;

        // ---------------- stable partition + child SSE ----------------
        const int nxt = cur ^ 1;
        for (int c = blockIdx.x; c < nch; c += G) {
            const CChunk ch = ld_chunk(&A.chunks[c]);
            const int sl = ch.slot;
            const int leaf = ldi(&A.slots[sl].leaf);
            const int start = ldi(&A.leaves[leaf].start), m = ldi(&A.leaves[leaf].m);
            const unsigned char* sd = A.side[s_fbuf[sl]];
            const int cb = ldi(&A.slots[sl].cbeg);
            // n1 of this slot and of earlier chunks (from the final pass partials)
            long long pre1 = 0, tot1 = 0;
            for (int c2 = cb; c2 < ldi(&A.slots[sl].cend); c2++) {
                const long long v = (long long)ldd(&A.part[(size_t)c2 * A.pstride + 2 * rho]);
                if (c2 < c) pre1 += v;
                tot1 += v;
            }
            const long long m0 = m - tot1;
            const long long pre0 = (ch.begin - start) - pre1;
            const double* c0 = cen0 + sl * rho;
            const double* c1 = cen1 + sl * rho;
            double se0 = 0.0, se1 = 0.0;
            long long run0 = 0, run1 = 0;
            for (int t0 = ch.begin; t0 < ch.end; t0 += blockDim.x) {
                const int t = t0 + tid;
                const bool ok = t < ch.end;
                const int s = ok ? (int)__ldcg(sd + t) : 0;
                const int f0 = (ok && s == 0) ? 1 : 0;
                // block exclusive scan of f0 (ballot per warp, warp totals scanned in shared memory)
                const unsigned bal = __ballot_sync(0xffffffffu, f0);
                if (lane == 0) s_scan[warp] = __popc(bal);
                __syncthreads();
                int wpre = 0, total0 = 0;
                for (int w = 0; w < kClWarps; w++) {
                    const int v = s_scan[w];
                    if (w < warp) wpre += v;
                    total0 += v;
                }
                const int incl = wpre + __popc(bal & ((lane == 31) ? 0xffffffffu : ((1u << (lane + 1)) - 1u)));
                __syncthreads();
                if (ok) {
                    const int rank0 = incl - f0;
                    const int rank1 = (t - t0) - rank0;
                    long long dst;
                    if (s == 0) dst = start + pre0 + run0 + rank0;
                    else dst = start + m0 + pre1 + run1 + rank1;
                    const float* x = P + (size_t)t * rho;
                    double dd = 0.0;
                    const double* cc = s ? c1 : c0;
                    for (int d = 0; d < rho; d++) {
                        const float v = __ldcg(x + d);
                        A.pts[nxt][(size_t)dst * rho + d] = v;
                        dd = d2_rn(dd, (double)v, cc[d]);
                    }
                    A.idx[nxt][dst] = __ldcg(A.idx[cur] + t);
                    if (s) se1 += dd; else se0 += dd;
                }
                const int nvalid = min((int)blockDim.x, ch.end - t0);
                run0 += total0;
                run1 += nvalid - total0;
            }
            se0 = warp_sum(se0);
            se1 = warp_sum(se1);
            if (lane == 0) { red[warp * nvL] = se0; red[warp * nvL + 1] = se1; }
            block_reduce_rows(red, 2, nvL, tmpv);
            if (tid == 0) {
                A.part[(size_t)c * A.pstride + 2 * rho + 2] = tmpv[0];
                A.part[(size_t)c * A.pstride + 2 * rho + 3] = tmpv[1];
            }
            __syncthreads();
        }
        grid.sync();
        // copy the partitioned segments back, record the computed splits
        for (int c = blockIdx.x; c < nch; c += G) {
            const CChunk ch = ld_chunk(&A.chunks[c]);
            for (long long e = (long long)ch.begin * rho + tid; e < (long long)ch.end * rho; e += blockDim.x)
                A.pts[cur][e] = __ldcg(A.pts[nxt] + e);
            for (int t = ch.begin + tid; t < ch.end; t += blockDim.x) A.idx[cur][t] = __ldcg(A.idx[nxt] + t);
        }
        for (int sl = blockIdx.x; sl < nslots; sl += G) {
            if (tid == 0) {
                const int leaf = ldi(&A.slots[sl].leaf);
                const int cb = ldi(&A.slots[sl].cbeg), ce = ldi(&A.slots[sl].cend);
                double s0 = 0.0, s1 = 0.0, n1 = 0.0;
                for (int c = cb; c < ce; c++) {
                    n1 += ldd(&A.part[(size_t)c * A.pstride + 2 * rho]);
                    s0 += ldd(&A.part[(size_t)c * A.pstride + 2 * rho + 2]);
                    s1 += ldd(&A.part[(size_t)c * A.pstride + 2 * rho + 3]);
                }
                const int m = ldi(&A.leaves[leaf].m);
                A.leaves[leaf].m0 = m - (int)n1;
                A.leaves[leaf].csse0 = s0;
                A.leaves[leaf].csse1 = s1;
                for (int d = 0; d < rho; d++) {
                    A.cmean0[leaf * rho + d] = cen0[sl * rho + d];
                    A.cmean1[leaf * rho + d] = cen1[sl * rho + d];
                }
                __threadfence();
                A.leaves[leaf].state = 1;
            }
        }
        if (blockIdx.x == 0 && tid == 0) A.ctrl[C_ITERS] = ldi(&A.ctrl[C_ITERS]) + it + 1;
        grid.sync();
    }

    // ---------------- outputs ----------------
    const int L = ldi(&A.ctrl[C_NLEAVES]);
    for (int e = gtid; e < K * rho; e += gthreads) {
        const int k = e / rho, d = e % rho;
        const int src = (k < L) ? k : 0;
        A.centres[e] = (float)ldd(&A.lmean[src * rho + d]);
    }
    if (A.labels) {
        for (int l = 0; l < L; l++) {
            const int start = ldi(&A.leaves[l].start), m = ldi(&A.leaves[l].m);
            for (long long t = gtid; t < m; t += gthreads) A.labels[__ldcg(A.idx[cur] + start + t)] = l;
        }
    }
    if (gtid == 0) {
        double e = 0.0;
        for (int l = 0; l < L; l++) e += ldd(&A.leaves[l].sse);
        *A.ek = e;
    }
}

}  // namespace hdf
