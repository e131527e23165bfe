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
//   * Concurrency without changing the result: SSE never increases from a leaf to its children,
//     so the leaves the sequential procedure will split in its remaining K - L steps are a prefix
//     of the current leaves ordered by (SSE desc, id asc).  Each round computes the splits of the
//     not-yet-split leaves among that prefix concurrently (lock-step Lloyd iterations, one grid
//     barrier per iteration), then commits splits in the sequential order for as long as the
//     current maximum leaf has a computed split.
//   * Work layout of a round: the active slots' segments are concatenated (T points) and block b
//     owns the range [T b / G, T (b+1) / G); it writes one partial record per slot it touches.
//     Records are double-buffered by iteration parity, so the next pass never overwrites records
//     another block is still reducing.  Every block reduces the records of every slot itself, in a
//     fixed order, so all blocks hold identical centres without a second barrier.
//   * Distances are fp64 with explicit round-to-nearest operations in dimension order (the exact
//     operation sequence of a plain loop); sums are fp64 with a fixed reduction tree, so the run
//     is deterministic and decisions match the fp64 oracle up to summation order.
#pragma once
#include <cooperative_groups.h>

#include "hdf_common.cuh"

namespace hdf {
namespace cg = cooperative_groups;

constexpr int kClThreads = 512;
constexpr int kClWarps = kClThreads / 32;
constexpr int kFpCap = 1024;      // farthest-pair stride-sample cap (R3)
constexpr int kMaxIter = 50;      // Lloyd cap (R4)
constexpr int kSlotCap = 32;      // concurrent splits per round (more rounds, same result)
constexpr int kMaxGrid = 1024;    // records bound: kMaxGrid + kSlotCap per buffer
constexpr int kDC = 8;            // dimensions accumulated per sweep
constexpr int kTraceCap = 4096;

struct CLeaf {
    int start, m, state, m0;      // state 1 = split computed (segment partitioned, children ready)
    double sse, csse0, csse1;
};
struct CSlot {
    int leaf, start, m;           // leaf segment [start, start + m) of the leaf storage
    int blo, bhi, rbase;          // blocks touching the slot; first record index
    long long pbeg;               // offset of the segment in the round's concatenated range
    int stride, s;                // farthest-pair stride sample: members[0::stride], s of them
};

// control words
enum { C_NLEAVES = 0, C_NSLOTS, C_STATUS, C_ROUNDS, C_ITERS, C_DONE, C_NUM };
// phase timers (ns, diagnostics)
enum { T_PLAN = 0, T_SEED, T_LLOYD, T_PART, T_SYNC, T_PASS, T_P_SIDE, T_P_SUM, T_P_RED, T_NUM };

struct ClusterArgs {
    const float* p;
    int N, rho, K, slotmax, maxrec, pstride;
    int tileF;         // floats of the shared point tile (multiple of 4)
    long long big;     // a round whose largest slot exceeds this many points runs grid-wide
    float* pts[2];
    int* idx[2];
    unsigned char* side[2];
    CLeaf* leaves;
    double* lmean;     // [K][rho]
    double* cmean0;    // [K][rho]  child means of a computed split (by leaf id)
    double* cmean1;
    CSlot* slots;      // [slotmax]
    double* c0g;       // [slotmax][rho] seed / reseed centres
    double* c1g;
    double* rec[2];    // [maxrec][pstride]: sum0[rho], sum1[rho], n1, changed, sse0, sse1
    double* fpd;       // [slotmax * kFpCap] farthest-pair row maxima
    int* fpi;          // [slotmax * kFpCap]
    int* ctrl;         // [C_NUM]
    long long* timers; // [T_NUM]
    long long* trace;  // [1 + 2 * kTraceCap] (tag, globaltimer) events of block 0, diagnostics
    float* centres;    // [K][rho] out
    int* labels;       // [N] out (may be null)
    double* ek;        // out
};

// ---------------------------------------------------------------------------- small helpers ---
HDF_DEV double ldd(const double* p) { return __ldcg(p); }
HDF_DEV int ldi(const int* p) { return __ldcg(p); }
HDF_DEV long long ldll(const long long* p) { return __ldcg(p); }
HDF_DEV long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Diagnostics state of block 0 (shared memory, so recording costs no global round trip).
struct DiagSm {
    long long timers[16];
    int ntrace;
};
HDF_DEV DiagSm& diag() {
    __shared__ DiagSm d;
    return d;
}
// Append (tag | clock64 << 16, globaltimer) to the trace (block 0, thread 0 only; stores only).
HDF_DEV void trace_ev(long long* tr, int tag) {
    if (tr == nullptr || blockIdx.x != 0 || threadIdx.x != 0) return;
    DiagSm& d = diag();
    const int n = d.ntrace;
    if (n < kTraceCap) {
        tr[1 + 2 * n] = (long long)tag | ((long long)(clock64() & 0xFFFFFFFFFFLL) << 16);
        tr[2 + 2 * n] = gtimer();
        d.ntrace = n + 1;
        tr[0] = n + 1;
    }
}
HDF_DEV void timer_add(int ph, long long dt) { diag().timers[ph] += dt; }

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

// Warp reduce-scatter of 16 doubles in a fixed butterfly order (deterministic).  Afterwards the
// even lane l holds the warp total of the returned value index.
HDF_DEV int warp_reduce_scatter16(double (&v)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int step = 0; step < 4; step++) {
        const int o = 16 >> step;
        const int half = 8 >> step;           // live values after this step
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; j++) {
            const double send = upper ? v[j] : v[j + half];
            const double keep = upper ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    // the upper half was kept at steps with lane bit set: index = sum of the chosen half sizes
    return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// Block reduction of 16 per-thread doubles -> out[0..15] (valid in every thread on return).
// red: shared [kClWarps][16].
HDF_DEV void block_reduce16(double (&v)[16], double* red, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int vi = warp_reduce_scatter16(v);
    if ((lane & 1) == 0) red[warp * 16 + vi] = v[0];
    __syncthreads();
    if (threadIdx.x < 16) {
        double s = 0.0;
        for (int w = 0; w < kClWarps; w++) s += red[w * 16 + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

// Block sum of a per-thread int (exact, order-free).
HDF_DEV int block_sum_int(int x, int* ired) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    x = __reduce_add_sync(0xffffffffu, x);
    if (lane == 0) ired[warp] = x;
    __syncthreads();
    int s = 0;
    for (int w = 0; w < kClWarps; w++) s += ired[w];
    __syncthreads();
    return s;
}

// Block range of the round's concatenated active points.
HDF_DEV long long blk_lo(long long T, int b, int G) { return T * b / G; }

// Farthest partner of sample row a (warp-cooperative, R3): the exact fp64 maximum of
// ||x_a - x_b||^2 over b > a, ties -> lowest b, as the oracle computes it.  Pass 1 finds the row's
// fp32 maximum M (|d32 - d| <= (rho + 3) u d for fp32 inputs, u = 2^-24); pass 2 re-evaluates in
// fp64 (the oracle's operation sequence) only the pairs with d32 >= M (1 - 8 (rho + 3) u), which
// contain every pair whose fp64 value can be the row maximum.  `base(q)` points at sample member q.
// RHO > 0: compile-time dimension (row point in registers, two candidates in flight per lane).
template <int RHO, class Base>
HDF_DEV float pair_d32(const float* xa_r, const float* xb, int rho) {
    float acc = 0.f;
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < (RHO > 0 ? RHO : 1); d++) {
            const float t = xa_r[d] - xb[d];
            acc = fmaf(t, t, acc);
        }
    } else {
        for (int d = 0; d < rho; d++) {
            const float t = xa_r[d] - xb[d];
            acc = fmaf(t, t, acc);
        }
    }
    return acc;
}

template <int RHO, class Base>
HDF_DEV void row_farthest_t(int a, int sN, int rho, Base base, double& best, int& arg) {
    const int lane = threadIdx.x & 31;
    constexpr float u = 5.9604644775390625e-08f;
    constexpr int RR = RHO > 0 ? RHO : 1;
    float xr[RR];
    const float* xa = base(a);
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) xr[d] = xa[d];
    }
    const float* xav = RHO > 0 ? xr : xa;
    float m = 0.f;
    int q = a + 1 + lane;
    for (; q + 32 < sN; q += 64) {
        const float d1 = pair_d32<RHO, Base>(xav, base(q), rho);
        const float d2 = pair_d32<RHO, Base>(xav, base(q + 32), rho);
        m = fmaxf(m, fmaxf(d1, d2));
    }
    if (q < sN) m = fmaxf(m, pair_d32<RHO, Base>(xav, base(q), rho));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float thr = m * (1.0f - 8.0f * (float)(rho + 3) * u);
    best = -1.0;
    arg = -1;
    for (q = a + 1 + lane; q < sN; q += 32) {
        const float* xb = base(q);
        if (pair_d32<RHO, Base>(xav, xb, rho) >= thr) {
            double dd = 0.0;
            for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)xa[d], (double)xb[d]);
            if (dd > best) { best = dd; arg = q; }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (oa >= 0 && (arg < 0 || ob > best || (ob == best && oa < arg))) { best = ob; arg = oa; }
    }
}

template <class Base>
HDF_DEV void row_farthest(int a, int sN, int rho, Base base, double& best, int& arg) {
    switch (rho) {
        case 1: row_farthest_t<1>(a, sN, rho, base, best, arg); break;
        case 2: row_farthest_t<2>(a, sN, rho, base, best, arg); break;
        case 3: row_farthest_t<3>(a, sN, rho, base, best, arg); break;
        case 4: row_farthest_t<4>(a, sN, rho, base, best, arg); break;
        case 6: row_farthest_t<6>(a, sN, rho, base, best, arg); break;
        default: row_farthest_t<0>(a, sN, rho, base, best, arg); break;
    }
}

// ------------------------------------------------------------------------------ plan (block 0) --
// Commit computed splits in sequential order; select the next batch of slots; lay out the blocks.
// Block 0 stages the leaf table in shared memory; thread 0 then runs the (serial) logic on it.
struct PlanSm {
    double sse[HDF_MAX_K], csse0[HDF_MAX_K], csse1[HDF_MAX_K];
    int start[HDF_MAX_K], m[HDF_MAX_K], state[HDF_MAX_K], m0[HDF_MAX_K], order[HDF_MAX_K];
    int cp_dst[HDF_MAX_K], cp_src[HDF_MAX_K];   // deferred lmean[dst] = cmean{0,1}[src] copies
    CSlot slots[kSlotCap];
    int L, status, ncp, nslots;
};

HDF_DEV void cl_plan(const ClusterArgs& A, int G, PlanSm& sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = A.K, rho = A.rho;
    const int L0 = ldi(&A.ctrl[C_NLEAVES]);
    for (int l = tid; l < L0; l += blockDim.x) {
        const CLeaf c = ld_leaf(&A.leaves[l]);
        sh.sse[l] = c.sse; sh.csse0[l] = c.csse0; sh.csse1[l] = c.csse1;
        sh.start[l] = c.start; sh.m[l] = c.m; sh.state[l] = c.state; sh.m0[l] = c.m0;
    }
    __syncthreads();
    // commits, in the sequential order: warp 0 finds the max-SSE leaf (ties -> lowest id) and
    // commits it while its split has been computed
    if (warp == 0) {
        int L = L0;
        int ncp = 0;
        int status = ldi(&A.ctrl[C_STATUS]);
        while (L < K) {
            double best = -1.0;
            int s = -1;
            for (int l = lane; l < L; l += 32)
                if (s < 0 || sh.sse[l] > best) { best = sh.sse[l]; s = l; }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int os = __shfl_xor_sync(0xffffffffu, s, o);
                if (os >= 0 && (s < 0 || ob > best || (ob == best && os < s))) { best = ob; s = os; }
            }
            if (!(best > 0.0)) { status = HDF_ERR_K; break; }
            if (sh.state[s] != 1) break;
            if (lane == 0) {   // parent keeps child 0, child 1 gets id L
                CLeaf c0, c1;
                c0.start = sh.start[s]; c0.m = sh.m0[s]; c0.state = 0; c0.m0 = 0; c0.sse = sh.csse0[s];
                c0.csse0 = c0.csse1 = 0.0;
                c1.start = sh.start[s] + sh.m0[s]; c1.m = sh.m[s] - sh.m0[s]; c1.state = 0; c1.m0 = 0;
                c1.sse = sh.csse1[s]; c1.csse0 = c1.csse1 = 0.0;
                // lmean[s] <- cmean0[s], lmean[L] <- cmean1[s]: deferred (encoded src = 2 s + side)
                sh.cp_dst[ncp] = s; sh.cp_src[ncp] = 2 * s; ncp++;
                sh.cp_dst[ncp] = L; sh.cp_src[ncp] = 2 * s + 1; ncp++;
                A.leaves[s] = c0;
                A.leaves[L] = c1;
                sh.sse[s] = c0.sse; sh.start[s] = c0.start; sh.m[s] = c0.m; sh.state[s] = 0; sh.m0[s] = 0;
                sh.sse[L] = c1.sse; sh.start[L] = c1.start; sh.m[L] = c1.m; sh.state[L] = 0; sh.m0[L] = 0;
            }
            __syncwarp();
            L++;
        }
        if (lane == 0) {
            sh.L = L;
            sh.status = status;
            sh.ncp = ncp;
            A.ctrl[C_NLEAVES] = L;
            A.ctrl[C_STATUS] = status;
        }
    }
    __syncthreads();
    // the deferred centre copies, all loads in flight at once
    for (int e = tid; e < sh.ncp * rho; e += blockDim.x) {
        const int c = e / rho, d = e - c * rho;
        const int src = sh.cp_src[c] >> 1;
        const double v = (sh.cp_src[c] & 1) ? ldd(&A.cmean1[src * rho + d]) : ldd(&A.cmean0[src * rho + d]);
        A.lmean[sh.cp_dst[c] * rho + d] = v;
    }
    const int L = sh.L;
    if (L >= K || sh.status != HDF_OK) {
        if (tid == 0) {
            A.ctrl[C_DONE] = 1;
            A.ctrl[C_NSLOTS] = 0;
        }
        return;
    }
    // order the leaves by (sse desc, id asc)
    for (int l = tid; l < L; l += blockDim.x) {
        const double v = sh.sse[l];
        int r = 0;
        for (int j = 0; j < L; j++) r += (sh.sse[j] > v) || (sh.sse[j] == v && j < l);
        sh.order[r] = l;
    }
    __syncthreads();
    if (tid == 0) {
    // batch: leaves among the top (K - L) without a computed split
    const int need = K - L;
    int nslots = 0;
    long long T = 0;
    for (int r = 0; r < need && r < L && nslots < A.slotmax; r++) {
        const int s = sh.order[r];
        if (!(sh.sse[s] > 0.0)) break;
        if (sh.state[s] == 1) continue;
        CSlot sl;
        sl.leaf = s;
        sl.start = sh.start[s];
        sl.m = sh.m[s];
        sl.stride = (sl.m + kFpCap - 1) / kFpCap;
        sl.s = (sl.m + sl.stride - 1) / sl.stride;
        sl.pbeg = T;
        T += sl.m;
        sh.slots[nslots++] = sl;
    }
    // block layout: block b owns [T b / G, T (b+1) / G)
    int rb = 0;
    for (int i = 0; i < nslots; i++) {
        CSlot& sl = sh.slots[i];
        const long long q0 = sl.pbeg, q1 = sl.pbeg + sl.m - 1;
        int b0 = (int)(q0 * G / T), b1 = (int)(q1 * G / T);
        while (b0 + 1 < G && blk_lo(T, b0 + 1, G) <= q0) b0++;
        while (b0 > 0 && blk_lo(T, b0, G) > q0) b0--;
        while (b1 + 1 < G && blk_lo(T, b1 + 1, G) <= q1) b1++;
        while (b1 > 0 && blk_lo(T, b1, G) > q1) b1--;
        sl.blo = b0;
        sl.bhi = b1;
        sl.rbase = rb;
        rb += b1 - b0 + 1;
    }
    sh.nslots = nslots;
    A.ctrl[C_NSLOTS] = nslots;
    A.ctrl[C_ROUNDS] += 1;   // only block 0 thread 0 ever writes it
    }
    __syncthreads();
    for (int i = tid; i < sh.nslots; i += blockDim.x) A.slots[i] = sh.slots[i];
}

// Per-round slot table copied to shared memory.
struct SSlot {
    int start, m, blo, rbase, nrec, stride, s;
    long long pbeg;
};

// Shared-memory point tile of the pass: A.tileF floats (points x rho, sized by the host to the
// shared memory left over) plus side bytes.
HDF_DEV int tile_pts(int tileF, int rho) { return min(tileF / rho, 16384); }
constexpr int kRecBuf = 4096;   // doubles of shared staging for record reduction
// Threads per dimension in the dimension-parallel sum phase: largest power of two <= NT / rho.
HDF_DEV int sum_tpd(int rho) {
    int t = 1;
    while (2 * t * rho <= kClThreads) t *= 2;
    return t;
}

// Block copy global -> shared of n floats with 8 loads in flight per thread (a load followed by a
// dependent shared store in a plain loop would cost one L2 round trip per iteration).
HDF_DEV void copy_g2s(float* dst, const float* src, long long n) {
    constexpr int U = 8;
    for (long long f0 = 0; f0 < n; f0 += (long long)U * kClThreads) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long f = f0 + (long long)u * kClThreads + threadIdx.x;
            v[u] = (f < n) ? __ldcg(src + f) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long f = f0 + (long long)u * kClThreads + threadIdx.x;
            if (f < n) dst[f] = v[u];
        }
    }
}

// Block copy of n bytes global -> shared (8 loads in flight per thread).
HDF_DEV void copy_bytes_g2s(unsigned char* dst, const unsigned char* src, int n) {
    constexpr int U = 8;
    for (int f0 = 0; f0 < n; f0 += U * kClThreads) {
        unsigned char v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int f = f0 + u * kClThreads + threadIdx.x;
            v[u] = (f < n) ? __ldcg(src + f) : (unsigned char)0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int f = f0 + u * kClThreads + threadIdx.x;
            if (f < n) dst[f] = v[u];
        }
    }
}

// Block copy global -> global (L2) of n floats, 8 loads in flight per thread.
HDF_DEV void copy_g2s_global(float* dst, const float* src, long long n) {
    constexpr int U = 8;
    for (long long f0 = 0; f0 < n; f0 += (long long)U * kClThreads) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long f = f0 + (long long)u * kClThreads + threadIdx.x;
            v[u] = (f < n) ? __ldcg(src + f) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long f = f0 + (long long)u * kClThreads + threadIdx.x;
            if (f < n) dst[f] = v[u];
        }
    }
}

// Copy the points of concatenated positions [q0, q1) of the round into dst.
HDF_DEV void stage_points(const float* P, int rho, int nslots, const SSlot* ss, long long q0, long long q1,
                          float* dst) {
    for (int sl = 0; sl < nslots; sl++) {
        const SSlot S = ss[sl];
        const long long a = max(q0, S.pbeg), e = min(q1, S.pbeg + (long long)S.m);
        if (a >= e) continue;
        copy_g2s(dst + (a - q0) * rho, P + ((long long)S.start + (a - S.pbeg)) * rho, (e - a) * rho);
    }
}

// Segmented, fixed-order block reduction of (s0, s1) over the `tpd` consecutive threads of each
// dimension; thread d < rho receives the totals in out[d], out[rho + d] (shared, valid on return).
HDF_DEV void block_reduce_dims(double s0, double s1, int rho, int tpd, double* red, double* out, int i0, int i1,
                               int* ired, int* iout) {
    const int tid = threadIdx.x;
    const int w = tpd < 32 ? tpd : 32;
    i0 = __reduce_add_sync(0xffffffffu, i0);
    i1 = __reduce_add_sync(0xffffffffu, i1);
    if ((tid & 31) == 0) {
        ired[2 * (tid >> 5)] = i0;
        ired[2 * (tid >> 5) + 1] = i1;
    }
    for (int o = w >> 1; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    const int ngroups = kClThreads / w;
    if ((tid % w) == 0) {
        red[2 * (tid / w)] = s0;
        red[2 * (tid / w) + 1] = s1;
    }
    __syncthreads();
    if (tid < rho) {
        const int gpd = tpd / w;   // groups per dimension
        double a = 0.0, b = 0.0;
        for (int g = tid * gpd; g < (tid + 1) * gpd && g < ngroups; g++) {
            a += red[2 * g];
            b += red[2 * g + 1];
        }
        out[tid] = a;
        out[rho + tid] = b;
    }
    if (tid == 0) {
        int a = 0, b = 0;
        for (int w2 = 0; w2 < kClWarps; w2++) {
            a += ired[2 * w2];
            b += ired[2 * w2 + 1];
        }
        iout[0] = a;
        iout[1] = b;
    }
    __syncthreads();
}

// Nearer-centre decision, certified.  The oracle decides d64(x, c0) <= d64(x, c1) in fp64 (R4).  Here
// the distances are first evaluated in fp32 against fp32-rounded centres f0, f1 (u = 2^-24):
//   t^ = fl(x - fl(c)),  d32 = FMA-accumulated sum of t^2,
//   |t^2 - t^2_exact| <= 3u (|t| + |c|)^2,   accumulation error <= rho u d32,
//   => |d32 - d| <= u ((rho + 7) d32 + 6.1 ||c||^2),
// and the fp64 evaluation error is ~2^-29 of that.  If |d32_0 - d32_1| exceeds twice the sum of the
// two bounds the fp64 decision is the same; otherwise the distances are re-evaluated in fp64 with the
// oracle's operation sequence.  Four points per thread are in flight for instruction-level
// parallelism.  cur/prev: side bytes of the tile; sw: optional global copy of the sides.
struct Centres2 {
    const double* c0;
    const double* c1;
    const float* f0;   // fp32-rounded centres
    const float* f1;
    float n0, n1;      // ||f0||^2, ||f1||^2
};

// Explicit shared-memory accesses (the pointers are generic; these avoid generic LD/ST).
HDF_DEV float lds_f(const float* p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}
HDF_DEV unsigned lds_u8(const unsigned char* p) {
    unsigned short v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(smem_u32(p)));
    return v;
}
HDF_DEV void sts_u8(unsigned char* p, unsigned v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(smem_u32(p)), "h"((unsigned short)v) : "memory");
}

template <int RHO>
HDF_DEV void side_phase_t(const float* xt, int np, int rho_rt, const Centres2& C2, const unsigned char* prev,
                          unsigned char* cur, unsigned char* sw, int it, int& n1, int& chg) {
    constexpr int U = 4;
    constexpr float u = 5.9604644775390625e-08f;   // 2^-24
    const int rho = RHO > 0 ? RHO : rho_rt;
    const float kc = 2.0f * u * 6.1f * (C2.n0 + C2.n1);
    const float kd = 2.0f * u * (float)(rho + 7);
    constexpr int RR = RHO > 0 ? RHO : 1;
    float g0r[RR], g1r[RR];
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) { g0r[d] = lds_f(C2.f0 + d); g1r[d] = lds_f(C2.f1 + d); }
    }
    for (int t0 = threadIdx.x; t0 < np; t0 += U * kClThreads) {
        float a0[U], a1[U];
#pragma unroll
        for (int q = 0; q < U; q++) { a0[q] = 0.f; a1[q] = 0.f; }
        if (RHO > 0) {
            float xv[U][RR];
#pragma unroll
            for (int q = 0; q < U; q++) {
                const int t = min(t0 + q * kClThreads, np - 1);
#pragma unroll
                for (int d = 0; d < RR; d++) xv[q][d] = lds_f(xt + (size_t)t * RR + d);
            }
#pragma unroll
            for (int q = 0; q < U; q++) {
#pragma unroll
                for (int d = 0; d < RR; d++) {
                    const float e0 = xv[q][d] - g0r[d], e1 = xv[q][d] - g1r[d];
                    a0[q] = fmaf(e0, e0, a0[q]);
                    a1[q] = fmaf(e1, e1, a1[q]);
                }
            }
        } else {
            for (int d = 0; d < rho; d++) {
                const float g0 = lds_f(C2.f0 + d), g1 = lds_f(C2.f1 + d);
#pragma unroll
                for (int q = 0; q < U; q++) {
                    const int t = min(t0 + q * kClThreads, np - 1);
                    const float x = lds_f(xt + (size_t)t * rho + d);
                    const float e0 = x - g0, e1 = x - g1;
                    a0[q] = fmaf(e0, e0, a0[q]);
                    a1[q] = fmaf(e1, e1, a1[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int t = t0 + q * kClThreads;
            if (t < np) {
                const float diff = a0[q] - a1[q];
                const float bound = kd * (a0[q] + a1[q]) + kc;
                int sd;
                if (fabsf(diff) > bound) {
                    sd = diff > 0.f ? 1 : 0;
                } else {   // inside the uncertainty band: the oracle's fp64 sequence
                    const float* x = xt + (size_t)t * rho;
                    double dd0 = 0.0, dd1 = 0.0;
                    for (int d = 0; d < rho; d++) {
                        const double v = (double)x[d];
                        dd0 = d2_rn(dd0, v, C2.c0[d]);
                        dd1 = d2_rn(dd1, v, C2.c1[d]);
                    }
                    sd = (dd0 <= dd1) ? 0 : 1;
                }
                if (it > 0 && sd != (int)lds_u8(prev + t)) chg++;
                sts_u8(cur + t, (unsigned)sd);
                if (sw) sw[t] = (unsigned char)sd;
                n1 += sd;
            }
        }
    }
}

HDF_DEV void side_phase(const float* xt, int np, int rho, const Centres2& C2, const unsigned char* prev,
                        unsigned char* cur, unsigned char* sw, int it, int& n1, int& chg) {
    switch (rho) {
        case 1: side_phase_t<1>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
        case 2: side_phase_t<2>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
        case 3: side_phase_t<3>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
        case 4: side_phase_t<4>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
        case 6: side_phase_t<6>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
        default: side_phase_t<0>(xt, np, rho, C2, prev, cur, sw, it, n1, chg); break;
    }
}

// Dimension-parallel fp64 sums of a tile by side: thread (dsum, jsum) adds points jsum, jsum + tpd,
// ... of dimension dsum, alternating over four accumulators per side (fixed order).
HDF_DEV void sum_phase(const float* xt, int np, int rho, const unsigned char* cur, int tpd, double (&s0)[4],
                       double (&s1)[4]) {
    const int dsum = threadIdx.x / tpd, jsum = threadIdx.x % tpd;
    if (dsum >= rho) return;
    for (int t0 = jsum; t0 < np; t0 += 4 * tpd) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int t = t0 + q * tpd;
            if (t < np) {
                const double v = (double)lds_f(xt + (size_t)t * rho + dsum);
                if (lds_u8(cur + t)) s1[q] += v;
                else s0[q] += v;
            }
        }
    }
}

// fp32 copies and squared norms of the two centres of a slot (threads d < rho).
HDF_DEV void make_centres2(const double* c0, const double* c1, int rho, float* f0, float* f1, float* norms) {
    for (int d = threadIdx.x; d < rho; d += kClThreads) {
        f0[d] = (float)c0[d];
        f1[d] = (float)c1[d];
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        const float* f = threadIdx.x ? f1 : f0;
        float nn = 0.f;
        for (int d = 0; d < rho; d++) nn = fmaf(f[d], f[d], nn);
        norms[threadIdx.x] = nn;
    }
    __syncthreads();
}

// One lock-step Lloyd pass over this block's range: assign every member to the nearer centre (ties
// -> first), count changes against the previous assignment, and write the block's partial record
// per slot (sum0[rho], sum1[rho], n1, changed).  `only` restricts to slots with only[sl] != 0.
// Points come from the shared tile: resident for the whole round when the block's range fits
// (then the previous sides are kept in shared memory too), otherwise staged tile by tile.
HDF_DEV void cl_pass(const ClusterArgs& A, const float* P, int nslots, const SSlot* ss, long long T,
                     const double* cen0, const double* cen1, const int* s_conv, const int* only, int it, int wb,
                     double* red, int* ired, double* outv, float* tp, unsigned char* tsd, bool resident) {
    const int rho = A.rho;
    const int tid = threadIdx.x;
    const int b = blockIdx.x, G = gridDim.x;
    const long long lo = blk_lo(T, b, G), hi = blk_lo(T, b + 1, G);
    if (lo >= hi) return;
    const int TP = tile_pts(A.tileF, rho);
    const int tpd = sum_tpd(rho);
    unsigned char* sw = A.side[wb];
    const unsigned char* sp = A.side[wb ^ 1];
    double* recb = A.rec[wb];
    const bool tm = (A.timers != nullptr) && b == 0 && tid == 0;
    long long tq = tm ? gtimer() : 0;
    auto tk = [&](int ph) {
        if (tm) {
            const long long t1 = gtimer();
            timer_add(ph, t1 - tq);
            tq = t1;
        }
    };
    for (int sl = 0; sl < nslots; sl++) {
        const SSlot S = ss[sl];
        if (S.pbeg + S.m <= lo || S.pbeg >= hi) continue;
        if (s_conv[sl]) continue;
        if (only && !only[sl]) continue;
        const int a = (int)(max(lo, S.pbeg) - S.pbeg), e = (int)(min(hi, S.pbeg + S.m) - S.pbeg);
        const double* c0 = cen0 + sl * rho;
        const double* c1 = cen1 + sl * rho;
        double* rec = recb + (size_t)(S.rbase + b - S.blo) * A.pstride;
        int n1 = 0, chg = 0;
        double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
        for (int ta = a; ta < e; ta += TP) {
            const int te = min(e, ta + TP), np = te - ta;
            const float* xt;
            unsigned char* cur_sd;
            const unsigned char* prev_sd;
            __syncthreads();   // previous tile fully consumed
            if (resident) {
                const long long off = S.pbeg + ta - lo;
                xt = tp + off * rho;
                cur_sd = tsd + (size_t)wb * TP + off;
                prev_sd = tsd + (size_t)(wb ^ 1) * TP + off;
            } else {
                stage_points(P, rho, 1, &S, S.pbeg + ta, S.pbeg + te, tp);
                xt = tp;
                cur_sd = tsd;
                prev_sd = tsd + TP;
                if (it > 0) copy_bytes_g2s(tsd + TP, sp + S.start + ta, np);
                __syncthreads();
            }
            // side phase (certified fp32, see side_phase) and per-side fp64 sums
            {
                __shared__ float f01[2 * HDF_MAX_RHO + 2];
                make_centres2(c0, c1, rho, f01, f01 + HDF_MAX_RHO, f01 + 2 * HDF_MAX_RHO);
                Centres2 C2{c0, c1, f01, f01 + HDF_MAX_RHO, f01[2 * HDF_MAX_RHO], f01[2 * HDF_MAX_RHO + 1]};
                side_phase(xt, np, rho, C2, prev_sd, cur_sd, sw + S.start + ta, it, n1, chg);
            }
            __syncthreads();
            tk(T_P_SIDE);
            sum_phase(xt, np, rho, cur_sd, tpd, s0, s1);
        }
        tk(T_P_SUM);
        int* iout = ired + 2 * kClWarps;
        block_reduce_dims((s0[0] + s0[1]) + (s0[2] + s0[3]), (s1[0] + s1[1]) + (s1[2] + s1[3]), rho, tpd, red, outv, n1,
                          chg, ired, iout);
        for (int d = tid; d < rho; d += kClThreads) {
            rec[d] = outv[d];
            rec[rho + d] = outv[rho + d];
        }
        if (tid == 0) {
            rec[2 * rho] = (double)iout[0];
            rec[2 * rho + 1] = (double)iout[1];
        }
        tk(T_P_RED);
    }
}

// Reduce the records of every listed slot, in a fixed order, into tmpv[sl][v0 .. v0 + nv).  The
// records of a group of slots are first staged in shared memory with all loads in flight at once
// (one L2 round trip), then a warp per (slot, value) pair sums them: lanes stride over the
// records, xor-tree finish.  Identical in every block, so every block derives bit-identical
// centres.  A slot whose records do not fit the buffer is reduced straight from L2.
HDF_DEV void cl_reduce_records(const ClusterArgs& A, const double* recb, int nslots, const SSlot* ss,
                               const int* skip, int v0, int nv, double* tmpv, double* sbuf, int* soff) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int sl0 = 0;
    while (sl0 < nslots) {
        // group [sl0, sl1) whose staged records fit kRecBuf (uniform across the block)
        int sl1 = sl0, size = 0;
        while (sl1 < nslots) {
            const int need = (skip && skip[sl1]) ? 0 : ss[sl1].nrec * nv;
            if (size + need > kRecBuf) break;
            size += need;
            sl1++;
        }
        if (sl1 == sl0) {   // one oversized slot: reduce from L2 directly
            if (!(skip && skip[sl0])) {
                const SSlot S = ss[sl0];
                for (int v = warp; v < nv; v += kClWarps) {
                    double sacc = 0.0;
#pragma unroll 4
                    for (int j = lane; j < S.nrec; j += 32) sacc += ldd(recb + (size_t)(S.rbase + j) * A.pstride + v0 + v);
                    sacc = warp_sum(sacc);
                    if (lane == 0) tmpv[sl0 * A.pstride + v0 + v] = sacc;
                }
            }
            __syncthreads();
            sl0++;
            continue;
        }
        if (tid == 0) {
            int o = 0;
            for (int sl = sl0; sl < sl1; sl++) {
                soff[sl] = o;
                o += (skip && skip[sl]) ? 0 : ss[sl].nrec * nv;
            }
        }
        __syncthreads();
        {
            // flattened over the group: 8 loads in flight per thread, then the shared stores
            constexpr int U = kRecBuf / kClThreads;
            double v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = u * kClThreads + tid;
                v[u] = 0.0;
                if (f < size) {
                    int sl = sl0;
                    while (sl + 1 < sl1 && soff[sl + 1] <= f) sl++;
                    const int q = f - soff[sl];
                    const int j = q / nv, vv = q - j * nv;
                    v[u] = ldd(recb + (size_t)(ss[sl].rbase + j) * A.pstride + v0 + vv);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = u * kClThreads + tid;
                if (f < size) sbuf[f] = v[u];
            }
        }
        __syncthreads();
        const int npairs = (sl1 - sl0) * nv;
        for (int pr = warp; pr < npairs; pr += kClWarps) {
            const int sl = sl0 + pr / nv, v = pr % nv;
            if (skip && skip[sl]) continue;
            const int nrec = ss[sl].nrec;
            const double* src = sbuf + soff[sl] + v;
            double sacc = 0.0;
            for (int j = lane; j < nrec; j += 32) sacc += src[j * nv];
            sacc = warp_sum(sacc);
            if (lane == 0) tmpv[sl * A.pstride + v0 + v] = sacc;
        }
        __syncthreads();
        sl0 = sl1;
    }
}

// Finalise one iteration for every active slot, redundantly in every block.  Returns 1 if some
// slot came out with an empty side (s_rs[sl] = 1: side 1 empty, 2: side 0 empty).
HDF_DEV int cl_finalize(const ClusterArgs& A, int nslots, const SSlot* ss, int it, int wb, double* cen0,
                        double* cen1, int* s_conv, int* s_rs, int* s_fbuf, bool redo, double* tmpv, double* sbuf,
                        int* soff) {
    const int rho = A.rho;
    const int tid = threadIdx.x;
    cl_reduce_records(A, A.rec[wb], nslots, ss, s_conv, 0, 2 * rho + 2, tmpv, sbuf, soff);
    int any = 0;
    // new centres: thread per (slot, dimension)
    for (int e = tid; e < nslots * rho; e += kClThreads) {
        const int sl = e / rho, d = e - sl * rho;
        if (s_conv[sl] || (redo && !s_rs[sl])) continue;
        const double* tv = tmpv + sl * A.pstride;
        const long long m = ss[sl].m;
        const long long n1 = (long long)tv[2 * rho];
        const long long chg = (long long)tv[2 * rho + 1];
        const bool empty_side = !redo && (n1 == 0 || n1 == m);
        const bool conv = it > 0 && chg == 0;
        if (!empty_side && !conv) {
            cen0[sl * rho + d] = tv[d] / (double)(m - n1);
            cen1[sl * rho + d] = tv[rho + d] / (double)n1;
        }
    }
    __syncthreads();
    // slot state: thread per slot
    for (int sl = tid; sl < nslots; sl += kClThreads) {
        if (s_conv[sl]) continue;
        if (redo && !s_rs[sl]) continue;
        const double* tv = tmpv + sl * A.pstride;
        const long long m = ss[sl].m;
        const long long n1 = (long long)tv[2 * rho];
        const long long chg = (long long)tv[2 * rho + 1];
        if (!redo && (n1 == 0 || n1 == m)) {
            any = 1;
            s_rs[sl] = (n1 == 0) ? 1 : 2;
        } else if (it > 0 && chg == 0) {
            s_conv[sl] = 1;
            s_fbuf[sl] = wb;
        } else {
            s_fbuf[sl] = wb;
        }
    }
    any = __syncthreads_or(any);
    if (redo) {
        for (int sl = tid; sl < nslots; sl += kClThreads) s_rs[sl] = 0;
        __syncthreads();
    }
    return any;
}

// Farthest member of a reseed slot's leaf from the non-empty side's centre (ties -> first in
// member order); the block owning the slot writes the new centre to c0g / c1g.
HDF_DEV void cl_reseed(const ClusterArgs& A, const float* P, int nslots, const SSlot* ss, const double* cen0,
                       const double* cen1, const int* s_rs, double* red) {
    const int rho = A.rho;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int sl = blockIdx.x; sl < nslots; sl += gridDim.x) {
        const int rs = s_rs[sl];
        if (!rs) continue;
        const int start = ss[sl].start, m = ss[sl].m;
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

// ------------------------------------------------------------- cluster mode (one split per cluster) --
// A round whose slots are all small enough runs every split inside one thread-block cluster of C CTAs
// (slots dealt round-robin to the clusters): farthest-pair seeding, Lloyd iterations, reseeds, the
// stable partition and the child SSE.  CTA r owns the members [m r / C, m (r+1) / C) of the leaf.
// Partial records are exchanged through distributed shared memory and reduced in rank order by every
// CTA (bit-identical centres in the cluster); one cluster barrier per Lloyd iteration.
struct ClSm {
    double part[2][2 * HDF_MAX_RHO + 4];   // parity-buffered partial record: sum0, sum1, n1, changed
    double best_v;                         // farthest-pair / reseed candidate of this CTA
    long long best_a, best_b;
    double sse[2];
};

// Lloyd pass over members [a, e) of a leaf stored at gbase: assignment (ties -> first centre),
// changes against the previous assignment, per-side fp64 sums.  Sums -> outv[0, 2 rho), n1 and the
// change count -> iout[0], iout[1].
HDF_DEV void cl_pass_range(const ClusterArgs& A, const float* P, long long gbase, int a, int e, const double* c0,
                           const double* c1, int it, int wb, bool resident, float* tp, unsigned char* tsd, int TP,
                           double* red, int* ired, double* outv, int* iout) {
    const int rho = A.rho;
    const int tpd = sum_tpd(rho);
    unsigned char* sw = A.side[wb];
    const unsigned char* sp = A.side[wb ^ 1];
    __shared__ float f01[2 * HDF_MAX_RHO + 2];
    make_centres2(c0, c1, rho, f01, f01 + HDF_MAX_RHO, f01 + 2 * HDF_MAX_RHO);
    const Centres2 C2{c0, c1, f01, f01 + HDF_MAX_RHO, f01[2 * HDF_MAX_RHO], f01[2 * HDF_MAX_RHO + 1]};
    int n1 = 0, chg = 0;
    double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
    for (int ta = a; ta < e; ta += TP) {
        const int te = min(e, ta + TP), np = te - ta;
        const float* xt;
        unsigned char* cur_sd;
        const unsigned char* prev_sd;
        __syncthreads();   // previous tile fully consumed
        if (resident) {
            xt = tp + (size_t)(ta - a) * rho;
            cur_sd = tsd + (size_t)wb * TP + (ta - a);
            prev_sd = tsd + (size_t)(wb ^ 1) * TP + (ta - a);
        } else {
            copy_g2s(tp, P + (gbase + ta) * rho, (long long)np * rho);
            xt = tp;
            cur_sd = tsd;
            prev_sd = tsd + TP;
            if (it > 0) copy_bytes_g2s(tsd + TP, sp + gbase + ta, np);
            __syncthreads();
        }
        trace_ev(A.trace, 40);
        side_phase(xt, np, rho, C2, prev_sd, cur_sd, resident ? nullptr : sw + gbase + ta, it, n1, chg);
        __syncthreads();
        trace_ev(A.trace, 41);
        sum_phase(xt, np, rho, cur_sd, tpd, s0, s1);
    }
    trace_ev(A.trace, 42);
    block_reduce_dims((s0[0] + s0[1]) + (s0[2] + s0[3]), (s1[0] + s1[1]) + (s1[2] + s1[3]), rho, tpd, red, outv, n1,
                      chg, ired, iout);
    trace_ev(A.trace, 43);
}

// (value desc, a asc) candidate order shared by the farthest-pair and farthest-member searches.
HDF_DEV bool cand_better(double v, long long a, double bv, long long ba) {
    return a >= 0 && (ba < 0 || v > bv || (v == bv && a < ba));
}

HDF_DEV void cl_split_cluster(const ClusterArgs& A, const SSlot& S, int leaf, int cur, double* cen0, double* cen1,
                              double* red, int* ired, double* outv, double* tmpv, double* sbuf, float* tp,
                              unsigned char* tsd, ClSm& X) {
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
    const int rho = A.rho, nv = 2 * rho + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* P = A.pts[cur];
    float* Pn = A.pts[cur ^ 1];
    const int m = S.m;
    const long long gbase = S.start;
    const int a = (int)((long long)m * r / C), e = (int)((long long)m * (r + 1) / C);
    __shared__ long long s_pair[2];
    const bool tm = (A.timers != nullptr) && blockIdx.x == 0 && tid == 0;
    long long tq = tm ? gtimer() : 0;
    auto tk = [&](int ph) {
        if (tm) {
            const long long t1 = gtimer();
            timer_add(ph, t1 - tq);
            tq = t1;
        }
    };

    // ---- 1. farthest pair of the stride sample members[0::stride] (R3) ----
    trace_ev(A.trace, 1);
    const int stride = S.stride, sN = S.s;
    const bool insm = (long long)sN * rho <= A.tileF;
    __syncthreads();
    if (insm) {
        constexpr int U = 8;
        for (int f0 = 0; f0 < sN * rho; f0 += U * kClThreads) {
            float v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = f0 + u * kClThreads + tid;
                const int q = f / rho, d = f - q * rho;
                v[u] = (f < sN * rho) ? __ldcg(P + (gbase + (long long)q * stride) * rho + d) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = f0 + u * kClThreads + tid;
                if (f < sN * rho) tp[f] = v[u];
            }
        }
    }
    __syncthreads();
    trace_ev(A.trace, 2);
    {
        double bv = -1.0;
        long long ba = -1, bb = -1;
        for (int ra = r + C * warp; ra < sN; ra += C * kClWarps) {   // rows ascending within the warp
            double best;
            int arg;
            const float* tpc = tp;
            if (insm)
                row_farthest(ra, sN, rho, [&](int q) { return tpc + (size_t)q * rho; }, best, arg);
            else
                row_farthest(ra, sN, rho, [&](int q) { return P + (gbase + (long long)q * stride) * rho; }, best, arg);
            if (arg >= 0 && (ba < 0 || best > bv)) { bv = best; ba = ra; bb = arg; }
        }
        if (lane == 0) {
            red[3 * warp] = bv;
            red[3 * warp + 1] = (double)ba;
            red[3 * warp + 2] = (double)bb;
        }
        __syncthreads();
        if (tid == 0) {
            double v = -1.0;
            long long ia = -1, ib = -1;
            for (int w = 0; w < kClWarps; w++) {
                const long long wa = (long long)red[3 * w + 1];
                if (cand_better(red[3 * w], wa, v, ia)) { v = red[3 * w]; ia = wa; ib = (long long)red[3 * w + 2]; }
            }
            X.best_v = v;
            X.best_a = ia;
            X.best_b = ib;
        }
    }
    trace_ev(A.trace, 3);
    cl.sync();
    trace_ev(A.trace, 4);
    if (tid == 0) {
        double v = -1.0;
        long long ia = -1, ib = -1;
        for (int q = 0; q < C; q++) {
            const ClSm* Y = cl.map_shared_rank(&X, q);
            const long long qa = Y->best_a;
            if (cand_better(Y->best_v, qa, v, ia)) { v = Y->best_v; ia = qa; ib = Y->best_b; }
        }
        if (ia < 0) { ia = 0; ib = 0; }
        s_pair[0] = ia;
        s_pair[1] = ib;
    }
    __syncthreads();
    for (int f = tid; f < 2 * rho; f += kClThreads) {
        const int w = f / rho, d = f - w * rho;
        const long long q = s_pair[w];
        const double v = insm ? (double)tp[q * rho + d] : (double)__ldcg(P + (gbase + q * stride) * rho + d);
        (w ? cen1 : cen0)[d] = v;
    }
    tk(T_P_SIDE);
    // ---- 2. the CTA's members stay resident in shared memory when they fit ----
    const int TP = tile_pts(A.tileF, rho);
    const bool resident = (e - a) <= TP;
    __syncthreads();
    if (resident) copy_g2s(tp, P + (gbase + a) * rho, (long long)(e - a) * rho);
    __syncthreads();
    trace_ev(A.trace, 5);

    // ---- 3. Lloyd iterations (R4) ----
    int* iout = ired + 2 * kClWarps;
    int fbuf = (kMaxIter - 1) & 1;
    int it = 0;
    for (; it < kMaxIter; it++) {
        const int wb = it & 1;
        bool redo = false;
        while (true) {
            cl_pass_range(A, P, gbase, a, e, cen0, cen1, it, wb, resident, tp, tsd, TP, red, ired, outv, iout);
            for (int v = tid; v < 2 * rho; v += kClThreads) X.part[wb][v] = outv[v];
            if (tid == 0) {
                X.part[wb][2 * rho] = (double)iout[0];
                X.part[wb][2 * rho + 1] = (double)iout[1];
            }
            trace_ev(A.trace, 10);
            cl.sync();
            trace_ev(A.trace, 11);
            // every CTA gathers the C partial records and sums them in rank order
            for (int f = tid; f < C * nv; f += kClThreads) {
                const int q = f / nv, v = f - q * nv;
                sbuf[f] = cl.map_shared_rank(&X, q)->part[wb][v];
            }
            __syncthreads();
            for (int v = tid; v < nv; v += kClThreads) {
                double acc = 0.0;
                for (int q = 0; q < C; q++) acc += sbuf[q * nv + v];
                tmpv[v] = acc;
            }
            __syncthreads();
            trace_ev(A.trace, 12);
            const long long n1 = (long long)tmpv[2 * rho];
            if (redo || !(n1 == 0 || n1 == m)) break;
            // empty side: move its centre to the member farthest from the other centre (ties ->
            // first in member order), then redo this iteration's assignment
            const int rs = (n1 == 0) ? 1 : 2;
            const double* cref = (rs == 1) ? cen0 : cen1;
            double best = -1.0;
            long long arg = -1;
            for (int t = a + tid; t < e; t += kClThreads) {
                const float* x = resident ? tp + (size_t)(t - a) * rho : P + (gbase + t) * rho;
                double dd = 0.0;
                for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)x[d], cref[d]);
                if (dd > best) { best = dd; arg = t; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const long long oa = __shfl_xor_sync(0xffffffffu, arg, o);
                if (cand_better(ob, oa, best, arg)) { best = ob; arg = oa; }
            }
            if (lane == 0) { red[2 * warp] = best; red[2 * warp + 1] = (double)arg; }
            __syncthreads();
            if (tid == 0) {
                double v = -1.0;
                long long ia = -1;
                for (int w = 0; w < kClWarps; w++) {
                    const long long wa = (long long)red[2 * w + 1];
                    if (cand_better(red[2 * w], wa, v, ia)) { v = red[2 * w]; ia = wa; }
                }
                X.best_v = v;
                X.best_a = ia;
            }
            cl.sync();   // also: every CTA has gathered this parity's records
            if (tid == 0) {
                double v = -1.0;
                long long ia = -1;
                for (int q = 0; q < C; q++) {
                    const ClSm* Y = cl.map_shared_rank(&X, q);
                    if (cand_better(Y->best_v, Y->best_a, v, ia)) { v = Y->best_v; ia = Y->best_a; }
                }
                s_pair[0] = ia;
            }
            __syncthreads();
            double* cnew = (rs == 1) ? cen1 : cen0;
            for (int d = tid; d < rho; d += kClThreads) cnew[d] = (double)__ldcg(P + (gbase + s_pair[0]) * rho + d);
            __syncthreads();
            redo = true;
        }
        const long long n1 = (long long)tmpv[2 * rho];
        const long long chg = (long long)tmpv[2 * rho + 1];
        fbuf = wb;
        if (it > 0 && chg == 0) break;   // converged: the final assignment is this pass
        for (int d = tid; d < rho; d += kClThreads) {
            cen0[d] = tmpv[d] / (double)(m - n1);
            cen1[d] = tmpv[rho + d] / (double)n1;
        }
        __syncthreads();
        trace_ev(A.trace, 13);
    }
    if (it == kMaxIter) it = kMaxIter - 1;
    if (r == 0 && tid == 0) atomicAdd(&A.ctrl[C_ITERS], it + 1);
    tk(T_P_SUM);

    // ---- 4. stable partition by side + child SSE ----
    // n1 of every CTA from the final partial records (parity fbuf, untouched since the last gather)
    if (tid == 0) {
        long long pre1 = 0, tot1 = 0;
        for (int q = 0; q < C; q++) {
            const long long v = (long long)cl.map_shared_rank(&X, q)->part[fbuf][2 * rho];
            if (q < r) pre1 += v;
            tot1 += v;
        }
        s_pair[0] = pre1;
        s_pair[1] = tot1;
    }
    __syncthreads();
    const long long pre1 = s_pair[0], tot1 = s_pair[1];
    const long long m0 = m - tot1, pre0 = a - pre1;
    // final sides: shared (resident) or global, through one generic pointer (no speculative loads)
    const unsigned char* sdsrc = resident ? tsd + (size_t)fbuf * TP - a : A.side[fbuf] + gbase;
    double se0 = 0.0, se1 = 0.0;
    long long run0 = 0, run1 = 0;
    for (int t0 = a; t0 < e; t0 += kClThreads) {
        const int t = t0 + tid;
        const bool ok = t < e;
        const int sd = ok ? (int)sdsrc[t] : 0;
        const int f0 = (ok && sd == 0) ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f0);
        if (lane == 0) ired[warp] = __popc(bal);
        __syncthreads();
        int wpre = 0, total0 = 0;
        for (int w = 0; w < kClWarps; w++) {
            const int v = ired[w];
            if (w < warp) wpre += v;
            total0 += v;
        }
        const int incl = wpre + __popc(bal & ((lane == 31) ? 0xffffffffu : ((1u << (lane + 1)) - 1u)));
        __syncthreads();
        if (ok) {
            const int rank0 = incl - f0;
            const int rank1 = (t - t0) - rank0;
            const long long dst = gbase + (sd == 0 ? pre0 + run0 + rank0 : m0 + pre1 + run1 + rank1);
            const float* x = P + (gbase + t) * rho;
            const double* cc = sd ? cen1 : cen0;
            double dd = 0.0;
            for (int d = 0; d < rho; d++) {
                const float v = __ldcg(x + d);
                Pn[dst * rho + d] = v;
                dd = d2_rn(dd, (double)v, cc[d]);
            }
            A.idx[cur ^ 1][dst] = __ldcg(A.idx[cur] + gbase + t);
            if (sd) se1 += dd;
            else se0 += dd;
        }
        const int nvalid = min(kClThreads, e - t0);
        run0 += total0;
        run1 += nvalid - total0;
    }
    {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0;
        acc[0] = se0;
        acc[1] = se1;
        block_reduce16(acc, red, outv);
    }
    if (tid == 0) {
        X.sse[0] = outv[0];
        X.sse[1] = outv[1];
    }
    trace_ev(A.trace, 20);
    __threadfence();
    cl.sync();   // the cluster's scatter is complete and visible
    trace_ev(A.trace, 21);
    // copy back the CTA's own range of the (now partitioned) segment
    copy_g2s_global(A.pts[cur] + (gbase + a) * rho, Pn + (gbase + a) * rho, (long long)(e - a) * rho);
    for (int t = a + tid; t < e; t += kClThreads) A.idx[cur][gbase + t] = __ldcg(A.idx[cur ^ 1] + gbase + t);
    if (r == 0 && tid == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int q = 0; q < C; q++) {
            const ClSm* Y = cl.map_shared_rank(&X, q);
            s0 += Y->sse[0];
            s1 += Y->sse[1];
        }
        A.leaves[leaf].m0 = (int)m0;
        A.leaves[leaf].csse0 = s0;
        A.leaves[leaf].csse1 = s1;
        for (int d = 0; d < rho; d++) {
            A.cmean0[leaf * rho + d] = cen0[d];
            A.cmean1[leaf * rho + d] = cen1[d];
        }
        __threadfence();
        A.leaves[leaf].state = 1;
    }
    trace_ev(A.trace, 22);
    cl.sync();   // X (sse, part) is read by rank 0 before any CTA reuses it for the next slot
    trace_ev(A.trace, 23);
    tk(T_P_RED);
}

// ------------------------------------------------------------------------------- the kernel ---
__global__ void __launch_bounds__(kClThreads) k_bisect_kmeans(const ClusterArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm_cl[];
    const int rho = A.rho, K = A.K;
    double* red = sm_cl;                              // [2 * kClThreads] reduction scratch
    double* cen0 = red + 2 * kClThreads;              // [slotmax][rho] block-local centres
    double* cen1 = cen0 + A.slotmax * rho;
    double* tmpv = cen1 + A.slotmax * rho;            // [slotmax][pstride]
    double* outv = tmpv + A.slotmax * A.pstride;      // [2 rho + 16]
    float* tp = reinterpret_cast<float*>(outv + 2 * rho + 16);          // [tileF] point tile
    double* sbuf = reinterpret_cast<double*>(tp + A.tileF);             // [kRecBuf] record staging
    unsigned char* tsd = reinterpret_cast<unsigned char*>(sbuf + kRecBuf); // [2][tile_pts] sides
    __shared__ int s_conv[kSlotCap];
    __shared__ int s_rs[kSlotCap];
    __shared__ int s_fbuf[kSlotCap];
    __shared__ int ired[2 * kClWarps + 2];
    __shared__ SSlot ss[kSlotCap];
    __shared__ PlanSm plan_sm;
    __shared__ int soff[kSlotCap];
    __shared__ ClSm clx;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const long long gtid = (long long)blockIdx.x * blockDim.x + tid;
    const long long gthreads = (long long)G * blockDim.x;
    const bool timer = (A.timers != nullptr) && blockIdx.x == 0 && tid == 0;
    long long t0 = timer ? gtimer() : 0;
    auto tick = [&](int ph) {
        if (timer) {
            const long long t1 = gtimer();
            timer_add(ph, t1 - t0);
            t0 = t1;
        }
    };
    int ph_cur = T_PLAN;   // phase the work before the next barrier belongs to
    auto gsync = [&]() {
        tick(ph_cur);
        grid.sync();
        tick(T_SYNC);
    };

    if (blockIdx.x == 0 && tid == 0) {
        for (int c = 0; c < 16; c++) diag().timers[c] = 0;
        diag().ntrace = 0;
    }
    // ---- init: copy Theta into leaf storage, root leaf = all pixels in pixel order -----------
    for (long long e = gtid; e < (long long)A.N * rho; e += gthreads) A.pts[0][e] = A.p[e];
    for (long long e = gtid; e < A.N; e += gthreads) A.idx[0][e] = (int)e;
    if (gtid == 0) {
        for (int c = 0; c < C_NUM; c++) A.ctrl[c] = 0;
        A.ctrl[C_NLEAVES] = 1;
        if (A.trace) A.trace[0] = 0;
    }
    // root mean and SSE: per-block records over a fixed contiguous range, reduced in block order
    const long long per = ((long long)A.N + G - 1) / G;
    const long long rb0 = min((long long)A.N, (long long)blockIdx.x * per), rb1 = min((long long)A.N, rb0 + per);
    for (int d0 = 0; d0 < rho; d0 += kDC) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0;
        for (long long t = rb0 + tid; t < rb1; t += blockDim.x) {
#pragma unroll
            for (int j = 0; j < kDC; j++)
                if (d0 + j < rho) acc[j] += (double)A.p[t * rho + d0 + j];
        }
        block_reduce16(acc, red, outv);
        if (tid < kDC && d0 + tid < rho) A.rec[0][(size_t)blockIdx.x * A.pstride + d0 + tid] = outv[tid];
    }
    grid.sync();
    for (int d = tid; d < rho; d += blockDim.x) {
        double s = 0.0;
        for (int bI = 0; bI < G; bI++) s += ldd(&A.rec[0][(size_t)bI * A.pstride + d]);
        tmpv[d] = s / (double)A.N;
    }
    __syncthreads();
    {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0;
        for (long long t = rb0 + tid; t < rb1; t += blockDim.x) {
            double dd = 0.0;
            for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)A.p[t * rho + d], tmpv[d]);
            acc[0] += dd;
        }
        block_reduce16(acc, red, outv);
        if (tid == 0) A.rec[1][(size_t)blockIdx.x * A.pstride] = outv[0];
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {
        double s = 0.0;
        for (int bI = 0; bI < G; bI++) s += ldd(&A.rec[1][(size_t)bI * A.pstride]);
        CLeaf r;
        r.start = 0; r.m = A.N; r.state = 0; r.m0 = 0; r.sse = s; r.csse0 = r.csse1 = 0.0;
        A.leaves[0] = r;
        for (int d = 0; d < rho; d++) A.lmean[d] = tmpv[d];
    }
    grid.sync();

    int cur = 0;   // which pts/idx buffer holds the leaf storage
    while (true) {
        // ---------------- plan ----------------
        ph_cur = T_PLAN;
        trace_ev(A.trace, 30);
        if (blockIdx.x == 0) cl_plan(A, G, plan_sm);
        trace_ev(A.trace, 31);
        gsync();
        trace_ev(A.trace, 32);
        ph_cur = T_SEED;
        if (ldi(&A.ctrl[C_DONE])) break;
        const int nslots = ldi(&A.ctrl[C_NSLOTS]);
        const float* P = A.pts[cur];
        for (int sl = tid; sl < nslots; sl += blockDim.x) {
            SSlot S;
            S.start = ldi(&A.slots[sl].start);
            S.m = ldi(&A.slots[sl].m);
            S.blo = ldi(&A.slots[sl].blo);
            S.rbase = ldi(&A.slots[sl].rbase);
            S.nrec = ldi(&A.slots[sl].bhi) - S.blo + 1;
            S.pbeg = ldll(&A.slots[sl].pbeg);
            S.stride = ldi(&A.slots[sl].stride);
            S.s = ldi(&A.slots[sl].s);
            ss[sl] = S;
        }
        __syncthreads();
        const long long T = ss[nslots - 1].pbeg + ss[nslots - 1].m;
        int maxm = 0;
        for (int sl = 0; sl < nslots; sl++) maxm = max(maxm, ss[sl].m);
        if (maxm <= A.big) {
            // ---------------- cluster mode: every split inside one thread-block cluster ----------
            cg::cluster_group cl = cg::this_cluster();
            const int C = (int)cl.num_blocks();
            const int cid = blockIdx.x / C, ncl = G / C;
            ph_cur = T_LLOYD;
            for (int sl = cid; sl < nslots; sl += ncl)
                cl_split_cluster(A, ss[sl], ldi(&A.slots[sl].leaf), cur, cen0, cen1, red, ired, outv, tmpv, sbuf, tp,
                                 tsd, clx);
            ph_cur = T_LLOYD;
            trace_ev(A.trace, 33);
            gsync();
            trace_ev(A.trace, 34);
            continue;
        }

#ifndef HDF_NO_MODE_A
        // ---------------- farthest pair rows (R3) ----------------
        // Work items (slot, c): rows a = c, c + kFpItems, ... of the slot's stride sample, so every
        // item holds about the same number of pairs.  The block stages the slot's sample into the
        // shared tile (when it fits) and its warps take the item's rows.
        {
            constexpr int kFpItems = 16;
            const int nitems = nslots * kFpItems;
            int staged = -1;
            for (int item = blockIdx.x; item < nitems; item += G) {
                const int sl = item / kFpItems, c = item % kFpItems;
                const int start = ss[sl].start, stride = ss[sl].stride, s = ss[sl].s;
                const bool insm = (long long)s * rho <= A.tileF;
                if (insm && staged != sl) {
                    __syncthreads();
                    constexpr int U = 8;
                    for (int f0 = 0; f0 < s * rho; f0 += U * kClThreads) {
                        float v[U];
#pragma unroll
                        for (int u = 0; u < U; u++) {
                            const int f = f0 + u * kClThreads + tid;
                            const int a = f / rho, d = f - a * rho;
                            v[u] = (f < s * rho) ? __ldcg(P + (size_t)(start + (long long)a * stride) * rho + d) : 0.f;
                        }
#pragma unroll
                        for (int u = 0; u < U; u++) {
                            const int f = f0 + u * kClThreads + tid;
                            if (f < s * rho) tp[f] = v[u];
                        }
                    }
                    __syncthreads();
                    staged = sl;
                }
                for (int a = c + kFpItems * warp; a < s; a += kFpItems * kClWarps) {
                    double best;
                    int arg;
                    const float* tpc = tp;
                    if (insm)
                        row_farthest(a, s, rho, [&](int q) { return tpc + (size_t)q * rho; }, best, arg);
                    else
                        row_farthest(a, s, rho, [&](int q) { return P + (size_t)(start + (long long)q * stride) * rho; },
                                     best, arg);
                    if (lane == 0) {
                        A.fpd[(size_t)sl * kFpCap + a] = best;
                        A.fpi[(size_t)sl * kFpCap + a] = arg;
                    }
                }
            }
        }
        gsync();
        // argmax over rows (ties -> first row), one block per slot; centres from the pair
        for (int sl = blockIdx.x; sl < nslots; sl += G) {
            const int s = ss[sl].s;
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
            __shared__ int s_fab[2];
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
                s_fab[0] = fa;
                s_fab[1] = fb;
            }
            __syncthreads();
            {
                const int start = ss[sl].start, stride = ss[sl].stride;
                for (int e = tid; e < 2 * rho; e += blockDim.x) {
                    const int w = e / rho, d = e - w * rho;
                    const double v = (double)__ldcg(P + (size_t)(start + (long long)s_fab[w] * stride) * rho + d);
                    (w ? A.c1g : A.c0g)[sl * rho + d] = v;
                }
            }
            __syncthreads();
        }
        gsync();
        for (int e = tid; e < nslots * rho; e += blockDim.x) {
            cen0[e] = ldd(&A.c0g[e]);
            cen1[e] = ldd(&A.c1g[e]);
        }
        for (int sl = tid; sl < nslots; sl += blockDim.x) { s_conv[sl] = 0; s_rs[sl] = 0; s_fbuf[sl] = (kMaxIter - 1) & 1; }
        // the block's range stays resident in shared memory for the whole round when it fits
        const long long blo_q = blk_lo(T, blockIdx.x, G), bhi_q = blk_lo(T, blockIdx.x + 1, G);
        const bool resident = (bhi_q - blo_q) <= tile_pts(A.tileF, rho);
        __syncthreads();
        if (resident) stage_points(P, rho, nslots, ss, blo_q, bhi_q, tp);
        __syncthreads();
        tick(T_SEED);
        ph_cur = T_LLOYD;

        // ---------------- lock-step Lloyd iterations ----------------
        int it = 0;
        for (; it < kMaxIter; it++) {
            const int wb = it & 1;
            ph_cur = T_PASS;
            cl_pass(A, P, nslots, ss, T, cen0, cen1, s_conv, nullptr, it, wb, red, ired, outv, tp, tsd, resident);
            gsync();
            ph_cur = T_LLOYD;
            const int any = cl_finalize(A, nslots, ss, it, wb, cen0, cen1, s_conv, s_rs, s_fbuf, false, tmpv, sbuf, soff);
            tick(T_LLOYD);
            if (any) {
                // Rare path (R4): a side came out empty.  Move that side's centre to the member
                // farthest from the other centre (ties -> first), redo this iteration's assignment.
                cl_reseed(A, P, nslots, ss, cen0, cen1, s_rs, red);
                gsync();   // also: every block has finished reading records of parity wb
                for (int sl = 0; sl < nslots; sl++) {
                    if (!s_rs[sl]) continue;
                    for (int d = tid; d < rho; d += blockDim.x) {
                        if (s_rs[sl] == 1) cen1[sl * rho + d] = ldd(&A.c1g[sl * rho + d]);
                        else cen0[sl * rho + d] = ldd(&A.c0g[sl * rho + d]);
                    }
                }
                __syncthreads();
                cl_pass(A, P, nslots, ss, T, cen0, cen1, s_conv, s_rs, it, wb, red, ired, outv, tp, tsd, resident);
                gsync();
                cl_finalize(A, nslots, ss, it, wb, cen0, cen1, s_conv, s_rs, s_fbuf, true, tmpv, sbuf, soff);
            }
            bool all = true;
            for (int sl = 0; sl < nslots; sl++) all = all && s_conv[sl];
            if (all) break;
        }
        if (it == kMaxIter) it = kMaxIter - 1;
        tick(T_LLOYD);
        ph_cur = T_PART;

        // ---------------- stable partition + child SSE ----------------
        // (the sse fields of the final records are written below; other fields are only read)
        const int nxt = cur ^ 1;
        {
            const int b = blockIdx.x;
            const long long lo = blk_lo(T, b, G), hi = blk_lo(T, b + 1, G);
            for (int sl = 0; sl < nslots && lo < hi; sl++) {
                const SSlot S = ss[sl];
                if (S.pbeg + S.m <= lo || S.pbeg >= hi) continue;
                const int a = (int)(max(lo, S.pbeg) - S.pbeg), e = (int)(min(hi, S.pbeg + S.m) - S.pbeg);
                const int fb = s_fbuf[sl];
                const unsigned char* sd = A.side[fb];
                const double* recb = A.rec[fb];
                const int jme = b - S.blo;
                // n1 of every record of the slot: loaded in parallel, summed in order
                __syncthreads();
                for (int j = tid; j < S.nrec; j += kClThreads)
                    sbuf[j] = ldd(recb + (size_t)(S.rbase + j) * A.pstride + 2 * rho);
                __syncthreads();
                long long pre1 = 0, tot1 = 0;
                for (int j = 0; j < S.nrec; j++) {
                    const long long v = (long long)sbuf[j];
                    if (j < jme) pre1 += v;
                    tot1 += v;
                }
                const long long m0 = S.m - tot1;
                const long long pre0 = a - pre1;
                const double* c0 = cen0 + sl * rho;
                const double* c1 = cen1 + sl * rho;
                double acc[16];
#pragma unroll
                for (int j = 0; j < 16; j++) acc[j] = 0.0;
                long long run0 = 0, run1 = 0;
                for (int t0 = a; t0 < e; t0 += kClThreads) {
                    const int t = t0 + tid;
                    const bool ok = t < e;
                    const long long gi = (long long)S.start + t;
                    const int s = ok ? (int)__ldcg(sd + gi) : 0;
                    const int f0 = (ok && s == 0) ? 1 : 0;
                    // block exclusive scan of f0 (ballot per warp, warp totals scanned in shared memory)
                    const unsigned bal = __ballot_sync(0xffffffffu, f0);
                    if (lane == 0) ired[warp] = __popc(bal);
                    __syncthreads();
                    int wpre = 0, total0 = 0;
                    for (int w = 0; w < kClWarps; w++) {
                        const int v = ired[w];
                        if (w < warp) wpre += v;
                        total0 += v;
                    }
                    const int incl = wpre + __popc(bal & ((lane == 31) ? 0xffffffffu : ((1u << (lane + 1)) - 1u)));
                    __syncthreads();
                    if (ok) {
                        const int rank0 = incl - f0;
                        const int rank1 = (t - t0) - rank0;
                        long long dst;
                        if (s == 0) dst = S.start + pre0 + run0 + rank0;
                        else dst = S.start + m0 + pre1 + run1 + rank1;
                        const float* x = P + gi * rho;
                        double dd = 0.0;
                        const double* cc = s ? c1 : c0;
                        for (int d = 0; d < rho; d++) {
                            const float v = __ldcg(x + d);
                            A.pts[nxt][(size_t)dst * rho + d] = v;
                            dd = d2_rn(dd, (double)v, cc[d]);
                        }
                        A.idx[nxt][dst] = __ldcg(A.idx[cur] + gi);
                        if (s) acc[1] += dd;
                        else acc[0] += dd;
                    }
                    const int nvalid = min(kClThreads, e - t0);
                    run0 += total0;
                    run1 += nvalid - total0;
                }
                block_reduce16(acc, red, outv);
                if (tid == 0) {
                    double* rec = A.rec[fb] + (size_t)(S.rbase + jme) * A.pstride;
                    rec[2 * rho + 2] = outv[0];
                    rec[2 * rho + 3] = outv[1];
                }
            }
        }
        gsync();
        // copy the partitioned segments back (each block its own range), record the computed splits
        {
            const int b = blockIdx.x;
            const long long lo = blk_lo(T, b, G), hi = blk_lo(T, b + 1, G);
            for (int sl = 0; sl < nslots && lo < hi; sl++) {
                const SSlot S = ss[sl];
                if (S.pbeg + S.m <= lo || S.pbeg >= hi) continue;
                const long long a = max(lo, S.pbeg) - S.pbeg + S.start, e = min(hi, S.pbeg + S.m) - S.pbeg + S.start;
                for (long long q = a * rho + tid; q < e * rho; q += blockDim.x) A.pts[cur][q] = __ldcg(A.pts[nxt] + q);
                for (long long q = a + tid; q < e; q += blockDim.x) A.idx[cur][q] = __ldcg(A.idx[nxt] + q);
            }
        }
        for (int sl = blockIdx.x; sl < nslots; sl += G) {
            const SSlot S = ss[sl];
            if (warp == 0) {
                const double* recb = A.rec[s_fbuf[sl]];
                double v0 = 0.0, v1 = 0.0, v2 = 0.0;   // n1, sse0, sse1
                for (int j = lane; j < S.nrec; j += 32) {
                    const double* r = recb + (size_t)(S.rbase + j) * A.pstride;
                    v0 += ldd(r + 2 * rho);
                    v1 += ldd(r + 2 * rho + 2);
                    v2 += ldd(r + 2 * rho + 3);
                }
                v0 = warp_sum(v0);
                v1 = warp_sum(v1);
                v2 = warp_sum(v2);
                if (lane == 0) {
                    const int leaf = ldi(&A.slots[sl].leaf);
                    A.leaves[leaf].m0 = S.m - (int)v0;
                    A.leaves[leaf].csse0 = v1;
                    A.leaves[leaf].csse1 = v2;
                    for (int d = 0; d < rho; d++) {
                        A.cmean0[leaf * rho + d] = cen0[sl * rho + d];
                        A.cmean1[leaf * rho + d] = cen1[sl * rho + d];
                    }
                    __threadfence();
                    A.leaves[leaf].state = 1;
                }
            }
        }
        if (blockIdx.x == 0 && tid == 0) A.ctrl[C_ITERS] = ldi(&A.ctrl[C_ITERS]) + it + 1;
        gsync();
        tick(T_PART);
#endif
    }

    // ---------------- outputs ----------------
    const int L = ldi(&A.ctrl[C_NLEAVES]);
    for (long long e = gtid; e < (long long)K * rho; e += gthreads) {
        const int k = (int)(e / rho), d = (int)(e % rho);
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
        if (A.timers)
            for (int c = 0; c < T_NUM; c++) A.timers[c] = diag().timers[c];
    }
}

}  // namespace hdf
