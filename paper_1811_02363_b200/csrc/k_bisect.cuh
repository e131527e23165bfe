// k_bisect.cuh -- step 1: bisecting K-means of Theta = {p(i)}.
//
// The sequential procedure (oracle/hdf_oracle.c orc_cluster, readings R1-R5): start from one leaf
// holding every pixel; K-1 times split the leaf of largest SSE (R2) by 2-means seeded with the
// farthest pair of the stride sample members[0::ceil(m/1024)] (R3), Lloyd iterations until no
// assignment changes or 50 iterations, an empty side reseeded at the member farthest from the
// other centre (R4).  The parent id keeps child 0, child 1 gets id = #leaves.
//
// Parallel formulation used here (same result).  Call the binary tree of all splits the procedure
// could ever make the "potential tree".  A child's SSE never exceeds its parent's (each side's own
// mean beats the parent mean), so the tree is heap-ordered by SSE, and "repeatedly split the
// largest leaf" visits its nodes in globally descending SSE order: the K-1 split nodes are exactly
// the K-1 nodes of largest SSE in the potential tree, and the split order is descending SSE.
// The kernel therefore expands the potential tree best-first, in parallel:
//   * a node table holds every computed node (SSE, size, segment, mean, state);
//   * a worker claims the FREE node of largest SSE, provided fewer than K-1 known nodes have a
//     larger SSE (otherwise it can never be among the K-1 largest: unknown nodes are descendants of
//     FREE nodes and have smaller SSE); the node of largest SSE among FREE nodes is always decided
//     exactly, the others are speculative (a wasted speculative split changes nothing);
//   * when no node is claimable and none is in progress, the K-1 largest nodes are the split set.
//     Leaf ids are then replayed: the j-th split (descending SSE) gives child 1 id j+1, child 0
//     inherits the parent's id -- the sequential procedure's numbering.
// Workers:
//   * phase 1 (grid mode): while the best claimable node does not fit one thread-block cluster's
//     shared memory, the whole cooperative grid splits it (lock-step, grid barriers, points
//     streamed through shared-memory tiles);
//   * phase 2 (cluster mode): every thread-block cluster is a worker; a claimed node's members stay
//     resident in the cluster's shared memory (TMA bulk copies) for the whole split; partial sums
//     are exchanged through distributed shared memory, one cluster barrier per Lloyd iteration.
// Every split writes its children's members as a stable partition of the parent's segment into the
// other ping-pong buffer (children are sub-segments of the parent's segment).
// Exactness vs the fp64 oracle: nearer-centre decisions are taken in fp32 with a proven error
// bound and re-evaluated with the oracle's fp64 operation sequence inside the uncertainty band; the
// farthest pair likewise (fp32 row maximum, fp64 for the candidates near it); sums are fp64 in a
// fixed order.  GPU and oracle differ only in the summation order of the means and SSEs.
#pragma once
#include <cooperative_groups.h>

#include "hdf_common.cuh"

namespace hdf {
namespace cg = cooperative_groups;

constexpr int kBT = 512;            // threads per CTA
constexpr int kBW = kBT / 32;       // warps per CTA
constexpr int kFpCap = 1024;        // farthest-pair stride-sample cap (R3)
constexpr int kMaxIter = 50;        // Lloyd cap (R4)
constexpr int kRecV = 2 * HDF_MAX_RHO + 8;   // exchanged record length (doubles)
constexpr int kSampRho = 8;         // the stride sample is staged in shared memory for rho <= 8
constexpr int kBisectTraceCap = 8192;

// control words
enum {
    B_NALLOC = 0,  // node ids allocated
    B_INPROG,      // claimed splits not yet published
    B_VERSION,     // number of publications
    B_STATUS,      // HDF_OK / HDF_ERR_K / internal error
    B_ACH,         // leaves reached (achievable K)
    B_TASK,        // phase-1 task (node id or -1)
    B_TASKC,       // phase-1 task: first child id
    B_SPLITS,      // splits computed (including wasted speculative ones)
    B_ITERS,       // Lloyd passes executed (all splits)
    B_GRIDSPLITS,  // splits computed in grid mode
    B_TRACE_N,     // trace events recorded
    B_ABORT,       // node table overflow (never expected)
    B_NUM
};
enum { ST_FREE = 0, ST_CLAIMED = 1, ST_DONE = 2, ST_NONE = 3 };
constexpr int kBufInput = 2;        // node buffer 2 = the caller's p (root only), identity index

struct BisectArgs {
    const float* p;
    int N, rho, K, maxn;
    int cap;            // points per CTA tile (multiple of kBT)
    int wcap;           // side words per CTA in the global scratch (streamed ranges)
    long long ccap;     // points a cluster keeps resident (C * cap)
    const float* pts[3];   // ping-pong leaf storage; pts[2] = p
    float* ptsw[2];
    int* idx[2];
    uint32_t* sidew;    // [grid][2][wcap] side words of streamed ranges
    double* rec;        // [2][grid][kRecV] grid-mode exchange records
    // node table (struct of arrays, coalesced warp scans)
    double* nsse;
    int* nm;
    int* nstart;
    int* nstate;
    int* nparent;
    int* nchild;
    int* nbuf;
    double* nmean;      // [maxn][rho]
    int* nfinal;        // [maxn] leaf id of the final leaf containing the node (labels)
    int* node_of;       // [N] deepest computed node of each pixel (labels only)
    int* ctl;           // [B_NUM]
    long long* trace;   // [1 + 2 * kBisectTraceCap] (tag|node|worker, globaltimer), or null
    float* centres;     // [K][rho] out
    int* labels;        // [N] out, or null
    double* ek;         // out
};

// --------------------------------------------------------------------------- memory helpers ---
HDF_DEV int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
HDF_DEV void st_rel(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
HDF_DEV long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
HDF_DEV float lds_f(const float* p) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}
HDF_DEV uint32_t lds_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)));
    return v;
}
// 1-D bulk copy global -> shared (TMA), completion on `bar`.  16-byte aligned, size % 16 == 0.
HDF_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

HDF_DEV void trace_ev(const BisectArgs& A, int tag, int node, int worker) {
    if (A.trace == nullptr) return;
    const int s = atomicAdd(&A.ctl[B_TRACE_N], 1);
    if (s < kBisectTraceCap) {
        A.trace[1 + 2 * s] = (long long)tag | ((long long)(node & 0xFFFFF) << 8) | ((long long)worker << 28);
        A.trace[2 + 2 * s] = gtimer();
    }
}

// Exactly rounded fp64 squared distance of fp32 x to fp64 c in dimension order, no contraction:
// the oracle's dist2 (oracle/hdf_oracle.c) operation for operation.
HDF_DEV double dist_rn(const float* x, const double* c, int rho) {
    double s = 0.0;
    for (int d = 0; d < rho; d++) s = d2_rn(s, (double)x[d], c[d]);
    return s;
}

HDF_DEV bool cand_better(double v, long long a, double bv, long long ba) {
    return a >= 0 && (ba < 0 || v > bv || (v == bv && a < ba));
}

// Warp reduce-scatter of 16 doubles in a fixed butterfly order (deterministic).  Afterwards the even
// lane l holds the warp total of the returned value index.
HDF_DEV int warp_reduce_scatter16(double (&v)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int step = 0; step < 4; step++) {
        const int o = 16 >> step;
        const int half = 8 >> step;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; j++) {
            const double send = upper ? v[j] : v[j + half];
            const double keep = upper ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// Block-wide exclusive scan of one int per thread; returns the prefix, *total = block sum.
HDF_DEV int block_exscan(int x, int* wsum, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kBW; w++) {
        const int v = wsum[w];
        pre += (w < warp) ? v : 0;
        tot += v;
    }
    __syncthreads();
    *total = tot;
    return pre + inc - x;
}

// ------------------------------------------------------------------------------ shared state ---
struct SplitSm {
    double c0[HDF_MAX_RHO], c1[HDF_MAX_RHO];   // centres (fp64, the oracle's values)
    float f0[HDF_MAX_RHO], f1[HDF_MAX_RHO];    // fp32-rounded centres
    double tot[kRecV];                          // gathered totals
    double rx[2][kRecV];                        // posted record (cluster mode, read over DSMEM)
    double red[kBW * 16];
    double wv[kBW];
    long long wa[kBW], wb[kBW];
    int wsum[kBW];
    int wp[kBT];                                // word prefix of a tile
    int iv[8];
    long long lv[4];
    uint64_t bar;                               // TMA mbarrier
    uint32_t tma_phase;
    int task, cbase;
};

// -------------------------------------------------------------------------------- groups ------
// A split runs on a group of CTAs: one thread-block cluster (records over DSMEM, cluster barrier)
// or the whole cooperative grid (records in global memory, grid barrier).
struct ClusterGrp {
    int rank, size;
    HDF_DEV void sync() const { cg::this_cluster().sync(); }
    HDF_DEV double* post(SplitSm& S, int par) const { return S.rx[par]; }
    HDF_DEV double peer(SplitSm& S, int par, int q, int v) const {
        const double* p = cg::this_cluster().map_shared_rank(&S.rx[par][0], q);
        return p[v];
    }
    static constexpr bool kGrid = false;
};
struct GridGrp {
    int rank, size;
    double* rec;
    HDF_DEV void sync() const { cg::this_grid().sync(); }
    HDF_DEV double* post(SplitSm&, int par) const { return rec + ((size_t)par * size + rank) * kRecV; }
    HDF_DEV double peer(SplitSm&, int par, int q, int v) const {
        return __ldcg(rec + ((size_t)par * size + q) * kRecV + v);
    }
    static constexpr bool kGrid = true;
};

// Sum record value v over the group's CTAs in rank order.
template <class Grp>
HDF_DEV double gather_sum(const Grp& g, SplitSm& S, int par, int v) {
    double s = 0.0;
    for (int q = 0; q < g.size; q++) s += g.peer(S, par, q, v);
    return s;
}

// ------------------------------------------------------------------------------- tile loads ---
// Load `tn` points (rho floats each) starting at global `src` into the shared tile `dyn`: the 16-byte
// aligned body with TMA bulk copies (completion on S.bar), the < 16-byte tail with plain loads (never
// reads past the end).  tile_issue returns the tile pointer (dyn offset by the source's
// misalignment); tile_wait must follow before the tile is read.
struct TileLd {
    const float* ptr;
    uint32_t body;
};
HDF_DEV TileLd tile_issue(const float* src, int tn, int rho, float* dyn, SplitSm& S) {
    const uintptr_t s = reinterpret_cast<uintptr_t>(src);
    const int delta = (int)((s & 15u) >> 2);
    const uintptr_t s0 = s - 4u * (uintptr_t)delta;
    const uintptr_t end = s + 4u * (uintptr_t)tn * (uintptr_t)rho;
    const uintptr_t body_end = end & ~(uintptr_t)15;
    const uint32_t body = body_end > s0 ? (uint32_t)(body_end - s0) : 0u;
    __syncthreads();   // the previous tile is fully consumed
    if (threadIdx.x == 0 && body > 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&S.bar, body);
        for (uint32_t off = 0; off < body; off += 32768u)
            bulk_g2s(reinterpret_cast<char*>(dyn) + off, reinterpret_cast<const char*>(s0) + off,
                     min(32768u, body - off), &S.bar);
    }
    const uintptr_t tb = body > 0 ? body_end : s0;   // tail floats [tb, end)
    const int tail = (int)((end - tb) >> 2);
    if (threadIdx.x < tail) {
        const float* tp = reinterpret_cast<const float*>(tb) + threadIdx.x;
        if (reinterpret_cast<uintptr_t>(tp) >= s) dyn[(tb - s0) / 4 + threadIdx.x] = __ldcg(tp);
    }
    return {dyn + delta, body};
}
HDF_DEV void tile_wait(SplitSm& S, const TileLd& t) {
    if (t.body > 0) mbar_wait(&S.bar, S.tma_phase);
    __syncthreads();
    if (threadIdx.x == 0 && t.body > 0) S.tma_phase ^= 1u;
    __syncthreads();
}
HDF_DEV const float* load_tile(const float* src, int tn, int rho, float* dyn, SplitSm& S) {
    const TileLd t = tile_issue(src, tn, rho, dyn, S);
    tile_wait(S, t);
    return t.ptr;
}

// ------------------------------------------------------------------------- farthest pair ------
// Farthest partner of sample row a (warp-cooperative, R3): the exact fp64 maximum of
// ||x_a - x_b||^2 over b > a, ties -> lowest b.  Pass 1 finds the row's fp32 maximum M
// (|d32 - d| <= (rho + 3) u d for fp32 inputs, u = 2^-24); pass 2 re-evaluates with the oracle's
// fp64 sequence only the pairs with d32 >= M (1 - 8 (rho + 3) u), which contain every pair whose
// fp64 value can be the row maximum.
template <int RHO, class Base>
HDF_DEV float pair_d32(const float* xa, const float* xb, int rho) {
    float acc = 0.f;
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < (RHO > 0 ? RHO : 1); d++) {
            const float t = xa[d] - xb[d];
            acc = fmaf(t, t, acc);
        }
    } else {
        for (int d = 0; d < rho; d++) {
            const float t = xa[d] - xb[d];
            acc = fmaf(t, t, acc);
        }
    }
    return acc;
}

template <int RHO, class Base>
HDF_DEV void row_farthest(int a, int sN, int rho, Base base, double& best, int& arg) {
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
    float mx = 0.f;
    int q = a + 1 + lane;
    for (; q + 32 < sN; q += 64) {
        const float d1 = pair_d32<RHO, Base>(xav, base(q), rho);
        const float d2 = pair_d32<RHO, Base>(xav, base(q + 32), rho);
        mx = fmaxf(mx, fmaxf(d1, d2));
    }
    if (q < sN) mx = fmaxf(mx, pair_d32<RHO, Base>(xav, base(q), rho));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float thr = mx * (1.0f - 8.0f * (float)(rho + 3) * u);
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

// ------------------------------------------------------------------------------- the pass -----
// Nearer-centre decision, certified.  The oracle decides d64(x, c0) <= d64(x, c1) in fp64 (R4).
// Here the distances are first evaluated in fp32 against fp32-rounded centres f0, f1 (u = 2^-24):
//   t^ = fl(x - fl(c)),  d32 = FMA-accumulated sum of t^2,
//   |t^2 - t^2_exact| <= 3u (|t| + |c|)^2,   accumulation error <= rho u d32,
//   => |d32 - d| <= u ((rho + 7) d32 + 6.1 ||c||^2),
// and the fp64 evaluation error is ~2^-29 of that.  If |d32_0 - d32_1| exceeds the sum of the two
// bounds the fp64 decision is the same; otherwise the distances are re-evaluated in fp64 with the
// oracle's operation sequence.
HDF_DEV int side_of(const float* x, int rho, float a0, float a1, float kd, float kc, const SplitSm& S) {
    const float diff = a0 - a1;
    const float bound = kd * (a0 + a1) + kc;
    if (fabsf(diff) > bound) return diff > 0.f ? 1 : 0;
    double dd0 = 0.0, dd1 = 0.0;
    for (int d = 0; d < rho; d++) {
        const double v = (double)x[d];
        dd0 = d2_rn(dd0, v, S.c0[d]);
        dd1 = d2_rn(dd1, v, S.c1[d]);
    }
    return (dd0 <= dd1) ? 0 : 1;
}

HDF_DEV void cert_consts(const SplitSm& S, int rho, float& kd, float& kc) {
    constexpr float u = 5.9604644775390625e-08f;   // 2^-24
    float n0 = 0.f, n1 = 0.f;
    for (int d = 0; d < rho; d++) {
        n0 = fmaf(S.f0[d], S.f0[d], n0);
        n1 = fmaf(S.f1[d], S.f1[d], n1);
    }
    kd = 2.0f * u * (float)(rho + 7);
    kc = 2.0f * u * 6.1f * (n0 + n1);
}

// Small rho (compile-time): thread per point, fp64 per-side sums in registers.  Tile points
// j = j0 + tid; word j/32 of the tile holds the sides of 32 consecutive points (bit = lane).
template <int RHO>
HDF_DEV void pass_small(const float* X, int tn, const uint32_t* prevW, uint32_t* curW, bool cmp, const SplitSm& S,
                        double (&s)[2 * RHO], int& n1, int& chg) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float f0[RHO], f1[RHO];
#pragma unroll
    for (int d = 0; d < RHO; d++) { f0[d] = S.f0[d]; f1[d] = S.f1[d]; }
    float kd, kc;
    cert_consts(S, RHO, kd, kc);
#pragma unroll 2
    for (int j0 = 0; j0 < tn; j0 += kBT) {
        const int j = j0 + tid;
        const bool ok = j < tn;
        float x[RHO];
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int d = 0; d < RHO; d++) {
            x[d] = ok ? lds_f(X + (size_t)j * RHO + d) : 0.f;
            const float e0 = x[d] - f0[d], e1 = x[d] - f1[d];
            a0 = fmaf(e0, e0, a0);
            a1 = fmaf(e1, e1, a1);
        }
        const int sd = ok ? side_of(x, RHO, a0, a1, kd, kc, S) : 0;
        const uint32_t w = __ballot_sync(0xffffffffu, sd != 0);
        if (lane == 0) {
            const int wi = (j0 >> 5) + warp;
            if (cmp) chg += __popc(w ^ prevW[wi]);
            curW[wi] = w;
        }
        n1 += sd;
#pragma unroll
        for (int d = 0; d < RHO; d++) {
            const double xd = (double)x[d];
            s[d] += sd ? 0.0 : xd;
            s[RHO + d] += sd ? xd : 0.0;
        }
    }
}

// Generic rho: side phase (thread per point) ...
HDF_DEV void pass_side_generic(const float* X, int tn, int rho, const uint32_t* prevW, uint32_t* curW, bool cmp,
                               const SplitSm& S, int& n1, int& chg) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float kd, kc;
    cert_consts(S, rho, kd, kc);
    for (int j0 = 0; j0 < tn; j0 += kBT) {
        const int j = j0 + tid;
        const bool ok = j < tn;
        int sd = 0;
        if (ok) {
            const float* x = X + (size_t)j * rho;
            float a0 = 0.f, a1 = 0.f;
            for (int d = 0; d < rho; d++) {
                const float v = lds_f(x + d);
                const float e0 = v - S.f0[d], e1 = v - S.f1[d];
                a0 = fmaf(e0, e0, a0);
                a1 = fmaf(e1, e1, a1);
            }
            sd = side_of(x, rho, a0, a1, kd, kc, S);
        }
        const uint32_t w = __ballot_sync(0xffffffffu, sd != 0);
        if (lane == 0) {
            const int wi = (j0 >> 5) + warp;
            if (cmp) chg += __popc(w ^ prevW[wi]);
            curW[wi] = w;
        }
        n1 += sd;
    }
}
// ... then dimension-parallel sums: warp w owns dimensions w, w + 16, ... (<= 4 of them), lanes
// stride over the tile's points (consecutive points per lane group, odd rho: conflict free).
constexpr int kGenDims = (HDF_MAX_RHO + kBW - 1) / kBW;
HDF_DEV void pass_sum_generic(const float* X, int tn, int rho, const uint32_t* curW, double (&a0)[kGenDims],
                              double (&a1)[kGenDims]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const uint32_t w = curW[j0 >> 5];
        const int j = j0 + lane;
        const bool ok = j < tn;
        const bool sd = (w >> lane) & 1u;
#pragma unroll
        for (int q = 0; q < kGenDims; q++) {
            const int d = warp + kBW * q;
            if (d < rho && ok) {
                const double v = (double)lds_f(X + (size_t)j * rho + d);
                a0[q] += sd ? 0.0 : v;
                a1[q] += sd ? v : 0.0;
            }
        }
    }
}

// ------------------------------------------------------------------------------- the split ----
struct SplitIO {
    float* dynX;        // tile area (cap * rho + 8 floats)
    uint32_t* dynW;     // resident side words [2][cap / 32 + 2]
    float* dynS;        // stride sample (rho <= kSampRho), else null
};

template <int RHO, class Grp>
HDF_DEV void split_node(const BisectArgs& A, const Grp& g, SplitSm& S, const SplitIO& io, int v, int cbase,
                        int worker) {
    const int rho = RHO > 0 ? RHO : A.rho;
    const int nv = 2 * rho + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = g.rank, C = g.size;
    const int m = __ldcg(&A.nm[v]), start = __ldcg(&A.nstart[v]), buf = __ldcg(&A.nbuf[v]);
    const int nbuf = (buf == kBufInput) ? 0 : (buf ^ 1);
    const int a = (int)((long long)m * r / C), e = (int)((long long)m * (r + 1) / C), np = e - a;
    const float* Pg = A.pts[buf] + (size_t)start * rho;   // the node's points
    const bool resident = (m + C - 1) / C <= A.cap;   // uniform over the group (np <= ceil(m / C))
    // Phase 1 splits every claimable node larger than a cluster's resident capacity, so a cluster
    // worker never streams (its range always fits); guard the invariant.
    if (!Grp::kGrid && !resident) {
        if (tid == 0) atomicExch(&A.ctl[B_ABORT], 1);
        return;
    }
    const int wsm = A.cap / 32 + 2;
    uint32_t* W0;
    uint32_t* W1;
    if (resident) {
        W0 = io.dynW;
        W1 = io.dynW + wsm;
    } else {
        W0 = A.sidew + (size_t)blockIdx.x * 2 * A.wcap;
        W1 = W0 + A.wcap;
    }
    const bool lead = (r == 0 && tid == 0);
    if (lead) trace_ev(A, 2, v, worker);
    int par = 0;

    // ---- 1. the CTA's members: resident tile, TMA issued now, awaited after the seed exchange ----
    TileLd rt{nullptr, 0u};
    if (resident) rt = tile_issue(Pg + (size_t)a * rho, np, rho, io.dynX, S);
    // ---- 2. farthest pair of the stride sample members[0::stride] (R3) ----
    const int stride = (m + kFpCap - 1) / kFpCap, sN = (m + stride - 1) / stride;
    const bool insm = io.dynS != nullptr;
    if (insm) {
        constexpr int U = 8;
        for (int f0 = 0; f0 < sN * rho; f0 += U * kBT) {
            float vv[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = f0 + u * kBT + tid;
                const int q = f / rho, d = f - q * rho;
                vv[u] = (f < sN * rho) ? __ldcg(Pg + (size_t)q * stride * rho + d) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int f = f0 + u * kBT + tid;
                if (f < sN * rho) io.dynS[f] = vv[u];
            }
        }
        __syncthreads();
    }
    {
        double bv = -1.0;
        long long ba = -1, bb = -1;
        for (int ra = r + C * warp; ra < sN; ra += C * kBW) {   // rows ascend within the warp
            double best;
            int arg;
            if (insm) {
                const float* sp = io.dynS;
                row_farthest<RHO>(ra, sN, rho, [&](int q) { return sp + (size_t)q * rho; }, best, arg);
            } else {
                row_farthest<RHO>(ra, sN, rho, [&](int q) { return Pg + (size_t)q * stride * rho; }, best, arg);
            }
            if (arg >= 0 && (ba < 0 || best > bv)) { bv = best; ba = ra; bb = arg; }
        }
        if (lane == 0) { S.wv[warp] = bv; S.wa[warp] = ba; S.wb[warp] = bb; }
        __syncthreads();
        if (tid == 0) {
            double bvv = -1.0;
            long long ia = -1, ib = -1;
            for (int w = 0; w < kBW; w++)
                if (cand_better(S.wv[w], S.wa[w], bvv, ia)) { bvv = S.wv[w]; ia = S.wa[w]; ib = S.wb[w]; }
            double* rp = g.post(S, par);
            rp[0] = bvv;
            rp[1] = (double)ia;
            rp[2] = (double)ib;
        }
    }
    if (Grp::kGrid) __threadfence();
    g.sync();
    if (tid == 0) {
        double bvv = -1.0;
        long long ia = -1, ib = -1;
        for (int q = 0; q < C; q++) {
            const double qv = g.peer(S, par, q, 0);
            const long long qa = (long long)g.peer(S, par, q, 1), qb = (long long)g.peer(S, par, q, 2);
            if (cand_better(qv, qa, bvv, ia)) { bvv = qv; ia = qa; ib = qb; }
        }
        if (ia < 0) { ia = 0; ib = (sN > 1) ? 1 : 0; }
        S.lv[0] = ia;
        S.lv[1] = ib;
    }
    par ^= 1;
    __syncthreads();
    for (int f = tid; f < 2 * rho; f += kBT) {
        const int w = f / rho, d = f - w * rho;
        const long long q = S.lv[w];
        const float x = insm ? io.dynS[q * rho + d] : __ldcg(Pg + (size_t)q * stride * rho + d);
        (w ? S.c1 : S.c0)[d] = (double)x;
        (w ? S.f1 : S.f0)[d] = x;
    }
    const float* X = rt.ptr;
    if (resident) tile_wait(S, rt);
    __syncthreads();
    if (lead) trace_ev(A, 3, v, worker);

    // ---- 3. Lloyd iterations (R4) ----
    int it = 0, fbw = 0;
    bool conv = false;
    for (; it < kMaxIter; it++) {
        uint32_t* curW = (it & 1) ? W1 : W0;
        const uint32_t* prevW = (it & 1) ? W0 : W1;
        bool redo = false;
        long long n1tot = 0, chgtot = 0;
        while (true) {
            int n1 = 0, chg = 0;
            double* rp = g.post(S, par);
            if (RHO > 0) {
                double s[2 * (RHO > 0 ? RHO : 1)];
#pragma unroll
                for (int q = 0; q < 2 * (RHO > 0 ? RHO : 1); q++) s[q] = 0.0;
                for (int t0 = 0; t0 < np; t0 += A.cap) {
                    const int tn = min(A.cap, np - t0);
                    const float* T = resident ? X : load_tile(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                    pass_small<(RHO > 0 ? RHO : 1)>(T, tn, prevW + (t0 >> 5), curW + (t0 >> 5), it > 0, S, s, n1, chg);
                }
                double vv[16];
#pragma unroll
                for (int q = 0; q < 16; q++) vv[q] = 0.0;
#pragma unroll
                for (int q = 0; q < 2 * (RHO > 0 ? RHO : 1); q++) vv[q] = s[q];
                vv[2 * rho] = (double)n1;
                vv[2 * rho + 1] = (double)chg;
                const int vi = warp_reduce_scatter16(vv);
                if ((lane & 1) == 0) S.red[warp * 16 + vi] = vv[0];
                __syncthreads();
                if (tid < nv) {
                    double acc = 0.0;
                    for (int w = 0; w < kBW; w++) acc += S.red[w * 16 + tid];
                    rp[tid] = acc;
                }
            } else {
                double s0[kGenDims], s1[kGenDims];
#pragma unroll
                for (int q = 0; q < kGenDims; q++) { s0[q] = 0.0; s1[q] = 0.0; }
                for (int t0 = 0; t0 < np; t0 += A.cap) {
                    const int tn = min(A.cap, np - t0);
                    const float* T = resident ? X : load_tile(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                    pass_side_generic(T, tn, rho, prevW + (t0 >> 5), curW + (t0 >> 5), it > 0, S, n1, chg);
                    __syncthreads();
                    pass_sum_generic(T, tn, rho, curW + (t0 >> 5), s0, s1);
                }
#pragma unroll
                for (int q = 0; q < kGenDims; q++) {
                    const int d = warp + kBW * q;
                    const double x0 = warp_sum(s0[q]), x1 = warp_sum(s1[q]);
                    if (lane == 0 && d < rho) { rp[d] = x0; rp[rho + d] = x1; }
                }
                n1 = __reduce_add_sync(0xffffffffu, n1);
                chg = __reduce_add_sync(0xffffffffu, chg);
                if (lane == 0) { S.red[warp * 2] = (double)n1; S.red[warp * 2 + 1] = (double)chg; }
                __syncthreads();
                if (tid < 2) {
                    double acc = 0.0;
                    for (int w = 0; w < kBW; w++) acc += S.red[w * 2 + tid];
                    rp[2 * rho + tid] = acc;
                }
            }
            if (Grp::kGrid) __threadfence();
            g.sync();
            // every CTA sums the records in rank order: bit-identical totals in the group
            if (tid < nv) S.tot[tid] = gather_sum(g, S, par, tid);
            par ^= 1;
            __syncthreads();
            n1tot = (long long)S.tot[2 * rho];
            chgtot = (long long)S.tot[2 * rho + 1];
            if (redo || !(n1tot == 0 || n1tot == m)) break;
            // Empty side: move its centre to the member farthest from the other centre (ties -> first
            // in member order), then redo this iteration's assignment (R4).
            const bool side1_empty = (n1tot == 0);
            const double* cref = side1_empty ? S.c0 : S.c1;
            double best = -1.0;
            long long arg = -1;
            for (int t0 = 0; t0 < np; t0 += A.cap) {
                const int tn = min(A.cap, np - t0);
                const float* T = resident ? X : load_tile(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                for (int j = tid; j < tn; j += kBT) {
                    const double dd = dist_rn(T + (size_t)j * rho, cref, rho);
                    if (dd > best) { best = dd; arg = a + t0 + j; }
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const long long oa = __shfl_xor_sync(0xffffffffu, arg, o);
                if (cand_better(ob, oa, best, arg)) { best = ob; arg = oa; }
            }
            if (lane == 0) { S.wv[warp] = best; S.wa[warp] = arg; }
            __syncthreads();
            if (tid == 0) {
                double bvv = -1.0;
                long long ia = -1;
                for (int w = 0; w < kBW; w++)
                    if (cand_better(S.wv[w], S.wa[w], bvv, ia)) { bvv = S.wv[w]; ia = S.wa[w]; }
                double* rq = g.post(S, par);
                rq[0] = bvv;
                rq[1] = (double)ia;
            }
            if (Grp::kGrid) __threadfence();
            g.sync();
            if (tid == 0) {
                double bvv = -1.0;
                long long ia = -1;
                for (int q = 0; q < C; q++) {
                    const double qv = g.peer(S, par, q, 0);
                    const long long qa = (long long)g.peer(S, par, q, 1);
                    if (cand_better(qv, qa, bvv, ia)) { bvv = qv; ia = qa; }
                }
                S.lv[2] = ia < 0 ? 0 : ia;
            }
            par ^= 1;
            __syncthreads();
            for (int d = tid; d < rho; d += kBT) {
                const float x = __ldcg(Pg + (size_t)S.lv[2] * rho + d);
                if (side1_empty) { S.c1[d] = (double)x; S.f1[d] = x; }
                else { S.c0[d] = (double)x; S.f0[d] = x; }
            }
            __syncthreads();
            redo = true;
        }
        fbw = it & 1;
        if (it > 0 && chgtot == 0) { conv = true; break; }   // the final partition is this pass's
        for (int d = tid; d < rho; d += kBT) {
            const double c0 = S.tot[d] / (double)(m - n1tot), c1 = S.tot[rho + d] / (double)n1tot;
            S.c0[d] = c0;
            S.c1[d] = c1;
            S.f0[d] = (float)c0;
            S.f1[d] = (float)c1;
        }
        __syncthreads();
    }
    if (!conv) it = kMaxIter - 1;
    if (lead) trace_ev(A, 4, v, worker);
    const uint32_t* FW = fbw ? W1 : W0;

    // ---- 4. child SSE (w.r.t. the child means = current centres) and side-0 counts ----
    {
        double se0 = 0.0, se1 = 0.0;
        int cnt0 = 0;
        for (int t0 = 0; t0 < np; t0 += A.cap) {
            const int tn = min(A.cap, np - t0);
            const float* T = resident ? X : load_tile(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
            for (int j0 = 0; j0 < tn; j0 += kBT) {
                const int j = j0 + tid;
                const uint32_t w = FW[((t0 + j0) >> 5) + warp];
                if (j < tn) {
                    const int sd = (w >> lane) & 1u;
                    const double dd = dist_rn(T + (size_t)j * rho, sd ? S.c1 : S.c0, rho);
                    if (sd) se1 += dd;
                    else { se0 += dd; cnt0++; }
                }
            }
        }
        double vv[16];
#pragma unroll
        for (int q = 0; q < 16; q++) vv[q] = 0.0;
        vv[0] = (double)cnt0;
        vv[1] = se0;
        vv[2] = se1;
        const int vi = warp_reduce_scatter16(vv);
        if ((lane & 1) == 0) S.red[warp * 16 + vi] = vv[0];
        __syncthreads();
        double* rp = g.post(S, par);
        if (tid < 3) {
            double acc = 0.0;
            for (int w = 0; w < kBW; w++) acc += S.red[w * 16 + tid];
            rp[tid] = acc;
        }
        if (Grp::kGrid) __threadfence();
        g.sync();
        if (tid < 4) {
            double acc = 0.0, pre = 0.0;
            for (int q = 0; q < C; q++) {
                const double x = g.peer(S, par, q, tid < 3 ? tid : 0);
                if (q < r) pre += x;
                acc += x;
            }
            S.tot[tid] = (tid == 3) ? pre : acc;   // tot[0] = m0, tot[1] = sse0, tot[2] = sse1, tot[3] = pre0
        }
        par ^= 1;
        __syncthreads();
    }
    const int m0 = (int)S.tot[0];
    const int pre0 = (int)S.tot[3], pre1 = a - pre0;

    // ---- 5. stable partition into the other buffer: children are [start, start+m0), [start+m0, start+m) ----
    {
        float* Po = A.ptsw[nbuf] + (size_t)start * rho;
        int* Io = A.idx[nbuf] + start;
        const int* Ii = (buf == kBufInput) ? nullptr : A.idx[buf] + start;
        int run0 = 0;
        for (int t0 = 0; t0 < np; t0 += A.cap) {
            const int tn = min(A.cap, np - t0);
            const float* T = resident ? X : load_tile(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
            const int nw = (tn + 31) >> 5;
            for (int w0 = 0; w0 < nw; w0 += kBT) {
                // word prefix of side-0 counts for words [w0, w0 + kBT) of the tile
                const int wi = w0 + tid;
                int z = 0;
                if (wi < nw) {
                    const int nb = min(32, tn - wi * 32);
                    const uint32_t valid = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
                    z = __popc(~FW[(t0 >> 5) + wi] & valid);
                }
                int ztot;
                const int zp = block_exscan(z, S.wsum, &ztot);
                S.wp[tid] = zp;
                __syncthreads();
                const int jlo = w0 * 32, jhi = min(tn, (w0 + kBT) * 32);
                for (int j0 = jlo; j0 < jhi; j0 += kBT) {
                    const int j = j0 + tid;
                    const int wl = ((j0 - jlo) >> 5) + warp;
                    const uint32_t w = FW[((t0 + j0) >> 5) + warp];
                    if (j < jhi) {
                        const int sd = (w >> lane) & 1u;
                        const int zb = S.wp[wl] + __popc(~w & ((1u << lane) - 1u));   // side-0 before j in the chunk
                        const int jj = t0 + j;                                       // CTA-relative index
                        const int z0 = run0 + zb;                                    // side-0 before jj
                        const int dst = sd ? (m0 + pre1 + (jj - z0)) : (pre0 + z0);
                        const float* x = T + (size_t)j * rho;
                        float* o = Po + (size_t)dst * rho;
                        for (int d = 0; d < rho; d++) o[d] = lds_f(x + d);
                        const int pix = Ii ? __ldcg(Ii + a + jj) : (start + a + jj);
                        Io[dst] = pix;
                        if (A.labels) A.node_of[pix] = cbase + sd;
                    }
                }
                run0 += ztot;
                __syncthreads();
            }
        }
    }
    __threadfence();
    g.sync();   // the whole group's scatter is complete and visible
    // ---- 6. publish the children ----
    if (lead) {
        const int c = cbase;
        A.nsse[c] = S.tot[1];
        A.nsse[c + 1] = S.tot[2];
        A.nm[c] = m0;
        A.nm[c + 1] = m - m0;
        A.nstart[c] = start;
        A.nstart[c + 1] = start + m0;
        A.nbuf[c] = nbuf;
        A.nbuf[c + 1] = nbuf;
        A.nparent[c] = v;
        A.nparent[c + 1] = v;
        A.nchild[c] = -1;
        A.nchild[c + 1] = -1;
        for (int d = 0; d < rho; d++) {
            A.nmean[(size_t)c * rho + d] = S.c0[d];
            A.nmean[(size_t)(c + 1) * rho + d] = S.c1[d];
        }
        A.nchild[v] = c;
        __threadfence();
        st_rel(&A.nstate[c], ST_FREE);
        st_rel(&A.nstate[c + 1], ST_FREE);
        st_rel(&A.nstate[v], ST_DONE);
        __threadfence();
        atomicAdd(&A.ctl[B_SPLITS], 1);
        atomicAdd(&A.ctl[B_ITERS], it + 1);
        if (Grp::kGrid) atomicAdd(&A.ctl[B_GRIDSPLITS], 1);
        atomicAdd(&A.ctl[B_VERSION], 1);
        atomicAdd(&A.ctl[B_INPROG], -1);
        trace_ev(A, 5, v, worker);
    }
}

// ------------------------------------------------------------------------------- the claim ----
// Warp-cooperative.  Chooses the FREE node of largest SSE (ties -> lowest id) with SSE > 0 and >= 2
// members, and claims it if fewer than K-1 published nodes precede it in (SSE desc, id asc) order.
// mode 1 (grid phase): only a node larger than `bigcap` points is claimed, else -1 is returned.
// mode 2 (cluster phase): when nothing is claimable, waits until a publication changes the table;
// returns -1 once nothing is claimable and no split is in progress.
struct Claim {
    int task, cbase;
};
HDF_DEV Claim claim_node(const BisectArgs& A, int mode, long long bigcap) {
    const int lane = threadIdx.x & 31;
    int backoff = 32;
    while (true) {
        if (ld_acq(&A.ctl[B_ABORT])) return {-1, 0};
        int ver0 = 0, n = 0;
        if (lane == 0) {
            ver0 = ld_acq(&A.ctl[B_VERSION]);
            n = ld_acq(&A.ctl[B_NALLOC]);
        }
        ver0 = __shfl_sync(0xffffffffu, ver0, 0);
        n = min(__shfl_sync(0xffffffffu, n, 0), A.maxn);
        double bs = -1.0;
        int bi = -1;
        const long long mmin = (mode == 1) ? bigcap + 1 : 2;   // phase 1: only nodes too big for a cluster
        for (int i = lane; i < n; i += 32) {
            if (ld_acq(&A.nstate[i]) == ST_FREE) {
                const double s = __ldcg(&A.nsse[i]);
                if (s > 0.0 && __ldcg(&A.nm[i]) >= mmin && (bi < 0 || s > bs)) { bs = s; bi = i; }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, bs, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || ob > bs || (ob == bs && oi < bi))) { bs = ob; bi = oi; }
        }
        if (bi >= 0) {
            int cnt = 0;
            for (int i = lane; i < n; i += 32) {
                if (ld_acq(&A.nstate[i]) != ST_NONE) {
                    const double s = __ldcg(&A.nsse[i]);
                    cnt += (s > bs || (s == bs && i < bi)) ? 1 : 0;
                }
            }
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (cnt < A.K - 1) {
                int got = 0, cb = 0;
                if (lane == 0) {
                    atomicAdd(&A.ctl[B_INPROG], 1);
                    if (atomicCAS(&A.nstate[bi], ST_FREE, ST_CLAIMED) == ST_FREE) {
                        cb = atomicAdd(&A.ctl[B_NALLOC], 2);
                        got = 1;
                        if (cb + 2 > A.maxn) {
                            atomicExch(&A.ctl[B_ABORT], 1);
                            got = 0;
                        }
                    } else {
                        atomicAdd(&A.ctl[B_INPROG], -1);
                    }
                }
                got = __shfl_sync(0xffffffffu, got, 0);
                cb = __shfl_sync(0xffffffffu, cb, 0);
                if (got) return {bi, cb};
                continue;
            }
        }
        if (mode == 1) return {-1, 0};
        int done = 0;
        if (lane == 0) {
            const int ip = ld_acq(&A.ctl[B_INPROG]);
            const int v1 = ld_acq(&A.ctl[B_VERSION]);
            done = (ip == 0 && v1 == ver0) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, done, 0)) return {-1, 0};
        __nanosleep(backoff);
        backoff = min(2 * backoff, 512);
    }
}

// ------------------------------------------------------------------------------ finalisation --
// Block 0: the split set (the K-1 published nodes of largest SSE), the sequential procedure's leaf
// ids, centres, E_K and, per node, the id of the final leaf containing it.
HDF_DEV void finalise(const BisectArgs& A, unsigned char* dyn) {
    const int tid = threadIdx.x;
    const int K = A.K, rho = A.rho;
    const int n = min(__ldcg(&A.ctl[B_NALLOC]), A.maxn);
    double* sse = reinterpret_cast<double*>(dyn);
    int* st = reinterpret_cast<int*>(sse + n);
    int* par = st + n;
    int* ch = par + n;
    int* rk = ch + n;
    int* fin = rk + n;
    int* inS = fin + n;
    double* lsse = reinterpret_cast<double*>(((uintptr_t)(inS + n) + 7) & ~(uintptr_t)7);   // [K]
    int* lnode = reinterpret_cast<int*>(lsse + K);                                           // [K]
    __shared__ int s_cnt[2];
    for (int i = tid; i < n; i += kBT) {
        st[i] = __ldcg(&A.nstate[i]);
        sse[i] = __ldcg(&A.nsse[i]);
        par[i] = __ldcg(&A.nparent[i]);
        ch[i] = __ldcg(&A.nchild[i]);
    }
    for (int k = tid; k < K; k += kBT) { lsse[k] = 0.0; lnode[k] = -1; }
    if (tid < 2) s_cnt[tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kBT) {
        int c = 0x7fffffff;
        if (st[i] != ST_NONE) {
            c = 0;
            for (int j = 0; j < n; j++)
                if (st[j] != ST_NONE && (sse[j] > sse[i] || (sse[j] == sse[i] && j < i))) c++;
        }
        rk[i] = c;
    }
    __syncthreads();
    for (int i = tid; i < n; i += kBT) {
        const bool s = st[i] != ST_NONE && rk[i] < K - 1 && sse[i] > 0.0;
        inS[i] = s ? 1 : 0;
        if (s) {
            atomicAdd(&s_cnt[0], 1);
            if (st[i] != ST_DONE) atomicAdd(&s_cnt[1], 1);   // must not happen
        }
    }
    __syncthreads();
    const int nS = s_cnt[0];
    // final leaves: the root if nothing is split, else children of split nodes that are not split
    for (int i = tid; i < n; i += kBT) {
        int f = -1;
        if (st[i] != ST_NONE && !inS[i] && (i == 0 || inS[par[i]])) {
            int j = i;
            while (j != 0 && ch[par[j]] == j) j = par[j];   // child 0 inherits the parent's id
            f = (j == 0) ? 0 : rk[par[j]] + 1;
            if (f < K) {
                lnode[f] = i;
                lsse[f] = sse[i];
            }
        }
        fin[i] = f;
    }
    __syncthreads();
    // every node -> id of the final leaf on its root path (speculative descendants included)
    for (int i = tid; i < n; i += kBT) {
        int j = i, f = -1;
        while (j >= 0 && st[j] != ST_NONE) {
            if (fin[j] >= 0) { f = fin[j]; break; }
            j = (j == 0) ? -1 : par[j];
        }
        A.nfinal[i] = f;
    }
    const int ach = nS + 1;
    for (int e = tid; e < K * rho; e += kBT) {
        const int k = e / rho, d = e - k * rho;
        const int src = (k < ach && lnode[k] >= 0) ? lnode[k] : lnode[0];
        A.centres[e] = (float)__ldcg(&A.nmean[(size_t)src * rho + d]);
    }
    if (tid == 0) {
        double ek = 0.0;
        for (int k = 0; k < min(K, ach); k++) ek += lsse[k];
        *A.ek = ek;
        int status = (nS < K - 1) ? HDF_ERR_K : HDF_OK;
        if (s_cnt[1] != 0 || __ldcg(&A.ctl[B_ABORT])) status = HDF_ERR_CUDA;
        A.ctl[B_STATUS] = status;
        A.ctl[B_ACH] = ach;
    }
}

// --------------------------------------------------------------------------------- kernel -----
template <int RHO>
__global__ void __launch_bounds__(kBT, 1) k_bisect(const __grid_constant__ BisectArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ SplitSm S;
    const int rho = RHO > 0 ? RHO : A.rho;
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const long long gtid = (long long)blockIdx.x * kBT + tid;
    const long long gth = (long long)G * kBT;
    const int wsm = A.cap / 32 + 2;
    SplitIO io;
    io.dynX = reinterpret_cast<float*>(dsm);
    io.dynW = reinterpret_cast<uint32_t*>(dsm + (((size_t)A.cap * rho + 8) * 4 + 15) / 16 * 16);
    io.dynS = rho <= kSampRho ? reinterpret_cast<float*>(io.dynW + 2 * wsm) : nullptr;

    if (tid == 0) {
        mbar_init(&S.bar, 1);
        fence_barrier_init();
        S.tma_phase = 0;
    }
    // ---- init: node table, root statistics (mean, SSE) in a fixed order ----
    for (long long i = gtid; i < A.maxn; i += gth) A.nstate[i] = ST_NONE;
    if (A.labels)
        for (long long i = gtid; i < A.N; i += gth) A.node_of[i] = 0;
    if (gtid < B_NUM) A.ctl[gtid] = 0;
    const long long per = ((long long)A.N + G - 1) / G;
    const long long rb0 = min((long long)A.N, (long long)blockIdx.x * per), rb1 = min((long long)A.N, rb0 + per);
    double* rec0 = A.rec;
    double* rec1 = A.rec + (size_t)G * kRecV;
    for (int d0 = 0; d0 < rho; d0 += 8) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0;
        for (long long t = rb0 + tid; t < rb1; t += kBT) {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (d0 + j < rho) acc[j] += (double)__ldg(A.p + t * rho + d0 + j);
        }
        const int vi = warp_reduce_scatter16(acc);
        if (((tid & 31) & 1) == 0) S.red[(tid >> 5) * 16 + vi] = acc[0];
        __syncthreads();
        if (tid < 8 && d0 + tid < rho) {
            double s = 0.0;
            for (int w = 0; w < kBW; w++) s += S.red[w * 16 + tid];
            rec0[(size_t)blockIdx.x * kRecV + d0 + tid] = s;
        }
        __syncthreads();
    }
    __threadfence();
    grid.sync();
    if (tid == 0 && blockIdx.x == 0) {
        A.ctl[B_NALLOC] = 1;
        A.ctl[B_TASK] = -1;
    }
    for (int d = tid; d < rho; d += kBT) {
        double s = 0.0;
        for (int b = 0; b < G; b++) s += __ldcg(rec0 + (size_t)b * kRecV + d);
        S.c0[d] = s / (double)A.N;
    }
    __syncthreads();
    {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0.0;
        for (long long t = rb0 + tid; t < rb1; t += kBT) acc[0] += dist_rn(A.p + t * rho, S.c0, rho);
        const int vi = warp_reduce_scatter16(acc);
        if (((tid & 31) & 1) == 0) S.red[(tid >> 5) * 16 + vi] = acc[0];
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < kBW; w++) s += S.red[w * 16];
            rec1[(size_t)blockIdx.x * kRecV] = s;
        }
    }
    __threadfence();
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {
        double s = 0.0;
        for (int b = 0; b < G; b++) s += __ldcg(rec1 + (size_t)b * kRecV);
        A.nsse[0] = s;
        A.nm[0] = A.N;
        A.nstart[0] = 0;
        A.nbuf[0] = kBufInput;
        A.nparent[0] = -1;
        A.nchild[0] = -1;
        for (int d = 0; d < rho; d++) A.nmean[d] = S.c0[d];
        __threadfence();
        st_rel(&A.nstate[0], ST_FREE);
    }
    __threadfence();
    grid.sync();

    // ---- phase 1: nodes too large for one cluster, split by the whole grid ----
    GridGrp gg{(int)blockIdx.x, G, A.rec};
    while (true) {
        if (blockIdx.x == 0 && tid < 32) {
            const Claim c = claim_node(A, 1, A.ccap);
            if (tid == 0) {
                A.ctl[B_TASK] = c.task;
                A.ctl[B_TASKC] = c.cbase;
                __threadfence();
            }
        }
        grid.sync();
        const int task = __ldcg(&A.ctl[B_TASK]);
        const int cb = __ldcg(&A.ctl[B_TASKC]);
        if (task < 0) break;
        split_node<RHO>(A, gg, S, io, task, cb, -1);
        grid.sync();
    }

    // ---- phase 2: every thread-block cluster is a worker ----
    {
        cg::cluster_group cl = cg::this_cluster();
        const ClusterGrp g{(int)cl.block_rank(), (int)cl.num_blocks()};
        const int worker = blockIdx.x / g.size;
        while (true) {
            if (g.rank == 0 && tid < 32) {
                if (tid == 0) trace_ev(A, 1, 0, worker);
                const Claim c = claim_node(A, 2, 0);
                if (tid == 0) { S.task = c.task; S.cbase = c.cbase; }
            }
            cl.sync();
            int* rt = cl.map_shared_rank(&S.task, 0);
            int* rc = cl.map_shared_rank(&S.cbase, 0);
            const int task = *rt, cb = *rc;
            cl.sync();
            if (task < 0) break;
            split_node<RHO>(A, g, S, io, task, cb, worker);
        }
    }
    __threadfence();
    grid.sync();

    // ---- phase 3: split set, leaf ids, centres, E_K, labels ----
    if (blockIdx.x == 0) finalise(A, dsm);
    __threadfence();
    grid.sync();
    if (A.labels) {
        for (long long i = gtid; i < A.N; i += gth) A.labels[i] = __ldcg(&A.nfinal[__ldcg(&A.node_of[i])]);
    }
}

}  // namespace hdf
