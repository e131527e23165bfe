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
//   * phase 2 (cluster mode): while a claimable node does not fit one CTA's tile, every
//     thread-block cluster is a worker; a claimed node's members stay resident in the cluster's
//     shared memory (TMA bulk copies) for the whole split; partial sums are pushed into every peer's
//     shared memory with st.async and counted by an mbarrier (no cluster barrier per iteration);
//   * phase 3 (CTA mode): every CTA is a worker on the remaining (small) nodes, no inter-CTA
//     synchronisation inside a split.
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
constexpr int kGB = 384;            // doubles of the shared staging of gathered peer records

// control words
enum {
    B_INPROG = 0,  // claimed splits not yet published   } one 64-bit word (updated atomically
    B_VERSION,     // number of publications             } together, read as one snapshot)
    B_NALLOC,      // node ids allocated
    B_STATUS,      // HDF_OK / HDF_ERR_K / internal error
    B_ACH,         // leaves reached (achievable K)
    B_TASK,        // phase-1 task (node id or -1)
    B_TASKC,       // phase-1 task: first child id
    B_SPLITS,      // splits computed (including wasted speculative ones)
    B_ITERS,       // Lloyd passes executed (all splits)
    B_GRIDSPLITS,  // splits computed in grid mode
    B_TRACE_N,     // trace events recorded
    B_ABORT,       // internal error: 1 node table overflow, 2 cluster range not resident (never expected)
    B_NOTDONE,     // diagnostics: split-set nodes without a computed split (never expected)
    B_DIAG0, B_DIAG1, B_DIAG2, B_DIAG3, B_DIAG4, B_DIAG5,   // diagnostics (grid exchange timeouts)
    B_PAD,
    B_PTPASS, B_PTPASS_HI,     // u64: sum over the K-1 split nodes of m * (Lloyd passes) (8-byte aligned)
    B_PTSPLIT, B_PTSPLIT_HI,   // u64: sum over the K-1 split nodes of m
    B_NUM
};
enum { ST_FREE = 0, ST_CLAIMED = 1, ST_DONE = 2, ST_NONE = 3 };
constexpr int kBufInput = 2;        // node buffer 2 = the caller's p (root only), identity index
constexpr int kTeamMax = 16;        // grid-mode teams per round

struct BisectArgs {
    const float* p;
    int N, rho, K, maxn;
    int cap;            // points per CTA tile (multiple of kBT)
    int wcap;           // side words per CTA in the global scratch (streamed ranges)
    long long ccap;     // points a cluster keeps resident (C * cap)
    long long gabove;   // nodes larger than this are split by the whole grid (>= ccap: clusters stream)
    long long ctamax;   // nodes of at most this many points go to single CTAs (<= cap)
    long long qmax;     // nodes of at most this many points go to groups of 4 CTAs (<= 4 cap)
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
    int* nit;           // Lloyd passes of each computed split
    double* nmean;      // [maxn][rho]
    int* nfinal;        // [maxn] leaf id of the final leaf containing the node (labels)
    int* ctl;           // [B_NUM]
    long long* trace;   // [1 + 2 * kBisectTraceCap] (tag|node|worker, globaltimer), or null
    unsigned long long* xw;   // grid exchange: [2][clusters][2 kRecV] tagged record words (seq << 32 | half)
    int* teams;         // grid-mode round: [kTeamMax][5] (node, cbase, first cluster, clusters, -), then
                        // [clusters] the team of each cluster
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
HDF_DEV int ld_rlx(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
HDF_DEV void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
HDF_DEV unsigned long long ld_acq64(const int* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
HDF_DEV void red_release_add64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// (in progress, version) word at ctl[B_INPROG]: low 32 bits in progress, high 32 bits version
HDF_DEV unsigned long long* syncword(const int* ctl) {
    return reinterpret_cast<unsigned long long*>(const_cast<int*>(ctl) + B_INPROG);
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
// Hot loops address shared memory through a 32-bit base taken once per loop (volatile: the compiler
// keeps it in a register instead of re-deriving the generic pointer, S2R SR_CgaCtaId included, at
// every access); ptxas folds the constant parts of base + offset into the LDS immediates.
HDF_DEV uint32_t smem_pin(const void* p) {
    uint32_t r;
    asm volatile("{\n\t.reg .u64 t;\n\tcvta.to.shared.u64 t, %1;\n\tcvt.u32.u64 %0, t;\n\t}" : "=r"(r) : "l"(p));
    return r;
}
HDF_DEV float lds_fa(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
HDF_DEV uint32_t lds_ua(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
HDF_DEV void sts_ua(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
// Side words of a pass (bit j of word j/32 = point j on side 1): this and the previous iteration's,
// in shared memory (resident nodes) or global memory (streamed nodes).
struct WordsSm {
    uint32_t prev, cur;   // shared addresses
    HDF_DEV uint32_t ld_prev(int i) const { return lds_ua(prev + 4u * i); }
    HDF_DEV uint32_t ld_cur(int i) const { return lds_ua(cur + 4u * i); }
    HDF_DEV void st_cur(int i, uint32_t v) const { sts_ua(cur + 4u * i, v); }
    HDF_DEV WordsSm at(int w) const { return {prev + 4u * w, cur + 4u * w}; }
};
struct WordsGl {
    const uint32_t* prev;
    uint32_t* cur;
    HDF_DEV uint32_t ld_prev(int i) const { return prev[i]; }
    HDF_DEV uint32_t ld_cur(int i) const { return cur[i]; }
    HDF_DEV void st_cur(int i, uint32_t v) const { cur[i] = v; }
    HDF_DEV WordsGl at(int w) const { return {prev + w, cur + w}; }
};
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
        A.trace[1 + 2 * s] = (long long)tag | ((long long)(node & 0xFFFFF) << 8) | ((long long)(worker & 0xFFF) << 28);
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
// Warp reduce-scatter of N (power of two, <= 32) doubles: returns the index of the total this lane
// ends up holding in v[0]; the 32 / N lanes holding one index hold equal values (lane & (32/N - 1)
// == 0 is one of them).  log2(N) halving steps, then log2(32 / N) butterfly steps.
template <int N>
HDF_DEV int warp_reduce_scatter(double (&v)[N]) {
    const int lane = threadIdx.x & 31;
    int idx = 0;
#pragma unroll
    for (int step = 0; (N >> step) > 1; step++) {
        const int o = 16 >> step;
        const int half = (N >> step) / 2;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; j++) {
            const double send = upper ? v[j] : v[j + half];
            const double keep = upper ? v[j + half] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
        idx += upper ? half : 0;
    }
#pragma unroll
    for (int o = 32 / N / 2; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    return idx;
}
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
constexpr int kPushV = 16;          // values per pushed record (small rho: 2 rho + 2 <= 16)
constexpr int kMaxC = 16;           // CTAs per cluster
struct SplitSm {
    double c0[HDF_MAX_RHO], c1[HDF_MAX_RHO];   // centres (fp64, the oracle's values)
    float f0[HDF_MAX_RHO], f1[HDF_MAX_RHO];    // fp32-rounded centres
    double tot[kRecV];                          // reduced totals
    double outv[kRecV];                         // this CTA's record of the current exchange
    union {
        double rxb[2][kMaxC][kPushV];           // pushed records of the cluster (push exchange)
        struct {
            double rx[2][kRecV];                // posted record (pull exchange over DSMEM)
            double gb[kGB];                     // staged peer records (pull / grid exchanges)
        };
    };
    double grx[2][16][16];                      // grid mode: the cluster's CTA records, at the leader
    double red[kBW * 16];
    double wv[kBW];
    long long wa[kBW], wb[kBW];
    int wsum[kBW];
    int wp[kBT];                                // word prefix of a tile
    double tcta[HDF_MAX_RHO];                   // the CTA's total of its members (small rho)
    float xmax[HDF_MAX_RHO];                    // max |p_d| over the guide (decision bounds)
    float fpc[HDF_MAX_RHO];                     // farthest-pair pruning: sample centroid
    float fpr[2];                               //   max squared radius, lower bound of the diameter
    float wt[HDF_MAX_RHO], mt[HDF_MAX_RHO];     // fp32 c1 - c0, c0 + c1 (linear side test)
    short fpo[kFpCap];                          // farthest pair: the sample's outer points
    int iv[8];
    long long lv[4];
    uint64_t bar;                               // TMA mbarrier
    uint64_t xbar[2];                           // push-exchange mbarriers (by parity)
    uint64_t gbar[2];                           // grid mode: the cluster leader's record mbarriers
    uint64_t bbar;                              // group broadcast mbarrier (PushGrp::bcast)
    int2 bcv;                                   // group broadcast value
    int btask[16], bcb[16], bn, bgran;          // a cluster batch: tasks of its groups, count, group size
    uint32_t tma_phase;
    int task, cbase;
};

HDF_DEV uint32_t mapa_u32(uint32_t laddr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
    return r;
}
HDF_DEV void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
HDF_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// -------------------------------------------------------------------------------- groups ------
// A split runs on a group of CTAs.  Every exchange: each CTA assembles its record in S.outv[0, nv)
// (visible to its threads), exchange() makes every CTA's record of parity `par` readable through
// peer(), and the reductions below combine them in rank order (identical results in every CTA).
//   GridGrp     the whole cooperative grid: records in global memory, grid barrier;
//   ClusterGrp  a thread-block cluster, pull: records in shared memory read over DSMEM after a
//               cluster barrier (any record length);
//   PushGrp     a thread-block cluster, push: every CTA stores its record into every peer's shared
//               memory with st.async, completion counted by the receiver's mbarrier (no barrier,
//               no remote read round trip; records <= kPushV values);
//   CtaGrp      one CTA.
enum { XSUM = 0, XARGMAX = 1 };
// The whole cooperative grid, hierarchically: CTA records are combined inside each thread-block
// cluster over DSMEM (sums in rank order, or the best candidate), the cluster's first CTA posts the
// cluster record to global memory, one grid barrier, and every CTA reads the (few) cluster records.
// Record-level accessors (nrec / rec) therefore see cluster records; the order of every sum is
// fixed (clusters in order, CTAs in rank order inside a cluster), so all CTAs agree bit for bit.
// Grid mode: the group is the whole grid.  Exchange: every CTA pushes its record to its cluster's
// leader (st.async + mbarrier; a DSMEM pull for records longer than kPushV), the leader combines the
// cluster's records in a fixed order and stores the cluster record to global memory as tagged 64-bit
// words (exchange number << 32 | one 32-bit half of a value); every CTA reads the cluster records by
// polling those words until the tags match.  No grid barrier: each word validates itself, and the
// two parities alternate, so a slot is rewritten only after every CTA has read it (a CTA's next
// record, which the next-but-one exchange waits for, follows its reads).
struct GridGrp {
    int rank, size;           // CTA rank / count in the team
    int crank, csize, cid;    // rank in the cluster, cluster size, cluster index (in the grid)
    int ncl;                  // clusters in the team: [c0, c0 + ncl)
    unsigned long long* xw;   // [2][nclg][2 kRecV] tagged words (slots by grid cluster index)
    int* ctl;
    int c0 = 0;               // the team's first cluster
    int nclg = 0;             // clusters in the grid (slot stride)
    uint32_t tagbase = 0;     // team id << 16 (unique per team formation: stale slots never match)
    uint32_t seq = 0;         // exchanges so far (the same in every CTA of the team)
    uint32_t sq[2] = {0, 0};  // tag held by each parity's slots
    uint32_t gph = 0;         // phase bits of S.gbar (leader)
    uint32_t pushed = 0;      // bit par: that exchange went through the push buffer
    static constexpr bool kGrid = true, kLocal = false;
    HDF_DEV void sync() { cg::this_grid().sync(); }
    HDF_DEV unsigned long long* slot(int par, int q, int v) const {   // q: team cluster index
        return xw + (((size_t)par * nclg + c0 + q) * kRecV + v) * 2;
    }
    HDF_DEV void exchange(SplitSm& S, int par, int nv, int kind = XSUM) {
        cg::cluster_group cl = cg::this_cluster();
        const int tid = threadIdx.x;
        sq[par] = tagbase | (++seq & 0xffffu);
        const bool push = nv <= kPushV;
        pushed = push ? (pushed | (1u << par)) : (pushed & ~(1u << par));
        if (push && csize == 1) {   // no cluster (e.g. a launch without the cluster attribute)
            if (tid < nv) S.grx[par][0][tid] = S.outv[tid];
            __syncthreads();
        } else if (push) {
            if (crank == 0 && tid == 0) mbar_arrive_expect_tx(&S.gbar[par], (uint32_t)(csize * nv * 8));
            if (tid < nv)
                st_async_f64(mapa_u32(smem_u32(&S.grx[par][crank][tid]), 0), S.outv[tid],
                             mapa_u32(smem_u32(&S.gbar[par]), 0));
            if (crank == 0) {
                mbar_wait_cluster(&S.gbar[par], (gph >> par) & 1u);
                gph ^= 1u << par;
            }
        } else {
            for (int v = tid; v < nv; v += kBT) S.rx[par][v] = S.outv[v];
            cl.sync();
        }
        if (crank != 0) {
            if (!push) cl.sync();   // the leader reads this CTA's posted record in between
            return;
        }
        const uint64_t tag = (uint64_t)sq[par] << 32;
        auto put = [&](int v, double x) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(x);
            unsigned long long* w = slot(par, cid - c0, v);
            __stcg(w, tag | (b & 0xffffffffull));
            __stcg(w + 1, tag | (b >> 32));
        };
        auto rec = [&](int q, int v) -> double {
            return push ? S.grx[par][q][v] : cl.map_shared_rank(&S.rx[par][0], q)[v];
        };
        if (kind == XSUM) {
            for (int v = tid; v < nv; v += kBT) {
                double x[kMaxC];
#pragma unroll
                for (int q = 0; q < kMaxC; q++) x[q] = (q < csize) ? rec(q, v) : 0.0;
#pragma unroll
                for (int h = kMaxC / 2; h >= 1; h >>= 1) {
#pragma unroll
                    for (int q = 0; q < h; q++) x[q] = x[2 * q] + x[2 * q + 1];
                }
                put(v, x[0]);
            }
        } else if (tid == 0) {
            double bvv = -1.0;
            long long ia = -1, ib = -1;
            for (int q = 0; q < csize; q++) {
                const double y0 = rec(q, 0);
                const long long qa = (long long)rec(q, 1), qb = (long long)rec(q, 2);
                if (cand_better(y0, qa, bvv, ia)) { bvv = y0; ia = qa; ib = qb; }
            }
            put(0, bvv);
            put(1, (double)ia);
            put(2, (double)ib);
        }
        if (!push) cl.sync();   // the peers' rx stay in place until the leader has read them
    }
    HDF_DEV int nrec() const { return ncl; }
    HDF_DEV double peer(SplitSm&, int par, int q, int v) const {
        const unsigned long long* w = slot(par, q, v);
        const uint32_t want = sq[par];
        unsigned long long lo, hi;
        long long spins = 0;
        do {
            lo = __ldcv(w);
            hi = __ldcv(w + 1);
            if (++spins > (1LL << 22)) {
                if (atomicCAS(&ctl[B_ABORT], 0, 7) == 0) {
                    ctl[B_DIAG0] = (int)want;
                    ctl[B_DIAG1] = (int)(lo >> 32);
                    ctl[B_DIAG2] = (int)(hi >> 32);
                    ctl[B_DIAG3] = par * 100000 + q * 1000 + v;
                    ctl[B_DIAG4] = rank;
                    ctl[B_DIAG5] = (int)sq[par ^ 1];
                }
                break;
            }
        } while ((uint32_t)(lo >> 32) != want || (uint32_t)(hi >> 32) != want);
        return __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
    }
    // sum of value v over the CTAs of lower grid rank (clusters before this one, then the CTAs of
    // this cluster before this CTA, from the leader's push buffer or the peers' posted records)
    HDF_DEV double prefix(SplitSm& S, int par, int v) const {
        double acc = 0.0;
        for (int c = 0; c < cid - c0; c++) acc += peer(S, par, c, v);
        cg::cluster_group cl = cg::this_cluster();
        if ((pushed >> par) & 1u) {
            const double* lr = cl.map_shared_rank(&S.grx[par][0][0], 0);
            for (int q = 0; q < crank; q++) acc += lr[q * kPushV + v];
        } else {
            for (int q = 0; q < crank; q++) acc += cl.map_shared_rank(&S.rx[par][0], q)[v];
        }
        return acc;
    }
};
struct ClusterGrp {
    int rank, size;
    static constexpr bool kGrid = false, kLocal = false;
    HDF_DEV void sync() { cg::this_cluster().sync(); }
    HDF_DEV void exchange(SplitSm& S, int par, int nv, int = XSUM) {
        for (int v = threadIdx.x; v < nv; v += kBT) S.rx[par][v] = S.outv[v];
        cg::this_cluster().sync();
    }
    HDF_DEV int nrec() const { return size; }
    HDF_DEV double peer(SplitSm& S, int par, int q, int v) const {
        const double* p = cg::this_cluster().map_shared_rank(&S.rx[par][0], q);
        return p[v];
    }
    HDF_DEV void send(SplitSm& S, int par, int v, double x) { S.rx[par][v] = x; }
    HDF_DEV void wait(SplitSm&, int, int) { cg::this_cluster().sync(); }
    HDF_DEV void wait_warp0(SplitSm& S, int par, int nv) { wait(S, par, nv); }
};
struct PushGrp {
    int rank, size;
    uint32_t ph;    // phase bits of S.xbar[0..1] (every thread keeps its own copy)
    int base = 0;   // cluster rank of group rank 0 (a group is `size` consecutive CTAs of a cluster)
    static constexpr bool kGrid = false, kLocal = true;
    HDF_DEV int nrec() const { return size; }
    HDF_DEV void exchange(SplitSm& S, int par, int nv, int = XSUM) {
        const int tid = threadIdx.x;
        if (tid == 0) mbar_arrive_expect_tx(&S.xbar[par], (uint32_t)(size * nv * 8));
        for (int t = tid; t < size * nv; t += kBT) {
            const int q = t / nv, v = t - q * nv;
            st_async_f64(mapa_u32(smem_u32(&S.rxb[par][rank][v]), base + q), S.outv[v],
                         mapa_u32(smem_u32(&S.xbar[par]), base + q));
        }
        mbar_wait_cluster(&S.xbar[par], (ph >> par) & 1u);
        ph ^= 1u << par;
    }
    HDF_DEV double peer(SplitSm& S, int par, int q, int v) const { return S.rxb[par][q][v]; }
    // push one value of this CTA's record to every CTA of the cluster (itself included)
    HDF_DEV void send(SplitSm& S, int par, int v, double x) {
        const uint32_t la = smem_u32(&S.rxb[par][rank][v]), lb = smem_u32(&S.xbar[par]);
        for (int q = 0; q < size; q++) st_async_f64(mapa_u32(la, base + q), x, mapa_u32(lb, base + q));
    }
    HDF_DEV void wait(SplitSm& S, int par, int nv) {
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&S.xbar[par], (uint32_t)(size * nv * 8));
        mbar_wait_cluster(&S.xbar[par], (ph >> par) & 1u);
        ph ^= 1u << par;
    }
    // group rank 0's (a, b) to every CTA of the group (its own buffer and mbarrier, phase bit 2 of ph);
    // rank 0 calls it with its warp-0 values, every thread returns them
    HDF_DEV int2 bcast(SplitSm& S, int a, int b) {
        const int tid = threadIdx.x;
        if (tid == 0) mbar_arrive_expect_tx(&S.bbar, 8u);
        if (rank == 0 && tid < size) {
            const uint32_t la = smem_u32(&S.bcv), lb = smem_u32(&S.bbar);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s32 [%0], {%1, %2}, [%3];" ::"r"(
                             mapa_u32(la, base + tid)),
                         "r"(a), "r"(b), "r"(mapa_u32(lb, base + tid))
                         : "memory");
        }
        mbar_wait_cluster(&S.bbar, (ph >> 2) & 1u);
        ph ^= 4u;
        return make_int2(S.bcv.x, S.bcv.y);
    }
    // only warp 0 waits (the other warps keep their phase bits in step)
    HDF_DEV void wait_warp0(SplitSm& S, int par, int nv) {
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) mbar_arrive_expect_tx(&S.xbar[par], (uint32_t)(size * nv * 8));
            mbar_wait_cluster(&S.xbar[par], (ph >> par) & 1u);
        }
        ph ^= 1u << par;
    }
};
struct CtaGrp {
    int rank = 0, size = 1;
    static constexpr bool kGrid = false, kLocal = true;
    HDF_DEV void sync() { __syncthreads(); }
    HDF_DEV void exchange(SplitSm&, int, int, int = XSUM) { __syncthreads(); }
    HDF_DEV int nrec() const { return 1; }
    HDF_DEV double peer(SplitSm& S, int, int, int v) const { return S.outv[v]; }
    HDF_DEV void send(SplitSm& S, int, int v, double x) { S.outv[v] = x; }
    HDF_DEV void wait(SplitSm&, int, int) { __syncthreads(); }
    HDF_DEV void wait_warp0(SplitSm&, int, int) { __syncwarp(); }
};

// out[v] = sum over the group's records (rank order) of value v, v < nv; pre[v] (optional) = the
// same sum over the CTAs of lower rank than this one.  Remote records are first staged in shared
// memory in chunks with every load in flight at once (one DSMEM / L2 round trip per chunk).
// Block-wide; out/pre are shared and valid on return.
template <class Grp>
HDF_DEV void group_sum(const Grp& g, SplitSm& S, int par, int nv, double* out, double* pre) {
    const int tid = threadIdx.x;
    const int nr = g.nrec();
    double acc = 0.0, pacc = 0.0;
    if (Grp::kLocal) {
        if (tid < nv) {
            for (int q = 0; q < nr; q++) {
                const double x = g.peer(S, par, q, tid);
                acc += x;
                if (q < g.rank) pacc += x;
            }
        }
    } else {
        const int qc = max(1, kGB / nv);
        for (int q0 = 0; q0 < nr; q0 += qc) {
            const int nq = min(qc, nr - q0);
            for (int f = tid; f < nq * nv; f += kBT) {
                const int q = f / nv, v = f - q * nv;
                S.gb[f] = g.peer(S, par, q0 + q, v);
            }
            __syncthreads();
            if (tid < nv) {
                for (int q = 0; q < nq; q++) {
                    const double x = S.gb[q * nv + tid];
                    acc += x;
                    if (!Grp::kGrid && q0 + q < g.rank) pacc += x;
                }
            }
            __syncthreads();
        }
        if constexpr (Grp::kGrid) {
            if (pre && tid < nv) pacc = g.prefix(S, par, tid);
        }
    }
    if (tid < nv) {
        out[tid] = acc;
        if (pre) pre[tid] = pacc;
    }
    __syncthreads();
}
// Best (value desc, a asc) candidate over the group's records (fields 0 = value, 1 = a, 2 = b).
// Returns it in S.lv[0], S.lv[1] (a, b); shared, valid on return.
template <class Grp>
HDF_DEV void group_argmax(const Grp& g, SplitSm& S, int par) {
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int qc = kGB / 3;
    const int nr = g.nrec();
    if (Grp::kLocal && nr <= 32) {
        // one warp: lane q holds record q, warp-wide (value desc, a asc) reduction
        if (tid < 32) {
            double bvv = -1.0;
            long long ia = -1, ib = -1;
            if (lane < nr) {
                bvv = g.peer(S, par, lane, 0);
                ia = (long long)g.peer(S, par, lane, 1);
                ib = (long long)g.peer(S, par, lane, 2);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bvv, o);
                const long long oa = __shfl_xor_sync(0xffffffffu, ia, o);
                const long long ob = __shfl_xor_sync(0xffffffffu, ib, o);
                if (cand_better(ov, oa, bvv, ia)) { bvv = ov; ia = oa; ib = ob; }
            }
            if (lane == 0) {
                S.lv[0] = ia;
                S.lv[1] = ib;
            }
        }
        __syncthreads();
        return;
    }
    double bvv = -1.0;
    long long ia = -1, ib = -1;
    for (int q0 = 0; q0 < nr; q0 += qc) {
        const int nq = min(qc, nr - q0);
        if (!Grp::kLocal) {
            for (int f = tid; f < nq * 3; f += kBT) {
                const int q = f / 3, v = f - q * 3;
                S.gb[f] = g.peer(S, par, q0 + q, v);
            }
            __syncthreads();
        }
        if (tid == 0) {
            for (int q = 0; q < nq; q++) {
                double qv, fa, fb;
                if (Grp::kLocal) {
                    qv = g.peer(S, par, q0 + q, 0);
                    fa = g.peer(S, par, q0 + q, 1);
                    fb = g.peer(S, par, q0 + q, 2);
                } else {
                    qv = S.gb[3 * q];
                    fa = S.gb[3 * q + 1];
                    fb = S.gb[3 * q + 2];
                }
                const long long qa = (long long)fa, qb = (long long)fb;
                if (cand_better(qv, qa, bvv, ia)) { bvv = qv; ia = qa; ib = qb; }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        S.lv[0] = ia;
        S.lv[1] = ib;
    }
    __syncthreads();
}
// Sum over the group's CTAs (rank order) of record value v, by the calling thread, for groups whose
// records are local (all loads issued back to back).
template <class Grp>
HDF_DEV double local_sum(const Grp& g, SplitSm& S, int par, int v) {
    double x[kMaxC];
#pragma unroll
    for (int q = 0; q < kMaxC; q++) x[q] = (q < g.size) ? g.peer(S, par, q, v) : 0.0;
    // pairwise, in a fixed tree (the same in every CTA, so the totals are bit-identical)
#pragma unroll
    for (int h = kMaxC / 2; h >= 1; h >>= 1) {
#pragma unroll
        for (int q = 0; q < h; q++) x[q] = x[2 * q] + x[2 * q + 1];
    }
    return x[0];
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
    uint64_t* bar = &S.bar;
    const uintptr_t s = reinterpret_cast<uintptr_t>(src);
    const int delta = (int)((s & 15u) >> 2);
    const uintptr_t s0 = s - 4u * (uintptr_t)delta;
    const uintptr_t end = s + 4u * (uintptr_t)tn * (uintptr_t)rho;
    const uintptr_t body_end = end & ~(uintptr_t)15;
    const uint32_t body = body_end > s0 ? (uint32_t)(body_end - s0) : 0u;
    __syncthreads();   // the previous tile is fully consumed
    if (threadIdx.x == 0 && body > 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, body);
        for (uint32_t off = 0; off < body; off += 32768u)
            bulk_g2s(reinterpret_cast<char*>(dyn) + off, reinterpret_cast<const char*>(s0) + off,
                     min(32768u, body - off), bar);
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
// Sample accessors: value d of sample q, from shared memory (rho <= kSampRho) or global memory.
struct SampSm {
    uint32_t base;   // shared address of the staged sample
    int rs;          // row stride (floats)
    HDF_DEV float operator()(int q, int d) const { return lds_fa(base + 4u * (uint32_t)(q * rs + d)); }
    HDF_DEV void store(int q, int d, float v) const {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + 4u * (uint32_t)(q * rs + d)), "f"(v) : "memory");
    }
};
struct SampGl {
    const float* p;   // the node's first member
    size_t rs;        // row stride (floats): stride * rho
    HDF_DEV float operator()(int q, int d) const { return __ldcg(p + (size_t)q * rs + d); }
    HDF_DEV void store(int, int, float) const {}
};
template <int RHO, bool IND, class Acc>
HDF_DEV void row_farthest(int a, int nO, int rho, const Acc& ld, const short* fpo, double& best, int& arg) {
    // One pass: a lane keeps its running fp32 maximum M_l and re-evaluates in fp64 every pair whose
    // d32 >= M_l (1 - 8 (rho + 3) u) at the time it is seen -- a superset of the pairs that can be
    // the lane's fp64 maximum, whose fp64 maximum is therefore exact.  Rows and columns are positions
    // in the outer list: samples fpo[q] (IND) or the compacted copy's rows q.  A lane takes its
    // columns four at a time (loads and fp32 distances in flight together), in ascending order.
    const int lane = threadIdx.x & 31;
    constexpr float u = 5.9604644775390625e-08f;
    constexpr int RR = RHO > 0 ? RHO : 1;
    constexpr int UC = 4;
    const float shrink = 1.0f - 8.0f * (float)(rho + 3) * u;
    const int qa = IND ? fpo[a] : a;
    float xr[RR];
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) xr[d] = ld(qa, d);
    }
    float mx = -1.0f;
    best = -1.0;
    arg = -1;
    for (int q0 = a + 1 + lane; q0 < nO; q0 += 32 * UC) {
        float d32[UC];
        int qb[UC];
#pragma unroll
        for (int c = 0; c < UC; c++) {
            const int q = q0 + 32 * c;
            qb[c] = (q < nO) ? (IND ? fpo[q] : q) : qa;
            float acc = 0.f;
            if (RHO > 0) {
#pragma unroll
                for (int d = 0; d < RR; d++) {
                    const float t = xr[d] - ld(qb[c], d);
                    acc = fmaf(t, t, acc);
                }
            } else {
                for (int d = 0; d < rho; d++) {
                    const float t = ld(qa, d) - ld(qb[c], d);
                    acc = fmaf(t, t, acc);
                }
            }
            d32[c] = (q < nO) ? acc : -2.0f;
        }
#pragma unroll
        for (int c = 0; c < UC; c++) {
            if (d32[c] >= mx * shrink) {
                mx = fmaxf(mx, d32[c]);
                double dd = 0.0;
                for (int d = 0; d < rho; d++) dd = d2_rn(dd, (double)ld(qa, d), (double)ld(qb[c], d));
                if (dd > best) { best = dd; arg = q0 + 32 * c; }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        if (oa >= 0 && (arg < 0 || ob > best || (ob == best && oa < arg))) { best = ob; arg = oa; }
    }
}

// Farthest pair of the stride sample, exact and pruned (R3).  Row pruning: for any point c,
// ||x_a - x_b|| <= ||x_a - c|| + R with R = max_b ||x_b - c||, so neither end of a pair reaching L (a
// lower bound of the largest pair distance) lies outside O = {q : (||x_q - c|| + R)^2 >= L}; pairs
// outside O are strictly below the maximum, so restricting rows and columns to O keeps the argmax and
// its tie-breaking.  c = the node's mean (in S.fpc), L = the farthest partner of the sample point
// farthest from c.  fp32 estimates carry 1e-4 relative margins (their errors are < 1e-5 for
// rho <= 64).  Three barriers: the per-warp farthest-from-c records, the per-warp partner maxima,
// then the compaction of O.  The CTA's best pair (over its rows) is left in S.outv[0..2].
template <int RHO, bool CPT, class Acc, class Mark>
HDF_DEV void sample_farthest_pair(const Acc& ld, int sN, int rho, int r, int C, SplitSm& S, Mark mark) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int RR = RHO > 0 ? RHO : 1;
    float fc[RR];
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) fc[d] = S.fpc[d];
    }
    auto dist_c = [&](int q) {
        float r2 = 0.f;
        if (RHO > 0) {
#pragma unroll
            for (int d = 0; d < RR; d++) {
                const float t = ld(q, d) - fc[d];
                r2 = fmaf(t, t, r2);
            }
        } else {
            for (int d = 0; d < rho; d++) {
                const float t = ld(q, d) - S.fpc[d];
                r2 = fmaf(t, t, r2);
            }
        }
        return r2;
    };
    // (1) the point farthest from c: per thread (ascending q), per warp, then per CTA in every thread
    float r2m = -1.f;
    int rmi = 0;
    for (int q = tid; q < sN; q += kBT) {
        const float r2 = dist_c(q);
        if (r2 > r2m) { r2m = r2; rmi = q; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float orr = __shfl_xor_sync(0xffffffffu, r2m, o);
        const int oi = __shfl_xor_sync(0xffffffffu, rmi, o);
        if (orr > r2m || (orr == r2m && oi < rmi)) { r2m = orr; rmi = oi; }
    }
    if (lane == 0) { S.wv[warp] = (double)r2m; S.wa[warp] = rmi; }
    __syncthreads();
    mark(14);
    float R2 = -1.f;
    int istar = 0;
#pragma unroll
    for (int w = 0; w < kBW; w++) {
        const float x = (float)S.wv[w];
        const int i = (int)S.wa[w];
        if (x > R2 || (x == R2 && i < istar)) { R2 = x; istar = i; }
    }
    // (2) L = max_q ||x_q - x_istar||^2
    float xi[RR];
    if (RHO > 0) {
#pragma unroll
        for (int d = 0; d < RR; d++) xi[d] = ld(istar, d);
    }
    float lm = 0.f;
    for (int q = tid; q < sN; q += kBT) {
        float d2 = 0.f;
        if (RHO > 0) {
#pragma unroll
            for (int d = 0; d < RR; d++) {
                const float t = ld(q, d) - xi[d];
                d2 = fmaf(t, t, d2);
            }
        } else {
            for (int d = 0; d < rho; d++) {
                const float t = ld(q, d) - ld(istar, d);
                d2 = fmaf(t, t, d2);
            }
        }
        lm = fmaxf(lm, d2);
    }
    for (int o = 16; o > 0; o >>= 1) lm = fmaxf(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    if (lane == 0) S.wb[warp] = __float_as_int(lm);
    __syncthreads();
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < kBW; w++) L = fmaxf(L, __int_as_float((int)S.wb[w]));
    mark(15);
    const float R = sqrtf(fmaxf(R2, 0.f));
    const float lowb = L * (1.0f - 1e-4f);
    // (3) O in sample order: the sample indices in S.fpo and (CPT: a shared sample with compile-time
    // rho) the coordinates compacted in place to the front of the sample.  A chunk reads all its
    // samples before the barrier inside block_exscan and writes only below its own positions.
    int nO = 0;
    for (int q0 = 0; q0 < sN; q0 += kBT) {
        const int q = q0 + tid;
        bool in = false;
        float xq[RR];
        if (q < sN) {
            float r2 = 0.f;
            if (CPT) {
#pragma unroll
                for (int d = 0; d < RR; d++) {
                    xq[d] = ld(q, d);
                    const float t = xq[d] - fc[d];
                    r2 = fmaf(t, t, r2);
                }
            } else {
                r2 = dist_c(q);
            }
            const float ub = (sqrtf(r2) + R) * (1.0f + 1e-4f);
            in = ub * ub >= lowb;
        }
        int tot;
        const int pos = block_exscan(in ? 1 : 0, S.wsum, &tot);
        if (in) {
            S.fpo[nO + pos] = (short)q;
            if (CPT) {
#pragma unroll
                for (int d = 0; d < RR; d++) ld.store(nO + pos, d, xq[d]);
            }
        }
        nO += tot;
    }
    __syncthreads();
    mark(16);
    // (4) rows of O over the group's warps (rows ascend within a warp), then the CTA's best pair
    double bv = -1.0;
    long long ba = -1, bb = -1;
    for (int ia = r + C * warp; ia < nO; ia += C * kBW) {
        double best;
        int arg;
        row_farthest<RHO, !CPT>(ia, nO, rho, ld, S.fpo, best, arg);
        if (arg >= 0 && (ba < 0 || best > bv)) { bv = best; ba = S.fpo[ia]; bb = S.fpo[arg]; }
    }
    if (lane == 0) { S.wv[warp] = bv; S.wa[warp] = ba; S.wb[warp] = bb; }
    __syncthreads();
    if (tid == 0) {
        double bvv = -1.0;
        long long ia = -1, ib = -1;
        for (int w = 0; w < kBW; w++)
            if (cand_better(S.wv[w], S.wa[w], bvv, ia)) { bvv = S.wv[w]; ia = S.wa[w]; ib = S.wb[w]; }
        S.outv[0] = bvv;
        S.outv[1] = (double)ia;
        S.outv[2] = (double)ib;
    }
    __syncthreads();
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

// Small rho (compile-time): the side is decided from the linear form
//   D = ||x - c0||^2 - ||x - c1||^2 = sum_d w_d (2 x_d - m_d),  w = c1 - c0,  m = c0 + c1,
// evaluated in fp32 with w, m rounded to fp32 (2 FMAs per dimension).  Error bound, u = 2^-24,
// X_d = max |p_d| over the guide (S.xmax):
//   |D~ - D| <= u sum_d |w~_d| ((4.05 + 2.02 rho) X_d + (3.05 + 1.01 rho) |m~_d|)     (rounding of w, m,
//   2x - m, products and the FMA chain), doubled for safety, plus the fp64 error of the oracle's own
//   distances 2^-51 (rho + 2) sum_d (X_d + |m~_d| + |w~_d|)^2.  |D~| above the bound decides the side
//   exactly as the oracle does (d0 <= d1 -> side 0); otherwise the oracle's fp64 sequence decides.
// Thread per point, two points per thread per step (points j0 + tid and j0 + kBT + tid).  Word j/32
// of the tile holds the sides of 32 consecutive points (bit = lane).  Per thread: fp64 sums of the
// side-1 points s1 (DFMA with a 0/1 factor) and, when TOT, of all points (the CTA's total T; side-0
// sums are T - s1).  The side-1 and change counts come from the ballots (lane 0's copy is reduced).
template <int RHO>
HDF_DEV void lin_consts(const SplitSm& S, float (&wt)[RHO], float (&mt)[RHO], float& bound) {
    constexpr float u = 5.9604644775390625e-08f;
    float b1 = 0.f, b2 = 0.f;
#pragma unroll
    for (int d = 0; d < RHO; d++) {
        wt[d] = S.wt[d];
        mt[d] = S.mt[d];
        const float aw = fabsf(wt[d]), am = fabsf(mt[d]), X = S.xmax[d];
        b1 = fmaf(aw, (4.05f + 2.02f * RHO) * X + (3.05f + 1.01f * RHO) * am, b1);
        b2 = fmaf(X + am + aw, X + am + aw, b2);
    }
    bound = (2.0f * u * b1 + 4.5e-16f * (RHO + 2) * b2) * 1.001f;   // fp32 evaluation margin
}
// fp32 w = c1 - c0, m = c0 + c1 of the current centres (threads d < rho; callers synchronise)
HDF_DEV void set_lin(SplitSm& S, int rho) {
    for (int d = threadIdx.x; d < rho; d += kBT) {
        S.wt[d] = (float)(S.c1[d] - S.c0[d]);
        S.mt[d] = (float)(S.c0[d] + S.c1[d]);
    }
}

// Whole blocks of U * kBT points (no validity tests), the side words built straight from ballots:
// wu = points inside the certification band (decided again in fp64, rare), wp = side-1 points.
// CMP: compare with the previous pass's words; FULL: sums start from zero (every side-1 point
// is added) instead of being updated by the points that moved.  Returns the first unprocessed point.
template <int RHO, int U, bool TOT, bool CMP, bool FULL, class Words>
HDF_DEV int pass_blocks(int j0, uint32_t xs, int tn, const Words& Wd, const SplitSm& S, const float (&wt)[RHO],
                        const float (&mt)[RHO], float bound, double (&s1)[RHO], double (&st)[RHO], int& n1,
                        int& chg) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cw = 0;
    for (; j0 + U * kBT <= tn; j0 += U * kBT) {
        float x[U][RHO];
        uint32_t wp[U], wu[U];
        uint32_t anyu = 0;
#pragma unroll
        for (int h = 0; h < U; h++) {
            float D = 0.f;
#pragma unroll
            for (int d = 0; d < RHO; d++) {
                x[h][d] = lds_fa(xs + 4u * (uint32_t)((j0 + h * kBT) * RHO + d));
                D = fmaf(wt[d], fmaf(2.0f, x[h][d], -mt[d]), D);
            }
            wu[h] = __ballot_sync(0xffffffffu, !(fabsf(D) > bound));
            wp[h] = __ballot_sync(0xffffffffu, D > 0.f);
            anyu |= wu[h];
        }
        if (anyu) {
#pragma unroll
            for (int h = 0; h < U; h++) {
                if (wu[h]) {
                    bool s64 = false;
                    if ((wu[h] >> lane) & 1u) {
                        double dd0 = 0.0, dd1 = 0.0;
#pragma unroll
                        for (int d = 0; d < RHO; d++) {
                            const double v = (double)x[h][d];
                            dd0 = d2_rn(dd0, v, S.c0[d]);
                            dd1 = d2_rn(dd1, v, S.c1[d]);
                        }
                        s64 = !(dd0 <= dd1);
                    }
                    wp[h] = (wp[h] & ~wu[h]) | (__ballot_sync(0xffffffffu, s64) & wu[h]);
                }
            }
        }
        uint32_t anym = 0, mk[U];
#pragma unroll
        for (int h = 0; h < U; h++) {
            const int wi = (j0 >> 5) + h * kBW + warp;
            if (lane == 0) Wd.st_cur(wi, wp[h]);
            n1 += __popc(wp[h]);
            if (CMP) {   // only whether anything changed is used (convergence)
                const uint32_t c = wp[h] ^ Wd.ld_prev(wi);
                cw |= c;
                mk[h] = FULL ? wp[h] : c;
            } else {
                mk[h] = wp[h];
            }
            anym |= mk[h];
        }
        if (anym) {
#pragma unroll
            for (int h = 0; h < U; h++) {
                const double k = ((mk[h] >> lane) & 1u) ? (((wp[h] >> lane) & 1u) ? 1.0 : -1.0) : 0.0;
#pragma unroll
                for (int d = 0; d < RHO; d++) s1[d] = fma(k, (double)x[h][d], s1[d]);
            }
        }
        if (TOT) {
#pragma unroll
            for (int d = 0; d < RHO; d++) {
                double acc = 0.0;
#pragma unroll
                for (int h = 0; h < U; h++) acc += (double)x[h][d];
                st[d] += acc;
            }
        }
    }
    chg += cw != 0u;
    return j0;
}

template <int RHO, bool TOT, class Words>
HDF_DEV void pass_small(const float* X, int tn, const Words& Wd, bool cmp, bool full,
                        const SplitSm& S, double (&s1)[RHO], double (&st)[RHO], int& n1, int& chg) {
    // Incremental side-1 sums: s1 persists across the Lloyd iterations; a pass adds the points that
    // moved to side 1 and subtracts those that left it (full: s1 starts from 0 and every side-1 point
    // is added).  After the first iterations few points move, so the fp64 work nearly vanishes.
    // Whole blocks go through pass_blocks; the tail loop below handles the last partial block.
    constexpr int U = 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float wt[RHO], mt[RHO], bound;
    lin_consts<RHO>(S, wt, mt, bound);
    const uint32_t xs = smem_pin(X) + 4u * (uint32_t)(tid * RHO);
    int jb;
    if (TOT || !cmp) {
        jb = pass_blocks<RHO, 4, TOT, false, true>(0, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
        jb = pass_blocks<RHO, 1, TOT, false, true>(jb, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
    } else if (!full) {
        jb = pass_blocks<RHO, 4, TOT, true, false>(0, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
        jb = pass_blocks<RHO, 1, TOT, true, false>(jb, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
    } else {
        jb = pass_blocks<RHO, 4, TOT, true, true>(0, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
        jb = pass_blocks<RHO, 1, TOT, true, true>(jb, xs, tn, Wd, S, wt, mt, bound, s1, st, n1, chg);
    }
    for (int j0 = jb; j0 < tn; j0 += U * kBT) {   // the ragged tail (< kBT points)
        float x[U][RHO];
        bool sd[U], cert[U];
        uint32_t pw[U];
        bool allc = true;
#pragma unroll
        for (int h = 0; h < U; h++) {
            const int wi = (j0 >> 5) + h * kBW + warp;
            // (per warp: a word past the range may belong to the next streamed tile -- never touch it)
            const bool has = j0 + h * kBT + warp * 32 < tn;
            pw[h] = (cmp && has) ? Wd.ld_prev(wi) : 0u;
            const int j = j0 + h * kBT + tid;
            const bool ok = j < tn;
            float D = 0.f;
#pragma unroll
            for (int d = 0; d < RHO; d++) {
                x[h][d] = ok ? lds_fa(xs + 4u * (uint32_t)((j0 + h * kBT) * RHO + d)) : 0.f;
                D = fmaf(wt[d], fmaf(2.0f, x[h][d], -mt[d]), D);
            }
            cert[h] = !ok || fabsf(D) > bound;
            sd[h] = ok && D > 0.f;
            allc = allc && cert[h];
        }
        if (__ballot_sync(0xffffffffu, !allc)) {   // rare: the oracle's fp64 sequence
#pragma unroll
            for (int h = 0; h < U; h++) {
                if (!cert[h]) {
                    double dd0 = 0.0, dd1 = 0.0;
#pragma unroll
                    for (int d = 0; d < RHO; d++) {
                        const double v = (double)x[h][d];
                        dd0 = d2_rn(dd0, v, S.c0[d]);
                        dd1 = d2_rn(dd1, v, S.c1[d]);
                    }
                    sd[h] = !(dd0 <= dd1);
                }
            }
        }
        uint32_t anym = 0;
        uint32_t mk[U];
#pragma unroll
        for (int h = 0; h < U; h++) {
            const uint32_t w = __ballot_sync(0xffffffffu, sd[h]);
            const bool has = j0 + h * kBT + warp * 32 < tn;
            if (lane == 0 && has) Wd.st_cur((j0 >> 5) + h * kBW + warp, w);
            if (cmp && has) chg += __popc(w ^ pw[h]);
            n1 += __popc(w);
            mk[h] = full ? w : (w ^ pw[h]);   // points whose sum term changes
            anym |= mk[h];
        }
        if (anym) {
#pragma unroll
            for (int h = 0; h < U; h++) {
                const double k = ((mk[h] >> lane) & 1u) ? (sd[h] ? 1.0 : -1.0) : 0.0;
#pragma unroll
                for (int d = 0; d < RHO; d++) s1[d] = fma(k, (double)x[h][d], s1[d]);
            }
        }
        if (TOT) {
#pragma unroll
            for (int d = 0; d < RHO; d++) {
                double acc = 0.0;
#pragma unroll
                for (int h = 0; h < U; h++) acc += (double)x[h][d];
                st[d] += acc;
            }
        }
    }
}

// Generic rho: side phase (thread per point) ...
template <class Words>
HDF_DEV void pass_side_generic(const float* X, int tn, int rho, const Words& Wd, bool cmp,
                               const SplitSm& S, int& n1, int& chg) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float kd, kc;
    cert_consts(S, rho, kd, kc);
    const uint32_t xs = smem_pin(X);
    for (int j0 = 0; j0 < tn; j0 += kBT) {
        const int j = j0 + tid;
        const bool ok = j < tn;
        int sd = 0;
        if (ok) {
            const float* x = X + (size_t)j * rho;
            const uint32_t xa = xs + 4u * (uint32_t)(j * rho);
            float a0 = 0.f, a1 = 0.f;
            for (int d = 0; d < rho; d++) {
                const float v = lds_fa(xa + 4u * d);
                const float e0 = v - S.f0[d], e1 = v - S.f1[d];
                a0 = fmaf(e0, e0, a0);
                a1 = fmaf(e1, e1, a1);
            }
            sd = side_of(x, rho, a0, a1, kd, kc, S);
        }
        const uint32_t w = __ballot_sync(0xffffffffu, sd != 0);
        if (lane == 0 && j0 + warp * 32 < tn) {   // (words past the range: the next tile's)
            const int wi = (j0 >> 5) + warp;
            if (cmp) chg += __popc(w ^ Wd.ld_prev(wi));
            Wd.st_cur(wi, w);
        }
        n1 += sd;
    }
}
// ... then dimension-parallel sums: warp w owns dimensions w, w + 16, ... (<= 4 of them), lanes
// stride over the tile's points (consecutive points per lane group, odd rho: conflict free).
constexpr int kGenDims = (HDF_MAX_RHO + kBW - 1) / kBW;
template <class Words>
HDF_DEV void pass_sum_generic(const float* X, int tn, int rho, const Words& Wd, double (&a0)[kGenDims],
                              double (&a1)[kGenDims]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t xs = smem_pin(X);
    for (int j0 = 0; j0 < tn; j0 += 32) {
        const uint32_t w = Wd.ld_cur(j0 >> 5);
        const int j = j0 + lane;
        const bool ok = j < tn;
        const bool sd = (w >> lane) & 1u;
#pragma unroll
        for (int q = 0; q < kGenDims; q++) {
            const int d = warp + kBW * q;
            if (d < rho && ok) {
                const double v = (double)lds_fa(xs + 4u * (uint32_t)(j * rho + d));
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
HDF_DEV void split_node(const BisectArgs& A, Grp& g, SplitSm& S, const SplitIO& io, int v, int cbase, int worker) {
    const int rho = RHO > 0 ? RHO : A.rho;
    const int nv = 2 * rho + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = g.rank, C = g.size;
    const int m = __ldcg(&A.nm[v]), start = __ldcg(&A.nstart[v]), buf = __ldcg(&A.nbuf[v]);
    const int nbuf = (buf == kBufInput) ? 0 : (buf ^ 1);
    const int a = (int)((long long)m * r / C), e = (int)((long long)m * (r + 1) / C), np = e - a;
    const float* Pg = A.pts[buf] + (size_t)start * rho;   // the node's points
    const bool resident = (m + C - 1) / C <= A.cap;      // uniform over the group (np <= ceil(m / C))
    // Nodes larger than the group's shared memory stream their points tile by tile (grid mode, and
    // cluster mode up to gabove); the side words then live in the CTA's global scratch (guarded).
    if (!resident && (m + C - 1) / C > 32LL * (A.wcap - 2)) {
        if (tid == 0) atomicExch(&A.ctl[B_ABORT], 2);
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
    const int stride = (m + kFpCap - 1) / kFpCap, sN = (m + stride - 1) / stride;
    // The stride sample is staged in shared memory: in its own area for rho <= kSampRho, else in the
    // tile area (sN <= cap), whose TMA is then issued after the farthest pair has read the sample (read
    // from global memory element by element, the sample cost ~30 us per seeding phase at rho = 31)
    const bool insm = io.dynS != nullptr;
    float* const sbuf = insm ? io.dynS : (sN <= A.cap ? io.dynX : nullptr);
    TileLd rt{nullptr, 0u};
    if (resident && insm) rt = tile_issue(Pg + (size_t)a * rho, np, rho, io.dynX, S);
    // ---- 2. farthest pair of the stride sample members[0::stride] (R3) ----
    if (sbuf) {
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
                if (f < sN * rho) sbuf[f] = vv[u];
            }
        }
        __syncthreads();
        if (lead) trace_ev(A, 7, v, worker);
    }
    if (tid < rho) S.fpc[tid] = (float)__ldcg(&A.nmean[(size_t)v * rho + tid]);
    __syncthreads();
    auto mark = [&](int tag) {
        if (lead) trace_ev(A, tag, v, worker);
    };
    if (insm) sample_farthest_pair<RHO, (RHO > 0)>(SampSm{smem_pin(io.dynS), rho}, sN, rho, r, C, S, mark);
    else if (sbuf) sample_farthest_pair<RHO, false>(SampSm{smem_pin(sbuf), rho}, sN, rho, r, C, S, mark);
    else sample_farthest_pair<RHO, false>(SampGl{Pg, (size_t)stride * rho}, sN, rho, r, C, S, mark);
    // the sample in the tile area has been read (sample_farthest_pair ends with a barrier): the tile now
    if (resident && !insm) rt = tile_issue(Pg + (size_t)a * rho, np, rho, io.dynX, S);
    if (lead) trace_ev(A, 8, v, worker);
    g.exchange(S, par, 3, XARGMAX);
    if (lead) trace_ev(A, 9, v, worker);
    group_argmax(g, S, par);
    par ^= 1;
    if (lead) trace_ev(A, 10, v, worker);
    if (tid == 0 && S.lv[0] < 0) { S.lv[0] = 0; S.lv[1] = (sN > 1) ? 1 : 0; }
    __syncthreads();
    for (int f = tid; f < 2 * rho; f += kBT) {
        const int w = f / rho, d = f - w * rho;
        const long long q = S.lv[w];
        const float x = __ldcg(Pg + (size_t)q * stride * rho + d);   // (the staged sample is compacted)
        (w ? S.c1 : S.c0)[d] = (double)x;
        (w ? S.f1 : S.f0)[d] = x;
    }
    __syncthreads();
    set_lin(S, rho);
    const float* X = rt.ptr;
    if (resident) tile_wait(S, rt);
    __syncthreads();
    if (lead) trace_ev(A, 3, v, worker);

    // ---- 3. Lloyd iterations (R4) ----
    // Record of a pass (per CTA): [0, rho) side-0 sums, [rho, 2 rho) side-1 sums, 2 rho: side-1 count,
    // 2 rho + 1: nonzero iff some side changed (a count of warps with changes).  Each value v is
    // reduced by thread v and sent straight from it.
    int it = 0, fbw = 0, fpar = 0;
    bool conv = false;
    long long tph[4] = {0, 0, 0, 0};   // diagnostics (lead thread): pass, reduce, exchange, update
    long long tq = lead ? gtimer() : 0;
    auto tick = [&](int ph) {
        if (lead && A.trace) {
            const long long t1 = gtimer();
            tph[ph] += t1 - tq;
            tq = t1;
        }
    };
    constexpr int RH = RHO > 0 ? RHO : 1;
    double s1p[RH], stp[RH];   // small rho: per-thread side-1 sums (persistent) and totals
#pragma unroll
    for (int q = 0; q < RH; q++) { s1p[q] = 0.0; stp[q] = 0.0; }
    long long n1tot = 0, chgtot = 0;
    for (; it < kMaxIter; it++) {
        uint32_t* curW = (it & 1) ? W1 : W0;
        const uint32_t* prevW = (it & 1) ? W0 : W1;
        bool redo = false;
        while (true) {
            int n1 = 0, chg = 0;
            if (RHO > 0) {
                const bool full = (it == 0) || redo;
                const bool tot = (it == 0 && !redo);   // the CTA's total T, once per split
                if (full) {
#pragma unroll
                    for (int q = 0; q < RH; q++) s1p[q] = 0.0;
                }
                if (resident) {
                    const WordsSm wd{smem_pin(prevW), smem_pin(curW)};
                    if (tot) pass_small<RH, true>(X, np, wd, it > 0, full, S, s1p, stp, n1, chg);
                    else pass_small<RH, false>(X, np, wd, it > 0, full, S, s1p, stp, n1, chg);
                } else {
                    // streamed: the tile's side words are staged in the (otherwise idle) shared word
                    // buffers, the previous ones loaded while the tile's TMA is in flight
                    const WordsSm wd{smem_pin(io.dynW), smem_pin(io.dynW + wsm)};
                    for (int t0 = 0; t0 < np; t0 += A.cap) {
                        const int tn = min(A.cap, np - t0), nw = (tn + 31) >> 5;
                        const TileLd tl = tile_issue(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                        if (it > 0)
                            for (int i = tid; i < nw; i += kBT) io.dynW[i] = __ldcg(prevW + (t0 >> 5) + i);
                        tile_wait(S, tl);
                        if (tot) pass_small<RH, true>(tl.ptr, tn, wd, it > 0, full, S, s1p, stp, n1, chg);
                        else pass_small<RH, false>(tl.ptr, tn, wd, it > 0, full, S, s1p, stp, n1, chg);
                        __syncthreads();
                        for (int i = tid; i < nw; i += kBT) curW[(t0 >> 5) + i] = io.dynW[wsm + i];
                    }
                }
                tick(0);
                constexpr int NR = (2 * RH + 2 <= 8) ? 8 : 16;
                double vv[NR];
#pragma unroll
                for (int q = 0; q < NR; q++) vv[q] = 0.0;
#pragma unroll
                for (int q = 0; q < RH; q++) { vv[q] = tot ? stp[q] : 0.0; vv[RH + q] = s1p[q]; }
                vv[2 * RH] = (lane == 0) ? (double)n1 : 0.0;     // ballot counts: lane 0's copy
                vv[2 * RH + 1] = (lane == 0) ? (double)chg : 0.0;
                const int vi = warp_reduce_scatter<NR>(vv);
                if ((lane & (32 / NR - 1)) == 0) S.red[warp * 16 + vi] = vv[0];
                __syncthreads();
                if constexpr (Grp::kLocal) {
                    // warp 0: the CTA's record, the exchange, the group totals and the new centres
                    if (warp == 0) {
                        double x = 0.0;
                        if (lane < nv) {
                            double t[kBW], u1[kBW];
#pragma unroll
                            for (int w = 0; w < kBW; w++) {
                                t[w] = S.red[w * 16 + lane];
                                u1[w] = (lane < RH) ? S.red[w * 16 + RH + lane] : 0.0;
                            }
                            double ts = 0.0, us = 0.0;
#pragma unroll
                            for (int w = 0; w < kBW; w++) { ts += t[w]; us += u1[w]; }
                            if (lane < RH) {   // side-0 sums = T - s1 (T of the first pass)
                                if (tot) S.tcta[lane] = ts;
                                x = (tot ? ts : S.tcta[lane]) - us;
                            } else {
                                x = ts;
                            }
                            g.send(S, par, lane, x);
                        }
                        tick(1);
                        g.wait_warp0(S, par, nv);
                        tick(2);
                        const double tv = (lane < nv) ? local_sum(g, S, par, lane) : 0.0;
                        const long long n1t = (long long)__shfl_sync(0xffffffffu, tv, 2 * RH);
                        const long long cht = (long long)__shfl_sync(0xffffffffu, tv, 2 * RH + 1);
                        const double t1 = __shfl_sync(0xffffffffu, tv, (RH + lane) & 31);
                        const bool upd = !(it > 0 && cht == 0) && (redo || !(n1t == 0 || n1t == m));
                        if (upd && lane < RH) {
                            const double c0 = tv / (double)(m - n1t), c1 = t1 / (double)n1t;
                            S.c0[lane] = c0;
                            S.c1[lane] = c1;
                            S.f0[lane] = (float)c0;
                            S.f1[lane] = (float)c1;
                            S.wt[lane] = (float)(c1 - c0);
                            S.mt[lane] = (float)(c0 + c1);
                        }
                        if (lane == 0) {
                            S.lv[2] = n1t;
                            S.lv[3] = cht;
                        }
                    } else {
                        g.wait_warp0(S, par, nv);   // phase bookkeeping only
                    }
                    __syncthreads();
                } else {
                    if (tid < nv) {
                        double x = 0.0;
                        if (tid < RH) {   // side-0 sums = T - s1 (T of the first pass)
                            double t = 0.0, u1 = 0.0;
                            for (int w = 0; w < kBW; w++) { t += S.red[w * 16 + tid]; u1 += S.red[w * 16 + RH + tid]; }
                            if (tot) S.tcta[tid] = t;
                            x = (tot ? t : S.tcta[tid]) - u1;
                        } else {
                            for (int w = 0; w < kBW; w++) x += S.red[w * 16 + tid];
                        }
                        S.outv[tid] = x;
                    }
                    __syncthreads();
                    tick(1);
                    g.exchange(S, par, nv);
                    tick(2);
                }
            } else {
                double s0[kGenDims], s1[kGenDims];
#pragma unroll
                for (int q = 0; q < kGenDims; q++) { s0[q] = 0.0; s1[q] = 0.0; }
                if (resident) {
                    const WordsSm wd{smem_pin(prevW), smem_pin(curW)};
                    pass_side_generic(X, np, rho, wd, it > 0, S, n1, chg);
                    __syncthreads();
                    pass_sum_generic(X, np, rho, wd, s0, s1);
                } else {
                    const WordsSm wd{smem_pin(io.dynW), smem_pin(io.dynW + wsm)};   // (staged, as above)
                    for (int t0 = 0; t0 < np; t0 += A.cap) {
                        const int tn = min(A.cap, np - t0), nw = (tn + 31) >> 5;
                        const TileLd tl = tile_issue(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                        if (it > 0)
                            for (int i = tid; i < nw; i += kBT) io.dynW[i] = __ldcg(prevW + (t0 >> 5) + i);
                        tile_wait(S, tl);
                        pass_side_generic(tl.ptr, tn, rho, wd, it > 0, S, n1, chg);
                        __syncthreads();
                        pass_sum_generic(tl.ptr, tn, rho, wd, s0, s1);
                        __syncthreads();
                        for (int i = tid; i < nw; i += kBT) curW[(t0 >> 5) + i] = io.dynW[wsm + i];
                    }
                }
#pragma unroll
                for (int q = 0; q < kGenDims; q++) {
                    const int d = warp + kBW * q;
                    const double x0 = warp_sum(s0[q]), x1 = warp_sum(s1[q]);
                    if (lane == 0 && d < rho) { S.outv[d] = x0; S.outv[rho + d] = x1; }
                }
                n1 = __reduce_add_sync(0xffffffffu, n1);
                chg = __reduce_add_sync(0xffffffffu, chg);
                if (lane == 0) { S.red[warp * 2] = (double)n1; S.red[warp * 2 + 1] = (double)chg; }
                __syncthreads();
                if (tid < 2) {
                    double acc = 0.0;
                    for (int w = 0; w < kBW; w++) acc += S.red[w * 2 + tid];
                    S.outv[2 * rho + tid] = acc;
                }
                __syncthreads();
                g.exchange(S, par, nv);
            }
            // totals over the group in rank order (bit-identical in every CTA); n1 and the change count
            // are read by every thread, the sums by the threads of the centre update below
            if (Grp::kLocal && RHO > 0) {   // warp 0 has reduced the totals and updated the centres
                n1tot = S.lv[2];
                chgtot = S.lv[3];
            } else if (Grp::kLocal) {
                n1tot = (long long)local_sum(g, S, par, 2 * rho);
                chgtot = (long long)local_sum(g, S, par, 2 * rho + 1);
            } else {
                group_sum(g, S, par, nv, S.tot, nullptr);
                n1tot = (long long)S.tot[2 * rho];
                chgtot = (long long)S.tot[2 * rho + 1];
            }
            fpar = par;
            par ^= 1;
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
                S.outv[0] = bvv;
                S.outv[1] = (double)ia;
                S.outv[2] = -1.0;
            }
            __syncthreads();
            g.exchange(S, par, 3, XARGMAX);
            group_argmax(g, S, par);
            par ^= 1;
            const long long pick = S.lv[0] < 0 ? 0 : S.lv[0];
            for (int d = tid; d < rho; d += kBT) {
                const float x = __ldcg(Pg + (size_t)pick * rho + d);
                if (side1_empty) { S.c1[d] = (double)x; S.f1[d] = x; }
                else { S.c0[d] = (double)x; S.f0[d] = x; }
            }
            __syncthreads();
            set_lin(S, rho);
            __syncthreads();
            redo = true;
        }
        fbw = it & 1;
        if (it > 0 && chgtot == 0) { conv = true; break; }   // the final partition is this pass's
        if (Grp::kLocal && RHO > 0) {                        // centres already updated by warp 0
            tick(3);
            continue;
        }
        for (int d = tid; d < rho; d += kBT) {
            double t0v, t1v;
            if (Grp::kLocal) {
                t0v = local_sum(g, S, fpar, d);
                t1v = local_sum(g, S, fpar, rho + d);
            } else {
                t0v = S.tot[d];
                t1v = S.tot[rho + d];
            }
            const double c0 = t0v / (double)(m - n1tot), c1 = t1v / (double)n1tot;
            S.c0[d] = c0;
            S.c1[d] = c1;
            S.f0[d] = (float)c0;
            S.f1[d] = (float)c1;
            S.wt[d] = (float)(c1 - c0);
            S.mt[d] = (float)(c0 + c1);
        }
        __syncthreads();
        tick(3);
    }
    if (!conv) it = kMaxIter - 1;
    if (lead) {
        trace_ev(A, 4, v, worker);
        trace_ev(A, 6, it + 1, worker);
        for (int q = 0; q < 4; q++) trace_ev(A, 20 + q, (int)(tph[q] / 100), worker);   // 0.1 us units
    }
    const uint32_t* FW = fbw ? W1 : W0;
    // final partition sizes from the last pass's records: side-1 members of lower ranks, total
    long long pre1l = 0;
    if (Grp::kLocal) {
        for (int q = 0; q < r; q++) pre1l += (long long)g.peer(S, fpar, q, 2 * rho);
    } else {
        group_sum(g, S, fpar, nv, S.tot, S.outv);   // outv: sums over the lower ranks
        pre1l = (long long)S.outv[2 * rho];
        __syncthreads();
    }
    const int m0 = m - (int)n1tot;
    const int pre1 = (int)pre1l, pre0 = a - pre1;

    // ---- 4. stable partition into the other buffer (children [start, start+m0), [start+m0, start+m)),
    //         fused with the children's SSE w.r.t. their means (= the final centres) ----
    {
        float* Po = A.ptsw[nbuf] + (size_t)start * rho;
        int* Io = A.idx[nbuf] + start;
        const int* Ii = (buf == kBufInput) ? nullptr : A.idx[buf] + start;
        double se0 = 0.0, se1 = 0.0;
        int run0 = 0;
        for (int t0 = 0; t0 < np; t0 += A.cap) {
            const int tn = min(A.cap, np - t0);
            const uint32_t* FWt = FW + (t0 >> 5);   // the tile's final side words
            const float* T = X;
            const int nw = (tn + 31) >> 5;
            if (!resident) {   // streamed: the words staged in shared memory under the tile's TMA
                const TileLd tl = tile_issue(Pg + (size_t)(a + t0) * rho, tn, rho, io.dynX, S);
                for (int i = tid; i < nw; i += kBT) io.dynW[i] = __ldcg(FWt + i);
                tile_wait(S, tl);
                T = tl.ptr;
                FWt = io.dynW;
            }
            const uint32_t Ts = smem_pin(T);
            for (int w0 = 0; w0 < nw; w0 += kBT) {
                // word prefix of side-0 counts for words [w0, w0 + kBT) of the tile
                const int wi = w0 + tid;
                int z = 0;
                if (wi < nw) {
                    const int nb = min(32, tn - wi * 32);
                    const uint32_t valid = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
                    z = __popc(~FWt[wi] & valid);
                }
                int ztot;
                const int zp = block_exscan(z, S.wsum, &ztot);
                S.wp[tid] = zp;
                __syncthreads();
                const int jlo = w0 * 32, jhi = min(tn, (w0 + kBT) * 32);
                constexpr int U = 4;   // pixel indices of U points in flight per thread
                for (int jb = jlo; jb < jhi; jb += U * kBT) {
                    int pix[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int jj = t0 + jb + u * kBT + tid;
                        pix[u] = (jb + u * kBT + tid < jhi) ? (Ii ? __ldcg(Ii + a + jj) : (start + a + jj)) : 0;
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int j0 = jb + u * kBT;
                        if (j0 >= jhi) break;
                        const int j = j0 + tid;
                        const int wl = ((j0 - jlo) >> 5) + warp;
                        const uint32_t w = FWt[(j0 >> 5) + warp];
                        if (j < jhi) {
                            const int sd = (w >> lane) & 1u;
                            const int zb = S.wp[wl] + __popc(~w & ((1u << lane) - 1u));   // side-0 before j (chunk)
                            const int jj = t0 + j;                                       // CTA-relative index
                            const int z0 = run0 + zb;                                    // side-0 before jj
                            const int dst = sd ? (m0 + pre1 + (jj - z0)) : (pre0 + z0);
                            const uint32_t xa = Ts + 4u * (uint32_t)(j * rho);
                            float* o = Po + (size_t)dst * rho;
                            const double* cc = sd ? S.c1 : S.c0;
                            double dd = 0.0;
                            for (int d = 0; d < rho; d++) {
                                const float xv = lds_fa(xa + 4u * d);
                                o[d] = xv;
                                dd = d2_rn(dd, (double)xv, cc[d]);
                            }
                            if (sd) se1 += dd;
                            else se0 += dd;
                            Io[dst] = pix[u];
                        }
                    }
                }
                run0 += ztot;
                __syncthreads();
            }
        }
        // the scatter is made visible before the SSE records are sent: the group leader publishes the
        // children once it has every record (no separate barrier for push groups)
        __threadfence();
        // children's SSE over the group
        double vv[2] = {se0, se1};
        const int vi = warp_reduce_scatter<2>(vv);
        if ((lane & 15) == 0) S.red[warp * 16 + vi] = vv[0];
        __syncthreads();
        if (tid < 2) {
            double x = 0.0;
            for (int w = 0; w < kBW; w++) x += S.red[w * 16 + tid];
            S.outv[tid] = x;
        }
        __syncthreads();
        if (lead) trace_ev(A, 12, v, worker);
        g.exchange(S, par, 2);
        group_sum(g, S, par, 2, S.tot + 1, nullptr);   // tot[1] = sse0, tot[2] = sse1
        par ^= 1;
    }

    if (lead) trace_ev(A, 13, v, worker);
    // Pull groups (ClusterGrp) still need a barrier; push and grid groups' SSE exchange has already
    // delivered every CTA's record, sent after its fence, to the lead.
    if constexpr (!Grp::kLocal && !Grp::kGrid) g.sync();
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
        A.nit[v] = it + 1;
        // st.release orders the records above before each state; the sync-word update (version + 1,
        // in progress - 1, one atomic) is a release too, after the states
        st_rel(&A.nstate[c], ST_FREE);
        st_rel(&A.nstate[c + 1], ST_FREE);
        st_rel(&A.nstate[v], ST_DONE);
        atomicAdd(&A.ctl[B_SPLITS], 1);
        atomicAdd(&A.ctl[B_ITERS], it + 1);
        if (Grp::kGrid) atomicAdd(&A.ctl[B_GRIDSPLITS], 1);
        red_release_add64(syncword(A.ctl), (1ULL << 32) - 1ULL);
        trace_ev(A, 5, v, worker);
        trace_ev(A, 17, c, v);   // children c, c + 1 of v (the worker field carries the parent)
    }
}

// ------------------------------------------------------------------------------- the claim ----
// Warp-cooperative.  Chooses the FREE node of largest SSE (ties -> lowest id) with SSE > 0 and >= 2
// members, and claims it if fewer than K-1 published nodes precede it in (SSE desc, id asc) order.
// Only nodes with bigcap < m <= maxm points are considered.  mode 1 (grid phase, a single claimer)
// and mode 3 (a group's follow-up claim inside a cluster batch): return -1 when nothing is claimable.  mode 2 (cluster / CTA phases): when nothing is claimable,
// waits until a publication changes the table; returns -1 once nothing is claimable and no split is
// in progress.
struct Claim {
    int task, cbase;
};
template <int kScan>   // node-table entries per lane: the table holds 32 kScan nodes
HDF_DEV Claim claim_node_t(const BisectArgs& A, int mode, long long bigcap, int wid, long long maxm) {
    const int lane = threadIdx.x & 31;
    int backoff = 16;
    while (true) {
        if (ld_acq(&A.ctl[B_ABORT])) return {-1, 0};
        int ver0 = 0, n = 0;
        if (lane == 0) {
            ver0 = (int)(ld_acq64(A.ctl) >> 32);
            n = ld_acq(&A.ctl[B_NALLOC]);
        }
        ver0 = __shfl_sync(0xffffffffu, ver0, 0);
        n = min(__shfl_sync(0xffffffffu, n, 0), A.maxn);
        const long long mmin = max(bigcap + 1, 2LL);
        // states (relaxed, all in flight), then one acquire fence before the fields they publish
        int stv[kScan];
#pragma unroll
        for (int u = 0; u < kScan; u++) {
            const int i = lane + 32 * u;
            stv[u] = (i < n) ? ld_rlx(&A.nstate[i]) : ST_NONE;
        }
        fence_acq_rel();
        double ssev[kScan];
        unsigned elig = 0;   // FREE, SSE > 0, large enough
#pragma unroll
        for (int u = 0; u < kScan; u++) {
            const int i = lane + 32 * u;
            ssev[u] = (stv[u] != ST_NONE) ? __ldcg(&A.nsse[i]) : -1.0;
            if (stv[u] == ST_FREE && ssev[u] > 0.0) {
                const int mi = __ldcg(&A.nm[i]);
                if (mi >= mmin && mi <= maxm) elig |= 1u << u;
            }
        }
        // Candidates in (SSE desc, id asc) order.  Idle workers start at different ranks of that order
        // (wid modulo the number of candidates, at most 8 deep) so that they do not all race for the
        // same node; a lost race moves on to the next candidate without rescanning.  A candidate that
        // fails the rank test ends the walk (every later one fails it too); if candidates were
        // skipped, the walk is repeated from the top.
        const int nel0 = __reduce_add_sync(0xffffffffu, __popc(elig));
        bool lost = false;
        for (int walk = 0; walk < 2 && nel0 > 0; walk++) {
            unsigned el = elig;
            int skip = (walk == 0 && mode != 1) ? (wid % min(nel0, 8)) : 0;
            const bool skipped = skip > 0;
            while (true) {
                double bs = -1.0;
                int bi = -1;
#pragma unroll
                for (int u = 0; u < kScan; u++) {
                    if ((el >> u) & 1u) {
                        const int i = lane + 32 * u;
                        if (bi < 0 || ssev[u] > bs) { bs = ssev[u]; bi = i; }
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, bs, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (oi >= 0 && (bi < 0 || ob > bs || (ob == bs && oi < bi))) { bs = ob; bi = oi; }
                }
                if (bi < 0) break;
                if ((bi & 31) == lane) el &= ~(1u << (bi >> 5));   // consumed from the local snapshot
                if (skip > 0) { skip--; continue; }
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < kScan; u++) {
                    const int i = lane + 32 * u;
                    if (stv[u] != ST_NONE) cnt += (ssev[u] > bs || (ssev[u] == bs && i < bi)) ? 1 : 0;
                }
                cnt = __reduce_add_sync(0xffffffffu, cnt);
                if (cnt >= A.K - 1) break;
                int got = 0, cb = 0;
                if (lane == 0) {
                    atomicAdd(syncword(A.ctl), 1ULL);
                    __threadfence();   // the in-progress count is visible before the claim is
                    if (atomicCAS(&A.nstate[bi], ST_FREE, ST_CLAIMED) == ST_FREE) {
                        cb = atomicAdd(&A.ctl[B_NALLOC], 2);
                        got = 1;
                        if (cb + 2 > A.maxn) {
                            atomicExch(&A.ctl[B_ABORT], 1);
                            got = 0;
                        }
                    } else {
                        atomicAdd(syncword(A.ctl), ~0ULL);   // in progress - 1 (no borrow: it was incremented)
                    }
                }
                got = __shfl_sync(0xffffffffu, got, 0);
                cb = __shfl_sync(0xffffffffu, cb, 0);
                if (got) return {bi, cb};
                lost = true;
            }
            if (!skipped) break;
        }
        if (mode != 2) return {-1, 0};   // modes 1, 3: no waiting
        if (lost) continue;   // lost races: rescan at once
        int done = 0;
        if (lane == 0) {
            const unsigned long long sw = ld_acq64(A.ctl);
            done = ((unsigned)sw == 0u && (int)(sw >> 32) == ver0) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, done, 0)) return {-1, 0};
        // wait for the next publication (or for the in-progress count to reach 0) before rescanning
        if (lane == 0) {
            for (int spin = 0; spin < 4096; spin++) {
                const unsigned long long sw = ld_acq64(A.ctl);
                if ((int)(sw >> 32) != ver0 || (unsigned)sw == 0u || ld_acq(&A.ctl[B_ABORT])) break;
                __nanosleep(backoff);
                backoff = min(2 * backoff, 256);
            }
        }
        __syncwarp();
    }
}

HDF_DEV Claim claim_node(const BisectArgs& A, int mode, long long bigcap, int wid, long long maxm = LLONG_MAX) {
    return A.maxn > 512 ? claim_node_t<32>(A, mode, bigcap, wid, maxm) : claim_node_t<16>(A, mode, bigcap, wid, maxm);
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
    if (tid < 32) {   // the split set's algorithmic work (bench roofline): sum m * passes, sum m
        unsigned long long pp = 0, pm = 0;
        for (int i = tid; i < n; i += 32)
            if (inS[i]) {
                const unsigned long long mi = (unsigned long long)__ldcg(&A.nm[i]);
                pp += mi * (unsigned long long)__ldcg(&A.nit[i]);
                pm += mi;
            }
        for (int o = 16; o > 0; o >>= 1) {
            pp += __shfl_xor_sync(0xffffffffu, pp, o);
            pm += __shfl_xor_sync(0xffffffffu, pm, o);
        }
        if (tid == 0) {
            *reinterpret_cast<unsigned long long*>(&A.ctl[B_PTPASS]) = pp;
            *reinterpret_cast<unsigned long long*>(&A.ctl[B_PTSPLIT]) = pm;
        }
    }
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
        A.ctl[B_NOTDONE] = s_cnt[1];
        A.ctl[B_STATUS] = status;
        A.ctl[B_ACH] = ach;
    }
}

// --------------------------------------------------------------------------------- kernel -----
// Instantiated per RHO in inst_bisect.cu (one translation unit each); the host code gets the
// launchable pointers from these accessors.
using BisectFn = void (*)(const BisectArgs);
BisectFn bisect_kernel_rho0();
BisectFn bisect_kernel_rho1();
BisectFn bisect_kernel_rho2();
BisectFn bisect_kernel_rho3();
BisectFn bisect_kernel_rho4();
BisectFn bisect_kernel_rho5();
BisectFn bisect_kernel_rho6();
BisectFn bisect_kernel_rho7();

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
        mbar_init(&S.xbar[0], 1);
        mbar_init(&S.xbar[1], 1);
        mbar_init(&S.gbar[0], 1);
        mbar_init(&S.gbar[1], 1);
        mbar_init(&S.bbar, 1);
        fence_barrier_init();
        S.tma_phase = 0;
    }
    cg::this_cluster().sync();   // the exchange mbarriers are initialised before any peer signals them
    const bool b0 = (blockIdx.x == 0 && tid == 0);
    if (b0 && A.trace) {   // (the counter is zeroed below; event 0 is written at slot 0 directly)
        A.trace[1] = 30;
        A.trace[2] = gtimer();
    }
    // ---- init: node table, root statistics (mean, SSE) in a fixed order ----
    for (long long i = gtid; i < A.maxn; i += gth) A.nstate[i] = ST_NONE;
    for (long long i = gtid; i < (long long)2 * G * kRecV * 2; i += gth) A.xw[i] = 0ull;
    if (gtid < B_NUM) A.ctl[gtid] = (gtid == B_TRACE_N && A.trace) ? 1 : 0;
    const long long per = ((long long)A.N + G - 1) / G;
    const long long rb0 = min((long long)A.N, (long long)blockIdx.x * per), rb1 = min((long long)A.N, rb0 + per);
    double* rec0 = A.rec;
    double* rec1 = A.rec + (size_t)G * kRecV;
    // Pass 1 over the CTA's contiguous range: per dimension the fp64 sum, max p_d and max -p_d
    // (record: rec0 [0, rho) sums, [HDF_MAX_RHO, +rho) max p_d; rec1 [0, rho) max -p_d).
    for (int d0 = 0; d0 < rho; d0 += 8) {
        constexpr int UP = 4;   // points per thread in flight
        double acc[8];
        float hi[8], nlo[8];
#pragma unroll
        for (int j = 0; j < 8; j++) { acc[j] = 0.0; hi[j] = -INFINITY; nlo[j] = -INFINITY; }
        for (long long t0 = rb0 + tid; t0 < rb1; t0 += UP * kBT) {
            float x[UP][8];
#pragma unroll
            for (int u = 0; u < UP; u++) {
                const long long t = t0 + (long long)u * kBT;
#pragma unroll
                for (int j = 0; j < 8; j++) x[u][j] = (t < rb1 && d0 + j < rho) ? __ldg(A.p + t * rho + d0 + j) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < UP; u++) {
                if (t0 + (long long)u * kBT < rb1) {
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        acc[j] += (double)x[u][j];
                        hi[j] = fmaxf(hi[j], x[u][j]);
                        nlo[j] = fmaxf(nlo[j], -x[u][j]);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++)
            for (int o = 16; o > 0; o >>= 1) {
                hi[j] = fmaxf(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], o));
                nlo[j] = fmaxf(nlo[j], __shfl_xor_sync(0xffffffffu, nlo[j], o));
            }
        double av[8];
#pragma unroll
        for (int j = 0; j < 8; j++) av[j] = acc[j];
        const int vi = warp_reduce_scatter<8>(av);
        if ((tid & 3) == 0) S.red[(tid >> 5) * 16 + vi] = av[0];
        if ((tid & 31) == 0)
#pragma unroll
            for (int j = 0; j < 4; j++) {   // hi and nlo packed as float pairs
                S.red[(tid >> 5) * 16 + 8 + j] = __hiloint2double(__float_as_int(hi[2 * j + 1]), __float_as_int(hi[2 * j]));
                S.red[(tid >> 5) * 16 + 12 + j] =
                    __hiloint2double(__float_as_int(nlo[2 * j + 1]), __float_as_int(nlo[2 * j]));
            }
        __syncthreads();
        if (tid < 8 && d0 + tid < rho) {
            double sm = 0.0;
            float h = -INFINITY, nl = -INFINITY;
            for (int w = 0; w < kBW; w++) {
                sm += S.red[w * 16 + tid];
                const double hp = S.red[w * 16 + 8 + tid / 2], np = S.red[w * 16 + 12 + tid / 2];
                h = fmaxf(h, __int_as_float((tid & 1) ? __double2hiint(hp) : __double2loint(hp)));
                nl = fmaxf(nl, __int_as_float((tid & 1) ? __double2hiint(np) : __double2loint(np)));
            }
            rec0[(size_t)blockIdx.x * kRecV + d0 + tid] = sm;
            rec0[(size_t)blockIdx.x * kRecV + HDF_MAX_RHO + d0 + tid] = (double)h;
            rec1[(size_t)blockIdx.x * kRecV + d0 + tid] = (double)nl;
        }
        __syncthreads();
    }
    __threadfence();
    grid.sync();
    if (tid == 0 && blockIdx.x == 0) {
        A.ctl[B_NALLOC] = 1;
        A.ctl[B_TASK] = -1;
    }
    // Every CTA gathers the G records, all loads in flight: quantity e (sum_d, max p_d, max -p_d) is
    // reduced by one warp, lanes over blocks then a fixed butterfly (bit-identical in every CTA).
    {
        const int lane = tid & 31, warp = tid >> 5;
        for (int e = warp; e < 3 * rho; e += kBW) {
            const int kind = e / rho, d = e - kind * rho;
            const double* src = (kind == 2) ? rec1 + d : rec0 + (kind == 1 ? HDF_MAX_RHO : 0) + d;
            double v = (kind == 0) ? 0.0 : -INFINITY;
            for (int b = lane; b < G; b += 32) {
                const double x = __ldcg(src + (size_t)b * kRecV);
                v = (kind == 0) ? v + x : fmax(v, x);
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double y = __shfl_xor_sync(0xffffffffu, v, o);
                v = (kind == 0) ? v + y : fmax(v, y);
            }
            if (lane == 0) {
                if (kind == 0) S.c0[d] = v / (double)A.N;
                else if (kind == 1) S.c1[d] = v;     // max p_d (staged)
                else S.tot[d] = v;                   // max -p_d (staged)
            }
        }
    }
    __syncthreads();
    bool constant = true;
    for (int d = 0; d < rho; d++) constant = constant && (S.c1[d] == -S.tot[d]);
    __syncthreads();
    for (int d = tid; d < rho; d += kBT) S.xmax[d] = (float)fmax(S.c1[d], S.tot[d]);
    // The root's SSE is only compared with its descendants' (it is the largest unless the guide is
    // constant, then 0) and enters E_K only when the root stays a leaf: a constant guide (0) or K = 1,
    // where pass 2 computes it in a fixed order.
    double root_sse = constant ? 0.0 : INFINITY;
    if (A.K == 1 && !constant) {
        __syncthreads();
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; j++) acc[j] = 0.0;
        for (long long t = rb0 + tid; t < rb1; t += kBT) acc[0] += dist_rn(A.p + t * rho, S.c0, rho);
        const int vi = warp_reduce_scatter<8>(acc);
        if ((tid & 3) == 0) S.red[(tid >> 5) * 16 + vi] = acc[0];
        __syncthreads();
        if (tid == 0) {
            double sm = 0.0;
            for (int w = 0; w < kBW; w++) sm += S.red[w * 16];
            rec1[(size_t)blockIdx.x * kRecV + HDF_MAX_RHO + 8] = sm;
        }
        __threadfence();
        grid.sync();
        if (blockIdx.x == 0 && tid == 0) {
            double sm = 0.0;
            for (int b = 0; b < G; b++) sm += __ldcg(rec1 + (size_t)b * kRecV + HDF_MAX_RHO + 8);
            root_sse = sm;
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        A.nsse[0] = root_sse;
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

    if (b0) trace_ev(A, 31, 0, 0);
    // ---- phase 1: nodes too large for one cluster, split by the whole grid ----
    cg::cluster_group cl = cg::this_cluster();
    const long long ccap = min(A.ccap, (long long)cl.num_blocks() * A.cap);
    // grid mode above gabove; a cluster streams at most its CTAs' side-word scratch
    const long long gab = max(ccap, min(A.gabove, (long long)cl.num_blocks() * 32LL * (A.wcap - 2)));
    {
        // Rounds: block 0 claims every claimable node larger than gab (best first) and gives each a
        // team of consecutive clusters, in proportion to its size (at least one); the teams split
        // their nodes concurrently (tagged-word exchanges inside the team), then the grid syncs.
        const int nclg = G / (int)cl.num_blocks(), cidg = (int)(blockIdx.x / cl.num_blocks());
        int round = 0;
        uint32_t gph = 0;   // phase bits of this CTA's S.gbar, carried across rounds (the barriers persist)
        while (A.N > gab) {   // (no node needs the grid otherwise)
            if (blockIdx.x == 0 && tid < 32) {
                // The best node first; then only nodes that fit resident in the clusters still free
                // (a streamed node is bandwidth-bound: splitting the grid would only slow it down).
                // Each team gets the clusters its node needs resident; the rest go round robin.
                int nt = 0, need = 0;
                int tk[kTeamMax], tcb[kTeamMax], tcl[kTeamMax];
                while (nt < min(nclg, kTeamMax) && need < nclg) {
                    const long long lim = nt == 0 ? LLONG_MAX : (long long)(nclg - need) * ccap;
                    const Claim c = claim_node(A, 1, gab, 0, lim);
                    if (c.task < 0) break;
                    const long long mi = __ldcg(&A.nm[c.task]);
                    tk[nt] = c.task;
                    tcb[nt] = c.cbase;
                    tcl[nt] = (int)min((long long)nclg, (mi + ccap - 1) / ccap);
                    need += tcl[nt];
                    nt++;
                }
                if (tid == 0) {
                    int used = 0;
                    for (int i = 0; i < nt; i++) used += tcl[i];
                    for (int i = 0; used < nclg && nt > 0; i = (i + 1) % nt, used++) tcl[i]++;
                    int c = 0;
                    for (int i = 0; i < nt; i++) {
                        A.teams[i * 5 + 0] = tk[i];
                        A.teams[i * 5 + 1] = tcb[i];
                        A.teams[i * 5 + 2] = c;
                        A.teams[i * 5 + 3] = tcl[i];
                        for (int q = 0; q < tcl[i]; q++) A.teams[kTeamMax * 5 + c + q] = i;
                        c += tcl[i];
                    }
                    A.ctl[B_TASK] = nt;
                    __threadfence();
                }
            }
            grid.sync();
            const int nt = __ldcg(&A.ctl[B_TASK]);
            if (nt <= 0) break;
            const int ti = __ldcg(&A.teams[kTeamMax * 5 + cidg]);
            const int task = __ldcg(&A.teams[ti * 5 + 0]), cb = __ldcg(&A.teams[ti * 5 + 1]);
            const int tc0 = __ldcg(&A.teams[ti * 5 + 2]), tn = __ldcg(&A.teams[ti * 5 + 3]);
            GridGrp gg{(cidg - tc0) * (int)cl.num_blocks() + (int)cl.block_rank(), tn * (int)cl.num_blocks(),
                       (int)cl.block_rank(), (int)cl.num_blocks(), cidg, tn, A.xw, A.ctl};
            gg.c0 = tc0;
            gg.nclg = nclg;
            gg.tagbase = (uint32_t)(round * kTeamMax + ti + 1) << 16;   // unique per team formation
            gg.gph = gph;
            split_node<RHO>(A, gg, S, io, task, cb, -1 - ti);
            gph = gg.gph;
            round++;
            grid.sync();
        }
    }

    if (b0) trace_ev(A, 32, 0, 0);
    // ---- phase 2: nodes larger than one CTA's tile; every thread-block cluster is a worker ----
    if (cl.num_blocks() > 1) {
        const int worker = blockIdx.x / (int)cl.num_blocks();
        auto run = [&](auto& g) {
            while (true) {
                if (g.rank == 0 && tid < 32) {
                    if (tid == 0) trace_ev(A, 1, 0, worker);
                    const Claim c = claim_node(A, 2, A.ctamax, worker);
                    if (tid == 0) { S.task = c.task; S.cbase = c.cbase; }
                }
                cl.sync();
                const int task = *cl.map_shared_rank(&S.task, 0);
                const int cb = *cl.map_shared_rank(&S.cbase, 0);
                cl.sync();
                if (task < 0) break;
                split_node<RHO>(A, g, S, io, task, cb, worker);
            }
        };
        if (RHO > 0) {
            // Cluster batches.  The cluster's rank 0 claims the best node; a node of at most qmax points
            // turns the cluster into groups of 4 CTAs (at most ctamax points: single CTAs) for this
            // batch, and rank 0 claims up to one node per group (no waiting).  A group that finishes
            // its node claims another one of at most its size limit (no waiting) and stops when there
            // is none; the cluster regroups when every group has stopped.
            const int cdim = (int)cl.num_blocks(), crank = (int)cl.block_rank();
            uint32_t ph = 0;
            while (true) {
                if (crank == 0 && tid < 32) {
                    if (tid == 0) trace_ev(A, 1, 0, worker);
                    const Claim c0 = claim_node(A, 2, 1, worker * 16);
                    int gsz = cdim, nt = 0;
                    int tk[16], cb[16];
                    if (c0.task >= 0) {
                        const int m0 = __ldcg(&A.nm[c0.task]);
                        if (m0 <= A.ctamax) gsz = 1;
                        else if (m0 <= A.qmax && cdim >= 4) gsz = 4;
                        tk[0] = c0.task;
                        cb[0] = c0.cbase;
                        nt = 1;
                        const long long lim = gsz == 1 ? A.ctamax : A.qmax;
                        for (int q = 1; q < cdim / gsz; q++) {
                            const Claim c = claim_node(A, 3, 1, worker * 16 + q, lim);
                            if (c.task < 0) break;
                            tk[q] = c.task;
                            cb[q] = c.cbase;
                            nt++;
                        }
                    } else {
                        tk[0] = -1;
                        cb[0] = 0;
                    }
                    // to every CTA of the cluster
                    for (int r = 0; r < cdim; r++) {
                        SplitSm* R = cl.map_shared_rank(&S, r);
                        if (tid == 0) { R->bn = nt; R->bgran = gsz; }
                        if (tid < 16) {
                            R->btask[tid] = (tid < nt) ? tk[tid] : -1;
                            R->bcb[tid] = (tid < nt) ? cb[tid] : 0;
                        }
                    }
                }
                cl.sync();
                const int gsz = S.bgran, gi = crank / gsz;
                int task = S.btask[gi], cbt = S.bcb[gi];
                const bool done = S.btask[0] < 0;
                if (done) break;
                PushGrp g{crank - gi * gsz, gsz, ph, gi * gsz};
                const long long lim = gsz == 1 ? A.ctamax : A.qmax;
                while (task >= 0) {
                    split_node<RHO>(A, g, S, io, task, cbt, worker * 16 + gi);
                    if (gsz == cdim) break;   // a whole-cluster node: back to the batch level
                    int nt = -1, nc = 0;
                    if (g.rank == 0 && tid < 32) {
                        const Claim c = claim_node(A, 3, 1, worker * 16 + gi, lim);
                        nt = c.task;
                        nc = c.cbase;
                    }
                    if (gsz == 1) {
                        if (tid == 0) { S.task = nt; S.cbase = nc; }
                        __syncthreads();
                        task = S.task;
                        cbt = S.cbase;
                        __syncthreads();
                    } else {
                        nt = __shfl_sync(0xffffffffu, nt, 0);
                        nc = __shfl_sync(0xffffffffu, nc, 0);
                        const int2 tc = g.bcast(S, nt, nc);   // (rank 0: lanes < gsz hold the values)
                        task = tc.x;
                        cbt = tc.y;
                    }
                }
                ph = g.ph;
                cl.sync();   // the batch ends when every group has stopped
            }
        } else {
            ClusterGrp g{(int)cl.block_rank(), (int)cl.num_blocks()};
            run(g);
        }
    }
    // ---- phase 3: every CTA is a worker (only needed when phase 2 left small nodes: rho > 7, or no
    //      thread-block clusters); with cluster batches phase 2 has split every node already ----
    const bool phase3 = !(RHO > 0 && cl.num_blocks() > 1);
    if (phase3) {
        __threadfence();
        grid.sync();
    }
    if (b0) trace_ev(A, 33, 0, 0);
    if (phase3) {
        CtaGrp g;
        const int worker = 1000 + blockIdx.x;
        while (true) {
            if (tid < 32) {
                if (tid == 0) trace_ev(A, 1, 0, worker);
                const Claim c = claim_node(A, 2, 0, blockIdx.x);
                if (tid == 0) { S.task = c.task; S.cbase = c.cbase; }
            }
            __syncthreads();
            const int task = S.task, cb = S.cbase;
            __syncthreads();
            if (task < 0) break;
            split_node<RHO>(A, g, S, io, task, cb, worker);
        }
    }
    __threadfence();
    grid.sync();

    // ---- phase 4: split set, leaf ids, centres, E_K, labels ----
    if (b0) trace_ev(A, 34, 0, 0);
    if (blockIdx.x == 0) finalise(A, dsm);
    if (b0) trace_ev(A, 35, 0, 0);
    __threadfence();
    grid.sync();
    if (A.labels) {
        // Pixel labels.  Every leaf of the computed tree (a node never split) holds its members at
        // positions [nstart, nstart + nm) of buffer nbuf (no later partition writes there), and its
        // label is nfinal.  A CTA walks a contiguous range of positions (index reads coalesced over
        // the threads) and finds the leaf covering a position by descending from the root over the
        // node table staged in shared memory, reusing it while the position stays inside.
        const int n = min(__ldcg(&A.ctl[B_NALLOC]), A.maxn);
        int* tst = reinterpret_cast<int*>(dsm);
        int* tch = tst + n;
        int* tsa = tch + n;
        int* tnm = tsa + n;
        int* tbf = tnm + n;
        int* tfn = tbf + n;
        for (int i = tid; i < n; i += kBT) {
            tst[i] = __ldcg(&A.nstate[i]);
            tch[i] = __ldcg(&A.nchild[i]);
            tsa[i] = __ldcg(&A.nstart[i]);
            tnm[i] = __ldcg(&A.nm[i]);
            tbf[i] = __ldcg(&A.nbuf[i]);
            tfn[i] = __ldcg(&A.nfinal[i]);
        }
        __syncthreads();
        long long ls = 0, le = 0;
        int lb = kBufInput, lf = 0;
        for (long long j = rb0 + tid; j < rb1; j += kBT) {
            if (j < ls || j >= le) {
                int v = 0;
                while (tst[v] == ST_DONE) {
                    const int c = tch[v];
                    v = (j < tsa[c + 1]) ? c : c + 1;
                }
                ls = tsa[v];
                le = ls + tnm[v];
                lb = tbf[v];
                lf = tfn[v];
            }
            const long long pix = (lb == kBufInput) ? j : (long long)__ldcg(A.idx[lb] + j);
            A.labels[pix] = lf;
        }
    }
}

}  // namespace hdf
