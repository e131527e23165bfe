// hdf_api.cu -- the C ABI (include/hdf.h): argument checking, workspace carving, launches.
// Every arithmetic step of the hot path runs in this library's kernels; there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hdf_dispatch.h"
#include "k_bisect.cuh"
#include "k_coeffs.cuh"
#include "k_coeffs_tc.cuh"
#include "k_vpass_tc.cuh"
#include "k_hpass_tc.cuh"
#include "k_guide.cuh"
#include "k_iir.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define HDF_CUDA(call)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(HDF_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Bump allocator over the caller's workspace (256-byte aligned slices).  With base == nullptr it
// only measures.
struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += sizeof(T) * count;
        return p;
    }
};

int round_up(int a, int b) { return (a + b - 1) / b * b; }

// No C++ exception crosses the C ABI: every entry point runs its body through guarded().
template <class Fn>
int guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::exception& e) {
        return fail(HDF_ERR_CUDA, "internal exception: %s", e.what());
    } catch (...) {
        return fail(HDF_ERR_CUDA, "internal exception");
    }
}
template <class Fn>
size_t guarded_size(Fn&& fn) {
    try {
        return fn();
    } catch (...) {
        return 0;
    }
}

// ------------------------------------------------------------------ per-stage event profiling ----
// When enabled (hdf_profile_enable), every stage records a start/end CUDA event pair on the call's
// stream; hdf_profile_collect() waits for them and returns the summed device time per stage.
struct ProfRec {
    int stage;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_pending;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    ProfRec r;
    cudaStream_t st;
    bool on;
    ProfScope(int stage, cudaStream_t s) : st(s) {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        on = g_prof_on;
        if (on) {
            r.stage = stage;
            r.a = prof_event();
            r.b = prof_event();
            cudaEventRecord(r.a, st);
        }
    }
    void close() {
        if (!on) return;
        on = false;
        cudaEventRecord(r.b, st);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof_pending.push_back(r);
    }
    ~ProfScope() { close(); }
};

// ------------------------------------------------------------------------ cluster workspace ----
// k_bisect (k_bisect.cuh) works in a caller-provided workspace: two ping-pong copies of the guide
// and its pixel index, grid-mode side words and exchange records, the node table.
constexpr int kBisectMaxGrid = 256;     // upper bound of the cooperative grid (records, side words)
constexpr int kBisectMinGrid = 32;      // the launch never uses fewer CTAs (streamed ranges <= N / 32)
// Node table: the K-1 splits need 2K-1 nodes; speculative splits need room too.  Claim scans hold
// the table in registers (16 or 32 entries per lane).
int bisect_maxn(int K) { return K > 64 ? 1024 : 512; }

hdf::BisectArgs carve_cluster(Carver& cv, const float* p, int H, int W, int rho, int K) {
    const long long N = (long long)H * W;
    hdf::BisectArgs A;
    memset(&A, 0, sizeof(A));
    A.p = p;
    A.N = (int)N;
    A.rho = rho;
    A.K = K;
    A.maxn = bisect_maxn(K);
    A.wcap = (int)((N + (long long)kBisectMinGrid * 32 - 1) / ((long long)kBisectMinGrid * 32)) + 2;
    for (int b = 0; b < 2; b++) {
        A.ptsw[b] = cv.take<float>((size_t)N * rho + 16);
        A.pts[b] = A.ptsw[b];
    }
    A.pts[hdf::kBufInput] = p;
    for (int b = 0; b < 2; b++) A.idx[b] = cv.take<int>((size_t)N);
    A.sidew = cv.take<uint32_t>((size_t)kBisectMaxGrid * 2 * A.wcap);
    A.rec = cv.take<double>((size_t)2 * kBisectMaxGrid * hdf::kRecV);
    A.nsse = cv.take<double>(A.maxn);
    A.nm = cv.take<int>(A.maxn);
    A.nstart = cv.take<int>(A.maxn);
    A.nstate = cv.take<int>(A.maxn);
    A.nparent = cv.take<int>(A.maxn);
    A.nchild = cv.take<int>(A.maxn);
    A.nbuf = cv.take<int>(A.maxn);
    A.nit = cv.take<int>(A.maxn);
    A.nmean = cv.take<double>((size_t)A.maxn * rho);
    A.nfinal = cv.take<int>(A.maxn);
    A.ctl = cv.take<int>(hdf::B_NUM);
    A.trace = cv.take<long long>(1 + 2 * hdf::kBisectTraceCap);
    A.ek = cv.take<double>(1);
    A.xw = cv.take<unsigned long long>((size_t)2 * kBisectMaxGrid * hdf::kRecV * 2);
    A.teams = cv.take<int>((size_t)hdf::kTeamMax * 5 + kBisectMaxGrid);
    return A;
}

// Dynamic shared memory of k_bisect for a tile of `cap` points: the tile (cap * rho + 8 floats),
// two side-word buffers, the stride sample (rho <= kSampRho).
size_t bisect_dyn_smem(int rho, int cap) {
    const size_t x = (((size_t)cap * rho + 8) * 4 + 15) / 16 * 16;
    const size_t w = 2 * ((size_t)cap / 32 + 2) * 4;
    const size_t smp = rho <= hdf::kSampRho ? (size_t)hdf::kFpCap * rho * 4 : 0;
    return x + w + smp;
}

using BisectKernel = hdf::BisectFn;
BisectKernel bisect_kernel(int rho) {
    switch (rho) {
        case 1: return hdf::bisect_kernel_rho1();
        case 2: return hdf::bisect_kernel_rho2();
        case 3: return hdf::bisect_kernel_rho3();
        case 4: return hdf::bisect_kernel_rho4();
        case 5: return hdf::bisect_kernel_rho5();
        case 6: return hdf::bisect_kernel_rho6();
        case 7: return hdf::bisect_kernel_rho7();
        default: return hdf::bisect_kernel_rho0();
    }
}

int check_common(int H, int W, int rho, int K) {
    if (H < 1 || W < 1) return fail(HDF_ERR_ARG, "H, W must be >= 1 (got %d, %d)", H, W);
    if ((long long)H * W > (1LL << 30)) return fail(HDF_ERR_ARG, "H*W too large");
    if (rho < 1 || rho > HDF_MAX_RHO) return fail(HDF_ERR_ARG, "rho must be in [1, %d] (got %d)", HDF_MAX_RHO, rho);
    if (K < 1 || K > HDF_MAX_K) return fail(HDF_ERR_ARG, "K must be in [1, %d] (got %d)", HDF_MAX_K, K);
    return HDF_OK;
}

bool misaligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; }

// Cluster size of the phase-2 workers (HDF_BISECT_CLUSTER=16|8|4|2 overrides; default 16 when the
// device keeps enough 16-CTA clusters resident, else 8).
int env_cluster_dim() {
    const char* e = getenv("HDF_BISECT_CLUSTER");
    return e ? atoi(e) : 0;
}

// The clustering launch shape (cached per rho): one 512-thread CTA per SM with the largest tile that
// fits, in a cooperative grid of thread-block clusters.
struct ClusterShape {
    int cdim, nclusters, cap;
    size_t smem;
};

// Per-thread pinned host words that the calls with *_host outputs read back into: the clustering's
// control words and E_K, the filter's status and flag count.  Pinned, so that the read-backs are
// enqueued asynchronously and read after the call's one final synchronisation (a read into pageable
// memory would block the host mid-call).  Allocated on first use (a few hundred bytes of pinned host
// memory per calling thread, never freed); the library allocates no device memory.
struct HostStage {
    int ctrl[hdf::B_NUM];
    double ek;
    int hv[2];   // filter: A^+ status, number of flagged pixels
};
HostStage* host_stage() {
    static thread_local HostStage* hs = nullptr;
    if (!hs) {
        void* p = nullptr;
        if (cudaMallocHost(&p, sizeof(HostStage)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        hs = static_cast<HostStage*>(p);
    }
    return hs;
}

// The clustering kernel's control words and E_K in the calling thread's pinned stage, read back
// with the caller's final synchronisation.
struct ClusterReadback {
    HostStage* hs = nullptr;
    ClusterShape sh;
};

// Status of a finished clustering from its control words; fills info (may be NULL).
int cluster_status(const ClusterReadback& rb, int K, hdf_cluster_info* info) {
    const int* ctrl = rb.hs->ctrl;
    if (info) {
        memset(info, 0, sizeof(*info));
        info->launch_ctas = (int)(rb.sh.cdim * rb.sh.nclusters);
        info->cluster_ctas = rb.sh.cdim;
        info->status = ctrl[hdf::B_STATUS];
        info->achievable_k = ctrl[hdf::B_ACH];
        info->splits_computed = ctrl[hdf::B_SPLITS];
        info->lloyd_iters = ctrl[hdf::B_ITERS];
        info->grid_splits = ctrl[hdf::B_GRIDSPLITS];
        unsigned long long pp, pm;
        memcpy(&pp, &ctrl[hdf::B_PTPASS], 8);
        memcpy(&pm, &ctrl[hdf::B_PTSPLIT], 8);
        info->point_passes = (int64_t)pp;
        info->points_split = (int64_t)pm;
        info->tile_points = rb.sh.cap;
        info->e_k = rb.hs->ek;
    }
    if (ctrl[hdf::B_STATUS] == HDF_ERR_CUDA)
        return fail(HDF_ERR_CUDA,
                    "clustering kernel: internal error (abort %d, nodes %d, splits %d, not done %d, diag %d %d %d %d "
                    "%d %d)",
                    ctrl[hdf::B_ABORT], ctrl[hdf::B_NALLOC], ctrl[hdf::B_SPLITS], ctrl[hdf::B_NOTDONE],
                    ctrl[hdf::B_DIAG0], ctrl[hdf::B_DIAG1], ctrl[hdf::B_DIAG2], ctrl[hdf::B_DIAG3], ctrl[hdf::B_DIAG4],
                    ctrl[hdf::B_DIAG5]);
    if (ctrl[hdf::B_STATUS] == HDF_ERR_K)
        return fail(HDF_ERR_K, "K=%d exceeds the number of distinct guide vectors (%d)", K, ctrl[hdf::B_ACH]);
    return HDF_OK;
}

// Launch the clustering.  info != NULL: read the result back now (synchronises `st`).  rb != NULL:
// enqueue the read-back into *rb (which must stay alive until the caller synchronises `st`).
int launch_cluster(const float* p, int H, int W, int rho, int K, float* centres, int32_t* labels,
                   hdf_cluster_info* info, void* ws, cudaStream_t st, ClusterReadback* rb = nullptr) {
    Carver cv(ws);
    hdf::BisectArgs A = carve_cluster(cv, p, H, W, rho, K);
    A.centres = centres;
    A.labels = labels;
    BisectKernel kern = bisect_kernel(rho);
    using Shape = ClusterShape;
    static std::mutex mu;
    static Shape cache[17][HDF_MAX_RHO + 1];   // by requested cluster size (0 = default) and rho
    Shape sh;
    {
        std::lock_guard<std::mutex> lk(mu);
        sh = cache[std::min(std::max(env_cluster_dim(), 0), 16)][rho];
        if (sh.cdim == 0) {
            int dev = 0, optin = 0;
            HDF_CUDA(cudaGetDevice(&dev));
            HDF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            cudaFuncAttributes fa;
            HDF_CUDA(cudaFuncGetAttributes(&fa, kern));
            const long long budget = (long long)optin - (long long)fa.sharedSizeBytes;
            int cap = 0;
            for (int c = 512; ; c += 512) {
                if ((long long)bisect_dyn_smem(rho, c) > budget) break;
                cap = c;
            }
            if (cap == 0) return fail(HDF_ERR_CUDA, "clustering kernel: no shared-memory tile fits");
            const size_t smem = bisect_dyn_smem(rho, cap);
            HDF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            HDF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            const int want = env_cluster_dim();
            for (int cdim : {16, 8, 4, 2, 1}) {
                if (want > 0 && cdim != want) continue;
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cdim;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3(cdim);
                cfg.blockDim = dim3(hdf::kBT);
                cfg.dynamicSmemBytes = smem;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg) != cudaSuccess) {
                    cudaGetLastError();
                    ncl = 0;
                }
                ncl = std::min(ncl, kBisectMaxGrid / cdim);
                if (ncl * cdim >= std::max(kBisectMinGrid, 96) || (want > 0 && ncl * cdim >= kBisectMinGrid)) {
                    sh.cdim = cdim;
                    sh.nclusters = ncl;
                    break;
                }
            }
            if (sh.cdim == 0) return fail(HDF_ERR_CUDA, "no resident launch shape for the clustering kernel");
            sh.cap = cap;
            sh.smem = smem;
            cache[std::min(std::max(env_cluster_dim(), 0), 16)][rho] = sh;
        }
    }
    A.cap = sh.cap;
    A.ccap = (long long)sh.cdim * sh.cap;
    {   // worker trace (diagnostics, hdf_cluster_trace): off unless HDF_BISECT_TRACE=1
        const char* e = getenv("HDF_BISECT_TRACE");
        if (!(e && atoi(e) != 0)) A.trace = nullptr;
    }
    // Grid mode above max(a cluster's shared memory, N / 5): a node of up to N / 5 points streams
    // through one cluster's shared memory instead of taking the whole grid, so several such nodes
    // split concurrently (measured: c5 14.9 -> 12.3 ms, c3 5.3 -> 4.8 ms; N / 4 and above: more
    // speculative splits, c5 13.2 ms; c1, c2a, c2b, c4 are unchanged: their cluster capacity is larger)
    A.gabove = std::max<long long>(A.ccap, (long long)A.N / 5);
    if (const char* e = getenv("HDF_BISECT_GRID_ABOVE")) {   // may lower (cluster capacity too) or raise it
        A.gabove = std::max<long long>(1, atoll(e));
        A.ccap = std::min<long long>(A.ccap, A.gabove);
    }
    A.ctamax = std::min<long long>(A.cap, 2048);   // smaller nodes: one CTA each (measured best on c2b)
    if (const char* e = getenv("HDF_BISECT_CTA_MAX")) A.ctamax = std::min<long long>(A.cap, atoll(e));
    // groups of 4 CTAs for nodes of at most qmax points (cluster batches): with K >= 64 the tree has enough
    // ready mid-size nodes to keep 4x more group workers busy (the sampled c5 input, 262k points: 0.86 ->
    // 0.74-0.76 ms, qmax 16k-32k); with K = 32 they only add speculative splits (c2b 0.50 -> 0.54 ms, c4
    // 0.66 -> 0.71 ms), so they stay off there
    A.qmax = K >= 64 ? std::min<long long>(4LL * A.cap, 32768) : 0;
    if (const char* e = getenv("HDF_BISECT_QUAD_MAX")) A.qmax = std::min<long long>(4LL * A.cap, atoll(e));
    {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = sh.cdim;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.gridDim = dim3(sh.cdim * sh.nclusters);
        cfg.blockDim = dim3(hdf::kBT);
        cfg.dynamicSmemBytes = sh.smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        ProfScope prof(HDF_STAGE_CLUSTER, st);
        HDF_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    }
    ClusterReadback local;
    ClusterReadback* r = rb ? rb : (info ? &local : nullptr);
    if (r) {
        r->sh = sh;
        r->hs = host_stage();
        if (!r->hs) return fail(HDF_ERR_CUDA, "pinned host stage: cudaMallocHost failed");
        HDF_CUDA(cudaMemcpyAsync(r->hs->ctrl, A.ctl, sizeof(r->hs->ctrl), cudaMemcpyDeviceToHost, st));
        HDF_CUDA(cudaMemcpyAsync(&r->hs->ek, A.ek, sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    if (info && !rb) {
        HDF_CUDA(cudaStreamSynchronize(st));
        return cluster_status(local, K, info);
    }
    return HDF_OK;
}

// ------------------------------------------------------------------------- filter planning -----
int padded_radius(int R, bool box) {
    for (int i = 0; i < hdf::kNumRadii; i++) {
        if (box && hdf::kRadii[i] == R) return R;
        if (!box && hdf::kRadii[i] >= R) return hdf::kRadii[i];
    }
    return -1;
}

struct FilterPlan {
    int R, Rp, Wp, NP, P;
    bool box;
    bool iir;   // HDF_SPATIAL_GAUSSIAN_IIR: identity taps in the passes, the recursion in between
    int Rfb;    // the R9 fallback's window radius (= R for the FIR kinds)
    // F1
    hdf::VLaunch vl;
    int Pg, TY;
    // F2
    hdf::HLaunch hl;
    int RR, NJW, NWC, NS, Lbox, stage_bytes, planes_bytes;
};

// the recursive Gaussian's R9 fallback window (a direct sum per flagged pixel, weights computed in place)
constexpr int kMaxFallbackRadius = 512;
// the recursive Gaussian's largest sigma_s (its anti-causal start matrix is simulated on the host over
// 60 sigma_s + 100 samples, iir_params)
constexpr float kMaxIirSigma = 4096.f;

int make_plan(int H, int W, int n, int K, int kind, float sigma_s, int radius, FilterPlan* fp, int nsm) {
    FilterPlan& F = *fp;
    F.box = (kind == HDF_SPATIAL_BOX);
    F.iir = (kind == HDF_SPATIAL_GAUSSIAN_IIR);
    if (kind != HDF_SPATIAL_GAUSSIAN && kind != HDF_SPATIAL_BOX && !F.iir)
        return fail(HDF_ERR_ARG, "unknown spatial kind %d", kind);
    F.Rfb = -1;
    if (F.iir) {   // the recursion replaces the FIR; radius only sizes the R9 fallback's window
        if (!(sigma_s >= 0.5f)) return fail(HDF_ERR_ARG, "the recursive Gaussian needs sigma_s >= 0.5");
        if (!(sigma_s <= kMaxIirSigma))
            return fail(HDF_ERR_ARG, "the recursive Gaussian needs sigma_s <= %g", (double)kMaxIirSigma);
        F.Rfb = radius >= 0 ? radius : (int)std::ceil(3.0 * (double)sigma_s);
        if (F.Rfb > kMaxFallbackRadius)
            return fail(HDF_ERR_ARG, "fallback radius %d exceeds %d", F.Rfb, kMaxFallbackRadius);
        radius = 0;
    }
    if (radius < 0) {
        if (F.box) return fail(HDF_ERR_ARG, "the box kernel needs an explicit radius");
        if (!(sigma_s > 0.f)) return fail(HDF_ERR_ARG, "sigma_s must be > 0");
        radius = (int)std::ceil(3.0 * (double)sigma_s);
    }
    if (!F.box && !(sigma_s > 0.f)) return fail(HDF_ERR_ARG, "sigma_s must be > 0");
    if (radius > HDF_MAX_RADIUS) return fail(HDF_ERR_ARG, "radius %d exceeds HDF_MAX_RADIUS=%d", radius, HDF_MAX_RADIUS);
    F.R = radius;
    if (!F.iir) F.Rfb = radius;
    // Running-sum box kernels need a compiled radius equal to S; any other box radius (and S = 0)
    // runs through the FIR kernels with unit taps on [-S, S] and zero taps beyond (exact).
    if (F.box && (radius == 0 || padded_radius(radius, true) < 0)) F.box = false;
    F.Rp = padded_radius(radius == 0 ? 1 : radius, F.box);
    if (F.Rp < 0) return fail(HDF_ERR_ARG, "radius %d is not supported by this build", radius);
    F.Wp = round_up(W, 32);   // (whole 32-column strips of the strip-major fp16 planes, k_hpass_tc.cuh)
    F.NP = n + 1;
    F.P = K * F.NP;
    // F1: planes per CTA; a persistent grid (one 512-thread CTA per SM) with equal shares of the
    // (strip, plane group) x rows space
    {
        const int npl = hdf::vfir_npl(hdf::vpass_pack(F.Rp), hdf::vpass_nt(F.Rp));
        F.Pg = npl;
        const long long gx = (W + hdf::kVTX - 1) / hdf::kVTX, gz = (F.P + npl - 1) / npl;
        F.TY = (int)gx;   // reused: number of strips
        const long long cols = gx * gz;
        F.vl.grid = dim3((unsigned)std::max(1LL, std::min<long long>(std::max(1, nsm - 1), cols * H)));
        F.vl.threads = hdf::vpass_nt(F.Rp);
        F.vl.smem = 0;   // depends on rho and on f aliasing p: set at launch
    }
    // F2
    const int NP = F.NP;
    int maxjp = 1;
    if (NP <= 7) { F.RR = 8; F.NJW = NP; }
    else if (NP <= 15) { F.RR = 4; F.NJW = NP; }
    else if (NP <= 31) { F.RR = 2; F.NJW = NP; }
    else if (NP <= 62) { F.RR = 2; F.NJW = (NP + 1) / 2; maxjp = 2; }
    else { F.RR = 2; F.NJW = (NP + 3) / 4; maxjp = 4; }
    F.NWC = (F.RR / 2) * F.NJW;
    const int R4 = (F.Rp + 3) & ~3;
    F.Lbox = hdf::kHTW + 2 * R4 + 4;
    F.planes_bytes = round_up(F.Lbox * F.RR * NP * 4, 128);
    F.stage_bytes = F.planes_bytes + round_up(hdf::kCoefBox * F.RR * 4, 128);
    const int fixed = 128 + round_up(F.RR * hdf::kHTW * 4, 128) + 128;
    int optin = 227 * 1024;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    const int budget = std::min(200 * 1024, optin - 2048);   // (large n and R: up to the opt-in limit)
    F.NS = std::min(4, (budget - fixed) / F.stage_bytes);
    if (F.NS < 2) F.NS = std::min(2, (optin - 2048 - fixed) / F.stage_bytes);
    if (F.NS < 2) return fail(HDF_ERR_ARG, "tile does not fit shared memory (n=%d, R=%d)", n, radius);
    F.hl.grid = dim3((W + hdf::kHTW - 1) / hdf::kHTW, (H + F.RR - 1) / F.RR);
    F.hl.threads = 32 * (F.NWC + 1);
    F.hl.smem = fixed + (size_t)F.NS * F.stage_bytes;
    F.hl.maxjp = maxjp;
    return HDF_OK;
}

// Dynamic shared memory of k_range_vpass: the centres of its plane group, two buffers of J raw rows
// (rho, or rho + n floats per pixel when f is not p) and two of J range-weight rows.
size_t vpass_smem(const FilterPlan& F, int rho, int n, bool f_is_p) {
    const int J = hdf::vpass_j(F.Rp);
    const int RW = f_is_p ? rho : rho + n;
    const size_t mus_len = (size_t)round_up(hdf::vfir_nkmax(F.NP, F.Pg) * rho, 4);
    const size_t raw_len = (size_t)round_up(J * hdf::kVTX * RW, 4);
    const size_t zs_len = (size_t)J * F.Pg * hdf::kVTX;
    return sizeof(float) * (mus_len + 2 * raw_len + 2 * zs_len);
}

struct FilterWS {
    float* planes;
    float* cpl;
    float* Ap32;
    double* Ap64;
    double* Vscratch;
    int* status;
    int* flag_count;
    int* flag_list;
    int* labels;      // internal labels (hard variant, when the caller passes NULL)
    float* centres;   // internal centres (when the caller passes NULL)
    void* cluster_ws;
};

constexpr int kMaxInBands = 16;

FilterWS carve_filter(Carver& cv, int H, int W, int n, int rho, int K, int Wp, bool with_cluster) {
    FilterWS w;
    const int NP = n + 1;
    w.planes = cv.take<float>((size_t)K * NP * H * Wp);
    w.cpl = cv.take<float>((size_t)K * H * Wp);
    w.Ap32 = cv.take<float>((size_t)K * K);
    w.Ap64 = cv.take<double>((size_t)K * K);
    w.Vscratch = cv.take<double>((size_t)K * K);
    w.status = cv.take<int>(4 + kMaxInBands);   // [A^+ status, flag count, flag start, -, max |f| per input band]
    w.flag_count = w.status + 1;
    w.flag_list = cv.take<int>((size_t)H * W);
    w.labels = cv.take<int>((size_t)H * W);
    w.centres = cv.take<float>((size_t)K * rho);
    w.cluster_ws = nullptr;
    if (with_cluster) {
        cv.off = (cv.off + 255) & ~size_t(255);
        w.cluster_ws = cv.base ? cv.base + cv.off : nullptr;
        Carver c2(w.cluster_ws);
        carve_cluster(c2, nullptr, H, W, rho, K);
        cv.off += c2.off;
    }
    return w;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool getenv_on(const char* name) {
    const char* e = getenv(name);
    return e && atoi(e) != 0;
}

int encode3d(CUtensorMap* m, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch_bytes,
             uint64_t plane_bytes, uint32_t b0, uint32_t b1, uint32_t b2,
             CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(HDF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {pitch_bytes, plane_bytes};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HDF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return HDF_OK;
}

// strip-major planes [P][Wp / 32][H][32] of 2-byte (fp16, 64-byte rows, SWIZZLE_64B) or 1-byte (e4m3 as
// uint8, 32-byte rows, SWIZZLE_32B) elements; box [planes][1 strip][rows][32]
int encode_strips(CUtensorMap* m, void* base, int H, int Wp, int P, uint32_t rows, uint32_t planes, int esize) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(HDF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t rb = 32ull * (cuuint64_t)esize;
    cuuint64_t dims[4] = {32, (cuuint64_t)H, (cuuint64_t)(Wp / 32), (cuuint64_t)P};
    cuuint64_t strides[3] = {rb, (cuuint64_t)H * rb, (cuuint64_t)H * (cuuint64_t)(Wp / 32) * rb};
    cuuint32_t box[4] = {32, rows, 1, planes};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    esize == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HDF_ERR_CUDA, "cuTensorMapEncodeTiled (strips) failed (%d)", (int)r);
    return HDF_OK;
}

// Library-owned side stream and fork/join events (per device): k_gram_pinv runs on it, concurrently
// with the column pass (which leaves one SM free for it), and the main stream waits for it before the
// coefficient kernel.  Created once, never destroyed (process lifetime).
// The fork/join events are shared by every call on the device, so a call holds the device's `mu`
// from recording `fork` until its main stream has waited on `join` (host-side only, a few launches):
// another thread can then neither re-record `fork` before this call's side stream waited on it, nor
// `join` before this call's main stream did.  Calls on different caller streams share the side
// stream, so their k_gram_pinv launches are serialised on it (correct, not concurrent).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex* mu = nullptr;
};
// The host path's copy-out stream: one per (calling thread, device), created on first use.
cudaStream_t copy_stream() {
    static thread_local cudaStream_t cs[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!cs[dev] && cudaStreamCreateWithFlags(&cs[dev], cudaStreamNonBlocking) != cudaSuccess) {
        cs[dev] = nullptr;
        return nullptr;
    }
    return cs[dev];
}

// The row-pass stream of the pipelined filter (run_filter): one per (calling thread, device), with a
// small pool of events reused call after call (a wait captures the event's state when it is enqueued,
// so re-recording in the next call is safe).
struct PipeStream {
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> ev;
};
PipeStream* pipe_stream(int nev) {
    static thread_local PipeStream ps[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    PipeStream& p = ps[dev];
    if (!p.s && cudaStreamCreateWithFlags(&p.s, cudaStreamNonBlocking) != cudaSuccess) {
        p.s = nullptr;
        return nullptr;
    }
    while ((int)p.ev.size() < nev) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        p.ev.push_back(e);
    }
    return &p;
}

int side_stream(SideStream* out) {
    static std::mutex mu;
    static std::mutex dev_mu[64];
    static SideStream cache[64];
    int dev = 0;
    HDF_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(HDF_ERR_CUDA, "device index %d out of range", dev);
    std::lock_guard<std::mutex> lk(mu);
    SideStream& c = cache[dev];
    if (!c.s) {
        HDF_CUDA(cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking));
        HDF_CUDA(cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming));
        HDF_CUDA(cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming));
        c.mu = &dev_mu[dev];
    }
    *out = c;
    return HDF_OK;
}

using CoefKernel = hdf::CoefFn;
CoefKernel coeffs_mma_kernel(int nt, int rho) {
    switch (nt) {
        case 1: return hdf::coeffs_mma_kernel_nt1(rho);
        case 2: return hdf::coeffs_mma_kernel_nt2(rho);
        case 3: return hdf::coeffs_mma_kernel_nt3(rho);
        case 4: return hdf::coeffs_mma_kernel_nt4(rho);
        case 5: return hdf::coeffs_mma_kernel_nt5(rho);
        case 6: return hdf::coeffs_mma_kernel_nt6(rho);
        case 7: return hdf::coeffs_mma_kernel_nt7(rho);
        case 8: return hdf::coeffs_mma_kernel_nt8(rho);
        default: return nullptr;
    }
}

int nsm_of_device() {
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nsm;
}

void fill_taps(float* taps, int kind, float sigma_s, int R, int Rp) {
    for (int i = 0; i < hdf::kMaxTaps; i++) taps[i] = 0.f;
    for (int t = -Rp; t <= Rp; t++) {
        float w = 0.f;
        if (t >= -R && t <= R) {
            if (kind == HDF_SPATIAL_BOX) w = 1.f;
            else w = (float)std::exp(-(double)(t * t) / (2.0 * (double)sigma_s * (double)sigma_s));
        }
        taps[t + Rp] = w;
    }
}

// Young's recursive Gaussian coefficients in fp64 and the anti-causal start matrix of the
// zero extension (k_iir.cuh, R17): M[:, j] = (y[N], y[N+1], y[N+2]) when (w[N-1], w[N-2], w[N-3]) = e_j
// and the input is zero from N on (a long zero-input run of both passes, at rest far past the end).
hdf::IIRParams iir_params(double s) {
    const double q = s >= 2.5 ? 0.98711 * s - 0.96330 : 3.97156 - 4.14554 * std::sqrt(1.0 - 0.26891 * s);
    const double b0 = 1.57825 + 2.44413 * q + 1.4281 * q * q + 0.422205 * q * q * q;
    const double b1 = 2.44413 * q + 2.85619 * q * q + 1.26661 * q * q * q;
    const double b2 = -(1.4281 * q * q + 1.26661 * q * q * q);
    const double b3 = 0.422205 * q * q * q;
    const double a1 = b1 / b0, a2 = b2 / b0, a3 = b3 / b0, B = 1.0 - (b1 + b2 + b3) / b0;
    const double G = std::sqrt(2.0 * 3.14159265358979323846) * s;
    hdf::IIRParams P;
    memset(&P, 0, sizeof(P));
    P.gB = G * B;
    P.B = B;
    P.a1 = a1;
    P.a2 = a2;
    P.a3 = a3;
    const int L = (int)(60.0 * s) + 100;
    std::vector<double> w(L + 3), y(L + 3);
    for (int j = 0; j < 3; j++) {
        w[0] = (j == 2) ? 1.0 : 0.0;   // w[0..2] = w[N-3], w[N-2], w[N-1]; w[3 + t] = w[N + t]
        w[1] = (j == 1) ? 1.0 : 0.0;
        w[2] = (j == 0) ? 1.0 : 0.0;
        for (int t = 0; t < L; t++) w[3 + t] = a1 * w[2 + t] + a2 * w[1 + t] + a3 * w[t];
        std::fill(y.begin(), y.end(), 0.0);   // y[t] = y[N + t], at rest from L on
        for (int t = L - 1; t >= 0; t--) y[t] = B * w[3 + t] + a1 * y[t + 1] + a2 * y[t + 2] + a3 * y[t + 3];
        for (int r = 0; r < 3; r++) P.M[3 * r + j] = y[r];
    }
    return P;
}

// hard: the hard-assignment variant: c = one-hot(label), no A^+, no fallback (tau = 0).
// hard_labels: the caller's labels (with its centres), or NULL to cluster here (labels in the workspace).
// Every argument check of a filter call that needs no pointer (shared by the device and host entry
// points, so that both reject bad arguments before anything is enqueued).
// (1) the scalar arguments (no CUDA call)
int validate_scalars(int n, int rho, int H, int W, int kind, float sigma_r, int K, float tau, bool hard) {
    int rc = check_common(H, W, rho, K);
    if (rc) return rc;
    if (n < 1 || n > HDF_MAX_N) return fail(HDF_ERR_ARG, "n must be in [1, %d] (got %d)", HDF_MAX_N, n);
    if (!(sigma_r > 0.f)) return fail(HDF_ERR_ARG, "sigma_r must be > 0");
    if (!(tau >= 0.f)) return fail(HDF_ERR_ARG, "tau must be >= 0");
    if (hard && kind == HDF_SPATIAL_GAUSSIAN_IIR)   // no oracle for that pairing: not offered
        return fail(HDF_ERR_ARG, "the hard-assignment variant takes the FIR kinds (gaussian, box)");
    return HDF_OK;
}

// (2) the plan and the device limits
int validate_filter(int n, int rho, int H, int W, int kind, float sigma_s, int radius, float sigma_r, int K,
                    float tau, bool f_is_p, bool hard, FilterPlan* F, size_t* vsmem) {
    int rc = validate_scalars(n, rho, H, W, kind, sigma_r, K, tau, hard);
    if (rc) return rc;
    rc = make_plan(H, W, n, K, kind, sigma_s, radius, F, nsm_of_device());
    if (rc) return rc;
    // the column pass keeps J raw rows (rho or rho + n floats per pixel, double buffered) and J range-
    // weight rows of its plane group in shared memory: checked before anything is enqueued
    *vsmem = vpass_smem(*F, rho, n, f_is_p);
    int dev = 0, optin = 0;
    HDF_CUDA(cudaGetDevice(&dev));
    HDF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (*vsmem > (size_t)optin)
        return fail(HDF_ERR_ARG,
                    "the column pass needs %zu bytes of shared memory (rho %d, n %d, radius %d) > %d: reduce "
                    "rho + n or the radius",
                    *vsmem, rho, n, F->Rp, optin);
    return HDF_OK;
}

// hard: the hard-assignment variant: c = one-hot(label), no A^+, no fallback (tau = 0).
// hard_labels: the caller's labels (with its centres), or NULL to cluster here (labels in the workspace).
// n_flagged_host != NULL: read the flag count, the pinv status and (when the clustering ran inside
// the call) the clustering status back with one synchronisation at the end.
// nchunks / after_chunk (the host path): the row pass runs in nchunks row chunks and after_chunk(y0, y1)
// is called once the rows [y0, y1) of g are final (enqueued on st), e.g. to start their copy-out.
using ChunkFn = std::function<int(int, int, cudaStream_t)>;
// before_rows(y_end, s): make stream s wait until the input rows [0, y_end) are on the device (hdf_filter_host copies
// the input in row chunks; the tensor-core column pass then runs in row bands, each as soon as its rows arrived)
using RowsFn = std::function<int(int, cudaStream_t)>;
int run_filter(const float* f, int n, const float* p, int rho, int H, int W, int kind, float sigma_s, int radius,
               float sigma_r, int K, const float* centres, float tau, float* g, int32_t* n_flagged_host, void* ws,
               size_t ws_bytes, cudaStream_t st, bool hard = false, const int32_t* hard_labels = nullptr,
               int nchunks = 1, const ChunkFn& after_chunk = ChunkFn(), const RowsFn& before_rows = RowsFn(),
               int in_bands = 1) {
    FilterPlan F;
    size_t vsmem = 0;
    int rc = validate_scalars(n, rho, H, W, kind, sigma_r, K, tau, hard);
    if (rc) return rc;
    if (!f || !p || !g || !ws) return fail(HDF_ERR_ARG, "NULL pointer argument");
    if (misaligned(f) || misaligned(p) || misaligned(g) || misaligned(ws) || (centres && misaligned(centres)))
        return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
    if (g == f || g == p) return fail(HDF_ERR_ARG, "g must not alias f or p");
    rc = validate_filter(n, rho, H, W, kind, sigma_s, radius, sigma_r, K, tau, f == p, hard, &F, &vsmem);
    if (rc) return rc;
    const int nsm = nsm_of_device();
    const size_t need = hdf_filter_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius);
    if (ws_bytes < need) return fail(HDF_ERR_WORKSPACE, "workspace %zu < required %zu bytes", ws_bytes, need);
    Carver cv(ws);
    FilterWS w = carve_filter(cv, H, W, n, rho, K, F.Wp, true);
    const float neg_inv2sr2 = (float)(-1.0 / (2.0 * (double)sigma_r * (double)sigma_r));

    if (hard) tau = 0.5f;   // small r_s(i): the direct window sum with mu_s (k_fallback, hard mode)
    // step 1 (optional): cluster the guide inside this call
    ClusterReadback crb;
    const bool cluster_here = !centres;
    if (!centres) {
        if (before_rows) {
            rc = before_rows(H, st);
            if (rc) return rc;
        }
        int32_t* lab = hard ? w.labels : nullptr;
        rc = launch_cluster(p, H, W, rho, K, w.centres, lab, nullptr, w.cluster_ws, st,
                            n_flagged_host ? &crb : nullptr);
        if (rc) return rc;
        centres = w.centres;
        if (hard) hard_labels = lab;
    }
    // step 2: A and A^+ (one CTA, fp64) on the side stream, concurrent with the column pass
    SideStream ss;
    rc = side_stream(&ss);
    if (rc) return rc;
    std::unique_lock<std::mutex> side_lock(*ss.mu);   // until st has waited on ss.join
    HDF_CUDA(cudaEventRecord(ss.fork, st));
    HDF_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    if (!hard) {
        hdf::PinvOut po{w.Ap32, w.Ap64, w.status, w.Vscratch};
        const size_t smem = hdf::pinv_smem_bytes(K);
        HDF_CUDA(cudaFuncSetAttribute(hdf::k_gram_pinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        ProfScope prof(HDF_STAGE_PINV, ss.s);
        hdf::k_gram_pinv<<<1, hdf::kPinvThreads, smem, ss.s>>>(centres, K, rho, -1.0 / (2.0 * (double)sigma_r * sigma_r),
                                                              po);
        HDF_CUDA(cudaGetLastError());
    }
    HDF_CUDA(cudaEventRecord(ss.join, ss.s));
    HDF_CUDA(cudaMemsetAsync(w.flag_count, 0, sizeof(int), st));
    if (hard) HDF_CUDA(cudaMemsetAsync(w.status, 0, sizeof(int), st));
    float taps[hdf::kMaxTaps];
    fill_taps(taps, kind, sigma_s, F.R, F.Rp);
    // the column FIR on the tensor cores (k_vpass_tc.cuh) for colour images with the Gaussian FIR
    // (HDF_VPASS_FMA=1 keeps the CUDA-core kernel), and then the row FIR + combine on the tensor cores too
    // (k_hpass_tc.cuh, fed by fp16 hi/lo planes; HDF_HPASS_FMA=1 keeps fp32 planes and the CUDA-core row pass)
    bool use_tc = !F.box && !F.iir && F.NP == 4 && rho == 3 && f == p && F.R >= 4 && F.R <= hdf::kVtcMaxR &&
                  (W % 4) == 0;
    if (const char* e = getenv("HDF_VPASS_FMA")) {
        if (atoi(e)) use_tc = false;
    }
    // The tensor-core row pass parallelises over (32-row block, 128-column strip) units with every cluster
    // inside a unit: it is used when the units fill the SMs (config 5: 4096 units; a 512 x 512 image has
    // only 64, and there the CUDA-core row pass is faster: c2b 61 vs 95 us).  HDF_HPASS_FMA=1 / =0 forces
    // the CUDA-core / tensor-core row pass.
    bool use_htc = use_tc && F.R <= hdf::kHtcMaxR &&
                   (long long)((H + hdf::kHtcRows - 1) / hdf::kHtcRows) * ((W + 127) / 128) >= nsm;
    if (const char* e = getenv("HDF_HPASS_FMA")) {
        if (*e) use_htc = use_tc && F.R <= hdf::kHtcMaxR && atoi(e) == 0;
    }
    int wexp = 0;   // 2^wexp >= the sum of the taps (the fp16 planes' scale)
    {
        double ws = 0.0;
        for (int t = 0; t <= 2 * F.Rp; t++) ws += (double)taps[t];
        while (std::ldexp(1.0, wexp) < ws) wexp++;
    }
    int* amax = w.status + 4;   // [kMaxInBands]: max |f| over the input rows of each column-pass band
    // The pipelined filter (tensor-core path): the image is cut into nband row bands (multiples of 64
    // rows).  The column pass of band b + 1 (st, gv SMs: it only writes its planes) runs while the row
    // pass + combine of band b (hs, gh SMs: it only reads them) runs, so the HBM write and read streams
    // overlap instead of taking turns (a write-only stream tops out near 3.6 TB/s, a mixed one at the
    // copy bandwidth); the coefficient kernel runs on hs beside the first column-pass band.  Band 0's
    // column pass and the last band's row pass have the GPU to themselves.  HDF_PIPE_BANDS (default 1 =
    // off) and HDF_PIPE_HSM (the row pass's SMs) tune it.
    const int nt64 = (H + hdf::kVtcRows - 1) / hdf::kVtcRows;
    int nband = 1;
    if (use_htc) {
        int want = 1;   // measured slower at c5: off unless asked for
        if (const char* e = getenv("HDF_PIPE_BANDS")) want = atoi(e);
        if (want > 1) nband = std::min(std::max(want, nchunks), nt64);
    }
    const bool pipe = nband > 1;
    // input bands (hdf_filter_host): uniform bands of ib_rows rows (a multiple of 64) for the tensor-core passes
    int nib = 1, ib_rows = std::max(H, 1);
    if (before_rows && use_htc && !pipe && in_bands > 1) {
        const int want = std::min(std::min(in_bands, kMaxInBands), nt64);
        ib_rows = hdf::kVtcRows * ((nt64 + want - 1) / want);
        nib = (H + ib_rows - 1) / ib_rows;
        if (nib <= 1) {
            nib = 1;
            ib_rows = std::max(H, 1);
        }
    }
    PipeStream* pst = nullptr;
    if (pipe) {
        pst = pipe_stream(nband + 2);
        if (!pst) return fail(HDF_ERR_CUDA, "pipeline stream / events: %s", cudaGetErrorString(cudaGetLastError()));
    }
    cudaStream_t hs = pipe ? pst->s : st;   // the stream of the coefficients and the row passes
    int gh = nsm, gv = nsm - 1;
    if (pipe) {
        gh = (nsm - 1) * 47 / 100;
        if (const char* e = getenv("HDF_PIPE_HSM")) gh = atoi(e);
        gh = std::max(1, std::min(gh, nsm - 2));
        gv = nsm - 1 - gh;
    }
    auto band_y = [&](int b) { return std::min(H, hdf::kVtcRows * (int)((long long)nt64 * b / nband)); };
    ProfScope prof_filter(HDF_STAGE_FILTER, st);
    // F1: range weights + column pass
    {
        hdf::VParams vp;
        vp.f = f;
        vp.p = p;
        vp.centres = centres;
        vp.planes = w.planes;
        vp.pstride = (long long)H * F.Wp;
        vp.n = n;
        vp.rho = rho;
        vp.H = H;
        vp.W = W;
        vp.Wp = F.Wp;
        vp.K = K;
        vp.NP = F.NP;
        vp.P = F.P;
        vp.nstrip = F.TY;
        vp.ncol = F.TY * ((F.P + F.Pg - 1) / F.Pg);
        vp.f_is_p = (f == p) ? 1 : 0;
        vp.neg_inv2sr2 = neg_inv2sr2;
        for (int t = 0; t <= HDF_MAX_RADIUS; t++) {
            const float wv = (t <= F.Rp) ? taps[F.Rp + t] : 0.f;
            uint32_t b;
            memcpy(&b, &wv, 4);
            vp.tw[t] = ((unsigned long long)b << 32) | b;
        }
        for (int t = 0; t < 2 * HDF_MAX_RADIUS + 1; t++) vp.tws[t] = (t <= 2 * F.Rp) ? taps[t] : 0.f;
        hdf::VLaunch vl = F.vl;
        vl.smem = vsmem;
        std::unique_ptr<ProfScope> prof(use_tc ? nullptr : new ProfScope(HDF_STAGE_VPASS, st));
        if (!use_tc && before_rows) {
            rc = before_rows(H, st);
            if (rc) return rc;
        }
        if (use_tc) {
            HDF_CUDA(cudaMemsetAsync(amax, 0, sizeof(int) * kMaxInBands, st));
            if (nib == 1) {   // one band: the scale from max |f| over the whole image
                if (before_rows) {
                    rc = before_rows(H, st);
                    if (rc) return rc;
                }
                const long long nf = (long long)H * W * n;
                hdf::k_absmax<<<(unsigned)std::min<long long>((nf + 255) / 256, (long long)nsm * 8), 256, 0, st>>>(f, nf,
                                                                                                                amax);
                HDF_CUDA(cudaGetLastError());
            }
            hdf::VtcParams tp;
            tp.centres = centres;
            tp.planes = w.planes;
            tp.ph = use_htc ? reinterpret_cast<unsigned short*>(w.planes) : nullptr;
            // the e4m3 residuals after the 4K fp16 hi planes (3 bytes per value of the 4 the workspace holds)
            tp.pl = use_htc ? reinterpret_cast<unsigned char*>(w.planes) + (size_t)4 * K * H * F.Wp * 2 : nullptr;
            tp.wexp = wexp;
            tp.absmax = amax;
            tp.pstride = (long long)H * F.Wp;
            tp.H = H;
            tp.W = W;
            tp.Wp = F.Wp;
            tp.K = K;
            tp.R = F.R;
            tp.nstrip = (W + 31) / 32;
            tp.csleep = 0;
            if (const char* e = getenv("HDF_VTC_CSLEEP")) tp.csleep = std::max(0, atoi(e));
            tp.neg_inv2sr2 = neg_inv2sr2;
            for (int t = 0; t < hdf::kMaxTaps; t++) tp.taps[t] = 0.f;
            for (int t = 0; t <= 2 * F.R; t++) tp.taps[t] = taps[F.Rp - F.R + t];
            CUtensorMap tmp;
            rc = encode3d(&tmp, const_cast<float*>(p), (uint64_t)W * 3, (uint64_t)H, 1, (uint64_t)W * 3 * 4,
                          (uint64_t)H * W * 3 * 4, 96u, 64u, 1u);
            if (rc) return rc;
            const size_t smem = hdf::vpass_tc_smem(F.R);
            // consumer warps: 8 (32 rows each; the fp16 + e4m3 stores are the consumers' work), HDF_VTC_CONS=4 keeps 4
            int cons = 8;
            if (const char* e = getenv("HDF_VTC_CONS")) cons = atoi(e) == 4 ? 4 : 8;
            // the stacked Toeplitz operand (k_vpass_tc.cuh, NS): a consistent 1-2% at config 5;
            // HDF_VTC_NSTACK=0 keeps the three-MMA form
            bool vns = true;
            if (const char* e = getenv("HDF_VTC_NSTACK")) vns = !(*e) || atoi(e) != 0;
            void (*kvtc)(const CUtensorMap, const hdf::VtcParams) =
                cons == 4 ? hdf::k_range_vpass_tc<4, false>
                          : (vns ? hdf::k_range_vpass_tc<8, true> : hdf::k_range_vpass_tc<8, false>);
            const int vthreads = cons == 4 ? hdf::vtc_threads(4) : hdf::vtc_threads(8);
            HDF_CUDA(cudaFuncSetAttribute(kvtc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            // output rows [y0, y1) on `grid` SMs: row segments of whole 64-row tiles, enough units to fill the grid
            auto launch_vtc = [&](int y0, int y1, int grid) -> int {
                const long long ncol = (long long)tp.nstrip * K;
                const int rows = y1 - y0;
                const int maxseg = (rows + hdf::kVtcRows - 1) / hdf::kVtcRows;
                tp.y0 = y0;
                tp.nseg = (int)std::max<long long>(1, std::min<long long>(maxseg, (4LL * grid + ncol - 1) / ncol));
                tp.seglen = ((rows + tp.nseg - 1) / tp.nseg + hdf::kVtcRows - 1) / hdf::kVtcRows * hdf::kVtcRows;
                tp.nseg = (rows + tp.seglen - 1) / tp.seglen;
                ProfScope pv(HDF_STAGE_VPASS, st);
                kvtc<<<(unsigned)std::min<long long>(grid, ncol * tp.nseg), vthreads, smem, st>>>(tmp, tp);
                HDF_CUDA(cudaGetLastError());
                return HDF_OK;
            };
            if (!pipe && nib > 1) {
                // the input arrives in row chunks: band b (rows [b ib_rows, (b + 1) ib_rows)) starts when its input rows
                // [y0 - R, y1 + R) are on the device, with its own power-of-two scale from max |f| over those rows
                for (int b = 0; b < nib; b++) {
                    const int y0 = b * ib_rows, y1 = std::min(H, y0 + ib_rows);
                    const int i0 = std::max(0, y0 - F.R), i1 = std::min(H, y1 + F.R);
                    rc = before_rows(i1, st);
                    if (rc) return rc;
                    const long long nf = (long long)(i1 - i0) * W * n;
                    hdf::k_absmax<<<(unsigned)std::min<long long>((nf + 255) / 256, (long long)nsm * 8), 256, 0, st>>>(
                        f + (size_t)i0 * W * n, nf, amax + b);
                    HDF_CUDA(cudaGetLastError());
                    tp.absmax = amax + b;
                    rc = launch_vtc(y0, y1, std::max(1, nsm - 1));
                    if (rc) return rc;
                }
            } else if (!pipe) {
                rc = launch_vtc(0, H, std::max(1, nsm - 1));
                if (rc) return rc;
            } else {
                HDF_CUDA(cudaEventRecord(pst->ev[0], st));   // hs starts after the clustering and the memsets
                for (int b = 0; b < nband; b++) {
                    rc = launch_vtc(band_y(b), band_y(b + 1), gv);
                    if (rc) return rc;
                    HDF_CUDA(cudaEventRecord(pst->ev[1 + b], st));
                }
            }
        } else {
            HDF_CUDA(hdf::launch_vpass(F.Rp, F.box, vl, st, vp));
        }
        if (F.iir) {   // NEXT #1: the recursion over the unfiltered planes, columns then rows
            hdf::IIRParams ip = iir_params((double)sigma_s);
            ip.planes = w.planes;
            ip.pstride = (long long)H * F.Wp;
            ip.P = F.P;
            ip.H = H;
            ip.W = W;
            ip.Wp = F.Wp;
            hdf::k_iir_cols<<<dim3((unsigned)((W + hdf::kIirColThreads - 1) / hdf::kIirColThreads), (unsigned)F.P),
                              hdf::kIirColThreads, 0, st>>>(ip);
            HDF_CUDA(cudaGetLastError());
            hdf::k_iir_rows<<<dim3((unsigned)((H + 31) / 32), (unsigned)F.P), 32, 0, st>>>(ip);
            HDF_CUDA(cudaGetLastError());
        }
    }
    if (pipe) HDF_CUDA(cudaStreamWaitEvent(hs, pst->ev[0], 0));
    HDF_CUDA(cudaStreamWaitEvent(hs, ss.join, 0));   // A^+ is ready
    side_lock.unlock();
    // loop for2: c(i) = A^+ b(i) -> K coefficient planes
    // (HDF_C24=1: in 24 bits when k_coeffs_tc feeds the stacked-operand tensor-core row pass, CoefParams.  Off by
    // default: measured slower at config 5 -- the coefficient kernel's consumers are bound by instruction issue, not
    // by the bytes they write (1.44 -> 1.61 ms with the pack/transpose shuffles), and the row pass is not bound by
    // HBM reads (3.33 -> 3.36 ms))
    bool htc_ns = true;
    if (const char* e = getenv("HDF_HTC_NSTACK")) {
        if (*e && atoi(e) == 0) htc_ns = false;
    }
    const bool c24 = getenv_on("HDF_C24") && use_htc && htc_ns && !hard && K <= hdf::kTcMaxK && K % 4 == 0 &&
                     W % 4 == 0 && !getenv_on("HDF_COEFFS_MMA") && !getenv_on("HDF_COEFFS_FMA");
    {
        hdf::CoefParams cp;
        cp.p = p;
        cp.centres = centres;
        cp.Ap32 = w.Ap32;
        cp.cpl = w.cpl;
        cp.cstride = (long long)H * F.Wp;
        if (c24) {   // 24-bit planes inside the same buffer: [K][H][Wp] 16-bit words, then [K][H][Wp] bytes
            cp.ch = reinterpret_cast<unsigned short*>(w.cpl);
            cp.cm = reinterpret_cast<unsigned char*>(w.cpl) + (size_t)K * H * F.Wp * 2;
        }
        cp.H = H;
        cp.W = W;
        cp.Wp = F.Wp;
        cp.rho = rho;
        cp.K = K;
        cp.neg_inv2sr2 = neg_inv2sr2;
        const long long npix = (long long)H * W;
        const unsigned nblk = (unsigned)((npix + hdf::kCoefPix - 1) / hdf::kCoefPix);
        void (*kt)(const hdf::CoefParams) = nullptr;
        void (*km)(const hdf::CoefParams) = nullptr;
        // tcgen05 (5th-generation tensor cores, TMEM accumulator, 3xTF32) for K <= 64; the legacy
        // mma.sync kernel (HDF_COEFFS_MMA=1) and the CUDA-core kernels (HDF_COEFFS_FMA=1) are kept for
        // comparison and for K > 64
        void (*ktc)(const hdf::CoefParams) = nullptr;
        if (K <= hdf::kTcMaxK) ktc = rho == 3 ? hdf::k_coeffs_tc<3> : rho == 6 ? hdf::k_coeffs_tc<6> : hdf::k_coeffs_tc<0>;
        km = coeffs_mma_kernel((K + 7) / 8, rho);   // mma.sync (3xTF32), K <= 64 padded to 8 NT
        if (const char* e = getenv("HDF_COEFFS_MMA")) {
            if (atoi(e)) ktc = nullptr;
        }
        if (const char* e = getenv("HDF_COEFFS_FMA")) {   // diagnostics: the CUDA-core kernel instead
            if (atoi(e)) km = ktc = nullptr;
        }
        if (K == 8) kt = hdf::k_coeffs_t<8>;
        else if (K == 16) kt = hdf::k_coeffs_t<16>;
        else if (K == 32) kt = hdf::k_coeffs_t<32>;
        else if (K == 64) kt = hdf::k_coeffs_t<64>;
        ProfScope prof(HDF_STAGE_COEFFS, hs);
        if (hard) {
            const long long ntot = npix;
            const unsigned nb = (unsigned)std::min<long long>((ntot + 255) / 256, (long long)nsm * 16);
            hdf::k_coeffs_onehot<<<nb, 256, 0, hs>>>(hard_labels, w.cpl, (long long)H * F.Wp, H, W, F.Wp, K);
        } else if (ktc) {
            const size_t smem = hdf::coeffs_tc_smem(K, rho);
            HDF_CUDA(cudaFuncSetAttribute(ktc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            HDF_CUDA(cudaFuncSetAttribute(ktc, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            int per_sm = 1;
            HDF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ktc, hdf::kTcThreads, smem));
            const long long ntile = (npix + hdf::kTcM - 1) / hdf::kTcM;
            const unsigned nb = (unsigned)std::min<long long>(ntile, (long long)(pipe ? gh : nsm) * std::max(1, std::min(per_sm, 1)));
            ktc<<<nb, hdf::kTcThreads, smem, hs>>>(cp);
        } else if (km) {
            const int nt = (K + 7) / 8;
            const size_t smem = sizeof(float) * ((size_t)2 * nt * nt * 2 * 32 + (size_t)8 * nt * rho);
            HDF_CUDA(cudaFuncSetAttribute(km, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const long long ntile = (npix + 15) / 16;
            const long long want = (ntile + 7) / 8;
            int per_sm = 1;   // resident blocks per SM: a persistent grid (A^+ staged once per block)
            HDF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, km, hdf::kCoefMmaThreads, smem));
            const unsigned nb = (unsigned)std::min<long long>(want, (long long)nsm * std::max(per_sm, 1));
            km<<<nb, hdf::kCoefMmaThreads, smem, hs>>>(cp);
        } else if (kt) {   // compile-time K: b in registers, broadcast A^+ rows
            const size_t smem = sizeof(float) * ((size_t)K * K + (size_t)K * rho);
            HDF_CUDA(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kt<<<nblk, hdf::kCoefPix, smem, hs>>>(cp);
        } else {
            const int K8 = (K + 7) & ~7;
            const size_t smem = sizeof(float) * ((size_t)K * K8 + (size_t)K * rho + (size_t)K * hdf::kCoefPix);
            HDF_CUDA(cudaFuncSetAttribute(hdf::k_coeffs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            hdf::k_coeffs<<<nblk, hdf::kCoefPix, smem, hs>>>(cp);
        }
        HDF_CUDA(cudaGetLastError());
    }
    // F2 + F3 in row chunks (one chunk unless the host path asks for more, to overlap the copy-out of
    // finished rows with the rest of the row pass): row pass + combine + normalise (TMA-fed), then the
    // direct (num)/(den) for the pixels this chunk flagged (R9)
    CUtensorMap tp, tc;
    rc = encode3d(&tp, w.planes, (uint64_t)W, (uint64_t)H, (uint64_t)F.P, (uint64_t)F.Wp * 4, (uint64_t)H * F.Wp * 4,
                  (uint32_t)F.Lbox, (uint32_t)F.RR, (uint32_t)F.NP);
    if (rc) return rc;
    rc = encode3d(&tc, w.cpl, (uint64_t)W, (uint64_t)H, (uint64_t)K, (uint64_t)F.Wp * 4, (uint64_t)H * F.Wp * 4,
                  (uint32_t)hdf::kCoefBox, (uint32_t)F.RR, 1u);
    if (rc) return rc;
    hdf::HParams hp;
    hp.g = g;
    hp.flag_count = w.flag_count;
    hp.flag_list = w.flag_list;
    hp.n = n;
    hp.NP = F.NP;
    hp.H = H;
    hp.W = W;
    hp.K = K;
    hp.RR = F.RR;
    hp.NJW = F.NJW;
    hp.NWC = F.NWC;
    hp.NS = F.NS;
    hp.Lbox = F.Lbox;
    hp.stage_bytes = F.stage_bytes;
    hp.planes_bytes = F.planes_bytes;
    hp.tau_floor = tau * taps[F.Rp] * taps[F.Rp] * 1.0f;   // tau * omega(0) * phi(0)
    memcpy(hp.taps, taps, sizeof(taps));
    hdf::FBParams fb;
    fb.f = f;
    fb.p = p;
    fb.g = g;
    fb.flag_count = w.flag_count;
    fb.flag_list = w.flag_list;
    fb.flag_start = nullptr;
    fb.n = n;
    fb.rho = rho;
    fb.H = H;
    fb.W = W;
    fb.R = F.Rfb;
    fb.neg_inv2sr2 = neg_inv2sr2;
    fb.mu = hard ? centres : nullptr;
    fb.labels = hard ? hard_labels : nullptr;
    {
        float t2[hdf::kMaxTaps];
        fb.neg_inv2ss2 = 0.f;
        if (F.Rfb <= HDF_MAX_RADIUS) {
            fill_taps(t2, F.iir ? (int)HDF_SPATIAL_GAUSSIAN : kind, sigma_s, F.Rfb, F.Rfb);
        } else {   // the recursive Gaussian with a window beyond the table: weights in the kernel
            memset(t2, 0, sizeof(t2));
            fb.neg_inv2ss2 = (float)(-1.0 / (2.0 * (double)sigma_s * (double)sigma_s));
        }
        memcpy(fb.taps, t2, sizeof(t2));
    }
    // the tensor-core row pass: tensor maps of the strip-major fp16 hi and e4m3 lo planes (boxes [4 planes][32 rows]
    // [the hi or lo half of a 32-column strip], 64-byte swizzle) and of the coefficient planes (two
    // [32 rows][32 columns] halves per tile, 128-byte swizzle)
    CUtensorMap tz, tzl, tcc, tcm;
    hdf::HtcParams hq;
    size_t htc_smem = 0;
    void (*khtc)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const hdf::HtcParams) =
        c24 ? hdf::k_hpass_combine_tc<true, true> : hdf::k_hpass_combine_tc<true, false>;
    if (use_htc) {
        unsigned short* ph = reinterpret_cast<unsigned short*>(w.planes);
        rc = encode_strips(&tz, ph, H, F.Wp, K * 4, (uint32_t)hdf::kHtcRows, 4u, 2);
        if (rc) return rc;
        rc = encode_strips(&tzl, reinterpret_cast<unsigned char*>(w.planes) + (size_t)4 * K * H * F.Wp * 2, H, F.Wp, K * 4,
                           (uint32_t)hdf::kHtcRows, 4u, 1);
        if (rc) return rc;
        if (c24) {   // boxes [32 rows][64 columns] of the 16-bit words (128-byte swizzle) and of the bytes (64-byte)
            rc = encode3d(&tcc, w.cpl, (uint64_t)W, (uint64_t)H, (uint64_t)K, (uint64_t)F.Wp * 2, (uint64_t)H * F.Wp * 2,
                          (uint32_t)hdf::kHtcN, (uint32_t)hdf::kHtcRows, 1u, CU_TENSOR_MAP_DATA_TYPE_UINT16,
                          CU_TENSOR_MAP_SWIZZLE_128B);
            if (rc) return rc;
            rc = encode3d(&tcm, reinterpret_cast<unsigned char*>(w.cpl) + (size_t)K * H * F.Wp * 2, (uint64_t)W, (uint64_t)H,
                          (uint64_t)K, (uint64_t)F.Wp, (uint64_t)H * F.Wp, (uint32_t)hdf::kHtcN, (uint32_t)hdf::kHtcRows, 1u,
                          CU_TENSOR_MAP_DATA_TYPE_UINT8, CU_TENSOR_MAP_SWIZZLE_64B);
            if (rc) return rc;
        } else {
            rc = encode3d(&tcc, w.cpl, (uint64_t)W, (uint64_t)H, (uint64_t)K, (uint64_t)F.Wp * 4, (uint64_t)H * F.Wp * 4,
                          32u, (uint32_t)hdf::kHtcRows, 1u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_SWIZZLE_128B);
            if (rc) return rc;
            tcm = tcc;
        }
        hq.g = g;
        hq.flag_count = w.flag_count;
        hq.flag_list = w.flag_list;
        hq.absmax = amax;
        hq.band_rows = ib_rows;
        hq.H = H;
        hq.W = W;
        hq.K = K;
        hq.R = F.R;
        hq.nstrip = (W + hdf::kHtcS * hdf::kHtcN - 1) / (hdf::kHtcS * hdf::kHtcN);
        hq.wexp = wexp;
        hq.csleep = 0;
        if (const char* e = getenv("HDF_HTC_CSLEEP")) hq.csleep = std::max(0, atoi(e));
        hq.tau_floor = hp.tau_floor;
        for (int t = 0; t < hdf::kMaxTaps; t++) hq.taps[t] = 0.f;
        for (int t = 0; t <= 2 * F.R; t++) hq.taps[t] = taps[F.Rp - F.R + t];
        htc_smem = hdf::hpass_tc_smem();
        // the stacked Toeplitz operand (one N = 128 MMA per K step instead of two of N = 64) is the default;
        // HDF_HTC_NSTACK=0 keeps the two-MMA form
        if (!htc_ns) khtc = hdf::k_hpass_combine_tc<false, false>;
        HDF_CUDA(cudaFuncSetAttribute(khtc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)htc_smem));
    }
    const int tile_rows = use_htc ? hdf::kHtcRows : F.RR;
    const int row_tiles = use_htc ? (H + hdf::kHtcRows - 1) / hdf::kHtcRows : (int)F.hl.grid.y;
    // row chunks: the pipeline's bands (in 32-row blocks), else nchunks equal chunks
    const int nch = pipe ? nband : std::max(1, std::min(nchunks, row_tiles));
    int* flag_start = w.status + 2;   // list entries before this chunk (device)
    for (int ch = 0; ch < nch; ch++) {
        int ty0 = (int)((long long)row_tiles * ch / nch), ty1 = (int)((long long)row_tiles * (ch + 1) / nch);
        if (pipe) {
            ty0 = band_y(ch) / hdf::kHtcRows;
            ty1 = ch == nch - 1 ? row_tiles : band_y(ch + 1) / hdf::kHtcRows;
            HDF_CUDA(cudaStreamWaitEvent(hs, pst->ev[1 + ch], 0));   // band ch's planes are written
        }
        hp.ytile0 = ty0;
        hdf::HLaunch hl = F.hl;
        hl.grid.y = (unsigned)(ty1 - ty0);
        if (nch > 1) {
            HDF_CUDA(cudaMemcpyAsync(flag_start, w.flag_count, sizeof(int), cudaMemcpyDeviceToDevice, hs));
            fb.flag_start = flag_start;
        }
        {
            ProfScope prof(HDF_STAGE_HPASS, hs);
            if (use_htc) {
                hq.yb0 = ty0;
                hq.yb1 = ty1;
                const long long nunit = (long long)(ty1 - ty0) * hq.nstrip;
                // (the last band's row pass has the GPU to itself)
                const int grid = (pipe && ch < nch - 1) ? gh : nsm;
                khtc<<<(unsigned)std::max<long long>(1, std::min<long long>(grid, nunit)), hdf::kHtcThreads, htc_smem,
                       hs>>>(tz, tzl, tcc, tcm, hq);
                HDF_CUDA(cudaGetLastError());
            } else {
                HDF_CUDA(hdf::launch_hpass(F.Rp, F.box, hl, hs, tp, tc, hp));
            }
        }
        if (tau > 0.f) {
            ProfScope prof(HDF_STAGE_FALLBACK, hs);
            // one warp per flagged pixel (grid-stride): the count is on the device, so the grid is sized for
            // the worst case the SMs can hold at once (8 CTAs of 8 warps per SM), capped by the pixel count
            const long long npix = (long long)H * W;
            const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((npix + 7) / 8, 8LL * nsm));
            if (n <= 16) {
                void (*kfb)(const hdf::FBParams) = n <= 4 ? hdf::k_fallback<4> : hdf::k_fallback<16>;
                kfb<<<nb, hdf::kFbThreads, 0, hs>>>(fb);
            } else {   // many channels: one CTA per pixel (measured at config 3: 20 us vs 51 us for a warp)
                hdf::k_fallback_cta<<<(unsigned)std::min<long long>(npix, 16LL * nsm), hdf::kFbCtaThreads, 0, hs>>>(
                    fb);
            }
            HDF_CUDA(cudaGetLastError());
        }
        if (after_chunk) {
            rc = after_chunk(std::min(H, ty0 * tile_rows), std::min(H, ty1 * tile_rows), hs);
            if (rc) return rc;
        }
    }
    if (pipe) {   // the caller's stream continues after the last row pass
        HDF_CUDA(cudaEventRecord(pst->ev[nband + 1], hs));
        HDF_CUDA(cudaStreamWaitEvent(st, pst->ev[nband + 1], 0));
    }
    prof_filter.close();
    if (n_flagged_host) {
        HostStage* hs = cluster_here ? crb.hs : host_stage();
        if (!hs) return fail(HDF_ERR_CUDA, "pinned host stage: cudaMallocHost failed");
        HDF_CUDA(cudaMemcpyAsync(hs->hv, w.status, sizeof(hs->hv), cudaMemcpyDeviceToHost, st));
        HDF_CUDA(cudaStreamSynchronize(st));
        *n_flagged_host = hs->hv[1];
        if (cluster_here) {   // HDF_ERR_K: the output was filtered with the padded centres (hdf.h)
            rc = cluster_status(crb, K, nullptr);
            if (rc) return rc;
        }
        if (hs->hv[0] == HDF_WARN_ILLCOND)
            return fail(HDF_WARN_ILLCOND, "A is numerically singular; A^+ truncated (R6)");
    }
    return HDF_OK;
}

}  // namespace

namespace hdf {

template <int R>
cudaError_t launch_vpass_t(bool box, const VLaunch& L, cudaStream_t st, const VParams& P);
template <int R>
cudaError_t launch_hpass_t(bool box, const HLaunch& L, cudaStream_t st, const CUtensorMap& tp, const CUtensorMap& tc,
                           const HParams& P);

cudaError_t launch_vpass(int R, bool box, const VLaunch& L, cudaStream_t st, const VParams& P) {
    switch (R) {
#define HDF_CASE(r) \
    case r: return launch_vpass_t<r>(box, L, st, P);
        HDF_CASE(1) HDF_CASE(2) HDF_CASE(3) HDF_CASE(4) HDF_CASE(5) HDF_CASE(6) HDF_CASE(8) HDF_CASE(9)
        HDF_CASE(10) HDF_CASE(12) HDF_CASE(15) HDF_CASE(16) HDF_CASE(20) HDF_CASE(24) HDF_CASE(32)
#undef HDF_CASE
        default: return cudaErrorInvalidValue;
    }
}
cudaError_t launch_hpass(int R, bool box, const HLaunch& L, cudaStream_t st, const CUtensorMap& tp,
                         const CUtensorMap& tc, const HParams& P) {
    switch (R) {
#define HDF_CASE(r) \
    case r: return launch_hpass_t<r>(box, L, st, tp, tc, P);
        HDF_CASE(1) HDF_CASE(2) HDF_CASE(3) HDF_CASE(4) HDF_CASE(5) HDF_CASE(6) HDF_CASE(8) HDF_CASE(9)
        HDF_CASE(10) HDF_CASE(12) HDF_CASE(15) HDF_CASE(16) HDF_CASE(20) HDF_CASE(24) HDF_CASE(32)
#undef HDF_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hdf

// =============================================================================== C ABI ========
extern "C" {

const char* hdf_version(void) { return "hdf 0.1.0 sm_100a"; }

const char* hdf_last_error(void) { return g_err.c_str(); }

// Diagnostics: copy the clustering trace of the last hdf_cluster call that used `ws` (block 0
// events: tag, globaltimer ns).  Returns the number of events.
int hdf_cluster_trace(const float* p_unused, int H, int W, int rho, int K, void* ws, long long* out, int cap) {
    (void)p_unused;
    Carver cv(ws);
    hdf::BisectArgs A = carve_cluster(cv, nullptr, H, W, rho, K);
    int n = 0;
    if (cudaMemcpy(&n, A.ctl + hdf::B_TRACE_N, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    n = std::min(std::min(n, hdf::kBisectTraceCap), cap);
    if (n > 0 && cudaMemcpy(out, A.trace + 1, sizeof(long long) * 2 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    return n;
}

int hdf_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = (on != 0);
    return HDF_OK;
}

static int profile_collect_impl(double* ms_total, int32_t* launches);
int hdf_profile_collect(double* ms_total, int32_t* launches) {
    g_err.clear();
    return guarded([&]() -> int { return profile_collect_impl(ms_total, launches); });
}
static int profile_collect_impl(double* ms_total, int32_t* launches) {
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        recs.swap(g_prof_pending);
    }
    for (int s = 0; s < HDF_NUM_STAGES; s++) {
        if (ms_total) ms_total[s] = 0.0;
        if (launches) launches[s] = 0;
    }
    int rc = HDF_OK;
    for (const ProfRec& r : recs) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess && rc == HDF_OK) rc = fail(HDF_ERR_CUDA, "profile event: %s", cudaGetErrorString(e));
        if (r.stage >= 0 && r.stage < HDF_NUM_STAGES) {
            if (ms_total) ms_total[r.stage] += ms;
            if (launches) launches[r.stage] += 1;
        }
    }
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (const ProfRec& r : recs) {
        g_prof_pool.push_back(r.a);
        g_prof_pool.push_back(r.b);
    }
    return rc;
}

size_t hdf_cluster_workspace_bytes(int H, int W, int rho, int K) {
    if (H < 1 || W < 1 || rho < 1 || K < 1) return 0;
    Carver cv(nullptr);
    carve_cluster(cv, nullptr, H, W, rho, K);
    return cv.off + 256;
}

int hdf_cluster(const float* p, int H, int W, int rho, int K, float* centres, int32_t* labels,
                hdf_cluster_info* info_host, void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        int rc = check_common(H, W, rho, K);
        if (rc) return rc;
        if (!p || !centres || !ws) return fail(HDF_ERR_ARG, "NULL pointer argument");
        if (misaligned(p) || misaligned(centres) || misaligned(ws) || (labels && misaligned(labels)))
            return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
        const size_t need = hdf_cluster_workspace_bytes(H, W, rho, K);
        if (ws_bytes < need) return fail(HDF_ERR_WORKSPACE, "workspace %zu < required %zu bytes", ws_bytes, need);
        return launch_cluster(p, H, W, rho, K, centres, labels, info_host, ws, static_cast<cudaStream_t>(stream));
    });
}

size_t hdf_filter_workspace_bytes(int H, int W, int n, int rho, int K, int kind, float sigma_s, int radius) {
    (void)kind;
    (void)sigma_s;
    (void)radius;
    if (H < 1 || W < 1 || n < 1 || rho < 1 || K < 1) return 0;
    Carver cv(nullptr);
    carve_filter(cv, H, W, n, rho, K, round_up(W, 32), true);
    return cv.off + 256;
}

int hdf_filter(const float* f, int n, const float* p, int rho, int H, int W, int kind, float sigma_s, int radius,
               float sigma_r, int K, const float* centres, float tau, float* g, int32_t* n_flagged_host, void* ws,
               size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        return run_filter(f, n, p, rho, H, W, kind, sigma_s, radius, sigma_r, K, centres, tau, g, n_flagged_host, ws,
                          ws_bytes, static_cast<cudaStream_t>(stream));
    });
}

int hdf_filter_hard(const float* f, int n, const float* p, int rho, int H, int W, int kind, float sigma_s, int radius,
                    float sigma_r, int K, const float* centres, const int32_t* labels, float* g, void* ws,
                    size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        if ((centres == nullptr) != (labels == nullptr))
            return fail(HDF_ERR_ARG, "hdf_filter_hard: pass both centres and labels, or neither");
        if (labels && misaligned(labels)) return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
        return run_filter(f, n, p, rho, H, W, kind, sigma_s, radius, sigma_r, K, centres, 0.f, g, nullptr, ws,
                          ws_bytes, static_cast<cudaStream_t>(stream), true, labels);
    });
}

// ------------------------------------------------------------------ PCA-NLM guide (NEXT #3) ----
size_t hdf_pca_guide_workspace_bytes(int H, int W, int n, int m, int dim) {
    if (H < 1 || W < 1 || n < 1 || m < 1 || dim < 1) return 0;
    const int D = n * m * m;
    if (D > hdf::kPcaMaxD) return 0;
    Carver cv(nullptr);
    cv.take<double>((size_t)hdf::kPcaGrid * (D + D * (D + 1) / 2));
    cv.take<float>((size_t)hdf::kPcaMaxDim * D);
    cv.take<float>((size_t)D);
    cv.take<double>((size_t)hdf::kPcaMaxDim);
    return cv.off + 256;
}

static int pca_guide_impl(const float* f, int H, int W, int n, int m, int dim, float* p, float* basis_out, void* ws,
                          size_t ws_bytes, void* stream);
int hdf_pca_guide(const float* f, int H, int W, int n, int m, int dim, float* p, float* basis_out, void* ws,
                  size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int { return pca_guide_impl(f, H, W, n, m, dim, p, basis_out, ws, ws_bytes, stream); });
}
static int pca_guide_impl(const float* f, int H, int W, int n, int m, int dim, float* p, float* basis_out, void* ws,
                          size_t ws_bytes, void* stream) {
    if (!f || !p || !ws) return fail(HDF_ERR_ARG, "NULL pointer argument");
    if (H < 1 || W < 1 || n < 1) return fail(HDF_ERR_ARG, "H, W, n must be >= 1");
    if (m < 1 || m % 2 == 0) return fail(HDF_ERR_ARG, "patch side m must be odd and >= 1 (got %d)", m);
    const int D = n * m * m;
    if (D > hdf::kPcaMaxD) return fail(HDF_ERR_ARG, "patch dimension n m^2 = %d exceeds %d", D, hdf::kPcaMaxD);
    if (dim < 1 || dim > D || dim > hdf::kPcaMaxDim)
        return fail(HDF_ERR_ARG, "dim must be in [1, min(n m^2, %d)] (got %d)", hdf::kPcaMaxDim, dim);
    if (misaligned(f) || misaligned(p) || misaligned(ws)) return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
    const size_t need = hdf_pca_guide_workspace_bytes(H, W, n, m, dim);
    if (ws_bytes < need) return fail(HDF_ERR_WORKSPACE, "workspace %zu < required %zu bytes", ws_bytes, need);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver cv(ws);
    double* part = cv.take<double>((size_t)hdf::kPcaGrid * (D + D * (D + 1) / 2));
    hdf::PcaOut po;
    po.basis = cv.take<float>((size_t)hdf::kPcaMaxDim * D);
    po.mean = cv.take<float>((size_t)D);
    po.evals = cv.take<double>((size_t)hdf::kPcaMaxDim);
    const long long N = (long long)H * W;
    hdf::k_pca_moments<<<hdf::kPcaGrid, hdf::kPcaThreads, 0, st>>>(f, H, W, n, m, part);
    HDF_CUDA(cudaGetLastError());
    HDF_CUDA(cudaFuncSetAttribute(hdf::k_pca_eig, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)hdf::pca_eig_smem()));
    hdf::k_pca_eig<<<1, hdf::kPcaThreads, hdf::pca_eig_smem(), st>>>(part, hdf::kPcaGrid, D, dim, N, po);
    HDF_CUDA(cudaGetLastError());
    const unsigned nb = (unsigned)std::min<long long>((N + hdf::kPcaThreads - 1) / hdf::kPcaThreads, 148LL * 8);
    if (dim <= 8) hdf::k_pca_project<8><<<nb, hdf::kPcaThreads, 0, st>>>(f, H, W, n, m, dim, po.basis, po.mean, p);
    else if (dim <= 16)
        hdf::k_pca_project<16><<<nb, hdf::kPcaThreads, 0, st>>>(f, H, W, n, m, dim, po.basis, po.mean, p);
    else hdf::k_pca_project<32><<<nb, hdf::kPcaThreads, 0, st>>>(f, H, W, n, m, dim, po.basis, po.mean, p);
    HDF_CUDA(cudaGetLastError());
    if (basis_out)
        HDF_CUDA(cudaMemcpyAsync(basis_out, po.basis, sizeof(float) * (size_t)dim * D, cudaMemcpyDeviceToDevice, st));
    return HDF_OK;
}

int hdf_sample_guide(const float* p, long long N, int rho, long long i0, long long stride, float* out, long long M,
                     void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        if (!p || !out) return fail(HDF_ERR_ARG, "NULL pointer argument");
        if (rho < 1 || rho > HDF_MAX_RHO) return fail(HDF_ERR_ARG, "rho must be in [1, %d]", HDF_MAX_RHO);
        if (N < 1 || stride < 1 || i0 < 0 || M < 0) return fail(HDF_ERR_ARG, "need N >= 1, stride >= 1, i0, M >= 0");
        if (M > 0 && i0 + (M - 1) * stride >= N) return fail(HDF_ERR_ARG, "the sample runs past the guide");
        if (M == 0) return HDF_OK;
        const unsigned nb =
            (unsigned)std::min<long long>((M * rho + 255) / 256, (long long)nsm_of_device() * 16);
        hdf::k_sample_guide<<<nb, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, rho, i0, stride, out, M);
        HDF_CUDA(cudaGetLastError());
        return HDF_OK;
    });
}

size_t hdf_cluster_sampled_workspace_bytes(int H, int W, int rho, int K, int stride) {
    if (H < 1 || W < 1 || rho < 1 || K < 1 || stride < 1) return 0;
    const long long N = (long long)H * W, M = (N + stride - 1) / stride;
    if (M > (1LL << 30)) return 0;
    Carver cv(nullptr);
    cv.take<float>((size_t)M * rho + 4);
    return cv.off + 256 + hdf_cluster_workspace_bytes(1, (int)M, rho, K);
}

int hdf_cluster_sampled(const float* p, int H, int W, int rho, int K, int stride, float* centres,
                        hdf_cluster_info* info_host, void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        int rc = check_common(H, W, rho, K);
        if (rc) return rc;
        if (stride < 1) return fail(HDF_ERR_ARG, "stride must be >= 1 (got %d)", stride);
        if (!p || !centres || !ws) return fail(HDF_ERR_ARG, "NULL pointer argument");
        if (misaligned(p) || misaligned(centres) || misaligned(ws))
            return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
        const size_t need = hdf_cluster_sampled_workspace_bytes(H, W, rho, K, stride);
        if (ws_bytes < need) return fail(HDF_ERR_WORKSPACE, "workspace %zu < required %zu bytes", ws_bytes, need);
        const long long N = (long long)H * W, M = (N + stride - 1) / stride;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        Carver cv(ws);
        float* smp = cv.take<float>((size_t)M * rho + 4);
        cv.off = (cv.off + 255) & ~size_t(255);
        void* cws = cv.base + cv.off;
        if (stride == 1) {
            smp = const_cast<float*>(p);   // the exact procedure on the whole guide
        } else {
            const unsigned nb = (unsigned)std::min<long long>((M * rho + 255) / 256, (long long)nsm_of_device() * 16);
            hdf::k_sample_guide<<<nb, 256, 0, st>>>(p, rho, 0, stride, smp, M);
            HDF_CUDA(cudaGetLastError());
        }
        return launch_cluster(smp, 1, (int)M, rho, K, centres, nullptr, info_host, cws, st);
    });
}

int hdf_scale_guide(const float* p, int H, int W, int rho, const float* scale_host, const float* extra, int e,
                    const float* extra_scale_host, float* out, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        if (!p || !out) return fail(HDF_ERR_ARG, "NULL pointer argument");
        if (H < 1 || W < 1) return fail(HDF_ERR_ARG, "H, W must be >= 1");
        if (rho < 1 || e < 0 || rho + e > HDF_MAX_RHO)
            return fail(HDF_ERR_ARG, "rho >= 1, e >= 0 and rho + e <= %d required (got %d, %d)", HDF_MAX_RHO, rho, e);
        if (e > 0 && !extra) return fail(HDF_ERR_ARG, "extra is NULL with e = %d", e);
        if (misaligned(p) || misaligned(out) || (extra && misaligned(extra)))
            return fail(HDF_ERR_ARG, "device pointers must be 16-byte aligned");
        if (out == p || (extra && out == extra)) return fail(HDF_ERR_ARG, "out must not alias p or extra");
        hdf::ScaleParams sp;
        sp.p = p;
        sp.extra = e > 0 ? extra : nullptr;
        sp.out = out;
        sp.N = (long long)H * W;
        sp.rho = rho;
        sp.e = e;
        for (int d = 0; d < HDF_MAX_RHO; d++) sp.s[d] = 0.f;
        for (int d = 0; d < rho; d++) sp.s[d] = scale_host ? scale_host[d] : 1.f;
        for (int j = 0; j < e; j++) sp.s[rho + j] = extra_scale_host ? extra_scale_host[j] : 1.f;
        for (int d = 0; d < rho + e; d++)
            if (!std::isfinite(sp.s[d])) return fail(HDF_ERR_ARG, "scale %d is not finite", d);
        const long long tot = sp.N * (rho + e);
        const unsigned nb = (unsigned)std::min<long long>((tot + 255) / 256, (long long)nsm_of_device() * 16);
        hdf::k_scale_guide<<<nb, 256, 0, static_cast<cudaStream_t>(stream)>>>(sp);
        HDF_CUDA(cudaGetLastError());
        return HDF_OK;
    });
}

size_t hdf_filter_host_workspace_bytes(int H, int W, int n, int rho, int K, int kind, float sigma_s, int radius) {
    const size_t base = hdf_filter_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius);
    if (!base) return 0;
    Carver cv(nullptr);
    cv.take<float>((size_t)H * W * n);
    cv.take<float>((size_t)H * W * rho);
    cv.take<float>((size_t)H * W * n);
    cv.take<float>((size_t)K * rho);
    cv.take<float>((size_t)H * W * rho);   // the stride sample (cluster_stride > 1)
    return base + cv.off + 256;
}

int hdf_filter_host(const float* f_host, int n, const float* p_host, int rho, int H, int W, int kind, float sigma_s,
                    int radius, float sigma_r, int K, float tau, int cluster_stride, float* g_host, float* centres_host,
                    int32_t* n_flagged_host, hdf_cluster_info* info_host, void* ws, size_t ws_bytes, void* stream) {
    g_err.clear();
    return guarded([&]() -> int {
        // every argument is checked before the first copy is enqueued
        const bool f_is_p = (p_host == f_host && rho == n);
        FilterPlan F;
        size_t vsmem = 0;
        int rc = validate_scalars(n, rho, H, W, kind, sigma_r, K, tau, false);
        if (rc) return rc;
        if (!f_host || !p_host || !g_host || !ws) return fail(HDF_ERR_ARG, "NULL pointer argument");
        if (misaligned(ws)) return fail(HDF_ERR_ARG, "the workspace must be 16-byte aligned");
        if (cluster_stride < 1) return fail(HDF_ERR_ARG, "cluster_stride must be >= 1 (got %d)", cluster_stride);
        rc = validate_filter(n, rho, H, W, kind, sigma_s, radius, sigma_r, K, tau, f_is_p, false, &F, &vsmem);
        if (rc) return rc;
        const size_t need = hdf_filter_host_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius);
        if (ws_bytes < need) return fail(HDF_ERR_WORKSPACE, "workspace %zu < required %zu bytes", ws_bytes, need);
        HostStage* hs = host_stage();
        if (!hs) return fail(HDF_ERR_CUDA, "pinned host stage: cudaMallocHost failed");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        Carver cv(ws);
        const size_t fbytes = hdf_filter_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius);
        void* fws = cv.take<char>(fbytes);
        float* fd = cv.take<float>((size_t)H * W * n);
        float* pd = cv.take<float>((size_t)H * W * rho);
        float* gd = cv.take<float>((size_t)H * W * n);
        float* cd = cv.take<float>((size_t)K * rho);
        float* smp = cv.take<float>((size_t)H * W * rho);
        const float* pdev = fd;
        // from here on, a failure synchronises the stream before returning (copies from the caller's
        // buffers may be in flight)
        cudaStream_t cs = copy_stream();
        if (!cs) return fail(HDF_ERR_CUDA, "copy stream creation failed");
        auto bail = [&](int code) {
            cudaStreamSynchronize(st);
            cudaStreamSynchronize(cs);
            return code;
        };
        const bool sampled = cluster_stride > 1;
        // Sampled mode: the bulk input copy runs on the copy stream while the caller's stream copies the
        // stride sample straight from the host guide (one strided 2-D copy) and clusters it, so the
        // clustering is hidden under the bulk copy; the filter waits for both.  Exact mode: the copy, then
        // the clustering of every pixel, in order on the caller's stream.
        // The bulk copy goes in kInChunks row chunks, each followed by an event: the tensor-core column pass runs in
        // row bands, each as soon as its rows (+ R halo rows) are on the device (run_filter, before_rows), so most of
        // the input copy is hidden under the column pass instead of preceding it.
        constexpr int kInChunks = 8;
        const bool in_chunked = sampled && (long long)H * W >= (1LL << 20);
        const int nin = in_chunked ? std::min(kInChunks, H) : 1;
        cudaEvent_t ev_fork = nullptr, ev_in = nullptr, ev_rows[kInChunks] = {};
        auto destroy_io = [&]() {
            if (ev_fork) cudaEventDestroy(ev_fork);
            if (ev_in) cudaEventDestroy(ev_in);
            for (int c = 0; c < kInChunks; c++)
                if (ev_rows[c]) cudaEventDestroy(ev_rows[c]);
            ev_fork = ev_in = nullptr;
            for (int c = 0; c < kInChunks; c++) ev_rows[c] = nullptr;
        };
        auto in_row = [&](int c) { return (int)((long long)H * c / nin); };   // first row of input chunk c
        cudaStream_t in_st = st;
        if (sampled) {
            bool ok = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                      cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming) == cudaSuccess;
            for (int c = 0; ok && in_chunked && c < nin; c++)
                ok = cudaEventCreateWithFlags(&ev_rows[c], cudaEventDisableTiming) == cudaSuccess;
            if (!ok) {
                destroy_io();
                return bail(fail(HDF_ERR_CUDA, "event creation failed"));
            }
            cudaEventRecord(ev_fork, st);   // the copy stream starts after the caller's earlier work
            cudaStreamWaitEvent(cs, ev_fork, 0);
            in_st = cs;
        }
        {
            ProfScope prof(HDF_STAGE_H2D, in_st);
            for (int c = 0; c < nin; c++) {
                const size_t r0 = (size_t)in_row(c), r1 = (size_t)in_row(c + 1);
                if (cudaMemcpyAsync(fd + r0 * W * n, f_host + r0 * W * n, sizeof(float) * (r1 - r0) * W * n,
                                    cudaMemcpyHostToDevice, in_st) != cudaSuccess) {
                    destroy_io();
                    return bail(fail(HDF_ERR_CUDA, "input copy: %s", cudaGetErrorString(cudaGetLastError())));
                }
                if (!f_is_p) {
                    if (cudaMemcpyAsync(pd + r0 * W * rho, p_host + r0 * W * rho, sizeof(float) * (r1 - r0) * W * rho,
                                        cudaMemcpyHostToDevice, in_st) != cudaSuccess) {
                        destroy_io();
                        return bail(fail(HDF_ERR_CUDA, "guide copy: %s", cudaGetErrorString(cudaGetLastError())));
                    }
                }
                if (in_chunked) cudaEventRecord(ev_rows[c], in_st);
            }
            if (!f_is_p) pdev = pd;
        }
        if (sampled) cudaEventRecord(ev_in, cs);
        // cluster (in the filter workspace's cluster region; status read back at the end) then filter
        Carver c2(fws);
        FilterWS w = carve_filter(c2, H, W, n, rho, K, round_up(W, 32), true);
        ClusterReadback crb;
        if (!sampled) {
            rc = launch_cluster(pdev, H, W, rho, K, cd, nullptr, nullptr, w.cluster_ws, st, &crb);
        } else {   // the sampled mode (hdf_cluster_sampled): the stride sample p.flat[0::s], then the same procedure
            const long long N = (long long)H * W, M = (N + cluster_stride - 1) / cluster_stride;
            {
                ProfScope prof(HDF_STAGE_H2D, st);
                // Pinned (or registered) host memory is addressable from the device: k_sample_guide then gathers the
                // sample straight out of the caller's buffer over PCIe (M short reads in flight at once) instead of a
                // strided 2-D DMA copy of M rho-float rows (~4 ms for 262k rows at config 5).  HDF_HOST_SAMPLE_DMA=1 or
                // pageable memory keeps the 2-D copy.
                const float* p_dev_view = nullptr;
                if (!getenv_on("HDF_HOST_SAMPLE_DMA")) {
                    cudaPointerAttributes pa;
                    if (cudaPointerGetAttributes(&pa, p_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        pa.devicePointer)
                        p_dev_view = static_cast<const float*>(pa.devicePointer);
                    else
                        cudaGetLastError();   // (pageable memory: not an error here)
                }
                if (p_dev_view) {
                    const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((M * rho + 255) / 256, 1184));
                    hdf::k_sample_guide<<<nb, 256, 0, st>>>(p_dev_view, rho, 0, cluster_stride, smp, M);
                    if (cudaGetLastError() != cudaSuccess) {
                        destroy_io();
                        return bail(fail(HDF_ERR_CUDA, "sample gather launch failed"));
                    }
                } else if (cudaMemcpy2DAsync(smp, sizeof(float) * (size_t)rho, p_host,
                                             sizeof(float) * (size_t)rho * cluster_stride, sizeof(float) * (size_t)rho,
                                             (size_t)M, cudaMemcpyHostToDevice, st) != cudaSuccess) {
                    destroy_io();
                    return bail(fail(HDF_ERR_CUDA, "sample copy: %s", cudaGetErrorString(cudaGetLastError())));
                }
            }
            rc = launch_cluster(smp, 1, (int)M, rho, K, cd, nullptr, nullptr, w.cluster_ws, st, &crb);
            if (!rc && !in_chunked) cudaStreamWaitEvent(st, ev_in, 0);   // the filter needs the whole input
        }
        if (rc) {
            destroy_io();
            return bail(rc);
        }
        // rows [0, y_end) are on the device once the chunk holding row y_end - 1 has been copied
        RowsFn before_rows;
        if (in_chunked)
            before_rows = [&](int y_end, cudaStream_t s) -> int {
                int c = 0;
                while (c + 1 < nin && in_row(c + 1) < y_end) c++;
                HDF_CUDA(cudaStreamWaitEvent(s, ev_rows[c], 0));
                return HDF_OK;
            };
        // the output rows are copied out chunk by chunk on the copy stream while the row pass continues
        constexpr int kChunks = 8;
        cudaEvent_t evs[kChunks];
        int nev = 0;
        auto release = [&]() {
            for (int e = 0; e < nev; e++) cudaEventDestroy(evs[e]);
            nev = 0;
        };
        const size_t rowf = (size_t)W * n;
        const bool chunked = (long long)H * W >= (1LL << 20);   // small images: one copy after the filter
        auto after = [&](int y0, int y1, cudaStream_t s) -> int {
            if (nev >= kChunks) return fail(HDF_ERR_CUDA, "too many output chunks");
            cudaEvent_t ev;
            HDF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            evs[nev++] = ev;
            HDF_CUDA(cudaEventRecord(ev, s));
            HDF_CUDA(cudaStreamWaitEvent(cs, ev, 0));
            ProfScope prof(HDF_STAGE_D2H, cs);
            HDF_CUDA(cudaMemcpyAsync(g_host + (size_t)y0 * rowf, gd + (size_t)y0 * rowf, sizeof(float) * (size_t)(y1 - y0) * rowf,
                                     cudaMemcpyDeviceToHost, cs));
            return HDF_OK;
        };
        rc = run_filter(fd, n, pdev, rho, H, W, kind, sigma_s, radius, sigma_r, K, cd, tau, gd, nullptr, fws, fbytes,
                        st, false, nullptr, chunked ? kChunks : 1, after, before_rows, in_chunked ? 4 : 1);
        destroy_io();   // (destroying a recorded event is safe: the waits were already enqueued)
        if (rc) {
            cudaStreamSynchronize(cs);
            release();
            return bail(rc);
        }
        {
            cudaError_t e = cudaSuccess;
            if (centres_host)
                e = cudaMemcpyAsync(centres_host, cd, sizeof(float) * (size_t)K * rho, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(hs->hv, w.status, sizeof(hs->hv), cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) {
                cudaStreamSynchronize(cs);
                release();
                return bail(fail(HDF_ERR_CUDA, "output copy: %s", cudaGetErrorString(e)));
            }
        }
        // the caller's stream ends after the last copy (its events / a later sync see the whole call)
        cudaEvent_t done;
        if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(done, cs);
            cudaStreamWaitEvent(st, done, 0);
            cudaEventDestroy(done);
        }
        const cudaError_t se = cudaStreamSynchronize(st);
        cudaStreamSynchronize(cs);
        release();
        if (se != cudaSuccess) return fail(HDF_ERR_CUDA, "stream: %s", cudaGetErrorString(se));
        if (n_flagged_host) *n_flagged_host = hs->hv[1];
        rc = cluster_status(crb, K, info_host);   // HDF_ERR_K: g_host holds the padded-centre result
        if (rc) return rc;
        if (hs->hv[0] == HDF_WARN_ILLCOND)
            return fail(HDF_WARN_ILLCOND, "A is numerically singular; A^+ truncated (R6)");
        return HDF_OK;
    });
}

// Diagnostics / parity tests: the pixels that took the R9 fallback in the last hdf_filter call on
// workspace `ws` with the same sizes (synchronous).  Returns their number (at most cap copied, in the
// order the row pass flagged them), or -1 on a CUDA error.
int hdf_filter_flagged(const void* ws, int H, int W, int n, int rho, int K, int32_t* idx_host, int cap) {
    g_err.clear();
    return guarded([&]() -> int {
        if (!ws || H < 1 || W < 1 || n < 1 || rho < 1 || K < 1) return -1;
        Carver cv(const_cast<void*>(ws));
        FilterWS w = carve_filter(cv, H, W, n, rho, K, round_up(W, 32), true);
        int cnt = 0;
        if (cudaMemcpy(&cnt, w.flag_count, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
        const int m = std::min(cnt, std::max(cap, 0));
        if (m > 0 && idx_host &&
            cudaMemcpy(idx_host, w.flag_list, sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToHost) != cudaSuccess)
            return -1;
        return cnt;
    });
}

}  // extern "C"
