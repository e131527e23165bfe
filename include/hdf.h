/*
 * hdf.h -- C ABI of the B200 (sm_100a) implementation of the fast high-dimensional bilateral /
 * nonlocal-means filter of Nair & Chaudhury (arXiv 1811.02363).
 *
 * Citations "P:n" are lines of the paper's text; "Rn" are the readings of the paper
 * listed in DESIGN.md section 3.  Every entry point below is plain C: device or host pointers,
 * sizes and a CUDA stream passed as void* (a cudaStream_t; NULL = legacy default stream).
 *
 * Conventions (all entry points):
 *  - Layout.  Images are row-major, channel-fastest ("HWC"): f [H][W][n], p [H][W][rho],
 *    g [H][W][n], float32.  Centres are [K][rho] float32.  Pixel (y, x) is index y*W + x.
 *  - Ownership.  The caller owns every buffer (inputs, outputs, workspace).  The library never
 *    allocates or frees device memory, and keeps no pointer after the enqueued work completes.
 *    Device buffers must stay alive until the stream has reached the end of the enqueued work.
 *  - Alignment.  Device pointers must be 16-byte aligned (torch allocations are 512-byte aligned).
 *  - Aliasing.  f may alias p (the bilateral filter, f = p).  g must not alias f, p or ws.
 *  - Asynchrony.  Calls enqueue work on `stream` and return without waiting, except where an
 *    optional *_host output pointer is non-NULL (documented per call): then the call
 *    synchronises `stream` before returning.  Argument errors are detected before anything is
 *    enqueued; nothing is launched on error.
 *  - Errors.  Every call returns an hdf_status.  hdf_last_error() gives a message for the last
 *    failing call on the calling thread.  Launch failures map to HDF_ERR_CUDA; asynchronous device
 *    faults surface at the caller's next synchronisation.
 *  - Finite inputs are a precondition and are not checked.
 *  - There is no CPU fallback: every arithmetic step runs in this library's CUDA kernels.
 */
#ifndef HDF_H_
#define HDF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HDF_OK = 0,
    HDF_ERR_ARG = 1,        /* invalid argument (shape, range, NULL, alignment, aliasing) */
    HDF_ERR_K = 2,          /* K exceeds the number of distinct guide vectors (R5)          */
    HDF_ERR_WORKSPACE = 3,  /* ws_bytes smaller than the *_workspace_bytes() requirement    */
    HDF_ERR_CUDA = 4,       /* a CUDA runtime call or launch failed                          */
    HDF_WARN_ILLCOND = 5    /* A (defAb) is numerically singular: A^+ truncated (R6)         */
} hdf_status;

typedef enum {
    HDF_SPATIAL_GAUSSIAN = 0, /* omega(i) = exp(-||i||^2 / 2 sigma_s^2) on [-S,S]^2 */
    HDF_SPATIAL_BOX = 1,      /* omega = 1 on [-S,S]^2 (nonlocal means)                 */
    HDF_SPATIAL_GAUSSIAN_IIR = 2 /* Young's O(1) recursive Gaussian, the paper's implementation of
                                    the Gaussian convolutions; 0.5 <= sigma_s <= 4096; zero
                                    outside the image, gain sqrt(2 pi) sigma_s per axis so that
                                    omega(0) ~ 1 (DESIGN R17); `radius` (or ceil(3 sigma_s)) only
                                    sizes the R9 fallback's direct window sum (exact FIR Gaussian,
                                    radius <= 512) */
} hdf_spatial_kind;

/* Limits of this build. */
#define HDF_MAX_K 128
#define HDF_MAX_RHO 64
#define HDF_MAX_N 64
#define HDF_MAX_RADIUS 32

/* Library version string, e.g. "hdf 0.1.0 sm_100a". */
const char *hdf_version(void);

/* Message of the last failing hdf_* call on this thread ("" if none).  Valid until the next
 * hdf_* call on the same thread. */
const char *hdf_last_error(void);

/* ---------------------------------------------------------------------------------------------
 * Step 1 -- cluster the range space Theta = {p(i)} (Algorithm 1 line "cluster" P:294)
 * with bisecting K-means: repeatedly split the leaf of largest SSE (R2) by 2-means seeded with the
 * farthest pair of a stride sample of <= 1024 members (R3), Lloyd iterations until no assignment
 * changes or 50 iterations (R4).  mu_k = centroid of C_k.  Runs as one persistent
 * cooperative kernel that expands the tree of splits best-first in parallel (thread-block clusters
 * as workers); the result is the sequential procedure's.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    int32_t status;          /* HDF_OK or HDF_ERR_K                                              */
    int32_t achievable_k;    /* leaves reached; the number of distinct guide vectors on HDF_ERR_K */
    int32_t splits_computed; /* 2-means splits computed, including speculative ones not needed   */
    int32_t lloyd_iters;     /* Lloyd passes executed over all computed splits                   */
    double e_k;              /* clustering error E_K = sum_k sum_{p(i) in C_k} ||p(i)-mu_k||^2     */
    int32_t grid_splits;     /* splits computed by the whole grid (nodes larger than a cluster)    */
    int32_t tile_points;     /* guide vectors a CTA keeps resident in shared memory                */
    int32_t launch_ctas;     /* CTAs of the cooperative launch                                      */
    int32_t cluster_ctas;    /* CTAs per thread-block cluster (one worker)                          */
    int64_t point_passes;    /* sum over the K-1 splits of the procedure: members x Lloyd passes    */
    int64_t points_split;    /* sum over the K-1 splits of the procedure: members                   */
} hdf_cluster_info;

/* ---------------------------------------------------------------------------------------------
 * Sampled clustering mode.  The paper notes that "any efficient clustering method" can provide the
 * centres.  hdf_cluster_sampled runs the same bisecting K-means (R2-R4) on the stride sample
 * {p(i) : i = 0, s, 2s, ...} of the pixels (flat index order) instead of all of them: mu_k are the
 * leaf means of the sample.  stride = 1 is hdf_cluster exactly.  Its quality is checked by the R15
 * rule (error against brute force within 5% of the exact oracle pipeline's, tests/test_gpu_cluster.py);
 * on the sample itself the result equals the oracle's bisecting K-means of the same sample.
 *   stride   s >= 1; the sample has M = ceil(H W / s) points
 *   info_host  as hdf_cluster (E_K, labels are those of the SAMPLE)
 *   ws         at least hdf_cluster_sampled_workspace_bytes(H, W, rho, K, stride)
 * Errors as hdf_cluster.
 * hdf_sample_guide: the gather on its own (the multi-GPU split gathers each rank's share of the
 * global sample, strips.py): out[j] = p[i0 + j stride], j < M, rho floats each; device pointers;
 * HDF_ERR_ARG if the sample runs past N; asynchronous.
 * ------------------------------------------------------------------------------------------- */
size_t hdf_cluster_sampled_workspace_bytes(int H, int W, int rho, int K, int stride);
int hdf_cluster_sampled(const float *p, int H, int W, int rho, int K, int stride, float *centres,
                        hdf_cluster_info *info_host, void *ws, size_t ws_bytes, void *stream);
int hdf_sample_guide(const float *p, long long N, int rho, long long i0, long long stride, float *out, long long M,
                     void *stream);

/* Device workspace (bytes) for hdf_cluster on an H x W guide of dimension rho. */
size_t hdf_cluster_workspace_bytes(int H, int W, int rho, int K);

/*
 * hdf_cluster
 *   p        [H][W][rho] float32, device (read only)
 *   K        1 <= K <= HDF_MAX_K number of clusters
 *   centres  [K][rho] float32, device, out: mu_k (rounded from fp64 means)
 *   labels   [H][W] int32, device, out: k such that p(i) in C_k; may be NULL
 *   info_host  hdf_cluster_info*, host, out; may be NULL.  Non-NULL synchronises `stream` and
 *              returns HDF_ERR_K if K exceeds the number of distinct guide vectors (R5).  With
 *              NULL the call is fully asynchronous and, in that (documented) error case, centres
 *              k >= achievable_k are copies of centre 0 (A then has duplicate centres and the
 *              pseudo-inverse handles the rank deficiency, R6).
 *   ws, ws_bytes  device workspace of at least hdf_cluster_workspace_bytes(H, W, rho, K)
 *   stream   cudaStream_t as void*
 */
int hdf_cluster(const float *p, int H, int W, int rho, int K, float *centres, int32_t *labels,
                hdf_cluster_info *info_host, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------------
 * Steps 2-6 -- Algorithm 1:
 *   A_kl = phi(mu_k - mu_l), A^+ (P:235-240);
 *   b_k(j) = phi(p(j) - mu_k), u_k = b_k f;
 *   v_k = omega * u_k, r_k = omega * b_k: K(n+1) separable convolutions, window clipped to Omega
 *   (zero extension, R8);
 *   c(i) = A^+ b(i); g(i) = sum_k c_k v_k / sum_k c_k r_k.
 * Degenerate normaliser (R9): if eta_hat(i) = sum_k c_k r_k < tau * omega(0) phi(0), g(i) is
 * replaced by the direct (num)/(den) value of P:43-51 at i, computed on the GPU.
 * ------------------------------------------------------------------------------------------- */

/* Device workspace (bytes) for hdf_filter.  radius < 0 means ceil(3 sigma_s) (Gaussian). */
size_t hdf_filter_workspace_bytes(int H, int W, int n, int rho, int K, int kind, float sigma_s, int radius);

/*
 * hdf_filter
 *   f        [H][W][n] float32, device (read only), 1 <= n <= HDF_MAX_N
 *   p        [H][W][rho] float32, device (read only), 1 <= rho <= HDF_MAX_RHO; may alias f
 *   kind     hdf_spatial_kind
 *   sigma_s  Gaussian spatial sigma (> 0; ignored for the box)
 *   radius   window half-width S; < 0 -> ceil(3 sigma_s) for the Gaussian; required for the
 *            box; 0 <= S <= HDF_MAX_RADIUS
 *   sigma_r  range sigma (> 0), phi(x) = exp(-||x||^2 / 2 sigma_r^2)
 *   K        number of centres, 1 <= K <= HDF_MAX_K
 *   Working-set limit: the column pass keeps 2 J rows of (rho, or rho + n when f is not p) floats for
 *   32 columns in shared memory (J = rows per step, 2..16 with the radius), so large rho + n need a
 *   small radius (e.g. rho + n = 67 works up to radius 2, rho + n = 6 up to 32); beyond that the call
 *   returns HDF_ERR_ARG before launching anything.
 *   centres  [K][rho] float32, device; NULL -> hdf_cluster is run first inside this call (then
 *            ws must also hold the clustering workspace, which hdf_filter_workspace_bytes includes)
 *   tau      degenerate-normaliser threshold (R9); 0 disables the rule; callers pass 0.5
 *   g        [H][W][n] float32, device, out
 *   n_flagged_host  int32*, host, out: number of pixels that took the R9 fallback; may be NULL.
 *            Non-NULL synchronises `stream` once, at the end of the call, and the call then reports
 *            what happened on the device: HDF_ERR_K (centres == NULL and K exceeds the number of
 *            distinct guide vectors, R5: g holds the result with the padded centres of hdf_cluster),
 *            HDF_ERR_CUDA (the clustering kernel failed), else HDF_WARN_ILLCOND when A was
 *            numerically singular (its pseudo-inverse truncated eigenvalues below tol, R6), else
 *            HDF_OK.  With NULL the call is fully asynchronous and reports argument errors only.
 *   ws, ws_bytes  device workspace of at least hdf_filter_workspace_bytes(...)
 *   stream   cudaStream_t as void*
 * Threads: calls from several host threads are safe (errors are per thread).  The pseudo-inverse
 * kernel runs on a library-owned side stream per device, forked from and joined back to `stream` by
 * events under a per-device lock; calls on different streams therefore serialise their (small)
 * pseudo-inverse kernels on that side stream.
 */
int hdf_filter(const float *f, int n, const float *p, int rho, int H, int W, int kind, float sigma_s,
               int radius, float sigma_r, int K, const float *centres, float tau, float *g,
               int32_t *n_flagged_host, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------------
 * hdf_pca_guide -- PCA-NLM guide on the GPU (reading R11).
 *   p(i) = the m x m patch of f around i, all n channels (D = n m^2 values, channel-major then rows
 *   then columns; replicate borders), minus the mean patch, projected on the `dim` leading
 *   eigenvectors of the patch covariance (fp64 moments and Jacobi eigen-decomposition; descending
 *   eigenvalues; each eigenvector signed so that its entry of largest magnitude is positive).
 *   f          [H][W][n] float32, device (read only)
 *   m          odd patch side; D = n m^2 <= 64
 *   dim        1 <= dim <= min(D, 32)
 *   p          [H][W][dim] float32, device, out: the guide (usable as hdf_filter's p)
 *   basis_out  [dim][D] float32, device, out (or NULL): the projection basis
 *   ws         device workspace of at least hdf_pca_guide_workspace_bytes(H, W, n, m, dim)
 * Errors: HDF_ERR_ARG (sizes, NULL, alignment), HDF_ERR_WORKSPACE; asynchronous on `stream`.
 */
size_t hdf_pca_guide_workspace_bytes(int H, int W, int n, int m, int dim);
int hdf_pca_guide(const float *f, int H, int W, int n, int m, int dim, float *p, float *basis_out, void *ws,
                  size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------------
 * hdf_scale_guide -- anisotropic and augmented guides.
 * The diagonal range kernel phi(x) = exp(-sum_d x_d^2 / 2 sigma_d^2) is the isotropic kernel with
 * sigma_r = 1 on the guide scaled per channel by 1 / sigma_d; an extra guide channel (the paper's
 * infrared band) is appended with its own scale.  Pass the result to hdf_cluster /
 * hdf_filter with sigma_r = 1.
 *   out(i) = (p(i)_d * scale[d])_{d < rho} ++ (extra(i)_j * extra_scale[j])_{j < e}
 *   p      [H][W][rho] float32, device (read only)
 *   scale_host        [rho] float32, host (NULL: all 1)
 *   extra  [H][W][e] float32, device, or NULL when e = 0
 *   extra_scale_host  [e] float32, host (NULL: all 1)
 *   out    [H][W][rho + e] float32, device, out; rho + e <= HDF_MAX_RHO; must not alias p or extra
 * Errors: HDF_ERR_ARG (sizes, NULL, alignment, aliasing, a non-finite scale); asynchronous on `stream`.
 */
int hdf_scale_guide(const float *p, int H, int W, int rho, const float *scale_host, const float *extra, int e,
                    const float *extra_scale_host, float *out, void *stream);

/* ---------------------------------------------------------------------------------------------
 * hdf_filter_hard -- the hard-assignment variant (coeffICIP)/(HDapprox2): every pixel keeps
 * only its own cluster's term, g(i) = v_s(i) / r_s(i) with s = label(i) (no pseudo-inverse, no
 * fallback: r_s(i) >= omega(0) phi(p(i) - mu_s) > 0).  Theorem 1 bounds its error
 * against the exact filter by C L^2 n |W|^2 E_K.
 *   centres, labels  [K][rho] float32 and [H][W] int32 (values in [0, K)), device: both given (e.g.
 *                    from hdf_cluster) or both NULL (clustering runs inside the call, labels kept in
 *                    the workspace); HDF_ERR_ARG otherwise
 *   kind             HDF_SPATIAL_GAUSSIAN or HDF_SPATIAL_BOX (HDF_ERR_ARG for the recursive Gaussian)
 *   other arguments, workspace (hdf_filter_workspace_bytes) and errors as hdf_filter; asynchronous.
 */
int hdf_filter_hard(const float *f, int n, const float *p, int rho, int H, int W, int kind, float sigma_s,
                    int radius, float sigma_r, int K, const float *centres, const int32_t *labels, float *g,
                    void *ws, size_t ws_bytes, void *stream);

/*
 * hdf_filter_host -- the whole hot path end to end from HOST buffers: copies f and p to the device
 * workspace, clusters, filters, and copies g back, all on `stream`, then synchronises it once.
 *   f_host [H][W][n], p_host [H][W][rho] (may be the same pointer), g_host [H][W][n]: host float32
 *   (pinned memory gives full-rate copies; pageable memory works but is slower).  With cluster_stride > 1 on
 *   images of 2^20 pixels or more the input is copied in row chunks and the tensor-core column pass starts on
 *   the rows that have arrived (same result: the planes' power-of-two scale is then taken per row band), and the
 *   stride sample is gathered straight from p_host by a kernel when that memory is pinned (device-addressable).
 *   cluster_stride  1: the exact clustering of every pixel (hdf_cluster); s > 1: the sampled mode
 *            (hdf_cluster_sampled with stride s)
 *   centres_host [K][rho] out, may be NULL.  n_flagged_host, info_host: out, may be NULL.
 *   ws: device workspace of at least hdf_filter_host_workspace_bytes(...).
 * Every argument is checked before the first copy is enqueued (HDF_ERR_ARG / HDF_ERR_WORKSPACE,
 * nothing enqueued).  A failure after that synchronises `stream` before returning.  Returns HDF_OK,
 * HDF_ERR_K (K exceeds the number of distinct guide vectors, R5; g_host then holds the result with
 * the padded centres), HDF_ERR_CUDA, or HDF_WARN_ILLCOND (A^+ truncated, R6; g_host is valid).
 * The status words are read back through a few bytes of pinned host memory per calling thread
 * (allocated by the library on first use), so the call does not block mid-way.
 */
size_t hdf_filter_host_workspace_bytes(int H, int W, int n, int rho, int K, int kind, float sigma_s, int radius);
int hdf_filter_host(const float *f_host, int n, const float *p_host, int rho, int H, int W, int kind,
                    float sigma_s, int radius, float sigma_r, int K, float tau, int cluster_stride, float *g_host,
                    float *centres_host, int32_t *n_flagged_host, hdf_cluster_info *info_host,
                    void *ws, size_t ws_bytes, void *stream);

/*
 * hdf_filter_flagged -- diagnostics and parity tests: the pixels (index y*W + x) that took the R9
 * fallback in the last hdf_filter / hdf_filter_hard call that used workspace `ws` with the same
 * H, W, n, rho, K.  Synchronous (device -> host copies).  Copies at most `cap` indices into idx_host
 * (host, may be NULL when cap is 0), in the order the row pass flagged them (not sorted); returns the
 * number of flagged pixels, or -1 on a CUDA error or a NULL workspace.
 */
int hdf_filter_flagged(const void *ws, int H, int W, int n, int rho, int K, int32_t *idx_host, int cap);

/* ---------------------------------------------------------------------------------------------
 * Per-stage device timing (benchmarking / tracing).  When enabled, every
 * stage of hdf_cluster / hdf_filter / hdf_filter_host records a pair of CUDA events on the call's
 * stream around its kernel launch (or copy).
 * ------------------------------------------------------------------------------------------- */
typedef enum {
    HDF_STAGE_CLUSTER = 0,   /* k_bisect_kmeans                        step 1               */
    HDF_STAGE_PINV = 1,      /* k_gram_pinv                            step 2               */
    HDF_STAGE_COEFFS = 2,    /* k_coeffs: c = A^+ b planes             step 5 (for2)        */
    HDF_STAGE_VPASS = 3,     /* k_range_vpass: b, u + column pass      steps 3, 4           */
    HDF_STAGE_HPASS = 4,     /* k_hpass_combine: row pass + combine    steps 4, 6           */
    HDF_STAGE_FALLBACK = 5,  /* k_fallback: direct (num)/(den), R9     step 6               */
    HDF_STAGE_H2D = 6,       /* hdf_filter_host input copies                                */
    HDF_STAGE_D2H = 7,       /* hdf_filter_host output copies                               */
    HDF_STAGE_FILTER = 8,    /* the whole filter (steps 3-6, all of the above but the       */
                             /* clustering): wall time on the call's stream, which covers   */
                             /* the pipelined column / row passes' overlap                  */
    HDF_NUM_STAGES = 9
} hdf_stage;

/* Diagnostics: events recorded by the clustering workers during the last hdf_cluster call that
 * used workspace `ws` with the same H, W, rho, K: out[2e] = tag | node << 8 | worker << 28 (tags:
 * 1 claim start, 2 split start, 3 seeds chosen, 4 Lloyd done, 5 children published; worker -1 =
 * the whole grid), out[2e+1] = globaltimer ns.  out: host [2 * cap]; returns the number of events
 * copied (synchronous), or -1 on a CUDA error. */
int hdf_cluster_trace(const float *p_unused, int H, int W, int rho, int K, void *ws, long long *out, int cap);

/* Turn event recording on (on != 0) or off.  Process-wide; returns HDF_OK. */
int hdf_profile_enable(int on);

/* Wait for every event pair recorded since the last collect, then write per-stage sums:
 *   ms_total [HDF_NUM_STAGES] host, out: summed device milliseconds per stage (may be NULL)
 *   launches [HDF_NUM_STAGES] host, out: number of recorded launches per stage (may be NULL)
 * Clears the recorded set.  Returns HDF_OK or HDF_ERR_CUDA. */
int hdf_profile_collect(double *ms_total, int32_t *launches);

#ifdef __cplusplus
}
#endif

#endif /* HDF_H_ */
