/*
 * hdf_oracle.c -- TEST INFRASTRUCTURE ONLY (not product code).
 *
 * A plain, slow, fp64 CPU oracle for Nair & Chaudhury, "Fast High-Dimensional Bilateral and
 * Nonlocal Means Filtering" (arXiv 1811.02363).  Citations "P:n" are lines of
 * /root/reference/PAPER.md; "Rn" are the readings listed in DESIGN.md section 3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no source, header, table or helper with the CUDA path under
 * paper_1811_02363_b200/csrc and never calls into it.
 *
 * Every routine follows the paper's definitions / Algorithm 1 in the paper's order, in double
 * precision, with no blocking, fusion or reordering beyond what the definition states.  OpenMP is
 * used only across independent output pixels / rows (each output is computed by one thread in a
 * fixed order), so results do not depend on the thread count.  Build with -ffp-contract=off.
 *
 * Parity status of each function is listed in DESIGN.md section 4 ("pins").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_K 2
#define ORC_ERR_MEM 3

#define ORC_SPATIAL_GAUSSIAN 0
#define ORC_SPATIAL_BOX 1

/* ------------------------------------------------------------------------------------------ */
/* Kernels                                                                         */
/* ------------------------------------------------------------------------------------------ */

/* Squared Euclidean distance, summed over dimensions in index order. */
static double dist2(const double *a, const double *b, int rho) {
    double s = 0.0;
    for (int d = 0; d < rho; d++) {
        double t = a[d] - b[d];
        s = s + t * t;
    }
    return s;
}

/* Range kernel phi(x) = exp(-||x||^2 / (2 sigma_r^2)), evaluated from ||x||^2. */
static double phi_from_d2(double d2, double sigma_r) {
    return exp(-d2 / (2.0 * sigma_r * sigma_r));
}

double orc_phi(const double *x, int rho, double sigma_r) {
    double s = 0.0;
    for (int d = 0; d < rho; d++) s = s + x[d] * x[d];
    return phi_from_d2(s, sigma_r);
}

/* Spatial radius: S = 3 sigma_s for the Gaussian, rounded up (R7); explicit for box. */
int orc_radius(int kind, double sigma_s, int radius) {
    if (radius >= 0) return radius;
    if (kind == ORC_SPATIAL_GAUSSIAN) return (int)ceil(3.0 * sigma_s);
    return -1;
}

/* 1-D taps w_t, t in [-R, R]: the 2-D spatial kernel is omega(j) = w_{j_y} w_{j_x}.
 * Gaussian: omega(i) = exp(-||i||^2 / 2 sigma_s^2) = product of 1-D Gaussians.
 * Box: omega = 1 on W = [-S,S]^2.  Taps are unnormalised (R13). */
int orc_spatial_taps(int kind, double sigma_s, int R, double *w) {
    if (R < 0) return ORC_ERR_ARG;
    for (int t = -R; t <= R; t++) {
        if (kind == ORC_SPATIAL_GAUSSIAN)
            w[t + R] = exp(-(double)(t * t) / (2.0 * sigma_s * sigma_s));
        else if (kind == ORC_SPATIAL_BOX)
            w[t + R] = 1.0;
        else
            return ORC_ERR_ARG;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Step 1: bisecting K-means on Theta = {p(i)} (R1-R5)             */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
    long *idx;   /* members, ascending pixel index (member order, R3) */
    long m;
    double *mean;
    double sse;  /* total within-cluster sum of squares ("variance", R2) */
} Leaf;

static void leaf_stats(const double *p, int rho, Leaf *L) {
    for (int d = 0; d < rho; d++) L->mean[d] = 0.0;
    for (long t = 0; t < L->m; t++) {
        const double *x = p + L->idx[t] * (long)rho;
        for (int d = 0; d < rho; d++) L->mean[d] = L->mean[d] + x[d];
    }
    for (int d = 0; d < rho; d++) L->mean[d] = L->mean[d] / (double)L->m;
    double s = 0.0;
    for (long t = 0; t < L->m; t++) s = s + dist2(p + L->idx[t] * (long)rho, L->mean, rho);
    L->sse = s;
}

/* Farthest pair within the stride sample members[0::stride], stride = ceil(m / cap), cap = 1024 (R3).
 * Ties keep the lexicographically smallest (a, b) in sample order. */
static void farthest_pair(const double *p, int rho, const Leaf *L, int cap, long *pa, long *pb) {
    long m = L->m;
    long stride = (m + cap - 1) / cap;
    long s = (m + stride - 1) / stride;
    double *rowbest = (double *)malloc(sizeof(double) * (size_t)s);
    long *rowarg = (long *)malloc(sizeof(long) * (size_t)s);
#pragma omp parallel for schedule(dynamic, 16)
    for (long a = 0; a < s; a++) {
        const double *xa = p + L->idx[a * stride] * (long)rho;
        double best = -1.0;
        long arg = -1;
        for (long b = a + 1; b < s; b++) {
            double d = dist2(xa, p + L->idx[b * stride] * (long)rho, rho);
            if (d > best) { best = d; arg = b; }
        }
        rowbest[a] = best;
        rowarg[a] = arg;
    }
    double best = -1.0;
    long ba = 0, bb = 1;
    for (long a = 0; a < s; a++) {
        if (rowarg[a] >= 0 && rowbest[a] > best) { best = rowbest[a]; ba = a; bb = rowarg[a]; }
    }
    free(rowbest);
    free(rowarg);
    if (s < 2) bb = ba;            /* single member: no pair (never split, SSE = 0) */
    *pa = L->idx[ba * stride];
    *pb = L->idx[bb * stride];
}

/* The seed step of one split on its own, for the pins (tests/test_oracle_pins.py): the farthest pair
 * of the stride sample of the members idx[0..m) (ascending pixel index, R3).  Writes the two
 * pixel indices; no arithmetic beyond farthest_pair above. */
int orc_farthest_pair(const double *p, int rho, const long *idx, long m, int cap, long *pa, long *pb) {
    if (!p || rho < 1 || !idx || m < 1 || cap < 2 || !pa || !pb) return ORC_ERR_ARG;
    Leaf L;
    L.idx = (long *)idx;
    L.m = m;
    L.mean = NULL;
    L.sse = 0.0;
    farthest_pair(p, rho, &L, cap, pa, pb);
    return ORC_OK;
}

/* Nearest of two centres, ties -> first (R4). */
static int nearer(const double *x, const double *c0, const double *c1, int rho) {
    return dist2(x, c0, rho) <= dist2(x, c1, rho) ? 0 : 1;
}

/* Member farthest from centre c; ties -> first in member order. */
static long farthest_member(const double *p, int rho, const Leaf *L, const double *c) {
    double best = -1.0;
    long arg = 0;
    for (long t = 0; t < L->m; t++) {
        double d = dist2(p + L->idx[t] * (long)rho, c, rho);
        if (d > best) { best = d; arg = t; }
    }
    return L->idx[arg];
}

static long assign_all(const double *p, int rho, const Leaf *L, const double *c0, const double *c1,
                       unsigned char *as) {
    long n1 = 0;
#pragma omp parallel for reduction(+ : n1)
    for (long t = 0; t < L->m; t++) {
        as[t] = (unsigned char)nearer(p + L->idx[t] * (long)rho, c0, c1, rho);
        n1 += as[t];
    }
    return n1;
}

/* 2-means of one leaf, seeded by the farthest pair, Lloyd iterations until no
 * assignment changes or max_iter (R4).  Writes the final side of each member to as[]. */
static void two_means(const double *p, int rho, const Leaf *L, int cap, int max_iter, unsigned char *as) {
    long m = L->m;
    double *c0 = (double *)calloc((size_t)rho, sizeof(double));
    double *c1 = (double *)calloc((size_t)rho, sizeof(double));
    unsigned char *prev = (unsigned char *)malloc((size_t)m);
    long a, b;
    farthest_pair(p, rho, L, cap, &a, &b);
    memcpy(c0, p + a * (long)rho, sizeof(double) * (size_t)rho);
    memcpy(c1, p + b * (long)rho, sizeof(double) * (size_t)rho);
    for (int it = 0; it < max_iter; it++) {
        long n1 = assign_all(p, rho, L, c0, c1, as);
        if (n1 == 0) {          /* empty side 1: reseed at the member farthest from c0 (R4) */
            long f = farthest_member(p, rho, L, c0);
            memcpy(c1, p + f * (long)rho, sizeof(double) * (size_t)rho);
            n1 = assign_all(p, rho, L, c0, c1, as);
        } else if (n1 == m) {   /* empty side 0: reseed at the member farthest from c1 */
            long f = farthest_member(p, rho, L, c1);
            memcpy(c0, p + f * (long)rho, sizeof(double) * (size_t)rho);
            n1 = assign_all(p, rho, L, c0, c1, as);
        }
        if (it > 0 && memcmp(as, prev, (size_t)m) == 0) break;   /* converged */
        /* new centres = means of the two sides, summed in member order */
        long cnt0 = 0, cnt1 = 0;
        for (int d = 0; d < rho; d++) { c0[d] = 0.0; c1[d] = 0.0; }
        for (long t = 0; t < m; t++) {
            const double *x = p + L->idx[t] * (long)rho;
            if (as[t] == 0) { cnt0++; for (int d = 0; d < rho; d++) c0[d] = c0[d] + x[d]; }
            else            { cnt1++; for (int d = 0; d < rho; d++) c1[d] = c1[d] + x[d]; }
        }
        for (int d = 0; d < rho; d++) { c0[d] = c0[d] / (double)cnt0; c1[d] = c1[d] / (double)cnt1; }
        memcpy(prev, as, (size_t)m);
    }
    /* If the loop ran out of iterations, the last centres are the means of prev; use prev. */
    memcpy(as, prev, (size_t)m);
    free(prev);
    free(c0);
    free(c1);
}

/*
 * orc_cluster: bisecting K-means (Algorithm 1 line "cluster").
 *   p        [N, rho] guide vectors (row-major pixel order)
 *   K        number of leaves
 *   cap      farthest-pair sample cap (1024, R3); max_iter Lloyd cap (50, R4)
 *   centres  out [K, rho] leaf means (mu_k = centroid of C_k)
 *   labels   out [N] leaf id of every pixel (may be NULL)
 *   leaf_sse out [K] (may be NULL); E_K out (may be NULL)
 *   achievable out: number of leaves reached (== number of distinct vectors on ORC_ERR_K, R5)
 * Returns ORC_OK, ORC_ERR_ARG, ORC_ERR_K.
 */
int orc_cluster(const double *p, long N, int rho, int K, int cap, int max_iter, double *centres,
                int32_t *labels, double *leaf_sse, double *E_K, int *achievable) {
    if (!p || N < 1 || rho < 1 || K < 1 || cap < 2 || max_iter < 1 || !centres) return ORC_ERR_ARG;
    Leaf *leaves = (Leaf *)calloc((size_t)K, sizeof(Leaf));
    leaves[0].m = N;
    leaves[0].idx = (long *)malloc(sizeof(long) * (size_t)N);
    for (long i = 0; i < N; i++) leaves[0].idx[i] = i;
    leaves[0].mean = (double *)calloc((size_t)rho, sizeof(double));
    leaf_stats(p, rho, &leaves[0]);
    int nleaves = 1;
    int status = ORC_OK;
    unsigned char *as = (unsigned char *)malloc((size_t)N);
    while (nleaves < K) {
        int s = 0;
        for (int l = 1; l < nleaves; l++)
            if (leaves[l].sse > leaves[s].sse) s = l;   /* ties -> lowest id */
        if (!(leaves[s].sse > 0.0)) { status = ORC_ERR_K; break; }
        Leaf *P = &leaves[s];
        two_means(p, rho, P, cap, max_iter, as);
        long m0 = 0;
        for (long t = 0; t < P->m; t++) m0 += (as[t] == 0);
        long m1 = P->m - m0;
        Leaf c0, c1;
        c0.m = m0; c1.m = m1;
        c0.idx = (long *)malloc(sizeof(long) * (size_t)(m0 > 0 ? m0 : 1));
        c1.idx = (long *)malloc(sizeof(long) * (size_t)(m1 > 0 ? m1 : 1));
        long i0 = 0, i1 = 0;
        for (long t = 0; t < P->m; t++) {          /* stable partition keeps member order */
            if (as[t] == 0) c0.idx[i0++] = P->idx[t]; else c1.idx[i1++] = P->idx[t];
        }
        c0.mean = P->mean;                          /* parent id keeps child 0 */
        c1.mean = (double *)calloc((size_t)rho, sizeof(double));
        leaf_stats(p, rho, &c0);
        leaf_stats(p, rho, &c1);
        free(P->idx);
        leaves[s] = c0;
        leaves[nleaves] = c1;                       /* child 1 gets id = #leaves */
        nleaves++;
    }
    if (achievable) *achievable = nleaves;
    if (status == ORC_OK) {
        double e = 0.0;
        for (int l = 0; l < K; l++) {
            for (int d = 0; d < rho; d++) centres[(long)l * rho + d] = leaves[l].mean[d];
            if (leaf_sse) leaf_sse[l] = leaves[l].sse;
            e = e + leaves[l].sse;
            if (labels)
                for (long t = 0; t < leaves[l].m; t++) labels[leaves[l].idx[t]] = l;
        }
        if (E_K) *E_K = e;
    }
    for (int l = 0; l < nleaves; l++) { free(leaves[l].idx); free(leaves[l].mean); }
    free(leaves);
    free(as);
    return status;
}

/* ------------------------------------------------------------------------------------------ */
/* Step 2: A_kl = phi(mu_k - mu_l) and its Moore-Penrose pseudo-inverse (R6) */
/* ------------------------------------------------------------------------------------------ */

int orc_gram(const double *mu, int K, int rho, double sigma_r, double *A) {
    if (!mu || K < 1 || rho < 1 || !A) return ORC_ERR_ARG;
    for (int k = 0; k < K; k++)
        for (int l = 0; l < K; l++)
            A[(long)k * K + l] = phi_from_d2(dist2(mu + (long)k * rho, mu + (long)l * rho, rho), sigma_r);
    return ORC_OK;
}

/* MATLAB eps(x): spacing of doubles at |x|. */
static double eps_of(double x) {
    x = fabs(x);
    if (x == 0.0) return DBL_MIN;
    int e;
    frexp(x, &e);                  /* x = f * 2^e, f in [0.5, 1) */
    return ldexp(1.0, e - 53);
}

/*
 * orc_pinv_sym: pinv of a symmetric matrix by cyclic Jacobi eigen-decomposition.
 * A = U diag(lambda) U^T; singular values are |lambda|; tol = K * eps(max|lambda|) (MATLAB
 * pinv default, R6); A^+ = sum_{|lambda_j| > tol} u_j u_j^T / lambda_j.
 * Outputs: Ap [K,K]; lambda [K] (may be NULL); rank (may be NULL); tol (may be NULL).
 */
int orc_pinv_sym(const double *A_in, int K, double *Ap, double *lambda, int *rank, double *tol_out) {
    if (!A_in || K < 1 || !Ap) return ORC_ERR_ARG;
    double *A = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *V = (double *)calloc((size_t)K * K, sizeof(double));
    memcpy(A, A_in, sizeof(double) * (size_t)K * K);
    for (int i = 0; i < K; i++) V[(long)i * K + i] = 1.0;
    double fro = 0.0;
    for (long i = 0; i < (long)K * K; i++) fro += A[i] * A[i];
    fro = sqrt(fro);
    for (int sweep = 0; sweep < 100; sweep++) {
        double off = 0.0;
        for (int i = 0; i < K; i++)
            for (int j = 0; j < K; j++)
                if (i != j) off += A[(long)i * K + j] * A[(long)i * K + j];
        if (sqrt(off) <= 1e-17 * fro || off == 0.0) break;
        for (int pp = 0; pp < K - 1; pp++) {
            for (int q = pp + 1; q < K; q++) {
                double apq = A[(long)pp * K + q];
                if (apq == 0.0) continue;
                double app = A[(long)pp * K + pp], aqq = A[(long)q * K + q];
                double tau = (aqq - app) / (2.0 * apq);
                double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                /* A <- J^T A J with J the (p,q) rotation [c s; -s c] */
                for (int k = 0; k < K; k++) {
                    double akp = A[(long)k * K + pp], akq = A[(long)k * K + q];
                    A[(long)k * K + pp] = c * akp - s * akq;
                    A[(long)k * K + q] = s * akp + c * akq;
                }
                for (int k = 0; k < K; k++) {
                    double apk = A[(long)pp * K + k], aqk = A[(long)q * K + k];
                    A[(long)pp * K + k] = c * apk - s * aqk;
                    A[(long)q * K + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < K; k++) {
                    double vkp = V[(long)k * K + pp], vkq = V[(long)k * K + q];
                    V[(long)k * K + pp] = c * vkp - s * vkq;
                    V[(long)k * K + q] = s * vkp + c * vkq;
                }
            }
        }
    }
    double lmax = 0.0;
    for (int j = 0; j < K; j++) if (fabs(A[(long)j * K + j]) > lmax) lmax = fabs(A[(long)j * K + j]);
    double tol = (double)K * eps_of(lmax);
    int r = 0;
    memset(Ap, 0, sizeof(double) * (size_t)K * K);
    for (int j = 0; j < K; j++) {
        double lj = A[(long)j * K + j];
        if (lambda) lambda[j] = lj;
        if (fabs(lj) > tol) {
            r++;
            for (int a = 0; a < K; a++)
                for (int b = 0; b < K; b++)
                    Ap[(long)a * K + b] += V[(long)a * K + j] * V[(long)b * K + j] / lj;
        }
    }
    if (rank) *rank = r;
    if (tol_out) *tol_out = tol;
    free(A);
    free(V);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Convolution omega * x with the window clipped to Omega (zero extension, R8)       */
/* ------------------------------------------------------------------------------------------ */

/* out(y,x) = sum_{ty,tx in [-R,R]} w_ty w_tx in(y-ty, x-tx), (y-ty, x-tx) in Omega.
 * Separable: rows (along x) first, then columns (along y). */
static void conv2_sep(const double *in, double *out, double *tmp, int H, int W, const double *w, int R) {
#pragma omp parallel for
    for (int y = 0; y < H; y++) {
        for (int x = 0; x < W; x++) {
            double s = 0.0;
            for (int t = -R; t <= R; t++) {
                int xx = x - t;
                if (xx < 0 || xx >= W) continue;
                s = s + w[t + R] * in[(long)y * W + xx];
            }
            tmp[(long)y * W + x] = s;
        }
    }
#pragma omp parallel for
    for (int y = 0; y < H; y++) {
        for (int x = 0; x < W; x++) {
            double s = 0.0;
            for (int t = -R; t <= R; t++) {
                int yy = y - t;
                if (yy < 0 || yy >= H) continue;
                s = s + w[t + R] * tmp[(long)yy * W + x];
            }
            out[(long)y * W + x] = s;
        }
    }
}

/* Exported for the convolution pins (P6). */
int orc_conv2(const double *in, double *out, int H, int W, int kind, double sigma_s, int radius) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!in || !out || H < 1 || W < 1 || R < 0) return ORC_ERR_ARG;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    double *tmp = (double *)malloc(sizeof(double) * (size_t)H * W);
    int st = orc_spatial_taps(kind, sigma_s, R, w);
    if (st == ORC_OK) conv2_sep(in, out, tmp, H, W, w, R);
    free(w);
    free(tmp);
    return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Brute force (num)/(den), window clipped to Omega (R8)                              */
/* ------------------------------------------------------------------------------------------ */

/* pix == NULL -> all pixels, in which case g has H*W*n entries; otherwise npix pixels. */
int orc_bruteforce_pixels(const double *f, int n, const double *p, int rho, int H, int W, int kind,
                          double sigma_s, int radius, double sigma_r, const long *pix, long npix,
                          double *g, double *eta) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!f || !p || n < 1 || rho < 1 || H < 1 || W < 1 || R < 0 || !g) return ORC_ERR_ARG;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    int st = orc_spatial_taps(kind, sigma_s, R, w);
    if (st != ORC_OK) { free(w); return st; }
    long count = pix ? npix : (long)H * W;
#pragma omp parallel
    {
        double *num = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 64)
        for (long q = 0; q < count; q++) {
            long i = pix ? pix[q] : q;
            int y = (int)(i / W), x = (int)(i % W);
            const double *pi = p + i * rho;
            double den = 0.0;
            for (int c = 0; c < n; c++) num[c] = 0.0;
            for (int ty = -R; ty <= R; ty++) {
                int yy = y - ty;
                if (yy < 0 || yy >= H) continue;
                for (int tx = -R; tx <= R; tx++) {
                    int xx = x - tx;
                    if (xx < 0 || xx >= W) continue;
                    long jj = (long)yy * W + xx;
                    double wt = w[ty + R] * w[tx + R] * phi_from_d2(dist2(p + jj * rho, pi, rho), sigma_r);
                    den = den + wt;
                    for (int c = 0; c < n; c++) num[c] = num[c] + wt * f[jj * n + c];
                }
            }
            for (int c = 0; c < n; c++) g[q * n + c] = num[c] / den;
            if (eta) eta[q] = den;
        }
        free(num);
    }
    free(w);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Algorithm 1: planes, coefficients, (n+1)K convolutions, combine, normalise      */
/* ------------------------------------------------------------------------------------------ */

/* Algorithm 1 loops for1 and for2: b_k(i) = phi(mu_k - p(i)) (defAb) and
 * c(i) = A^+ b(i), stored as K planes each ([K][N]). */
static void for1_for2(const double *p, long N, int rho, const double *mu, int K, double sigma_r,
                      const double *Ap, double *b, double *c) {
#pragma omp parallel for
    for (long i = 0; i < N; i++)
        for (int k = 0; k < K; k++)
            b[(long)k * N + i] = phi_from_d2(dist2(mu + (long)k * rho, p + i * rho, rho), sigma_r);
#pragma omp parallel for
    for (long i = 0; i < N; i++)
        for (int k = 0; k < K; k++) {
            double s = 0.0;
            for (int l = 0; l < K; l++) s = s + Ap[(long)k * K + l] * b[(long)l * N + i];
            c[(long)k * N + i] = s;
        }
}

/* Exported for pins P5: b [K][N], c [K][N] for guide p [N, rho]. */
int orc_coefficients(const double *p, long N, int rho, const double *mu, int K, double sigma_r,
                     double *b, double *c) {
    if (!p || !mu || !b || !c || N < 1 || rho < 1 || K < 1) return ORC_ERR_ARG;
    double *A = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *Ap = (double *)malloc(sizeof(double) * (size_t)K * K);
    orc_gram(mu, K, rho, sigma_r, A);
    orc_pinv_sym(A, K, Ap, NULL, NULL, NULL);
    for1_for2(p, N, rho, mu, K, sigma_r, Ap, b, c);
    free(A);
    free(Ap);
    return ORC_OK;
}

/*
 * orc_filter: the fast filter (HDapprox)/(approxDen), computed as Algorithm 1.
 *   f [H,W,n], p [H,W,rho], centres mu [K,rho] (fp64; parity runs pass fp32-rounded centres, R14)
 *   kind/sigma_s/radius: spatial kernel (radius < 0 -> ceil(3 sigma_s) for the Gaussian)
 *   tau: degenerate-normaliser rule R9: if eta_hat(i) < tau*omega(0)*phi(0), g(i) is replaced by
 *        the brute-force (num)/(den) value at i and the pixel is flagged (tau = 0 disables).
 *   g [H,W,n] out; eta_hat [H,W] out (may be NULL); flagged [H,W] out (may be NULL);
 *   n_flagged out (may be NULL).
 */
int orc_filter(const double *f, int n, const double *p, int rho, int H, int W, int kind, double sigma_s,
               int radius, double sigma_r, int K, const double *mu, double tau, double *g,
               double *eta_hat, unsigned char *flagged, long *n_flagged) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!f || !p || !mu || !g || n < 1 || rho < 1 || H < 1 || W < 1 || K < 1 || R < 0) return ORC_ERR_ARG;
    long N = (long)H * W;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    if (orc_spatial_taps(kind, sigma_s, R, w) != ORC_OK) { free(w); return ORC_ERR_ARG; }
    double *A = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *Ap = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *b = (double *)malloc(sizeof(double) * (size_t)K * N);     /* b_k(i), K planes */
    double *c = (double *)malloc(sizeof(double) * (size_t)K * N);     /* c_k(i), K planes */
    double *v = (double *)calloc((size_t)n * N, sizeof(double));      /* v accumulator, n planes */
    double *r = (double *)calloc((size_t)N, sizeof(double));          /* r accumulator */
    double *u = (double *)malloc(sizeof(double) * (size_t)N);
    double *cv = (double *)malloc(sizeof(double) * (size_t)N);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)N);
    if (!A || !Ap || !b || !c || !v || !r || !u || !cv || !tmp) {
        free(w); free(A); free(Ap); free(b); free(c); free(v); free(r); free(u); free(cv); free(tmp);
        return ORC_ERR_MEM;
    }
    /* line "pinv": A (defAb) and A^+ */
    orc_gram(mu, K, rho, sigma_r, A);
    orc_pinv_sym(A, K, Ap, NULL, NULL, NULL);
    /* loops for1 (b_k(i); u_k = b_k f is formed in for3 just before use) and for2 (c = A^+ b) */
    for1_for2(p, N, rho, mu, K, sigma_r, Ap, b, c);
    /* loop for3: v += c_k (omega * u_k), r += c_k (omega * b_k), k ascending */
    for (int k = 0; k < K; k++) {
        const double *bk = b + (long)k * N;
        const double *ck = c + (long)k * N;
        for (int ch = 0; ch < n; ch++) {
            for (long i = 0; i < N; i++) u[i] = bk[i] * f[i * n + ch];
            conv2_sep(u, cv, tmp, H, W, w, R);
            for (long i = 0; i < N; i++) v[(long)ch * N + i] = v[(long)ch * N + i] + ck[i] * cv[i];
        }
        conv2_sep(bk, cv, tmp, H, W, w, R);
        for (long i = 0; i < N; i++) r[i] = r[i] + ck[i] * cv[i];
    }
    /* g = v / r, then the degenerate-normaliser rule R9 */
    double floor_ = tau * w[R] * w[R] * phi_from_d2(0.0, sigma_r);
    long nf = 0;
    for (long i = 0; i < N; i++) {
        for (int ch = 0; ch < n; ch++) g[i * n + ch] = v[(long)ch * N + i] / r[i];
        if (eta_hat) eta_hat[i] = r[i];
        int fl = (tau > 0.0) && (r[i] < floor_);
        if (flagged) flagged[i] = (unsigned char)fl;
        if (fl) nf++;
    }
    if (nf > 0) {
        long *pix = (long *)malloc(sizeof(long) * (size_t)nf);
        double *gb = (double *)malloc(sizeof(double) * (size_t)nf * n);
        long q = 0;
        for (long i = 0; i < N; i++)
            if ((tau > 0.0) && (r[i] < floor_)) pix[q++] = i;
        orc_bruteforce_pixels(f, n, p, rho, H, W, kind, sigma_s, R, sigma_r, pix, nf, gb, NULL);
        for (long t = 0; t < nf; t++)
            for (int ch = 0; ch < n; ch++) g[pix[t] * n + ch] = gb[t * n + ch];
        free(pix);
        free(gb);
    }
    if (n_flagged) *n_flagged = nf;
    free(w); free(A); free(Ap); free(b); free(c); free(v); free(r); free(u); free(cv); free(tmp);
    return ORC_OK;
}

/*
 * orc_filter_pixels: the same fast filter evaluated at selected pixels only (for parity at sizes
 * where full fp64 planes do not fit): v_k(i) = sum_{j in W} omega(j) b_k(i-j) f(i-j) and
 * r_k(i) = sum_j omega(j) b_k(i-j) are the definitions (temp1)/(temp2) written out;
 * c(i) = A^+ b(i); g(i) = sum_k c_k v_k / sum_k c_k r_k with rule R9.
 * Outputs per selected pixel: g [npix, n], eta_hat [npix] (may be NULL), flagged [npix] (may be NULL).
 */
int orc_filter_pixels(const double *f, int n, const double *p, int rho, int H, int W, int kind,
                      double sigma_s, int radius, double sigma_r, int K, const double *mu, double tau,
                      const long *pix, long npix, double *g, double *eta_hat, unsigned char *flagged) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!f || !p || !mu || !g || !pix || n < 1 || rho < 1 || H < 1 || W < 1 || K < 1 || R < 0) return ORC_ERR_ARG;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    if (orc_spatial_taps(kind, sigma_s, R, w) != ORC_OK) { free(w); return ORC_ERR_ARG; }
    double *A = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *Ap = (double *)malloc(sizeof(double) * (size_t)K * K);
    orc_gram(mu, K, rho, sigma_r, A);
    orc_pinv_sym(A, K, Ap, NULL, NULL, NULL);
    double floor_ = tau * w[R] * w[R] * phi_from_d2(0.0, sigma_r);
    long nbf = 0;
#pragma omp parallel reduction(+ : nbf)
    {
        double *bi = (double *)malloc(sizeof(double) * (size_t)K);
        double *ci = (double *)malloc(sizeof(double) * (size_t)K);
        double *bj = (double *)malloc(sizeof(double) * (size_t)K);
        double *vk = (double *)malloc(sizeof(double) * (size_t)K * n);
        double *rk = (double *)malloc(sizeof(double) * (size_t)K);
#pragma omp for schedule(dynamic, 4)
        for (long q = 0; q < npix; q++) {
            long i = pix[q];
            int y = (int)(i / W), x = (int)(i % W);
            for (int k = 0; k < K; k++) bi[k] = phi_from_d2(dist2(mu + (long)k * rho, p + i * rho, rho), sigma_r);
            for (int k = 0; k < K; k++) {
                double s = 0.0;
                for (int l = 0; l < K; l++) s = s + Ap[(long)k * K + l] * bi[l];
                ci[k] = s;
            }
            for (long t = 0; t < (long)K * n; t++) vk[t] = 0.0;
            for (int k = 0; k < K; k++) rk[k] = 0.0;
            for (int ty = -R; ty <= R; ty++) {
                int yy = y - ty;
                if (yy < 0 || yy >= H) continue;
                for (int tx = -R; tx <= R; tx++) {
                    int xx = x - tx;
                    if (xx < 0 || xx >= W) continue;
                    long jj = (long)yy * W + xx;
                    double wt = w[ty + R] * w[tx + R];
                    for (int k = 0; k < K; k++) {
                        bj[k] = phi_from_d2(dist2(mu + (long)k * rho, p + jj * rho, rho), sigma_r);
                        rk[k] = rk[k] + wt * bj[k];
                        for (int ch = 0; ch < n; ch++) vk[(long)k * n + ch] = vk[(long)k * n + ch] + wt * (bj[k] * f[jj * n + ch]);
                    }
                }
            }
            double den = 0.0;
            for (int k = 0; k < K; k++) den = den + ci[k] * rk[k];
            for (int ch = 0; ch < n; ch++) {
                double num = 0.0;
                for (int k = 0; k < K; k++) num = num + ci[k] * vk[(long)k * n + ch];
                g[q * n + ch] = num / den;
            }
            if (eta_hat) eta_hat[q] = den;
            int fl = (tau > 0.0) && (den < floor_);
            if (flagged) flagged[q] = (unsigned char)fl;
            if (fl) {
                nbf++;
                orc_bruteforce_pixels(f, n, p, rho, H, W, kind, sigma_s, R, sigma_r, &pix[q], 1, &g[q * n], NULL);
            }
        }
        free(bi); free(ci); free(bj); free(vk); free(rk);
    }
    free(w); free(A); free(Ap);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Appendix A written as a direct window sum: the "Nystrom" kernel                 */
/*   phi~(i, i') = b(i)^T A^+ b(i') = sum_k c_k(i) phi(p(i') - mu_k)                           */
/* g(i) = sum_j omega(j) phi~(i, i-j) f(i-j) / sum_j omega(j) phi~(i, i-j).  Used for pin P7.   */
/* ------------------------------------------------------------------------------------------ */
int orc_nystrom_pixels(const double *f, int n, const double *p, int rho, int H, int W, int kind,
                       double sigma_s, int radius, double sigma_r, int K, const double *mu,
                       const long *pix, long npix, double *g, double *eta) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!f || !p || !mu || !g || n < 1 || rho < 1 || H < 1 || W < 1 || K < 1 || R < 0) return ORC_ERR_ARG;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    orc_spatial_taps(kind, sigma_s, R, w);
    double *A = (double *)malloc(sizeof(double) * (size_t)K * K);
    double *Ap = (double *)malloc(sizeof(double) * (size_t)K * K);
    orc_gram(mu, K, rho, sigma_r, A);
    orc_pinv_sym(A, K, Ap, NULL, NULL, NULL);
    long count = pix ? npix : (long)H * W;
#pragma omp parallel
    {
        double *bi = (double *)malloc(sizeof(double) * (size_t)K);
        double *Apbi = (double *)malloc(sizeof(double) * (size_t)K);
        double *num = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
        for (long q = 0; q < count; q++) {
            long i = pix ? pix[q] : q;
            int y = (int)(i / W), x = (int)(i % W);
            for (int k = 0; k < K; k++) bi[k] = phi_from_d2(dist2(mu + (long)k * rho, p + i * rho, rho), sigma_r);
            for (int k = 0; k < K; k++) {
                double s = 0.0;
                for (int l = 0; l < K; l++) s = s + Ap[(long)k * K + l] * bi[l];
                Apbi[k] = s;
            }
            double den = 0.0;
            for (int ch = 0; ch < n; ch++) num[ch] = 0.0;
            for (int ty = -R; ty <= R; ty++) {
                int yy = y - ty;
                if (yy < 0 || yy >= H) continue;
                for (int tx = -R; tx <= R; tx++) {
                    int xx = x - tx;
                    if (xx < 0 || xx >= W) continue;
                    long jj = (long)yy * W + xx;
                    double kt = 0.0;
                    for (int k = 0; k < K; k++)
                        kt = kt + Apbi[k] * phi_from_d2(dist2(mu + (long)k * rho, p + jj * rho, rho), sigma_r);
                    double wt = w[ty + R] * w[tx + R] * kt;
                    den = den + wt;
                    for (int ch = 0; ch < n; ch++) num[ch] = num[ch] + wt * f[jj * n + ch];
                }
            }
            for (int ch = 0; ch < n; ch++) g[q * n + ch] = num[ch] / den;
            if (eta) eta[q] = den;
        }
        free(bi); free(Apbi); free(num);
    }
    free(w); free(A); free(Ap);
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Hard-assignment variant (coeffICIP)/(HDapprox2): g(i) = v_s(i) / r_s(i)           */
/* ------------------------------------------------------------------------------------------ */
int orc_filter_hard(const double *f, int n, const double *p, int rho, int H, int W, int kind,
                    double sigma_s, int radius, double sigma_r, int K, const double *mu,
                    const int32_t *labels, double *g) {
    int R = orc_radius(kind, sigma_s, radius);
    if (!f || !p || !mu || !labels || !g || n < 1 || rho < 1 || H < 1 || W < 1 || K < 1 || R < 0) return ORC_ERR_ARG;
    long N = (long)H * W;
    double *w = (double *)malloc(sizeof(double) * (size_t)(2 * R + 1));
    orc_spatial_taps(kind, sigma_s, R, w);
    double *bk = (double *)malloc(sizeof(double) * (size_t)N);
    double *u = (double *)malloc(sizeof(double) * (size_t)N);
    double *cv = (double *)malloc(sizeof(double) * (size_t)N);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)N);
    double *rs = (double *)malloc(sizeof(double) * (size_t)N);
    for (int k = 0; k < K; k++) {
        for (long i = 0; i < N; i++) bk[i] = phi_from_d2(dist2(mu + (long)k * rho, p + i * rho, rho), sigma_r);
        conv2_sep(bk, cv, tmp, H, W, w, R);
        for (long i = 0; i < N; i++) if (labels[i] == k) rs[i] = cv[i];
        for (int ch = 0; ch < n; ch++) {
            for (long i = 0; i < N; i++) u[i] = bk[i] * f[i * n + ch];
            conv2_sep(u, cv, tmp, H, W, w, R);
            for (long i = 0; i < N; i++) if (labels[i] == k) g[i * n + ch] = cv[i];
        }
    }
    for (long i = 0; i < N; i++)
        for (int ch = 0; ch < n; ch++) g[i * n + ch] = g[i * n + ch] / rs[i];
    free(w); free(bk); free(u); free(cv); free(tmp); free(rs);
    return ORC_OK;
}
