// k_coeffs.cuh -- step 2 (A and A^+) and loop for2 (c(i) = A^+ b(i)) of Algorithm 1.
//
//  k_gram_pinv: one CTA.  A_kl = phi(mu_k - mu_l) in fp64 (defAb).  A is symmetric
//    positive (semi)definite.  Fast path: in-place Gauss-Jordan inverse (no pivoting, SPD) with an
//    infinity-norm condition estimate; when kappa_inf(A) <= 1e8 every eigenvalue is far above
//    MATLAB's pinv tolerance K*eps(lambda_max) (R6), so A^+ = A^{-1}.  Otherwise the slow path
//    computes the eigen-decomposition by cyclic Jacobi and truncates eigenvalues <= tol exactly as
//    pinv does, and flags HDF_WARN_ILLCOND when something was truncated.
//  k_coeffs: c(i) = A^+ b(i), b_k(i) = phi(mu_k - p(i)), written as K planes
//    [K][H][Wp] (fp32) that the horizontal pass streams with TMA.
#pragma once
#include "hdf_common.cuh"

namespace hdf {

struct PinvOut {
    float* Ap32;       // [K][K] fp32 copy for the per-pixel matvec
    double* Ap64;      // [K][K] fp64 (diagnostics)
    int* status;       // device word: 0 ok, HDF_WARN_ILLCOND
    double* Vscratch;  // [K][K] fp64 global scratch for the Jacobi slow path
};

constexpr int kPinvThreads = 512;

__global__ void __launch_bounds__(kPinvThreads) k_gram_pinv(const float* __restrict__ centres, int K, int rho,
                                                             double neg_inv2sr2, PinvOut out) {
    extern __shared__ double sm_pinv[];
    double* A = sm_pinv;              // [K][K]
    double* col = A + K * K;          // [K]
    double* rowsum = col + K;         // [K]
    __shared__ int fail;
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;

    // Gram matrix in fp64 (exact promotion of the fp32 centres).
    for (int e = tid; e < K * K; e += nt) {
        int k = e / K, l = e % K;
        double s = 0.0;
        for (int d = 0; d < rho; d++) s = d2_rn(s, (double)centres[k * rho + d], (double)centres[l * rho + d]);
        A[e] = (k == l) ? 1.0 : exp(s * neg_inv2sr2);
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int k = tid; k < K; k += nt) {
        double s = 0.0;
        for (int l = 0; l < K; l++) s += fabs(A[k * K + l]);
        rowsum[k] = s;
    }
    __syncthreads();
    double normA = 0.0;
    for (int k = 0; k < K; k++) normA = fmax(normA, rowsum[k]);

    // In-place Gauss-Jordan inversion (SPD, no pivoting).
    for (int k = 0; k < K; k++) {
        double piv = A[k * K + k];
        if (!(piv > 0.0) || !isfinite(piv)) { if (tid == 0) fail = 1; break; }
        double pinv = 1.0 / piv;
        for (int i = tid; i < K; i += nt) col[i] = A[i * K + k];
        __syncthreads();
        for (int j = tid; j < K; j += nt) A[k * K + j] = ((j == k) ? 1.0 : A[k * K + j]) * pinv;
        __syncthreads();
        for (int e = tid; e < K * K; e += nt) {
            int i = e / K, j = e % K;
            if (i != k) A[e] = ((j == k) ? 0.0 : A[e]) - col[i] * A[k * K + j];
        }
        __syncthreads();
    }
    __syncthreads();
    bool use_inverse = (fail == 0);
    if (use_inverse) {
        double mx = 0.0;
        for (int k = tid; k < K; k += nt) {
            double s = 0.0;
            for (int l = 0; l < K; l++) s += fabs(A[k * K + l]);
            mx = fmax(mx, s);
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((tid & 31) == 0) red[tid >> 5] = mx;
        __syncthreads();
        double norminv = 0.0;
        for (int w = 0; w < (nt + 31) / 32; w++) norminv = fmax(norminv, red[w]);
        if (!(normA * norminv <= 1e8) || !isfinite(norminv)) use_inverse = false;
    }
    __syncthreads();
    int warn = 0;
    if (!use_inverse) {
        // Slow path: cyclic Jacobi eigen-decomposition A = V diag(lam) V^T (V in global scratch),
        // then A^+ = sum_{|lam_j| > tol} v_j v_j^T / lam_j with MATLAB's tol = K eps(max|lam|).
        double* V = out.Vscratch;
        for (int e = tid; e < K * K; e += nt) {
            int k = e / K, l = e % K;
            double s = 0.0;
            for (int d = 0; d < rho; d++) s = d2_rn(s, (double)centres[k * rho + d], (double)centres[l * rho + d]);
            A[e] = (k == l) ? 1.0 : exp(s * neg_inv2sr2);
            V[e] = (k == l) ? 1.0 : 0.0;
        }
        __syncthreads();
        for (int sweep = 0; sweep < 60; sweep++) {
            double off = 0.0, fro = 0.0;
            for (int e = 0; e < K * K; e++) { double a = A[e]; fro += a * a; if (e / K != e % K) off += a * a; }
            if (off <= 1e-34 * fro) break;
            for (int p = 0; p < K - 1; p++) {
                for (int q = p + 1; q < K; q++) {
                    double apq = A[p * K + q];
                    if (apq == 0.0) continue;      // uniform across the block
                    double app = A[p * K + p], aqq = A[q * K + q];
                    double tau = (aqq - app) / (2.0 * apq);
                    double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                    __syncthreads();
                    for (int k = tid; k < K; k += nt) {
                        double akp = A[k * K + p], akq = A[k * K + q];
                        A[k * K + p] = c * akp - s * akq;
                        A[k * K + q] = s * akp + c * akq;
                        double vkp = V[k * K + p], vkq = V[k * K + q];
                        V[k * K + p] = c * vkp - s * vkq;
                        V[k * K + q] = s * vkp + c * vkq;
                    }
                    __syncthreads();
                    for (int k = tid; k < K; k += nt) {
                        double apk = A[p * K + k], aqk = A[q * K + k];
                        A[p * K + k] = c * apk - s * aqk;
                        A[q * K + k] = s * apk + c * aqk;
                    }
                    __syncthreads();
                }
            }
        }
        double lmax = 0.0;
        for (int j = 0; j < K; j++) lmax = fmax(lmax, fabs(A[j * K + j]));
        int e2;
        frexp(lmax, &e2);
        const double tol = (double)K * ldexp(1.0, e2 - 53);
        __syncthreads();
        for (int j = tid; j < K; j += nt) col[j] = A[j * K + j];   // eigenvalues
        __syncthreads();
        for (int j = 0; j < K; j++) if (!(fabs(col[j]) > tol)) warn = 1;
        for (int e = tid; e < K * K; e += nt) {
            int a = e / K, b = e % K;
            double s = 0.0;
            for (int j = 0; j < K; j++)
                if (fabs(col[j]) > tol) s += V[a * K + j] * V[b * K + j] / col[j];
            out.Ap64[e] = s;
            out.Ap32[e] = (float)s;
        }
        if (tid == 0) *out.status = warn ? HDF_WARN_ILLCOND : HDF_OK;
        return;
    }
    for (int e = tid; e < K * K; e += nt) {
        out.Ap64[e] = A[e];
        out.Ap32[e] = (float)A[e];
    }
    if (tid == 0) *out.status = warn ? HDF_WARN_ILLCOND : HDF_OK;
}

// Shared memory needed by k_gram_pinv.
inline size_t pinv_smem_bytes(int K) { return sizeof(double) * (size_t)(K * K + 2 * K); }

// ---------------------------------------------------------------------------------------------
// c(i) = A^+ b(i).  One thread per pixel; b staged in shared memory [K][kCoefPix]; A^+ (fp32) in
// shared memory, read as broadcast float4.  Output planes cpl[k][y][x] with row pitch Wp.
// ---------------------------------------------------------------------------------------------
constexpr int kCoefPix = 256;

struct CoefParams {
    const float* p;
    const float* centres;
    const float* Ap32;
    float* cpl;
    long long cstride;   // H * Wp
    int H, W, Wp, rho, K;
    float neg_inv2sr2;
};

__global__ void __launch_bounds__(kCoefPix) k_coeffs(const CoefParams P) {
    extern __shared__ float sm_coef[];
    const int K = P.K, rho = P.rho;
    const int K8 = (K + 7) & ~7;
    float* Aps = sm_coef;                 // [K][K8]  Aps[l*K8 + k] = A^+[k][l] (zero-padded in k)
    float* mus = Aps + K * K8;            // [K][rho]
    float* bs = mus + K * rho;            // [K][kCoefPix]
    const int tid = threadIdx.x;
    for (int e = tid; e < K * K8; e += blockDim.x) {
        int l = e / K8, k = e % K8;
        Aps[e] = (k < K) ? P.Ap32[k * K + l] : 0.f;
    }
    for (int e = tid; e < K * rho; e += blockDim.x) mus[e] = P.centres[e];
    __syncthreads();
    const long long npix = (long long)P.H * P.W;
    const long long i = (long long)blockIdx.x * kCoefPix + tid;
    if (i >= npix) return;
    const float* pi = P.p + i * rho;
    for (int k = 0; k < K; k++) {
        float d2 = 0.f;
        for (int d = 0; d < rho; d++) {
            float t = __ldg(pi + d) - mus[k * rho + d];
            d2 = fmaf(t, t, d2);
        }
        bs[k * kCoefPix + tid] = expf(d2 * P.neg_inv2sr2);
    }
    const int y = (int)(i / P.W), x = (int)(i % P.W);
    float* out = P.cpl + (long long)y * P.Wp + x;
    for (int k0 = 0; k0 < K; k0 += 8) {
        float acc[8];
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = 0.f;
        for (int l = 0; l < K; l++) {
            const float bl = bs[l * kCoefPix + tid];
            const float* a = Aps + l * K8 + k0;
#pragma unroll
            for (int u = 0; u < 8; u++) acc[u] = fmaf(a[u], bl, acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (k0 + u < K) out[(long long)(k0 + u) * P.cstride] = acc[u];
    }
}

}  // namespace hdf
