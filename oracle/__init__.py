"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Thin ctypes binding over oracle/hdf_oracle.c (plain C, fp64).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package.  It shares no code with paper_1811_02363_b200 (the CUDA path) and never imports it.

Functions follow PAPER.md (see the C file for per-function citations):
  cluster        bisecting K-means (readings R1-R5)
  farthest_pair  its seed step on its own (R3), for the pins
  gram, pinv     A_kl = phi(mu_k - mu_l) and MATLAB-style pinv (R6)
  filter         Algorithm 1 with the R9 degenerate-normaliser rule
  filter_pixels  the same filter evaluated at selected pixels from (temp1)/(temp2)
  bruteforce     (num)/(den), window clipped to Omega (R8)
  nystrom        Appendix A identity written as a direct window sum
  filter_hard    hard-assignment variant (coeffICIP)/(HDapprox2)
  pca_guide      PCA-NLM patch guide (reading R11), numpy fp64
  phi_aniso, bruteforce_aniso, filter_aniso
                 the diagonal (anisotropic) range kernel (NEXT #3) and Algorithm 1
                 with it, numpy fp64 (small images)
  young_coeffs, young1d, young2d, filter_iir
                 Young's O(1) recursive Gaussian (the reference the paper cites) and
                 Algorithm 1 with it in place of the FIR (NEXT #1; readings R17), numpy fp64
  conv2          omega * x with the clipped window
  mse, psnr      (rmse), intensities normalised by R
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hdf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, ERR_ARG, ERR_K, ERR_MEM = 0, 1, 2, 3
KIND = {"gaussian": 0, "box": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp64, -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = C.CDLL(_LIB)
            D = C.POINTER(C.c_double)
            I32 = C.POINTER(C.c_int32)
            LP = C.POINTER(C.c_long)
            U8 = C.POINTER(C.c_uint8)
            i, d, l = C.c_int, C.c_double, C.c_long
            lib.orc_phi.argtypes = [D, i, d]; lib.orc_phi.restype = d
            lib.orc_radius.argtypes = [i, d, i]; lib.orc_radius.restype = i
            lib.orc_spatial_taps.argtypes = [i, d, i, D]
            lib.orc_cluster.argtypes = [D, l, i, i, i, i, D, I32, D, D, C.POINTER(C.c_int)]
            lib.orc_gram.argtypes = [D, i, i, d, D]
            lib.orc_pinv_sym.argtypes = [D, i, D, D, C.POINTER(C.c_int), D]
            lib.orc_conv2.argtypes = [D, D, i, i, i, d, i]
            lib.orc_bruteforce_pixels.argtypes = [D, i, D, i, i, i, i, d, i, d, LP, l, D, D]
            lib.orc_filter.argtypes = [D, i, D, i, i, i, i, d, i, d, i, D, d, D, D, U8, LP]
            lib.orc_filter_pixels.argtypes = [D, i, D, i, i, i, i, d, i, d, i, D, d, LP, l, D, D, U8]
            lib.orc_nystrom_pixels.argtypes = [D, i, D, i, i, i, i, d, i, d, i, D, LP, l, D, D]
            lib.orc_coefficients.argtypes = [D, l, i, D, i, d, D, D]
            lib.orc_filter_hard.argtypes = [D, i, D, i, i, i, i, d, i, d, i, D, I32, D]
            lib.orc_farthest_pair.argtypes = [D, i, LP, l, i, LP, LP]
            for fn in ("orc_spatial_taps", "orc_cluster", "orc_gram", "orc_pinv_sym", "orc_conv2",
                       "orc_bruteforce_pixels", "orc_filter", "orc_filter_pixels",
                       "orc_nystrom_pixels", "orc_filter_hard", "orc_coefficients", "orc_farthest_pair"):
                getattr(lib, fn).restype = C.c_int
            _lib = lib
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(st: int, what: str):
    if st != OK:
        raise RuntimeError(f"oracle {what} failed with status {st}")


class OracleKError(ValueError):
    def __init__(self, achievable: int):
        super().__init__(f"K exceeds the number of distinct guide vectors ({achievable})")
        self.achievable = achievable


def radius(kind: str, sigma_s: float, r: int = -1) -> int:
    return _L().orc_radius(KIND[kind], float(sigma_s), int(r))


def phi(x, sigma_r: float) -> float:
    x = _d(x).reshape(-1)
    return _L().orc_phi(_pd(x), x.size, float(sigma_r))


def spatial_taps(kind: str, sigma_s: float, r: int = -1) -> np.ndarray:
    R = radius(kind, sigma_s, r)
    w = np.zeros(2 * R + 1)
    _check(_L().orc_spatial_taps(KIND[kind], float(sigma_s), R, _pd(w)), "taps")
    return w


def cluster(p, K: int, cap: int = 1024, max_iter: int = 50):
    """Bisecting K-means of the guide p [..., rho].  Returns (centres [K,rho] fp64, labels [N]
    int32, leaf_sse [K], E_K)."""
    p = _d(p)
    rho = p.shape[-1]
    P = p.reshape(-1, rho)
    N = P.shape[0]
    cen = np.zeros((K, rho))
    lab = np.zeros(N, dtype=np.int32)
    sse = np.zeros(K)
    ek = C.c_double(0.0)
    ach = C.c_int(0)
    st = _L().orc_cluster(_pd(P), N, rho, int(K), int(cap), int(max_iter), _pd(cen),
                          lab.ctypes.data_as(C.POINTER(C.c_int32)), _pd(sse), C.byref(ek), C.byref(ach))
    if st == ERR_K:
        raise OracleKError(ach.value)
    _check(st, "cluster")
    return cen, lab, sse, ek.value


def farthest_pair(p, members, cap: int = 1024):
    """The seed step of one split (R3): the farthest pair of the stride sample
    members[0::ceil(m/cap)] of the given members (ascending pixel indices).  Returns the two pixel
    indices (a, b) of the lexicographically smallest pair in sample order among the maximisers."""
    p = _d(p)
    rho = p.shape[-1]
    P = p.reshape(-1, rho)
    mem = np.ascontiguousarray(np.asarray(members, dtype=np.int64).reshape(-1))
    a, b = C.c_long(0), C.c_long(0)
    _check(_L().orc_farthest_pair(_pd(P), rho, mem.ctypes.data_as(C.POINTER(C.c_long)), mem.size, int(cap),
                                  C.byref(a), C.byref(b)), "farthest_pair")
    return a.value, b.value


def gram(mu, sigma_r: float) -> np.ndarray:
    mu = _d(mu)
    K, rho = mu.shape
    A = np.zeros((K, K))
    _check(_L().orc_gram(_pd(mu), K, rho, float(sigma_r), _pd(A)), "gram")
    return A


def pinv(A):
    """Returns (A^+, eigenvalues, rank, tol) by cyclic Jacobi, MATLAB tolerance (R6)."""
    A = _d(A)
    K = A.shape[0]
    Ap = np.zeros((K, K))
    lam = np.zeros(K)
    rank = C.c_int(0)
    tol = C.c_double(0.0)
    _check(_L().orc_pinv_sym(_pd(A), K, _pd(Ap), _pd(lam), C.byref(rank), C.byref(tol)), "pinv")
    return Ap, lam, rank.value, tol.value


def coefficients(p, mu, sigma_r: float):
    """Algorithm 1 loops for1/for2: returns (b [N,K], c [N,K]) with c(i) = A^+ b(i)."""
    p = _d(p)
    rho = p.shape[-1]
    P = p.reshape(-1, rho)
    N = P.shape[0]
    mu = _d(mu)
    K = mu.shape[0]
    b = np.zeros((K, N))
    c = np.zeros((K, N))
    _check(_L().orc_coefficients(_pd(P), N, rho, _pd(mu), K, float(sigma_r), _pd(b), _pd(c)), "coefficients")
    return b.T.copy(), c.T.copy()


def conv2(x, kind: str, sigma_s: float, r: int = -1) -> np.ndarray:
    x = _d(x)
    H, W = x.shape
    out = np.zeros_like(x)
    _check(_L().orc_conv2(_pd(x), _pd(out), H, W, KIND[kind], float(sigma_s), int(r)), "conv2")
    return out


def _fp(f, p):
    f = _d(f)
    p = _d(p)
    if f.ndim == 2:
        f = f[..., None]
    if p.ndim == 2:
        p = p[..., None]
    assert f.shape[:2] == p.shape[:2]
    return f, p


def _pix(pix):
    if pix is None:
        return None, 0
    a = np.ascontiguousarray(np.asarray(pix, dtype=np.int64).reshape(-1))
    return a, a.size


def bruteforce(f, p, kind: str, sigma_s: float, sigma_r: float, r: int = -1, pix=None):
    """(num)/(den) of P:43-51.  Returns (g, eta): full images, or per selected pixel if pix given."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    rho = p.shape[2]
    a, npx = _pix(pix)
    cnt = npx if a is not None else H * W
    g = np.zeros((cnt, n))
    eta = np.zeros(cnt)
    lp = a.ctypes.data_as(C.POINTER(C.c_long)) if a is not None else None
    _check(_L().orc_bruteforce_pixels(_pd(f), n, _pd(p), rho, H, W, KIND[kind], float(sigma_s), int(r),
                                      float(sigma_r), lp, npx, _pd(g), _pd(eta)), "bruteforce")
    if a is None:
        return g.reshape(H, W, n), eta.reshape(H, W)
    return g, eta


def filter(f, p, kind: str, sigma_s: float, sigma_r: float, mu, r: int = -1, tau: float = 0.5):
    """Algorithm 1 with rule R9.  Returns (g [H,W,n], eta_hat [H,W], flagged [H,W] bool, n_flagged)."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    rho = p.shape[2]
    mu = _d(mu)
    K = mu.shape[0]
    g = np.zeros((H, W, n))
    eta = np.zeros((H, W))
    fl = np.zeros((H, W), dtype=np.uint8)
    nf = C.c_long(0)
    st = _L().orc_filter(_pd(f), n, _pd(p), rho, H, W, KIND[kind], float(sigma_s), int(r), float(sigma_r),
                         K, _pd(mu), float(tau), _pd(g), _pd(eta), fl.ctypes.data_as(C.POINTER(C.c_uint8)),
                         C.byref(nf))
    _check(st, "filter")
    return g, eta, fl.astype(bool), nf.value


def filter_pixels(f, p, kind: str, sigma_s: float, sigma_r: float, mu, pix, r: int = -1, tau: float = 0.5):
    """The same filter at selected pixels.  Returns (g [npix,n], eta_hat [npix], flagged [npix])."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    rho = p.shape[2]
    mu = _d(mu)
    K = mu.shape[0]
    a, npx = _pix(pix)
    g = np.zeros((npx, n))
    eta = np.zeros(npx)
    fl = np.zeros(npx, dtype=np.uint8)
    st = _L().orc_filter_pixels(_pd(f), n, _pd(p), rho, H, W, KIND[kind], float(sigma_s), int(r),
                                float(sigma_r), K, _pd(mu), float(tau), a.ctypes.data_as(C.POINTER(C.c_long)),
                                npx, _pd(g), _pd(eta), fl.ctypes.data_as(C.POINTER(C.c_uint8)))
    _check(st, "filter_pixels")
    return g, eta, fl.astype(bool)


def nystrom(f, p, kind: str, sigma_s: float, sigma_r: float, mu, r: int = -1, pix=None):
    """Appendix A identity as a direct window sum (pin P7).  Returns (g, eta)."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    rho = p.shape[2]
    mu = _d(mu)
    K = mu.shape[0]
    a, npx = _pix(pix)
    cnt = npx if a is not None else H * W
    g = np.zeros((cnt, n))
    eta = np.zeros(cnt)
    lp = a.ctypes.data_as(C.POINTER(C.c_long)) if a is not None else None
    _check(_L().orc_nystrom_pixels(_pd(f), n, _pd(p), rho, H, W, KIND[kind], float(sigma_s), int(r),
                                   float(sigma_r), K, _pd(mu), lp, npx, _pd(g), _pd(eta)), "nystrom")
    if a is None:
        return g.reshape(H, W, n), eta.reshape(H, W)
    return g, eta


def filter_hard(f, p, kind: str, sigma_s: float, sigma_r: float, mu, labels, r: int = -1):
    """Hard-assignment variant g(i) = v_s(i)/r_s(i), s = label of i."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    rho = p.shape[2]
    mu = _d(mu)
    K = mu.shape[0]
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32).reshape(-1))
    g = np.zeros((H, W, n))
    _check(_L().orc_filter_hard(_pd(f), n, _pd(p), rho, H, W, KIND[kind], float(sigma_s), int(r),
                                float(sigma_r), K, _pd(mu), lab.ctypes.data_as(C.POINTER(C.c_int32)), _pd(g)),
           "filter_hard")
    return g


def mse(a, b, R: float = 1.0) -> float:
    """(rmse): |Omega|^-1 sum_i ||a(i) - b(i)||^2 on intensities divided by R."""
    a = _d(a)
    b = _d(b)
    if a.ndim == 2:
        a = a[..., None]
        b = b[..., None]
    d = (a - b) / R
    return float(np.mean(np.sum(d * d, axis=-1)))


def psnr(a, b, R: float = 1.0) -> float:
    m = mse(a, b, R)
    return float("inf") if m == 0.0 else float(-10.0 * np.log10(m))


# ------------------------------------------------------------------ PCA-NLM patch guide ----------
def pca_guide(img, m: int = 3, dim: int = 6):
    """NLM guide (reading R11): p(i) = the m x m patch of img around i (all n channels,
    rho = n m^2 values in (channel, dy, dx) order; replicate borders), mean-centred over all pixels
    and projected on the `dim` leading eigenvectors of the patch covariance (PCA-NLM).
    Eigenvectors in descending eigenvalue order, each signed so that its entry of largest magnitude
    is positive.  fp64.  Returns (guide [H, W, dim], basis [n m^2, dim], mean [n m^2], eigenvalues)."""
    x = _d(img)
    H, W, n = x.shape
    r = m // 2
    cols = []
    for c in range(n):
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                yy = np.clip(np.arange(H) + dy, 0, H - 1)
                xx = np.clip(np.arange(W) + dx, 0, W - 1)
                cols.append(x[yy][:, xx, c])
    P = np.stack(cols, axis=-1).reshape(H * W, n * m * m)
    mean = P.mean(axis=0)
    Pc = P - mean
    C = (Pc.T @ Pc) / P.shape[0]
    evals, evecs = np.linalg.eigh(C)
    order = np.argsort(-evals, kind="stable")[:dim]
    B = evecs[:, order].copy()
    for j in range(dim):
        k = int(np.argmax(np.abs(B[:, j])))
        if B[k, j] < 0:
            B[:, j] = -B[:, j]
    return (Pc @ B).reshape(H, W, dim), B, mean, evals[order]


# ------------------------------------------------ anisotropic range kernel (NEXT #3) --
def phi_aniso(x, sigmas) -> np.ndarray:
    """The diagonal Gaussian range kernel phi(x) = exp(-sum_d x_d^2 / (2 sigma_d^2)) (per-
    dimension range widths; sigma_r = 50 on the PCA dimensions, 10 on the infrared band),
    evaluated on the last axis of x, summed over d in index order.  fp64."""
    x = _d(x)
    s = _d(sigmas).reshape(-1)
    q = np.zeros(x.shape[:-1])
    for d in range(x.shape[-1]):
        q = q + (x[..., d] * x[..., d]) / (s[d] * s[d])
    return np.exp(-q / 2.0)


def bruteforce_aniso(f, p, kind: str, sigma_s: float, sigmas, r: int = -1, pix=None):
    """(num)/(den) of P:43-51 with the diagonal range kernel, window clipped to Omega (R8), written out
    pixel by pixel (small images).  Returns (g [npix, n], eta [npix]) for the pixels pix (flat indices;
    None: all)."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    R = radius(kind, sigma_s, r)
    w = spatial_taps(kind, sigma_s, R)
    idx = np.arange(H * W) if pix is None else np.asarray(pix, dtype=np.int64).reshape(-1)
    g = np.zeros((idx.size, n))
    eta = np.zeros(idx.size)
    for t, i in enumerate(idx):
        y, x = divmod(int(i), W)
        y0, y1, x0, x1 = max(0, y - R), min(H, y + R + 1), max(0, x - R), min(W, x + R + 1)
        om = w[y0 - y + R:y1 - y + R, None] * w[None, x0 - x + R:x1 - x + R]
        wt = om * phi_aniso(p[y0:y1, x0:x1] - p[y, x], sigmas)
        eta[t] = wt.sum()
        g[t] = (wt[..., None] * f[y0:y1, x0:x1]).sum((0, 1)) / eta[t]
    return g, eta


def filter_aniso(f, p, kind: str, sigma_s: float, sigmas, mu, r: int = -1, tau: float = 0.5):
    """Algorithm 1 with the diagonal range kernel phi_aniso, step by step in the paper's
    order (small images, numpy fp64): A_kl = phi(mu_k - mu_l) and A^+ (the oracle's MATLAB-style pinv,
    R6); loop for1: b_k(i) = phi(mu_k - p(i)); loop for2: c(i) = A^+ b(i); loop for3: v += c_k (omega *
    (b_k f)), r += c_k (omega * b_k) with the oracle's clipped-window convolution (R8); g = v / r; rule R9
    with the direct (num)/(den) of bruteforce_aniso at flagged pixels.  Returns (g, eta_hat, flagged,
    n_flagged) like filter()."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    mu = _d(mu)
    K = mu.shape[0]
    R = radius(kind, sigma_s, r)
    A = phi_aniso(mu[:, None, :] - mu[None, :, :], sigmas)
    Ap, _, _, _ = pinv(A)
    b = np.stack([phi_aniso(mu[k] - p, sigmas) for k in range(K)])            # [K, H, W]
    c = np.einsum("kl,lhw->khw", Ap, b)
    v = np.zeros((n, H, W))
    rr = np.zeros((H, W))
    for k in range(K):
        for ch in range(n):
            v[ch] = v[ch] + c[k] * conv2(b[k] * f[..., ch], kind, sigma_s, R)
        rr = rr + c[k] * conv2(b[k], kind, sigma_s, R)
    g = np.ascontiguousarray(np.moveaxis(v / rr, 0, -1))
    w = spatial_taps(kind, sigma_s, R)
    floor = tau * w[R] * w[R] * 1.0
    fl = (rr < floor) if tau > 0 else np.zeros((H, W), bool)
    if fl.any():
        pix = np.nonzero(fl.reshape(-1))[0]
        gb, _ = bruteforce_aniso(f, p, kind, sigma_s, sigmas, R, pix)
        g.reshape(-1, n)[pix] = gb
    return g, rr, fl, int(fl.sum())


# ---------------------------------------------------------------- recursive Gaussian (NEXT #1) --
def young_coeffs(sigma_s: float):
    """Young & van Vliet's recursive Gaussian, the O(1) convolution the paper uses for the Gaussian
    steps: q from sigma (two ranges), the third-order recursion's b0..b3 and the input
    gain B = 1 - (b1 + b2 + b3) / b0 (unit DC gain per pass).  Returns (B, b1/b0, b2/b0, b3/b0).
    Reading R17: sigma_s >= 0.5 (the range the q formula is given for)."""
    s = float(sigma_s)
    if s < 0.5:
        raise ValueError("the recursive Gaussian needs sigma_s >= 0.5")
    q = 0.98711 * s - 0.96330 if s >= 2.5 else 3.97156 - 4.14554 * math.sqrt(1.0 - 0.26891 * s)
    b0 = 1.57825 + 2.44413 * q + 1.4281 * q * q + 0.422205 * q ** 3
    b1 = 2.44413 * q + 2.85619 * q * q + 1.26661 * q ** 3
    b2 = -(1.4281 * q * q + 1.26661 * q ** 3)
    b3 = 0.422205 * q ** 3
    return 1.0 - (b1 + b2 + b3) / b0, b1 / b0, b2 / b0, b3 / b0


def young1d(x, sigma_s: float, axis: int = 0) -> np.ndarray:
    """One axis of the recursive Gaussian, readings R17: the causal pass
    w[t] = G B x[t] + a1 w[t-1] + a2 w[t-2] + a3 w[t-3], then the anti-causal pass
    y[t] = B w[t] + a1 y[t+1] + a2 y[t+2] + a3 y[t+3], on the signal extended by zeros outside the image
    (the signal is 0 outside Omega, as under the FIR's clipped window; written out as zero padding past
    the end, long enough for the tails to vanish) and G = sqrt(2 pi) sigma_s, so that the response
    peaks near 1 like the unnormalised FIR taps exp(-t^2 / 2 sigma^2) (omega(0) = 1 for rule R9)."""
    B, a1, a2, a3 = young_coeffs(sigma_s)
    G = math.sqrt(2.0 * math.pi) * float(sigma_s)
    x = np.moveaxis(np.asarray(x, dtype=np.float64), axis, 0)
    N = x.shape[0]
    L = int(60.0 * float(sigma_s)) + 100           # zero padding after the end: the tails fall below 1e-16
    M = N + L
    xp = np.zeros((M,) + x.shape[1:])
    xp[:N] = x
    w = np.zeros((M + 3,) + x.shape[1:])          # w[t + 3] = w_t; w_-1..w_-3 = 0 (rest before the start)
    for t in range(M):
        w[t + 3] = G * B * xp[t] + a1 * w[t + 2] + a2 * w[t + 1] + a3 * w[t]
    y = np.zeros((M + 3,) + x.shape[1:])          # y[t] = y_t; at rest L samples past the end
    for t in range(M - 1, -1, -1):
        y[t] = B * w[t + 3] + a1 * y[t + 1] + a2 * y[t + 2] + a3 * y[t + 3]
    return np.moveaxis(y[:N], 0, axis)


def young2d(x, sigma_s: float) -> np.ndarray:
    """The separable 2-D recursive Gaussian: columns (axis 0), then rows (axis 1)."""
    return young1d(young1d(x, sigma_s, axis=0), sigma_s, axis=1)


def filter_iir(f, p, sigma_s: float, sigma_r: float, mu, tau: float = 0.5):
    """Algorithm 1 with the recursive Gaussian for the convolutions of loop for3
    (P:332-333), in the paper's order: b_k and c = A^+ b (loops for1/for2), then per k
    v += c_k (omega * (b_k f)), r += c_k (omega * b_k), g = v / r.  Rule R9 as in `filter`: eta_hat
    below tau omega(0) phi(0) = tau (omega(0) = 1 by the gain of R17) -> the brute-force (num)/(den)
    with the truncated FIR Gaussian, R = ceil(3 sigma_s).  Returns (g, eta_hat, flagged, n_flagged)."""
    f, p = _fp(f, p)
    H, W, n = f.shape
    b, c = coefficients(p, mu, sigma_r)
    K = b.shape[1]
    v = np.zeros((H, W, n))
    r = np.zeros((H, W))
    for k in range(K):
        bk = b[:, k].reshape(H, W)
        ck = c[:, k].reshape(H, W)
        for ch in range(n):
            v[:, :, ch] += ck * young2d(bk * f[:, :, ch], sigma_s)
        r += ck * young2d(bk, sigma_s)
    g = v / r[..., None]
    floor = tau * phi(np.zeros(1), sigma_r)
    fl = (tau > 0.0) & (r < floor)
    if fl.any():
        pix = np.flatnonzero(fl)
        gb, _ = bruteforce(f, p, "gaussian", sigma_s, sigma_r, -1, pix=pix)
        g.reshape(-1, n)[pix] = gb
    return g, r, fl, int(fl.sum())
