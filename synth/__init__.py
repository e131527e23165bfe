"""Seeded synthetic workloads shaped like the paper's.

This module holds NO arithmetic of the method (no clustering, range kernel, convolution or
combine).  It only draws the inputs f, p that both the fp64 oracle (oracle/) and the CUDA path
(paper_1811_02363_b200) consume, so neither side depends on the other for its inputs.

Stand-ins (the paper's images/datasets are not available):
  C1  tiny 64x64x3 colour bilateral      (BASELINE.json configs[0])
  C2  512x512x3 colour bilateral, K=16/32 (configs[1]; stands in for Lena/Barbara/Peppers)
  C3  512x512x31 hyperspectral bilateral  (configs[2]; stands in for the 33-band set / Pavia)
  C4  512x512x3 colour NLM, PCA-6 guide   (configs[3]; stands in for Kodak NLM)
  C5  4096x4096x3 colour bilateral, K=64  (configs[4]; 4K shape of Table III)

All generators: numpy default_rng(seed) (PCG64), float64 generation, cast to float32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Config", "CONFIGS", "make", "gen_rectangles", "gen_voronoi", "gen_hyperspectral",
           "gen_nlm", "gen_kdistinct", "gen_ir", "pca_patch_guide"]


@dataclass(frozen=True)
class Config:
    name: str
    H: int
    W: int
    n: int
    rho: int
    kind: str            # "gaussian" | "box"
    sigma_s: float       # Gaussian sigma_s (ignored for box)
    radius: int          # window half-width S (R = ceil(3 sigma_s) for Gaussian configs)
    sigma_r: float
    K: int
    seed: int
    R_range: float       # intensity range R of f, used for PSNR normalisation
    bilateral: bool = True   # f is p (f may alias p)
    note: str = ""
    extra: dict = field(default_factory=dict)


NLM_SIGMA = 20.0
CONFIGS = {
    "c1": Config("c1", 64, 64, 3, 3, "gaussian", 3.0, 9, 30.0, 8, 1, 255.0,
                 note="tiny colour bilateral, BASELINE configs[0]"),
    "c2a": Config("c2a", 512, 512, 3, 3, "gaussian", 5.0, 15, 40.0, 16, 2, 255.0,
                  note="colour bilateral K=16, configs[1]"),
    "c2b": Config("c2b", 512, 512, 3, 3, "gaussian", 5.0, 15, 40.0, 32, 2, 255.0,
                  note="colour bilateral K=32, configs[1]"),
    "c3": Config("c3", 512, 512, 31, 31, "gaussian", 3.0, 9, 0.2, 32, 3, 1.0,
                 note="hyperspectral bilateral, configs[2]"),
    "c4": Config("c4", 512, 512, 3, 6, "box", 0.0, 10, 0.4 * NLM_SIGMA * math.sqrt(27.0), 32, 4, 255.0,
                 bilateral=False, note="colour NLM, PCA-6 patch guide, box 21x21, configs[3]"),
    "c5": Config("c5", 4096, 4096, 3, 3, "gaussian", 8.0, 24, 40.0, 64, 5, 255.0,
                 note="large colour bilateral, configs[4]"),
}


def _grid01(H: int, W: int):
    yy = (np.arange(H, dtype=np.float64) / max(H - 1, 1))[:, None, None]
    xx = (np.arange(W, dtype=np.float64) / max(W - 1, 1))[None, :, None]
    return yy, xx


def gen_rectangles(H: int = 64, W: int = 64, seed: int = 1, noise: float = 10.0) -> np.ndarray:
    """C1: background U(0,255)^3; 4 axis-aligned rectangles (sides U{8..31}, colour U(0,255)^3);
    per-channel linear ramp with y and x amplitudes U(-40,40); + N(0, noise^2); clip [0,255]."""
    rng = np.random.default_rng(seed)
    bg = rng.uniform(0.0, 255.0, 3)
    img = np.broadcast_to(bg, (H, W, 3)).copy()
    for _ in range(4):
        h = int(rng.integers(8, 32))
        w = int(rng.integers(8, 32))
        y0 = int(rng.integers(0, max(H - h, 0) + 1))
        x0 = int(rng.integers(0, max(W - w, 0) + 1))
        img[y0:y0 + h, x0:x0 + w] = rng.uniform(0.0, 255.0, 3)
    ay = rng.uniform(-40.0, 40.0, 3)
    ax = rng.uniform(-40.0, 40.0, 3)
    yy, xx = _grid01(H, W)
    img = img + ay * yy + ax * xx
    if noise > 0:
        img = img + rng.normal(0.0, noise, (H, W, 3))
    return np.clip(img, 0.0, 255.0).astype(np.float32)


def _voronoi_labels(H: int, W: int, sites: np.ndarray) -> np.ndarray:
    from scipy.spatial import cKDTree
    tree = cKDTree(sites)
    lab = np.empty((H, W), dtype=np.int32)
    xs = np.arange(W, dtype=np.float64)
    step = max(1, (1 << 20) // W)
    for y0 in range(0, H, step):
        y1 = min(H, y0 + step)
        ys = np.arange(y0, y1, dtype=np.float64)
        pts = np.stack(np.meshgrid(ys, xs, indexing="ij"), axis=-1).reshape(-1, 2)
        _, idx = tree.query(pts)
        lab[y0:y1] = idx.reshape(y1 - y0, W)
    return lab


def gen_voronoi(H: int = 512, W: int = 512, n_cells: int = 40, seed: int = 2,
                noise: float = 10.0) -> np.ndarray:
    """C2/C5: n_cells Voronoi sites U over the image; cell colour U(0,255)^3; per-cell ramp with
    gradients U(-30,30) per channel along y and x (normalised coordinates); + N(0, noise^2); clip."""
    rng = np.random.default_rng(seed)
    sites = rng.uniform(0.0, 1.0, (n_cells, 2)) * np.array([H, W], dtype=np.float64)
    colour = rng.uniform(0.0, 255.0, (n_cells, 3))
    gy = rng.uniform(-30.0, 30.0, (n_cells, 3))
    gx = rng.uniform(-30.0, 30.0, (n_cells, 3))
    lab = _voronoi_labels(H, W, sites)
    yy, xx = _grid01(H, W)
    img = colour[lab] + gy[lab] * yy + gx[lab] * xx
    if noise > 0:
        img = img + rng.normal(0.0, noise, (H, W, 3))
    return np.clip(img, 0.0, 255.0).astype(np.float32)


def gen_hyperspectral(H: int = 512, W: int = 512, bands: int = 31, seed: int = 3,
                      n_spectra: int = 5, n_regions: int = 30) -> np.ndarray:
    """C3: bands on lambda in [0,1]; n_spectra spectra, each a sum of 3 Gaussian bumps (amplitude
    U(.2,1), centre U(0,1), width U(.05,.3)) rescaled to [0.05,0.95]; n_regions Voronoi regions with
    mean abundance a_r ~ Dir(1^5); pixel abundance ~ Dir(50 a_r + 1e-3); f = abundance . spectra
    + N(0, 0.01^2); clip [0,1]."""
    rng = np.random.default_rng(seed)
    lam = np.linspace(0.0, 1.0, bands)
    spectra = np.zeros((n_spectra, bands))
    for s in range(n_spectra):
        for _ in range(3):
            a = rng.uniform(0.2, 1.0)
            c = rng.uniform(0.0, 1.0)
            w = rng.uniform(0.05, 0.3)
            spectra[s] += a * np.exp(-(lam - c) ** 2 / (2.0 * w * w))
        lo, hi = spectra[s].min(), spectra[s].max()
        spectra[s] = 0.05 + 0.9 * (spectra[s] - lo) / max(hi - lo, 1e-12)
    sites = rng.uniform(0.0, 1.0, (n_regions, 2)) * np.array([H, W], dtype=np.float64)
    mean_ab = rng.dirichlet(np.ones(n_spectra), size=n_regions)
    lab = _voronoi_labels(H, W, sites)
    alpha = 50.0 * mean_ab[lab] + 1e-3                        # [H, W, n_spectra]
    g = rng.gamma(alpha)                                      # Dirichlet via normalised gammas
    ab = g / np.maximum(g.sum(axis=-1, keepdims=True), 1e-300)
    img = ab @ spectra + rng.normal(0.0, 0.01, (H, W, bands))
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def pca_patch_guide(img: np.ndarray, m: int = 3, dim: int = 6) -> np.ndarray:
    """NLM guide (R11): m x m x n patches of img with replicate borders, mean-centred
    over all pixels, projected on the top-`dim` eigenvectors of the patch covariance (fp64,
    P:598; sign: largest-magnitude entry positive).  Input preparation, not the method."""
    H, W, n = img.shape
    r = m // 2
    x = img.astype(np.float64)
    pad = np.pad(x, ((r, r), (r, r), (0, 0)), mode="edge")
    cols = []
    for c in range(n):
        for dy in range(m):
            for dx in range(m):
                cols.append(pad[dy:dy + H, dx:dx + W, c])
    P = np.stack(cols, axis=-1).reshape(-1, n * m * m)
    P = P - P.mean(axis=0, keepdims=True)
    C = (P.T @ P) / P.shape[0]
    evals, evecs = np.linalg.eigh(C)
    order = np.argsort(evals)[::-1][:dim]
    B = evecs[:, order]
    sgn = np.sign(B[np.argmax(np.abs(B), axis=0), np.arange(dim)])
    B = B * sgn
    return (P @ B).reshape(H, W, dim).astype(np.float32)


def gen_nlm(H: int = 512, W: int = 512, seed: int = 4, sigma: float = NLM_SIGMA, n_cells: int = 40):
    """C4 (R12): clean = C2 generator without noise; noisy = clean + N(0, sigma^2), clipped;
    guide = PCA-6 of 3x3x3 patches of the noisy image (R11).  Returns (noisy, guide, clean)."""
    clean = gen_voronoi(H, W, n_cells, seed, noise=0.0)
    rng = np.random.default_rng(seed + 1000)
    noisy = np.clip(clean.astype(np.float64) + rng.normal(0.0, sigma, clean.shape), 0.0, 255.0)
    noisy = noisy.astype(np.float32)
    guide = pca_patch_guide(noisy, 3, 6)
    return noisy, guide, clean


def gen_ir(f: np.ndarray, seed: int = 9, noise: float = 5.0) -> np.ndarray:
    """An infrared-like extra guide channel for the low-light use case (the
    paper's IR images are not available): a different linear mix of the image's channels (their mean
    when f has fewer than 3), a smooth random shading, N(0, noise^2), clipped to [0, 255].  [H, W]
    float32."""
    rng = np.random.default_rng(seed)
    x = np.asarray(f, dtype=np.float64)
    H, W = x.shape[:2]
    mix = rng.dirichlet(np.ones(3)) if x.shape[2] >= 3 else None
    base = x[..., :3] @ mix if mix is not None else x.mean(-1)
    yy, xx = _grid01(H, W)
    shade = 30.0 * np.sin(np.pi * (rng.uniform(0.5, 2.0) * yy[..., 0] + rng.uniform(0.5, 2.0) * xx[..., 0]))
    ir = 0.8 * base + shade + rng.normal(0.0, noise, (H, W))
    return np.clip(ir, 0.0, 255.0).astype(np.float32)


def gen_kdistinct(H: int, W: int, K: int, rho: int, seed: int, spread: float = 255.0,
                  min_sep: float = 0.0):
    """Guide taking exactly K distinct values (for the exactness pin P3): a palette of K vectors
    U(0, spread)^rho assigned to blocky regions.  Returns (labels [H,W] int32, palette [K,rho] fp32,
    p [H,W,rho] fp32).  Every palette entry is used at least once."""
    rng = np.random.default_rng(seed)
    for _ in range(1000):
        pal = rng.uniform(0.0, spread, (K, rho))
        d = np.sqrt(((pal[:, None, :] - pal[None, :, :]) ** 2).sum(-1)) + np.eye(K) * 1e9
        if d.min() >= min_sep:
            break
    pal = pal.astype(np.float32)
    by = max(1, H // 8)
    bx = max(1, W // 8)
    blocks = rng.integers(0, K, ((H + by - 1) // by, (W + bx - 1) // bx))
    lab = np.repeat(np.repeat(blocks, by, axis=0), bx, axis=1)[:H, :W].astype(np.int32)
    lab.reshape(-1)[:K] = np.arange(K, dtype=np.int32)        # every value present
    return lab, pal, pal[lab]


def make(name: str, H: int | None = None, W: int | None = None):
    """Inputs of a named config: returns (cfg, f, p) with f [H,W,n], p [H,W,rho] float32
    (p is f for bilateral configs).  H/W override the size (same recipe, for parity cases)."""
    cfg = CONFIGS[name]
    Hh = H or cfg.H
    Ww = W or cfg.W
    if name == "c1":
        f = gen_rectangles(Hh, Ww, cfg.seed)
        return cfg, f, f
    if name in ("c2a", "c2b"):
        f = gen_voronoi(Hh, Ww, 40, cfg.seed)
        return cfg, f, f
    if name == "c3":
        f = gen_hyperspectral(Hh, Ww, 31, cfg.seed)
        return cfg, f, f
    if name == "c4":
        noisy, guide, _clean = gen_nlm(Hh, Ww, cfg.seed)
        return cfg, noisy, guide
    if name == "c5":
        f = gen_voronoi(Hh, Ww, 200, cfg.seed)
        return cfg, f, f
    raise KeyError(name)
