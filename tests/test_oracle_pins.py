"""Pins of the fp64 oracle against what the paper and the mathematics fix.

Every test here runs on CPU (no GPU) and checks the oracle against something other than itself:
closed forms, invariants, special cases reducing to textbook/library routines, or brute force on
tiny inputs.  Pin ids (P1..P13) follow SURVEY.md section 8(c).
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


# ---------------------------------------------------------------- P1: kernels -----
def test_p1_range_kernel_closed_form():
    assert oracle.phi([0.0, 0.0, 0.0], 17.0) == 1.0
    g = GOLD["phi_sigma30_x30"]
    assert abs(oracle.phi([30.0], 30.0) - g["value"]) < 1e-15
    # isotropic in rho dims: only ||x|| matters
    assert abs(oracle.phi([18.0, 24.0], 30.0) - g["value"]) < 1e-15
    assert oracle.phi([1e4], 1.0) == 0.0 or oracle.phi([1e4], 1.0) < 1e-300


def test_p1_spatial_taps_closed_form():
    w = oracle.spatial_taps("gaussian", 5.0, 15)
    assert w.shape == (31,)
    assert w[15] == 1.0
    g = GOLD["omega_sigma5_j50"]
    assert abs(w[15 + 5] * w[15] - g["value"]) < 1e-15      # omega((5,0)) = w_5 w_0
    assert np.allclose(w, w[::-1])
    assert oracle.radius("gaussian", 3.0) == 9 and oracle.radius("gaussian", 8.0) == 24
    assert oracle.radius("gaussian", 2.5) == 8                   # ceil(3 sigma_s) (R7)
    assert np.all(oracle.spatial_taps("box", 0.0, 10) == 1.0)


# ---------------------------------------------------------------- P2: clustering ---------------
def _blobs(seed, centres, per, spread):
    rng = np.random.default_rng(seed)
    pts = np.concatenate([c + rng.uniform(-spread, spread, (per, len(c))) for c in centres])
    return pts


def test_p2_k1_is_global_mean():
    _, f, _ = synth.make("c1")
    cen, lab, sse, ek = oracle.cluster(f, 1)
    P = f.reshape(-1, 3).astype(np.float64)
    assert np.allclose(cen[0], P.mean(axis=0), rtol=0, atol=1e-9)
    assert np.all(lab == 0)
    assert abs(ek - ((P - P.mean(0)) ** 2).sum()) <= 1e-9 * ek


def test_p2_k_distinct_values_gives_zero_error():
    lab, pal, p = synth.gen_kdistinct(32, 32, 6, 3, seed=7)
    cen, labels, sse, ek = oracle.cluster(p, 6)
    assert ek == 0.0
    # centres equal the distinct values as a set
    got = sorted(map(tuple, np.round(cen, 9)))
    want = sorted(map(tuple, np.round(pal.astype(np.float64), 9)))
    assert got == want
    with pytest.raises(oracle.OracleKError) as e:
        oracle.cluster(p, 7)
    assert e.value.achievable == 6                               # R5 names the achievable K


def test_p2_two_blobs_split_exactly():
    pts = _blobs(3, [np.zeros(3), np.full(3, 200.0)], 100, 1.0)
    cen, lab, _, _ = oracle.cluster(pts, 2)
    assert set(lab[:100]) == {lab[0]} and set(lab[100:]) == {lab[100]} and lab[0] != lab[100]
    assert np.allclose(cen[lab[0]], pts[:100].mean(0), atol=1e-9)
    assert np.allclose(cen[lab[100]], pts[100:].mean(0), atol=1e-9)


@pytest.mark.parametrize("seed", [0, 1])
def test_p2_centres_are_leaf_means_and_ek_is_sse(seed):
    rng = np.random.default_rng(seed)
    pts = rng.normal(0, 30, (3000, 4)) + rng.integers(0, 4, (3000, 1)) * 60.0
    K = 9
    cen, lab, sse, ek = oracle.cluster(pts, K)
    assert sorted(set(lab.tolist())) == list(range(K))          # K non-empty leaves
    tot = 0.0
    for k in range(K):
        m = pts[lab == k]
        assert np.allclose(cen[k], m.mean(0), rtol=0, atol=1e-9)
        s = ((m - m.mean(0)) ** 2).sum()
        assert abs(sse[k] - s) <= 1e-9 * max(s, 1.0)
        tot += s
    assert abs(ek - tot) <= 1e-9 * tot


def test_p2_bisection_refines_the_max_sse_leaf():
    """R2: going from K to K+1 leaves splits exactly the leaf of largest SSE (ties: lowest id),
    keeps its id for child 0 and gives child 1 the id K; E_K is non-increasing in K."""
    _, f, _ = synth.make("c1")
    prev = None
    eks = []
    for K in range(1, 13):
        cen, lab, sse, ek = oracle.cluster(f, K)
        eks.append(ek)
        if prev is not None:
            plab, psse = prev
            s = int(np.argmax(psse))
            assert psse[s] == psse.max()
            same = plab != s
            assert np.all(lab[same] == plab[same])               # other leaves untouched
            split = plab == s
            assert set(lab[split].tolist()) == {s, K - 1}
        prev = (lab, sse)
    assert all(eks[i + 1] <= eks[i] * (1 + 1e-12) for i in range(len(eks) - 1))


def test_p2_lloyd_fixed_point():
    """R4: after a converged 2-means split every member is assigned to the nearer of the two
    child means (ties -> first); brute-force check of the Lloyd fixed point on a small leaf."""
    rng = np.random.default_rng(11)
    pts = rng.normal(0, 1, (400, 2)) * [3.0, 1.0]
    cen, lab, _, _ = oracle.cluster(pts, 2)
    d0 = ((pts - cen[0]) ** 2).sum(1)
    d1 = ((pts - cen[1]) ** 2).sum(1)
    nearest = np.where(d0 <= d1, 0, 1)
    assert np.array_equal(nearest, lab)
    # and the split is the best 2-partition along the separating hyperplane direction:
    # SSE after split must be below the parent SSE
    assert ((pts[lab == 0] - cen[0]) ** 2).sum() + ((pts[lab == 1] - cen[1]) ** 2).sum() < \
        ((pts - pts.mean(0)) ** 2).sum()


def test_p2_farthest_pair_seed_on_line():
    """P:329 seeds 2-means with the farthest pair.  On collinear points 0..m-1 the farthest pair is
    (0, m-1), so the first Lloyd step splits at the midpoint and converges to the two halves."""
    m = 101
    pts = np.arange(m, dtype=np.float64)[:, None]
    cen, lab, _, _ = oracle.cluster(pts, 2)
    assert np.array_equal(lab, (np.arange(m) > 50).astype(np.int32))
    assert np.allclose(sorted(cen[:, 0]), [25.0, 75.5])


def _bruteforce_farthest_pair(P, members, cap):
    """R3 written out by brute force: every pair (a < b) of the stride sample members[0::ceil(m/cap)],
    squared distance summed over dimensions in index order, the lexicographically smallest (a, b)
    among the maximisers."""
    m = len(members)
    stride = -(-m // cap)
    smp = np.asarray(members)[0::stride]
    X = P[smp]
    best, arg = -1.0, (0, 0)
    for a in range(len(smp) - 1):
        diff = X[a + 1:] - X[a]
        d = np.zeros(len(diff))
        for k in range(P.shape[1]):            # (d0^2 + d1^2) + d2^2 ..., the definition's order
            d = d + diff[:, k] * diff[:, k]
        j = int(np.argmax(d))                  # first maximiser in the row
        if d[j] > best:
            best, arg = float(d[j]), (a, a + 1 + j)
    if len(smp) < 2:
        return int(smp[0]), int(smp[0])
    return int(smp[arg[0]]), int(smp[arg[1]])


@pytest.mark.parametrize("m,cap,integer,seed", [(1024, 1024, False, 1), (1025, 1024, False, 2),
                                                (5000, 1024, False, 3), (100000, 1024, False, 4),
                                                (3000, 1024, True, 5), (6001, 1024, True, 6),
                                                (700, 64, True, 7), (1, 1024, False, 8)])
def test_p2_farthest_pair_stride_sample_against_bruteforce(m, cap, integer, seed):
    """R3: the seeds are the farthest pair of the stride sample members[0::ceil(m/1024)] in
    member order (ascending pixel index), ties -> lexicographically smallest pair.  The members are a
    sparse ascending subset of the pixels; the farthest pair of ALL members is planted off the
    sample (so a search over every member, or another stride, gives a different pair), and integer
    coordinates in a small range make many pairs tie."""
    rng = np.random.default_rng(seed)
    N = 3 * m + 10
    P = (rng.integers(0, 12, (N, 3)).astype(np.float64) if integer else rng.normal(0, 10, (N, 3)))
    members = np.sort(rng.choice(N, m, replace=False))
    stride = -(-m // cap)
    if stride > 1 and not integer:
        P[members[1]] = (1e3, 1e3, 1e3)        # off the sample: index 1 is not a multiple of the stride
        P[members[-2 if (m - 2) % stride else -3]] = (-1e3, -1e3, -1e3)
    a, b = oracle.farthest_pair(P, members, cap)
    assert (a, b) == _bruteforce_farthest_pair(P, members, cap)
    if stride > 1 and not integer:
        assert 1e3 not in (P[a][0], P[b][0])   # the planted pair is not seen


def test_p2_empty_side_is_reseeded_at_the_farthest_member():
    """R4: when one side of a 2-means step is empty it is reseeded at the member farthest from the
    other centre.  Construction: 2048 points, so the stride sample (stride 2) holds only the even
    pixels, which are all v = 0; the farthest pair of the sample is two copies of v, every point
    ties to the first centre, side 1 is empty.  The odd pixels are 400 copies of a = (100, 0, 0)
    followed by 624 copies of c = (-40, 0, 0).  The member farthest from v is the first a (ties ->
    first), so c1 = a, and Lloyd converges to {v, c} | {a}: centres (-40 * 624 / 1648, 0, 0) and a,
    E_K = the two leaves' SSE written out in closed form."""
    N = 2048
    P = np.zeros((N, 3))
    odd = np.arange(1, N, 2)
    P[odd[:400]] = (100.0, 0.0, 0.0)
    P[odd[400:]] = (-40.0, 0.0, 0.0)
    cen, lab, sse, ek = oracle.cluster(P, 2)
    want = np.zeros(N, dtype=np.int32)
    want[odd[:400]] = 1
    assert np.array_equal(lab, want)
    m0 = 1024 + 624
    x0 = -40.0 * 624 / m0
    assert np.allclose(cen[0], (x0, 0, 0), rtol=0, atol=1e-12) and np.array_equal(cen[1], (100.0, 0, 0))
    sse0 = 1024 * x0 ** 2 + 624 * (-40.0 - x0) ** 2
    assert abs(ek - sse0) <= 1e-9 * sse0 and sse[1] == 0.0


# ---------------------------------------------------------------- P4: A and A^+ ----------------
def test_p4_gram_closed_form():
    g = GOLD["gram_K2"]
    A = oracle.gram(np.array(g["mu"]), g["sigma_r"])
    assert np.allclose(A, np.array(g["A"]), rtol=0, atol=1e-15)


@pytest.mark.parametrize("K,dup", [(5, False), (16, False), (7, True)])
def test_p4_pinv_moore_penrose(K, dup):
    rng = np.random.default_rng(K)
    mu = rng.uniform(0, 255, (K, 3))
    if dup:
        mu[3] = mu[1]                                            # rank-deficient A
    A = oracle.gram(mu, 40.0)
    Ap, lam, rank, tol = oracle.pinv(A)
    assert rank == (K - 1 if dup else K)
    nrm = np.linalg.norm(A)
    assert np.linalg.norm(A @ Ap @ A - A) <= 1e-10 * nrm
    assert np.linalg.norm(Ap @ A @ Ap - Ap) <= 1e-10 * np.linalg.norm(Ap)
    assert np.linalg.norm((A @ Ap).T - A @ Ap) <= 1e-10 * np.linalg.norm(A @ Ap)
    assert np.linalg.norm((Ap @ A).T - Ap @ A) <= 1e-10 * np.linalg.norm(Ap @ A)
    ref = np.linalg.pinv(A, rcond=tol / np.abs(lam).max(), hermitian=True)    # library routine
    assert np.linalg.norm(Ap - ref) <= 1e-9 * np.linalg.norm(ref)
    assert abs(tol - K * np.spacing(np.abs(lam).max())) <= 1e-30               # MATLAB default


# ---------------------------------------------------------------- P5: coefficients -------------
def test_p5_b_closed_form_and_unit_coefficients():
    g = GOLD["b_K2"]
    b, c = oracle.coefficients(np.array([g["p"]]), np.array(g["mu"]), g["sigma_r"])
    assert np.allclose(b[0], g["b"], rtol=0, atol=1e-15)
    rng = np.random.default_rng(5)
    mu = rng.uniform(0, 255, (8, 3))
    b, c = oracle.coefficients(mu, mu, 40.0)                     # p(i) = mu_s  =>  c = e_s
    assert np.allclose(c, np.eye(8), atol=1e-10)


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_p5_nystrom_diagonal_in_unit_interval(name):
    """0 <= c(i)^T b(i) = b^T A^+ b <= phi(0) = 1: Schur complement of the PSD Gaussian kernel
    matrix on {mu_k} u {p(i)}; holds for any guide."""
    cfg, f, p = synth.make(name, 48, 48)
    cen, _, _, _ = oracle.cluster(p, cfg.K)
    b, c = oracle.coefficients(p, cen.astype(np.float32), cfg.sigma_r)
    q = (b * c).sum(1)
    assert q.min() >= -1e-9 and q.max() <= 1 + 1e-9


def test_p5_surrogate_optimality():
    """c(i) = A^+ b(i) minimises ||A c - b(i)|| (opt): no random competitor does better."""
    rng = np.random.default_rng(9)
    mu = rng.uniform(0, 255, (6, 3))
    p = rng.uniform(0, 255, (20, 3))
    b, c = oracle.coefficients(p, mu, 40.0)
    A = oracle.gram(mu, 40.0)
    for i in range(20):
        best = np.linalg.norm(A @ c[i] - b[i])
        for _ in range(100):
            v = c[i] + rng.normal(0, 0.1, 6)
            assert np.linalg.norm(A @ v - b[i]) >= best - 1e-12


# ---------------------------------------------------------------- P6: convolution --------------
@pytest.mark.parametrize("kind,s,r", [("gaussian", 2.0, -1), ("gaussian", 1.3, 4), ("box", 0.0, 2)])
def test_p6_separable_equals_direct_window_sum(kind, s, r):
    rng = np.random.default_rng(1)
    H, W = 13, 17
    x = rng.normal(0, 1, (H, W))
    out = oracle.conv2(x, kind, s, r)
    R = oracle.radius(kind, s, r)
    w = oracle.spatial_taps(kind, s, r)
    ref = np.zeros_like(x)
    for y in range(H):
        for xx in range(W):
            acc = 0.0
            for ty in range(-R, R + 1):
                for tx in range(-R, R + 1):
                    yy, x2 = y - ty, xx - tx
                    if 0 <= yy < H and 0 <= x2 < W:
                        acc += w[ty + R] * w[tx + R] * x[yy, x2]
            ref[y, xx] = acc
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    from scipy.ndimage import correlate                                  # library routine
    assert np.allclose(out, correlate(x, np.outer(w, w), mode="constant", cval=0.0), atol=1e-12)


def test_p6_impulse_response_is_taps_and_linearity():
    H = W = 41
    x = np.zeros((H, W))
    x[20, 20] = 1.0
    out = oracle.conv2(x, "gaussian", 3.0)
    w = oracle.spatial_taps("gaussian", 3.0)
    R = 9
    assert np.allclose(out[20 - R:21 + R, 20 - R:21 + R], np.outer(w, w), atol=1e-15)
    assert np.abs(out).sum() - np.outer(w, w).sum() < 1e-12
    rng = np.random.default_rng(2)
    a, b = rng.normal(size=(2, 20, 23))
    lhs = oracle.conv2(2.5 * a - 0.5 * b, "gaussian", 2.0)
    rhs = 2.5 * oracle.conv2(a, "gaussian", 2.0) - 0.5 * oracle.conv2(b, "gaussian", 2.0)
    assert np.allclose(lhs, rhs, atol=1e-11)


# ---------------------------------------------------------------- P3 / P7: filter identities ---
def test_p3_k_distinct_exactness_fast_equals_bruteforce():
    """Guide with exactly K distinct values and centres = those values: b(i) = A e_s, c(i) = e_s,
    so Algorithm 1 equals (num)/(den) (opt, defAb)."""
    lab, pal, p = synth.gen_kdistinct(40, 36, 8, 3, seed=3, spread=255.0, min_sep=60.0)
    rng = np.random.default_rng(4)
    f = rng.uniform(0, 255, (40, 36, 3)).astype(np.float32)
    for (kind, s, r, sr) in [("gaussian", 3.0, 9, 40.0), ("box", 0.0, 4, 60.0)]:
        g, eta, fl, nf = oracle.filter(f, p, kind, s, sr, pal, r=r, tau=0.0)
        gb, etab = oracle.bruteforce(f, p, kind, s, sr, r=r)
        assert np.abs(g - gb).max() <= 1e-9
        assert np.abs(eta - etab).max() <= 1e-9 * etab.max()
        gh = oracle.filter_hard(f, p, kind, s, sr, pal, lab, r=r)       # hard variant too
        assert np.abs(gh - gb).max() <= 1e-9


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_p7_nystrom_identity(name):
    """Appendix A: sum_k c_k(i) v_k(i) = sum_j omega(j) b(i)^T A^+ b(i-j) f(i-j): the
    plane-based Algorithm 1 equals the direct window evaluation with phi~(i,i') = b(i)^T A^+ b(i')."""
    cfg, f, p = synth.make(name, 40, 44)
    cen, _, _, _ = oracle.cluster(p, min(cfg.K, 12))
    mu = cen.astype(np.float32)
    r = min(cfg.radius, 6)
    g, eta, _, _ = oracle.filter(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, mu, r=r, tau=0.0)
    gn, etan = oracle.nystrom(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, mu, r=r)
    ok = np.abs(etan) > 1e-3
    assert np.abs(eta - etan).max() <= 1e-9 * np.abs(etan).max()
    assert np.abs(g - gn)[ok].max() <= 1e-8 * cfg.R_range
    # and the per-pixel evaluator agrees with the plane-based filter
    pix = np.random.default_rng(0).choice(40 * 44, 50, replace=False)
    gp, etap, _ = oracle.filter_pixels(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, mu, pix, r=r, tau=0.0)
    assert np.abs(gp - g.reshape(-1, cfg.n)[pix]).max() <= 1e-9 * cfg.R_range
    assert np.abs(etap - eta.reshape(-1)[pix]).max() <= 1e-12 * np.abs(eta).max()


# ---------------------------------------------------------------- P8 / P9: special cases -------
def test_p8_large_sigma_r_is_normalised_blur():
    """sigma_r -> inf: A -> all-ones (rank 1), phi -> 1, g = (omega*f)/(omega*1)."""
    from scipy.ndimage import correlate1d
    _, f, p = synth.make("c1", 30, 33)
    cen, _, _, _ = oracle.cluster(p, 4)
    g, eta, _, _ = oracle.filter(f, p, "gaussian", 2.0, 1e9, cen, tau=0.0)
    w = oracle.spatial_taps("gaussian", 2.0)
    def blur(x):
        t = correlate1d(x, w, axis=1, mode="constant", cval=0.0)
        return correlate1d(t, w, axis=0, mode="constant", cval=0.0)
    ones = blur(np.ones((30, 33)))
    ref = np.stack([blur(f[..., c].astype(np.float64)) for c in range(3)], -1) / ones[..., None]
    assert np.abs(g - ref).max() <= 1e-6


def test_p9_constant_image_maps_to_itself():
    rng = np.random.default_rng(8)
    p = rng.uniform(0, 255, (24, 28, 3))
    f = np.full((24, 28, 2), 77.25)
    mu = rng.uniform(0, 255, (6, 3))
    for kind, s, r in [("gaussian", 2.0, -1), ("box", 0.0, 3)]:
        g, eta, fl, nf = oracle.filter(f, p, kind, s, 40.0, mu, r=r, tau=0.0)
        ok = np.abs(eta) > 1e-6
        assert np.abs(g - 77.25)[ok].max() <= 1e-8
        gb, _ = oracle.bruteforce(f, p, kind, s, 40.0, r=r)
        assert np.abs(gb - 77.25).max() <= 1e-10


def test_r9_flagged_pixels_take_bruteforce_values():
    cfg, f, p = synth.make("c4", 48, 48)
    cen, _, _, _ = oracle.cluster(p, cfg.K)
    g, eta, fl, nf = oracle.filter(f, p, "box", 0.0, cfg.sigma_r, cen.astype(np.float32), r=cfg.radius, tau=0.5)
    assert nf == fl.sum()
    assert np.all((eta < 0.5) == fl)
    if nf:
        gb, _ = oracle.bruteforce(f, p, "box", 0.0, cfg.sigma_r, r=cfg.radius)
        assert np.array_equal(g[fl], gb[fl])


# ---------------------------------------------------------------- P10: error falls with K ------
@pytest.mark.parametrize("seed", [1, 2])
def test_p10_error_falls_as_k_grows(seed):
    """approximation error against (num)/(den) falls as K grows."""
    from scipy.stats import spearmanr
    f = synth.gen_rectangles(48, 48, seed)
    gb, _ = oracle.bruteforce(f, f, "gaussian", 3.0, 30.0)
    Ks = [1, 2, 4, 8, 16, 32]
    m = []
    for K in Ks:
        cen, _, _, _ = oracle.cluster(f, K)
        g, _, _, _ = oracle.filter(f, f, "gaussian", 3.0, 30.0, cen, tau=0.0)
        m.append(oracle.mse(g, gb, 255.0))
    rho_s = spearmanr(Ks, m).correlation
    assert rho_s <= -0.9, (m, rho_s)
    assert m[-1] < m[2] < m[0]


# ---------------------------------------------------------------- P11: Theorem 1 ---------------
@pytest.mark.parametrize("seed", range(4))
def test_p11_theorem1_bound_hard_variant(seed):
    """Theorem 1: sum_i ||g_hard(i) - g(i)||^2 <= C L^2 n |W|^2 E_K with
    C = 2 sqrt(R)/(omega(0) phi(0)), L = e^{-1/2}/sigma_r."""
    rng = np.random.default_rng(seed)
    f = rng.uniform(0, 255, (20, 20, 3))
    sr, s = 40.0, 2.0
    R = oracle.radius("gaussian", s)
    gb, _ = oracle.bruteforce(f, f, "gaussian", s, sr)
    for K in (2, 4, 8):
        cen, lab, _, ek = oracle.cluster(f, K)
        gh = oracle.filter_hard(f, f, "gaussian", s, sr, cen, lab)
        lhs = ((gh - gb) ** 2).sum()
        C = 2.0 * math.sqrt(255.0) / 1.0
        L = math.exp(-0.5) / sr
        rhs = C * L * L * 3 * ((2 * R + 1) ** 2) ** 2 * ek
        assert lhs <= rhs


def test_p11_hard_is_cluster_by_cluster_ratio():
    """(HDapprox2): g_hard(i) = v_s(i)/r_s(i) -- check against planes built with numpy."""
    from scipy.ndimage import correlate1d
    _, f, p = synth.make("c1", 24, 26)
    cen, lab, _, _ = oracle.cluster(p, 5)
    gh = oracle.filter_hard(f, p, "gaussian", 2.0, 30.0, cen, lab)
    w = oracle.spatial_taps("gaussian", 2.0)
    def blur(x):
        return correlate1d(correlate1d(x, w, axis=1, mode="constant"), w, axis=0, mode="constant")
    lab2 = lab.reshape(24, 26)
    P = p.astype(np.float64)
    ref = np.zeros((24, 26, 3))
    for k in range(5):
        bk = np.exp(-((P - cen[k]) ** 2).sum(-1) / (2 * 30.0 ** 2))
        rk = blur(bk)
        for c in range(3):
            vk = blur(bk * f[..., c])
            ref[..., c] = np.where(lab2 == k, vk / rk, ref[..., c])
    assert np.abs(gh - ref).max() <= 1e-9


# ---------------------------------------------------------------- P12: metric ------------------
def test_p12_psnr_closed_form():
    g = GOLD["psnr_uniform_offset"]
    a = np.zeros((10, 10, 3))
    b = a + g["delta"]
    assert abs(oracle.mse(a, b, 1.0) - g["mse"]) < 1e-15
    assert abs(oracle.psnr(a, b, 1.0) - g["psnr"]) < 1e-9
    assert abs(oracle.psnr(a * 255, b * 255, 255.0) - g["psnr"]) < 1e-9
    assert oracle.psnr(a, a) == float("inf")


# ---------------------------------------------------------------- P13: determinism -------------
def test_p13_thread_count_independent():
    code = ("import numpy as np, oracle, synth, hashlib;"
            "cfg,f,p=synth.make('c1',32,40);"
            "c,l,s,e=oracle.cluster(p,6);"
            "g,eta,fl,nf=oracle.filter(f,p,'gaussian',3.0,30.0,c.astype(np.float32));"
            "print(hashlib.sha256(c.tobytes()+l.tobytes()+g.tobytes()).hexdigest())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = set()
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=root)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert len(outs) == 1


# ------------------------------------------------------- PCA-NLM patch guide (NEXT #3) -----------
def _patch_bruteforce(img, i, j, m):
    """The patch of pixel (i, j) written out: channel-major, rows then columns, replicate borders."""
    H, W, n = img.shape
    r = m // 2
    return np.array([img[min(max(i + dy, 0), H - 1), min(max(j + dx, 0), W - 1), c]
                     for c in range(n) for dy in range(-r, r + 1) for dx in range(-r, r + 1)])


def test_pca_guide_full_rank_reconstructs_patches():
    """With dim = n m^2 the projection is invertible: guide @ B^T + mean gives back every patch, which
    is checked against patches written out pixel by pixel (order, borders, centring)."""
    rng = np.random.default_rng(7)
    img = rng.uniform(0, 255, (6, 7, 2))
    g, B, mu, ev = oracle.pca_guide(img, 3, 18)
    rec = g.reshape(-1, 18) @ B.T + mu
    for (i, j) in [(0, 0), (0, 6), (5, 0), (5, 6), (2, 3), (3, 1)]:
        assert np.allclose(rec[i * 7 + j], _patch_bruteforce(img, i, j, 3), atol=1e-9)


def test_pca_guide_matches_svd_and_is_orthonormal():
    """Independent route: the right singular vectors of the centred patch matrix (SVD) span the same
    leading directions with eigenvalues s^2 / N; the basis is orthonormal, sorted, sign-normalised."""
    rng = np.random.default_rng(8)
    img = rng.uniform(0, 1, (12, 10, 3))
    g, B, mu, ev = oracle.pca_guide(img, 3, 6)
    P = np.stack([_patch_bruteforce(img, i, j, 3) for i in range(12) for j in range(10)])
    Pc = P - P.mean(0)
    U, s, Vt = np.linalg.svd(Pc, full_matrices=False)
    assert np.allclose(ev, (s[:6] ** 2) / P.shape[0], rtol=1e-10)
    for k in range(6):
        v = Vt[k] * np.sign(Vt[k][np.argmax(np.abs(Vt[k]))])
        assert np.allclose(B[:, k], v, atol=1e-8)
    assert np.allclose(B.T @ B, np.eye(6), atol=1e-12)
    assert all(ev[k] >= ev[k + 1] for k in range(5))
    assert all(B[np.argmax(np.abs(B[:, k])), k] > 0 for k in range(6))
    cov = g.reshape(-1, 6).T @ g.reshape(-1, 6) / P.shape[0]
    assert np.allclose(cov, np.diag(ev), atol=1e-9 * ev[0])


def test_pca_guide_constant_image_is_zero():
    g, B, mu, ev = oracle.pca_guide(np.full((5, 6, 3), 42.0), 3, 4)
    assert np.all(g == 0.0) and np.allclose(mu, 42.0)


# ---------------------------------------- NEXT #1: Young's recursive Gaussian -----
# The recursion is pinned by what its design fixes: unit DC gain per pass (B = 1 - sum a), a
# zero-phase (symmetric) impulse response from the causal + anti-causal pair, a Gaussian shape of
# the requested sigma within the approximation's known error, and separability; the filter built on
# it by the paper's invariants (a constant image maps to itself; close to the FIR filter).
@pytest.mark.parametrize("s", [0.5, 1.0, 2.0, 2.5, 5.0, 8.0])
def test_iir_dc_gain_and_symmetry(s):
    G = math.sqrt(2.0 * math.pi) * s
    c = oracle.young1d(np.ones(60 * int(math.ceil(s)) + 200), s)
    mid = c.size // 2
    assert abs(c[mid] / G - 1.0) < 1e-10              # unit DC gain per pass, times the R17 gain G
    x = np.zeros(c.size)
    x[mid] = 1.0
    h = oracle.young1d(x, s)
    t = np.arange(1, int(8 * s) + 2)
    assert np.max(np.abs(h[mid + t] - h[mid - t])) < 1e-12 * h[mid]   # zero phase
    assert abs(h.sum() / G - 1.0) < 1e-9               # the impulse response integrates to G


@pytest.mark.parametrize("s", [0.5, 1.3, 2.5, 4.0, 8.0])
def test_iir_impulse_response_closed_form(s):
    """The causal recursion w_t = G B x_t + a1 w_{t-1} + a2 w_{t-2} + a3 w_{t-3} has the impulse response
    G B sum_i r_i p_i^t (t >= 0), p_i the roots of z^3 - a1 z^2 - a2 z - a3, r_i = p_i^2 / prod_{j != i}
    (p_i - p_j); the anti-causal pass mirrors it with gain B.  Their cascade, away from the image ends, is
    y_t = G B^2 sum_{i,j} r_i r_j p_i^|t| / (1 - p_i p_j) -- a closed form from the coefficients alone
    (numpy's polynomial roots), so a wrong index, sign or pass direction in the oracle's loops fails it."""
    B, a1, a2, a3 = oracle.young_coeffs(s)
    G = math.sqrt(2.0 * math.pi) * s
    pr = np.roots([1.0, -a1, -a2, -a3]).astype(np.complex128)
    assert np.all(np.abs(pr) < 1.0)                      # a stable causal recursion
    r = np.array([pr[i] ** 2 / np.prod([pr[i] - pr[j] for j in range(3) if j != i]) for i in range(3)])
    n = int(60 * s) + 301
    x = np.zeros(n)
    x[n // 2] = 1.0
    h = oracle.young1d(x, s)
    t = np.arange(int(6 * s) + 3)
    want = np.real(G * B * B * np.einsum("i,j,it,ij->t", r, r, pr[:, None] ** t[None, :],
                                         1.0 / (1.0 - pr[:, None] * pr[None, :])))
    assert np.max(np.abs(h[n // 2 + t] - want)) < 1e-11 * abs(want[0])
    assert np.max(np.abs(h[n // 2 - t] - want)) < 1e-11 * abs(want[0])


@pytest.mark.parametrize("s,tol", [(0.5, 0.1), (1.0, 0.1), (2.0, 0.07), (2.5, 0.06), (5.0, 0.04), (8.0, 0.03)])
def test_iir_impulse_response_is_gaussian(s, tol):
    n = int(20 * s) + 41
    x = np.zeros(n)
    x[n // 2] = 1.0
    h = oracle.young1d(x, s)
    t = np.arange(n) - n // 2
    assert np.max(np.abs(h - np.exp(-t * t / (2.0 * s * s)))) < tol     # peak ~1 (omega(0) = 1, R17)
    if s >= 2.0:   # the width: h(sigma) / h(0) = exp(-1/2) of a Gaussian of that sigma
        hs = np.interp(s, t, h)
        assert abs(hs / h[n // 2] - math.exp(-0.5)) < (0.08 if s < 3.0 else 0.03)   # wider at small sigma


def test_iir_separable_and_zero_outside():
    rng = np.random.default_rng(5)
    a, b = rng.random(37), rng.random(23)
    y = oracle.young2d(np.outer(a, b), 2.0)
    assert np.allclose(y, np.outer(oracle.young1d(a, 2.0), oracle.young1d(b, 2.0)), rtol=1e-12, atol=1e-14)
    # zero outside Omega at both ends (R17): the result is the convolution of the zero-extended signal
    # with the symmetric impulse response, so reversing the input reverses the output
    for s in (0.7, 2.0, 6.0):
        assert np.allclose(oracle.young1d(a[::-1], s), oracle.young1d(a, s)[::-1], rtol=0, atol=1e-12)
        # and zeros added outside change nothing on the support
        z = np.concatenate([np.zeros(50), a, np.zeros(7)])
        assert np.allclose(oracle.young1d(z, s)[50:50 + a.size], oracle.young1d(a, s), rtol=0, atol=1e-12)


def test_iir_filter_constant_image_and_close_to_fir():
    cfg, f, p = synth.make("c1", 40, 44)
    mu = oracle.cluster(p, 6)[0]
    g, eta, fl, nf = oracle.filter_iir(np.full_like(f, 77.0), np.full_like(p, 77.0), 3.0, 30.0, np.full((1, 3), 77.0))
    assert np.allclose(g, 77.0, rtol=0, atol=1e-9)
    gi, _, _, _ = oracle.filter_iir(f, p, cfg.sigma_s, cfg.sigma_r, mu)
    gf, _, _, _ = oracle.filter(f, p, "gaussian", cfg.sigma_s, cfg.sigma_r, mu)
    d = np.abs(gi - gf) * 255.0 / cfg.R_range
    assert d.mean() < 1.0 and d.max() < 12.0    # the recursion approximates the truncated Gaussian


# ------------------------------------------- anisotropic range kernel (NEXT #3) ------
def _aniso_case(seed, H=24, W=30):
    rng = np.random.default_rng(seed)
    cfg, f, p = synth.make("c1", H, W)
    ir = synth.gen_ir(f, seed=seed)                         # an extra guide channel
    pg = np.concatenate([p.astype(np.float64), ir[..., None]], -1)
    sig = np.array([30.0, 45.0, 60.0, 12.0])
    return f, pg, sig, rng


def test_aniso_phi_closed_form():
    """phi(x) = exp(-sum_d x_d^2 / 2 sigma_d^2): one standard deviation along each axis gives e^-1/2."""
    sig = np.array([3.0, 50.0, 10.0])
    for d in range(3):
        x = np.zeros(3)
        x[d] = sig[d]
        assert abs(oracle.phi_aniso(x, sig) - math.exp(-0.5)) <= 1e-15
    assert oracle.phi_aniso(np.array([3.0, 50.0, 10.0]), sig) == pytest.approx(math.exp(-1.5), rel=1e-15)


def test_aniso_equal_sigmas_is_the_isotropic_oracle():
    """Special case: every sigma_d = sigma_r reduces filter_aniso / bruteforce_aniso to the (pinned)
    isotropic C oracle."""
    cfg, f, p = synth.make("c1", 26, 31)
    cen, _, _, _ = oracle.cluster(p, 6)
    g1, e1, fl1, _ = oracle.filter(f, p, "gaussian", 2.0, 30.0, cen, r=6)
    g2, e2, fl2, _ = oracle.filter_aniso(f, p, "gaussian", 2.0, [30.0] * 3, cen, r=6)
    assert np.allclose(g1, g2, rtol=0, atol=1e-9) and np.allclose(e1, e2, rtol=1e-12, atol=1e-12)
    pix = np.arange(0, 26 * 31, 7)
    b1, _ = oracle.bruteforce(f, p, "gaussian", 2.0, 30.0, r=6, pix=pix)
    b2, _ = oracle.bruteforce_aniso(f, p, "gaussian", 2.0, [30.0] * 3, r=6, pix=pix)
    assert np.allclose(b1, b2, rtol=0, atol=1e-9)


@pytest.mark.parametrize("seed", [1, 2])
def test_aniso_equals_isotropic_on_the_scaled_guide(seed):
    """The identity behind the GPU path: per-channel scaling of the guide by 1/sigma_d
    with sigma_r = 1 equals the anisotropic kernel, for the filter (the centres scaled alike) and for
    brute force; here against the isotropic C oracle on the scaled guide."""
    f, pg, sig, rng = _aniso_case(seed)
    ps = pg / sig
    cen_s, _, _, _ = oracle.cluster(ps, 5)
    g_iso, e_iso, _, nf = oracle.filter(f, ps, "gaussian", 2.0, 1.0, cen_s, r=6)
    g_an, e_an, _, nf2 = oracle.filter_aniso(f, pg, "gaussian", 2.0, sig, cen_s * sig, r=6)
    assert nf == nf2
    assert np.allclose(g_iso, g_an, rtol=0, atol=1e-8) and np.allclose(e_iso, e_an, rtol=1e-10, atol=1e-10)
    b_iso, _ = oracle.bruteforce(f, ps, "box", 0.0, 1.0, r=3, pix=np.arange(0, 24 * 30, 5))
    b_an, _ = oracle.bruteforce_aniso(f, pg, "box", 0.0, sig, r=3, pix=np.arange(0, 24 * 30, 5))
    assert np.allclose(b_iso, b_an, rtol=0, atol=1e-9)


def test_aniso_k_distinct_exactness_against_bruteforce():
    """P3 with the diagonal kernel: a guide with exactly K well-separated values and the centres equal
    to them gives b(i) = A e_s, c(i) = e_s, so the fast filter equals brute force (num)/(den)."""
    lab, pal, p = synth.gen_kdistinct(20, 22, 5, 4, seed=3, spread=255.0, min_sep=80.0)
    rng = np.random.default_rng(4)
    f = rng.uniform(0, 255, (20, 22, 3))
    sig = np.array([40.0, 60.0, 25.0, 90.0])
    g, _, _, _ = oracle.filter_aniso(f, p, "gaussian", 1.5, sig, pal, r=5, tau=0.0)
    gb, _ = oracle.bruteforce_aniso(f, p, "gaussian", 1.5, sig, r=5)
    assert np.allclose(g.reshape(-1, 3), gb, rtol=0, atol=1e-8)
