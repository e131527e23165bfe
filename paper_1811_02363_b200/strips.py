"""Row strips: one image filtered by several ranks.

The filter is local in space: output row y depends on input rows [y - R, y + R] only (the separable
window, clipped to the image, R8) and on the centres (and A^+, from the centres).  So rank r of
`world` filters its strip of output rows [y0, y1) from the input rows [max(0, y0 - R), min(H, y1 + R))
with the same centres, and keeps rows [y0, y1): the result is the single-GPU result row for row
(the image borders stay where they are; a strip border is never treated as one).

The clustering needs the whole guide.  Two ways:
* exact (cluster_stride None): rank 0 clusters the whole guide and broadcasts the K x rho centres,
  one collective of a few hundred bytes; the other ranks wait for rank 0's clustering;
* sharded sample (cluster_stride s): the sampled mode of hdf_cluster_sampled split over the
  ranks -- rank r gathers the members of the global stride sample p.flat[0::s] that lie in its own
  output rows (hdf_sample_guide), one all_gather assembles the whole sample in pixel order (rank
  order = row order), and every rank runs the same deterministic bisecting K-means on it, so all ranks
  hold identical centres with no further exchange: the result equals the single-GPU sampled mode.
Host-side orchestration only: every step runs in the CUDA path through the C ABI (`filter`,
`cluster`, `sample_guide`), or in the functions passed as `filt` / `cluster` / `sample`.
"""
from __future__ import annotations

import math


def radius_of(kind: str, sigma_s: float, radius: int) -> int:
    """The window half-width the library uses (R7: ceil(3 sigma_s) for the Gaussian by default)."""
    if radius >= 0:
        return int(radius)
    if kind == "box":
        raise ValueError("the box kernel needs an explicit radius")
    return int(math.ceil(3.0 * sigma_s))


def strip_bounds(H: int, world: int, R: int):
    """[(y0, y1, h0, h1)] per rank: output rows [y0, y1) (balanced), input rows [h0, h1) with the halo."""
    out = []
    for r in range(world):
        y0, y1 = H * r // world, H * (r + 1) // world
        out.append((y0, y1, max(0, y0 - R), min(H, y1 + R)))
    return out


def sample_share(H: int, W: int, y0: int, y1: int, s: int):
    """(i0, M): the members i0, i0 + s, ... (M of them) of the global stride sample {0, s, 2s, ...} of
    the H*W pixels that lie in rows [y0, y1)."""
    a, b = y0 * W, y1 * W
    i0 = -(-a // s) * s
    M = 0 if i0 >= b else (b - 1 - i0) // s + 1
    return i0, M


def sharded_sample(p, s: int, dist=None, sample=None):
    """The global stride sample p.flat[0::s] ([M, rho], pixel order) assembled from every rank's share of
    its own row strip (balanced strips of strip_bounds) with one all_gather."""
    import torch

    rank = dist.get_rank() if dist is not None else 0
    world = dist.get_world_size() if dist is not None else 1
    H, W = p.shape[0], p.shape[1]
    rho = p.shape[2] if p.dim() == 3 else 1
    if sample is None:
        import paper_1811_02363_b200 as hdf
        sample = hdf.sample_guide
    bounds = strip_bounds(H, world, 0)
    shares = [sample_share(H, W, b[0], b[1], s) for b in bounds]
    i0, M = shares[rank]
    mine = sample(p, i0, s, M)
    if dist is None or world == 1:
        return mine
    mmax = max(m for _, m in shares)
    pad = torch.zeros((mmax, rho), dtype=mine.dtype, device=mine.device)
    pad[:M] = mine
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][:shares[r][1]] for r in range(world)], 0)


def filter_strips(f, p=None, *, kind: str = "gaussian", sigma_s: float = 1.0, radius: int = -1,
                  sigma_r: float = 1.0, K: int = 16, tau: float = 0.5, centres=None, gather: bool = True,
                  dist=None, filt=None, cluster=None, cluster_stride: int | None = None, sample=None):
    """Filter the image f [H, W, n] (guide p, None: bilateral) split in row strips over the ranks of
    `dist` (torch.distributed, initialised; None: one rank).  Every rank passes the whole image (only
    its strip and halo are read).  Returns the full result on every rank (gather=True, all_gather) or
    this rank's strip rows.

    filt(f_strip, p_strip, centres) -> g_strip and cluster(p) -> centres default to the library's
    CUDA path (`paper_1811_02363_b200.filter` / `.cluster`); tests inject the CPU oracle.
    cluster_stride s: the sharded sampled clustering (module docstring); cluster then receives the
    assembled sample as a [1, M, rho] guide, and sample(p, i0, s, M) defaults to hdf.sample_guide."""
    import torch

    if p is None:
        p = f
    if kind == "gaussian_iir":
        # Young's recursion has infinite support: a strip filtered with zero extension at its own
        # edges differs from the whole image near the strip borders, so strips are not exact
        raise ValueError("row strips need a finite window (kind 'gaussian' or 'box'), not 'gaussian_iir'")
    rank = dist.get_rank() if dist is not None else 0
    world = dist.get_world_size() if dist is not None else 1
    H = f.shape[0]
    R = radius_of(kind, sigma_s, radius)
    if filt is None or cluster is None:
        import paper_1811_02363_b200 as hdf
        if cluster is None:
            def cluster(pp):
                return hdf.cluster(pp, K)[0]
        if filt is None:
            def filt(fs, ps, cen):
                return hdf.filter(fs, ps, kind=kind, sigma_s=sigma_s, radius=R, sigma_r=sigma_r, K=cen.shape[0],
                                  centres=cen, tau=tau).g
    if centres is None and cluster_stride is not None:
        # every rank clusters the same assembled sample: identical centres, no broadcast
        smp = sharded_sample(p, int(cluster_stride), dist, sample)
        centres = cluster(smp.reshape(1, smp.shape[0], smp.shape[1])).contiguous()
    # centres: rank 0 clusters the whole guide, one broadcast of K x rho floats
    if centres is None:
        if rank == 0:
            centres = cluster(p).contiguous()
        else:
            centres = torch.empty((K, p.shape[2]), dtype=torch.float32, device=p.device)
        if dist is not None:
            dist.broadcast(centres, src=0)
    y0, y1, h0, h1 = strip_bounds(H, world, R)[rank]
    fs = f[h0:h1].contiguous()
    ps = fs if p is f else p[h0:h1].contiguous()
    g = filt(fs, ps, centres)[y0 - h0:y1 - h0].contiguous()
    if not gather or dist is None:
        return g
    # all_gather of unequal strips: pad to the largest strip
    hmax = max(b[1] - b[0] for b in strip_bounds(H, world, R))
    pad = torch.zeros((hmax,) + tuple(g.shape[1:]), dtype=g.dtype, device=g.device)
    pad[: g.shape[0]] = g
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: b[1] - b[0]] for r, b in enumerate(strip_bounds(H, world, R))], dim=0)
