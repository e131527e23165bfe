"""Row strips: one image filtered by several ranks.

The filter is local in space: output row y depends on input rows [y - R, y + R] only (the separable
window, clipped to the image, R8) and on the centres (and A^+, from the centres).  So rank r of
`world` filters its strip of output rows [y0, y1) from the input rows [max(0, y0 - R), min(H, y1 + R))
with the same centres, and keeps rows [y0, y1): the result is the single-GPU result row for row
(the image borders stay where they are; a strip border is never treated as one).

The clustering needs the whole guide, so rank 0 clusters it and broadcasts the K x rho centres: the
only collective on the data path (a few hundred bytes).  Host-side orchestration only: every step of
the filter runs in the CUDA path through the C ABI (`filter`), or in the function passed as `filt`.
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


def filter_strips(f, p=None, *, kind: str = "gaussian", sigma_s: float = 1.0, radius: int = -1,
                  sigma_r: float = 1.0, K: int = 16, tau: float = 0.5, centres=None, gather: bool = True,
                  dist=None, filt=None, cluster=None):
    """Filter the image f [H, W, n] (guide p, None: bilateral) split in row strips over the ranks of
    `dist` (torch.distributed, initialised; None: one rank).  Every rank passes the whole image (only
    its strip and halo are read).  Returns the full result on every rank (gather=True, all_gather) or
    this rank's strip rows.

    filt(f_strip, p_strip, centres) -> g_strip and cluster(p) -> centres default to the library's
    CUDA path (`paper_1811_02363_b200.filter` / `.cluster`); tests inject the CPU oracle."""
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
