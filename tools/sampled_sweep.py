"""Sampled clustering mode (hdf_cluster_sampled): time and R15 quality per stride, on the GPU.

    python tools/sampled_sweep.py c5 1 4 16 64

For each stride: the clustering time (CUDA events, median of 5 after 2 warm-ups) and the MSE against
brute force on a seeded 2^16-pixel sample (all pixels when the image is smaller), relative to the exact
oracle pipeline's MSE (R15 asks for <= 1.05)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1811_02363_b200 as hdf
import synth

name = sys.argv[1]
strides = [int(s) for s in sys.argv[2:]] or [1, 4, 16]
cfg, f, p = synth.make(name)
H, W = cfg.H, cfg.W
pd = torch.from_numpy(p).cuda()
fd = pd if cfg.bilateral else torch.from_numpy(f).cuda()
rng = np.random.default_rng(5 << 16)
pix = np.sort(rng.choice(H * W, min(1 << 16, H * W), replace=False))
g_bf, _ = oracle.bruteforce(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, r=cfg.radius, pix=pix)
cen_o, _, _, ek_o = oracle.cluster(p, cfg.K)
g_o, _, _ = oracle.filter_pixels(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, cen_o, pix, r=cfg.radius)
mse_o = oracle.mse(g_o, g_bf, cfg.R_range)
ws = hdf.Workspace()
for s in strides:
    for _ in range(2):
        hdf.cluster_sampled(pd, cfg.K, s, info=False, ws=ws)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        hdf.cluster_sampled(pd, cfg.K, s, info=False, ws=ws)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    cen, info = hdf.cluster_sampled(pd, cfg.K, s, ws=ws)
    g = hdf.filter(fd, pd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r,
                   centres=cen).g.cpu().numpy().reshape(-1, cfg.n)[pix]
    mse_g = oracle.mse(g, g_bf, cfg.R_range)
    print(json.dumps({"config": name, "stride": s, "sample": (H * W + s - 1) // s, "cluster_ms": round(float(np.median(ts)), 4),
                      "mse_ratio": round(mse_g / mse_o, 5), "e_k_sample": info.e_k, "e_k_oracle_full": ek_o}), flush=True)
