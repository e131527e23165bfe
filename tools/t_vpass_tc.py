"""Quick check of the tensor-core column pass against the CUDA-core one (same inputs, same centres)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1811_02363_b200 as hdf
import synth

for name, H, W in [("c1", None, None), ("c2b", None, None), ("c1", 61, 77), ("c2a", 200, 333)]:
    cfg, f, p = synth.make(name, H, W)
    fd = torch.from_numpy(f).cuda()
    cen, _, _ = hdf.cluster(fd, cfg.K)
    os.environ["HDF_VPASS_FMA"] = "0"
    a = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g
    torch.cuda.synchronize()
    os.environ["HDF_VPASS_FMA"] = "1"
    b = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g
    torch.cuda.synchronize()
    d = (a - b).abs()
    print(name, H, W, "max", d.max().item(), "mean", d.mean().item(), flush=True)
