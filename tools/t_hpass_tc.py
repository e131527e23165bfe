"""Quick check of the tensor-core row pass (k_hpass_combine_tc) against the CUDA-core one (same inputs, same
centres), plus the stage times at config 5."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1811_02363_b200 as hdf
import synth


def run(name, H=None, W=None, timing=False):
    cfg, f, p = synth.make(name, H, W)
    fd = torch.from_numpy(f).cuda()
    cen, _, _ = hdf.cluster(fd, cfg.K)
    out = {}
    for mode in ("0", "1"):
        os.environ["HDF_HPASS_FMA"] = mode
        r = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen,
                       tau=0.5, count_flagged=True)
        torch.cuda.synchronize()
        out[mode] = r
        if timing:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen)
            hdf.profile_collect()
            hdf.profile_enable(True)
            s.record()
            for _ in range(5):
                hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen)
            e.record()
            torch.cuda.synchronize()
            pr = hdf.profile_collect()
            hdf.profile_enable(False)
            print(f"  HDF_HPASS_FMA={mode}: filter {s.elapsed_time(e) / 5:.3f} ms", flush=True)
            print("   ", {k: round(v[0] / max(v[1], 1), 3) for k, v in pr.items()}, flush=True)
    d = (out["0"].g - out["1"].g).abs()
    print(name, H, W, "max", d.max().item(), "mean", d.mean().item(), "flagged", out["0"].n_flagged,
          out["1"].n_flagged, flush=True)


for name, H, W in [("c1", None, None), ("c2b", None, None), ("c1", 61, 76), ("c2a", 200, 332), ("c2a", 33, 100)]:
    run(name, H, W)
run("c5", None, None, timing=True)
