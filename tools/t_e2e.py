"""Per-stage times of one end-to-end call (hdf_filter_host, host buffers) at config 5 (sampled clustering)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1811_02363_b200 as hdf
import synth

cfg, f, p = synth.make("c5")
fh = torch.from_numpy(f).pin_memory()
gh = torch.empty_like(fh).pin_memory()
ws = hdf.Workspace()
kw = dict(kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, K=cfg.K, out=gh, ws=ws,
          cluster_stride=64)
for _ in range(3):
    hdf.filter_host(fh, fh, **kw)
torch.cuda.synchronize()
hdf.profile_collect()
hdf.profile_enable(True)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
hdf.filter_host(fh, fh, **kw)
e.record()
torch.cuda.synchronize()
pr = hdf.profile_collect()
hdf.profile_enable(False)
print(f"e2e step {s.elapsed_time(e):.3f} ms", {k: (round(v[0], 3), v[1]) for k, v in pr.items() if v[1]}, flush=True)
