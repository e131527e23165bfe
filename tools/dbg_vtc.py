import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1811_02363_b200 as hdf, synth
cfg, f, p = synth.make("c2b")
fd = torch.from_numpy(f).cuda()
cen, _, _ = hdf.cluster(fd, cfg.K)
os.environ["HDF_VPASS_FMA"] = "0"
a = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g.cpu().numpy()
os.environ["HDF_VPASS_FMA"] = "1"
b = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g.cpu().numpy()
d = np.abs(a - b).max(-1)
rows = d.max(1); cols = d.max(0)
print("bad rows", np.nonzero(rows > 1e-3)[0][:40], len(np.nonzero(rows > 1e-3)[0]))
print("bad cols", np.nonzero(cols > 1e-3)[0][:40], len(np.nonzero(cols > 1e-3)[0]))
