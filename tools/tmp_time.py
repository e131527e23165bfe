import os, sys, shutil
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
var = sys.argv[1]
if var != "base":
    shutil.copy(os.path.join(ROOT, "tools", "tmp_" + var, "libhdf.so"), os.path.join(ROOT, "paper_1811_02363_b200", "libhdf.so"))
import torch, paper_1811_02363_b200 as hdf, synth
cfg, f, p = synth.make("c5")
fd = torch.from_numpy(f).cuda()
cen, _, _ = hdf.cluster(fd, cfg.K)
for _ in range(2):
    hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen)
torch.cuda.synchronize()
hdf.profile_collect(); hdf.profile_enable(True)
for _ in range(5):
    hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen)
pr = hdf.profile_collect()
print(var, {k: round(v[0] / max(v[1], 1), 3) for k, v in pr.items() if v[1]}, flush=True)
a = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g.clone()
os.environ["HDF_VPASS_FMA"] = "1"
b = hdf.filter(fd, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, centres=cen).g
os.environ["HDF_VPASS_FMA"] = "0"
print("   max |tc - fma| =", (a - b).abs().max().item(), flush=True)
