import sys; sys.path.insert(0,'.')
import torch, synth, paper_1811_02363_b200 as hdf
name = sys.argv[1] if len(sys.argv) > 1 else "c2b"
cfg, f, p = synth.make(name)
pd = torch.from_numpy(p).cuda()
try:
    cen, lab, info = hdf.cluster(pd, cfg.K, labels=True)
    torch.cuda.synchronize()
    print("cluster ok", info.status, info.splits_computed, info.grid_splits)
except Exception as e:
    print("cluster error", e)
fd = torch.from_numpy(f).cuda()
try:
    r = hdf.filter(fd, pd if not cfg.bilateral else None, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, K=cfg.K)
    torch.cuda.synchronize()
    print("filter ok")
except Exception as e:
    print("filter error", e)
