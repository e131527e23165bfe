import sys; sys.path.insert(0,'.')
import torch, synth, paper_1811_02363_b200 as hdf
cfg, f, p = synth.make("c2a")
pd = torch.from_numpy(p).cuda()
cen, lab, info = hdf.cluster(pd, cfg.K, labels=True)
torch.cuda.synchronize()
print("ok", info.status, info.splits_computed)
