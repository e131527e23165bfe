import sys; sys.path.insert(0,'.')
import torch, synth, paper_1811_02363_b200 as hdf
cfg, f, p = synth.make("c4")
fd = torch.from_numpy(f).cuda()
for _ in range(3): hdf.pca_guide(fd, 3, 6)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); hdf.pca_guide(fd, 3, 6); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("pca_guide c4 ms: min %.4f median %.4f" % (min(ts), sorted(ts)[5]))
