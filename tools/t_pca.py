"""Times the on-GPU PCA-NLM guide (hdf_pca_guide) at config 4's size and checks it against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1811_02363_b200 as hdf
import synth

noisy, _, _ = synth.gen_nlm(512, 512, 4)
fd = torch.from_numpy(noisy).cuda()
for _ in range(3):
    p, B = hdf.pca_guide(fd, 3, 6, basis=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    p, B = hdf.pca_guide(fd, 3, 6, basis=True)
e.record()
torch.cuda.synchronize()
print(f"pca_guide 512x512x3 m=3 dim=6: {s.elapsed_time(e) / 10:.3f} ms", flush=True)
if "--check" in sys.argv:
    po = oracle.pca_guide(noisy, 3, 6)
    po = po[0] if isinstance(po, tuple) else po
    print("max |p - oracle| =", float(np.abs(p.cpu().numpy() - po).max()), flush=True)
