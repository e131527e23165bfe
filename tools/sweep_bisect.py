"""Sweeps the clustering's worker-size knobs (HDF_BISECT_CTA_MAX, HDF_BISECT_QUAD_MAX) on the exact and
sampled clustering inputs: min of 7 timed runs per setting, E_K unchanged check."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1811_02363_b200 as hdf
import synth

inputs = {}
for name in sys.argv[1].split(","):
    base, _, stride = name.partition("s")
    cfg, f, p = synth.make(base)
    pd = torch.from_numpy(p).cuda()
    if stride:
        st = int(stride)
        M = (pd.numel() // cfg.rho + st - 1) // st
        pd = hdf.sample_guide(pd, 0, st, M).reshape(M, 1, cfg.rho)
    inputs[name] = (pd, cfg.K)
settings = [s.split(":") for s in sys.argv[2].split(",")]   # "cta:quad" pairs
for name, (pd, K) in inputs.items():
    ref = None
    for cta, quad in settings:
        os.environ["HDF_BISECT_CTA_MAX"] = cta
        os.environ["HDF_BISECT_QUAD_MAX"] = quad
        ts = []
        for _ in range(7):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            cen, _, info = hdf.cluster(pd, K)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ref = ref if ref is not None else info.e_k
        print(f"{name} cta_max {cta} quad_max {quad}: {min(ts):.3f} ms  E_K rel diff {abs(info.e_k - ref) / ref:.1e} "
              f"splits {info.splits_computed}", flush=True)
