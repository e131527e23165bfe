"""Clustering diagnostics on the GPU: python tools/dbg_cluster.py c1 c2b ...
Times hdf.cluster, compares with the oracle, and summarises the worker trace (per-node split spans)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1811_02363_b200 as hdf
_a = torch.randn(8192, 8192, device="cuda")       # warm the clocks up
for _ in range(20):
    _a @ _a
torch.cuda.synchronize()
for name in sys.argv[1:]:
    cfg, f, p = synth.make(name)
    pd = torch.from_numpy(p).cuda()
    ts = []
    for rep in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        cen, lab, info = hdf.cluster(pd, cfg.K, labels=True)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"{name}: K={cfg.K} status {info.status} splits {info.splits_computed} (grid {info.grid_splits}) "
          f"iters {info.lloyd_iters} E_K {info.e_k:.10e} ms {min(ts):.3f} (reps {' '.join('%.3f' % t for t in ts)}) "
          f"grid {info.launch_ctas} cl {info.cluster_ctas} tile {info.tile_points}")
    tr = hdf.cluster_trace(pd, cfg.K)
    if tr:
        t0 = min(t for _, t in tr)
        spans = {}
        for w, t in tr:
            tag, node, worker = w & 0xFF, (w >> 8) & 0xFFFFF, w >> 28
            if tag in (2, 3, 4, 5):
                spans.setdefault(node, {})[tag] = (t - t0) / 1e3
                spans[node]["w"] = worker
        last = max(t for _, t in tr)
        print(f"   trace: {len(tr)} events, span {(last - t0) / 1e3:.1f} us")
        for node in sorted(spans, key=lambda n: spans[n].get(2, 0)):
            s = spans[node]
            print(f"     node {node:4d} w{s['w']:3d} start {s.get(2, -1):8.1f} seeds +{s.get(3, 0) - s.get(2, 0):6.1f} "
                  f"lloyd +{s.get(4, 0) - s.get(3, 0):6.1f} part +{s.get(5, 0) - s.get(4, 0):6.1f} end {s.get(5, -1):8.1f}")
    c, l, s, ek = oracle.cluster(p, cfg.K)
    print('   oracle E_K %.10e' % ek, 'max centre diff', np.abs(cen.cpu().numpy() - c).max(),
          'labels eq', (lab.cpu().numpy().reshape(-1) == l).mean(), flush=True)
