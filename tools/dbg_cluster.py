"""Clustering diagnostics on the GPU: python tools/dbg_cluster.py c1 c2b c5s64 ...
Times hdf.cluster, compares with the oracle, and summarises the worker trace (per-node split spans)."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1811_02363_b200 as hdf
_a = torch.randn(8192, 8192, device="cuda")       # warm the clocks up
for _ in range(20):
    _a @ _a
torch.cuda.synchronize()
for name in sys.argv[1:]:
    # "c5s64": the sampled mode's input, the stride-64 sample of config 5 (R18)
    base, _, stride = name.partition("s")
    cfg, f, p = synth.make(base)
    pd = torch.from_numpy(p).cuda()
    if stride:
        st = int(stride)
        M = (pd.numel() // cfg.rho + st - 1) // st
        pd = hdf.sample_guide(pd, 0, st, M).reshape(M, 1, cfg.rho)
        p = pd.cpu().numpy()
    os.environ["HDF_BISECT_TRACE"] = "0"
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
    os.environ["HDF_BISECT_TRACE"] = "1"
    hdf.cluster(pd, cfg.K, labels=True)
    os.environ["HDF_BISECT_TRACE"] = "0"
    tr = hdf.cluster_trace(pd, cfg.K)
    if tr:
        t0 = min(t for _, t in tr)
        last = max(t for _, t in tr)
        print(f"   trace: {len(tr)} events, span {(last - t0) / 1e3:.1f} us")
        marks = {30: "start", 31: "root ready", 32: "cluster phase", 33: "CTA phase", 34: "finalise", 35: "done"}
        print("   timeline: " + "  ".join(f"{marks[w & 0xFF]} {(t - t0) / 1e3:.1f}" for w, t in sorted(tr, key=lambda x: x[1])
                                         if (w & 0xFF) in marks))
        # per worker, events in time order; a split = tag 2 .. tag 5 of one node
        byw = {}
        for w, t in sorted(tr, key=lambda x: x[1]):
            byw.setdefault(w >> 28, []).append((w & 0xFF, (w >> 8) & 0xFFFFF, (t - t0) / 1e3))
        names = {1: "claim", 2: "start", 7: "sample", 14: "R", 15: "L", 16: "O", 8: "rows", 9: "sync", 10: "argmax", 3: "seeds", 4: "lloyd",
                 11: "sse", 12: "part", 13: "ssex", 5: "publ"}
        rows = []
        for wk, evs in byw.items():
            cur = None
            for tag, node, t in evs:
                if tag == 2:
                    cur = {"w": wk, "node": node, "t": {2: t}, "it": 0}
                    rows.append(cur)
                elif tag == 6 and cur is not None:
                    cur["it"] = node
                elif 20 <= tag < 24 and cur is not None:
                    cur.setdefault("ph", [0, 0, 0, 0])[tag - 20] = node / 10.0
                elif cur is not None and tag in names:
                    cur["t"][tag] = t
        # critical path: parent links from the tag-17 events, chain ending at the last publication
        parent = {}
        for w, t in tr:
            if (w & 0xFF) == 17:
                c, pnode = (w >> 8) & 0xFFFFF, (w >> 28) & 0xFFF
                parent[c] = pnode
                parent[c + 1] = pnode
        byn = {r["node"]: r for r in rows if 5 in r["t"]}
        if byn:
            last = max(byn.values(), key=lambda r: r["t"][5])
            chain, v = [], last["node"]
            while v in byn:
                chain.append(byn[v])
                v = parent.get(v, -1)
            chain.reverse()
            tot_l = sum(r["t"].get(4, 0) - r["t"].get(3, 0) for r in chain)
            tot_s = sum(r["t"][5] - r["t"][2] for r in chain)
            gaps = sum(b["t"][2] - a["t"][5] for a, b in zip(chain, chain[1:]))
            print(f"   critical chain: {len(chain)} splits, {tot_s:.1f} us in splits ({tot_l:.1f} Lloyd, "
                  f"{sum(r['it'] for r in chain)} iterations), {gaps:.1f} us waiting between them; nodes "
                  + " ".join(str(r["node"]) for r in chain))
            for a, b in zip(chain, chain[1:]):
                t0, t1 = a["t"][5], b["t"][2]
                if t1 - t0 < 3:
                    continue
                busy = [f"w{r['w']}:n{r['node']}[{r['t'][2]:.0f}-{r['t'].get(5, 0):.0f}]" for r in rows
                        if r["t"][2] < t1 and r["t"].get(5, 1e9) > t0]
                print(f"     gap {t1 - t0:5.1f} us before node {b['node']} (ready {t0:.1f}): " + " ".join(busy))
        for rw in sorted(rows, key=lambda r: r["t"][2]):
            tt = rw["t"]
            seq = [2, 7, 14, 15, 16, 8, 9, 10, 3, 4, 11, 12, 13, 5]
            parts = []
            prev = tt[2]
            for tag in seq[1:]:
                if tag in tt:
                    parts.append(f"{names[tag]}+{tt[tag] - prev:.1f}")
                    prev = tt[tag]
            ph = rw.get("ph")
            phs = f" [pass {ph[0]:.1f} red {ph[1]:.1f} xchg {ph[2]:.1f} upd {ph[3]:.1f}]" if ph else ""
            print(f"     node {rw['node']:4d} w{rw['w']:4d} it {rw['it']:2d} @{tt[2]:7.1f} " + " ".join(parts) + phs)
    c, l, s, ek = oracle.cluster(p, cfg.K)
    print('   oracle E_K %.10e' % ek, 'max centre diff', np.abs(cen.cpu().numpy() - c).max(),
          'labels eq', (lab.cpu().numpy().reshape(-1) == l).mean(), flush=True)
