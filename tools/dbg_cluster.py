import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle, paper_1811_02363_b200 as hdf
# warm the GPU up (clocks ramp from idle) before timing
_a = torch.randn(8192, 8192, device="cuda")
for _ in range(20):
    _a @ _a
torch.cuda.synchronize()
for name in sys.argv[1:]:
    cfg, f, p = synth.make(name)
    pd = torch.from_numpy(p).cuda()
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        cen, lab, info = hdf.cluster(pd, cfg.K, labels=True)
        dt = time.perf_counter() - t
    print(name, 'status', info.status, 'rounds', info.rounds, 'iters', info.lloyd_iters, 'E_K %.10e' % info.e_k,
          'wall %.3f ms' % (dt * 1e3), 'grid', info.launch_ctas, 'cl', info.cluster_ctas, 'plan %.1f seed %.1f pass %.1f (side %.1f sum %.1f red %.1f) fin %.1f part %.1f sync %.1f us' % (info.t_plan_us, info.t_seed_us, info.t_pass_us, info.t_pass_side_us, info.t_pass_sum_us, info.t_pass_red_us, info.t_lloyd_us, info.t_part_us, info.t_sync_us))
    tr = hdf.cluster_trace(pd, cfg.K)
    agg = {}
    prev = tr[0][1] if tr else 0
    for tag, t in tr:
        a = agg.setdefault(tag & 0xFFFF, [0, 0.0])
        a[0] += 1
        a[1] += (t - prev) / 1e3
        prev = t
    print("   trace: " + "  ".join("%d:n=%d,sum=%.1f,avg=%.2f" % (k, v[0], v[1], v[1] / v[0]) for k, v in sorted(agg.items())))
    c, l, s, ek = oracle.cluster(p, cfg.K)
    print('   oracle E_K %.10e' % ek, 'max centre diff', np.abs(cen.cpu().numpy() - c).max(), 'labels eq', (lab.cpu().numpy().reshape(-1) == l).mean())

