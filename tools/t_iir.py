"""IIR precision vs sigma on the GPU (diagnostic): max / mean |dg| against oracle.filter_iir."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth, paper_1811_02363_b200 as hdf
for s, H, W in [(3.0, 130, 260), (8.0, 130, 260), (12.0, 130, 260), (16.0, 130, 260), (24.0, 130, 260)]:
    cfg, f, p = synth.make("c1", H, W)
    mu = oracle.cluster(p, 8)[0].astype(np.float32)
    g_o, eta, fl, nf = oracle.filter_iir(f, p, s, cfg.sigma_r, mu)
    fd = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).cuda()
    r = hdf.filter(fd, fd, kind="gaussian_iir", sigma_s=s, sigma_r=cfg.sigma_r, centres=torch.from_numpy(mu).cuda(),
                   count_flagged=True)
    d = np.abs(r.g.cpu().numpy() - g_o)
    i = np.unravel_index(np.argmax(d), d.shape)
    print(f"sigma {s}: max {d.max():.3e} mean {d.mean():.3e} flagged gpu {r.n_flagged} oracle {nf} at {i} eta {eta[i[:2]]:.3e}")
