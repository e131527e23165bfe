import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_1811_02363_b200 as hdf
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
H = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg, f, p = synth.make(name, H, H)
cen, lab, info = hdf.cluster(torch.from_numpy(p).cuda(), cfg.K, labels=True)
print('status', info.status, 'ach', info.achievable_k, 'rounds', info.rounds, 'iters', info.lloyd_iters, 'E_K', info.e_k)
import oracle
c, l, s, ek = oracle.cluster(p, cfg.K)
print('oracle E_K', ek, 'max centre diff', np.abs(cen.cpu().numpy() - c).max(), 'labels eq', (lab.cpu().numpy().reshape(-1) == l).mean())
