"""Multi-process host logic on CPU (gloo, world_size 2): the row-strip decomposition (NEXT #4,
paper_1811_02363_b200/strips.py) with the oracle standing in for the per-strip filter, and the
weak-scaling bench's max-over-ranks reduction.  No GPU."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out):
    import torch.distributed as dist

    from paper_1811_02363_b200 import strips
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, f, p = synth.make(name, 45, 38)
    R = strips.radius_of(cfg.kind, cfg.sigma_s, cfg.radius)

    def filt(fs, ps, cen):
        g, _, _, _ = oracle.filter(fs.numpy(), ps.numpy(), cfg.kind, cfg.sigma_s, cfg.sigma_r,
                                   cen.numpy().astype(np.float64), r=R, tau=0.5)
        return torch.from_numpy(g)

    def clus(pp):
        return torch.from_numpy(oracle.cluster(pp.numpy(), cfg.K)[0].astype(np.float32))

    ft = torch.from_numpy(f)
    pt = None if cfg.bilateral else torch.from_numpy(p)
    g = strips.filter_strips(ft, pt, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r,
                             K=cfg.K, dist=dist, filt=filt, cluster=clus)
    # weak-scaling bench: the step time is the max over ranks
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(out, g.numpy())
        np.save(out + ".t.npy", t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_row_strips_reproduce_the_whole_image(tmp_path, name):
    """Two ranks, each its strip plus an R-row halo, centres broadcast from rank 0: the gathered
    result equals the whole-image oracle filter with the same centres (window clipped only at the
    true image borders, R8)."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    g = np.load(out)
    cfg, f, p = synth.make(name, 45, 38)
    cen = oracle.cluster(p, cfg.K)[0].astype(np.float32).astype(np.float64)
    ref, _, _, _ = oracle.filter(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, cen, r=cfg.radius, tau=0.5)
    assert g.shape == ref.shape
    assert np.allclose(g, ref, rtol=0, atol=1e-9)
    assert float(np.load(out + ".t.npy")[0]) == 2.0


def _worker_sampled(rank, world, port, name, s, out):
    import torch.distributed as dist

    from paper_1811_02363_b200 import strips
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, f, p = synth.make(name, 45, 38)
    R = strips.radius_of(cfg.kind, cfg.sigma_s, cfg.radius)
    seen = {}

    def filt(fs, ps, cen):
        g, _, _, _ = oracle.filter(fs.numpy(), ps.numpy(), cfg.kind, cfg.sigma_s, cfg.sigma_r,
                                   cen.numpy().astype(np.float64), r=R, tau=0.5)
        return torch.from_numpy(g)

    def clus(pp):
        seen["sample"] = pp.numpy().copy()
        return torch.from_numpy(oracle.cluster(pp.numpy(), cfg.K)[0].astype(np.float32))

    def sample(pp, i0, st, M):       # the gather (data movement only)
        return pp.reshape(-1, pp.shape[-1])[i0::st][:M].clone()

    ft = torch.from_numpy(f)
    pt = None if cfg.bilateral else torch.from_numpy(p)
    g = strips.filter_strips(ft, pt, kind=cfg.kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r,
                             K=cfg.K, dist=dist, filt=filt, cluster=clus, cluster_stride=s, sample=sample)
    np.save(out + f".smp{rank}.npy", seen["sample"])
    if rank == 0:
        np.save(out, g.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,s", [("c1", 2, 3), ("c4", 3, 7), ("c1", 2, 1)])
def test_sharded_sampled_clustering(tmp_path, name, world, s):
    """the clustering split over the ranks.  Each rank gathers its rows' share of the
    global stride sample p.flat[0::s], one all_gather assembles it, every rank clusters it: every rank
    sees exactly the single-process sample (s = 1: the whole guide, the exact procedure), and the
    stitched result equals the whole-image oracle filter with the oracle's centres of that sample."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker_sampled, args=(world, _free_port(), name, s, out), nprocs=world, join=True)
    cfg, f, p = synth.make(name, 45, 38)
    want = p.reshape(-1, p.shape[-1])[0::s]
    for r in range(world):
        got = np.load(out + f".smp{r}.npy").reshape(-1, p.shape[-1])
        assert np.array_equal(got, want)
    cen = oracle.cluster(want, cfg.K)[0].astype(np.float32).astype(np.float64)
    ref, _, _, _ = oracle.filter(f, p, cfg.kind, cfg.sigma_s, cfg.sigma_r, cen, r=cfg.radius, tau=0.5)
    assert np.allclose(np.load(out), ref, rtol=0, atol=1e-9)


def test_sample_shares_partition_the_global_sample():
    from paper_1811_02363_b200 import strips
    for H, W, world, s in [(45, 38, 2, 3), (512, 512, 8, 16), (7, 5, 3, 4), (100, 3, 4, 1), (9, 9, 2, 100)]:
        idx = []
        for y0, y1, _, _ in strips.strip_bounds(H, world, 0):
            i0, M = strips.sample_share(H, W, y0, y1, s)
            idx += list(range(i0, i0 + M * s, s))
        assert idx == list(range(0, H * W, s))


def test_strip_bounds_cover_the_image():
    from paper_1811_02363_b200 import strips
    for H, world, R in [(512, 8, 15), (7, 3, 9), (100, 1, 24), (5, 5, 0)]:
        b = strips.strip_bounds(H, world, R)
        assert b[0][0] == 0 and b[-1][1] == H
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert all(h0 == max(0, y0 - R) and h1 == min(H, y1 + R) for y0, y1, h0, h1 in b)
