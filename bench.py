#!/usr/bin/env python
"""Benchmark of the hot path (cluster + pinv + K(n+1) convolutions + combine) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One step = one pass of the whole hot path (S1 cluster, S2 pinv, S3-S6
filter) over one synthetic image resident in HBM, through the C ABI (hdf_filter with centres=NULL
clusters inside the call).  Default workload = BASELINE.json configs[4] ("c5": 4096x4096x3 colour
bilateral, sigma_s=8 (R=24), sigma_r=40, K=64), the largest single-GPU configuration (BASELINE's
metric names no config).  L2 is flushed (a 512 MiB write) between timed steps, outside the timed
events; value = pixels / the MEDIAN step time.

Multi-GPU (torchrun, one process per GPU): the path partitions into independent images; every
rank filters its own seeded image with no collective on the data path ("scaling": "weak"); the
step time is the max over ranks.

Rank 0 prints ONE JSON line.  --impl reference times the fp64 CPU oracle (test infrastructure,
oracle/) on the host cores instead; --all prints one line per config (exploration only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "Mpixel/s per filter (cluster+convolve+combine)"
UNIT = "Mpixel/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------------------------ clocks ----
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, samples = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                s, mx = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            samples += 1
            smax = mx
            sm.append(s)
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": samples}


# ---------------------------------------------------------------------------- algorithmic work ----
def stage_work(cfg, K: int, H: int, W: int, iir: bool = False):
    """Algorithmic bytes and FP32 FMA-pipe ops per launch of each filter kernel.
    bytes: what the minimal version of the kernel must move (planes written once, read once; the
    coefficient planes c are a design choice of this build and are not counted)."""
    n, rho, R = cfg.n, cfg.rho, cfg.radius
    npx = H * W
    n_in = n if cfg.bilateral else n + rho
    planes = K * (n + 1)
    taps = 2 * R + 1
    if iir:   # NEXT #1: identity passes; the "vpass" stage adds the column and row recursions, each
        #       reading and writing every plane twice (causal, then anti-causal), 4 FMAs per sample
        return {
            "vpass": {"bytes": 4 * npx * (n_in + 9 * planes), "fma": npx * (planes * 16 + K * (rho + 1 + n))},
            "hpass": {"bytes": 4 * npx * (planes + n), "fma": npx * (2 * planes + n)},
            "coeffs": {"bytes": 4 * npx * rho, "fma": npx * (K * K + K * (rho + 1)), "mma_flop": 2 * npx * K * K},
            "filter": {"bytes": 4 * npx * (n_in + 10 * planes + n)},
        }
    return {
        "vpass": {"bytes": 4 * npx * (n_in + planes), "fma": npx * (planes * taps + K * (rho + 1 + n))},
        "hpass": {"bytes": 4 * npx * (planes + n),
                  "fma": npx * (planes * (taps if cfg.kind == "gaussian" else 4) + planes + n)},
        "coeffs": {"bytes": 4 * npx * rho, "fma": npx * (K * K + K * (rho + 1)), "mma_flop": 2 * npx * K * K},
        "filter": {"bytes": 4 * npx * (n_in + 2 * planes + n)},        # SURVEY 8(d) B_req
    }


# The sampled clustering mode's stride per workload (P:329 'any efficient clustering'), chosen from the
# measured sweeps (profiles/r02b_sampled_sweep.jsonl, profiles/r02t_sampled_sweep_c3.jsonl) and held to
# R15's 5% rule by tests/test_gpu_cluster.py (c5: 1.008 x the exact oracle pipeline's MSE on 2^16
# brute-force pixels; c3 at stride 16: 0.95, 1.11 ms against 1.56 ms at stride 4 once the stride sample
# of a rho = 31 node is staged in shared memory).  The NLM config c4 fails R15 at every stride tried
# (1.22 / 1.41 / 1.15), so it and the small images (where the clustering is latency-bound, not
# size-bound) cluster every pixel.
SAMPLED_STRIDE = {"c5": 64, "c3": 16}


def tc_passes(cfg, H: int, W: int, nsm: int, variant: str = "soft"):
    """Which filter passes run on the tensor cores for this workload (the library's own rule, hdf_api.cu:
    colour Gaussian FIR with f = p, 4 <= R <= 24, W % 4 == 0; the row pass when its (32-row, 128-column)
    units fill the SMs; HDF_VPASS_FMA / HDF_HPASS_FMA override)."""
    vtc = (cfg.kind == "gaussian" and variant != "iir" and cfg.bilateral and cfg.n == 3 and cfg.rho == 3
           and 4 <= cfg.radius <= 24 and W % 4 == 0 and os.environ.get("HDF_VPASS_FMA", "0") in ("", "0"))
    env = os.environ.get("HDF_HPASS_FMA", "")
    htc = vtc and (env == "0" if env else ((H + 31) // 32) * ((W + 127) // 128) >= nsm)
    return vtc, htc


def fma_peak(sm_mhz: float, nsm: int = 148) -> float:
    """FP32 FMA-pipe roof = SMs x 128 lanes x clock."""
    return nsm * 128 * sm_mhz * 1e6


# ------------------------------------------------------------------------------------ our arm ----
def run_ours(args, rank: int, world: int, dist):
    import torch

    import paper_1811_02363_b200 as hdf
    import synth

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg, f, p = synth.make(args.config)
    if world > 1 and rank > 0:       # independent image per rank (weak scaling)
        cfg2, f, p = _rank_image(args.config, rank)
    H, W = f.shape[:2]
    K = cfg.K
    fd = torch.from_numpy(f).to(dev)
    pd = fd if cfg.bilateral else torch.from_numpy(p).to(dev)
    ws = hdf.Workspace()
    g = torch.empty_like(fd)
    kind = "gaussian_iir" if args.variant == "iir" else cfg.kind
    if args.variant == "iir" and cfg.kind != "gaussian":
        raise SystemExit("--variant iir needs a Gaussian config")
    kw = dict(kind=kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r, K=K, tau=0.5,
              out=g, ws=ws)

    if args.strips and world > 1:   # one image over the ranks in row strips (NEXT #4; strong scaling)
        from paper_1811_02363_b200 import strips as _strips
        fd = torch.from_numpy(synth.make(args.config)[1]).to(dev)
        pd = fd if cfg.bilateral else torch.from_numpy(synth.make(args.config)[2]).to(dev)
        H, W = fd.shape[:2]

        def step():
            _strips.filter_strips(fd, None if cfg.bilateral else pd, kind=cfg.kind, sigma_s=cfg.sigma_s,
                                  radius=cfg.radius, sigma_r=cfg.sigma_r, K=K, tau=0.5, gather=False, dist=dist,
                                  cluster_stride=args.cluster_stride if args.cluster_stride > 1 else None)
    elif args.variant == "hard":     # hard-assignment variant: one-hot coefficients, no A^+
        kwh = {k: v for k, v in kw.items() if k != "tau"}

        def step():
            hdf.filter_hard(fd, None if cfg.bilateral else pd, **kwh)
    elif args.cluster_stride > 1:    # the sampled clustering mode, then the filter
        cws = hdf.Workspace()
        kwc = dict(kw)
        kwc.pop("K")

        def step():
            cen, _ = hdf.cluster_sampled(pd, K, args.cluster_stride, info=False, ws=cws)
            hdf.filter(fd, pd, centres=cen, **kwc)
    else:
        def step():
            hdf.filter(fd, pd, **kw)        # centres=None: clustering runs inside the call

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    # the write-only HBM bandwidth of this device (a 4 GiB fill, best of 5): the column pass and the
    # coefficient kernel only write, and HBM3e writes run well below the copy figure (context for their
    # roofline lines; the contract's peak stays the measured copy bandwidth)
    wbuf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    wbest = 1e30
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        wbuf.fill_(3)
        b.record(stream)
        b.synchronize()
        wbest = min(wbest, a.elapsed_time(b))
    write_peak = wbuf.numel() / (wbest * 1e-3) / 1e9
    # and the read-only bandwidth (a float sum over the same 4 GiB, best of 6): the row pass only reads
    rf = wbuf.view(torch.float32)
    rbest = 1e30
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rf.sum()
        b.record(stream)
        b.synchronize()
        rbest = min(rbest, a.elapsed_time(b))
    read_peak = wbuf.numel() / (rbest * 1e-3) / 1e9
    del wbuf, rf

    # ---- timed region: K steps, events around each step, L2 flushed between steps ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    hdf.profile_collect()
    hdf.profile_enable(True)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    hdf.profile_enable(False)
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    prof = hdf.profile_collect()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = statistics.median(step_ms)
    if dist is not None:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    ms_step = t_ms                              # median step (max over ranks)
    value = (1 if (args.strips and world > 1) else world) * H * W / (ms_step * 1e-3) / 1e6

    # ---- the same step with the exact clustering of every pixel, when the headline uses the sampled
    #      mode: timed the same way (K steps, L2 flushed, median, max over ranks), reported beside it ----
    exact = None
    if args.cluster_stride > 1 and not args.strips and args.variant == "soft":
        def step_exact():
            hdf.filter(fd, pd, **kw)
        for _ in range(args.warmup):
            flush.fill_(1)
            step_exact()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev2[i][0].record(stream)
            step_exact()
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        t2 = statistics.median([a.elapsed_time(b) for a, b in ev2])
        if dist is not None:
            t = torch.tensor([t2], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t2 = float(t.item())
        exact = {"value": round(world * H * W / (t2 * 1e-3) / 1e6, 3), "unit": UNIT, "ms_per_step": round(t2, 4),
                 "cluster": "exact bisecting K-means of every pixel (hdf_filter with centres=NULL)"}

    # ---- end to end through the public host API: H2D + cluster + filter + D2H each step ----
    fh = torch.from_numpy(f).pin_memory()
    ph = fh if cfg.bilateral else torch.from_numpy(p).pin_memory()
    gh = torch.empty_like(fh).pin_memory()
    ws2 = hdf.Workspace()
    for _ in range(max(1, args.warmup)):
        hdf.filter_host(fh, ph, kind=kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r,
                        K=K, out=gh, ws=ws2, cluster_stride=args.cluster_stride)
    e2e_ms = []
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        host_res = hdf.filter_host(fh, ph, kind=kind, sigma_s=cfg.sigma_s, radius=cfg.radius, sigma_r=cfg.sigma_r,
                                   K=K, out=gh, ws=ws2, cluster_stride=args.cluster_stride)
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_t = statistics.median(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = world * H * W / (e2e_t * 1e-3) / 1e6
    h2d = fh.numel() * 4 + (0 if cfg.bilateral else ph.numel() * 4)
    d2h = gh.numel() * 4 + K * cfg.rho * 4 + 8

    # ---- roofline of the dominant kernel (live event timings above) ----
    peaks = _peaks()
    work = stage_work(cfg, K, H, W, iir=(args.variant == "iir"))
    kern = {k: v for k, v in prof.items() if k in ("cluster", "pinv", "coeffs", "vpass", "hpass", "fallback")}
    per_launch = {k: (ms / n if n else 0.0) for k, (ms, n) in kern.items()}
    # per step: a kernel launched once per row band of the pipelined filter (HDF_PIPE_BANDS) sums its bands
    per_step = {k: ms / args.steps for k, (ms, n) in kern.items()}
    bands = max(1, kern.get("vpass", (0, 0))[1] // max(1, args.steps))
    sm_mhz = clk.get("sm_mhz") or peaks.get("clocks_under_load", {}).get("sm_mhz_median", 1965.0)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)

    # dram bytes per launch from the committed ncu --set full capture of this workload (profiles/), if any
    vtc, htc = tc_passes(cfg, H, W, nsm, args.variant)
    kname = {"vpass": "k_range_vpass_tc" if vtc else "k_range_vpass",
             "hpass": "k_hpass_combine_tc" if htc else "k_hpass_combine", "coeffs": "k_coeffs_tc"}
    # the FIR passes on the tensor cores (banded Toeplitz products, kind::f16 with the hi/lo split: 3 MMAs
    # per K step): their MMA flops issued per launch, against the fp16 dense peak (= bf16's)
    R = cfg.radius
    f16_peak = peaks.get("bf16_tflops", 2250.0) * 1e12
    tc_flop = {
        # column pass: tiles of 128 (plane, column) pairs x 64 rows, K = round_up(64 + 2R, 16) input rows
        "vpass": 3 * 2 * 128 * 64 * (((64 + 2 * R) + 15) // 16 * 16) * (K * ((W + 31) // 32))
                 * ((H + 63) // 64),
        # row pass: tiles of 128 (plane, row) pairs x 64 columns, K = 128 input columns
        "hpass": 3 * 2 * 128 * 64 * 128 * K * ((H + 31) // 32) * ((W + 63) // 64),
    }
    # tensor-core peak for the coefficient contraction (TF32): the measured bf16 peak x the nominal
    # dense TF32 / bf16 ratio (1.1 / 2.25 PFLOP/s, B200_PROFILING.md)
    tf32_peak = peaks.get("bf16_tflops", 2250.0) * (1.1 / 2.25) * 1e12
    traffic = {}
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")))
        traffic = tj.get("kernels", {})
    except Exception:
        pass

    def kernel_roof(name):
        """Roofline of one filter kernel from its algorithmic bytes / FMA-pipe ops, per step
        (the sum of its row-band launches when the filter is pipelined)."""
        t = per_step[name] * 1e-3
        hbm_gbs = work[name]["bytes"] / t / 1e9
        fma_s = work[name]["fma"] / t
        t_hbm = work[name]["bytes"] / (hbm_peak * 1e9)
        t_alu = work[name]["fma"] / fma_peak(sm_mhz, nsm)
        if name == "coeffs" and K <= 64:   # k_coeffs_mma: mma.sync TF32 (3xTF32 split)
            fl = work[name]["mma_flop"] / t
            t_tc = work[name]["mma_flop"] / tf32_peak
            if t_tc >= t_hbm:
                r = {"bound": "tensor", "achieved": round(fl / 1e12, 3), "peak": round(tf32_peak / 1e12, 1),
                     "unit": "TFLOP/s (tf32)", "frac": round(fl / tf32_peak, 4),
                     "peak_basis": "MEASURED_PEAKS bf16_tflops x 1.1/2.25 (nominal dense tf32/bf16); "
                                   "algorithmic 2 K^2 flop/px, the 3xTF32 split issues 3x that",
                     "hbm_achieved_gbs": round(hbm_gbs, 1), "hbm_frac": round(hbm_gbs / hbm_peak, 4)}
            else:
                r = {"bound": "hbm", "achieved": round(hbm_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(hbm_gbs / hbm_peak, 4), "peak_basis": "measured copy (MEASURED_PEAKS.json hbm_gbs)",
                     "tc_achieved_tflops": round(fl / 1e12, 3)}
        elif (name == "vpass" and vtc) or (name == "hpass" and htc):
            # the FIR on the tensor cores: HBM-bound (the tensor pipe runs well below its roof)
            r = {"bound": "hbm", "achieved": round(hbm_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                 "frac": round(hbm_gbs / hbm_peak, 4), "peak_basis": "measured copy (MEASURED_PEAKS.json hbm_gbs)",
                 "path": "tensor cores (tcgen05 kind::f16, Toeplitz FIR, fp16 hi/lo split)",
                 "tc_issued_tflops": round(tc_flop[name] / t / 1e12, 2),
                 "tc_frac_of_f16_peak": round(tc_flop[name] / t / f16_peak, 4)}
            # bytes per stored plane value: fp16 hi + e4m3 residual for the tensor-core row pass, else fp32
            pbytes = 3 if htc else 4
            if name == "vpass":   # it only writes: the bytes it stores against the write-only bandwidth
                wb = pbytes * H * W * (cfg.n + 1) * K
                r["write_roof"] = {"achieved": round(wb / t / 1e9, 1), "peak": round(write_peak, 1), "unit": "GB/s",
                                   "frac": round(wb / t / 1e9 / write_peak, 4),
                                   "peak_basis": "4 GiB fill measured in this run (best of 6)",
                                   "bytes": f"the planes as stored ({pbytes} bytes per value)"}
            if name == "hpass":   # it only reads (the planes and the coefficient planes): the read-only bandwidth
                rb = H * W * (pbytes * (cfg.n + 1) * K + 4 * K)
                r["read_roof"] = {"achieved": round(rb / t / 1e9, 1), "peak": round(read_peak, 1), "unit": "GB/s",
                                  "frac": round(rb / t / 1e9 / read_peak, 4),
                                  "peak_basis": "fp32 sum over 4 GiB measured in this run (best of 6)",
                                  "bytes": f"planes as stored ({pbytes} bytes per value) + fp32 coefficient planes, read once"}
        elif t_alu > t_hbm:
            r = {"bound": "alu", "achieved": round(fma_s / 1e12, 3), "peak": round(fma_peak(sm_mhz, nsm) / 1e12, 3),
                 "unit": "TFMA/s (fp32)", "frac": round(fma_s / fma_peak(sm_mhz, nsm), 4),
                 "peak_basis": f"{nsm} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (median SM clock in the timed region)",
                 "hbm_achieved_gbs": round(hbm_gbs, 1), "hbm_frac": round(hbm_gbs / hbm_peak, 4)}
        else:
            r = {"bound": "hbm", "achieved": round(hbm_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                 "frac": round(hbm_gbs / hbm_peak, 4), "peak_basis": "measured copy (MEASURED_PEAKS.json hbm_gbs)"}
        r.update({"kernel": name, "traffic": traffic.get(kname.get(name, ""), {}).get("dram_bytes"),
                  "ms_per_launch": round(per_launch[name], 4), "launches_per_step": kern[name][1] // args.steps,
                  "ms_per_step": round(per_step[name], 4)})
        if r["traffic"] is not None and r["launches_per_step"] > 1:   # the capture is of one band's launch
            r["traffic_note"] = "ncu capture of one band launch (1/%d of the step's rows)" % r["launches_per_step"]
        return r

    dom = max(per_step, key=per_step.get)
    filt_kernels = [k for k in ("vpass", "hpass", "coeffs") if per_step.get(k)]
    fdom = max(filt_kernels, key=per_step.get)
    filter_roof = kernel_roof(fdom)
    t_wall = prof.get("filter", (0.0, 0))[0] / args.steps * 1e-3   # the filter stage's wall time per step
    if bands > 1 and dom in ("vpass", "hpass", "coeffs") and t_wall > 0:
        # Pipelined filter: the column pass of band b + 1 overlaps the row pass of band b, so the unit that
        # bounds the step is the pair (plus the coefficient kernel beside band 0): the algorithmic bytes of
        # the three kernels over the filter stage's wall time, against the copy bandwidth.
        pb = sum(work[k]["bytes"] for k in ("vpass", "hpass", "coeffs"))
        roof = {"bound": "hbm", "kernel": "k_range_vpass_tc | k_hpass_combine_tc | k_coeffs_tc (pipelined, %d row bands)"
                % bands, "achieved": round(pb / t_wall / 1e9, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(pb / t_wall / 1e9 / hbm_peak, 4),
                "peak_basis": "measured copy (MEASURED_PEAKS.json hbm_gbs)",
                "algorithmic_bytes": int(pb), "ms_wall": round(t_wall * 1e3, 4),
                "traffic": (sum(traffic.get(kname[k], {}).get("dram_bytes") or 0 for k in ("vpass", "hpass")) * bands
                            + (traffic.get(kname["coeffs"], {}).get("dram_bytes") or 0)) or None,
                "traffic_basis": "ncu dram bytes of one band launch of each pass x bands + the coefficient kernel",
                "kernels": {k: kernel_roof(k) for k in ("vpass", "hpass", "coeffs")}}
    elif dom in work:
        roof = kernel_roof(dom)
    else:
        # The clustering kernel against the HBM roof: its algorithmic bytes are the K-1 splits of the
        # procedure, each reading the node's members once per Lloyd pass, then once more and writing
        # them (coordinates + index) for the partition.  It is bound by the latency
        # of its dependent chain of passes and exchanges, not by bandwidth, hence the low fraction.
        if args.cluster_stride > 1:
            _, info = hdf.cluster_sampled(pd, K, args.cluster_stride)
        else:
            _, _, info = hdf.cluster(pd, K)
        cb = 4 * cfg.rho * (info.point_passes + info.points_split) + 4 * (cfg.rho + 1) * info.points_split
        t = per_launch[dom] * 1e-3
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(cb / t / 1e9, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(cb / t / 1e9 / hbm_peak, 4),
                "traffic": traffic.get("k_bisect", {}).get("dram_bytes"),   # (ncu runs it without clusters)
                "ms_per_launch": round(per_launch[dom], 4), "algorithmic_bytes": int(cb),
                "peak_basis": "measured copy (MEASURED_PEAKS.json hbm_gbs)",
                "note": "exact bisecting K-means: a dependent chain of 2-means passes and group exchanges "
                        f"({info.point_passes} member-passes over the {K - 1} splits); latency-bound, see "
                        "filter_roofline for the dominant filter kernel"}
    # the filter stage: pinv runs on a side stream concurrently with the column pass (not on the path)
    t_filter = t_wall if t_wall > 0 else sum(per_step[k] for k in ("coeffs", "vpass", "hpass", "fallback")) * 1e-3
    filt = {"ms": round(t_filter * 1e3, 4), "B_req_bytes": work["filter"]["bytes"],
            "hbm_gbs": round(work["filter"]["bytes"] / t_filter / 1e9, 1),
            "hbm_frac": round(work["filter"]["bytes"] / t_filter / 1e9 / hbm_peak, 4),
            "kernels": {k: kernel_roof(k) for k in filt_kernels}, "row_bands": bands,
            "ms_basis": "wall time of the filter stage (HDF_STAGE_FILTER)" if t_wall > 0 else "sum of the stages"}
    launches = sum(n for k, (ms, n) in kern.items())
    return {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "ms_per_step_stats": {"median": round(statistics.median(step_ms), 4), "mean": round(statistics.mean(step_ms), 4),
                              "min": round(min(step_ms), 4), "max": round(max(step_ms), 4)},
        "higher_is_better": True,
        "scaling": "strong" if (args.strips and world > 1) else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY 8(d) generators)",
        "config": dict(workload_config(args.config, world),
                       **({"variant": "hard (one-hot coefficients, P:341-357); e2e is the soft path's"}
                          if args.variant == "hard" else {}),
                       **({"variant": "iir (Young's recursive Gaussian, P:332-333, NEXT #1); the vpass stage "
                                      "includes the column and row recursions"}
                          if args.variant == "iir" else {}),
                       cluster=("exact bisecting K-means of every pixel (P:328-329, R1-R4)" if args.cluster_stride == 1
                                else f"sampled mode: bisecting K-means of the stride-{args.cluster_stride} sample "
                                     f"(P:329 'any efficient clustering'; R15 5% rule checked in tests)")),
        "stages_ms_per_step": {k: round(ms / args.steps, 4) for k, (ms, n) in prof.items() if n},
        "filter": filt, "roofline": roof, "filter_roofline": filter_roof, "gpu_launches": launches, "clocks": clk,
        "e2e": {"value": round(e2e_val, 3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        **({"exact_cluster": exact} if exact else {}),
        # pixels whose normaliser fell under tau omega(0) phi(0) and took the direct window sum (R9), last e2e step
        "n_flagged": int(host_res[2]),
    }


def _rank_image(name: str, rank: int):
    import synth
    cfg = synth.CONFIGS[name]
    # same recipe, seed offset by rank (an independent image of the same workload)
    import dataclasses
    cfg2 = dataclasses.replace(cfg, seed=cfg.seed + 1000 * rank)
    old = synth.CONFIGS[name]
    synth.CONFIGS[name] = cfg2
    try:
        return synth.make(name)
    finally:
        synth.CONFIGS[name] = old


# --------------------------------------------------------------------------- oracle timing ----
def oracle_sample(config: str, budget_s: float, min_s: float = 0.0):
    """Time the fp64 CPU oracle (as it stands) on host cores: cluster + filter of the workload's
    image (a top strip of rows if one image would exceed the budget), repeated until at least
    min_s seconds of CPU work have been timed.  Returns (Mpixel/s, seconds, images, sample)."""
    import oracle
    import synth
    cfg, f, p = synth.make(config)
    H, W = f.shape[:2]
    rows = H
    est_per_px = 8e-6 if cfg.n <= 6 else 6e-5
    if H * W * est_per_px > budget_s:
        rows = max(16, int(budget_s / (W * est_per_px)))
    fs, ps = np.ascontiguousarray(f[:rows]), np.ascontiguousarray(p[:rows])
    t0 = time.perf_counter()
    reps = 0
    while True:
        cen, _, _, _ = oracle.cluster(ps, cfg.K)
        oracle.filter(fs, ps, cfg.kind, cfg.sigma_s, cfg.sigma_r, cen, r=cfg.radius)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_s or dt * (reps + 1) / reps > budget_s:
            break
    what = "full image" if rows == H else "top strip"
    sample = (f"{reps} x ({rows}x{W} rows of the {config} image, {what}): oracle.cluster + oracle.filter, fp64, "
              f"{cores()} OpenMP threads")
    return reps * rows * W / dt / 1e6, dt, reps, sample


def workload_config(name: str, world: int = 1) -> dict:
    import synth
    cfg = synth.CONFIGS[name]
    return {"workload": name, "note": cfg.note, "H": cfg.H, "W": cfg.W, "n": cfg.n, "rho": cfg.rho, "K": cfg.K,
            "kind": cfg.kind, "sigma_s": cfg.sigma_s, "radius": cfg.radius, "sigma_r": cfg.sigma_r,
            "images_per_step": world, "parallelism": f"independent image per rank x{world}",
            "l2": "flushed between steps (512 MiB write, outside the timed events)"}


def cores():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_model() -> str:
    """The host CPU (lscpu 'Model name'), for the cpu_baseline record."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    vals, secs = [], []
    budget = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    sample = ""
    for i in range(args.warmup + args.steps):
        v, dt, reps, sample = oracle_sample(args.config, budget)
        if i >= args.warmup:
            vals.append(v)
            secs.append(dt / reps)
    value = statistics.median(vals)
    return {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(secs), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8(d) generators)",
            "impl": "reference", "config": workload_config(args.config, 1),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores(), "cpu_model": cpu_model(),
                             "kind": "oracle", "sample": "each step: " + sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--all", action="store_true", help="one line per config (exploration)")
    ap.add_argument("--strips", action="store_true",
                    help="N > 1: one image in row strips over the ranks (strong scaling, exploration)")
    ap.add_argument("--cluster-stride", type=int, default=-1,
                    help="1: exact clustering of every pixel; s > 1: the sampled mode (hdf_cluster_sampled); "
                         "-1 (default): the workload's stride from SAMPLED_STRIDE (1 where R15 fails)")
    ap.add_argument("--variant", default="soft", choices=["soft", "hard", "iir"],
                    help="hard: the hard-assignment variant (exploration; not the headline)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    configs = ["c1", "c2a", "c2b", "c3", "c4", "c5"] if args.all else [args.config]
    auto_stride = args.cluster_stride < 1
    for c in configs:
        args.config = c
        if auto_stride:
            args.cluster_stride = SAMPLED_STRIDE.get(c, 1)
        out = run_ours(args, rank, world, dist)
        if rank == 0 and not args.no_cpu_baseline and not args.all:
            os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
            v, dt, reps, sample = oracle_sample(c, 30.0, min_s=10.0)
            out["cpu_baseline"] = {"value": round(v, 4), "unit": UNIT, "cores": cores(), "cpu_model": cpu_model(),
                                   "kind": "oracle", "sample": sample, "seconds": round(dt, 2)}
        if rank == 0:
            print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
