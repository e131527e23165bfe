"""B200 (sm_100a) implementation of the fast high-dimensional bilateral / nonlocal-means filter of
Nair & Chaudhury (arXiv 1811.02363) -- thin Python binding over the C ABI in include/hdf.h.

This module only marshals arguments (torch tensors -> device pointers, the current CUDA stream,
workspace allocation).  Every arithmetic step runs in libhdf.so's CUDA kernels; there is no CPU
fallback, and importing the binding fails loudly if the library is missing.

Names follow the paper: f (image, [H,W,n]), p (guide, [H,W,rho]), sigma_s / radius S (spatial
kernel omega), sigma_r (range kernel phi), K clusters with centres mu_k, g (output).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdf.so")

OK, ERR_ARG, ERR_K, ERR_WORKSPACE, ERR_CUDA, WARN_ILLCOND = 0, 1, 2, 3, 4, 5
GAUSSIAN, BOX, GAUSSIAN_IIR = 0, 1, 2
KIND = {"gaussian": GAUSSIAN, "box": BOX, "gaussian_iir": GAUSSIAN_IIR}
MAX_K, MAX_RHO, MAX_N, MAX_RADIUS = 128, 64, 64, 32

# every symbol include/hdf.h declares (checked by the CPU tests)
EXPORTS = ("hdf_version", "hdf_last_error", "hdf_cluster_workspace_bytes", "hdf_cluster",
           "hdf_filter_workspace_bytes", "hdf_filter", "hdf_filter_hard", "hdf_filter_host_workspace_bytes",
           "hdf_filter_host", "hdf_pca_guide_workspace_bytes", "hdf_pca_guide",
           "hdf_profile_enable", "hdf_profile_collect", "hdf_cluster_trace", "hdf_filter_flagged", "hdf_scale_guide",
           "hdf_cluster_sampled_workspace_bytes", "hdf_cluster_sampled", "hdf_sample_guide")
STAGES = ("cluster", "pinv", "coeffs", "vpass", "hpass", "fallback", "h2d", "d2h", "filter")


class HdfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hdf status {status}: {msg}")
        self.status = status


class HdfKError(HdfError):
    def __init__(self, status: int, msg: str, achievable: int):
        super().__init__(status, msg)
        self.achievable = achievable


class ClusterInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("achievable_k", C.c_int32), ("splits_computed", C.c_int32),
                ("lloyd_iters", C.c_int32), ("e_k", C.c_double), ("grid_splits", C.c_int32),
                ("tile_points", C.c_int32), ("launch_ctas", C.c_int32), ("cluster_ctas", C.c_int32),
                ("point_passes", C.c_int64), ("points_split", C.c_int64)]


_lib = None


def lib():
    """Load libhdf.so (raises if it has not been built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1811_02363_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, i, f, sz = C.c_void_p, C.c_int, C.c_float, C.c_size_t
        L.hdf_version.restype = C.c_char_p
        L.hdf_last_error.restype = C.c_char_p
        L.hdf_cluster_workspace_bytes.argtypes = [i, i, i, i]
        L.hdf_cluster_workspace_bytes.restype = sz
        L.hdf_cluster.argtypes = [vp, i, i, i, i, vp, vp, C.POINTER(ClusterInfo), vp, sz, vp]
        L.hdf_cluster.restype = i
        L.hdf_filter_workspace_bytes.argtypes = [i, i, i, i, i, i, f, i]
        L.hdf_filter_workspace_bytes.restype = sz
        L.hdf_filter.argtypes = [vp, i, vp, i, i, i, i, f, i, f, i, vp, f, vp, C.POINTER(C.c_int32), vp, sz, vp]
        L.hdf_filter.restype = i
        L.hdf_pca_guide_workspace_bytes.argtypes = [i, i, i, i, i]
        L.hdf_pca_guide_workspace_bytes.restype = sz
        L.hdf_pca_guide.argtypes = [vp, i, i, i, i, i, vp, vp, vp, sz, vp]
        L.hdf_pca_guide.restype = i
        L.hdf_filter_hard.argtypes = [vp, i, vp, i, i, i, i, f, i, f, i, vp, vp, vp, vp, sz, vp]
        L.hdf_filter_hard.restype = i
        L.hdf_filter_host_workspace_bytes.argtypes = [i, i, i, i, i, i, f, i]
        L.hdf_filter_host_workspace_bytes.restype = sz
        L.hdf_filter_host.argtypes = [vp, i, vp, i, i, i, i, f, i, f, i, f, i, vp, vp, C.POINTER(C.c_int32),
                                      C.POINTER(ClusterInfo), vp, sz, vp]
        L.hdf_cluster_sampled_workspace_bytes.argtypes = [i, i, i, i, i]
        L.hdf_cluster_sampled_workspace_bytes.restype = sz
        L.hdf_cluster_sampled.argtypes = [vp, i, i, i, i, i, vp, C.POINTER(ClusterInfo), vp, sz, vp]
        L.hdf_cluster_sampled.restype = i
        ll = C.c_longlong
        L.hdf_sample_guide.argtypes = [vp, ll, i, ll, ll, vp, ll, vp]
        L.hdf_sample_guide.restype = i
        L.hdf_filter_host.restype = i
        L.hdf_profile_enable.argtypes = [i]
        L.hdf_profile_enable.restype = i
        L.hdf_profile_collect.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.hdf_profile_collect.restype = i
        L.hdf_cluster_trace.argtypes = [vp, i, i, i, i, vp, C.POINTER(C.c_longlong), i]
        L.hdf_cluster_trace.restype = i
        L.hdf_filter_flagged.argtypes = [vp, i, i, i, i, i, C.POINTER(C.c_int32), i]
        L.hdf_filter_flagged.restype = i
        L.hdf_scale_guide.argtypes = [vp, i, i, i, vp, vp, i, vp, vp, vp]
        L.hdf_scale_guide.restype = i
        _lib = L
    return _lib


def version() -> str:
    return lib().hdf_version().decode()


def _raise(st: int):
    msg = lib().hdf_last_error().decode()
    raise HdfError(st, msg)


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dev_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _out(out, shape, device, name="out") -> torch.Tensor:
    """The caller's output tensor: float32, contiguous, of exactly `shape`, on `device` (the kernels
    write shape-many floats through its pointer)."""
    t = _dev_f32(out, name)
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)} (got {tuple(t.shape)})")
    if t.device != device:
        raise ValueError(f"{name} must be on {device} (got {t.device})")
    return t


def _same_device(t: torch.Tensor, device, name: str):
    if t.device != device:
        raise ValueError(f"{name} must be on {device} (got {t.device})")


def _hwc(t: torch.Tensor, name: str):
    if t.dim() == 2:
        return t.shape[0], t.shape[1], 1
    if t.dim() != 3:
        raise ValueError(f"{name} must be [H,W] or [H,W,c]")
    return t.shape[0], t.shape[1], t.shape[2]


class Workspace:
    """A reusable device workspace (grown on demand; the library never allocates)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_default_ws = Workspace()


def cluster_workspace_bytes(H: int, W: int, rho: int, K: int) -> int:
    return int(lib().hdf_cluster_workspace_bytes(H, W, rho, K))


def filter_workspace_bytes(H, W, n, rho, K, kind="gaussian", sigma_s=1.0, radius=-1) -> int:
    return int(lib().hdf_filter_workspace_bytes(H, W, n, rho, K, KIND[kind], float(sigma_s), int(radius)))


def cluster(p: torch.Tensor, K: int, labels: bool = False, info: bool = True, ws: Workspace | None = None,
            stream=None):
    """Step 1: bisecting K-means of the guide p [H,W,rho].

    Returns (centres [K,rho] fp32, labels [H,W] int32 or None, ClusterInfo or None).  With
    info=True the call synchronises and raises HdfKError if K exceeds the number of distinct
    guide vectors (R5)."""
    p = _dev_f32(p, "p")
    H, W, rho = _hwc(p, "p")
    cen = torch.empty((K, rho), dtype=torch.float32, device=p.device)
    lab = torch.empty((H, W), dtype=torch.int32, device=p.device) if labels else None
    wsb = (ws or _default_ws).get(cluster_workspace_bytes(H, W, rho, K), p.device)
    inf = ClusterInfo() if info else None
    st = lib().hdf_cluster(p.data_ptr(), H, W, rho, K, cen.data_ptr(), lab.data_ptr() if lab is not None else None,
                           C.byref(inf) if inf is not None else None, wsb.data_ptr(), wsb.numel(),
                           _stream_ptr(stream))
    if st == ERR_K:
        raise HdfKError(st, lib().hdf_last_error().decode(), inf.achievable_k)
    if st != OK:
        _raise(st)
    return cen, lab, inf


def cluster_sampled(p: torch.Tensor, K: int, stride: int, info: bool = True, ws: Workspace | None = None,
                    stream=None):
    """The sampled clustering mode ("any efficient clustering method"): bisecting K-means of the
    stride sample p.flat[0::stride] (include/hdf.h, hdf_cluster_sampled).  stride = 1 is cluster().
    Returns (centres [K,rho] fp32, ClusterInfo of the sample or None)."""
    p = _dev_f32(p, "p")
    H, W, rho = _hwc(p, "p")
    cen = torch.empty((K, rho), dtype=torch.float32, device=p.device)
    need = int(lib().hdf_cluster_sampled_workspace_bytes(H, W, rho, K, int(stride)))
    wsb = (ws or _default_ws).get(max(need, 256), p.device)
    inf = ClusterInfo() if info else None
    st = lib().hdf_cluster_sampled(p.data_ptr(), H, W, rho, K, int(stride), cen.data_ptr(),
                                   C.byref(inf) if inf is not None else None, wsb.data_ptr(), wsb.numel(),
                                   _stream_ptr(stream))
    if st == ERR_K:
        raise HdfKError(st, lib().hdf_last_error().decode(), inf.achievable_k)
    if st != OK:
        _raise(st)
    return cen, inf


def sample_guide(p: torch.Tensor, i0: int, stride: int, M: int, stream=None) -> torch.Tensor:
    """Gather p.flat[i0 + j stride], j < M ([M, rho]; include/hdf.h, hdf_sample_guide)."""
    p = _dev_f32(p, "p")
    rho = p.shape[-1] if p.dim() == 3 else 1
    N = p.numel() // rho
    out = torch.empty((max(M, 0), rho), dtype=torch.float32, device=p.device)
    st = lib().hdf_sample_guide(p.data_ptr(), N, rho, int(i0), int(stride), out.data_ptr(), int(M),
                                _stream_ptr(stream))
    if st != OK:
        _raise(st)
    return out


@dataclass
class FilterResult:
    g: torch.Tensor
    n_flagged: int | None
    status: int


def filter(f: torch.Tensor, p: torch.Tensor | None = None, *, kind: str = "gaussian", sigma_s: float = 1.0,
           radius: int = -1, sigma_r: float = 1.0, K: int = 16, centres: torch.Tensor | None = None,
           tau: float = 0.5, out: torch.Tensor | None = None, count_flagged: bool = False,
           ws: Workspace | None = None, stream=None) -> FilterResult:
    """Steps 2-6 (Algorithm 1): the fast filter g = (HDapprox)/(approxDen).

    f [H,W,n] and guide p [H,W,rho] (p=None -> bilateral, p = f).  centres [K,rho] (None -> the
    library clusters p first).  kind: "gaussian" (exact FIR, radius -1 -> ceil(3 sigma_s)), "box"
    (radius required) or "gaussian_iir" (Young's recursive Gaussian; radius only sizes
    the R9 fallback's window).  tau: rule R9 threshold.  count_flagged synchronises and returns
    the number of pixels that took the direct (num)/(den) fallback."""
    f = _dev_f32(f, "f")
    if p is None:
        p = f
    p = _dev_f32(p, "p")
    H, W, n = _hwc(f, "f")
    Hp, Wp, rho = _hwc(p, "p")
    if (Hp, Wp) != (H, W):
        raise ValueError("f and p must have the same H, W")
    _same_device(p, f.device, "p")
    if centres is not None:
        centres = _dev_f32(centres, "centres")
        if centres.dim() != 2 or centres.shape[1] != rho:
            raise ValueError("centres must be [K, rho]")
        _same_device(centres, f.device, "centres")
        K = centres.shape[0]
    g = _out(out, (H, W, n), f.device) if out is not None else \
        torch.empty((H, W, n), dtype=torch.float32, device=f.device)
    need = filter_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius)
    wsb = (ws or _default_ws).get(need, f.device)
    nfl = C.c_int32(-1)
    st = lib().hdf_filter(f.data_ptr(), n, p.data_ptr(), rho, H, W, KIND[kind], float(sigma_s), int(radius),
                          float(sigma_r), int(K), centres.data_ptr() if centres is not None else None, float(tau),
                          g.data_ptr(), C.byref(nfl) if count_flagged else None, wsb.data_ptr(), wsb.numel(),
                          _stream_ptr(stream))
    if st == ERR_K:
        raise HdfKError(st, lib().hdf_last_error().decode(), -1)
    if st not in (OK, WARN_ILLCOND):
        _raise(st)
    return FilterResult(g, nfl.value if count_flagged else None, st)


def filter_hard(f: torch.Tensor, p: torch.Tensor | None = None, *, kind: str = "gaussian", sigma_s: float = 1.0,
                radius: int = -1, sigma_r: float = 1.0, K: int = 16, centres: torch.Tensor | None = None,
                labels: torch.Tensor | None = None, out: torch.Tensor | None = None, ws: Workspace | None = None,
                stream=None) -> torch.Tensor:
    """Hard-assignment variant (coeffICIP)/(HDapprox2): g(i) = v_s(i) / r_s(i), s = label(i).

    centres [K,rho] and labels [H,W] int32 (e.g. from cluster(..., labels=True)) together, or neither
    (the library clusters p first)."""
    f = _dev_f32(f, "f")
    if p is None:
        p = f
    p = _dev_f32(p, "p")
    H, W, n = _hwc(f, "f")
    Hp, Wp, rho = _hwc(p, "p")
    if (Hp, Wp) != (H, W):
        raise ValueError("f and p must have the same H, W")
    if (centres is None) != (labels is None):
        raise ValueError("pass both centres and labels, or neither")
    _same_device(p, f.device, "p")
    if centres is not None:
        centres = _dev_f32(centres, "centres")
        if centres.dim() != 2 or centres.shape[1] != rho:
            raise ValueError("centres must be [K, rho]")
        K = centres.shape[0]
        if not (labels.is_cuda and labels.dtype == torch.int32 and labels.is_contiguous()
                and labels.numel() == H * W):
            raise TypeError("labels must be a contiguous int32 CUDA tensor of H*W elements")
        _same_device(centres, f.device, "centres")
        _same_device(labels, f.device, "labels")
    g = _out(out, (H, W, n), f.device) if out is not None else \
        torch.empty((H, W, n), dtype=torch.float32, device=f.device)
    need = filter_workspace_bytes(H, W, n, rho, K, kind, sigma_s, radius)
    wsb = (ws or _default_ws).get(need, f.device)
    st = lib().hdf_filter_hard(f.data_ptr(), n, p.data_ptr(), rho, H, W, KIND[kind], float(sigma_s), int(radius),
                               float(sigma_r), int(K), centres.data_ptr() if centres is not None else None,
                               labels.data_ptr() if labels is not None else None, g.data_ptr(), wsb.data_ptr(),
                               wsb.numel(), _stream_ptr(stream))
    if st != OK:
        _raise(st)
    return g


def pca_guide(f: torch.Tensor, m: int = 3, dim: int = 6, *, basis: bool = False, ws: Workspace | None = None,
              stream=None):
    """PCA-NLM guide: m x m x n patches of f projected on the `dim` leading eigenvectors of
    their covariance.  Returns the guide [H, W, dim] (and the basis [dim, n m^2] with basis=True)."""
    f = _dev_f32(f, "f")
    H, W, n = _hwc(f, "f")
    p = torch.empty((H, W, dim), dtype=torch.float32, device=f.device)
    B = torch.empty((dim, n * m * m), dtype=torch.float32, device=f.device) if basis else None
    need = int(lib().hdf_pca_guide_workspace_bytes(H, W, n, int(m), int(dim)))
    wsb = (ws or _default_ws).get(max(need, 256), f.device)
    st = lib().hdf_pca_guide(f.data_ptr(), H, W, n, int(m), int(dim), p.data_ptr(),
                             B.data_ptr() if B is not None else None, wsb.data_ptr(), wsb.numel(),
                             _stream_ptr(stream))
    if st != OK:
        _raise(st)
    return (p, B) if basis else p


def scale_guide(p: torch.Tensor, scale=None, extra: torch.Tensor | None = None, extra_scale=None,
                stream=None) -> torch.Tensor:
    """Anisotropic / augmented guide: [p * scale, extra * extra_scale] per channel
    (include/hdf.h, hdf_scale_guide).  With scale = 1 / sigma_d the isotropic filter at sigma_r = 1 on
    the result is the filter with the diagonal range kernel exp(-sum_d x_d^2 / 2 sigma_d^2)."""
    p = _dev_f32(p, "p")
    H, W, rho = _hwc(p, "p")
    e = 0
    if extra is not None:
        extra = _dev_f32(extra, "extra")
        He, We, e = _hwc(extra, "extra")
        if (He, We) != (H, W):
            raise ValueError("extra must have the guide's H, W")
        _same_device(extra, p.device, "extra")
    sc = (C.c_float * rho)(*[float(v) for v in scale]) if scale is not None else None
    es = (C.c_float * e)(*[float(v) for v in extra_scale]) if (extra_scale is not None and e) else None
    if scale is not None and len(scale) != rho:
        raise ValueError(f"scale must have {rho} entries")
    if extra_scale is not None and len(extra_scale) != e:
        raise ValueError(f"extra_scale must have {e} entries")
    out = torch.empty((H, W, rho + e), dtype=torch.float32, device=p.device)
    st = lib().hdf_scale_guide(p.data_ptr(), H, W, rho, sc, extra.data_ptr() if extra is not None else None, e,
                               es, out.data_ptr(), _stream_ptr(stream))
    if st != OK:
        _raise(st)
    return out


def anisotropic_guide(p: torch.Tensor, sigmas, extra: torch.Tensor | None = None, extra_sigmas=None,
                      stream=None) -> torch.Tensor:
    """The guide for per-channel range sigmas (e.g. sigma_r = 50 on PCA dimensions and 10 on an
    appended infrared channel): scale_guide with scale = 1 / sigma; filter it at sigma_r = 1."""
    return scale_guide(p, [1.0 / float(s) for s in sigmas], extra,
                       [1.0 / float(s) for s in extra_sigmas] if extra_sigmas is not None else None, stream)


def filter_host(f_host: torch.Tensor, p_host: torch.Tensor | None = None, *, kind: str = "gaussian",
                sigma_s: float = 1.0, radius: int = -1, sigma_r: float = 1.0, K: int = 16, tau: float = 0.5,
                cluster_stride: int = 1, out: torch.Tensor | None = None, ws: Workspace | None = None, device=None,
                stream=None):
    """End-to-end from HOST buffers (pinned preferred): H2D copy, cluster (exact, or the sampled mode
    with cluster_stride > 1), filter, D2H copy, all inside the library on one stream.  Returns
    (g_host, centres_host, n_flagged, ClusterInfo)."""
    if p_host is None:
        p_host = f_host
    for t, nm in ((f_host, "f"), (p_host, "p")):
        if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
            raise TypeError(f"{nm} must be a contiguous float32 host tensor")
    H, W, n = _hwc(f_host, "f")
    Hp, Wp, rho = _hwc(p_host, "p")
    if (Hp, Wp) != (H, W):
        raise ValueError("f and p must have the same H, W")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if out is not None:
        if out.is_cuda or out.dtype != torch.float32 or not out.is_contiguous() or out.numel() != H * W * n:
            raise ValueError(f"out must be a contiguous float32 host tensor of {H * W * n} elements")
        g = out
    else:
        g = torch.empty((H, W, n), dtype=torch.float32, pin_memory=True)
    cen = torch.empty((K, rho), dtype=torch.float32)
    need = int(lib().hdf_filter_host_workspace_bytes(H, W, n, rho, K, KIND[kind], float(sigma_s), int(radius)))
    wsb = (ws or _default_ws).get(need, dev)
    nfl = C.c_int32(0)
    inf = ClusterInfo()
    st = lib().hdf_filter_host(f_host.data_ptr(), n, p_host.data_ptr(), rho, H, W, KIND[kind], float(sigma_s),
                               int(radius), float(sigma_r), int(K), float(tau), int(cluster_stride), g.data_ptr(),
                               cen.data_ptr(),
                               C.byref(nfl), C.byref(inf), wsb.data_ptr(), wsb.numel(), _stream_ptr(stream))
    if st == ERR_K:
        raise HdfKError(st, lib().hdf_last_error().decode(), inf.achievable_k)
    if st not in (OK, WARN_ILLCOND):
        _raise(st)
    return g, cen, nfl.value, inf


def flagged_pixels(ws: Workspace, H: int, W: int, n: int, rho: int, K: int):
    """The pixel indices (y*W + x, sorted) that took the R9 fallback in the last filter() call on
    workspace ws with these sizes (include/hdf.h, hdf_filter_flagged).  Synchronous."""
    import numpy as np
    buf = (C.c_int32 * max(H * W, 1))()
    cnt = lib().hdf_filter_flagged(ws.buf.data_ptr(), H, W, n, rho, K, buf, H * W)
    if cnt < 0:
        _raise(ERR_CUDA)
    return np.sort(np.frombuffer(buf, dtype=np.int32, count=cnt).copy())


def profile_enable(on: bool = True) -> None:
    """Record CUDA events around every stage launch (include/hdf.h, hdf_profile_enable)."""
    lib().hdf_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """Wait for the recorded events; returns {stage: (total_ms, launches)} and clears the record."""
    ms = (C.c_double * len(STAGES))()
    n = (C.c_int32 * len(STAGES))()
    st = lib().hdf_profile_collect(ms, n)
    if st != OK:
        _raise(st)
    return {name: (ms[i], n[i]) for i, name in enumerate(STAGES)}


def cluster_trace(p: torch.Tensor, K: int, ws: Workspace | None = None):
    """Diagnostics: (tag | node << 8 | worker << 28, globaltimer ns) events of the clustering workers
    in the last cluster() call on workspace ws (see hdf_cluster_trace in include/hdf.h)."""
    H, W, rho = _hwc(p, "p")
    buf = (C.c_longlong * (2 * 8192))()
    n = lib().hdf_cluster_trace(None, H, W, rho, K, (ws or _default_ws).buf.data_ptr(), buf, 8192)
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(max(n, 0))]
