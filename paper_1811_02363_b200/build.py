"""In-tree build of libhdf.so (the C-ABI library, include/hdf.h) for sm_100a.

nvcc cross-compiles without a GPU.  The radius-templated filter kernels are instantiated once per
compiled radius (inst_r.cu with -DHDF_R=<R>) and those compilations run in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhdf.so")
OBJ = os.path.join(HERE, "_obj")
RADII = (1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 20, 24, 32)   # keep in sync with hdf_dispatch.h kRadii

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")] + os.environ.get("HDF_EXTRA_FLAGS", "").split()


def _sources_digest() -> str:
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cu", ".cuh", ".h")):
                with open(os.path.join(d, name), "rb") as fh:
                    h.update(name.encode() + fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def _compile(src: str, obj: str, defs=()) -> str:
    cmd = [NVCC, *FLAGS, *defs, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)} {defs}:\n{r.stderr[-6000:]}")
    return r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source into libhdf.so (skipped when the sources are unchanged)."""
    os.makedirs(OBJ, exist_ok=True)
    stamp = os.path.join(OBJ, "digest")
    dig = _sources_digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    jobs = [(os.path.join(CSRC, "hdf_api.cu"), os.path.join(OBJ, "hdf_api.o"), ())]
    for r in RADII:
        jobs.append((os.path.join(CSRC, "inst_r.cu"), os.path.join(OBJ, f"inst_r{r}.o"), (f"-DHDF_R={r}",)))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), max(2, os.cpu_count() or 2))) as ex:
        for (src, obj, defs), log in zip(jobs, ex.map(lambda j: _compile(*j), jobs)):
            logs.append(f"== {os.path.basename(src)} {' '.join(defs)}\n{log}")
    with open(os.path.join(OBJ, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", tmp,
           *[j[1] for j in jobs], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-6000:]}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
