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


def _deps(path: str, seen=None) -> list:
    """The file and every local header it includes, transitively (#include "...")."""
    import re
    seen = set() if seen is None else seen
    path = os.path.normpath(path)
    if path in seen or not os.path.exists(path):
        return []
    seen.add(path)
    out = [path]
    with open(path) as fh:
        for inc in re.findall(r'^\s*#include\s+"([^"]+)"', fh.read(), re.M):
            out += _deps(os.path.join(os.path.dirname(path), inc), seen)
    return out


def _digest(src: str, defs=()) -> str:
    h = hashlib.sha256()
    for p in sorted(_deps(src)):
        with open(p, "rb") as fh:
            h.update(os.path.basename(p).encode() + fh.read())
    h.update(" ".join(FLAGS + list(defs)).encode())
    return h.hexdigest()


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
    for r in range(8):     # k_bisect<RHO>, RHO = 0 (runtime) .. 7
        jobs.append((os.path.join(CSRC, "inst_bisect.cu"), os.path.join(OBJ, f"inst_bisect{r}.o"), (f"-DHDF_BRHO={r}",)))
    for nt in range(1, 9):  # k_coeffs_mma<NT, *>, K <= 8 NT
        jobs.append((os.path.join(CSRC, "inst_coeffs.cu"), os.path.join(OBJ, f"inst_coeffs{nt}.o"), (f"-DHDF_CNT={nt}",)))
    # per object: recompile only when its source, a header it includes or the flags changed
    todo = []
    for src, obj, defs in jobs:
        dg = _digest(src, defs)
        st = obj + ".digest"
        if force or not os.path.exists(obj) or not os.path.exists(st) or open(st).read() != dg:
            todo.append((src, obj, defs, dg))
    logs = []

    def run(j):
        src, obj, defs, dg = j
        log = _compile(src, obj, defs)
        with open(obj + ".digest", "w") as fh:
            fh.write(dg)
        with open(obj + ".ptxas.log", "w") as fh:
            fh.write(log)
        return log

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), max(2, os.cpu_count() or 2)))) as ex:
        for (src, obj, defs, _), log in zip(todo, ex.map(run, todo)):
            logs.append(f"== {os.path.basename(src)} {' '.join(defs)}\n{log}")
    with open(os.path.join(OBJ, "ptxas.log"), "w") as fh:
        for src, obj, defs in jobs:
            lp = obj + ".ptxas.log"
            fh.write(f"== {os.path.basename(src)} {' '.join(defs)}\n" + (open(lp).read() if os.path.exists(lp) else "")
                     + "\n")
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
