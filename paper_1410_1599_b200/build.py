"""Build libmpgpu.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repository snapshot to the GPU box).

    python paper_1410_1599_b200/build.py [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libmpgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["gemm.cu", "gemm_tc.cu", "metrics.cu", "elementwise.cu", "elementwise_fused8.cu",
           "elementwise_fused16.cu", "elementwise_fused32.cu", "lu.cu", "capi.cu", "group.cu",
           "gemm_wide.cu", "metrics_wide.cu"] + \
    [f"{k}_wide{L}.cu" for k in ("elementwise", "lu") for L in (64, 128, 256, 288)]
HEADERS = ["mp_arith.cuh", "kernels.h", "wmp.cuh", "wkern.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-I" + str(ROOT / "include")]


def _newest_dep() -> float:
    deps = [CSRC / h for h in HEADERS] + [ROOT / "include" / "mpgpu.h"]
    return max(p.stat().st_mtime for p in deps if p.exists())


def _compile(src: str, force: bool) -> Path:
    obj = BUILD / (src + ".o")
    s = CSRC / src
    srcs = [s] + ([CSRC / re.sub(r"_(wide|fused)\d*", "", src)] if ("_wide" in src or "_fused" in src) else [])  # *_wide*.cu / *_fused*.cu include *.cu
    if (not force and obj.exists() and all(obj.stat().st_mtime >= x.stat().st_mtime for x in srcs)
            and obj.stat().st_mtime >= _newest_dep()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if (force or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs)):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(LIB), *map(str, objs),
               "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
