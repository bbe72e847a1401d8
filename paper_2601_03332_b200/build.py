"""Build liblutkan_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

Usage: python -m paper_2601_03332_b200.build  (or __graft_entry__.build()).
Incremental: an object is rebuilt only when its source or a header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# A/B experiments: LKG_BUILD_TAG=x builds into _build_x/ and ab/liblutkan_x.so with LKG_NVCC_EXTRA flags
# (load it with LKG_LIB=ab/liblutkan_x.so); the default build is unaffected.
_TAG = os.environ.get("LKG_BUILD_TAG", "")
BUILD = os.path.join(PKG, "_build" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(ROOT, "ab", f"liblutkan_{_TAG}.so") if _TAG else os.path.join(PKG, "liblutkan_b200.so")
EXTRA = os.environ.get("LKG_NVCC_EXTRA", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include")]
# The compile kernel must not contract f64 multiply-adds (bit-exact LUT bytes).
PER_FILE = {"compile.cu": ["-fmad=false"], "eval.cu": ["-fmad=false"], "elements.cu": ["-fmad=false"]}


def _newer(src: str, obj: str, headers: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or any(os.path.getmtime(h) > t for h in headers)


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
               glob.glob(os.path.join(ROOT, "include", "*.h")))
    objs, cmds = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))):
        name = os.path.basename(src)
        obj = os.path.join(BUILD, name + ".o")
        objs.append(obj)
        if not _newer(src, obj, headers):
            continue
        cmds.append([NVCC, *ARCH, *COMMON, *EXTRA, *PER_FILE.get(name, []), "-c", src, "-o", obj])
    # the translation units compile side by side (forward_tiled.cu alone takes minutes)
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 4))) as ex:
        list(ex.map(run, cmds))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", LIB, *objs, "-ldl", "-lz"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
