"""Builds the sm_100a CUDA library in-tree (lib/libmigsim_b200.so).

nvcc cross-compiles for B200 without a GPU. Device code uses explicit
round-to-nearest double intrinsics and is additionally compiled with
--fmad=false, so no FMA contraction can change a Goodput value (SURVEY.md
Appendix B rule 3).
"""
from __future__ import annotations

import os
import subprocess
import sys

from .capi import LIB_DIR, LIB_PATH, PKG_DIR

ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
SOURCES = ["space.cu", "goodput.cu", "dp.cu", "dp2.cu", "bruteforce.cu", "table.cu", "wb.cu", "replay.cu", "preinit.cu", "feasible.cu", "shard.cu", "scan.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
    "-I", os.path.join(ROOT, "include"), "-I", CSRC,
] + (["-DMGS_MINB=" + os.environ["MGS_MINB"]] if os.environ.get("MGS_MINB") else [])


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(LIB_DIR, exist_ok=True)
    obj_dir = os.path.join(LIB_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "migsim_b200.h"))
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC] + FLAGS + ["-dc", "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB_PATH, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_PATH] + objs + \
              ["-Xcompiler", "-fPIC", "-cudart", "static", "-ldl"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB_PATH


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
