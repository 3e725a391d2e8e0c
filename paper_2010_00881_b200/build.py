"""Build the sm_100a shared library libfcm_mg.so in-tree with nvcc (no torch types,
plain C ABI from include/fcm_mg.h).  Usage: python -m paper_2010_00881_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfcm_mg.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("fcm_mg.cu", "quad.cu", "gen.cpp", "slab.cpp")]
HEADERS = sorted(os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                 if f.endswith((".cuh", ".hpp", ".h"))) + [os.path.join(ROOT, "include", "fcm_mg.h")]


def nvcc_cmd(out=LIB, extra=()):
    return ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
            "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-O3", "-shared", "-o", out,
            *SOURCES, "-lgomp", *extra]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = True) -> str:
    if force or stale():
        cmd = nvcc_cmd()
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
