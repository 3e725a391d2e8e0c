"""Build the sm_100a shared library libfcm_mg.so in-tree with nvcc (no torch types,
plain C ABI from include/fcm_mg.h).  Usage: python -m paper_2010_00881_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfcm_mg.so")
SOURCES = [os.path.join(HERE, "csrc", f)
           for f in ("fcm_mg.cu", "hpmg.cu", "quad.cu", "gen.cpp", "gen_hp.cpp", "slab.cpp")]
OBJDIR = os.path.join(HERE, "csrc", "_obj")
HEADERS = sorted(os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
                 if f.endswith((".cuh", ".hpp", ".h"))) + [os.path.join(ROOT, "include", "fcm_mg.h")]


FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-O3"]


def nvcc_cmd(out=LIB, extra=()):
    """One-shot command (all sources, used by tools that want a variant build)."""
    return ["nvcc", *FLAGS, "-shared", "-o", out, *SOURCES, "-lgomp", *extra]


def _obj(src):
    return os.path.join(OBJDIR, os.path.basename(src) + ".o")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = True) -> str:
    """Compile every translation unit to an object in parallel (nvcc -c, sm_100a), then link the
    shared library."""
    if force or stale():
        from concurrent.futures import ThreadPoolExecutor
        os.makedirs(OBJDIR, exist_ok=True)
        hdr_t = max(os.path.getmtime(f) for f in HEADERS)

        def compile_one(src):
            o = _obj(src)
            if not force and os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(src), hdr_t):
                return
            cmd = ["nvcc", *FLAGS, "-c", "-o", o, src]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True, cwd=HERE)

        with ThreadPoolExecutor(len(SOURCES)) as ex:
            list(ex.map(compile_one, SOURCES))
        cmd = ["nvcc", *FLAGS, "-shared", "-o", LIB, *[_obj(s) for s in SOURCES], "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
