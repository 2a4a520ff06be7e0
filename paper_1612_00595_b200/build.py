"""Builds the engine's C-ABI shared library in-tree for sm_100a.

    python -m paper_1612_00595_b200.build

produces paper_1612_00595_b200/_lib/libseis_b200.so (nvcc cross-compiles
without a GPU). --fmad=false keeps the reference's fp64 expressions
uncontracted; FMA is used only where the kernels spell it out.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libseis_b200.so")
SOURCES = [os.path.join(CSRC, "engine.cu"), os.path.join(CSRC, "worldgen.cpp"),
           os.path.join(CSRC, "evaluation.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("engine.cuh", "kernels.cuh")] + [
    os.path.join(ROOT, "include", f) for f in ("seis_b200.h", "seis_philox.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-shared",
              "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in DEPS if os.path.exists(f))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES,
           "-lpthread"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
