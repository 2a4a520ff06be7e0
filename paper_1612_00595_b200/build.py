"""Builds the engine's C-ABI shared library in-tree for sm_100a.

    python -m paper_1612_00595_b200.build [--force] [--fast] [-DNAME=VALUE ...] [--out PATH]

produces paper_1612_00595_b200/_lib/libseis_b200.so (nvcc cross-compiles
without a GPU). --fmad=false keeps the reference's fp64 expressions
uncontracted; FMA is used only where the kernels spell it out.

The region-sweep kernel k_phase is compiled one instantiation per object
(csrc/phase_inst.cu with -DINST_*: signal type x mode x chain capacity x
version kinds x item order = 20 objects), in parallel with engine.cu and the
host C++ sources, then linked. Objects are kept under _lib/obj/<key>/ and
rebuilt only when a source they depend on is newer. --fast (development)
builds only the fp32 row-only production kernels (-DSEIS_FAST_BUILD).
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libseis_b200.so")
HEADERS = [os.path.join(CSRC, f) for f in ("engine.cuh", "kernels.cuh", "phase.cuh",
                                            "phase_api.h")] + [
    os.path.join(ROOT, "include", f) for f in ("seis_b200.h", "seis_philox.h")]
SOURCES = [os.path.join(CSRC, f) for f in ("engine.cu", "worldgen.cpp", "evaluation.cpp")]
PHASE_SRC = os.path.join(CSRC, "phase_inst.cu")
DEPS = SOURCES + [PHASE_SRC] + HEADERS

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off",
              "-Xptxas", "-warn-spills"]

MAXOWN, SERIAL_CAP = 64, 1024  # engine.cuh (checked by a static_assert in phase_inst.cu)


def phase_variants(fast: bool, maxown: int = MAXOWN):
    """(YT, MODE, CAP, GEN, TM) of every k_phase instantiation engine.cu launches"""
    out = []
    for yt in ("float",) if fast else ("float", "double"):
        for tm in (1, 0):
            out.append((yt, 0, maxown, 0, tm))
            if fast:
                continue
            for mode in (0, 1):
                out.append((yt, mode, maxown, 1, tm))
                out.append((yt, mode, SERIAL_CAP, 1, tm))
    return out


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in DEPS if os.path.exists(f))


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in deps if os.path.exists(f))


def build(force: bool = False, verbose: bool = False, defs=(), fast: bool = False,
          out: str = LIB) -> str:
    """compile (in parallel) and link; returns the library path. Spill warnings
    of ptxas are printed."""
    defs = list(defs) + (["-DSEIS_FAST_BUILD=1"] if fast else [])
    if not force and not defs and out == LIB and up_to_date():
        return LIB
    key = hashlib.sha1(" ".join(sorted(defs)).encode()).hexdigest()[:10] if defs else "default"
    objdir = os.path.join(LIBDIR, "obj", key)
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]
    jobs = []  # (object, command, deps)
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        jobs.append((obj, [nvcc(), *NVCC_FLAGS, *defs, *inc, "-c", src, "-o", obj],
                     [src] + HEADERS))
    maxown = MAXOWN
    for d_ in defs:  # -DSEIS_MAXOWN=N (A/B builds) changes the region chains' capacity
        if d_.startswith("-DSEIS_MAXOWN="):
            maxown = int(d_.split("=")[1])
    for yt, mode, cap, gen, tm in phase_variants(fast, maxown):
        obj = os.path.join(objdir, f"phase_{yt}_m{mode}_c{cap}_g{gen}_t{tm}.o")
        inst = [f"-DINST_YT={yt}", f"-DINST_MODE={mode}", f"-DINST_CAP={cap}",
                f"-DINST_GEN={gen}", f"-DINST_TM={tm}"]
        jobs.append((obj, [nvcc(), *NVCC_FLAGS, *defs, *inst, *inc, "-c", PHASE_SRC, "-o", obj],
                     [PHASE_SRC] + HEADERS))
    todo = [j for j in jobs if force or _newer(j[0], j[2])]

    def run(job):
        if verbose:
            print(" ".join(job[1]), file=sys.stderr)
        r = subprocess.run(job[1], capture_output=True, text=True)
        return job, r

    workers = max(1, min(len(todo), int(os.environ.get("SEIS_BUILD_JOBS", os.cpu_count() or 4))))
    failed = None
    if todo:
        with ThreadPoolExecutor(workers) as ex:
            for job, r in ex.map(run, todo):
                for line in r.stderr.splitlines():
                    if "spill" in line.lower() or r.returncode:
                        print(f"[{os.path.basename(job[0])}] {line}", file=sys.stderr)
                if r.returncode and failed is None:
                    failed = job
    if failed is not None:
        raise subprocess.CalledProcessError(1, failed[1])
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out,
            *[j[0] for j in jobs], "-lpthread"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    return out


if __name__ == "__main__":
    argv = sys.argv[1:]
    out_path = LIB
    if "--out" in argv:
        out_path = os.path.abspath(argv[argv.index("--out") + 1])
    print(build(force="--force" in argv, verbose="-v" in argv,
                defs=[a for a in argv if a.startswith("-D")], fast="--fast" in argv,
                out=out_path))
