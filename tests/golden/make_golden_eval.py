"""Golden vectors for the evaluation bridge (evaluation.hpp:51-171), produced
by the reference itself (headers compiled unchanged into oracle/_ref through
oracle/ref_shim.cpp). Run in the build container (needs /root/reference):

    python tests/golden/make_golden_eval.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    R = O.Oracle("ref")
    lib = R.lib
    boot = lib.sr_bootstrap_ci
    P = C.c_void_p
    boot.argtypes = [P, C.c_int64, C.c_double, C.c_int32, C.c_uint64, P]
    boot.restype = C.c_int
    rng = np.random.default_rng(20261019)
    save = {}
    mcases = []
    for i in range(8):
        nt = int(rng.integers(0, 160))
        tx, tt = rng.uniform(0, 100, nt), rng.uniform(0, 300, nt)
        keep = rng.random(nt) < 0.8
        ix = np.concatenate([tx[keep] + rng.normal(0, 4, keep.sum()), rng.uniform(0, 100, 20)])
        it = np.concatenate([tt[keep] + rng.normal(0, 4, keep.sum()), rng.uniform(0, 300, 20)])
        if i % 3 == 0 and nt > 4:  # exact ties in (t, x) and in distance
            ix[:3] = tx[0]
            it[:3] = tt[0]
            tx[1], tt[1] = tx[0], tt[0]
        thr = [12.0, 5.0, 30.0, 0.5][i % 4]
        ti = np.arange(nt, dtype=np.uint64) + 7
        ii = (np.arange(len(ix), dtype=np.uint64) * 3 + 1)[rng.permutation(len(ix))]
        T = O.Events(ti, tx, tt, np.zeros((nt, 1)))
        I = O.Events(ii, ix, it, np.zeros((len(ix), 1)))
        pr, rc, le, nm = R.match_events(T, I, thr)
        for k, v in (("ti", ti), ("tx", tx), ("tt", tt), ("ii", ii), ("ix", ix), ("it", it)):
            save[f"m{i}_{k}"] = v
        mcases.append((thr, pr, rc, le, nm))
    save["match"] = np.array(mcases)
    bcases = []
    for i in range(6):
        n = int(rng.integers(1, 400))
        v = rng.normal(0.7, 0.2, n)
        level = [0.95, 0.9, 0.5][i % 3]
        res = [1000, 1, 37][i % 3]
        seed = int(rng.integers(0, 1 << 62))
        out = np.zeros(4)
        assert boot(v.ctypes.data_as(P), n, level, res, seed, out.ctypes.data_as(P)) == 0
        save[f"b{i}_v"] = v
        bcases.append((level, res, seed, *out))
    save["boot"] = np.array(bcases, dtype=object).astype(np.float64)
    save["boot_seed"] = np.array([int(b[2]) for b in bcases], np.uint64)
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **save)
    print("eval.npz", os.path.getsize(os.path.join(HERE, "eval.npz")))


if __name__ == "__main__":
    main()
