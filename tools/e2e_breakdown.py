"""Wall-clock breakdown of bench.py's e2e step (config[1]) into its four C-ABI calls.

    gpurun -- python tools/e2e_breakdown.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_1612_00595_b200 as E  # noqa: E402


def pinned(shape, dtype):
    nb = int(np.prod(shape)) * np.dtype(dtype).itemsize
    t_ = torch.empty(max(nb, 1), dtype=torch.uint8, pin_memory=True)
    return t_.numpy()[:nb].view(dtype).reshape(shape)


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    c = dict(bench.CONFIGS[cfg])
    m, ev, sig = bench.make_world(c, os.cpu_count() or 1)
    cap = int(max(1024, ev.N * 2 + 256))
    eng = E.Engine(m, sig, event_capacity=cap)
    pin = pinned(sig.shape, sig.dtype)
    pin[...] = sig
    S = c["S"]
    p_in = E.Events(pinned((ev.N,), np.uint64), pinned((ev.N,), np.float64),
                    pinned((ev.N,), np.float64), pinned((ev.N, S), np.float64))
    p_in.ids[...] = ev.ids
    p_in.x[...] = ev.x
    p_in.t[...] = ev.t
    p_in.arrivals[...] = ev.arrivals
    ocap = min(cap, 2 * ev.N + 1024)
    p_out = E.Events(pinned((ocap,), np.uint64), pinned((ocap,), np.float64),
                     pinned((ocap,), np.float64), pinned((ocap, S), np.float64))
    names = ["upload_signals", "set_hypothesis", "run_chromatic", "get_hypothesis"]
    acc = {k: [] for k in names}
    dev = []
    for i in range(13):
        t = [time.perf_counter()]
        eng.upload_signals(pin)
        t.append(time.perf_counter())
        eng.set_hypothesis(p_in)
        t.append(time.perf_counter())
        tr = eng.run_chromatic(bench.sampler_for(c, 500 + i), final=False, row_cap=4)
        t.append(time.perf_counter())
        eng.get_hypothesis(out=p_out)
        t.append(time.perf_counter())
        if i >= 3:
            for k, a, b in zip(names, t, t[1:]):
                acc[k].append((b - a) * 1e3)
            dev.append(tr.stats["total_ms"])
    tot = 0.0
    for k in names:
        v = float(np.median(acc[k]))
        tot += v
        print(f"{k:16s} {v:8.3f} ms")
    print(f"{'sum':16s} {tot:8.3f} ms; run_chromatic device total_ms {np.median(dev):.3f}")
    print(f"signals {sig.nbytes / 1e6:.1f} MB, arrivals in {ev.N * S * 8 / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
