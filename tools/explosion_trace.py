"""Event count per color phase of configs 3/4 at their stated k (DESIGN.md
"Configs 3 and 4"): the world streamed, the truth hypothesis loaded, then
`--epochs` sweeps in one run with a trace row after every phase.

    python tools/explosion_trace.py --config 3 --epochs 3 --capacity 4000000
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--capacity", type=int, default=4_000_000)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--storage", default="compact")
    a = ap.parse_args()
    import paper_1612_00595_b200 as E
    c = dict(bench.CONFIGS[a.config])
    if a.k:
        c["k"] = a.k
    threads = os.cpu_count() or 1
    t0 = time.time()
    m, ev, sig = bench.make_world(c, threads, streamed=bench.huge(c))
    eng = E.Engine(m, sig, event_capacity=a.capacity)
    eng.arrival_storage = a.storage
    bench.load_truth(E, eng, m, ev, threads)
    print(f"world {time.time() - t0:.1f} s, N {ev.N}, pool rows {eng.pool_slots}", flush=True)
    ncr = (c["n_regions"] + 1) // 2
    sc = E.SamplerConfig(algorithm="chromatic-dynamic" if c["dynamic"] else "chromatic-static",
                         steps_per_epoch=c["k"], epochs=a.epochs, n_regions=c["n_regions"],
                         seed=1, record_every=ncr * c["k"])
    t1 = time.time()
    try:
        tr = eng.run_chromatic(sc, final=False)
        st = tr.stats
        print(json.dumps({"config": a.config, "k": c["k"], "row_step": tr.row_step.tolist(),
                          "row_count": tr.row_count.tolist(), "wall_s": time.time() - t1,
                          "device_ms": st["total_ms"], "proposals": st["total_steps"],
                          "generated_versions": st["generated_versions"],
                          "proposals_per_s": st["total_steps"] / (st["total_ms"] / 1e3)}))
    except RuntimeError as e:
        print("failed:", e, f"after {time.time() - t1:.1f} s")


if __name__ == "__main__":
    main()
