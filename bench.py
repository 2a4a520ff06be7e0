#!/usr/bin/env python
"""Benchmark of the chromatic region-sweep hot path (BASELINE.json metric:
MH proposals/s and region sweeps/s on 1 B200; likelihood-delta % of roofline).

One "step" = one chromatic sweep (every color x every region x k MH steps).
The default workload is config[2] (SURVEY §8(d) 1-D mapping: S = 16384
stations, T = 3600 samples fp32, Poisson(5000) events, 4096 time regions,
k = 64, dynamic partition offsets redrawn every sweep), the largest
BASELINE config that runs at its mapped parameters on one GPU, started from
the world's truth hypothesis so every step is a steady-state sweep.

    python bench.py [--gpus N --steps K --warmup W --config C --impl ours|reference]

Timing. Configs whose inputs exceed the 126 MB L2 (2-4: >= 236 MB of
signals plus counts and arrival versions) run the K timed sweeps as one
run_chromatic call of K epochs (dynamic offsets live, as in a real run);
configs 0/1 fit in L2 and run one call per sweep with a 256 MiB L2 flush in
between. Device time from CUDA events on the engine's stream, covering every
kernel the run launches (partition, barriers, trace rows included).

--impl reference times the reference's own CPU implementation (oracle/_ref:
the reference headers compiled unchanged, run_region_steps on the truth world,
one region chain per host thread) on the same config and metric. That arm
builds its world with the reference's own generator (sr_sample_world /
sr_make_world_with_events) and never imports this package. Multi-GPU
(torchrun): independent replica chains per rank ("replicas only", weak
scaling), barrier + max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# side -> x_max, trace length -> T (1 Hz), Poisson mean -> lambda T,
# G x G stations -> S evenly spaced, R x R regions -> R^2 time regions,
# v = 1.2 x_max n_regions / T (l / tau_max = 1.2)
CONFIGS = {
    0: dict(x_max=1000.0, T=3600.0, events=20, S=100, n_regions=16, k=500, dynamic=0,
            dtype="f64", fits_l2=True,
            desc="config[0] small: 10x10 stations, 4x4 regions, fp64"),
    1: dict(x_max=4000.0, T=3600.0, events=400, S=1600, n_regions=256, k=64, dynamic=0,
            dtype="f32", fits_l2=True,
            desc="config[1] medium: 40x40 stations x 3600 fp32, 16x16 regions"),
    2: dict(x_max=16000.0, T=3600.0, events=5000, S=16384, n_regions=4096, k=64, dynamic=1,
            dtype="f32", fits_l2=False,
            desc="config[2] large: 128x128 stations x 3600 fp32, 64x64 regions, "
                 "dynamic offsets"),
    3: dict(x_max=16000.0, T=1800.0, events=20000, S=65536, n_regions=16384, k=256, dynamic=1,
            dtype="f32", fits_l2=False,
            desc="config[3] dense: 256x256 stations x 1800 fp32, 128x128 regions, "
                 "dynamic offsets"),
    4: dict(x_max=32000.0, T=1024.0, events=None, S=262144, n_regions=65536, k=64, dynamic=1,
            dtype="f32", fits_l2=False,
            desc="config[4] clustered (Thomas): 512x512 stations x 1024 fp32, "
                 "256x256 regions, dynamic offsets"),
}
DEFAULT_CONFIG = 2
METRIC = "MH proposals/sec (and region sweeps/sec) on 1 B200; likelihood-delta % of roofline"


def model_params(c):
    v = 1.2 * c["x_max"] * c["n_regions"] / c["T"]
    lam = (c["events"] or 20000) / c["T"]
    st = c["x_max"] * np.arange(c["S"], dtype=np.float64) / (c["S"] - 1)
    return dict(lambda_rate=lam, T=c["T"], x_max=c["x_max"], v=v, stations=st)


def thomas_args(c):
    return (0, c["x_max"], c["T"], 2000.0, 10.0, 50.0, 0.0015625 * c["T"])


def config_block(c, args):
    """the workload description, identical in both arms"""
    alg = "naive" if args.algorithm == "naive" else (
        "chromatic-dynamic" if c["dynamic"] else "chromatic-static")
    out = {"workload": c["desc"], "algorithm": alg,
           "start": "empty hypothesis" if args.algorithm == "naive" or args.start == "empty"
           else "truth hypothesis",
           "stations": c["S"], "samples": int(round(c["T"])), "regions": c["n_regions"],
           "k": c["k"], "signals": "fp32" if c["dtype"] == "f32" else "fp64",
           "world_seed": 0}
    if "k_mapped" in c:
        out["k_mapped"] = c["k_mapped"]
    return out


def huge(c):
    """configs whose N x S arrival matrix (10.5 GB at [3], 42 GB at [4]) is not
    materialised on the host: streamed generation and hypothesis upload"""
    return c["S"] * (c["events"] or 20000) * 8 > 4e9


def make_world(c, threads, streamed=False):
    """the config's world; streamed: events without their arrivals
    (Events.arrivals None; world_arrivals regenerates them)"""
    import paper_1612_00595_b200 as E
    m = E.ModelConfig(**model_params(c))
    dt = E.F64 if c["dtype"] == "f64" else E.F32
    if c["events"] is None:
        cx, ct = E.thomas_events(*thomas_args(c))
        if streamed:
            ev, sig = E.make_world_with_events_signals(m, cx, ct, 0, dtype=dt, threads=threads)
        else:
            ev, sig = E.make_world_with_events(m, cx, ct, 0, dtype=dt, threads=threads)
    elif streamed:
        ev, sig = E.sample_world_events(m, 0, dtype=dt, threads=threads)
    else:
        ev, sig = E.sample_world(m, 0, dtype=dt, threads=threads)
    return m, ev, sig


def load_truth(E, eng, m, ev, threads, out=None):
    """the truth hypothesis into the engine; streamed worlds regenerate the
    arrival rows chunk by chunk (into `out` when given, e.g. a pinned buffer)"""
    if ev.arrivals is not None:
        eng.set_hypothesis(ev)
        return
    S = m.n_stations()
    chunk = max(1, (512 << 20) // (8 * S))

    def rows(i0, n):
        dst = None if out is None else out[i0:i0 + n]
        return E.world_arrivals(m, 0, i0, ev.x[i0:i0 + n], ev.t[i0:i0 + n], threads, out=dst)
    eng.set_hypothesis_streamed(ev.ids, ev.x, ev.t, rows, chunk=chunk)


def sampler_for(c, seed, epochs=1, algorithm="chromatic"):
    from paper_1612_00595_b200 import SamplerConfig
    alg = "naive" if algorithm == "naive" else (
        "chromatic-dynamic" if c["dynamic"] else "chromatic-static")
    return SamplerConfig(algorithm=alg, steps_per_epoch=c["k"], epochs=epochs,
                         n_regions=c["n_regions"], seed=seed, record_every=1 << 30)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # first sample before the timed region starts
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_id):
    """DRAM bytes per k_phase launch from the committed ncu --set full capture"""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(f"config{cfg_id}")
    return None


def ref_threads(c, n_events):
    """host threads for the reference's run_region_steps: each holds a World
    copy (N S 8 arrival bytes + S n 8 signal bytes); keep them under ~120 GB"""
    per = n_events * c["S"] * 8 + c["S"] * int(round(c["T"])) * 8
    return max(1, min(os.cpu_count() or 1, int(120e9 // max(per, 1))))


def cpu_baseline_ref(c, w, seconds, threads, seed=1):
    """reference run_region_steps (oracle/_ref) on the truth world, one chain per thread."""
    from oracle import oracle as O
    s = O.Sampler(steps_per_epoch=c["k"], epochs=1, n_regions=c["n_regions"], seed=seed)
    return O.ref_bench_region_steps(w, w.events, s, threads, seconds, 1 << 40)


def oracle_world(c, ev, sig):
    """the engine-generated world as oracle inputs (the same values: the
    generator is bit-exact with the reference's; fp32 signals widened)"""
    from oracle import oracle as O
    om = O.Model(**model_params(c))
    return O.World(om, O.Events(ev.ids, ev.x, ev.t, ev.arrivals), sig.astype(np.float64))


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        return ws, rank, local, dist
    return 1, 0, 0, None


def reduce_max(dist, v):
    if dist is None:
        return v
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(dist, v):
    if dist is None:
        return v
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def run_reference(args, c, ws, rank, dist):
    """The reference arm: the reference's own CPU implementation, world from
    the reference's own generator; this package is never imported."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    if not O.have_ref():
        O.build()
    if not O.have_ref():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref (reference compiled in place) absent"}))
        return 0
    om = O.Model(**model_params(c))
    ref = O.Oracle("ref")
    t0 = time.perf_counter()
    if c["events"] is None:
        cx, ct = O.ref_thomas_events(*thomas_args(c))
        w = ref.make_world_with_events(om, cx, ct, 0)
    else:
        w = ref.sample_world(om, 0, cap=2 * c["events"] + 2048)
    if c["dtype"] == "f32":  # identical inputs: the fp32-rounded signals, widened
        w.signals = w.signals.astype(np.float32).astype(np.float64)
    gen_s = time.perf_counter() - t0
    threads = ref_threads(c, w.events.N)
    per_step = args.ref_seconds
    total_p, total_w, step_ms = 0, 0.0, []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline_ref(c, w, per_step if i >= args.warmup else min(1.0, per_step),
                             threads, seed=1 + i)
        if i >= args.warmup:
            total_p += r[0]
            total_w += r[1]
            step_ms.append(1e3 * r[1])
    value = total_p / total_w
    sample = (f"{args.steps} timed steps x {per_step:.0f} s of reference run_region_steps on "
              f"the truth world ({total_p} proposals, {threads} threads, one region chain per "
              f"thread; a step is a bounded sample of the sweep, not a whole sweep)")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "proposals/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(step_ms), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generative model sample_world, world seed 0)",
        "config": config_block(c, args),
        "detail": {"sweeps_per_s": value / (c["n_regions"] * c["k"]), "world_gen_s": gen_s,
                   "world_generator": "reference (oracle/_ref sr_sample_world / "
                                      "sr_make_world_with_events)",
                   "events": int(w.events.N),
                   "engine_imported": "paper_1612_00595_b200" in sys.modules},
        "cpu_baseline": {"value": value, "unit": "proposals/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "proposals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algorithm", default="chromatic", choices=["chromatic", "naive"],
                    help="naive: the uncolored comparison sampler (run_naive_parallel, "
                         "samplers.hpp:321-394) from the empty hypothesis")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--k", type=int, default=0,
                    help="override steps per region per sweep")
    ap.add_argument("--capacity", type=int, default=0,
                    help="event capacity (default 2N + 256; 2 M for configs 3/4)")
    ap.add_argument("--storage", default="", choices=["", "rows", "compact"],
                    help="arrival storage (default: the engine's choice, compact when the "
                         "pool cannot hold two stored rows per event)")
    ap.add_argument("--start", default="truth", choices=["truth", "empty"],
                    help="truth: steady state from the world's events (default); empty: the "
                         "reference's own start (samplers.hpp:409), the chain evolving over "
                         "the warm-up and timed sweeps (no e2e leg)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.k:
        c["k_mapped"] = c["k"]
        c["k"] = args.k
    ws, rank, local, dist = dist_init()
    if args.impl == "reference":
        return run_reference(args, c, ws, rank, dist)

    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3 (timing rules)")
    import torch
    import paper_1612_00595_b200 as E
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a GPU (the engine has no CPU fallback)")
    torch.cuda.set_device(local)
    threads = os.cpu_count() or 1
    big = huge(c)
    t_gen = time.perf_counter()
    m, ev, sig = make_world(c, threads, streamed=big)
    t_gen = time.perf_counter() - t_gen
    naive = args.algorithm == "naive"
    start = "empty" if naive else args.start
    # configs 3/4 at their k: the hypothesis swings between 4 k and 425 k events
    # from 20 k true ones (profiles/r02_explosion_config{3,4}.log),
    # so room for 2 M events (compact arrival storage: no row per event)
    cap = args.capacity or int(2_000_000 if big else max(1024, ev.N * 2 + 256))
    eng = E.Engine(m, sig, event_capacity=cap)
    if args.storage:
        eng.arrival_storage = args.storage
    truth = E.Events(ev.ids, ev.x, ev.t, ev.arrivals)
    empty = E.Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0), np.zeros((0, c["S"])))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    seed0 = 1000 * rank
    per_sweep = c["fits_l2"] and not naive

    def run(seed, epochs):
        return eng.run_chromatic(sampler_for(c, seed, epochs, args.algorithm), final=False,
                                 row_cap=4)

    if start == "truth":
        load_truth(E, eng, m, ev, threads)
    # warm-up: W sweeps (one call per sweep for the L2-resident configs)
    if per_sweep:
        for i in range(args.warmup):
            run(seed0 + i, 1)
    else:
        run(seed0, args.warmup)
        if naive:
            eng.set_hypothesis(empty)
    torch.cuda.synchronize()
    acc = dict(total_ms=0.0, sweep_ms=0.0, bytes=0.0, steps=0, scored=0, launches=0,
               changed=0, arrvals=0, phases=0, accepted=0, spec=0)

    def add(st):
        acc["total_ms"] += st["total_ms"]
        acc["sweep_ms"] += st["sweep_kernel_ms"]
        acc["bytes"] += st["algorithmic_bytes"]
        acc["steps"] += st["total_steps"]
        acc["scored"] += st["scored_proposals"]
        acc["launches"] += st["kernel_launches"]
        acc["changed"] += st["changed_samples"]
        acc["arrvals"] += st["arrival_values"]
        acc["accepted"] += st["total_accepted"]
        acc["spec"] += st["speculative_discarded"]
        acc["phases"] += st["phases"]
        acc["final_events"] = st["final_events"]
        acc["gen"] = st["generated_versions"]

    barrier(dist)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        if per_sweep:
            for i in range(args.steps):
                flush.zero_()  # L2 flush between timed sweeps (256 MiB > 126 MB L2)
                torch.cuda.synchronize()
                add(run(seed0 + args.warmup + i, 1).stats)
        else:
            add(run(seed0 + 1, args.steps).stats)
    torch.cuda.synchronize()
    barrier(dist)
    t_max = reduce_max(dist, acc["total_ms"])
    steps_all = reduce_sum(dist, acc["steps"])
    value = steps_all / (t_max / 1e3)
    peak, peak_kind = peaks()
    achieved = acc["bytes"] / (acc["sweep_ms"] / 1e3) / 1e9
    nph = max(1, acc["phases"])
    res = {
        "metric": METRIC, "value": value, "unit": "proposals/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generative model sample_world, world seed 0; "
                f"{'fp32' if c['dtype'] == 'f32' else 'fp64'} signals)",
        "config": config_block(c, args),
        "detail": {"sweeps_per_s": ws * args.steps / (t_max / 1e3),
                   "scored_proposals_per_s": reduce_sum(dist, acc["scored"]) / (t_max / 1e3),
                   "parallelism": "replicas" if ws > 1 else "single",
                   "events": int(ev.N), "final_events": int(acc.get("final_events", 0)),
                   "event_capacity": cap, "arrival_storage": eng.arrival_storage,
                   "pool_slots": int(eng.pool_slots),
                   "generated_versions_after": int(acc.get("gen", 0)),
                   "world_generation_s": t_gen,
                   "world_generation": "streamed (no N x S arrival matrix on the host)"
                                       if big else "in memory",
                   "timing": ("one call per sweep, L2 flushed between timed sweeps (256 MiB "
                              "write)" if per_sweep else
                              f"one call of {args.steps} epochs; inputs larger than L2 "
                              f"({sig.nbytes / 1e6:.0f} MB signals + counts + arrival versions)"),
                   "sweep_kernel_ms_per_step": acc["sweep_ms"] / args.steps,
                   "acceptance": acc["accepted"] / max(1, acc["steps"]),
                   "speculative_discarded_frac": acc["spec"] / max(1, acc["steps"]),
                   "dtype_note": "scoring arithmetic fp64 over fp32 signals / uint16 counts"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                     "peak_kind": peak_kind, "kernel": "k_phase (region sweep, fused delta)",
                     "bytes_per_launch": acc["bytes"] / nph,
                     "avg_launch_ms": acc["sweep_ms"] / nph, "launches": acc["phases"]},
        "gpu_launches": int(acc["launches"]),
    }
    res["clocks"] = clk.summary()
    # e2e through the C-ABI with host buffers: per step upload the observed
    # signals from pinned memory, load the start hypothesis, one sweep, read
    # the final hypothesis back
    if not args.no_e2e and start == "truth":
        pin = torch.empty(sig.size * sig.itemsize, dtype=torch.uint8, pin_memory=True)
        pin_np = pin.numpy().view(sig.dtype).reshape(sig.shape)
        pin_np[...] = sig
        eng.upload_signals(pin_np)

        def pinned(shape, dtype):
            nb = int(np.prod(shape)) * np.dtype(dtype).itemsize
            t_ = torch.empty(max(nb, 1), dtype=torch.uint8, pin_memory=True)
            return t_.numpy()[:nb].view(dtype).reshape(shape)
        S_ = c["S"]
        p_in = E.Events(pinned((ev.N,), np.uint64), pinned((ev.N,), np.float64),
                        pinned((ev.N,), np.float64), pinned((ev.N, S_), np.float64))
        p_in.ids[...] = truth.ids
        p_in.x[...] = truth.x
        p_in.t[...] = truth.t
        if truth.arrivals is not None:
            p_in.arrivals[...] = truth.arrivals
        else:  # streamed world: the truth's arrivals generated into the pinned buffer
            ch = max(1, (512 << 20) // (8 * S_))
            for i0 in range(0, ev.N, ch):
                n_ = min(ch, ev.N - i0)
                E.world_arrivals(m, 0, i0, ev.x[i0:i0 + n_], ev.t[i0:i0 + n_], threads,
                                 out=p_in.arrivals[i0:i0 + n_])
        # the result read back every step: the final hypothesis with its
        # arrivals (configs 0-2), or its events (id, x, t) for the streamed
        # configs, whose arrivals stay on the device
        out_arr = not big
        ocap = min(cap, 2 * ev.N + 1024) if out_arr else cap
        p_out = E.Events(pinned((ocap,), np.uint64), pinned((ocap,), np.float64),
                         pinned((ocap,), np.float64),
                         pinned((ocap, S_), np.float64) if out_arr else None)
        h2d = sig.nbytes + ev.N * (24 + 8 * S_)
        d2h = 0
        e2e_steps = max(3, min(args.steps, 10)) if not big else 3

        def e2e_step(i):
            eng.upload_signals(pin_np)
            eng.set_hypothesis(p_in)
            tr = run(seed0 + 500 + i, 1)
            try:
                fin = eng.get_hypothesis(arrivals=out_arr, out=p_out)
            except ValueError:  # the hypothesis outgrew the pinned buffer
                fin = eng.get_hypothesis(arrivals=out_arr)
            return tr.total_steps, len(fin.ids)

        e2e_step(-1)  # untimed: the engine's per-call scratch reaches its size
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        props = 0
        for i in range(e2e_steps):
            n_steps, n_final = e2e_step(i)
            props += n_steps
            d2h = n_final * (24 + (8 * S_ if out_arr else 0))
        torch.cuda.synchronize()
        wall = reduce_max(dist, time.perf_counter() - t0)
        res["e2e"] = {"value": reduce_sum(dist, props) / wall, "unit": "proposals/s",
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "path": "seis_upload_signals + seis_set_hypothesis + seis_run_chromatic "
                              "(one sweep) + seis_get_hypothesis"
                              + ("" if out_arr else " (id, x, t; arrivals stay on the device)")
                              + ", pinned host buffers, wall clock"}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and start == "truth":
        from oracle import oracle as O
        if O.have_ref():
            if ev.arrivals is None:  # streamed world: the truth's arrivals regenerated
                ev = E.Events(ev.ids, ev.x, ev.t,
                              E.world_arrivals(m, 0, 0, ev.x, ev.t, threads))
            ow = oracle_world(c, ev, sig)
            th = ref_threads(c, ev.N)
            r = cpu_baseline_ref(c, ow, args.cpu_seconds, th)
            res["cpu_baseline"] = {
                "value": r[0] / r[1], "unit": "proposals/s", "cores": th, "kind": "reference",
                "sample": f"{r[0]} proposals in {r[1]:.1f} s: reference run_region_steps on the "
                          f"truth world, one region chain per thread ({th} threads)"}
        else:
            res["cpu_baseline"] = None
    if rank == 0:
        print(json.dumps(res))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
