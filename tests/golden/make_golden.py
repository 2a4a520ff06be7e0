"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference headers compiled in place). Run in the container that holds
/root/reference:  python tests/golden/make_golden.py

Every fixture is seeded and small; the GPU box never needs /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def main():
    O.build()
    assert O.have_ref(), "needs oracle/_ref (reference tree present)"
    R = O.Oracle("ref")
    out = {}
    # --- partition KATs (test_partition.cpp:11-140 cases + a grid)
    cases = [(240, 60, 0, 50), (240, 60, 25, 50), (240, 240, 0, 50), (240, 30, 0, 50),
             (240, 20, 0, 50), (240, 0, 0, 50), (240, 300, 0, 50), (240, 60, 60, 50),
             (240, 60, -1, 50)]
    rng = np.random.default_rng(7)
    for _ in range(60):
        T = float(rng.choice([240.0, 3600.0, 1800.0, 1024.0]))
        nr = int(rng.choice([4, 16, 256, 64, 7, 13]))
        l = T / nr
        tau = l / float(rng.choice([1.2, 1.0, 1.7, 2.5, 0.9]))
        u = float(rng.uniform(0, l)) if rng.uniform() < 0.6 else 0.0
        cases.append((T, l, u, tau))
    P = []
    for (T, l, u, tau) in cases:
        rc, msg, b, c, k = R.partition(T, l, u, tau)
        probes = []
        if rc == 0:
            probes = list(b) + list((b[:-1] + b[1:]) / 2) + [np.nextafter(v, -1) for v in b[1:]]
            probes = [p for p in probes if 0 <= p <= T]
        regs = [R.region_of(b, p) for p in probes] if rc == 0 else []
        P.append(dict(T=T, l=l, u=u, tau=tau, rc=rc, b=b, c=c, k=k,
                      probes=np.array(probes), regions=np.array(regs, np.int64)))
    np.savez_compressed(os.path.join(HERE, "partition.npz"),
                        cases=np.array([(p["T"], p["l"], p["u"], p["tau"]) for p in P]),
                        rc=np.array([p["rc"] for p in P]),
                        k=np.array([p["k"] for p in P]),
                        **{f"b{i}": p["b"] for i, p in enumerate(P) if p["rc"] == 0},
                        **{f"c{i}": p["c"] for i, p in enumerate(P) if p["rc"] == 0},
                        **{f"probe{i}": p["probes"] for i, p in enumerate(P) if p["rc"] == 0},
                        **{f"reg{i}": p["regions"] for i, p in enumerate(P) if p["rc"] == 0})
    # --- offsets (samplers.hpp:488-491)
    offs = np.array([[R.partition_offset(seed, ep, l) for ep in range(1, 20)]
                     for seed, l in [(0, 60.0), (1, 14.0625), (123456789, 0.87890625)]])
    # --- rng streams
    import ctypes as C
    L = R.lib
    L.sr_derive_draws.argtypes = [C.c_uint64] * 5 + [C.c_int64, C.c_void_p, C.c_void_p,
                                                      C.c_uint64, C.c_void_p]
    uni, nor, idx = [], [], []
    for key in [(0, 5, 0, 0, 0), (1, 5, 3, 1, 7), (2024, 2, 11, 0, 0), (44, 4, 3, 0, 0)]:
        u = np.zeros(64)
        n = np.zeros(64)
        ix = np.zeros(64, np.uint64)
        L.sr_derive_draws(*key, 64, u.ctypes.data, n.ctypes.data, 1000003, ix.ctypes.data)
        uni.append(u)
        nor.append(n)
        idx.append(ix)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), offsets=offs, uniforms=np.array(uni),
                        normals=np.array(nor), indices=np.array(idx))
    # --- worlds (worldgen.hpp:20-86): reference default model, seeds 0..3; a
    # wider mapped world; a planted world
    m = O.Model()
    worlds = {}
    for seed in range(4):
        w = R.sample_world(m, seed)
        worlds[f"w{seed}"] = w
    mw = O.Model(lambda_rate=40 / 900.0, T=900.0, x_max=400.0, v=400.0 * 16 / 900.0 * 1.2,
                 stations=O.stations_line(64, 400.0))
    wide = R.sample_world(mw, 5)
    planted = R.make_world_with_events(m, [20.0, 80.0, 50.0], [30.0, 100.0, 190.0], 9)
    save = {}
    for name, w in list(worlds.items()) + [("wide", wide), ("planted", planted)]:
        save[f"{name}_ids"] = w.events.ids
        save[f"{name}_x"] = w.events.x
        save[f"{name}_t"] = w.events.t
        save[f"{name}_arr"] = w.events.arr
        save[f"{name}_sig"] = w.signals
    save["wide_model"] = np.array([mw.lambda_rate, mw.T, mw.x_max, mw.v])
    np.savez_compressed(os.path.join(HERE, "worlds.npz"), **save)
    # --- deltas on random changes (test_model.cpp:309-348 style) on the wide world
    drng = np.random.default_rng(2024)
    ev = wide.events
    D = []
    for i in range(300):
        pick = drng.uniform()
        if pick < 0.34:
            x, t = drng.uniform(0, mw.x_max), drng.uniform(0, mw.T)
            a = np.array([t + abs(x - s) / mw.v for s in mw.stations]) + drng.normal(0, 2, mw.S)
            rem, add = [], [(10000 + i, x, t, a)]
        elif pick < 0.67:
            rem, add = [int(drng.integers(ev.N))], []
        else:
            j = int(drng.integers(ev.N))
            x = ev.x[j] + drng.normal(0, 5)
            t = ev.t[j] + drng.normal(0, 5)
            a = ev.arr[j] + drng.normal(0, 30 if drng.uniform() < 0.3 else 1, mw.S)
            rem, add = [j], [(int(ev.ids[j]), x, t, a)]
        added = O.Events(np.array([q[0] for q in add], np.uint64), np.array([q[1] for q in add]),
                         np.array([q[2] for q in add]),
                         np.array([q[3] for q in add]).reshape(len(add), mw.S))
        d = R.delta(mw, wide.signals, ev, rem, added)
        D.append((rem, add, d))
    np.savez_compressed(
        os.path.join(HERE, "deltas.npz"),
        n_rem=np.array([len(r) for r, _, _ in D]), rem=np.array([r[0] if r else -1 for r, _, _ in D]),
        n_add=np.array([len(a) for _, a, _ in D]),
        add_id=np.array([a[0][0] if a else 0 for _, a, _ in D], np.uint64),
        add_x=np.array([a[0][1] if a else 0.0 for _, a, _ in D]),
        add_t=np.array([a[0][2] if a else 0.0 for _, a, _ in D]),
        add_arr=np.array([a[0][3] if a else np.zeros(mw.S) for _, a, _ in D]),
        delta=np.array([d for _, _, d in D]),
        log_joint=np.array([R.log_joint(mw, wide.signals, ev)]))
    # --- chromatic tapes (run_chromatic through the reference's functions)
    for name, world, model, sc in [
            ("default_static", worlds["w1"], m,
             O.Sampler(steps_per_epoch=100, epochs=6, n_regions=4, seed=3, dynamic=0)),
            ("default_dynamic", worlds["w2"], m,
             O.Sampler(steps_per_epoch=100, epochs=6, n_regions=4, seed=4, dynamic=1)),
            ("wide_dynamic", wide, mw,
             O.Sampler(steps_per_epoch=32, epochs=4, n_regions=16, seed=5, dynamic=1))]:
        r = R.run_chromatic(world, sc, tape=True, rowlj=True)
        np.savez_compressed(os.path.join(HERE, f"tape_{name}.npz"), tape=r["tape"],
                            tape_arr=r["tape_arr"], row_step=r["row_step"], row_lj=r["row_lj"],
                            row_count=r["row_count"], final_ids=r["final"].ids,
                            final_x=r["final"].x, final_t=r["final"].t,
                            final_arr=r["final"].arr, total_steps=r["total_steps"],
                            total_accepted=r["total_accepted"],
                            sampler=np.array([sc.steps_per_epoch, sc.epochs, sc.n_regions,
                                              sc.seed, sc.dynamic]))
    # --- posterior statistics of the reference's own run_sampler
    # (chromatic-dynamic from empty; acceptance.cpp:154-194 style), final
    # hypothesis matched to the truth with match_events (evaluation.hpp:51-103)
    post = []
    for ws in range(8):
        w = R.sample_world(m, 300 + ws)
        for rs in (1, 2, 3):
            sc = O.Sampler(steps_per_epoch=500, epochs=40, n_regions=4, seed=rs, dynamic=1,
                           burn_in_fraction=0.0, record_every=1 << 30)
            r = O.ref_run_sampler(w, sc, workers=1)
            pr, rc, le, nm = R.match_events(w.events, r["final"])
            post.append((300 + ws, rs, pr, rc, le, r["final"].N, w.events.N,
                         r["total_accepted"]))
    # naive-parallel comparison (samplers.hpp:321-394) on the same worlds
    for ws in range(8):
        w = R.sample_world(m, 300 + ws)
        for rs in (1, 2, 3):
            sc = O.Sampler(steps_per_epoch=500, epochs=40, n_regions=4, seed=rs,
                           burn_in_fraction=0.0, record_every=1 << 30)
            r = O.ref_run_sampler(w, sc, workers=1, naive=True)
            pr, rc, le, nm = R.match_events(w.events, r["final"])
            post.append((1000 + 300 + ws, rs, pr, rc, le, r["final"].N, w.events.N,
                         r["total_accepted"]))
    np.savez_compressed(os.path.join(HERE, "posterior.npz"), rows=np.array(post, np.float64),
                        cols=np.array(["world_seed", "run_seed", "precision", "recall",
                                       "location_error", "n_final", "n_true", "accepted"]),
                        sampler=np.array([500, 40, 4, 1]))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
