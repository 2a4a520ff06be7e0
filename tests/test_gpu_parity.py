"""GPU parity: the B200 engine (through its C-ABI) against the reference's
golden vectors and the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): region assignment, coloring and replay
accept/reject decisions bit-exact except where |log alpha - log u| < 1e-9;
per-proposal deltas within 1e-5 relative (asserted here much tighter, 1e-9);
production trajectories identical to the oracle's philox-spec replay.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import (default_model, engine_model, engine_sampler, golden, golden_world,
                           tape_sampler, wide_model)

pytestmark = pytest.mark.gpu

TIE = 1e-9
DTOL = 1e-9


@pytest.fixture(scope="module")
def E(built):
    import paper_1612_00595_b200 as E
    return E


@pytest.fixture(scope="module")
def oc(built):
    return O.Oracle("c")


def close(a, b, tol=DTOL):
    if np.isinf(a) or np.isinf(b):
        return a == b
    return abs(a - b) <= tol * max(1.0, abs(b))


# ------------------------------------------------------------------ partition
def test_partition_bit_exact(E):
    g = golden("partition.npz")
    for i, (T, l, u, tau) in enumerate(g["cases"]):
        if g["rc"][i]:
            with pytest.raises(ValueError):
                E.partition(T, l, u, tau)
            continue
        p = E.partition(T, l, u, tau)
        assert np.array_equal(p.boundaries, g[f"b{i}"]), i
        assert np.array_equal(p.colors, g[f"c{i}"]) and p.n_colors == g["k"][i]


def test_region_of_bit_exact(E):
    g = golden("partition.npz")
    for i in range(len(g["rc"])):
        if g["rc"][i] or len(g[f"probe{i}"]) == 0:
            continue
        got = E.assign_regions(g[f"b{i}"], g[f"probe{i}"])
        assert np.array_equal(got, g[f"reg{i}"]), i


def test_partition_offsets(E):
    g = golden("rng.npz")
    for r, (seed, l) in enumerate([(0, 60.0), (1, 14.0625), (123456789, 0.87890625)]):
        got = [E.partition_offset(seed, ep, l) for ep in range(1, 20)]
        assert np.array_equal(got, g["offsets"][r])


# ------------------------------------------------------------------ delta
def _golden_changes(m):
    g = golden("deltas.npz")
    w = golden_world("wide", m)
    out = []
    for i in range(len(g["delta"])):
        rem = [int(w.events.ids[g["rem"][i]])] if g["n_rem"][i] else []
        add = [(g["add_x"][i], g["add_t"][i], g["add_arr"][i])] if g["n_add"][i] else []
        out.append((rem, add))
    return w, out, g["delta"]


def test_score_batch_matches_reference_fp64(E):
    m = wide_model()
    w, changes, ref = _golden_changes(m)
    eng = E.Engine(engine_model(m), w.signals, event_capacity=256)
    eng.set_hypothesis(E.Events(w.events.ids, w.events.x, w.events.t, w.events.arr))
    got = eng.delta_log_joint(changes)
    bad = [(i, got[i], ref[i]) for i in range(len(ref)) if not close(got[i], ref[i])]
    assert not bad, bad[:5]
    assert close(eng.log_joint(), golden("deltas.npz")["log_joint"][0], 1e-12)


def test_score_batch_fp32_signals_vs_oracle(E, oc):
    m = wide_model()
    w, changes, _ = _golden_changes(m)
    sig32 = w.signals.astype(np.float32)
    eng = E.Engine(engine_model(m), sig32, event_capacity=256)
    eng.set_hypothesis(E.Events(w.events.ids, w.events.x, w.events.t, w.events.arr))
    got = eng.delta_log_joint(changes)
    sig = sig32.astype(np.float64)  # identical inputs: the widened fp32 values
    idx = {int(v): i for i, v in enumerate(w.events.ids)}
    for i, (rem, add) in enumerate(changes):
        a = None
        if add:
            a = O.Events(np.array([7], np.uint64), np.array([add[0][0]]), np.array([add[0][1]]),
                         np.array(add[0][2])[None, :])
        ref = oc.delta(m, sig, w.events, [idx[r] for r in rem], a)
        assert close(got[i], ref), (i, got[i], ref)


def test_score_batch_restricted_window_and_support(E, oc):
    m = wide_model()
    w, changes, _ = _golden_changes(m)
    eng = E.Engine(engine_model(m), w.signals, event_capacity=256)
    eng.set_hypothesis(E.Events(w.events.ids, w.events.x, w.events.t, w.events.arr))
    idx = {int(v): i for i, v in enumerate(w.events.ids)}
    win, sup = (100, 500), (50.0, 400.0, 0)  # naive-mode style ScoreOptions
    got = eng.delta_log_joint(changes[:80], window=win, support=sup)
    for i, (rem, add) in enumerate(changes[:80]):
        a = None
        if add:
            a = O.Events(np.array([7], np.uint64), np.array([add[0][0]]), np.array([add[0][1]]),
                         np.array(add[0][2])[None, :])
        ref = oc.delta(m, w.signals, w.events, [idx[r] for r in rem], a, window=win, support=sup)
        assert close(got[i], ref), (i, got[i], ref)


def test_score_batch_empty_world_and_unknown_id(E):
    m = default_model()
    g = golden_world("w0", m)
    eng = E.Engine(engine_model(m), g.signals)
    d = eng.delta_log_joint([([], [(10.0, 30.0, 30.0 + np.abs(10.0 - m.stations) / m.v)])])
    assert np.isfinite(d[0])
    with pytest.raises(ValueError):
        eng.delta_log_joint([([12345], [])])


# ------------------------------------------------------------------ replay
def _replay_check(E, world, model, tape, tape_arr, sampler, final, dtype=np.float64):
    eng = E.Engine(engine_model(model), world.signals.astype(dtype), event_capacity=512)
    tr = eng.run_chromatic(engine_sampler(sampler), tape=tape, tape_arrivals=tape_arr)
    out = tr.step_out
    scored = tape["scored"] == 1
    assert np.array_equal(out["scored"], tape["scored"])
    # decisions: bit-exact except near ties |log alpha - log u| < 1e-9
    lr = tape["log_r"]
    tie = np.zeros(len(tape), bool)
    drawn = tape["u_drawn"] == 1
    tie[drawn] = np.abs(lr[drawn] - np.log(tape["u"][drawn])) < TIE
    tie |= scored & (np.abs(lr) < TIE)
    mism = (out["accepted"] != tape["accepted"]) & ~tie
    assert not mism.any(), np.where(mism)[0][:10]
    for i in np.where(scored)[0]:
        assert close(out["delta"][i], tape["delta"][i]), (i, out["delta"][i], tape["delta"][i])
        assert close(out["log_r"][i], tape["log_r"][i]), i
    fin = tr.final
    assert np.array_equal(fin.ids, final["ids"])
    assert np.array_equal(fin.x, final["x"]) and np.array_equal(fin.t, final["t"])
    assert np.array_equal(fin.arrivals, final["arr"])
    return tr


@pytest.mark.parametrize("name", ["default_static", "default_dynamic", "wide_dynamic"])
def test_replay_golden_tapes(E, name):
    g = golden(f"tape_{name}.npz")
    s = tape_sampler(g["sampler"])
    if name.startswith("default"):
        m = default_model()
        w = golden_world("w1" if "static" in name else "w2", m)
    else:
        m = wide_model()
        w = golden_world("wide", m)
    _replay_check(E, w, m, g["tape"], g["tape_arr"], s,
                  dict(ids=g["final_ids"], x=g["final_x"], t=g["final_t"], arr=g["final_arr"]))


def _mapped_model(S, T, n_regions, x_max, lam_events):
    # SURVEY §8(d) mapping: l / tau = 1.2
    v = 1.2 * x_max * n_regions / T
    return O.Model(lambda_rate=lam_events / T, T=T, x_max=x_max, v=v,
                   stations=O.stations_line(S, x_max))


def test_replay_fp32_mapped_world(E, oc):
    # a config[1]-shaped slice small enough for the O(S N) oracle: fp32 signals,
    # overlapping same-color windows (tau + t_s > l) exercise the frozen snapshot
    m = _mapped_model(S=96, T=600.0, n_regions=40, x_max=4000.0, lam_events=60)
    w = oc.sample_world(m, 3)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=16, epochs=3, n_regions=40, seed=9, dynamic=1)
    r = oc.run_chromatic(w32, s, init=w.events, tape=True)
    eng = E.Engine(engine_model(m), w32.signals.astype(np.float32), event_capacity=1024)
    eng.set_hypothesis(E.Events(w.events.ids, w.events.x, w.events.t, w.events.arr))
    tr = eng.run_chromatic(engine_sampler(s), tape=r["tape"], tape_arrivals=r["tape_arr"])
    t = r["tape"]
    drawn = t["u_drawn"] == 1
    tie = np.zeros(len(t), bool)
    tie[drawn] = np.abs(t["log_r"][drawn] - np.log(t["u"][drawn])) < TIE
    assert not ((tr.step_out["accepted"] != t["accepted"]) & ~tie).any()
    sc = t["scored"] == 1
    assert np.allclose(tr.step_out["delta"][sc], t["delta"][sc], rtol=1e-11, atol=1e-9)
    assert np.array_equal(tr.final.ids, r["final"].ids)
    assert np.array_equal(tr.final.arrivals, r["final"].arr)


# ------------------------------------------------------------------ production
def _decisions_match(so, t, rtol):
    """per-step production decisions (driver order) vs the oracle's tape"""
    assert len(so) == len(t)
    assert np.array_equal(so["accepted"], t["accepted"])
    assert np.array_equal(so["scored"] != 0, t["scored"] == 1)
    sc = t["scored"] == 1
    fin = sc & np.isfinite(t["delta"])
    assert np.array_equal(np.isfinite(so["delta"][sc]), np.isfinite(t["delta"][sc]))
    assert np.allclose(so["delta"][fin], t["delta"][fin], rtol=rtol, atol=1e-9)


def _prod_vs_oracle(E, oc, m, w, s, init=None, dtype=np.float64, rowlj=False):
    ro = oc.run_chromatic(w, s, init=init, tape=True, rowlj=rowlj)
    eng = E.Engine(engine_model(m), w.signals.astype(dtype), event_capacity=2048)
    if init is not None:
        eng.set_hypothesis(E.Events(init.ids, init.x, init.t, init.arr))
    tr = eng.run_chromatic(engine_sampler(s, record_log_joint=rowlj), decisions=len(ro["tape"]))
    _decisions_match(tr.step_out, ro["tape"], 1e-11 if dtype == np.float64 else 1e-5)
    assert tr.total_steps == ro["total_steps"]
    assert tr.total_accepted == ro["total_accepted"]
    assert np.array_equal(tr.final.ids, ro["final"].ids)
    assert np.array_equal(tr.final.x, ro["final"].x)
    assert np.array_equal(tr.final.t, ro["final"].t)
    assert np.array_equal(tr.final.arrivals, ro["final"].arr)
    assert np.array_equal(tr.row_step, ro["row_step"])
    assert np.array_equal(tr.row_count, ro["row_count"])
    if rowlj:
        assert np.allclose(tr.row_log_joint, ro["row_lj"], rtol=1e-12, atol=1e-8)
    return tr, ro


@pytest.mark.parametrize("dyn", [0, 1])
def test_production_matches_oracle_philox_default(E, oc, dyn):
    m = default_model()
    w = golden_world("w3", m)
    s = O.Sampler(steps_per_epoch=100, epochs=12, n_regions=4, seed=17, dynamic=dyn,
                  rng_mode=1, record_every=400)
    _prod_vs_oracle(E, oc, m, w, s, rowlj=True)


def test_production_matches_oracle_philox_mapped_fp32(E, oc):
    m = _mapped_model(S=96, T=600.0, n_regions=40, x_max=4000.0, lam_events=60)
    w = oc.sample_world(m, 4)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=16, epochs=4, n_regions=40, seed=3, dynamic=1, rng_mode=1)
    _prod_vs_oracle(E, oc, m, w32, s, init=w.events, dtype=np.float32)


def test_production_from_empty_three_colors(E, oc):
    # l in [tau/2, tau): three colors (partition.hpp:68-71)
    m = O.Model(lambda_rate=0.03, T=300.0, x_max=100.0, v=2.0 * 1.5, stations=O.stations_line(8, 100.0))
    w = oc.sample_world(m, 8)
    s = O.Sampler(steps_per_epoch=60, epochs=6, n_regions=12, seed=5, dynamic=1, rng_mode=1)
    _prod_vs_oracle(E, oc, m, w, s)


def test_sampler_validation_errors(E):
    m = default_model()
    g = golden_world("w0", m)
    eng = E.Engine(engine_model(m), g.signals)
    with pytest.raises(ValueError):
        eng.run_chromatic(E.SamplerConfig(steps_per_epoch=0))
    with pytest.raises(ValueError):
        eng.run_chromatic(E.SamplerConfig(weights=(0.5, 0.5, 0.5, 0.0, 0.0)))
    with pytest.raises(ValueError):  # l < tau / 2
        eng.run_chromatic(E.SamplerConfig(n_regions=12))
    with pytest.raises(ValueError):
        E.Engine(engine_model(O.Model(var_event=0.5)), g.signals)


# ------------------------------------------------------------------ posterior
def test_posterior_statistics_within_seed_spread(E, oc):
    """north_star: posterior precision, recall and mean location error agree
    with the reference within seed-to-seed spread. Reference numbers: the
    reference's own run_sampler (tests/golden/posterior.npz, 8 worlds x 3
    seeds); engine: production mode (philox stream) on the same worlds, 6
    seeds each."""
    g = golden("posterior.npz")
    rows = g["rows"][g["rows"][:, 0] < 1000]
    k, ep, nr, dyn = [int(v) for v in g["sampler"]]
    m = default_model()
    stats = []
    for ws in sorted(set(int(v) for v in rows[:, 0])):
        w = oc.sample_world(m, ws)
        eng = E.Engine(engine_model(m), w.signals)
        for rs in range(11, 17):
            sc = E.SamplerConfig(algorithm="chromatic-dynamic" if dyn else "chromatic-static",
                                 steps_per_epoch=k, epochs=ep, n_regions=nr, seed=rs,
                                 burn_in_fraction=0.0, record_every=1 << 30)
            eng.set_hypothesis(E.Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0),
                                        np.zeros((0, m.S))))
            tr = eng.run_chromatic(sc)
            f = tr.final
            p, rc, le, _ = oc.match_events(w.events, O.Events(f.ids, f.x, f.t, f.arrivals))
            stats.append((p, rc, le))
    gpu = np.array(stats)
    ref = rows[:, 2:5]
    for c, name in enumerate(["precision", "recall", "location_error"]):
        a, b = gpu[:, c], ref[:, c]
        se = np.sqrt(a.var(ddof=1) / len(a) + b.var(ddof=1) / len(b))
        assert abs(a.mean() - b.mean()) <= 2.5 * se + 0.02, (name, a.mean(), b.mean(), se)


def test_production_many_regions(E, oc):
    # more same-colored regions than SMs (several CTA waves per phase, as at
    # configs 2-4); trajectories must still match the oracle
    m = _mapped_model(S=24, T=2400.0, n_regions=400, x_max=1000.0, lam_events=150)
    w = oc.sample_world(m, 21)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=8, epochs=3, n_regions=400, seed=13, dynamic=1, rng_mode=1)
    _prod_vs_oracle(E, oc, m, w32, s, init=w.events, dtype=np.float32)


def test_replay_many_regions(E, oc):
    m = _mapped_model(S=24, T=2400.0, n_regions=400, x_max=1000.0, lam_events=150)
    w = oc.sample_world(m, 22)
    s = O.Sampler(steps_per_epoch=8, epochs=2, n_regions=400, seed=14, dynamic=1)
    r = oc.run_chromatic(w, s, init=w.events, tape=True)
    eng = E.Engine(engine_model(m), w.signals, event_capacity=1024)
    eng.set_hypothesis(E.Events(w.events.ids, w.events.x, w.events.t, w.events.arr))
    tr = eng.run_chromatic(engine_sampler(s), tape=r["tape"], tape_arrivals=r["tape_arr"])
    t = r["tape"]
    drawn = t["u_drawn"] == 1
    tie = np.zeros(len(t), bool)
    tie[drawn] = np.abs(t["log_r"][drawn] - np.log(t["u"][drawn])) < TIE
    assert not ((tr.step_out["accepted"] != t["accepted"]) & ~tie).any()
    assert np.array_equal(tr.final.ids, r["final"].ids)
    assert np.array_equal(tr.final.arrivals, r["final"].arr)


def test_trace_rows_and_snapshots(E, oc, tmp_path):
    # Trace rows / snapshots (samplers.hpp:73-103,424-434): rows at record
    # points, snapshots from burn-in on, the last one equal to the final
    m = default_model()
    w = golden_world("w1", m)
    s = O.Sampler(steps_per_epoch=100, epochs=10, n_regions=4, seed=5, dynamic=1, rng_mode=1,
                  record_every=300, burn_in_fraction=0.5)
    ro = oc.run_chromatic(w, s, tape=False, rowlj=True)
    eng = E.Engine(engine_model(m), w.signals)
    eng.set_snapshot_capacity(10000, 64)
    tr = eng.run_chromatic(engine_sampler(s, record_log_joint=True))
    assert np.array_equal(tr.row_step, ro["row_step"])
    assert np.array_equal(tr.row_count, ro["row_count"])
    burn = int(0.5 * s.epochs * s.steps_per_epoch * s.n_regions)
    want = [int(v) for v in ro["row_step"][1:] if v >= burn]
    assert [sn.step for sn in tr.snapshots] == want
    for sn, c in zip(tr.snapshots, [int(c) for st, c in zip(ro["row_step"][1:], ro["row_count"][1:])
                                     if st >= burn]):
        assert len(sn.ids) == c
    last = tr.snapshots[-1]
    assert np.array_equal(last.ids, ro["final"].ids) and np.array_equal(last.x, ro["final"].x)
    tr.write_trace_csv(str(tmp_path / "trace.csv"))
    tr.write_samples_csv(str(tmp_path / "samples.csv"))
    lines = open(tmp_path / "samples.csv").read().splitlines()
    assert lines[0] == "snapshot_id,event_id,x,t"
    assert len(lines) == 1 + sum(len(sn.ids) for sn in tr.snapshots)



# ------------------------------------------------------------------ naive mode
def _naive_sampler(E, s):
    return E.SamplerConfig(algorithm="naive", steps_per_epoch=s.steps_per_epoch,
                           epochs=s.epochs, n_regions=s.n_regions, seed=s.seed,
                           burn_in_fraction=s.burn_in_fraction, record_every=s.record_every,
                           record_log_joint=True)


@pytest.mark.parametrize("ws", [0, 2, 3])
def test_naive_production_matches_oracle_philox(E, oc, ws):
    m = default_model()
    w = golden_world(f"w{ws}", m)
    s = O.Sampler(steps_per_epoch=100, epochs=8, n_regions=4, seed=31 + ws, rng_mode=1,
                  record_every=130, burn_in_fraction=0.0)
    ro = oc.run_chromatic(w, s, tape=True, rowlj=True, naive=True)
    eng = E.Engine(engine_model(m), w.signals)
    tr = eng.run_chromatic(_naive_sampler(E, s), decisions=len(ro["tape"]))
    _decisions_match(tr.step_out, ro["tape"], 1e-11)
    assert tr.total_steps == ro["total_steps"]
    assert tr.total_accepted == ro["total_accepted"]
    assert np.array_equal(tr.final.ids, ro["final"].ids)
    assert np.array_equal(tr.final.arrivals, ro["final"].arr)
    assert np.array_equal(tr.row_step, ro["row_step"])
    assert np.array_equal(tr.row_count, ro["row_count"])
    assert close(tr.row_log_joint[-1], ro["row_lj"][-1], 1e-12)


def test_naive_replay_reference_tape(E, oc):
    m = _mapped_model(S=32, T=600.0, n_regions=12, x_max=400.0, lam_events=25)
    w = oc.sample_world(m, 6)
    s = O.Sampler(steps_per_epoch=50, epochs=4, n_regions=12, seed=2, record_every=1 << 30,
                  burn_in_fraction=0.0)
    r = oc.run_chromatic(w, s, tape=True, naive=True)
    eng = E.Engine(engine_model(m), w.signals)
    tr = eng.run_chromatic(_naive_sampler(E, s), tape=r["tape"], tape_arrivals=r["tape_arr"])
    t = r["tape"]
    drawn = t["u_drawn"] == 1
    tie = np.zeros(len(t), bool)
    tie[drawn] = np.abs(t["log_r"][drawn] - np.log(t["u"][drawn])) < TIE
    assert not ((tr.step_out["accepted"] != t["accepted"]) & ~tie).any()
    sc = t["scored"] == 1
    assert np.allclose(tr.step_out["delta"][sc], t["delta"][sc], rtol=1e-11, atol=1e-9)
    assert np.array_equal(tr.final.ids, r["final"].ids)
    assert np.array_equal(tr.final.arrivals, r["final"].arr)


def test_naive_posterior_within_seed_spread(E, oc):
    g = golden("posterior.npz")
    rows = g["rows"][g["rows"][:, 0] >= 1000]
    k, ep, nr, _ = [int(v) for v in g["sampler"]]
    m = default_model()
    stats = []
    for ws in sorted(set(int(v) % 1000 for v in rows[:, 0])):
        w = oc.sample_world(m, ws)
        eng = E.Engine(engine_model(m), w.signals)
        for rs in range(11, 17):
            eng.set_hypothesis(E.Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0),
                                        np.zeros((0, m.S))))
            sc = E.SamplerConfig(algorithm="naive", steps_per_epoch=k, epochs=ep, n_regions=nr,
                                 seed=rs, burn_in_fraction=0.0, record_every=1 << 30)
            f = eng.run_chromatic(sc).final
            stats.append(oc.match_events(w.events, O.Events(f.ids, f.x, f.t, f.arrivals))[:3])
    gpu = np.array(stats)
    ref = rows[:, 2:5]
    for c, name in enumerate(["precision", "recall", "location_error"]):
        a, b = gpu[:, c], ref[:, c]
        se = np.sqrt(a.var(ddof=1) / len(a) + b.var(ddof=1) / len(b))
        assert abs(a.mean() - b.mean()) <= 2.5 * se + 0.02, (name, a.mean(), b.mean(), se)


# ------------------------------------------------------------------ serial mode
def _serial_sampler(E, s, record_log_joint=True):
    return E.SamplerConfig(algorithm="serial", steps_per_epoch=s.steps_per_epoch,
                           epochs=s.epochs, n_regions=s.n_regions, seed=s.seed,
                           burn_in_fraction=s.burn_in_fraction, record_every=s.record_every,
                           record_log_joint=record_log_joint)


def test_serial_replay_reference_tape(E, oc):
    """run_serial (samplers.hpp:282-315) replayed from the oracle's tape, which
    test_oracle pins bit-exact to the reference's."""
    m = default_model()
    w = golden_world("w1", m)
    s = O.Sampler(steps_per_epoch=200, epochs=3, n_regions=4, seed=9, record_every=170,
                  burn_in_fraction=0.0)
    r = oc.run_chromatic(w, s, tape=True, serial=True, rowlj=True)
    eng = E.Engine(engine_model(m), w.signals)
    tr = eng.run_chromatic(_serial_sampler(E, s), tape=r["tape"], tape_arrivals=r["tape_arr"])
    t = r["tape"]
    assert np.array_equal(tr.step_out["scored"], t["scored"])
    drawn = t["u_drawn"] == 1
    tie = np.zeros(len(t), bool)
    tie[drawn] = np.abs(t["log_r"][drawn] - np.log(t["u"][drawn])) < TIE
    assert not ((tr.step_out["accepted"] != t["accepted"]) & ~tie).any()
    sc = (t["scored"] == 1) & np.isfinite(t["delta"])
    assert np.allclose(tr.step_out["delta"][sc], t["delta"][sc], rtol=1e-11, atol=1e-9)
    assert np.array_equal(tr.final.ids, r["final"].ids)
    assert np.array_equal(tr.final.arrivals, r["final"].arr)
    assert np.array_equal(tr.row_step, r["row_step"]) and np.array_equal(tr.row_count, r["row_count"])
    assert np.allclose(tr.row_log_joint, r["row_lj"], rtol=1e-12, atol=1e-8)


@pytest.mark.parametrize("ws", [0, 3])
def test_serial_production_matches_oracle_philox(E, oc, ws):
    m = default_model()
    w = golden_world(f"w{ws}", m)
    s = O.Sampler(steps_per_epoch=250, epochs=4, n_regions=4, seed=41 + ws, rng_mode=1,
                  record_every=300, burn_in_fraction=0.5)
    ro = oc.run_chromatic(w, s, tape=True, rowlj=True, serial=True)
    eng = E.Engine(engine_model(m), w.signals)
    eng.set_snapshot_capacity(1 << 14, 16)
    tr = eng.run_chromatic(_serial_sampler(E, s), decisions=len(ro["tape"]))
    _decisions_match(tr.step_out, ro["tape"], 1e-11)
    assert tr.total_steps == ro["total_steps"] and tr.total_accepted == ro["total_accepted"]
    assert np.array_equal(tr.final.ids, ro["final"].ids)
    assert np.array_equal(tr.final.arrivals, ro["final"].arr)
    assert np.array_equal(tr.row_step, ro["row_step"]) and np.array_equal(tr.row_count, ro["row_count"])
    assert np.allclose(tr.row_log_joint, ro["row_lj"], rtol=1e-12, atol=1e-8)
    # snapshots at every record point past burn-in (samplers.hpp:309-312)
    assert [sn.step for sn in tr.snapshots] == [int(v) for v in ro["row_step"][1:] if v >= 500]


# ------------------------------------------------------------------ limits
def test_count_overflow_is_detected(E):
    """more than 65535 events over one (sample, station): the uint16 counts
    would wrap; the engine refuses the hypothesis and stays usable."""
    m = O.Model(lambda_rate=0.01, T=100.0, x_max=10.0, v=2.0, stations=O.stations_line(2, 10.0))
    em = engine_model(m)
    sig = np.zeros((2, 100))
    N = 65536
    eng = E.Engine(em, sig, event_capacity=N + 8)
    arr = np.tile(np.array([[50.0, 55.0]]), (N, 1))
    ev = E.Events(np.arange(N, dtype=np.uint64), np.zeros(N), np.full(N, 50.0), arr)
    with pytest.raises(RuntimeError, match="overflow"):
        eng.set_hypothesis(ev)
    assert eng.get_hypothesis().ids.size == 0
    ok = E.Events(ev.ids[:65535], ev.x[:65535], ev.t[:65535], arr[:65535])
    eng.set_hypothesis(ok)
    assert eng.get_hypothesis(arrivals=False).ids.size == 65535
    with pytest.raises(ValueError):  # above event_capacity
        E.Engine(em, sig, event_capacity=4).set_hypothesis(ok)


def test_capacity_and_region_limits_fail_loudly(E, oc):
    m = default_model()
    w = golden_world("w0", m)
    # births past a tiny event table: status 3, not a silent wrap
    eng = E.Engine(engine_model(m), w.signals, event_capacity=2)
    with pytest.raises(RuntimeError):
        eng.run_chromatic(E.SamplerConfig(steps_per_epoch=400, epochs=6, n_regions=4, seed=1))
    # the serial chain lives in one CTA: more than 1024 events is refused
    many = oc.sample_world(O.Model(lambda_rate=1100 / 240.0), 5)
    assert many.events.N > 1024
    eng2 = E.Engine(engine_model(many.model), many.signals, event_capacity=2048)
    eng2.set_hypothesis(E.Events(many.events.ids, many.events.x, many.events.t, many.events.arr))
    with pytest.raises(RuntimeError, match="per-chain event limit"):
        eng2.run_chromatic(E.SamplerConfig(algorithm="serial", steps_per_epoch=10, epochs=1))


def test_production_dense_regions_generic_band(E, oc):
    """many events per region and long chains: a region's own diff grows past
    four effective windows per station, the generic band path (density.hpp:
    263-301 with the frozen view) against the oracle."""
    m = O.Model(lambda_rate=48 / 240.0)
    w = oc.sample_world(m, 21)
    s = O.Sampler(steps_per_epoch=400, epochs=3, n_regions=4, seed=8, dynamic=1, rng_mode=1)
    tr, ro = _prod_vs_oracle(E, oc, m, w, s, init=w.events)
    assert tr.final.ids.size > 20


@pytest.mark.parametrize("depth", [1, 2, 4])
@pytest.mark.parametrize("S", [96, 2080])
def test_production_independent_of_speculation_depth(E, oc, monkeypatch, depth, S):
    """The speculative rounds (up to M proposals scored against one state, the
    next round's proposals generated during the decision) must reproduce the
    sequential chain for every depth M (SEIS_SPEC; default 3): decisions,
    deltas and the final hypothesis equal the oracle's. S = 96 runs the
    proposal-major item order with the per-round diff-window cache, S = 2080
    (65 station tiles) the tile-major order."""
    monkeypatch.setenv("SEIS_SPEC", str(depth))
    m = _mapped_model(S=S, T=400.0, n_regions=24, x_max=4000.0, lam_events=30)
    w = oc.sample_world(m, 11)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=24, epochs=3, n_regions=24, seed=21, dynamic=1, rng_mode=1)
    _prod_vs_oracle(E, oc, m, w32, s, init=w.events, dtype=np.float32)


@pytest.mark.parametrize("steps", [200, 800])
def test_production_burn_in_from_empty_many_windows(E, oc, steps):
    """Burn-in from the reference's empty start: regions accept many births
    within a phase, so stations see five to eight own diff windows (the
    eight-window band fed by the round cache's overflow array) and, with the
    longer chains, more than eight (the generic band); every decision, delta
    and the final hypothesis against the oracle."""
    m = _mapped_model(S=64, T=300.0, n_regions=6, x_max=1000.0, lam_events=40)
    w = oc.sample_world(m, 5)
    s = O.Sampler(steps_per_epoch=steps, epochs=3, n_regions=6, seed=13, dynamic=0, rng_mode=1)
    tr, ro = _prod_vs_oracle(E, oc, m, w, s)
    assert tr.final.ids.size > 10


@pytest.mark.parametrize("toggle", ["SEIS_TERMS", "SEIS_FIRST"])
def test_tile_major_fast_paths_equal_the_direct_paths(E, oc, monkeypatch, toggle):
    """The tile-major pass's shortcuts must not change a result: the per-sample
    term cache (k_terms, summed by band1_terms / dense_pair_terms instead of
    the direct band; SEIS_TERMS=0 disables it) and rounds that end at their
    first scored proposal, births and deaths taking the next ones along
    (SEIS_FIRST=0: three proposals scored per round).
    With the shortcut off and on: every delta and decision bit-identical
    (same operations in the same order), the final hypothesis identical, and
    both equal to the oracle (density.hpp:214-305, samplers.hpp:115-138)."""
    m = _mapped_model(S=4200, T=300.0, n_regions=12, x_max=4000.0, lam_events=14)
    w = oc.sample_world(m, 23)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=20, epochs=2, n_regions=12, seed=33, dynamic=1, rng_mode=1)
    outs = []
    # SEIS_FIRST: 0 = three proposals scored per round, 1 = rounds end at the
    # first scored one, 2 / 3 = births and deaths take one more / as many as
    # the batch holds along (3 is the tile-major default)
    for val in ("0", "1") if toggle == "SEIS_TERMS" else ("0", "1", "2", "3"):
        monkeypatch.setenv(toggle, val)
        tr, ro = _prod_vs_oracle(E, oc, m, w32, s, init=w.events, dtype=np.float32)
        outs.append(tr)
    a, b = outs[0], outs[-1]
    for o in outs[1:]:
        assert np.array_equal(a.step_out["accepted"], o.step_out["accepted"])
        assert np.array_equal(a.final.arrivals, o.final.arrivals)
    assert np.array_equal(a.step_out["accepted"], b.step_out["accepted"])
    if toggle == "SEIS_TERMS":  # same operations in the same order
        assert np.array_equal(a.step_out["delta"], b.step_out["delta"])
    else:  # the per-lane partial sums take the tiles in pairs: last-bit differences
        fin = np.isfinite(a.step_out["delta"])
        assert np.array_equal(fin, np.isfinite(b.step_out["delta"]))
        assert np.allclose(a.step_out["delta"][fin], b.step_out["delta"][fin], rtol=1e-12,
                           atol=1e-9)
    assert np.array_equal(a.final.arrivals, b.final.arrivals)
