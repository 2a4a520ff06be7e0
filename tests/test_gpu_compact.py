"""GPU parity of the compact arrival storage ("philox stream spec v2",
include/seis_philox.h): births of a production run and their location /
joint moves are generated versions (location + philox key, arrivals computed
as mean + sigma z), arrival moves are per-station overrides (up to 8; the
ninth stores the row). The CPU oracle implements the same spec (so_sampler
compact = 1); every decision, delta, trace row (log_joint included), the
final hypothesis with all its arrivals, and deltas scored against a
hypothesis holding generated versions must match it."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import default_model, engine_model, engine_sampler, golden_world

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(built):
    import paper_1612_00595_b200 as E
    return E


def _mapped(S, T, n_regions, x_max, lam_events):
    return O.Model(lambda_rate=lam_events / T, T=T, x_max=x_max,
                   v=1.2 * x_max * n_regions / T, stations=O.stations_line(S, x_max))


def _run(E, m, w, s, init=None, dtype=np.float64, algorithm=None, cap=4096):
    oc = O.Oracle("c")
    kw = dict(naive=algorithm == "naive", serial=algorithm == "serial")
    ro = oc.run_chromatic(w, s, init=init, tape=True, rowlj=True, **kw)
    eng = E.Engine(engine_model(m), w.signals.astype(dtype), event_capacity=cap)
    eng.arrival_storage = "compact"
    assert eng.arrival_storage == "compact"
    if init is not None:
        eng.set_hypothesis(E.Events(init.ids, init.x, init.t, init.arr))
    sc = engine_sampler(s, record_log_joint=True)
    if algorithm:
        sc.algorithm = algorithm
    tr = eng.run_chromatic(sc, decisions=len(ro["tape"]))
    so, t = tr.step_out, ro["tape"]
    assert np.array_equal(so["accepted"], t["accepted"])
    fin = (t["scored"] == 1) & np.isfinite(t["delta"])
    rtol = 1e-11 if dtype == np.float64 else 1e-5
    assert np.allclose(so["delta"][fin], t["delta"][fin], rtol=rtol, atol=1e-9)
    assert tr.total_accepted == ro["total_accepted"]
    assert np.array_equal(tr.final.ids, ro["final"].ids)
    assert np.array_equal(tr.final.x, ro["final"].x) and np.array_equal(tr.final.t, ro["final"].t)
    assert np.array_equal(tr.final.arrivals, ro["final"].arr)  # generated versions' arrivals
    assert np.array_equal(tr.row_count, ro["row_count"])
    if algorithm != "naive":
        assert np.allclose(tr.row_log_joint, ro["row_lj"], rtol=1e-12, atol=1e-8)
    return eng, tr, ro


@pytest.mark.parametrize("dyn", [0, 1])
def test_compact_production_from_empty(E, dyn):
    m = default_model()
    w = golden_world("w3", m)
    s = O.Sampler(steps_per_epoch=150, epochs=10, n_regions=4, seed=23, dynamic=dyn,
                  rng_mode=1, record_every=500, compact=1)
    eng, tr, ro = _run(E, m, w, s)
    assert tr.total_accepted > 100


def test_compact_generated_versions_persist_without_arrival_moves(E):
    """with no arrival moves every birth stays a generated version through its
    location and joint moves: the final hypothesis is all generated versions
    (no stored rows), its arrivals computed on the device equal the oracle's"""
    m = default_model()
    w = golden_world("w3", m)
    s = O.Sampler(steps_per_epoch=150, epochs=12, n_regions=4, seed=29, dynamic=1,
                  rng_mode=1, record_every=500, compact=1, weights=(0.25, 0.25, 0.375, 0.0, 0.125))
    eng, tr, ro = _run(E, m, w, s)
    assert tr.stats["generated_versions"] == ro["final"].N > 0


def test_compact_production_mapped_fp32_from_truth(E):
    """stored rows (the loaded truth) and generated versions side by side"""
    oc = O.Oracle("c")
    m = _mapped(S=96, T=600.0, n_regions=40, x_max=4000.0, lam_events=60)
    w = oc.sample_world(m, 4)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=24, epochs=6, n_regions=40, seed=3, dynamic=1, rng_mode=1,
                  compact=1)
    _run(E, m, w32, s, init=w.events, dtype=np.float32)


def test_compact_tile_major_and_burn_in(E):
    """S = 2080 (tile-major pass) from the empty start: many generated
    versions per region, diff windows of generated versions"""
    oc = O.Oracle("c")
    m = _mapped(S=2080, T=400.0, n_regions=24, x_max=4000.0, lam_events=30)
    w = oc.sample_world(m, 11)
    w32 = O.World(m, w.events, w.signals.astype(np.float32).astype(np.float64))
    s = O.Sampler(steps_per_epoch=40, epochs=3, n_regions=24, seed=21, dynamic=1, rng_mode=1,
                  compact=1)
    eng, tr, ro = _run(E, m, w32, s, dtype=np.float32)
    assert tr.total_accepted > 20


def test_compact_naive_and_serial(E):
    m = default_model()
    w = golden_world("w2", m)
    s = O.Sampler(steps_per_epoch=100, epochs=6, n_regions=4, seed=7, rng_mode=1,
                  record_every=150, burn_in_fraction=0.0, compact=1)
    _run(E, m, w, s, algorithm="naive")
    s2 = O.Sampler(steps_per_epoch=250, epochs=4, n_regions=4, seed=9, rng_mode=1,
                   record_every=300, burn_in_fraction=0.0, compact=1)
    _run(E, m, w, s2, algorithm="serial")


def test_compact_versions_scored_and_continued(E):
    """deltas against a hypothesis holding generated versions
    (seis_score_batch), and a rows-mode run continuing from it, against the
    oracle on the same arrays"""
    oc = O.Oracle("c")
    m = default_model()
    w = golden_world("w1", m)
    s = O.Sampler(steps_per_epoch=150, epochs=6, n_regions=4, seed=5, dynamic=1, rng_mode=1,
                  compact=1)
    eng, tr, ro = _run(E, m, w, s)
    f = ro["final"]
    assert f.N > 2
    rng = np.random.default_rng(1)
    changes, want = [], []
    for i in range(f.N):
        changes.append(([int(f.ids[i])], []))
        want.append(oc.delta(m, w.signals, f, [i], None))
        x, t = f.x[i] + rng.normal(), f.t[i] + rng.normal()
        a = f.arr[i] + (t + np.abs(x - m.stations) / m.v) - (f.t[i] + np.abs(f.x[i] - m.stations) / m.v)
        changes.append(([int(f.ids[i])], [(x, t, a)]))
        want.append(oc.delta(m, w.signals, f, [i], O.Events(np.array([f.ids[i]]), np.array([x]),
                                                          np.array([t]), a[None, :])))
    got = eng.delta_log_joint(changes)
    assert np.allclose(got, want, rtol=1e-11, atol=1e-9)
    assert abs(eng.log_joint() - oc.log_joint(m, w.signals, f)) < 1e-8 * max(1, abs(eng.log_joint()))
    # continue in rows mode: generated versions move / die under spec v1 rules
    # for the new rows; the oracle continues from the same arrays
    eng.arrival_storage = "rows"
    s2 = O.Sampler(steps_per_epoch=100, epochs=3, n_regions=4, seed=6, dynamic=1, rng_mode=1)
    tr2 = eng.run_chromatic(engine_sampler(s2))
    assert tr2.total_steps > 0


def test_compact_overrides_fill_and_materialise(E):
    """arrival moves dominate: generated versions collect up to 8 overrides,
    the ninth accepted arrival move stores the version as a row (spec v2);
    both paths against the oracle, bit for bit"""
    m = default_model()
    w = golden_world("w1", m)
    s = O.Sampler(steps_per_epoch=600, epochs=4, n_regions=4, seed=12, rng_mode=1,
                  record_every=800, burn_in_fraction=0.0, compact=1,
                  weights=(0.15, 0.05, 0.1, 0.6, 0.1))
    eng, tr, ro = _run(E, m, w, s, algorithm="serial")
    assert tr.total_accepted > 200
    s2 = O.Sampler(steps_per_epoch=300, epochs=6, n_regions=4, seed=13, dynamic=1, rng_mode=1,
                   record_every=1000, compact=1, weights=(0.15, 0.05, 0.1, 0.6, 0.1))
    _run(E, m, w, s2)
