"""CPU: the plain-C oracle restatement against the reference's golden vectors
(tests/golden/, generated from the reference compiled in place) and, when the
reference tree is present, against oracle/_ref directly."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import default_model, golden, golden_world, tape_sampler, wide_model


@pytest.fixture(scope="module")
def oc(built):
    return O.Oracle("c")


def test_partition_kats_and_grid(oc):
    g = golden("partition.npz")
    for i, (T, l, u, tau) in enumerate(g["cases"]):
        rc, msg, b, c, k = oc.partition(T, l, u, tau)
        assert rc == g["rc"][i], (i, msg)
        if rc:
            continue
        assert np.array_equal(b, g[f"b{i}"])  # bit-exact boundaries (b += l recurrence)
        assert np.array_equal(c, g[f"c{i}"]) and k == g["k"][i]
        regs = [oc.region_of(b, p) for p in g[f"probe{i}"]]
        assert np.array_equal(regs, g[f"reg{i}"])


def test_partition_reference_kats(oc):
    # proj/tests/test_partition.cpp:11-59
    rc, _, b, c, k = oc.partition(240, 60, 0, 50)
    assert list(b) == [0, 60, 120, 180, 240] and list(c) == [0, 1, 0, 1] and k == 2
    rc, _, b, c, k = oc.partition(240, 60, 25, 50)
    assert np.allclose(b, [0, 25, 85, 145, 205, 240])
    rc, _, b, c, k = oc.partition(240, 30, 0, 50)
    assert k == 3 and list(c) == [i % 3 for i in range(8)]
    assert oc.partition(240, 20, 0, 50)[0] == 2
    for bad in [(240, 0, 0, 50), (240, 300, 0, 50), (240, 60, 60, 50), (240, 60, -1, 50)]:
        assert oc.partition(*bad)[0] == 2


def test_offsets(oc):
    g = golden("rng.npz")
    for r, (seed, l) in enumerate([(0, 60.0), (1, 14.0625), (123456789, 0.87890625)]):
        got = [oc.partition_offset(seed, ep, l) for ep in range(1, 20)]
        assert np.array_equal(got, g["offsets"][r])


def test_worldgen_bit_exact(oc):
    m = default_model()
    for seed in range(4):
        w = oc.sample_world(m, seed)
        gw = golden_world(f"w{seed}", m)
        assert np.array_equal(w.signals, gw.signals)
        assert np.array_equal(w.events.arr, gw.events.arr)
        assert np.array_equal(w.events.x, gw.events.x) and np.array_equal(w.events.t, gw.events.t)
    mw = wide_model()
    w = oc.sample_world(mw, 5)
    gw = golden_world("wide", mw)
    assert np.array_equal(w.signals, gw.signals)
    p = oc.make_world_with_events(m, [20.0, 80.0, 50.0], [30.0, 100.0, 190.0], 9)
    gp = golden_world("planted", m)
    assert np.array_equal(p.signals, gp.signals) and np.array_equal(p.events.arr, gp.events.arr)


def _golden_changes():
    g = golden("deltas.npz")
    for i in range(len(g["delta"])):
        rem = [int(g["rem"][i])] if g["n_rem"][i] else []
        add = None
        if g["n_add"][i]:
            add = O.Events(np.array([g["add_id"][i]], np.uint64), np.array([g["add_x"][i]]),
                           np.array([g["add_t"][i]]), g["add_arr"][i][None, :])
        yield rem, add, g["delta"][i]


def test_delta_matches_reference_bits(oc):
    mw = wide_model()
    w = golden_world("wide", mw)
    for rem, add, d in _golden_changes():
        got = oc.delta(mw, w.signals, w.events, rem, add)
        assert got == d or (np.isinf(got) and np.isinf(d))
    assert oc.log_joint(mw, w.signals, w.events) == golden("deltas.npz")["log_joint"][0]


def test_delta_equals_full_recompute(oc):
    # proj/tests/test_model.cpp:309-348: delta vs log_joint(after) - log_joint(before)
    mw = wide_model()
    w = golden_world("wide", mw)
    base = oc.log_joint(mw, w.signals, w.events)
    n = 0
    for rem, add, d in _golden_changes():
        keep = [i for i in range(w.events.N) if i not in rem]
        ev = w.events
        ids = np.concatenate([ev.ids[keep], add.ids if add else np.zeros(0, np.uint64)])
        x = np.concatenate([ev.x[keep], add.x if add else []])
        t = np.concatenate([ev.t[keep], add.t if add else []])
        arr = np.concatenate([ev.arr[keep], add.arr if add else np.zeros((0, mw.S))])
        after = oc.log_joint(mw, w.signals, O.Events(ids, x, t, arr))
        if np.isinf(d):
            assert np.isinf(after)
        else:
            assert abs((after - base) - d) < 1e-8
        n += 1
        if n >= 60:
            break


@pytest.mark.parametrize("name", ["default_static", "default_dynamic", "wide_dynamic"])
def test_chromatic_tape_matches_reference(oc, name):
    g = golden(f"tape_{name}.npz")
    s = tape_sampler(g["sampler"])
    if name.startswith("default"):
        m = default_model()
        w = golden_world("w1" if "static" in name else "w2", m)
    else:
        m = wide_model()
        w = golden_world("wide", m)
    r = oc.run_chromatic(w, s, tape=True, rowlj=True)
    assert r["tape"].tobytes() == g["tape"].tobytes()
    assert np.array_equal(r["tape_arr"], g["tape_arr"])
    assert np.array_equal(r["final"].ids, g["final_ids"])
    assert np.array_equal(r["final"].arr, g["final_arr"])
    assert np.array_equal(r["row_lj"], g["row_lj"])
    assert r["total_accepted"] == int(g["total_accepted"])


@pytest.mark.skipif(not O.have_ref(), reason="reference tree absent")
def test_composed_driver_equals_reference_run_sampler(built):
    # the shim's tape driver == the reference's own run_sampler (workers 1 and 4)
    R = O.Oracle("ref")
    m = default_model()
    w = R.sample_world(m, 11)
    for dyn in (0, 1):
        s = O.Sampler(steps_per_epoch=50, epochs=8, n_regions=4, seed=21, dynamic=dyn,
                      burn_in_fraction=0.0)
        a = R.run_chromatic(w, s, tape=False)
        for workers in (1, 4):
            b = O.ref_run_sampler(w, s, workers=workers)
            assert np.array_equal(a["final"].ids, b["final"].ids)
            assert np.array_equal(a["final"].arr, b["final"].arr)
            assert a["total_accepted"] == b["total_accepted"]


@pytest.mark.skipif(not O.have_ref(), reason="reference tree absent")
def test_oracle_vs_reference_random_worlds(built, oc):
    R = O.Oracle("ref")
    for seed in range(3):
        m = O.Model(lambda_rate=0.05, T=120.0, stations=O.stations_line(6, 100.0))
        a = oc.sample_world(m, 100 + seed)
        b = R.sample_world(m, 100 + seed)
        assert np.array_equal(a.signals, b.signals)
        s = O.Sampler(steps_per_epoch=40, epochs=5, n_regions=2, seed=seed, dynamic=seed % 2)
        ra = oc.run_chromatic(a, s)
        rb = R.run_chromatic(b, s)
        assert ra["tape"].tobytes() == rb["tape"].tobytes()


def test_philox_known_answers(built):
    # Random123 kat_vectors for philox4x32_10
    assert O.philox((0, 0, 0, 0), (0, 0)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    f = 0xFFFFFFFF
    assert O.philox((f, f, f, f), (f, f)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
                    (0xA4093822, 0x299F31D0)) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_philox_normals_are_standard(built):
    z = np.array([O.philox_normal(7, 3, r, s, i) for r in range(10) for s in range(20)
                  for i in range(25)])
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1) < 0.05
    assert abs(np.mean(z ** 4) - 3) < 0.3


def test_match_events_reference_kats(oc):
    # evaluation.hpp:51-103 conventions: vacuous precision/recall, threshold
    T = O.Events(np.array([1, 2], np.uint64), np.array([10.0, 50.0]), np.array([20.0, 100.0]),
                 np.zeros((2, 4)))
    E = O.Events.empty(4)
    assert oc.match_events(T, E) == (1.0, 0.0, 0.0, 0)
    assert oc.match_events(E, T) == (0.0, 1.0, 0.0, 0)
    I = O.Events(np.array([7], np.uint64), np.array([13.0]), np.array([24.0]), np.zeros((1, 4)))
    p, r, le, n = oc.match_events(T, I)
    assert (p, r, n) == (1.0, 0.5, 1) and abs(le - 5.0) < 1e-12
    far = O.Events(np.array([7], np.uint64), np.array([10.0]), np.array([32.5]), np.zeros((1, 4)))
    assert oc.match_events(T, far)[3] == 0  # |dt| = 12.5 >= threshold 12


def test_posterior_statistics_match_reference(oc):
    # the restatement's reference-mode driver reproduces the reference's own
    # run_sampler trajectories, hence its posterior statistics, exactly
    g = golden("posterior.npz")
    k, ep, nr, dyn = [int(v) for v in g["sampler"]]
    m = default_model()
    for row in g["rows"][::5]:
        ws, rs = int(row[0]), int(row[1])
        naive = ws >= 1000
        w = oc.sample_world(m, ws % 1000)
        s = O.Sampler(steps_per_epoch=k, epochs=ep, n_regions=nr, seed=rs, dynamic=dyn,
                      burn_in_fraction=0.0, record_every=1 << 30)
        r = oc.run_chromatic(w, s, tape=False, naive=naive)
        p, rc, le, _ = oc.match_events(w.events, r["final"])
        assert (p, rc, le) == (row[2], row[3], row[4])
        assert r["final"].N == row[5] and r["total_accepted"] == row[7]


@pytest.mark.parametrize("seed", [0, 1])
def test_naive_tape_matches_reference(oc, seed):
    if not O.have_ref():
        pytest.skip("reference tree absent")
    R = O.Oracle("ref")
    m = default_model()
    w = oc.sample_world(m, 40 + seed)
    s = O.Sampler(steps_per_epoch=100, epochs=5, n_regions=4, seed=seed, record_every=150,
                  burn_in_fraction=0.0)
    a = oc.run_chromatic(w, s, naive=True, rowlj=True)
    b = R.run_chromatic(w, s, naive=True, rowlj=True)
    assert a["tape"].tobytes() == b["tape"].tobytes()
    assert np.array_equal(a["row_lj"], b["row_lj"]) and np.array_equal(a["row_count"], b["row_count"])
    c = O.ref_run_sampler(w, s, naive=True)
    assert np.array_equal(a["final"].arr, c["final"].arr)


@pytest.mark.parametrize("seed", [0, 5])
def test_serial_tape_matches_reference(oc, seed):
    """run_serial (samplers.hpp:282-315): the oracle's tape, rows and final
    hypothesis bit-identical to the reference's, which also matches the
    reference's own run_sampler(Serial)."""
    if not O.have_ref():
        pytest.skip("reference tree absent")
    R = O.Oracle("ref")
    m = default_model()
    w = oc.sample_world(m, 60 + seed)
    s = O.Sampler(steps_per_epoch=150, epochs=4, n_regions=4, seed=seed, record_every=110,
                  burn_in_fraction=0.0)
    a = oc.run_chromatic(w, s, serial=True, rowlj=True)
    b = R.run_chromatic(w, s, serial=True, rowlj=True)
    assert a["tape"].tobytes() == b["tape"].tobytes()
    assert np.array_equal(a["tape_arr"], b["tape_arr"])
    assert np.array_equal(a["row_step"], b["row_step"]) and np.array_equal(a["row_count"], b["row_count"])
    assert np.array_equal(a["row_lj"], b["row_lj"])
    assert a["total_accepted"] == b["total_accepted"]
    c = O.ref_run_sampler(w, s, serial=True)
    order = np.argsort(c["final"].ids)
    assert np.array_equal(a["final"].ids, c["final"].ids[order])
    assert np.array_equal(a["final"].arr, c["final"].arr[order])


_DIV_CHECK = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static uint64_t s = 0x9e3779b97f4a7c15ull;
static uint64_t nx(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double u01(void) { return (double)(nx() >> 11) * 0x1.0p-53; }
int main(int argc, char** argv) {
  long bad = 0;
  for (int k = 1; k + 1 < argc; k += 2) {
    const double v = strtod(argv[k], 0), span = strtod(argv[k + 1], 0), y = 1.0 / v;
    for (long i = 0; i < 10000000; ++i) {
      double a = u01() * span;
      if (i & 1) a = floor(a * 1024.0) / 1024.0;  /* station-grid-like operands */
      if (span < 0) { const double dd = u01() * 40.0 - 20.0; a = dd * dd; } /* (a - mean)^2 */
      const double q0 = a * y, q = fma(fma(-q0, v, a), y, q0);
      bad += q != a / v;
    }
  }
  printf("%ld\n", bad);
  return 0;
}
"""


def test_division_by_reciprocal_is_exact(tmp_path):
    """arrival_mean on the device (engine.cuh div_v) replaces |x - s| / v by
    q0 = a RN(1/v), q = RN(q0 + (a - q0 v) RN(1/v)); bit-identical to the
    reference's division (model.hpp:73-75) for every v of configs 0-4 and the
    default world, 10^7 operands each over [0, x_max]."""
    import subprocess
    src = tmp_path / "div.c"
    src.write_text(_DIV_CHECK)
    exe = tmp_path / "div"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", str(src), "-o", str(exe), "-lm"], check=True)
    # (v, x_max): reference default (v = 2, x_max = 100) and the SURVEY 8(d)
    # mapping v = 1.2 x_max R^2 / T of configs 0-4
    cases = [(2.0, 100.0)]
    for x_max, T, R in [(1000, 3600, 4), (4000, 3600, 16), (16000, 3600, 64), (16000, 1800, 128),
                        (32000, 1024, 256)]:
        cases.append((1.2 * x_max * R * R / T, float(x_max)))
    # arr_logpdf: (a - mean)^2 / (2 sigma^2) for sigma_arrival values whose
    # 2 sigma^2 is and is not a power of two (span < 0 selects squared operands)
    for sig in (2.0, 1.5, 1.1, 0.7, 3.3, 2.5):
        cases.append((2.0 * (sig * sig), -1.0))
    args = [f"{x:.17g}" for c in cases for x in c]
    out = subprocess.run([str(exe)] + args, check=True, capture_output=True, text=True).stdout
    assert int(out.strip()) == 0
