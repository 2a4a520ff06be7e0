"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
the host-side world generator is bit-exact with the reference generator."""
import re
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import default_model, engine_model, golden_world, wide_model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(seis_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(built):
    from paper_1612_00595_b200 import engine
    L = engine.load_library()
    names = declared("seis_b200.h")
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(engine.EXPORTS) == set(names)


def test_oracle_has_no_product_dependency():
    # the product never imports, links or calls the oracle
    bad = re.compile(r"(from\s+oracle|import\s+oracle|libseis_oracle|seis_oracle\.h|libseisref|so_delta)")
    for root, _, files in os.walk(os.path.join(ROOT, "paper_1612_00595_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(root, f)).read()
                assert not bad.search(src), f


def test_product_worldgen_bit_exact(built):
    from paper_1612_00595_b200 import F32, F64, make_world_with_events, sample_world
    m = default_model()
    for seed in range(4):
        ev, sig = sample_world(engine_model(m), seed, dtype=F64, threads=3)
        g = golden_world(f"w{seed}", m)
        assert np.array_equal(sig, g.signals)
        assert np.array_equal(ev.arrivals, g.events.arr)
    mw = wide_model()
    ev, sig = sample_world(engine_model(mw), 5, dtype=F32, threads=4)
    g = golden_world("wide", mw)
    assert np.array_equal(sig, g.signals.astype(np.float32))
    ev, sig = make_world_with_events(engine_model(m), [20.0, 80.0, 50.0], [30.0, 100.0, 190.0],
                                     9, dtype=F64)
    g = golden_world("planted", m)
    assert np.array_equal(sig, g.signals) and np.array_equal(ev.arrivals, g.events.arr)


def test_engine_fails_loudly_without_gpu(built):
    import torch
    if torch.cuda.is_available():
        return
    from paper_1612_00595_b200 import Engine
    m = default_model()
    g = golden_world("w0", m)
    try:
        Engine(engine_model(m), g.signals)
    except RuntimeError as e:
        assert "CUDA" in str(e) or "device" in str(e)
    else:
        raise AssertionError("engine constructed without a GPU")


def test_evaluation_bridge_bit_exact_vs_reference(built):
    """match_events / bootstrap_ci (evaluation.hpp:51-171) through the C-ABI
    against the reference's own outputs (tests/golden/make_golden_eval.py)."""
    import paper_1612_00595_b200 as E
    from tests.helpers import golden
    g = golden("eval.npz")
    for i, (thr, pr, rc, le, nm) in enumerate(g["match"]):
        T = E.Events(g[f"m{i}_ti"], g[f"m{i}_tx"], g[f"m{i}_tt"], np.zeros((len(g[f"m{i}_ti"]), 1)))
        I = E.Events(g[f"m{i}_ii"], g[f"m{i}_ix"], g[f"m{i}_it"], np.zeros((len(g[f"m{i}_ii"]), 1)))
        r = E.match_events(T, I, thr)
        assert (r.precision, r.recall, r.location_error, r.n_matched) == (pr, rc, le, int(nm)), i
        assert r.n_true == len(T.ids) and r.n_inferred == len(I.ids)
        assert len(set(r.pair_inferred_id.tolist())) == r.n_matched  # degrees <= 1
        if r.n_matched:
            assert abs(r.pair_distance.mean() - r.location_error) <= 1e-12 * max(1.0, le)
    for i, row in enumerate(g["boot"]):
        level, res = row[0], int(row[1])
        ci = E.bootstrap_ci(g[f"b{i}_v"], level, res, int(g["boot_seed"][i]))
        assert (ci.mean, ci.lo, ci.hi, ci.level) == tuple(row[3:7]), i
    with pytest.raises(ValueError):
        E.bootstrap_ci([], 0.95, 10, 0)
    with pytest.raises(ValueError):
        E.bootstrap_ci([1.0], 1.5, 10, 0)
    with pytest.raises(ValueError):
        E.match_events(T, I, 0.0)
    # vacuous conventions (evaluation.hpp:46-49)
    empty = E.Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0), np.zeros((0, 1)))
    r = E.match_events(empty, empty)
    assert (r.precision, r.recall, r.location_error) == (1.0, 1.0, 0.0)


def test_world_file_round_trip(built, tmp_path):
    """seis world v1 (binary replacement of the reference's CSV world files,
    SURVEY §8(f)3): save -> load is bit-identical, and loads as memory maps."""
    import paper_1612_00595_b200 as E
    m = engine_model(default_model())
    for dt in (E.F64, E.F32):
        ev, sig = E.sample_world(m, 11, dtype=dt, threads=2)
        p = str(tmp_path / f"w{dt}.seisworld")
        E.save_world(p, m, ev, sig)
        m2, ev2, sig2 = E.load_world(p)
        assert isinstance(sig2, np.memmap) and sig2.dtype == sig.dtype
        assert np.array_equal(sig2, sig) and np.array_equal(ev2.arrivals, ev.arrivals)
        assert np.array_equal(ev2.ids, ev.ids) and np.array_equal(ev2.x, ev.x)
        assert np.array_equal(ev2.t, ev.t) and np.array_equal(m2.stations, m.stations)
        assert (m2.T, m2.v, m2.lambda_rate, m2.t_s) == (m.T, m.v, m.lambda_rate, m.t_s)
    empty = E.Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0), np.zeros((0, 4)))
    p = str(tmp_path / "empty.seisworld")
    E.save_world(p, m, empty, sig)
    assert E.load_world(p)[1].ids.size == 0
    with open(p, "r+b") as f:
        f.write(b"NOTWORLD")
    with pytest.raises(ValueError):
        E.load_world(p)


@pytest.mark.skipif(not O.have_ref(), reason="needs oracle/_ref (reference tree)")
def test_thomas_events_match_reference_rng(built):
    """config[4]'s Thomas cluster process: the engine's host generator and the
    same draws made with the reference's own Rng (oracle/_ref, used by the
    reference arm of bench.py) give identical events"""
    from paper_1612_00595_b200 import thomas_events
    for T, x_max, pm in ((1024.0, 32000.0, 2000.0), (240.0, 100.0, 5.0)):
        cx, ct = thomas_events(3, x_max, T, pm, 10.0, 50.0, 0.0015625 * T)
        rx, rt = O.ref_thomas_events(3, x_max, T, pm, 10.0, 50.0, 0.0015625 * T)
        assert len(cx) > 0 and np.array_equal(cx, rx) and np.array_equal(ct, rt)


@pytest.mark.skipif(not os.path.isdir(O.REF_INC), reason="needs the reference headers")
def test_cpp_binding_compiles_against_reference_headers(built):
    """include/seis_b200.hpp (INTEGRATION.md's binding) compiles against the
    unmodified reference headers and links the engine; without a GPU its
    errors follow the reference's: std::invalid_argument for validation,
    std::runtime_error for the missing device"""
    import subprocess
    import torch
    exe = O.build_binding()
    assert exe and os.path.exists(exe)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_gpu_baseline_parity")
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK cpu" in r.stdout, r.stdout + r.stderr


def test_streaming_worldgen_bit_exact(built):
    """f3: the streamed generator (no N x S arrival matrix) gives the same
    events and signals as sample_world / make_world_with_events, and
    world_arrivals regenerates any event range's arrivals bit-exactly"""
    import paper_1612_00595_b200 as E
    from oracle.oracle import stations_line
    m = E.ModelConfig(lambda_rate=60 / 600.0, T=600.0, x_max=400.0, v=8.0,
                      stations=stations_line(40, 400.0))
    for dt in (E.F64, E.F32):
        ev, sig = E.sample_world(m, 7, dtype=dt, threads=3)
        ev2, sig2 = E.sample_world_events(m, 7, dtype=dt, threads=5)
        assert ev2.arrivals is None and np.array_equal(ev.ids, ev2.ids)
        assert np.array_equal(ev.x, ev2.x) and np.array_equal(ev.t, ev2.t)
        assert np.array_equal(sig, sig2)
        rows = E.world_arrivals(m, 7, 10, ev.x[10:25], ev.t[10:25], threads=2)
        assert np.array_equal(rows, ev.arrivals[10:25])
    cx, ct = [20.0, 380.0, 200.0, 5.0], [30.0, 100.0, 590.0, 300.0]
    ev, sig = E.make_world_with_events(m, cx, ct, 9)
    ev2, sig2 = E.make_world_with_events_signals(m, cx, ct, 9, threads=3)
    assert np.array_equal(sig, sig2)
    assert np.array_equal(E.world_arrivals(m, 9, 0, cx, ct), ev.arrivals)
    # the reference's own generator on the default world (golden vectors)
    g = golden_world("w2", default_model())
    ev3, sig3 = E.sample_world_events(engine_model(default_model()), 2, threads=2)
    assert np.array_equal(sig3, g.signals)
