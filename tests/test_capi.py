"""CPU: the C-ABI library loads and exports every symbol include/*.h declares;
the host-side world generator is bit-exact with the reference generator."""
import re
import os

import numpy as np

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
