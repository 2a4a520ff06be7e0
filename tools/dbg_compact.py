import sys; sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
from tests.helpers import default_model, engine_model, engine_sampler, golden_world
import paper_1612_00595_b200 as E
m = default_model(); w = golden_world("w3", m)
s = O.Sampler(steps_per_epoch=150, epochs=10, n_regions=4, seed=23, dynamic=0, rng_mode=1, record_every=500, compact=1)
eng = E.Engine(engine_model(m), w.signals, event_capacity=4096)
print("storage before", eng.arrival_storage, "pool", eng.pool_slots)
eng.arrival_storage = "compact"
print("storage after", eng.arrival_storage)
tr = eng.run_chromatic(engine_sampler(s))
print({k: v for k, v in tr.stats.items()})
