"""Generates tests/golden/posterior_mapped.npz from the REFERENCE itself
(oracle/_ref): posterior statistics of the reference's own run_sampler on a
BASELINE-mapped shape (SURVEY §8(d) mapping with S = 96 evenly spaced
stations, l / tau_max = 1.2, 32 time regions, ~40 events), for the GPU
posterior-parity test (acceptance.cpp:154-194 style: final hypothesis
matched to the truth with match_events, evaluation.hpp:51-103).

    python tests/golden/make_golden_mapped.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

# mapped shape: S, T, n_regions, x_max, expected events
SHAPE = (96, 1200.0, 32, 2000.0, 40.0)
SAMPLER = (100, 24, 32)  # steps_per_epoch, epochs, n_regions
THRESHOLD = 12.0 * 2000.0 / 100.0  # match radius scaled with x_max from the default world's 12


def mapped_model():
    S, T, nr, x_max, ev = SHAPE
    return O.Model(lambda_rate=ev / T, T=T, x_max=x_max, v=1.2 * x_max * nr / T,
                   stations=O.stations_line(S, x_max))


def main():
    O.build()
    assert O.have_ref(), "needs oracle/_ref (reference tree present)"
    R = O.Oracle("ref")
    m = mapped_model()
    k, ep, nr = SAMPLER
    rows = []
    for ws in range(4):
        w = R.sample_world(m, 500 + ws)
        for rs in (1, 2, 3):
            sc = O.Sampler(steps_per_epoch=k, epochs=ep, n_regions=nr, seed=rs, dynamic=1,
                           burn_in_fraction=0.0, record_every=1 << 30)
            r = O.ref_run_sampler(w, sc, workers=4)
            pr, rc, le, nm = R.match_events(w.events, r["final"], THRESHOLD)
            rows.append((500 + ws, rs, pr, rc, le, r["final"].N, w.events.N,
                         r["total_accepted"]))
            print(rows[-1], flush=True)
    np.savez_compressed(os.path.join(HERE, "posterior_mapped.npz"),
                        rows=np.array(rows, np.float64),
                        cols=np.array(["world_seed", "run_seed", "precision", "recall",
                                       "location_error", "n_final", "n_true", "accepted"]),
                        shape=np.array(SHAPE), sampler=np.array(SAMPLER),
                        threshold=np.array([THRESHOLD]))


if __name__ == "__main__":
    main()
