"""Shared test helpers: golden loading and model construction."""
import os

import numpy as np

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def default_model():
    return O.Model()


def wide_model():
    g = golden("worlds.npz")
    lam, T, x_max, v = g["wide_model"]
    return O.Model(lambda_rate=lam, T=T, x_max=x_max, v=v, stations=O.stations_line(64, x_max))


def golden_world(name, model):
    g = golden("worlds.npz")
    ev = O.Events(g[f"{name}_ids"], g[f"{name}_x"], g[f"{name}_t"], g[f"{name}_arr"])
    return O.World(model, ev, g[f"{name}_sig"])


def engine_model(m):
    """oracle Model -> engine ModelConfig"""
    from paper_1612_00595_b200 import ModelConfig
    return ModelConfig(lambda_rate=m.lambda_rate, T=m.T, x_max=m.x_max, v=m.v,
                       sigma_arrival=m.sigma_arrival, t_s=m.t_s, var_noise=m.var_noise,
                       var_event=m.var_event, sample_rate=m.sample_rate,
                       stations=np.array(m.stations, np.float64))


def tape_sampler(arr):
    k, epochs, n_regions, seed, dynamic = [int(v) for v in arr]
    return O.Sampler(steps_per_epoch=k, epochs=epochs, n_regions=n_regions, seed=seed,
                     dynamic=dynamic)


def engine_sampler(s, record_every=None, record_log_joint=False):
    from paper_1612_00595_b200 import SamplerConfig
    return SamplerConfig(algorithm="chromatic-dynamic" if s.dynamic else "chromatic-static",
                         steps_per_epoch=s.steps_per_epoch, epochs=s.epochs,
                         n_regions=s.n_regions, seed=s.seed,
                         burn_in_fraction=s.burn_in_fraction,
                         record_every=record_every or s.record_every, weights=s.weights,
                         step_location_x=s.step_location_x, step_location_t=s.step_location_t,
                         step_arrival=s.step_arrival, step_joint=s.step_joint,
                         record_log_joint=record_log_joint)
