"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU oracle.

Loads either the plain-C restatement (oracle/libseis_oracle.so, prefix ``so_``)
or the reference compiled in place (oracle/_ref/libseisref.so, prefix ``sr_``)
behind one interface, so the same test reads against both. Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libseis_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libseisref.so")

i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double
P = C.c_void_p


class SoModel(C.Structure):
    _fields_ = [(n, f64) for n in ("lambda_rate", "T", "x_max", "v", "sigma_arrival", "t_s",
                                   "var_noise", "var_event", "sample_rate")] + [
        ("n_stations", i64), ("stations", P)]


class SoSampler(C.Structure):
    _fields_ = [("steps_per_epoch", i64), ("epochs", i64), ("n_regions", i64), ("seed", u64),
                ("burn_in_fraction", f64), ("record_every", i64), ("weights", f64 * 5),
                ("step_location_x", f64), ("step_location_t", f64), ("step_arrival", f64),
                ("step_joint", f64), ("rng_mode", i64), ("dynamic", i64), ("compact", i64)]


TAPE_DTYPE = np.dtype([
    ("epoch", "<i8"), ("color", "<i8"), ("region", "<i8"), ("slot", "<i8"), ("step", "<i8"),
    ("type", "<i8"), ("is_null", "<i8"), ("n_removed", "<i8"), ("n_added", "<i8"),
    ("u_drawn", "<i8"), ("scored", "<i8"), ("accepted", "<i8"), ("constrained_out", "<i8"),
    ("removed_id", "<u8", (2,)), ("added_id", "<u8", (2,)), ("added_x", "<f8", (2,)),
    ("added_t", "<f8", (2,)), ("logq_f", "<f8"), ("logq_r", "<f8"), ("u", "<f8"),
    ("delta", "<f8"), ("log_r", "<f8"), ("added_arr_off", "<i8")])
assert TAPE_DTYPE.itemsize == 216


@dataclass
class Model:
    """reference ModelConfig (model.hpp:55-104); defaults are the reference's."""
    lambda_rate: float = 0.02
    T: float = 240.0
    x_max: float = 100.0
    v: float = 2.0
    sigma_arrival: float = 2.0
    t_s: float = 20.0
    var_noise: float = 1.0
    var_event: float = 4.0
    sample_rate: float = 1.0
    stations: np.ndarray = field(default_factory=lambda: np.array([0.0, 33.0, 66.0, 100.0]))

    @property
    def S(self) -> int:
        return len(self.stations)

    @property
    def n(self) -> int:
        return int(round(self.sample_rate * self.T))

    def c(self):
        st = np.ascontiguousarray(self.stations, dtype=np.float64)
        m = SoModel(self.lambda_rate, self.T, self.x_max, self.v, self.sigma_arrival, self.t_s,
                    self.var_noise, self.var_event, self.sample_rate, len(st),
                    st.ctypes.data_as(P))
        m._keep = st
        return m


@dataclass
class Sampler:
    """reference SamplerConfig (samplers.hpp:47-71) for the chromatic drivers."""
    steps_per_epoch: int = 500
    epochs: int = 100
    n_regions: int = 4
    seed: int = 1
    burn_in_fraction: float = 0.5
    record_every: int = 1000
    weights: tuple = (0.2, 0.2, 0.3, 0.2, 0.1)
    step_location_x: float = 4.0
    step_location_t: float = 4.0
    step_arrival: float = 1.0
    step_joint: float = 1.0
    rng_mode: int = 0
    dynamic: int = 0
    compact: int = 0  # rng_mode 1: generated arrival versions (philox stream spec v2)

    def c(self):
        return SoSampler(self.steps_per_epoch, self.epochs, self.n_regions, self.seed,
                         self.burn_in_fraction, self.record_every, (f64 * 5)(*self.weights),
                         self.step_location_x, self.step_location_t, self.step_arrival,
                         self.step_joint, self.rng_mode, self.dynamic, self.compact)


@dataclass
class Events:
    ids: np.ndarray
    x: np.ndarray
    t: np.ndarray
    arr: np.ndarray  # [N, S]

    @property
    def N(self) -> int:
        return len(self.ids)

    @staticmethod
    def empty(S: int) -> "Events":
        return Events(np.zeros(0, np.uint64), np.zeros(0), np.zeros(0), np.zeros((0, S)))


@dataclass
class World:
    model: Model
    events: Events
    signals: np.ndarray  # [S, n] station-major fp64


def _p(a):
    return a.ctypes.data_as(P) if a is not None and a.size else None


def build(quiet: bool = True) -> None:
    """Compile oracle/libseis_oracle.so (+ oracle/_ref when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


REF_INC = "/root/reference/proj/include"
BINDING_CHECK = os.path.join(HERE, "_ref", "binding_check")


def build_binding() -> str | None:
    """Compile tests/binding/binding_check.cpp — include/seis_b200.hpp (the
    C++ binding of INTEGRATION.md) against the unmodified reference headers,
    linked to the engine library — into oracle/_ref/binding_check. Needs the
    reference tree (this container) and the built engine; the binary travels
    to the GPU box. Returns the path, or None when it cannot be built here."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tests", "binding", "binding_check.cpp")
    lib = os.path.join(root, "paper_1612_00595_b200", "_lib")
    deps = [src, os.path.join(root, "include", "seis_b200.hpp"),
            os.path.join(root, "include", "seis_b200.h"), os.path.join(lib, "libseis_b200.so")]
    if not os.path.isdir(os.path.join(REF_INC, "seismic")) or not os.path.exists(deps[-1]):
        return BINDING_CHECK if os.path.exists(BINDING_CHECK) else None
    if os.path.exists(BINDING_CHECK) and all(
            os.path.getmtime(d) <= os.path.getmtime(BINDING_CHECK) for d in deps):
        return BINDING_CHECK
    os.makedirs(os.path.dirname(BINDING_CHECK), exist_ok=True)
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-pthread", "-I", REF_INC,
                    "-I", os.path.join(root, "include"), src, "-L", lib, "-lseis_b200",
                    "-Wl,-rpath,$ORIGIN/../../paper_1612_00595_b200/_lib", "-o", BINDING_CHECK],
                   check=True)
    return BINDING_CHECK


class Oracle:
    def __init__(self, which: str = "c"):
        path, pre = (ORACLE_SO, "so_") if which == "c" else (REF_SO, "sr_")
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.which = which
        self.lib = C.CDLL(path)
        self.pre = pre
        L = self.lib
        g = lambda n: getattr(L, pre + n)  # noqa: E731
        self._delta = g("delta")
        self._delta.restype = f64
        self._delta.argtypes = [P, P, i64, P, P, P, P, i64, P, i64, P, P, P, P, i64, i64, f64,
                                f64, i64]
        self._lj = g("log_joint")
        self._lj.restype = f64
        self._lj.argtypes = [P, P, i64, P, P, P, P]
        self._sw = g("sample_world")
        self._sw.argtypes = [P, u64, i64, P, P, P, P, P, P]
        self._sw.restype = C.c_int
        self._mw = g("make_world_with_events")
        self._mw.argtypes = [P, i64, P, P, u64, P, P, P, P, P]
        self._mw.restype = C.c_int
        self._part = g("partition")
        self._part.argtypes = [f64, f64, f64, f64, i64, P, P, P, P]
        self._part.restype = C.c_int
        self._rof = g("region_of")
        self._rof.argtypes = [P, i64, f64]
        self._rof.restype = i64
        self._off = g("partition_offset")
        self._off.argtypes = [u64, i64, f64]
        self._off.restype = f64
        self._sigw = g("signal_window")
        self._sigw.argtypes = [f64, f64, f64, f64, f64, P, P]
        self._ar = g("arrival_range")
        self._ar.argtypes = [P, f64, P, P]
        self._err = g("last_error")
        self._err.restype = C.c_char_p
        self._run = g("run_chromatic")
        self._run.restype = P
        self._run.argtypes = [P, P, P, i64, P, P, P, P, i64, i64]
        self._naive = g("run_naive")
        self._naive.restype = P
        self._naive.argtypes = [P, P, P, i64, i64]
        self._serial = g("run_serial")
        self._serial.restype = P
        self._serial.argtypes = [P, P, P, i64, P, P, P, P, i64, i64]
        for n in ("run_status",):
            getattr(L, pre + n).argtypes = [P]
        g("run_counts").argtypes = [P] + [P] * 6
        g("run_tape").argtypes = [P, P, P]
        g("run_rows").argtypes = [P, P, P, P]
        g("run_final").argtypes = [P, P, P, P, P]
        g("run_free").argtypes = [P]

    def err(self) -> str:
        return self._err().decode()

    # -- worldgen.hpp
    def sample_world(self, model: Model, seed: int, cap: int = 1 << 16) -> World:
        S, n = model.S, model.n
        ids = np.zeros(cap, np.uint64)
        x = np.zeros(cap)
        t = np.zeros(cap)
        arr = np.zeros((cap, S))
        sig = np.zeros((S, n))
        N = i64(0)
        m = model.c()
        rc = self._sw(C.byref(m), seed, cap, C.byref(N), _p(ids), _p(x), _p(t), _p(arr), _p(sig))
        if rc:
            raise RuntimeError(self.err())
        k = N.value
        return World(model, Events(ids[:k].copy(), x[:k].copy(), t[:k].copy(),
                                   arr[:k].copy()), sig)

    def make_world_with_events(self, model: Model, cx, ct, seed: int) -> World:
        S, n = model.S, model.n
        cx = np.ascontiguousarray(cx, np.float64)
        ct = np.ascontiguousarray(ct, np.float64)
        k = len(cx)
        ids = np.zeros(max(k, 1), np.uint64)
        x = np.zeros(max(k, 1))
        t = np.zeros(max(k, 1))
        arr = np.zeros((max(k, 1), S))
        sig = np.zeros((S, n))
        m = model.c()
        rc = self._mw(C.byref(m), k, _p(cx), _p(ct), seed, _p(ids), _p(x), _p(t), _p(arr),
                      _p(sig))
        if rc:
            raise RuntimeError(self.err())
        return World(model, Events(ids[:k].copy(), x[:k].copy(), t[:k].copy(),
                                   arr[:k].copy()), sig)

    # -- density.hpp
    def log_joint(self, model: Model, signals, ev: Events) -> float:
        m = model.c()
        sig = np.ascontiguousarray(signals, np.float64)
        arr = np.ascontiguousarray(ev.arr, np.float64)
        ids = np.ascontiguousarray(ev.ids, np.uint64)
        x = np.ascontiguousarray(ev.x, np.float64)
        t = np.ascontiguousarray(ev.t, np.float64)
        return self._lj(C.byref(m), _p(sig), ev.N, _p(ids), _p(x), _p(t), _p(arr))

    def delta(self, model: Model, signals, ev: Events, removed_idx, added: Events | None,
              window=None, support=None) -> float:
        m = model.c()
        sig = np.ascontiguousarray(signals, np.float64)
        arr = np.ascontiguousarray(ev.arr, np.float64)
        ids = np.ascontiguousarray(ev.ids, np.uint64)
        x = np.ascontiguousarray(ev.x, np.float64)
        t = np.ascontiguousarray(ev.t, np.float64)
        ridx = np.ascontiguousarray(removed_idx, np.int64)
        if added is None:
            added = Events.empty(model.S)
        aid = np.ascontiguousarray(added.ids, np.uint64)
        ax = np.ascontiguousarray(added.x, np.float64)
        at = np.ascontiguousarray(added.t, np.float64)
        aarr = np.ascontiguousarray(added.arr, np.float64)
        wlo, whi = window if window is not None else (0, model.n)
        slo, shi, sc = support if support is not None else (0.0, model.T, 1)
        return self._delta(C.byref(m), _p(sig), ev.N, _p(ids), _p(x), _p(t), _p(arr), len(ridx),
                           _p(ridx), added.N, _p(aid), _p(ax), _p(at), _p(aarr), wlo, whi, slo,
                           shi, sc)

    def arrival_range(self, model: Model, a: float):
        m = model.c()
        lo, hi = i64(0), i64(0)
        self._ar(C.byref(m), a, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    # -- partition.hpp
    def partition(self, T, l, offset, tau):
        cap = int(T / l) + 16 if l > 0 else 16
        b = np.zeros(cap)
        col = np.zeros(cap, np.int32)
        nr = i64(0)
        nc = C.c_int32(0)
        rc = self._part(T, l, offset, tau, cap, C.byref(nr), _p(b), _p(col), C.byref(nc))
        if rc:
            return rc, self.err(), None, None, 0
        k = nr.value
        return 0, "", b[:k + 1].copy(), col[:k].copy(), nc.value

    def region_of(self, boundaries, t) -> int:
        b = np.ascontiguousarray(boundaries, np.float64)
        return self._rof(_p(b), len(b) - 1, t)

    def partition_offset(self, seed, epoch, l) -> float:
        return self._off(seed, epoch, l)

    def signal_window(self, lo, hi, tau, T, rate):
        a, b = i64(0), i64(0)
        self._sigw(lo, hi, tau, T, rate, C.byref(a), C.byref(b))
        return a.value, b.value

    # -- evaluation.hpp
    def match_events(self, truth: Events, inferred: Events, threshold: float = 12.0):
        """match_events (evaluation.hpp:51-103) -> (precision, recall, location_error, n)."""
        f = getattr(self.lib, self.pre + "match_events")
        f.argtypes = [i64, P, P, P, i64, P, P, P, f64, P]
        f.restype = C.c_int
        out = np.zeros(4)
        a = [np.ascontiguousarray(v, dt) for v, dt in ((truth.ids, np.uint64), (truth.x, np.float64),
                                                        (truth.t, np.float64))]
        b = [np.ascontiguousarray(v, dt) for v, dt in ((inferred.ids, np.uint64),
                                                        (inferred.x, np.float64),
                                                        (inferred.t, np.float64))]
        rc = f(truth.N, *[_p(v) for v in a], inferred.N, *[_p(v) for v in b], threshold, _p(out))
        if rc:
            raise ValueError(self.err())
        return out[0], out[1], out[2], int(out[3])

    # -- samplers.hpp
    def run_chromatic(self, world: World, sampler: Sampler, init: Events | None = None,
                      tape: bool = True, rowlj: bool = False, naive: bool = False,
                      serial: bool = False) -> dict:
        model = world.model
        m = model.c()
        s = sampler.c()
        sig = np.ascontiguousarray(world.signals, np.float64)
        if init is None:
            init = Events.empty(model.S)
        ids = np.ascontiguousarray(init.ids, np.uint64)
        x = np.ascontiguousarray(init.x, np.float64)
        t = np.ascontiguousarray(init.t, np.float64)
        arr = np.ascontiguousarray(init.arr, np.float64)
        pre = self.pre
        if naive:
            h = self._naive(C.byref(m), _p(sig), C.byref(s), int(tape), int(rowlj))
        elif serial:
            h = self._serial(C.byref(m), _p(sig), C.byref(s), init.N, _p(ids), _p(x), _p(t),
                             _p(arr), int(tape), int(rowlj))
        else:
            h = self._run(C.byref(m), _p(sig), C.byref(s), init.N, _p(ids), _p(x), _p(t),
                          _p(arr), int(tape), int(rowlj))
        L = self.lib
        try:
            st = getattr(L, pre + "run_status")(h)
            if st:
                raise RuntimeError(f"run status {st}: {self.err()}")
            cnt = [i64(0) for _ in range(6)]
            getattr(L, pre + "run_counts")(h, *[C.byref(c) for c in cnt])
            n_tape, n_tarr, n_rows, n_final, total_steps, total_acc = [c.value for c in cnt]
            recs = np.zeros(n_tape, TAPE_DTYPE)
            tarr = np.zeros(max(n_tarr, 1))
            getattr(L, pre + "run_tape")(h, _p(recs), _p(tarr))
            rs = np.zeros(n_rows, np.int64)
            rl = np.zeros(n_rows)
            rc = np.zeros(n_rows, np.int64)
            getattr(L, pre + "run_rows")(h, _p(rs), _p(rl), _p(rc))
            S = model.S
            fi = np.zeros(max(n_final, 1), np.uint64)
            fx = np.zeros(max(n_final, 1))
            ft = np.zeros(max(n_final, 1))
            fa = np.zeros((max(n_final, 1), S))
            getattr(L, pre + "run_final")(h, _p(fi), _p(fx), _p(ft), _p(fa))
        finally:
            getattr(L, pre + "run_free")(h)
        return dict(tape=recs, tape_arr=tarr[:n_tarr], row_step=rs, row_lj=rl, row_count=rc,
                    final=Events(fi[:n_final], fx[:n_final], ft[:n_final], fa[:n_final]),
                    total_steps=total_steps, total_accepted=total_acc)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref_run_sampler(world: World, sampler: Sampler, workers: int = 1, cap: int = 1 << 16,
                    naive: bool = False, serial: bool = False):
    """The reference's own run_sampler (chromatic static/dynamic, naive or
    serial, from empty)."""
    if naive or serial:
        import copy
        sampler = copy.copy(sampler)
        sampler.dynamic = 2 if naive else 3
    L = C.CDLL(REF_SO)
    f = L.sr_run_sampler
    f.argtypes = [P, P, P, i64, i64, P, P, P, P, P, P, P, P]
    m = world.model.c()
    s = sampler.c()
    S = world.model.S
    ids = np.zeros(cap, np.uint64)
    x = np.zeros(cap)
    t = np.zeros(cap)
    arr = np.zeros((cap, S))
    n = i64(0)
    ts = i64(0)
    ta = i64(0)
    wall = f64(0)
    sig = np.ascontiguousarray(world.signals, np.float64)
    rc = f(C.byref(m), _p(sig), C.byref(s), workers, cap, C.byref(n), _p(ids), _p(x), _p(t),
           _p(arr), C.byref(ts), C.byref(ta), C.byref(wall))
    if rc:
        L.sr_last_error.restype = C.c_char_p
        raise RuntimeError(L.sr_last_error().decode())
    k = n.value
    return dict(final=Events(ids[:k], x[:k], t[:k], arr[:k]), total_steps=ts.value,
                total_accepted=ta.value, wall=wall.value)


def ref_bench_region_steps(world: World, truth: Events, sampler: Sampler, threads: int,
                           seconds: float, max_steps: int):
    """CPU baseline: reference run_region_steps per thread on the truth world."""
    L = C.CDLL(REF_SO)
    f = L.sr_bench_region_steps
    f.argtypes = [P, P, i64, P, P, P, P, P, i64, f64, i64, P, P]
    m = world.model.c()
    s = sampler.c()
    sig = np.ascontiguousarray(world.signals, np.float64)
    ids = np.ascontiguousarray(truth.ids, np.uint64)
    x = np.ascontiguousarray(truth.x, np.float64)
    t = np.ascontiguousarray(truth.t, np.float64)
    arr = np.ascontiguousarray(truth.arr, np.float64)
    props = i64(0)
    wall = f64(0)
    rc = f(C.byref(m), _p(sig), truth.N, _p(ids), _p(x), _p(t), _p(arr), C.byref(s), threads,
           seconds, max_steps, C.byref(props), C.byref(wall))
    if rc:
        L.sr_last_error.restype = C.c_char_p
        raise RuntimeError(L.sr_last_error().decode())
    return props.value, wall.value


def ref_thomas_events(seed, x_max, T, parent_mean=2000.0, child_mean=10.0, sx=50.0, st=None,
                      cap=1 << 20):
    """Thomas cluster process of config[4] drawn with the reference's own Rng
    (oracle/_ref sr_thomas_events); returns (cx, ct)."""
    L = C.CDLL(REF_SO)
    f = L.sr_thomas_events
    f.argtypes = [u64, f64, f64, f64, f64, f64, f64, i64, P, P, P]
    st = 0.0015625 * T if st is None else st
    cx = np.zeros(cap)
    ct = np.zeros(cap)
    n = i64(0)
    rc = f(seed, x_max, T, parent_mean, child_mean, sx, st, cap, C.byref(n), _p(cx), _p(ct))
    if rc:
        L.sr_last_error.restype = C.c_char_p
        raise RuntimeError(L.sr_last_error().decode())
    return cx[:n.value].copy(), ct[:n.value].copy()


def philox(c, k):
    L = C.CDLL(ORACLE_SO)
    o = (C.c_uint32 * 4)()
    L.so_philox(*[C.c_uint32(v) for v in (*c, *k)], o)
    return list(o)


def philox_normal(seed, sweep, region, step, i):
    L = C.CDLL(ORACLE_SO)
    L.so_philox_normal.restype = C.c_float
    L.so_philox_normal.argtypes = [u64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
    return L.so_philox_normal(seed, sweep, region, step, i)


def stations_line(S: int, x_max: float) -> np.ndarray:
    """SURVEY §8(d) mapping: S stations evenly spaced, s_j = x_max j / (S - 1)."""
    return x_max * np.arange(S, dtype=np.float64) / (S - 1)
