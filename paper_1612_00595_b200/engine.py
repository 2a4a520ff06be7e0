"""Python mirror of the reference sampler/model API over the engine's C-ABI.

Names follow the reference (proj/include/seismic/): ``ModelConfig``
(model.hpp:55-104), ``SamplerConfig`` (samplers.hpp:47-71), ``run_chromatic`` /
``run_sampler`` (samplers.hpp:401-509), ``delta_log_joint`` (density.hpp:214-305,
batched here), ``log_joint`` (density.hpp:146-154), ``build_partition`` +
``color_partition`` (partition.hpp:40-90) and ``Partition.region_of``
(partition.hpp:33-37). Validation errors raise ``ValueError`` (the reference's
std::invalid_argument, CLI exit 2), runtime errors ``RuntimeError`` (exit 3).

Everything computes in libseis_b200.so on the GPU; there is no CPU fallback.
Loading fails loudly if the library is missing or no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import build as _build

i32, i64, u64, f64, P = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p

F32, F64 = 0, 1


class _ModelC(C.Structure):
    _fields_ = [(n, f64) for n in ("lambda_rate", "T", "x_max", "v", "sigma_arrival", "t_s",
                                   "var_noise", "var_event", "sample_rate")]


class _SamplerC(C.Structure):
    _fields_ = [("steps_per_epoch", i64), ("epochs", i64), ("n_regions", i64), ("seed", u64),
                ("burn_in_fraction", f64), ("record_every", i64), ("weights", f64 * 5),
                ("step_location_x", f64), ("step_location_t", f64), ("step_arrival", f64),
                ("step_joint", f64), ("dynamic", i32), ("record_log_joint", i32)]


class _ChangeC(C.Structure):
    _fields_ = [("n_removed", i32), ("n_added", i32), ("removed_id", u64 * 2),
                ("added_x", f64 * 2), ("added_t", f64 * 2), ("added_row", i64 * 2),
                ("window_lo", i64), ("window_hi", i64), ("support_lo", f64),
                ("support_hi", f64), ("support_closed", i32), ("pad_", i32)]


class _StatsC(C.Structure):
    _fields_ = [("total_steps", i64), ("total_accepted", i64), ("scored_proposals", i64),
                ("changed_samples", i64), ("arrival_values", i64), ("algorithmic_bytes", f64),
                ("sweep_kernel_ms", f64), ("total_ms", f64), ("kernel_launches", i64),
                ("n_rows", i64), ("final_events", i64), ("speculative_discarded", i64),
                ("phases", i64), ("generated_versions", i64)]


class _PhaseC(C.Structure):
    _fields_ = [("epoch", i64), ("color", i32), ("pad_", i32), ("region", i64), ("steps", i64)]


PHASE_DTYPE = np.dtype([("epoch", "<i8"), ("color", "<i4"), ("pad_", "<i4"), ("region", "<i8"),
                        ("steps", "<i8")])


TAPE_DTYPE = np.dtype([
    ("epoch", "<i8"), ("color", "<i8"), ("region", "<i8"), ("slot", "<i8"), ("step", "<i8"),
    ("type", "<i8"), ("is_null", "<i8"), ("n_removed", "<i8"), ("n_added", "<i8"),
    ("u_drawn", "<i8"), ("scored", "<i8"), ("accepted", "<i8"), ("constrained_out", "<i8"),
    ("removed_id", "<u8", (2,)), ("added_id", "<u8", (2,)), ("added_x", "<f8", (2,)),
    ("added_t", "<f8", (2,)), ("logq_f", "<f8"), ("logq_r", "<f8"), ("u", "<f8"),
    ("delta", "<f8"), ("log_r", "<f8"), ("added_arr_off", "<i8")])
STEP_OUT_DTYPE = np.dtype([("delta", "<f8"), ("log_r", "<f8"), ("scored", "<i4"),
                           ("accepted", "<i4")])

EXPORTS = ("seis_last_error", "seis_engine_create", "seis_engine_destroy", "seis_upload_signals",
           "seis_set_hypothesis", "seis_get_hypothesis", "seis_partition", "seis_assign_regions",
           "seis_partition_offset", "seis_score_batch", "seis_log_joint", "seis_run_chromatic",
           "seis_world_last_error", "seis_world_generate", "seis_world_with_events",
           "seis_thomas_events", "seis_set_snapshot_capacity", "seis_get_snapshots",
           "seis_run_naive", "seis_run_serial", "seis_engine_pool_slots", "seis_eval_last_error",
           "seis_match_events", "seis_bootstrap_ci", "seis_get_phases", "seis_get_row_wall",
           "seis_set_hypothesis_begin", "seis_set_hypothesis_rows", "seis_set_hypothesis_end",
           "seis_world_generate_events", "seis_world_with_events_signals", "seis_world_arrivals",
           "seis_set_arrival_storage", "seis_get_arrival_storage")

_LIB = None


def load_library(path: str | None = None) -> C.CDLL:
    """dlopen libseis_b200.so (in-tree). Raises if it is absent: no fallback."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    # SEIS_LIB: an alternative build of the same library (A/B measurements)
    path = path or os.environ.get("SEIS_LIB") or _build.LIB
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_1612_00595_b200.build` "
                          "(the engine has no CPU fallback)")
    L = C.CDLL(path)
    L.seis_last_error.restype = C.c_char_p
    L.seis_world_last_error.restype = C.c_char_p
    L.seis_engine_create.argtypes = [P, P, i64, P, i32, i64, P]
    L.seis_engine_destroy.argtypes = [P]
    L.seis_engine_pool_slots.argtypes = [P]
    L.seis_engine_pool_slots.restype = C.c_int64
    L.seis_upload_signals.argtypes = [P, P]
    L.seis_set_hypothesis.argtypes = [P, i64, P, P, P, P]
    L.seis_get_hypothesis.argtypes = [P, i64, P, P, P, P, P]
    L.seis_partition.argtypes = [f64, f64, f64, f64, i64, P, P, P, P]
    L.seis_assign_regions.argtypes = [P, i64, i64, P, P]
    L.seis_partition_offset.argtypes = [u64, i64, f64, P]
    L.seis_score_batch.argtypes = [P, i64, P, P, i64, P]
    L.seis_log_joint.argtypes = [P, P]
    L.seis_run_chromatic.argtypes = [P, P, i32, P, i64, P, i64, P, i64, P, P, P, P]
    L.seis_run_naive.argtypes = [P, P, i32, P, i64, P, i64, P, i64, P, P, P, P]
    L.seis_run_serial.argtypes = [P, P, i32, P, i64, P, i64, P, i64, P, P, P, P]
    L.seis_world_generate.argtypes = [P, P, i64, u64, i64, P, P, P, P, P, P, i32, i32]
    L.seis_world_with_events.argtypes = [P, P, i64, i64, P, P, u64, P, P, i32, i32]
    L.seis_thomas_events.argtypes = [u64, f64, f64, f64, f64, f64, f64, i64, P, P, P]
    L.seis_eval_last_error.restype = C.c_char_p
    L.seis_match_events.argtypes = [i64, P, P, P, i64, P, P, P, f64, P, P, P, P]
    L.seis_bootstrap_ci.argtypes = [P, i64, f64, i32, u64, P]
    L.seis_set_snapshot_capacity.argtypes = [P, i64, i64]
    L.seis_get_snapshots.argtypes = [P, i64, P, P, P, i64, P, P, P]
    L.seis_get_phases.argtypes = [P, i64, P, P]
    L.seis_set_hypothesis_begin.argtypes = [P, i64, P, P, P]
    L.seis_set_arrival_storage.argtypes = [P, i32]
    L.seis_get_arrival_storage.argtypes = [P]
    L.seis_get_arrival_storage.restype = i32
    L.seis_set_hypothesis_rows.argtypes = [P, i64, i64, P]
    L.seis_set_hypothesis_end.argtypes = [P]
    L.seis_world_generate_events.argtypes = [P, P, i64, u64, i64, P, P, P, P, P, i32, i32]
    L.seis_world_with_events_signals.argtypes = [P, P, i64, i64, P, P, u64, P, i32, i32]
    L.seis_world_arrivals.argtypes = [P, P, i64, u64, i64, i64, P, P, P, i32]
    L.seis_get_row_wall.argtypes = [P, i64, P, P]
    if path == _build.LIB:
        _LIB = L
    return L


def _p(a):
    return a.ctypes.data_as(P) if a is not None and a.size else None


def _check(rc: int, L=None):
    if rc == 0:
        return
    msg = (L or load_library()).seis_last_error().decode()
    if rc == 2:
        raise ValueError(msg)
    raise RuntimeError(msg)


@dataclass
class ModelConfig:
    """reference ModelConfig (model.hpp:55-65); defaults are the reference's."""
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

    def n_samples(self) -> int:
        return int(round(self.sample_rate * self.T))

    def n_stations(self) -> int:
        return len(self.stations)

    def tau_max(self) -> float:
        return self.x_max / self.v

    def _c(self):
        return _ModelC(self.lambda_rate, self.T, self.x_max, self.v, self.sigma_arrival,
                       self.t_s, self.var_noise, self.var_event, self.sample_rate)


@dataclass
class SamplerConfig:
    """reference SamplerConfig (samplers.hpp:47-58) for every driver:
    algorithm serial, naive, chromatic-static or chromatic-dynamic."""
    algorithm: str = "chromatic-static"
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
    record_log_joint: bool = False

    def _c(self):
        if self.algorithm not in ("chromatic-static", "chromatic-dynamic", "naive", "serial"):
            raise ValueError(f"unknown sampler '{self.algorithm}' (this engine runs "
                             "chromatic-static, chromatic-dynamic, naive or serial)")
        return _SamplerC(self.steps_per_epoch, self.epochs, self.n_regions, self.seed,
                         self.burn_in_fraction, self.record_every, (f64 * 5)(*self.weights),
                         self.step_location_x, self.step_location_t, self.step_arrival,
                         self.step_joint, int(self.algorithm == "chromatic-dynamic"),
                         int(self.record_log_joint))


@dataclass
class Events:
    """an event set (reference Event, model.hpp:44-53) as arrays."""
    ids: np.ndarray
    x: np.ndarray
    t: np.ndarray
    arrivals: np.ndarray | None  # [N, S]

    @property
    def N(self) -> int:
        return len(self.ids)


@dataclass
class Snapshot:
    """reference Snapshot (samplers.hpp:80-85): the hypothesis at a trace row."""
    id: int
    step: int
    ids: np.ndarray
    x: np.ndarray
    t: np.ndarray
    wall_seconds: float = 0.0


@dataclass
class Trace:
    """reference Trace (samplers.hpp:97-103) + engine measurement counters."""
    row_step: np.ndarray
    row_log_joint: np.ndarray
    row_count: np.ndarray
    total_steps: int
    total_accepted: int
    stats: dict
    final: Events | None = None
    step_out: np.ndarray | None = None
    snapshots: list = field(default_factory=list)
    # TraceRow::wall_seconds (device time since the run started, CUDA events)
    row_wall: np.ndarray | None = None
    # Trace::phases (PhaseRecord, samplers.hpp:87-95): PHASE_DTYPE records
    phases: np.ndarray | None = None

    def write_trace_csv(self, path: str) -> None:
        """write_trace_csv (samplers.hpp:511-516)."""
        wall = self.row_wall if self.row_wall is not None else np.zeros(len(self.row_step))
        with open(path, "w") as f:
            f.write("wall_seconds,step,log_joint,event_count\n")
            for w, st, lj, c in zip(wall, self.row_step, self.row_log_joint, self.row_count):
                f.write(f"{_fmt(w)},{int(st)},{_fmt(lj)},{int(c)}\n")

    def write_samples_csv(self, path: str) -> None:
        """write_samples_csv (samplers.hpp:518-524)."""
        with open(path, "w") as f:
            f.write("snapshot_id,event_id,x,t\n")
            for sn in self.snapshots:
                for i, x, t in zip(sn.ids, sn.x, sn.t):
                    f.write(f"{sn.id},{int(i)},{_fmt(x)},{_fmt(t)}\n")


def _fmt(v: float) -> str:
    """format_double (csv.hpp:15-19): shortest round-trip decimal."""
    v = float(v)
    if v == float("inf"):
        return "inf"
    if v == float("-inf"):
        return "-inf"
    r = repr(v)
    return r[:-2] if r.endswith(".0") else r


@dataclass
class Partition:
    """reference Partition after color_partition (partition.hpp:16-38)."""
    boundaries: np.ndarray
    colors: np.ndarray
    n_colors: int

    def n_regions(self) -> int:
        return len(self.boundaries) - 1

    def region_of(self, t):
        return assign_regions(self.boundaries, t)


def partition(T: float, l: float, offset: float, tau: float) -> Partition:
    """build_partition(T, l, offset) + color_partition(., tau), on the GPU."""
    L = load_library()
    cap = int(T / l) + 16 if (l > 0 and np.isfinite(T / l)) else 16
    b = np.zeros(cap)
    c = np.zeros(cap, np.int32)
    nr = i64(0)
    nc = i32(0)
    _check(L.seis_partition(T, l, offset, tau, cap, C.byref(nr), _p(b), _p(c), C.byref(nc)), L)
    k = nr.value
    return Partition(b[:k + 1].copy(), c[:k].copy(), nc.value)


def assign_regions(boundaries, t) -> np.ndarray:
    """Partition::region_of for every t, on the GPU."""
    L = load_library()
    b = np.ascontiguousarray(boundaries, np.float64)
    t = np.ascontiguousarray(np.atleast_1d(t), np.float64)
    out = np.zeros(len(t), np.int64)
    _check(L.seis_assign_regions(_p(b), len(b) - 1, len(t), _p(t), _p(out)), L)
    return out


def partition_offset(seed: int, epoch: int, l: float) -> float:
    """dynamic-partition offset of `epoch` (samplers.hpp:488-491), on the GPU."""
    L = load_library()
    u = f64(0)
    _check(L.seis_partition_offset(seed, epoch, l, C.byref(u)), L)
    return u.value


def sample_world(config: ModelConfig, seed: int, dtype=F64, threads: int = 0,
                 cap: int = 1 << 20):
    """reference sample_world (worldgen.hpp:20-53): (Events, signals [S][n])."""
    L = load_library()
    threads = threads or os.cpu_count() or 1
    S, n = config.n_stations(), config.n_samples()
    lam = config.lambda_rate * config.T
    cap = int(min(cap, lam + 20 * np.sqrt(lam) + 64))
    st = np.ascontiguousarray(config.stations, np.float64)
    ids = np.zeros(cap, np.uint64)
    x = np.zeros(cap)
    t = np.zeros(cap)
    arr = np.zeros((cap, S))
    sig = np.zeros((S, n), np.float64 if dtype == F64 else np.float32)
    N = i64(0)
    m = config._c()
    rc = L.seis_world_generate(C.byref(m), _p(st), S, seed, cap, C.byref(N), _p(ids), _p(x),
                               _p(t), _p(arr), _p(sig), dtype, threads)
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    k = N.value
    return Events(ids[:k].copy(), x[:k].copy(), t[:k].copy(), arr[:k].copy()), sig


def make_world_with_events(config: ModelConfig, cx, ct, seed: int, dtype=F64, threads: int = 0):
    """reference make_world_with_events (worldgen.hpp:57-86)."""
    L = load_library()
    threads = threads or os.cpu_count() or 1
    S, n = config.n_stations(), config.n_samples()
    cx = np.ascontiguousarray(cx, np.float64)
    ct = np.ascontiguousarray(ct, np.float64)
    N = len(cx)
    st = np.ascontiguousarray(config.stations, np.float64)
    arr = np.zeros((max(N, 1), S))
    sig = np.zeros((S, n), np.float64 if dtype == F64 else np.float32)
    m = config._c()
    rc = L.seis_world_with_events(C.byref(m), _p(st), S, N, _p(cx), _p(ct), seed, _p(arr),
                                  _p(sig), dtype, threads)
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    return Events(np.arange(N, dtype=np.uint64), cx.copy(), ct.copy(), arr[:N].copy()), sig


def sample_world_events(config: ModelConfig, seed: int, dtype=F64, threads: int = 0,
                        cap: int = 1 << 22):
    """sample_world (worldgen.hpp:20-53) streamed: the events without their
    N x S arrivals (Events.arrivals is None) and the signals, identical to
    sample_world's; arrivals on demand with world_arrivals."""
    L = load_library()
    threads = threads or os.cpu_count() or 1
    S, n = config.n_stations(), config.n_samples()
    lam = config.lambda_rate * config.T
    cap = int(min(cap, lam + 20 * np.sqrt(lam) + 64))
    st = np.ascontiguousarray(config.stations, np.float64)
    ids = np.zeros(cap, np.uint64)
    x = np.zeros(cap)
    t = np.zeros(cap)
    sig = np.zeros((S, n), np.float64 if dtype == F64 else np.float32)
    N = i64(0)
    m = config._c()
    rc = L.seis_world_generate_events(C.byref(m), _p(st), S, seed, cap, C.byref(N), _p(ids),
                                      _p(x), _p(t), _p(sig), dtype, threads)
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    k = N.value
    return Events(ids[:k].copy(), x[:k].copy(), t[:k].copy(), None), sig


def make_world_with_events_signals(config: ModelConfig, cx, ct, seed: int, dtype=F64,
                                   threads: int = 0):
    """make_world_with_events (worldgen.hpp:57-86) streamed (arrivals None)."""
    L = load_library()
    threads = threads or os.cpu_count() or 1
    S, n = config.n_stations(), config.n_samples()
    cx = np.ascontiguousarray(cx, np.float64)
    ct = np.ascontiguousarray(ct, np.float64)
    st = np.ascontiguousarray(config.stations, np.float64)
    sig = np.zeros((S, n), np.float64 if dtype == F64 else np.float32)
    m = config._c()
    rc = L.seis_world_with_events_signals(C.byref(m), _p(st), S, len(cx), _p(cx), _p(ct), seed,
                                          _p(sig), dtype, threads)
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    return Events(np.arange(len(cx), dtype=np.uint64), cx.copy(), ct.copy(), None), sig


def world_arrivals(config: ModelConfig, seed: int, i0: int, x, t, threads: int = 0,
                   out: np.ndarray | None = None) -> np.ndarray:
    """Arrivals [n][S] of events i0 .. i0 + n - 1 of a generated world (their
    per-event streams, worldgen.hpp:34-38), x / t those events' coordinates."""
    L = load_library()
    threads = threads or os.cpu_count() or 1
    S = config.n_stations()
    x = np.ascontiguousarray(x, np.float64)
    t = np.ascontiguousarray(t, np.float64)
    n = len(x)
    if out is None:
        out = np.zeros((n, S))
    st = np.ascontiguousarray(config.stations, np.float64)
    m = config._c()
    rc = L.seis_world_arrivals(C.byref(m), _p(st), S, seed, i0, n, _p(x), _p(t), _p(out),
                               threads)
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    return out


# ------------------------------------------------------------ world files
# "seis world v1": a binary world (model, events with arrivals, signals) in
# place of the reference's CSV files (worldgen.hpp:157-161; 268 M rows at
# config[4]). Layout: 8-byte magic, u64 header length, JSON header, then the
# arrays at 64-byte-aligned offsets listed in the header, little-endian.
# load_world maps them without copying, so Engine uploads straight from the
# page cache.
_WORLD_MAGIC = b"SEISWLD1"
_MODEL_FIELDS = ("lambda_rate", "T", "x_max", "v", "sigma_arrival", "t_s", "var_noise",
                 "var_event", "sample_rate")


def save_world(path: str, config: ModelConfig, events: "Events", signals: np.ndarray) -> None:
    S, n = config.n_stations(), config.n_samples()
    sig = np.ascontiguousarray(signals)
    if sig.dtype not in (np.float32, np.float64) or sig.shape != (S, n):
        raise ValueError(f"signals must be float32/float64 [S={S}][n={n}]")
    N = len(events.ids)
    arrays = [("stations", np.ascontiguousarray(config.stations, "<f8")),
              ("ids", np.ascontiguousarray(events.ids, "<u8")),
              ("x", np.ascontiguousarray(events.x, "<f8")),
              ("t", np.ascontiguousarray(events.t, "<f8")),
              ("arrivals", np.ascontiguousarray(events.arrivals, "<f8").reshape(N, S)),
              ("signals", sig.astype(sig.dtype.newbyteorder("<"), copy=False))]
    head = {"version": 1, "model": {k: float(getattr(config, k)) for k in _MODEL_FIELDS},
            "S": S, "n": n, "N": N, "signal_dtype": "f32" if sig.dtype == np.float32 else "f64",
            "arrays": {}}
    # two passes: offsets depend on the header length
    for _ in range(2):
        hb = json.dumps(head, sort_keys=True).encode()
        off = (16 + len(hb) + 63) // 64 * 64
        for name, a in arrays:
            head["arrays"][name] = [off, a.nbytes]
            off = (off + a.nbytes + 63) // 64 * 64
    hb = json.dumps(head, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(_WORLD_MAGIC)
        f.write(np.uint64(len(hb)).tobytes())
        f.write(hb)
        for name, a in arrays:
            f.seek(head["arrays"][name][0])
            f.write(a.tobytes(order="C"))
        f.truncate(max(v[0] + v[1] for v in head["arrays"].values()))


def load_world(path: str):
    """-> (ModelConfig, Events, signals [S][n]); arrays are read-only memory maps."""
    with open(path, "rb") as f:
        if f.read(8) != _WORLD_MAGIC:
            raise ValueError(f"{path}: not a seis world v1 file")
        hl = int(np.frombuffer(f.read(8), "<u8")[0])
        head = json.loads(f.read(hl))
    if head.get("version") != 1:
        raise ValueError(f"{path}: unsupported world version {head.get('version')}")
    S, n, N = head["S"], head["n"], head["N"]
    sd = "<f4" if head["signal_dtype"] == "f32" else "<f8"
    shapes = {"stations": ("<f8", (S,)), "ids": ("<u8", (N,)), "x": ("<f8", (N,)),
              "t": ("<f8", (N,)), "arrivals": ("<f8", (N, S)), "signals": (sd, (S, n))}
    out = {}
    for name, (dt, shape) in shapes.items():
        off, nb = head["arrays"][name]
        if nb == 0:
            out[name] = np.zeros(shape, dt)
        else:
            out[name] = np.memmap(path, dtype=dt, mode="r", offset=off, shape=shape)
    cfg = ModelConfig(**head["model"], stations=np.array(out["stations"]))
    return cfg, Events(out["ids"], out["x"], out["t"], out["arrivals"]), out["signals"]


def thomas_events(seed, x_max, T, parent_mean, child_mean, sx, st, cap=1 << 22):
    L = load_library()
    cx = np.zeros(cap)
    ct = np.zeros(cap)
    n = i64(0)
    rc = L.seis_thomas_events(seed, x_max, T, parent_mean, child_mean, sx, st, cap, C.byref(n),
                              _p(cx), _p(ct))
    if rc:
        raise RuntimeError(L.seis_world_last_error().decode())
    return cx[:n.value].copy(), ct[:n.value].copy()


# ---------------------------------------------------------------- evaluation
class _MatchC(C.Structure):
    _fields_ = [("precision", f64), ("recall", f64), ("location_error", f64),
                ("n_true", i64), ("n_inferred", i64), ("n_matched", i64)]


class _CIC(C.Structure):
    _fields_ = [("mean", f64), ("lo", f64), ("hi", f64), ("level", f64), ("resamples", i32)]


@dataclass
class MatchReport:
    """reference MatchReport (evaluation.hpp:35-43); pairs in truth (t, x) order."""
    precision: float
    recall: float
    location_error: float
    n_true: int
    n_inferred: int
    n_matched: int
    pair_true_id: np.ndarray
    pair_inferred_id: np.ndarray
    pair_distance: np.ndarray


@dataclass
class BootstrapCI:
    """reference BootstrapCI (evaluation.hpp:128-134)."""
    mean: float
    lo: float
    hi: float
    level: float
    resamples: int


def _points(ev):
    ids = np.ascontiguousarray(ev.ids, np.uint64)
    return ids, np.ascontiguousarray(ev.x, np.float64), np.ascontiguousarray(ev.t, np.float64)


def _eval_check(rc, L):
    if rc == 2:
        raise ValueError(L.seis_eval_last_error().decode())
    if rc:
        raise RuntimeError(L.seis_eval_last_error().decode())


def match_events(true_events, inferred_events, threshold: float = 12.0) -> MatchReport:
    """match_events (evaluation.hpp:51-105): greedy nearest matching in (x, t),
    pairs within `threshold` in both |dt| and |dx|. Accepts anything with
    ids/x/t (Events, Snapshot)."""
    L = load_library()
    ti, tx, tt = _points(true_events)
    ii, ix, it = _points(inferred_events)
    k = max(1, min(len(ti), len(ii)))
    pt, pi, pd = np.zeros(k, np.uint64), np.zeros(k, np.uint64), np.zeros(k)
    r = _MatchC()
    _eval_check(L.seis_match_events(len(ti), _p(ti), _p(tx), _p(tt), len(ii), _p(ii), _p(ix),
                                    _p(it), float(threshold), C.byref(r), _p(pt), _p(pi),
                                    _p(pd)), L)
    m = r.n_matched
    return MatchReport(r.precision, r.recall, r.location_error, r.n_true, r.n_inferred, m,
                       pt[:m].copy(), pi[:m].copy(), pd[:m].copy())


def metric_trace(snapshots, true_events, threshold: float = 12.0) -> list:
    """metric_trace (evaluation.hpp:115-126): (snapshot id, precision, recall,
    location error) per snapshot (no wall-clock column, see Trace)."""
    if not snapshots:
        raise ValueError("metric_trace: no snapshots")
    out = []
    for sn in snapshots:
        r = match_events(true_events, sn, threshold)
        out.append((sn.id, r.precision, r.recall, r.location_error))
    return out


def bootstrap_ci(values, level: float = 0.95, resamples: int = 1000, seed: int = 0) -> BootstrapCI:
    """bootstrap_ci (evaluation.hpp:136-169): percentile bootstrap of the mean
    on the reference's kBootstrap stream (bit-exact)."""
    L = load_library()
    v = np.ascontiguousarray(values, np.float64)
    out = _CIC()
    _eval_check(L.seis_bootstrap_ci(_p(v), len(v), float(level), int(resamples), int(seed),
                                    C.byref(out)), L)
    return BootstrapCI(out.mean, out.lo, out.hi, out.level, out.resamples)


class Engine:
    """World{config, events, signals} resident on one B200 (seis_engine)."""

    def __init__(self, config: ModelConfig, signals: np.ndarray, event_capacity: int = 4096):
        self.L = load_library()
        self.config = config
        sig = np.ascontiguousarray(signals)
        if sig.dtype == np.float64:
            self.dtype = F64
        elif sig.dtype == np.float32:
            self.dtype = F32
        else:
            raise ValueError("signals must be float32 or float64")
        if sig.shape != (config.n_stations(), config.n_samples()):
            raise ValueError(f"signals must be [S={config.n_stations()}][n={config.n_samples()}]")
        st = np.ascontiguousarray(config.stations, np.float64)
        h = P()
        m = config._c()
        _check(self.L.seis_engine_create(C.byref(m), _p(st), len(st), _p(sig), self.dtype,
                                         event_capacity, C.byref(h)), self.L)
        self.h = h
        self.capacity = event_capacity
        self.pool_slots = int(self.L.seis_engine_pool_slots(h))

    def close(self):
        if getattr(self, "h", None):
            self.L.seis_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def upload_signals(self, signals: np.ndarray):
        sig = np.ascontiguousarray(signals, np.float64 if self.dtype == F64 else np.float32)
        _check(self.L.seis_upload_signals(self.h, _p(sig)), self.L)

    def set_hypothesis(self, ev: Events):
        S = self.config.n_stations()
        ids = np.ascontiguousarray(ev.ids, np.uint64)
        x = np.ascontiguousarray(ev.x, np.float64)
        t = np.ascontiguousarray(ev.t, np.float64)
        a = np.ascontiguousarray(ev.arrivals, np.float64).reshape(len(ids), S)
        _check(self.L.seis_set_hypothesis(self.h, len(ids), _p(ids), _p(x), _p(t), _p(a)),
               self.L)

    @property
    def arrival_storage(self) -> str:
        """'rows' (philox stream spec v1: every version stores its S arrivals)
        or 'compact' (spec v2: births and their moves as generated versions)."""
        return "compact" if self.L.seis_get_arrival_storage(self.h) == 1 else "rows"

    @arrival_storage.setter
    def arrival_storage(self, mode: str):
        if mode not in ("rows", "compact"):
            raise ValueError("arrival storage must be 'rows' or 'compact'")
        _check(self.L.seis_set_arrival_storage(self.h, 1 if mode == "compact" else 0), self.L)

    def set_hypothesis_streamed(self, ids, x, t, rows, chunk: int = 1024):
        """Load a hypothesis whose arrivals come in pieces: rows(i0, n) returns
        the [n][S] arrival rows of input events i0 .. i0 + n - 1
        (seis_set_hypothesis_begin / _rows / _end)."""
        ids = np.ascontiguousarray(ids, np.uint64)
        x = np.ascontiguousarray(x, np.float64)
        t = np.ascontiguousarray(t, np.float64)
        N = len(ids)
        _check(self.L.seis_set_hypothesis_begin(self.h, N, _p(ids), _p(x), _p(t)), self.L)
        try:
            for i0 in range(0, N, chunk):
                n = min(chunk, N - i0)
                a = np.ascontiguousarray(rows(i0, n), np.float64)
                _check(self.L.seis_set_hypothesis_rows(self.h, i0, n, _p(a)), self.L)
        finally:
            _check(self.L.seis_set_hypothesis_end(self.h), self.L)

    def get_hypothesis(self, arrivals: bool = True, out: Events | None = None) -> Events:
        """The resident hypothesis (id order). `out`: caller-owned buffers (for
        example pinned host memory) with room for the events; the result views
        their first N rows."""
        n = i64(0)
        _check(self.L.seis_get_hypothesis(self.h, 0, C.byref(n), None, None, None, None), self.L)
        N = n.value
        S = self.config.n_stations()
        if out is not None:
            if len(out.ids) < N or (arrivals and out.arrivals.shape[0] < N):
                raise ValueError(f"get_hypothesis: out holds fewer than {N} events")
            ids, x, t = out.ids, out.x, out.t
            a = out.arrivals if arrivals else None
            for v in (ids, x, t) + ((a,) if arrivals else ()):
                if not v.flags.c_contiguous:
                    raise ValueError("get_hypothesis: out arrays must be C-contiguous")
        else:
            ids = np.zeros(max(N, 1), np.uint64)
            x = np.zeros(max(N, 1))
            t = np.zeros(max(N, 1))
            a = np.zeros((max(N, 1), S)) if arrivals else None
        _check(self.L.seis_get_hypothesis(self.h, N, C.byref(n), _p(ids), _p(x), _p(t),
                                          _p(a) if arrivals else None), self.L)
        return Events(ids[:N], x[:N], t[:N], a[:N] if arrivals else None)

    def set_snapshot_capacity(self, max_events: int, max_snapshots: int = 4096):
        """keep trace snapshots (reference Trace::snapshots) of the next runs."""
        _check(self.L.seis_set_snapshot_capacity(self.h, max_events, max_snapshots), self.L)
        self._snap_cap = (max_events, max_snapshots)

    def _get_snapshots(self) -> list:
        cap = getattr(self, "_snap_cap", (0, 0))
        if cap[0] == 0:
            return []
        ns = i64(0)
        steps = np.zeros(cap[1], np.int64)
        counts = np.zeros(cap[1], np.int64)
        ids = np.zeros(max(cap[0], 1), np.uint64)
        x = np.zeros(max(cap[0], 1))
        t = np.zeros(max(cap[0], 1))
        _check(self.L.seis_get_snapshots(self.h, cap[1], C.byref(ns), _p(steps), _p(counts),
                                         cap[0], _p(ids), _p(x), _p(t)), self.L)
        out, off = [], 0
        for i in range(min(ns.value, cap[1])):
            c = int(counts[i])
            out.append(Snapshot(i, int(steps[i]), ids[off:off + c].copy(), x[off:off + c].copy(),
                                t[off:off + c].copy()))
            off += c
        return out

    def log_joint(self) -> float:
        out = f64(0)
        _check(self.L.seis_log_joint(self.h, C.byref(out)), self.L)
        return out.value

    def delta_log_joint(self, changes: list, window=None, support=None) -> np.ndarray:
        """Batched delta_log_joint against the resident hypothesis.

        Each change is (removed_ids, added) with added a list of
        (x, t, arrivals[S]) tuples.
        """
        S = self.config.n_stations()
        n = self.config.n_samples()
        wlo, whi = window if window is not None else (0, n)
        slo, shi, sc = support if support is not None else (0.0, self.config.T, 1)
        arr_rows = []
        cs = (_ChangeC * max(len(changes), 1))()
        for i, (rem, add) in enumerate(changes):
            c = cs[i]
            c.n_removed = len(rem)
            c.n_added = len(add)
            for q, rid in enumerate(rem):
                c.removed_id[q] = int(rid)
            for q, (ax, at, aa) in enumerate(add):
                c.added_x[q] = ax
                c.added_t[q] = at
                c.added_row[q] = len(arr_rows)
                arr_rows.append(np.asarray(aa, np.float64).reshape(S))
            c.window_lo, c.window_hi = wlo, whi
            c.support_lo, c.support_hi, c.support_closed = slo, shi, sc
        rows = np.ascontiguousarray(np.stack(arr_rows) if arr_rows else np.zeros((0, S)))
        out = np.zeros(len(changes))
        _check(self.L.seis_score_batch(self.h, len(changes), C.cast(cs, P), _p(rows),
                                       len(arr_rows), _p(out)), self.L)
        return out

    def run_chromatic(self, sc: SamplerConfig, tape: np.ndarray | None = None,
                      tape_arrivals: np.ndarray | None = None, row_cap: int = 1 << 16,
                      final: bool = True, decisions: int = 0) -> Trace:
        """run_chromatic (samplers.hpp:401-498) from the resident hypothesis;
        run_serial (samplers.hpp:282-315) when sc.algorithm == "serial"; or
        run_naive_parallel (samplers.hpp:321-394) when sc.algorithm == "naive"
        (from the empty hypothesis).

        Without `tape`: production mode (philox stream spec v1). With `tape`
        (oracle TAPE_DTYPE records in driver order): replay mode, returning the
        engine's per-step delta / log_r / decision in Trace.step_out.
        `decisions` > 0 (production only): capacity for the run's own per-step
        decisions, returned in Trace.step_out (driver order).
        """
        s = sc._c()
        mode = 0
        n_tape = 0
        tarr = None
        out = None
        if tape is not None:
            mode = 1
            tape = np.ascontiguousarray(tape, TAPE_DTYPE)
            n_tape = len(tape)
            tarr = np.ascontiguousarray(tape_arrivals if tape_arrivals is not None
                                        else np.zeros(1), np.float64)
            out = np.zeros(n_tape, STEP_OUT_DTYPE)
        elif decisions > 0:
            n_tape = int(decisions)
            out = np.zeros(n_tape, STEP_OUT_DTYPE)
        rs = np.zeros(row_cap, np.int64)
        rl = np.zeros(row_cap)
        rc = np.zeros(row_cap, np.int64)
        st = _StatsC()
        fn = {"naive": self.L.seis_run_naive,
              "serial": self.L.seis_run_serial}.get(sc.algorithm, self.L.seis_run_chromatic)
        _check(fn(self.h, C.byref(s), mode, _p(tape), n_tape, _p(tarr),
                  0 if tarr is None else len(tarr), _p(out), row_cap, _p(rs), _p(rl), _p(rc),
                  C.byref(st)), self.L)
        nr = min(st.n_rows, row_cap)
        stats = {f: getattr(st, f) for f, _ in _StatsC._fields_}
        if out is not None and mode == 0:
            out = out[:st.total_steps]
        tr = Trace(rs[:nr], rl[:nr], rc[:nr], st.total_steps, st.total_accepted, stats,
                   step_out=out)
        if final:
            tr.final = self.get_hypothesis()
        tr.row_wall = self.row_wall()[:nr]
        tr.phases = self.phases()
        tr.snapshots = self._get_snapshots()
        wall_at = {int(s_): float(w_) for s_, w_ in zip(tr.row_step, tr.row_wall)}
        for sn in tr.snapshots:
            sn.wall_seconds = wall_at.get(sn.step, 0.0)
        return tr

    def phases(self) -> np.ndarray:
        """Trace::phases of the last run (seis_get_phases)."""
        n = i64(0)
        _check(self.L.seis_get_phases(self.h, 0, C.byref(n), None), self.L)
        out = np.zeros(n.value, PHASE_DTYPE)
        if n.value:
            _check(self.L.seis_get_phases(self.h, n.value, C.byref(n), _p(out)), self.L)
        return out

    def row_wall(self) -> np.ndarray:
        """TraceRow::wall_seconds of the last run (seis_get_row_wall)."""
        n = i64(0)
        _check(self.L.seis_get_row_wall(self.h, 0, C.byref(n), None), self.L)
        out = np.zeros(n.value)
        if n.value:
            _check(self.L.seis_get_row_wall(self.h, n.value, C.byref(n), _p(out)), self.L)
        return out


def run_sampler(config: ModelConfig, signals: np.ndarray, sc: SamplerConfig,
                event_capacity: int = 4096) -> Trace:
    """reference run_sampler (samplers.hpp:500-509) for every algorithm
    (serial, naive, chromatic static/dynamic): from the empty hypothesis,
    through the C-ABI with host buffers."""
    eng = Engine(config, signals, event_capacity)
    try:
        return eng.run_chromatic(sc)
    finally:
        eng.close()
