"""B200-native engine for the chromatic region-sweep hot path of arXiv 1612.00595.

The product is the CUDA C-ABI library ``_lib/libseis_b200.so`` (built by
``paper_1612_00595_b200.build``); ``engine`` mirrors the reference's
sampler/model API over it. See DESIGN.md.
"""
from .engine import (  # noqa: F401
    F32, F64, BootstrapCI, Engine, Events, MatchReport, ModelConfig, Partition, SamplerConfig,
    Snapshot, Trace, assign_regions, bootstrap_ci, match_events, metric_trace,
    load_library, load_world, make_world_with_events, partition, partition_offset, run_sampler,
    sample_world, sample_world_events, make_world_with_events_signals, save_world,
    thomas_events, world_arrivals)
