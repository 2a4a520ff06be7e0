/*
 * seis_b200.h — C-ABI of the B200 chromatic region-sweep engine.
 *
 * The reference (arXiv 1612.00595, header-only C++, no FFI) exposes the hot
 * path as C++ templates over value types; see SURVEY.md §8(b). Each entry
 * point below replaces one reference seam (paths relative to
 * /root/reference/proj/include/seismic/):
 *
 *   seis_engine_create   World{config, {}, signals} + ModelConfig::validate
 *                        (model.hpp:55-121); uploads ObservedSignals once
 *   seis_set_hypothesis  the World::events a driver starts from (the
 *                        reference always starts empty, samplers.hpp:409;
 *                        this is the extension SURVEY §8(b) asks for)
 *   seis_get_hypothesis  Trace::snapshots[...].events (samplers.hpp:80-85)
 *   seis_partition       build_partition + color_partition
 *                        (partition.hpp:40-90), bit-exact, on device
 *   seis_assign_regions  Partition::region_of (partition.hpp:33-37), on device
 *   seis_partition_offset derive_stream(seed, kPartitionOffset, epoch)
 *                        .uniform(0, l) (samplers.hpp:488-491), on device
 *   seis_score_batch     delta_log_joint(world, change, opts)
 *                        (density.hpp:214-305), batched
 *   seis_log_joint       log_joint(world) (density.hpp:146-154)
 *   seis_run_chromatic   run_sampler / run_chromatic (samplers.hpp:401-509):
 *                        production mode (philox stream spec v1,
 *                        include/seis_philox.h) or replay mode (host tape of
 *                        proposals + uniforms, run_region_steps/mh_step
 *                        semantics, samplers.hpp:115-138,
 *                        proposals.hpp:265-293)
 *
 * Conventions: inputs are caller-owned host buffers; no C++
 * exceptions cross the ABI; every call returns 0 on success, 2 for a
 * validation error (the reference's std::invalid_argument, CLI exit 2) and 3
 * for a runtime error (std::runtime_error / logic_error, CLI exit 3), with the
 * message in seis_last_error() (thread-local). One CUDA stream per engine;
 * calls on one handle must be serialised by the caller. There is no CPU
 * fallback: without a usable sm_100 device seis_engine_create returns 3.
 */
#ifndef SEIS_B200_H
#define SEIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEIS_OK 0
#define SEIS_EINVAL 2
#define SEIS_ERUNTIME 3

#define SEIS_F32 0
#define SEIS_F64 1

typedef struct seis_engine seis_engine;

/* reference ModelConfig (model.hpp:55-65), stations passed separately */
typedef struct {
  double lambda_rate, T, x_max, v, sigma_arrival, t_s, var_noise, var_event, sample_rate;
} seis_model_cfg;

/* reference SamplerConfig (samplers.hpp:47-58); the algorithm is the entry point called */
typedef struct {
  int64_t steps_per_epoch; /* k steps per region between barriers */
  int64_t epochs;          /* sweeps */
  int64_t n_regions;
  uint64_t seed;
  double burn_in_fraction;
  int64_t record_every;    /* trace row cadence in executed steps */
  double weights[5];       /* birth, death, location, arrival, joint */
  double step_location_x, step_location_t, step_arrival, step_joint;
  int32_t dynamic;         /* 0 chromatic-static, 1 chromatic-dynamic */
  int32_t record_log_joint;/* evaluate log_joint on device at trace rows */
} seis_sampler_cfg;

/* One MH step of a reference chain (the replay tape); layout
 * identical to the oracle's so_tape_rec. Only the proposal fields are read:
 * type, is_null, n_removed/removed_id, n_added/added_*, logq_f, logq_r,
 * u_drawn, u. */
typedef struct {
  int64_t epoch, color, region, slot, step, type, is_null, n_removed, n_added, u_drawn, scored,
      accepted, constrained_out;
  uint64_t removed_id[2], added_id[2];
  double added_x[2], added_t[2];
  double logq_f, logq_r, u, delta, log_r;
  int64_t added_arr_off;
} seis_tape_step;

/* per-step result of replay mode */
typedef struct {
  double delta;  /* likelihood delta (-inf when out of support) */
  double log_r;  /* log acceptance ratio */
  int32_t scored, accepted;
} seis_step_out;

/* One proposed edit for seis_score_batch (reference Change + ScoreOptions,
 * density.hpp:160-189). Removed events are named by id and must be in the
 * engine's hypothesis; added arrivals are rows of `added_arrivals`. */
typedef struct {
  int32_t n_removed, n_added;
  uint64_t removed_id[2];
  double added_x[2], added_t[2];
  int64_t added_row[2];   /* row index into added_arrivals [rows][S] */
  int64_t window_lo, window_hi;   /* samples [lo, hi) */
  double support_lo, support_hi;  /* prior support on the time axis */
  int32_t support_closed;
  int32_t pad_;
} seis_change;

/* run summary + measurement counters */
typedef struct {
  int64_t total_steps, total_accepted;  /* reference Trace fields (samplers.hpp:97-103) */
  int64_t scored_proposals;             /* non-null, not constrained out */
  int64_t changed_samples;              /* sum of n_j(p) over scored proposals */
  int64_t arrival_values;               /* sum of A(p) over scored proposals */
  double algorithmic_bytes;             /* SURVEY §8(d) B(p) summed */
  double sweep_kernel_ms;               /* CUDA-event time of the region-sweep kernels */
  double total_ms;                      /* CUDA-event time of the whole run */
  int64_t kernel_launches;              /* kernels launched by the run */
  int64_t n_rows;                       /* trace rows produced */
  int64_t final_events;
  int64_t speculative_discarded;        /* proposals evaluated ahead of an accept, then dropped */
  int64_t phases;                       /* region-sweep kernel launches (color phases) */
  int64_t generated_versions;           /* live generated versions after the run (spec v2) */
} seis_run_stats;

/* reference PhaseRecord (samplers.hpp:87-95): one per committed region
 * segment, in commit order (run_chromatic samplers.hpp:479; run_naive_parallel
 * samplers.hpp:370; run_serial records none) */
typedef struct {
  int64_t epoch;
  int32_t color, pad_;
  int64_t region;
  int64_t steps;
} seis_phase_record;

const char* seis_last_error(void);

/* event_capacity (1 .. 2^22): live events the hypothesis may hold. Coverage
 * counts stay uint16: a run that puts more than 65535 events over one
 * (sample, station) fails with status 3 instead of wrapping. */
int seis_engine_create(const seis_model_cfg* cfg, const double* stations, int64_t n_stations,
                       const void* signals /* [S][n] station-major, dtype */, int32_t dtype,
                       int64_t event_capacity, seis_engine** out);
void seis_engine_destroy(seis_engine* eng);

/* Stored arrival rows the engine allocated: min(2 * event_capacity + 2048,
 * what fits in free HBM less a reserve). Rows-mode runs need the live events
 * plus the phase-start versions they replaced; fewer rows than events of
 * capacity select the compact storage by default (generated versions need no
 * row). A loaded hypothesis is stored rows: at most this many events. */
int64_t seis_engine_pool_slots(const seis_engine* eng);

/* Arrival storage of the versions production runs create. SEIS_ARR_ROWS
 * (philox stream spec v1): every version stores its S fp64 arrivals, exactly
 * the reference's arithmetic. SEIS_ARR_COMPACT (spec v2, include/seis_philox.h):
 * a birth's version is its location plus its philox key, arrivals computed as
 * mean + sigma z; location and joint moves of such a version keep the
 * residual z exactly, a first arrival move is one per-station override, a
 * second one stores the row. Memory per version O(1) instead of 8 S bytes
 * (configs 3 and 4 at their stated k). The default is COMPACT when the
 * arrival pool cannot hold two stored rows per event of capacity, else ROWS.
 * Replay mode always stores rows. */
#define SEIS_ARR_ROWS 0
#define SEIS_ARR_COMPACT 1
int seis_set_arrival_storage(seis_engine* eng, int32_t mode);
int32_t seis_get_arrival_storage(const seis_engine* eng);

/* Replace the signals (same shape/dtype) — one host->device copy. */
int seis_upload_signals(seis_engine* eng, const void* signals);

int seis_set_hypothesis(seis_engine* eng, int64_t n, const uint64_t* ids, const double* x,
                        const double* t, const double* arrivals /* [n][S] */);
/* The same in pieces, for hypotheses whose arrivals do not fit in host memory
 * at once: _begin takes the events, _rows uploads the arrival rows of input
 * events i0 .. i0 + n - 1 (any order, every row exactly once), _end builds the
 * coverage counts. Other calls on the engine between _begin and _end are an
 * error (status 2). */
int seis_set_hypothesis_begin(seis_engine* eng, int64_t n, const uint64_t* ids, const double* x,
                              const double* t);
int seis_set_hypothesis_rows(seis_engine* eng, int64_t i0, int64_t n,
                             const double* arrivals /* [n][S] */);
int seis_set_hypothesis_end(seis_engine* eng);
/* arrivals may be NULL; *n receives the event count, at most cap are written */
int seis_get_hypothesis(seis_engine* eng, int64_t cap, int64_t* n, uint64_t* ids, double* x,
                        double* t, double* arrivals);

/* Trace snapshots (reference Trace::snapshots, samplers.hpp:80-85,430-433):
 * with a capacity set, seis_run_chromatic stores the event table (id, x, t)
 * at every trace row once executed >= burn_in_fraction * planned steps.
 * Snapshots are packed back to back: snapshot i holds snap_count[i] events. */
int seis_set_snapshot_capacity(seis_engine* eng, int64_t max_events, int64_t max_snapshots);
/* ids == NULL: only snap_step / snap_count are written (sizes the event buffers) */
int seis_get_snapshots(seis_engine* eng, int64_t cap_snap, int64_t* n_snap, int64_t* snap_step,
                       int64_t* snap_count, int64_t cap_ev, uint64_t* ids, double* x, double* t);

/* Trace::phases of the engine's last run (*n = count, at most cap written). */
int seis_get_phases(seis_engine* eng, int64_t cap, int64_t* n, seis_phase_record* out);
/* TraceRow::wall_seconds (= Snapshot::wall_seconds at the same step,
 * samplers.hpp:73-85) of the last run's trace rows: device time from the
 * start of the run to the row, from CUDA events on the engine's stream. */
int seis_get_row_wall(seis_engine* eng, int64_t cap, int64_t* n, double* wall_seconds);

int seis_partition(double T, double l, double offset, double tau, int64_t cap,
                   int64_t* n_regions, double* boundaries /* cap */, int32_t* colors /* cap */,
                   int32_t* n_colors);
int seis_assign_regions(const double* boundaries, int64_t n_regions, int64_t n, const double* t,
                        int64_t* region_out);
int seis_partition_offset(uint64_t seed, int64_t epoch, double l, double* u_out);

int seis_score_batch(seis_engine* eng, int64_t n_changes, const seis_change* changes,
                     const double* added_arrivals, int64_t n_rows, double* delta_out);

int seis_log_joint(seis_engine* eng, double* out);

/* mode 0: production (philox stream spec v1); mode 1: replay `tape` (n_tape
 * steps in driver order, arrivals in tape_arr) writing step_out[n_tape].
 * In mode 0 a non-NULL step_out (capacity n_tape >= the run's steps, tape
 * NULL) receives the production run's own per-step decisions, driver order.
 * Trace rows go to row_step/row_log_joint/row_count (capacity row_cap, may be
 * NULL). The final hypothesis stays on the engine (seis_get_hypothesis). */
int seis_run_chromatic(seis_engine* eng, const seis_sampler_cfg* sc, int32_t mode,
                       const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                       int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                       int64_t* row_step, double* row_log_joint, int64_t* row_count,
                       seis_run_stats* stats);

/* run_serial (samplers.hpp:282-315): plain MH over [0, T] (no region
 * constraint, full window, area T), epochs x steps_per_epoch steps from the
 * resident hypothesis (the reference starts empty), a trace row + snapshot
 * after every record_every steps. Same arguments as seis_run_chromatic
 * (n_regions, dynamic ignored); production draws follow the philox spec with
 * sweep = region = 0 and the chain step as the step counter. */
int seis_run_serial(seis_engine* eng, const seis_sampler_cfg* sc, int32_t mode,
                    const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                    int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                    int64_t* row_step, double* row_log_joint, int64_t* row_count,
                    seis_run_stats* stats);

/* run_naive_parallel (samplers.hpp:321-394), the uncolored comparison
 * sampler: every region runs epochs x steps_per_epoch steps from the empty
 * hypothesis (the engine's must be empty) against its own events only, prior
 * support = the region, likelihood window = signal_window (partition.hpp:94-102).
 * Same arguments as seis_run_chromatic (sc->dynamic ignored); the union of the
 * regions' final events becomes the engine's hypothesis. Trace rows: union
 * event counts at every checkpoint, log_joint at the last row only. */
int seis_run_naive(seis_engine* eng, const seis_sampler_cfg* sc, int32_t mode,
                   const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                   int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                   int64_t* row_step, double* row_log_joint, int64_t* row_count,
                   seis_run_stats* stats);

/* ---- synthetic inputs (worldgen.hpp:20-86, bit-exact with the reference
 * generator; host C++ so the fp64 libm draws match). Not on the hot path. */
const char* seis_world_last_error(void);
int seis_world_generate(const seis_model_cfg* cfg, const double* stations, int64_t S,
                        uint64_t seed, int64_t cap, int64_t* n_events, uint64_t* ids, double* x,
                        double* t, double* arrivals /* [cap][S] */,
                        void* signals /* [S][n] */, int32_t dtype, int32_t threads);
int seis_world_with_events(const seis_model_cfg* cfg, const double* stations, int64_t S,
                           int64_t n, const double* cx, const double* ct, uint64_t seed,
                           double* arrivals /* [n][S] */, void* signals /* [S][n] */,
                           int32_t dtype, int32_t threads);
/* Streaming generation (no N x S arrival matrix in host memory): the same
 * events and signals as seis_world_generate / seis_world_with_events, the
 * coverage counts accumulated per station from chunks of events; arrivals of
 * any event range regenerated with seis_world_arrivals (for
 * seis_set_hypothesis_begin/_rows/_end). */
int seis_world_generate_events(const seis_model_cfg* cfg, const double* stations, int64_t S,
                               uint64_t seed, int64_t cap, int64_t* n_events, uint64_t* ids,
                               double* x, double* t, void* signals /* [S][n] */, int32_t dtype,
                               int32_t threads);
int seis_world_with_events_signals(const seis_model_cfg* cfg, const double* stations, int64_t S,
                                   int64_t n, const double* cx, const double* ct, uint64_t seed,
                                   void* signals /* [S][n] */, int32_t dtype, int32_t threads);
int seis_world_arrivals(const seis_model_cfg* cfg, const double* stations, int64_t S,
                        uint64_t seed, int64_t i0, int64_t n, const double* x, const double* t,
                        double* arrivals /* [n][S] */, int32_t threads);
int seis_thomas_events(uint64_t seed, double x_max, double T, double parent_mean,
                       double child_mean, double sx, double st, int64_t cap, int64_t* n,
                       double* cx, double* ct);

/* ---- evaluation bridge (evaluation.hpp:51-171): greedy event matching and
 * the percentile bootstrap, host C++, bit-exact with the reference. Feeds on
 * seis_get_hypothesis / seis_get_snapshots output. Errors: status 2 with the
 * message in seis_eval_last_error(). Not on the hot path. */
typedef struct {
  double precision, recall, location_error;
  int64_t n_true, n_inferred, n_matched;
} seis_match_report;

typedef struct {
  double mean, lo, hi, level;
  int32_t resamples;
} seis_ci;

const char* seis_eval_last_error(void);
/* pair_* (capacity min(n_true, n_inf), may be NULL): matched pairs in truth
 * (t, x) order. */
int seis_match_events(int64_t n_true, const uint64_t* true_id, const double* true_x,
                      const double* true_t, int64_t n_inf, const uint64_t* inf_id,
                      const double* inf_x, const double* inf_t, double threshold,
                      seis_match_report* report, uint64_t* pair_true_id,
                      uint64_t* pair_inf_id, double* pair_dist);
int seis_bootstrap_ci(const double* values, int64_t n, double level, int32_t resamples,
                      uint64_t seed, seis_ci* out);

#ifdef __cplusplus
}
#endif
#endif
