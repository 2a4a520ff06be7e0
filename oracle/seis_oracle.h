/*
 * seis_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's chromatic region-sweep path
 * (arXiv 1612.00595 reference, proj/include/seismic/ headers) used as the
 * parity checker for the B200 engine. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product path (paper_1612_00595_b200/) never links or calls it.
 *
 * Pinned against the reference itself: oracle/ref_shim.cpp compiles the
 * reference headers unchanged into oracle/_ref/libseisref.so exposing the
 * same flat API (prefix sr_), and tests/golden/ holds vectors generated from
 * it (tests/golden/make_golden.py).
 */
#ifndef SEIS_ORACLE_H
#define SEIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* reference ModelConfig (model.hpp:55-104) */
typedef struct {
  double lambda_rate, T, x_max, v, sigma_arrival, t_s, var_noise, var_event, sample_rate;
  int64_t n_stations;
  const double* stations;
} so_model;

/* reference SamplerConfig (samplers.hpp:47-71) + the RNG mode switch */
typedef struct {
  int64_t steps_per_epoch, epochs;
  int64_t n_regions;
  uint64_t seed;
  double burn_in_fraction;
  int64_t record_every;
  double weights[5]; /* birth, death, location, arrival, joint */
  double step_location_x, step_location_t, step_arrival, step_joint;
  int64_t rng_mode; /* 0: reference xoshiro streams, 1: philox stream spec v1 */
  int64_t dynamic;  /* 0: chromatic-static, 1: chromatic-dynamic */
  int64_t compact;  /* rng_mode 1: arrival storage spec v2 (generated versions) */
} so_sampler;

/* one MH step of a chain, as seen by the driver */
typedef struct {
  int64_t epoch, color, region, slot, step, type, is_null, n_removed, n_added, u_drawn, scored,
      accepted, constrained_out;
  uint64_t removed_id[2], added_id[2];
  double added_x[2], added_t[2];
  double logq_f, logq_r, u, delta, log_r;
  int64_t added_arr_off; /* offset (in doubles) of added[0] arrivals in the arrival pool */
} so_tape_rec;

enum { SO_OK = 0, SO_EINVAL = 2, SO_ERUNTIME = 3 };

/* ---- rng.hpp ---- */
uint64_t so_splitmix64(uint64_t* state);
typedef struct {
  uint64_t s[4];
} so_rng;
so_rng so_rng_from_key(uint64_t key);
so_rng so_derive_stream(uint64_t seed, uint64_t purpose, uint64_t i0, uint64_t i1, uint64_t i2);
uint64_t so_next_u64(so_rng* r);
double so_uniform(so_rng* r);
double so_uniform_range(so_rng* r, double lo, double hi);
uint64_t so_uniform_index(so_rng* r, uint64_t n);
double so_normal(so_rng* r, double mean, double stddev);
uint64_t so_poisson(so_rng* r, double mean);

/* ---- model/density ---- */
const char* so_last_error(void);
int so_validate_model(const so_model* m);
int64_t so_n_samples(const so_model* m);
void so_arrival_range(const so_model* m, double a, int64_t* lo, int64_t* hi);

/* World given as flat arrays: ids[N], x[N], t[N], arr[N*S] (event-major),
 * signals[S*n] (station-major, the reference's ObservedSignals layout). */
double so_log_joint(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                    const double* x, const double* t, const double* arr);

/* delta_log_joint (density.hpp:214-305). Removed events are given by index
 * into the world arrays; added events by value. window = [wlo, whi) samples,
 * prior support = [slo, shi) (closed at shi when sclosed). */
double so_delta(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                const double* x, const double* t, const double* arr, int64_t n_removed,
                const int64_t* removed_idx, int64_t n_added, const uint64_t* added_ids,
                const double* added_x, const double* added_t, const double* added_arr,
                int64_t wlo, int64_t whi, double slo, double shi, int64_t sclosed);

/* ---- worldgen.hpp ---- */
/* returns event count in *n_events (<= cap) and fills signals[S*n] */
int so_sample_world(const so_model* m, uint64_t seed, int64_t cap, int64_t* n_events,
                    uint64_t* ids, double* x, double* t, double* arr, double* signals);
int so_make_world_with_events(const so_model* m, int64_t n, const double* cx, const double* ct,
                              uint64_t seed, uint64_t* ids, double* x, double* t, double* arr,
                              double* signals);

/* ---- partition.hpp ---- */
int so_partition(double T, double l, double offset, double tau, int64_t cap, int64_t* n_regions,
                 double* boundaries, int32_t* colors, int32_t* n_colors);
int64_t so_region_of(const double* boundaries, int64_t n_regions, double t);
double so_partition_offset(uint64_t seed, int64_t epoch, double l);
void so_signal_window(double lo, double hi, double tau, double T, double rate, int64_t* wlo,
                      int64_t* whi);

/* ---- samplers.hpp: chromatic driver with tape ---- */
typedef struct so_run so_run;
so_run* so_run_chromatic(const so_model* m, const double* signals, const so_sampler* sc,
                         int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                         const double* arr, int64_t want_tape, int64_t want_rowlj);
so_run* so_run_serial(const so_model* m, const double* signals, const so_sampler* sc,
                      int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                      const double* arr, int64_t want_tape, int64_t want_rowlj);
so_run* so_run_naive(const so_model* m, const double* signals, const so_sampler* sc,
                     int64_t want_tape, int64_t want_rowlj);
int so_run_status(const so_run* r);
void so_run_counts(const so_run* r, int64_t* n_tape, int64_t* n_tape_arr, int64_t* n_rows,
                   int64_t* n_final, int64_t* total_steps, int64_t* total_accepted);
void so_run_tape(const so_run* r, so_tape_rec* recs, double* arr);
void so_run_rows(const so_run* r, int64_t* step, double* log_joint, int64_t* event_count);
void so_run_final(const so_run* r, uint64_t* ids, double* x, double* t, double* arr);
void so_run_free(so_run* r);

/* ---- evaluation.hpp: match_events; out = {precision, recall, location_error, n_matched} */
int so_match_events(int64_t nt, const uint64_t* tid, const double* tx, const double* tt,
                    int64_t ni, const uint64_t* iid, const double* ix, const double* it,
                    double threshold, double* out);

/* ---- philox stream spec v1 (include/seis_philox.h) probes ---- */
void so_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
               uint32_t* out);
float so_philox_normal(uint64_t seed, uint32_t sweep, uint32_t region, uint32_t step, uint32_t i);
float so_bm(uint32_t w0, uint32_t w1);

#ifdef __cplusplus
}
#endif
#endif
