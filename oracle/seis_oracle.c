/*
 * seis_oracle.c — TEST INFRASTRUCTURE ONLY (see seis_oracle.h).
 *
 * Plain-C restatement of the reference's chromatic region-sweep path. Every
 * function cites the reference lines it follows; paths are relative to
 * /root/reference/proj/include/seismic/. Build with -ffp-contract=off (the
 * reference's integer outputs come from fp64 expressions).
 */
#include "seis_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/seis_philox.h"

static const double kLog2Pi = 1.8378770664093454835606594728112;
static char g_err[512];

const char* so_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ rng.hpp */

/* rng.hpp:21-26 */
uint64_t so_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:30-34 */
so_rng so_rng_from_key(uint64_t key) {
  so_rng r;
  for (int i = 0; i < 4; ++i) r.s[i] = so_splitmix64(&key);
  if ((r.s[0] | r.s[1] | r.s[2] | r.s[3]) == 0) r.s[0] = 1;
  return r;
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:36-46 (xoshiro256++) */
uint64_t so_next_u64(so_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

/* rng.hpp:49-51 */
double so_uniform(so_rng* r) { return (double)(so_next_u64(r) >> 11) * 0x1.0p-53; }
double so_uniform_range(so_rng* r, double lo, double hi) { return lo + (hi - lo) * so_uniform(r); }

/* rng.hpp:54-57 */
uint64_t so_uniform_index(so_rng* r, uint64_t n) {
  return (uint64_t)(((unsigned __int128)so_next_u64(r) * n) >> 64);
}

/* rng.hpp:60-65 */
double so_normal(so_rng* r, double mean, double stddev) {
  const double u1 = 1.0 - so_uniform(r);
  const double u2 = so_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  return mean + stddev * rr * cos(6.283185307179586476925286766559 * u2);
}

/* rng.hpp:82-89 */
static uint64_t poisson_small(so_rng* r, double mean) {
  const double limit = exp(-mean);
  uint64_t k = 0;
  double p = 1.0;
  do {
    ++k;
    p *= so_uniform(r);
  } while (p > limit);
  return k - 1;
}

/* rng.hpp:69-80 */
uint64_t so_poisson(so_rng* r, double mean) {
  uint64_t total = 0;
  while (mean > 60.0) {
    total += poisson_small(r, 60.0);
    mean -= 60.0;
  }
  return total + poisson_small(r, mean);
}

/* rng.hpp:110-121 */
so_rng so_derive_stream(uint64_t seed, uint64_t purpose, uint64_t i0, uint64_t i1, uint64_t i2) {
  uint64_t key = seed;
  uint64_t k = so_splitmix64(&key);
  const uint64_t words[4] = {purpose, i0, i1, i2};
  for (int i = 0; i < 4; ++i) {
    uint64_t w = words[i];
    k ^= so_splitmix64(&w);
    k = so_splitmix64(&k);
  }
  return so_rng_from_key(k);
}

/* ---------------------------------------------------------------- model.hpp */

/* model.hpp:79-103 */
int so_validate_model(const so_model* m) {
  if (!(m->lambda_rate > 0)) return fail(SO_EINVAL, "ModelConfig: lambda_rate must be > 0");
  if (!(m->T > 0)) return fail(SO_EINVAL, "ModelConfig: T must be > 0");
  if (!(m->x_max > 0)) return fail(SO_EINVAL, "ModelConfig: x_max must be > 0");
  if (!(m->v > 0)) return fail(SO_EINVAL, "ModelConfig: v must be > 0");
  if (!(m->sigma_arrival > 0)) return fail(SO_EINVAL, "ModelConfig: sigma_arrival must be > 0");
  if (!(m->t_s > 0)) return fail(SO_EINVAL, "ModelConfig: t_s must be > 0");
  if (!(m->var_noise > 0)) return fail(SO_EINVAL, "ModelConfig: var_noise must be > 0");
  if (!(m->var_event > m->var_noise))
    return fail(SO_EINVAL, "ModelConfig: var_event must exceed var_noise");
  if (!(m->sample_rate > 0)) return fail(SO_EINVAL, "ModelConfig: sample_rate must be > 0");
  const double n = m->sample_rate * m->T;
  if (fabs(n - (double)llround(n)) > 1e-9)
    return fail(SO_EINVAL, "ModelConfig: sample_rate * T must be an integer sample count");
  if (m->n_stations < 2) return fail(SO_EINVAL, "ModelConfig: need at least 2 stations");
  for (int64_t j = 0; j < m->n_stations; ++j) {
    if (m->stations[j] < 0 || m->stations[j] > m->x_max)
      return fail(SO_EINVAL, "ModelConfig: station outside [0, x_max]");
    if (j > 0 && !(m->stations[j - 1] < m->stations[j]))
      return fail(SO_EINVAL, "ModelConfig: stations must be sorted strictly ascending");
  }
  return SO_OK;
}

/* model.hpp:67-69 */
int64_t so_n_samples(const so_model* m) { return (int64_t)llround(m->sample_rate * m->T); }

/* model.hpp:73-75 */
static double arrival_mean(const so_model* m, double x, double t, int64_t j) {
  return t + fabs(x - m->stations[j]) / m->v;
}

/* -------------------------------------------------------------- density.hpp */

/* density.hpp:15-18 */
static double log_gaussian(double x, double mean, double var) {
  const double d = x - mean;
  return -0.5 * (kLog2Pi + log(var)) - d * d / (2.0 * var);
}

/* density.hpp:21-25 */
static double log_factorial(int64_t n) {
  double acc = 0.0;
  for (int64_t i = 2; i <= n; ++i) acc += log((double)i);
  return acc;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* density.hpp:29-36 */
void so_arrival_range(const so_model* m, double a, int64_t* lo, int64_t* hi) {
  const double n = (double)so_n_samples(m);
  double l = ceil(a * m->sample_rate);
  double h = ceil((a + m->t_s) * m->sample_rate);
  l = clampd(l, 0.0, n);
  h = clampd(h, 0.0, n);
  *lo = (int64_t)l;
  *hi = (int64_t)h;
}

/* model.hpp:27-32 */
static int region_contains(double lo, double hi, int closed, double t) {
  return t >= lo && (t < hi || (closed && t == hi));
}

/* density.hpp:45-61 */
static double log_event_prior(const so_model* m, int64_t N, const double* x, const double* t,
                              double slo, double shi, int sclosed) {
  const double area_t = shi - slo;
  const double lambda_area = m->lambda_rate * area_t;
  for (int64_t i = 0; i < N; ++i)
    if (x[i] < 0.0 || x[i] > m->x_max || !region_contains(slo, shi, sclosed, t[i]))
      return -INFINITY;
  return -lambda_area + (double)N * log(lambda_area) - log_factorial(N) +
         (double)N * (-log(m->x_max) - log(area_t));
}

/* density.hpp:63-75 */
static double log_arrival_densities(const so_model* m, double x, double t, const double* a) {
  double acc = 0.0;
  const double s = m->sigma_arrival;
  for (int64_t j = 0; j < m->n_stations; ++j)
    acc += log_gaussian(a[j], arrival_mean(m, x, t, j), s * s);
  return acc;
}

/* density.hpp:79-84 */
static void add_coverage(int32_t* counts, int64_t wb, int64_t we, int64_t sb, int64_t se,
                         int32_t delta) {
  const int64_t lo = wb > sb ? wb : sb;
  const int64_t hi = we < se ? we : se;
  for (int64_t s = lo; s < hi; ++s) counts[s - wb] += delta;
}

/* density.hpp:89-108 */
static double station_loglik(const so_model* m, const double* samples, int64_t wb, int64_t we,
                             const int32_t* counts) {
  double acc = 0.0;
  int32_t last = -1;
  double log_term = 0.0, inv_2var = 0.0;
  for (int64_t s = wb; s < we; ++s) {
    const int32_t c = counts[s - wb];
    if (c != last) {
      const double var = m->var_noise + c * m->var_event;
      log_term = -0.5 * (kLog2Pi + log(var));
      inv_2var = 0.5 / var;
      last = c;
    }
    const double y = samples[s];
    acc += log_term - y * y * inv_2var;
  }
  return acc;
}

/* density.hpp:131-144 */
static double log_signal_likelihood(const so_model* m, const double* signals, int64_t N,
                                    const double* arr, int64_t wb, int64_t we) {
  const int64_t S = m->n_stations, n = so_n_samples(m);
  double acc = 0.0;
  int32_t* counts = (int32_t*)calloc((size_t)(we > wb ? we - wb : 0) + 1, sizeof(int32_t));
  for (int64_t j = 0; j < S; ++j) {
    memset(counts, 0, sizeof(int32_t) * (size_t)(we - wb));
    for (int64_t e = 0; e < N; ++e) {
      int64_t lo, hi;
      so_arrival_range(m, arr[e * S + j], &lo, &hi);
      add_coverage(counts, wb, we, lo, hi, 1);
    }
    acc += station_loglik(m, signals + j * n, wb, we, counts);
  }
  free(counts);
  return acc;
}

/* density.hpp:146-154 */
double so_log_joint(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                    const double* x, const double* t, const double* arr) {
  (void)ids;
  const double prior = log_event_prior(m, N, x, t, 0.0, m->T, 1);
  if (prior == -INFINITY) return -INFINITY;
  double arrivals = 0.0;
  for (int64_t e = 0; e < N; ++e)
    arrivals += log_arrival_densities(m, x[e], t[e], arr + e * m->n_stations);
  return prior + arrivals + log_signal_likelihood(m, signals, N, arr, 0, so_n_samples(m));
}

typedef struct {
  int64_t b, e;
} range_t;

/* density.hpp:193-206 */
static int64_t merge_ranges(range_t* r, int64_t k) {
  for (int64_t i = 1; i < k; ++i) /* insertion sort by begin (k <= 4) */
    for (int64_t j = i; j > 0 && r[j].b < r[j - 1].b; --j) {
      range_t tmp = r[j];
      r[j] = r[j - 1];
      r[j - 1] = tmp;
    }
  int64_t out = 0;
  for (int64_t i = 0; i < k; ++i) {
    if (r[i].e <= r[i].b) continue;
    if (out > 0 && r[i].b <= r[out - 1].e) {
      if (r[i].e > r[out - 1].e) r[out - 1].e = r[i].e;
    } else {
      r[out++] = r[i];
    }
  }
  return out;
}

/* delta_log_joint, density.hpp:214-305, restated over flat arrays. */
double so_delta(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                const double* x, const double* t, const double* arr, int64_t n_removed,
                const int64_t* removed_idx, int64_t n_added, const uint64_t* added_ids,
                const double* added_x, const double* added_t, const double* added_arr,
                int64_t wlo, int64_t whi, double slo, double shi, int64_t sclosed) {
  (void)added_ids;
  const int64_t S = m->n_stations, n = so_n_samples(m);
  /* 218-221: support */
  for (int64_t a = 0; a < n_added; ++a)
    if (added_x[a] < 0.0 || added_x[a] > m->x_max ||
        !region_contains(slo, shi, (int)sclosed, added_t[a]))
      return -INFINITY;
  /* 223-237: prior */
  const int64_t n0 = N;
  const int64_t n1 = n0 - n_removed + n_added;
  const double area_t = shi - slo;
  const double log_lambda_area = log(m->lambda_rate * area_t);
  double delta = 0.0;
  if (n1 > n0) {
    for (int64_t i = n0 + 1; i <= n1; ++i) delta += log_lambda_area - log((double)i);
  } else if (n1 < n0) {
    for (int64_t i = n1 + 1; i <= n0; ++i) delta -= log_lambda_area - log((double)i);
  }
  delta += (double)(n1 - n0) * (-log(m->x_max) - log(area_t));
  /* 239-240: arrival densities */
  for (int64_t a = 0; a < n_added; ++a)
    delta += log_arrival_densities(m, added_x[a], added_t[a], added_arr + a * S);
  for (int64_t r = 0; r < n_removed; ++r) {
    const int64_t e = removed_idx[r];
    delta -= log_arrival_densities(m, x[e], t[e], arr + e * S);
  }
  /* 244-301: likelihood over merged affected ranges per station */
  int32_t* oc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* nc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < S; ++j) {
    range_t rg[8];
    int64_t k = 0;
    for (int64_t r = 0; r < n_removed; ++r) {
      int64_t lo, hi;
      so_arrival_range(m, arr[removed_idx[r] * S + j], &lo, &hi);
      if (lo < wlo) lo = wlo;
      if (hi > whi) hi = whi;
      if (hi > lo) rg[k++] = (range_t){lo, hi};
    }
    for (int64_t a = 0; a < n_added; ++a) {
      int64_t lo, hi;
      so_arrival_range(m, added_arr[a * S + j], &lo, &hi);
      if (lo < wlo) lo = wlo;
      if (hi > whi) hi = whi;
      if (hi > lo) rg[k++] = (range_t){lo, hi};
    }
    k = merge_ranges(rg, k);
    for (int64_t q = 0; q < k; ++q) {
      const int64_t rb = rg[q].b, re = rg[q].e;
      memset(oc, 0, sizeof(int32_t) * (size_t)(re - rb));
      for (int64_t e = 0; e < N; ++e) {
        int removed = 0;
        for (int64_t r = 0; r < n_removed; ++r)
          if (ids[removed_idx[r]] == ids[e]) {
            removed = 1;
            break;
          }
        if (!removed) {
          int64_t lo, hi;
          so_arrival_range(m, arr[e * S + j], &lo, &hi);
          add_coverage(oc, rb, re, lo, hi, 1);
        }
      }
      memcpy(nc, oc, sizeof(int32_t) * (size_t)(re - rb));
      for (int64_t r = 0; r < n_removed; ++r) {
        int64_t lo, hi;
        so_arrival_range(m, arr[removed_idx[r] * S + j], &lo, &hi);
        add_coverage(oc, rb, re, lo, hi, 1);
      }
      for (int64_t a = 0; a < n_added; ++a) {
        int64_t lo, hi;
        so_arrival_range(m, added_arr[a * S + j], &lo, &hi);
        add_coverage(nc, rb, re, lo, hi, 1);
      }
      const double* samples = signals + j * n;
      int32_t last_old = -1, last_new = -1;
      double old_log = 0, old_inv = 0, new_log = 0, new_inv = 0;
      for (int64_t s = rb; s < re; ++s) {
        const int32_t co = oc[s - rb], cn = nc[s - rb];
        if (co == cn) continue;
        if (co != last_old) {
          const double var = m->var_noise + co * m->var_event;
          old_log = -0.5 * (kLog2Pi + log(var));
          old_inv = 0.5 / var;
          last_old = co;
        }
        if (cn != last_new) {
          const double var = m->var_noise + cn * m->var_event;
          new_log = -0.5 * (kLog2Pi + log(var));
          new_inv = 0.5 / var;
          last_new = cn;
        }
        const double y2 = samples[s] * samples[s];
        delta += (new_log - y2 * new_inv) - (old_log - y2 * old_inv);
      }
    }
  }
  free(oc);
  free(nc);
  return delta;
}

/* ------------------------------------------------------------- worldgen.hpp */

static void gen_signals(const so_model* m, uint64_t seed, int64_t N, const double* arr,
                        double* signals) {
  const int64_t S = m->n_stations, n = so_n_samples(m);
  int32_t* counts = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t j = 0; j < S; ++j) {
    /* worldgen.hpp:42-43 variance_profile (density.hpp:112-129) */
    memset(counts, 0, sizeof(int32_t) * (size_t)n);
    for (int64_t e = 0; e < N; ++e) {
      int64_t lo, hi;
      so_arrival_range(m, arr[e * S + j], &lo, &hi);
      add_coverage(counts, 0, n, lo, hi, 1);
    }
    /* worldgen.hpp:44-51 */
    so_rng noise = so_derive_stream(seed, 4, (uint64_t)j, 0, 0);
    for (int64_t s = 0; s < n; ++s) {
      const double var = m->var_noise + counts[s] * m->var_event;
      signals[j * n + s] = so_normal(&noise, 0.0, sqrt(var));
    }
  }
  free(counts);
}

static void gen_arrivals(const so_model* m, uint64_t seed, uint64_t i, double x, double t,
                         double* a) {
  so_rng r = so_derive_stream(seed, 3, i, 0, 0); /* worldgen.hpp:34-38 */
  for (int64_t j = 0; j < m->n_stations; ++j)
    a[j] = so_normal(&r, arrival_mean(m, x, t, j), m->sigma_arrival);
}

/* worldgen.hpp:20-53 */
int so_sample_world(const so_model* m, uint64_t seed, int64_t cap, int64_t* n_events,
                    uint64_t* ids, double* x, double* t, double* arr, double* signals) {
  int rc = so_validate_model(m);
  if (rc) return rc;
  so_rng count_rng = so_derive_stream(seed, 1, 0, 0, 0);
  const uint64_t N = so_poisson(&count_rng, m->lambda_rate * m->T);
  *n_events = (int64_t)N;
  if ((int64_t)N > cap) return fail(SO_ERUNTIME, "so_sample_world: event capacity too small");
  for (uint64_t i = 0; i < N; ++i) {
    so_rng c = so_derive_stream(seed, 2, i, 0, 0);
    ids[i] = i;
    x[i] = so_uniform_range(&c, 0.0, m->x_max);
    t[i] = so_uniform_range(&c, 0.0, m->T);
    gen_arrivals(m, seed, i, x[i], t[i], arr + i * m->n_stations);
  }
  gen_signals(m, seed, (int64_t)N, arr, signals);
  return SO_OK;
}

/* worldgen.hpp:57-86 */
int so_make_world_with_events(const so_model* m, int64_t n, const double* cx, const double* ct,
                              uint64_t seed, uint64_t* ids, double* x, double* t, double* arr,
                              double* signals) {
  int rc = so_validate_model(m);
  if (rc) return rc;
  for (int64_t i = 0; i < n; ++i) {
    ids[i] = (uint64_t)i;
    x[i] = cx[i];
    t[i] = ct[i];
    gen_arrivals(m, seed, (uint64_t)i, x[i], t[i], arr + i * m->n_stations);
  }
  gen_signals(m, seed, n, arr, signals);
  return SO_OK;
}

/* ------------------------------------------------------------ partition.hpp */

/* partition.hpp:40-61 + 66-90 */
int so_partition(double T, double l, double offset, double tau, int64_t cap, int64_t* n_regions,
                 double* boundaries, int32_t* colors, int32_t* n_colors) {
  if (!(T > 0)) return fail(SO_EINVAL, "build_partition: T must be > 0");
  if (!(l > 0) || l > T) return fail(SO_EINVAL, "build_partition: need 0 < l <= T");
  if (offset < 0 || offset >= l) return fail(SO_EINVAL, "build_partition: need 0 <= offset < l");
  int64_t nb = 0;
  if (nb >= cap) return fail(SO_ERUNTIME, "partition capacity");
  boundaries[nb++] = 0.0;
  double b = offset > 0 ? offset : l;
  while (b < T - 1e-9) {
    if (nb >= cap) return fail(SO_ERUNTIME, "partition capacity");
    boundaries[nb++] = b;
    b += l;
  }
  if (nb >= cap) return fail(SO_ERUNTIME, "partition capacity");
  boundaries[nb++] = T;
  const int64_t n = nb - 1;
  *n_regions = n;
  if (!(tau >= 0)) return fail(SO_EINVAL, "color_partition: tau_max must be >= 0");
  int k;
  if (l >= tau)
    k = 2;
  else if (l >= tau / 2)
    k = 3;
  else
    return fail(SO_EINVAL, "color_partition: region length is below tau_max/2");
  *n_colors = k;
  for (int64_t i = 0; i < n; ++i) colors[i] = (int32_t)(i % k);
  /* separation invariant, partition.hpp:84-88 (O(n^2) as the reference) */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (colors[i] == colors[j] && boundaries[j] - boundaries[i + 1] < tau - 1e-9)
        return fail(SO_ERUNTIME, "color_partition: separation invariant violated");
  return SO_OK;
}

/* partition.hpp:33-37 */
int64_t so_region_of(const double* boundaries, int64_t n_regions, double t) {
  for (int64_t i = 0; i + 1 < n_regions; ++i)
    if (t < boundaries[i + 1]) return i;
  return n_regions - 1;
}

/* samplers.hpp:488-491 */
double so_partition_offset(uint64_t seed, int64_t epoch, double l) {
  so_rng r = so_derive_stream(seed, 6, (uint64_t)epoch, 0, 0);
  return so_uniform_range(&r, 0.0, l);
}

/* partition.hpp:94-102 */
void so_signal_window(double lo, double hi, double tau, double T, double rate, int64_t* wlo,
                      int64_t* whi) {
  const double h = fmin(hi + tau, T);
  *wlo = (int64_t)ceil(lo * rate - 1e-9);
  *whi = (int64_t)ceil(h * rate - 1e-9);
}

/* ------------------------------------------------------------- samplers.hpp */

/* an event version; gen = 1: a generated version of arrival storage spec v2
 * (include/seis_philox.h): its arrivals are arrival_mean(x, t, j) + sigma z_j
 * with z_j the philox normal of its birth (key gseed, counter gsweep / gregion
 * / gstep), plus its overrides (ovr_d[k] at station ovr_st[k], in order);
 * `a` always holds those values */
typedef struct {
  uint64_t id;
  double x, t;
  double* a;
  int gen, n_ovr;
  uint64_t gseed;
  uint32_t gsweep, gregion, gstep, pad_;
  int ovr_st[8]; /* kGenOvr overrides, in acceptance order */
  double ovr_d[8];
} ev_t;

typedef struct {
  ev_t* e;
  int64_t n, cap;
} evlist_t;

static void evl_push(evlist_t* l, ev_t e) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 16;
    l->e = (ev_t*)realloc(l->e, sizeof(ev_t) * (size_t)l->cap);
  }
  l->e[l->n++] = e;
}

static ev_t ev_copy(const ev_t* src, int64_t S) {
  ev_t e = *src;
  e.a = (double*)malloc(sizeof(double) * (size_t)S);
  memcpy(e.a, src->a, sizeof(double) * (size_t)S);
  return e;
}

static void evl_free(evlist_t* l) {
  for (int64_t i = 0; i < l->n; ++i) free(l->e[i].a);
  free(l->e);
  l->e = NULL;
  l->n = l->cap = 0;
}

static evlist_t evl_clone(const evlist_t* src, int64_t S) {
  evlist_t l = {0, 0, 0};
  for (int64_t i = 0; i < src->n; ++i) evl_push(&l, ev_copy(&src->e[i], S));
  return l;
}

static int cmp_id(const void* a, const void* b) {
  const ev_t* x = (const ev_t*)a;
  const ev_t* y = (const ev_t*)b;
  return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

/* flat view of a list for so_delta / so_log_joint */
typedef struct {
  uint64_t* ids;
  double *x, *t, *arr;
  int64_t cap;
} flat_t;

static void flat_fill(flat_t* f, const evlist_t* l, int64_t S) {
  if (l->n > f->cap) {
    f->cap = l->n * 2 + 8;
    f->ids = (uint64_t*)realloc(f->ids, sizeof(uint64_t) * (size_t)f->cap);
    f->x = (double*)realloc(f->x, sizeof(double) * (size_t)f->cap);
    f->t = (double*)realloc(f->t, sizeof(double) * (size_t)f->cap);
    f->arr = (double*)realloc(f->arr, sizeof(double) * (size_t)(f->cap * S));
  }
  for (int64_t i = 0; i < l->n; ++i) {
    f->ids[i] = l->e[i].id;
    f->x[i] = l->e[i].x;
    f->t[i] = l->e[i].t;
    memcpy(f->arr + i * S, l->e[i].a, sizeof(double) * (size_t)S);
  }
}

static void flat_free(flat_t* f) {
  free(f->ids);
  free(f->x);
  free(f->t);
  free(f->arr);
}

struct so_run {
  int status;
  int64_t S;
  so_tape_rec* tape;
  int64_t n_tape, cap_tape;
  double* tarr;
  int64_t n_tarr, cap_tarr;
  int64_t* row_step;
  double* row_lj;
  int64_t* row_count;
  int64_t n_rows, cap_rows;
  evlist_t final;
  int64_t total_steps, total_accepted;
};

static void run_push_row(struct so_run* r, int64_t step, double lj, int64_t count) {
  if (r->n_rows == r->cap_rows) {
    r->cap_rows = r->cap_rows ? 2 * r->cap_rows : 64;
    r->row_step = (int64_t*)realloc(r->row_step, sizeof(int64_t) * (size_t)r->cap_rows);
    r->row_lj = (double*)realloc(r->row_lj, sizeof(double) * (size_t)r->cap_rows);
    r->row_count = (int64_t*)realloc(r->row_count, sizeof(int64_t) * (size_t)r->cap_rows);
  }
  r->row_step[r->n_rows] = step;
  r->row_lj[r->n_rows] = lj;
  r->row_count[r->n_rows] = count;
  r->n_rows++;
}

static so_tape_rec* run_push_tape(struct so_run* r) {
  if (r->n_tape == r->cap_tape) {
    r->cap_tape = r->cap_tape ? 2 * r->cap_tape : 1024;
    r->tape = (so_tape_rec*)realloc(r->tape, sizeof(so_tape_rec) * (size_t)r->cap_tape);
  }
  so_tape_rec* t = &r->tape[r->n_tape++];
  memset(t, 0, sizeof *t);
  return t;
}

static int64_t run_push_arr(struct so_run* r, const double* a, int64_t S) {
  if (r->n_tarr + S > r->cap_tarr) {
    r->cap_tarr = (r->cap_tarr + S) * 2;
    r->tarr = (double*)realloc(r->tarr, sizeof(double) * (size_t)r->cap_tarr);
  }
  const int64_t off = r->n_tarr;
  memcpy(r->tarr + off, a, sizeof(double) * (size_t)S);
  r->n_tarr += S;
  return off;
}

/* Proposal (proposals.hpp:57-63) */
typedef struct {
  int type, is_null;
  int n_removed, n_added;
  int64_t removed_idx[2]; /* indices into the local list */
  ev_t added[2];          /* owned arrivals */
  double logq_f, logq_r;
} prop_t;

static void prop_free(prop_t* p) {
  for (int i = 0; i < p->n_added; ++i) free(p->added[i].a);
  p->n_added = 0;
}

/* chain context: region, rng */
typedef struct {
  const so_model* m;
  const so_sampler* sc;
  double rlo, rhi;
  int rclosed;
  /* mode 0 */
  so_rng rng;
  /* mode 1 */
  uint32_t sweep, region, step;
  uint32_t step_base; /* global step index of this call's first step */
  /* ScoreOptions (density.hpp:182-189): chromatic = full window and [0, T]
   * (samplers.hpp:410); naive = signal_window and the region
   * (samplers.hpp:345-347) */
  int64_t wlo, whi;
  double slo, shi;
  int sclosed;
  int unconstrained; /* run_serial: no region constraint (samplers.hpp:300) */
} chain_t;

/* proposals.hpp:65-71 */
static int64_t events_in_region(const evlist_t* l, const chain_t* c, int64_t* idx) {
  int64_t k = 0;
  for (int64_t i = 0; i < l->n; ++i)
    if (region_contains(c->rlo, c->rhi, c->rclosed, l->e[i].t)) idx[k++] = i;
  return k;
}

static double draw_normal(chain_t* c, uint32_t i, double mean, double sd) {
  if (c->sc->rng_mode == 0) return so_normal(&c->rng, mean, sd);
  return mean + sd * (double)seis_normal(c->sc->seed, c->sweep, c->region, c->step, i);
}

/* cross_swap, proposals.hpp:182-194 */
static void cross_swap(double x1, double t1, double x2, double t2, double xl, double xr, double v,
                       double* nx1, double* nt1, double* nx2, double* nt2) {
  const double al1 = t1 + fabs(x1 - xl) / v;
  const double ar1 = t1 + fabs(x1 - xr) / v;
  const double al2 = t2 + fabs(x2 - xl) / v;
  const double ar2 = t2 + fabs(x2 - xr) / v;
  *nx1 = 0.5 * (xl + xr) + 0.5 * v * (al1 - ar2);
  *nt1 = 0.5 * (al1 + ar2) - (xr - xl) / (2.0 * v);
  *nx2 = 0.5 * (xl + xr) + 0.5 * v * (al2 - ar1);
  *nt2 = 0.5 * (al2 + ar1) - (xr - xl) / (2.0 * v);
}

static ev_t shifted(const so_model* m, const ev_t* before, double nx, double nt) {
  ev_t after = ev_copy(before, m->n_stations);
  after.x = nx;
  after.t = nt;
  if (before->gen) { /* spec v2: the residual sigma z of the birth kept exactly */
    for (int64_t j = 0; j < m->n_stations; ++j) {
      after.a[j] = arrival_mean(m, after.x, after.t, j) +
                   m->sigma_arrival * (double)seis_normal(before->gseed, before->gsweep,
                                                         before->gregion, before->gstep,
                                                         (uint32_t)j);
      for (int k = 0; k < before->n_ovr; ++k)
        if (before->ovr_st[k] == j) after.a[j] = after.a[j] + before->ovr_d[k];
    }
    return after;
  }
  for (int64_t j = 0; j < m->n_stations; ++j)
    after.a[j] += arrival_mean(m, after.x, after.t, j) - arrival_mean(m, before->x, before->t, j);
  return after;
}

/* propose_move, proposals.hpp:84-253; draw order follows the reference in
 * mode 0 and philox stream spec v1 (include/seis_philox.h) in mode 1. */
static void propose(chain_t* c, int type, const evlist_t* l, uint64_t new_id, int64_t* idxbuf,
                    prop_t* p) {
  const so_model* m = c->m;
  const so_sampler* sc = c->sc;
  const int64_t S = m->n_stations;
  memset(p, 0, sizeof *p);
  p->type = type;
  const int64_t k = events_in_region(l, c, idxbuf);
  seis_u32x4 d1 = {{0, 0, 0, 0}}, d2 = {{0, 0, 0, 0}};
  if (sc->rng_mode == 1) {
    d1 = seis_draw(sc->seed, c->sweep, c->region, c->step, SEIS_DRAW_SCALAR);
    d2 = seis_draw(sc->seed, c->sweep, c->region, c->step, SEIS_DRAW_PAIR);
  }
  const double sig = m->sigma_arrival;
  switch (type) {
    case 0: { /* birth, proposals.hpp:84-107 */
      ev_t e;
      memset(&e, 0, sizeof e);
      e.id = new_id;
      if (sc->rng_mode == 1 && sc->compact) { /* spec v2: a generated version */
        e.gen = 1;
        e.gseed = sc->seed;
        e.gsweep = c->sweep;
        e.gregion = c->region;
        e.gstep = c->step;
      }
      if (sc->rng_mode == 0) {
        e.t = so_uniform_range(&c->rng, c->rlo, c->rhi);
        e.x = so_uniform_range(&c->rng, 0.0, m->x_max);
      } else {
        e.t = c->rlo + (c->rhi - c->rlo) * seis_u53(d1.w[0], d1.w[1]);
        e.x = 0.0 + (m->x_max - 0.0) * seis_u53(d1.w[2], d1.w[3]);
      }
      e.a = (double*)malloc(sizeof(double) * (size_t)S);
      double alq = 0.0;
      for (int64_t j = 0; j < S; ++j) {
        const double mean = arrival_mean(m, e.x, e.t, j);
        e.a[j] = draw_normal(c, (uint32_t)j, mean, sig);
        alq += log_gaussian(e.a[j], mean, sig * sig);
      }
      p->logq_f = log(sc->weights[0]) - log(c->rhi - c->rlo) - log(m->x_max) + alq;
      p->logq_r = log(sc->weights[1]) - log((double)k + 1.0);
      p->n_added = 1;
      p->added[0] = e;
      return;
    }
    case 1: { /* death, proposals.hpp:111-138 */
      if (k == 0) {
        p->is_null = 1;
        return;
      }
      const uint64_t pick = sc->rng_mode == 0 ? so_uniform_index(&c->rng, (uint64_t)k)
                                              : seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
      const ev_t* v = &l->e[idxbuf[pick]];
      double alq = 0.0;
      for (int64_t j = 0; j < S; ++j)
        alq += log_gaussian(v->a[j], arrival_mean(m, v->x, v->t, j), sig * sig);
      p->logq_f = log(sc->weights[1]) - log((double)k);
      p->logq_r = log(sc->weights[0]) - log(c->rhi - c->rlo) - log(m->x_max) + alq;
      p->n_removed = 1;
      p->removed_idx[0] = idxbuf[pick];
      return;
    }
    case 2: { /* location, proposals.hpp:143-159 */
      if (k == 0) {
        p->is_null = 1;
        return;
      }
      const uint64_t pick = sc->rng_mode == 0 ? so_uniform_index(&c->rng, (uint64_t)k)
                                              : seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
      const ev_t* b = &l->e[idxbuf[pick]];
      const double nx = b->x + draw_normal(c, 0, 0.0, sc->step_location_x);
      const double nt = b->t + draw_normal(c, 1, 0.0, sc->step_location_t);
      p->n_removed = 1;
      p->removed_idx[0] = idxbuf[pick];
      p->n_added = 1;
      p->added[0] = shifted(m, b, nx, nt);
      return;
    }
    case 3: { /* arrival, proposals.hpp:161-174 */
      if (k == 0) {
        p->is_null = 1;
        return;
      }
      uint64_t pick, st;
      if (sc->rng_mode == 0) {
        pick = so_uniform_index(&c->rng, (uint64_t)k);
        st = so_uniform_index(&c->rng, (uint64_t)S);
      } else {
        pick = seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        st = seis_lemire(seis_u64(d1.w[2], d1.w[3]), (uint64_t)S);
      }
      const ev_t* b = &l->e[idxbuf[pick]];
      ev_t after = ev_copy(b, S);
      const double da = draw_normal(c, 0, 0.0, sc->step_arrival);
      after.a[st] += da;
      if (b->gen) { /* spec v2: up to 8 overrides stay generated, the next stores the row */
        if (b->n_ovr < 8) {
          after.ovr_st[after.n_ovr] = (int)st;
          after.ovr_d[after.n_ovr] = da;
          after.n_ovr++;
        } else {
          after.gen = 0;
        }
      }
      p->n_removed = 1;
      p->removed_idx[0] = idxbuf[pick];
      p->n_added = 1;
      p->added[0] = after;
      return;
    }
    default: { /* joint pair, proposals.hpp:200-234 */
      if (k < 2) {
        p->is_null = 1;
        return;
      }
      uint64_t i1, i2, pair;
      if (sc->rng_mode == 0) {
        i1 = so_uniform_index(&c->rng, (uint64_t)k);
        i2 = so_uniform_index(&c->rng, (uint64_t)k - 1);
      } else {
        i1 = seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        i2 = seis_lemire(seis_u64(d1.w[2], d1.w[3]), (uint64_t)k - 1);
      }
      if (i2 >= i1) ++i2;
      const ev_t* e1 = &l->e[idxbuf[i1]];
      const ev_t* e2 = &l->e[idxbuf[i2]];
      if (sc->rng_mode == 0)
        pair = so_uniform_index(&c->rng, (uint64_t)S - 1);
      else
        pair = seis_lemire(seis_u64(d2.w[0], d2.w[1]), (uint64_t)S - 1);
      const double xl = m->stations[pair], xr = m->stations[pair + 1];
      double n1x, n1t, n2x, n2t;
      cross_swap(e1->x, e1->t, e2->x, e2->t, xl, xr, m->v, &n1x, &n1t, &n2x, &n2t);
      n1x += draw_normal(c, 0, 0.0, sc->step_joint);
      n1t += draw_normal(c, 1, 0.0, sc->step_joint / m->v);
      n2x += draw_normal(c, 2, 0.0, sc->step_joint);
      n2t += draw_normal(c, 3, 0.0, sc->step_joint / m->v);
      p->n_removed = 2;
      p->removed_idx[0] = idxbuf[i1];
      p->removed_idx[1] = idxbuf[i2];
      p->n_added = 2;
      p->added[0] = shifted(m, e1, n1x, n1t);
      p->added[1] = shifted(m, e2, n2x, n2t);
      return;
    }
  }
}

/* apply_change, density.hpp:171-180: erase-by-id (order preserving), then
 * push_back the added events. Consumes p->added. */
static void apply_change(evlist_t* l, prop_t* p) {
  uint64_t rid[2];
  for (int r = 0; r < p->n_removed; ++r) rid[r] = l->e[p->removed_idx[r]].id;
  for (int r = 0; r < p->n_removed; ++r) {
    int64_t i = 0;
    while (i < l->n && l->e[i].id != rid[r]) ++i;
    free(l->e[i].a);
    memmove(&l->e[i], &l->e[i + 1], sizeof(ev_t) * (size_t)(l->n - i - 1));
    l->n--;
  }
  for (int a = 0; a < p->n_added; ++a) evl_push(l, p->added[a]);
  p->n_added = 0;
}

/* run_region_steps (samplers.hpp:115-138) with mh_step (proposals.hpp:265-293)
 * inlined, recording every step on the tape. */
static int64_t run_region_steps(struct so_run* run, chain_t* c, evlist_t* local,
                                const double* signals, int64_t steps, uint64_t id_base,
                                int want_tape, int64_t epoch, int64_t color, int64_t slot,
                                flat_t* flat, int64_t* idxbuf, int64_t* births_out) {
  const so_model* m = c->m;
  const so_sampler* sc = c->sc;
  const int64_t S = m->n_stations;
  int64_t births = 0, accepted = 0;
  for (int64_t i = 0; i < steps; ++i) {
    c->step = (uint32_t)(c->step_base + i);
    seis_u32x4 d0 = {{0, 0, 0, 0}};
    double um;
    if (sc->rng_mode == 0) {
      um = so_uniform(&c->rng);
    } else {
      d0 = seis_draw(sc->seed, c->sweep, c->region, c->step, SEIS_DRAW_MOVE);
      um = seis_u53(d0.w[0], d0.w[1]);
    }
    /* MoveDistribution::sample, proposals.hpp:33-41 */
    int type = 4;
    double cum = 0.0;
    for (int q = 0; q < 5; ++q) {
      cum += sc->weights[q];
      if (um < cum) {
        type = q;
        break;
      }
    }
    prop_t p;
    propose(c, type, local, id_base + (uint64_t)births, idxbuf, &p);
    so_tape_rec* rec = NULL;
    if (want_tape) {
      rec = run_push_tape(run);
      rec->epoch = epoch;
      rec->color = color;
      rec->region = c->region;
      rec->slot = slot;
      rec->step = (int64_t)c->step_base + i;
      rec->type = type;
      rec->is_null = p.is_null;
      rec->n_removed = p.n_removed;
      rec->n_added = p.n_added;
      for (int r = 0; r < p.n_removed; ++r) rec->removed_id[r] = local->e[p.removed_idx[r]].id;
      for (int a = 0; a < p.n_added; ++a) {
        rec->added_id[a] = p.added[a].id;
        rec->added_x[a] = p.added[a].x;
        rec->added_t[a] = p.added[a].t;
        const int64_t off = run_push_arr(run, p.added[a].a, S);
        if (a == 0) rec->added_arr_off = off;
      }
      rec->logq_f = p.logq_f;
      rec->logq_r = p.logq_r;
      rec->delta = -INFINITY;
    }
    int acc = 0;
    if (!p.is_null) {
      int constrained_out = 0;
      for (int a = 0; a < p.n_added && !c->unconstrained; ++a)
        if (!region_contains(c->rlo, c->rhi, c->rclosed, p.added[a].t)) {
          constrained_out = 1;
          break;
        }
      double log_r;
      double delta = -INFINITY;
      if (constrained_out) {
        log_r = -INFINITY;
      } else {
        flat_fill(flat, local, S);
        double ax[2], at[2];
        uint64_t aid[2];
        double* aarr = (double*)malloc(sizeof(double) * (size_t)(S * 2));
        for (int a = 0; a < p.n_added; ++a) {
          ax[a] = p.added[a].x;
          at[a] = p.added[a].t;
          aid[a] = p.added[a].id;
          memcpy(aarr + a * S, p.added[a].a, sizeof(double) * (size_t)S);
        }
        delta = so_delta(m, signals, local->n, flat->ids, flat->x, flat->t, flat->arr, p.n_removed,
                         p.removed_idx, p.n_added, aid, ax, at, aarr, c->wlo, c->whi, c->slo,
                         c->shi, c->sclosed);
        free(aarr);
        /* log_accept_ratio, proposals.hpp:255-258 */
        log_r = delta == -INFINITY ? -INFINITY : delta + p.logq_r - p.logq_f;
      }
      if (rec) {
        rec->constrained_out = constrained_out;
        rec->scored = !constrained_out;
        rec->delta = delta;
        rec->log_r = log_r;
      }
      if (log_r >= 0.0) {
        acc = 1;
      } else {
        const double u =
            sc->rng_mode == 0 ? so_uniform(&c->rng) : seis_u53(d0.w[2], d0.w[3]);
        if (rec) {
          rec->u_drawn = 1;
          rec->u = u;
        }
        if (log(u) < log_r) acc = 1;
      }
    }
    if (acc) {
      if (type == 0) births++;
      accepted++;
      apply_change(local, &p);
    }
    if (rec) rec->accepted = acc;
    prop_free(&p);
  }
  if (births_out) *births_out = births;
  return accepted;
}

/* run_chromatic, samplers.hpp:401-498 (+ an optional initial hypothesis; the
 * reference always starts empty, samplers.hpp:409). */
so_run* so_run_chromatic(const so_model* m, const double* signals, const so_sampler* sc,
                         int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                         const double* arr, int64_t want_tape, int64_t want_rowlj) {
  struct so_run* run = (struct so_run*)calloc(1, sizeof(struct so_run));
  const int64_t S = m->n_stations;
  run->S = S;
  int rc = so_validate_model(m);
  if (rc) {
    run->status = rc;
    return run;
  }
  /* SamplerConfig::validate, samplers.hpp:59-70; MoveDistribution::validate,
   * proposals.hpp:23-31 */
  if (sc->steps_per_epoch < 1 || sc->epochs < 1 || sc->n_regions < 1 || sc->record_every < 1 ||
      sc->burn_in_fraction < 0 || sc->burn_in_fraction >= 1) {
    run->status = fail(SO_EINVAL, "SamplerConfig: invalid");
    return run;
  }
  {
    double wsum = 0.0;
    for (int q = 0; q < 5; ++q) {
      if (sc->weights[q] < 0) {
        run->status = fail(SO_EINVAL, "MoveDistribution: negative weight");
        return run;
      }
      wsum += sc->weights[q];
    }
    if (fabs(wsum - 1.0) > 1e-12) {
      run->status = fail(SO_EINVAL, "MoveDistribution: weights must sum to 1");
      return run;
    }
  }
  const double tau = m->x_max / m->v;
  const double l = m->T / (double)sc->n_regions;
  const int64_t bcap = sc->n_regions + 8;
  double* bnd = (double*)malloc(sizeof(double) * (size_t)bcap);
  int32_t* col = (int32_t*)malloc(sizeof(int32_t) * (size_t)bcap);
  int64_t nreg;
  int32_t ncol;
  rc = so_partition(m->T, l, 0.0, tau, bcap, &nreg, bnd, col, &ncol);
  if (rc) {
    run->status = rc;
    free(bnd);
    free(col);
    return run;
  }
  evlist_t global = {0, 0, 0};
  uint64_t next_base = 0;
  for (int64_t i = 0; i < n_init; ++i) {
    ev_t e;
    memset(&e, 0, sizeof e);
    e.id = ids[i];
    e.x = x[i];
    e.t = t[i];
    e.a = (double*)malloc(sizeof(double) * (size_t)S);
    memcpy(e.a, arr + i * S, sizeof(double) * (size_t)S);
    evl_push(&global, e);
    if (ids[i] + 1 > next_base) next_base = ids[i] + 1;
  }
  qsort(global.e, (size_t)global.n, sizeof(ev_t), cmp_id);
  flat_t flat = {0, 0, 0, 0, 0};
  int64_t* idxbuf = NULL;
  int64_t idxcap = 0;
  const int64_t k = sc->steps_per_epoch;
  int64_t executed = 0, last_recorded = 0;
  const int64_t planned = sc->epochs * sc->steps_per_epoch * sc->n_regions;
  (void)planned;
  if (want_rowlj) {
    flat_fill(&flat, &global, S);
    run_push_row(run, 0, so_log_joint(m, signals, global.n, flat.ids, flat.x, flat.t, flat.arr),
                 global.n);
  } else {
    run_push_row(run, 0, 0.0, global.n);
  }
  int64_t* cr = (int64_t*)malloc(sizeof(int64_t) * (size_t)bcap);
  for (int64_t epoch = 0; epoch < sc->epochs; ++epoch) {
    for (int color = 0; color < ncol; ++color) {
      int64_t ncr = 0;
      for (int64_t i = 0; i < nreg; ++i)
        if (col[i] == color) cr[ncr++] = i;
      if (ncr == 0) continue;
      evlist_t* results = (evlist_t*)calloc((size_t)ncr, sizeof(evlist_t));
      for (int64_t slot = 0; slot < ncr; ++slot) {
        const int64_t ri = cr[slot];
        chain_t c;
        memset(&c, 0, sizeof c);
        c.m = m;
        c.sc = sc;
        c.rlo = bnd[ri];
        c.rhi = bnd[ri + 1];
        c.rclosed = (ri + 1 == nreg);
        c.sweep = (uint32_t)epoch;
        c.region = (uint32_t)ri;
        c.wlo = 0;
        c.whi = so_n_samples(m);
        c.slo = 0.0;
        c.shi = m->T;
        c.sclosed = 1;
        if (sc->rng_mode == 0)
          c.rng = so_derive_stream(sc->seed, 5, (uint64_t)epoch, (uint64_t)color, (uint64_t)ri);
        evlist_t local = evl_clone(&global, S); /* samplers.hpp:448 */
        if (local.n + k + 8 > idxcap) {
          idxcap = local.n + k + 8;
          idxbuf = (int64_t*)realloc(idxbuf, sizeof(int64_t) * (size_t)idxcap);
        }
        const uint64_t id_base = next_base + (uint64_t)slot * (uint64_t)k;
        run->total_accepted += run_region_steps(run, &c, &local, signals, k, id_base, (int)want_tape,
                                                epoch, color, slot, &flat, idxbuf, NULL);
        /* samplers.hpp:459-462: own events in local order */
        for (int64_t i = 0; i < local.n; ++i)
          if (region_contains(c.rlo, c.rhi, c.rclosed, local.e[i].t))
            evl_push(&results[slot], ev_copy(&local.e[i], S));
        evl_free(&local);
      }
      /* barrier merge, samplers.hpp:471-482 */
      evlist_t merged = {0, 0, 0};
      for (int64_t i = 0; i < global.n; ++i) {
        const int64_t r = so_region_of(bnd, nreg, global.e[i].t);
        if (col[r] != color) evl_push(&merged, ev_copy(&global.e[i], S));
      }
      for (int64_t slot = 0; slot < ncr; ++slot) {
        for (int64_t i = 0; i < results[slot].n; ++i) evl_push(&merged, results[slot].e[i]);
        free(results[slot].e);
      }
      free(results);
      qsort(merged.e, (size_t)merged.n, sizeof(ev_t), cmp_id);
      evl_free(&global);
      global = merged;
      next_base += (uint64_t)ncr * (uint64_t)k;
      executed += ncr * k;
      /* record(false), samplers.hpp:424-434 */
      if (executed - last_recorded >= sc->record_every) {
        last_recorded = executed;
        double lj = 0.0;
        if (want_rowlj) {
          flat_fill(&flat, &global, S);
          lj = so_log_joint(m, signals, global.n, flat.ids, flat.x, flat.t, flat.arr);
        }
        run_push_row(run, executed, lj, global.n);
      }
    }
    if (sc->dynamic && epoch + 1 < sc->epochs) { /* samplers.hpp:488-493 */
      const double u = so_partition_offset(sc->seed, epoch + 1, l);
      rc = so_partition(m->T, l, u, tau, bcap, &nreg, bnd, col, &ncol);
      if (rc) {
        run->status = rc;
        break;
      }
    }
  }
  if (run->status == 0 && last_recorded != executed) {
    double lj = 0.0;
    if (want_rowlj) {
      flat_fill(&flat, &global, S);
      lj = so_log_joint(m, signals, global.n, flat.ids, flat.x, flat.t, flat.arr);
    }
    run_push_row(run, executed, lj, global.n);
  }
  run->total_steps = executed;
  run->final = global;
  free(cr);
  free(idxbuf);
  flat_free(&flat);
  free(bnd);
  free(col);
  return run;
}


/* run_naive_parallel, samplers.hpp:321-394: independent per-region chains
 * from the empty hypothesis, no coloring, prior restricted to the region and
 * the likelihood to the region's signal window; the trace is the union of
 * the per-region checkpoints (every record_every local steps). */
so_run* so_run_naive(const so_model* m, const double* signals, const so_sampler* sc,
                     int64_t want_tape, int64_t want_rowlj) {
  struct so_run* run = (struct so_run*)calloc(1, sizeof(struct so_run));
  const int64_t S = m->n_stations;
  run->S = S;
  int rc = so_validate_model(m);
  if (rc) {
    run->status = rc;
    return run;
  }
  if (sc->steps_per_epoch < 1 || sc->epochs < 1 || sc->n_regions < 1 || sc->record_every < 1 ||
      sc->burn_in_fraction < 0 || sc->burn_in_fraction >= 1) {
    run->status = fail(SO_EINVAL, "SamplerConfig: invalid");
    return run;
  }
  const double tau = m->x_max / m->v;
  const double l = m->T / (double)sc->n_regions;
  const int64_t bcap = sc->n_regions + 8;
  double* bnd = (double*)malloc(sizeof(double) * (size_t)bcap);
  int64_t nreg = 0;
  /* build_partition only (no color_partition), samplers.hpp:326-327 */
  {
    int64_t nb = 0;
    if (!(l > 0) || l > m->T) {
      run->status = fail(SO_EINVAL, "build_partition: need 0 < l <= T");
      free(bnd);
      return run;
    }
    bnd[nb++] = 0.0;
    double b = l;
    while (b < m->T - 1e-9) {
      bnd[nb++] = b;
      b += l;
    }
    bnd[nb++] = m->T;
    nreg = nb - 1;
  }
  const int64_t spr = sc->epochs * sc->steps_per_epoch;
  const int64_t n_cp = (spr + sc->record_every - 1) / sc->record_every + 1;
  evlist_t* cps = (evlist_t*)calloc((size_t)(nreg * n_cp), sizeof(evlist_t));
  int64_t* cp_steps = (int64_t*)calloc((size_t)n_cp, sizeof(int64_t));
  flat_t flat = {0, 0, 0, 0, 0};
  int64_t idxcap = spr + 16;
  int64_t* idxbuf = (int64_t*)malloc(sizeof(int64_t) * (size_t)idxcap);
  for (int64_t r = 0; r < nreg; ++r) {
    chain_t c;
    memset(&c, 0, sizeof c);
    c.m = m;
    c.sc = sc;
    c.rlo = bnd[r];
    c.rhi = bnd[r + 1];
    c.rclosed = (r + 1 == nreg);
    c.sweep = 0;
    c.region = (uint32_t)r;
    so_signal_window(c.rlo, c.rhi, tau, m->T, m->sample_rate, &c.wlo, &c.whi);
    c.slo = c.rlo;
    c.shi = c.rhi;
    c.sclosed = c.rclosed;
    if (sc->rng_mode == 0) c.rng = so_derive_stream(sc->seed, 5, 0, 0, (uint64_t)r);
    uint64_t id_base = ((uint64_t)r + 1) << 32;
    evlist_t local = {0, 0, 0};
    cps[r * n_cp + 0] = evl_clone(&local, S);
    int64_t done = 0, ci = 0;
    while (done < spr) {
      const int64_t chunk = sc->record_every < spr - done ? sc->record_every : spr - done;
      c.step_base = (uint32_t)done;
      int64_t births = 0;
      run->total_accepted += run_region_steps(run, &c, &local, signals, chunk, id_base,
                                              (int)want_tape, 0, 0, r, &flat, idxbuf, &births);
      id_base += (uint64_t)births;
      done += chunk;
      ++ci;
      cps[r * n_cp + ci] = evl_clone(&local, S);
      cp_steps[ci] = done;
    }
    evl_free(&local);
  }
  /* union trace rows, samplers.hpp:366-392 */
  for (int64_t ci = 0; ci < n_cp; ++ci) {
    evlist_t merged = {0, 0, 0};
    for (int64_t r = 0; r < nreg; ++r)
      for (int64_t i = 0; i < cps[r * n_cp + ci].n; ++i)
        evl_push(&merged, ev_copy(&cps[r * n_cp + ci].e[i], S));
    qsort(merged.e, (size_t)merged.n, sizeof(ev_t), cmp_id);
    double lj = 0.0;
    if (want_rowlj) {
      flat_fill(&flat, &merged, S);
      lj = so_log_joint(m, signals, merged.n, flat.ids, flat.x, flat.t, flat.arr);
    }
    run_push_row(run, cp_steps[ci] * nreg, lj, merged.n);
    if (ci + 1 == n_cp) {
      run->final = merged;
    } else {
      evl_free(&merged);
    }
  }
  for (int64_t i = 0; i < nreg * n_cp; ++i) evl_free(&cps[i]);
  free(cps);
  free(cp_steps);
  free(idxbuf);
  flat_free(&flat);
  free(bnd);
  run->total_steps = spr * nreg;
  return run;
}

int so_run_status(const so_run* r) { return r->status; }

void so_run_counts(const so_run* r, int64_t* n_tape, int64_t* n_tape_arr, int64_t* n_rows,
                   int64_t* n_final, int64_t* total_steps, int64_t* total_accepted) {
  *n_tape = r->n_tape;
  *n_tape_arr = r->n_tarr;
  *n_rows = r->n_rows;
  *n_final = r->final.n;
  *total_steps = r->total_steps;
  *total_accepted = r->total_accepted;
}

void so_run_tape(const so_run* r, so_tape_rec* recs, double* arr) {
  if (r->n_tape) memcpy(recs, r->tape, sizeof(so_tape_rec) * (size_t)r->n_tape);
  if (r->n_tarr) memcpy(arr, r->tarr, sizeof(double) * (size_t)r->n_tarr);
}

void so_run_rows(const so_run* r, int64_t* step, double* log_joint, int64_t* event_count) {
  for (int64_t i = 0; i < r->n_rows; ++i) {
    step[i] = r->row_step[i];
    log_joint[i] = r->row_lj[i];
    event_count[i] = r->row_count[i];
  }
}

void so_run_final(const so_run* r, uint64_t* ids, double* x, double* t, double* arr) {
  for (int64_t i = 0; i < r->final.n; ++i) {
    ids[i] = r->final.e[i].id;
    x[i] = r->final.e[i].x;
    t[i] = r->final.e[i].t;
    memcpy(arr + i * r->S, r->final.e[i].a, sizeof(double) * (size_t)r->S);
  }
}

void so_run_free(so_run* r) {
  if (!r) return;
  struct so_run* q = (struct so_run*)r;
  free(q->tape);
  free(q->tarr);
  free(q->row_step);
  free(q->row_lj);
  free(q->row_count);
  evl_free(&q->final);
  free(q);
}

/* ------------------------------------------------ philox stream spec v1 probes */
void so_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
               uint32_t* out) {
  const seis_u32x4 r = seis_philox4x32_10(c0, c1, c2, c3, k0, k1);
  for (int i = 0; i < 4; ++i) out[i] = r.w[i];
}

float so_philox_normal(uint64_t seed, uint32_t sweep, uint32_t region, uint32_t step,
                       uint32_t i) {
  return seis_normal(seed, sweep, region, step, i);
}

float so_bm(uint32_t w0, uint32_t w1) { return seis_bm(w0, w1); }

/* ------------------------------------------------------------ evaluation.hpp */

typedef struct {
  uint64_t id;
  double x, t;
} pt_t;

static int cmp_tx(const void* a, const void* b) {
  const pt_t* p = (const pt_t*)a;
  const pt_t* q = (const pt_t*)b;
  if (p->t != q->t) return p->t < q->t ? -1 : 1;
  if (p->x != q->x) return p->x < q->x ? -1 : 1;
  return p->id < q->id ? -1 : (p->id > q->id ? 1 : 0);
}

/* match_events, evaluation.hpp:51-103: greedy matching in ascending (t, x)
 * order; a pair counts when within threshold in time and in distance
 * separately. out = {precision, recall, location_error, n_matched}. */
int so_match_events(int64_t nt, const uint64_t* tid, const double* tx, const double* tt,
                    int64_t ni, const uint64_t* iid, const double* ix, const double* it,
                    double threshold, double* out) {
  if (!(threshold > 0)) return fail(SO_EINVAL, "match_events: threshold must be > 0");
  pt_t* T = (pt_t*)malloc(sizeof(pt_t) * (size_t)(nt + 1));
  pt_t* I = (pt_t*)malloc(sizeof(pt_t) * (size_t)(ni + 1));
  char* taken = (char*)calloc((size_t)ni + 1, 1);
  for (int64_t i = 0; i < nt; ++i) T[i] = (pt_t){tid[i], tx[i], tt[i]};
  for (int64_t i = 0; i < ni; ++i) I[i] = (pt_t){iid[i], ix[i], it[i]};
  qsort(T, (size_t)nt, sizeof(pt_t), cmp_tx);
  qsort(I, (size_t)ni, sizeof(pt_t), cmp_tx);
  int64_t matched = 0;
  double sum = 0.0;
  for (int64_t a = 0; a < nt; ++a) {
    int64_t best = ni;
    double best_dist = 0.0;
    for (int64_t i = 0; i < ni; ++i) {
      if (taken[i]) continue;
      const double dx = T[a].x - I[i].x;
      const double dt = T[a].t - I[i].t;
      const double dist = sqrt(dx * dx + dt * dt);
      if (best == ni || dist < best_dist) {
        best = i;
        best_dist = dist;
      }
    }
    if (best == ni) continue;
    if (fabs(T[a].t - I[best].t) < threshold && fabs(T[a].x - I[best].x) < threshold) {
      taken[best] = 1;
      ++matched;
      sum += best_dist;
    }
  }
  out[0] = ni == 0 ? 1.0 : (double)matched / (double)ni;
  out[1] = nt == 0 ? 1.0 : (double)matched / (double)nt;
  out[2] = matched ? sum / (double)matched : 0.0;
  out[3] = (double)matched;
  free(T);
  free(I);
  free(taken);
  return SO_OK;
}


/* run_serial, samplers.hpp:282-315: one chain over config.full_region()
 * without the region constraint, default ScoreOptions (full window, [0, T]),
 * stream derive_stream(seed, kChain, 0, 0, 0) in rng_mode 0 and philox
 * (sweep 0, region 0, chain step) in rng_mode 1; a trace row after every
 * record_every steps. The final list is returned sorted by id (the engine's
 * order; the reference keeps list order, a permutation of it). */
so_run* so_run_serial(const so_model* m, const double* signals, const so_sampler* sc,
                      int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                      const double* arr, int64_t want_tape, int64_t want_rowlj) {
  struct so_run* run = (struct so_run*)calloc(1, sizeof(struct so_run));
  const int64_t S = m->n_stations;
  run->S = S;
  int rc = so_validate_model(m);
  if (rc) {
    run->status = rc;
    return run;
  }
  if (sc->steps_per_epoch < 1 || sc->epochs < 1 || sc->n_regions < 1 || sc->record_every < 1 ||
      sc->burn_in_fraction < 0 || sc->burn_in_fraction >= 1) {
    run->status = fail(SO_EINVAL, "SamplerConfig: invalid");
    return run;
  }
  chain_t c;
  memset(&c, 0, sizeof c);
  c.m = m;
  c.sc = sc;
  c.rlo = 0.0;
  c.rhi = m->T;
  c.rclosed = 1;
  c.unconstrained = 1;
  c.wlo = 0;
  c.whi = so_n_samples(m);
  c.slo = 0.0;
  c.shi = m->T;
  c.sclosed = 1;
  if (sc->rng_mode == 0) c.rng = so_derive_stream(sc->seed, 5, 0, 0, 0);
  const int64_t total = sc->epochs * sc->steps_per_epoch;
  flat_t flat = {0, 0, 0, 0, 0};
  int64_t* idxbuf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 16));
  /* the reference starts empty (samplers.hpp:291); an initial hypothesis (the
   * engine's resident one) starts in id order, births numbered above it */
  evlist_t local = {0, 0, 0};
  uint64_t id_base = 0;
  for (int64_t i = 0; i < n_init; ++i) {
    ev_t e;
    memset(&e, 0, sizeof e);
    e.id = ids[i];
    e.x = x[i];
    e.t = t[i];
    e.a = (double*)malloc(sizeof(double) * (size_t)S);
    memcpy(e.a, arr + i * S, sizeof(double) * (size_t)S);
    evl_push(&local, e);
    if (ids[i] + 1 > id_base) id_base = ids[i] + 1;
  }
  if (local.n) qsort(local.e, (size_t)local.n, sizeof(ev_t), cmp_id);
  int64_t done = 0;
  run_push_row(run, 0, 0.0, local.n);
  if (want_rowlj) {
    flat_fill(&flat, &local, S);
    run->row_lj[0] = so_log_joint(m, signals, local.n, flat.ids, flat.x, flat.t, flat.arr);
  }
  while (done < total) {
    const int64_t chunk = sc->record_every < total - done ? sc->record_every : total - done;
    c.step_base = (uint32_t)done;
    int64_t births = 0;
    run->total_accepted += run_region_steps(run, &c, &local, signals, chunk, id_base,
                                            (int)want_tape, 0, 0, 0, &flat, idxbuf, &births);
    id_base += (uint64_t)births;
    done += chunk;
    double lj = 0.0;
    if (want_rowlj) {
      flat_fill(&flat, &local, S);
      lj = so_log_joint(m, signals, local.n, flat.ids, flat.x, flat.t, flat.arr);
    }
    run_push_row(run, done, lj, local.n);
  }
  qsort(local.e, (size_t)local.n, sizeof(ev_t), cmp_id);
  run->final = local;
  run->total_steps = total;
  free(idxbuf);
  flat_free(&flat);
  return run;
}
