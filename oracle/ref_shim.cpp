// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNCHANGED reference headers (/root/reference/proj/include,
// read in place, never copied) into oracle/_ref/libseisref.so and exposes them
// through the same flat C API as the C restatement (seis_oracle.h), with the
// prefix sr_ instead of so_. Used (a) to pin the restatement and generate the
// golden vectors under tests/golden/, and (b) as the reference CPU arm of
// bench.py (sr_bench_region_steps, sr_bench_run_sampler).
//
// The tape-recording chromatic driver below composes the reference's own
// building blocks (build_partition/color_partition, derive_stream,
// MoveDistribution::sample, propose_move, delta_log_joint, apply_change) in
// the order of run_chromatic / run_region_steps / mh_step
// (samplers.hpp:115-138,401-498; proposals.hpp:265-293); sr_run_sampler runs
// the reference's run_sampler itself so tests can check the composed driver
// against it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "seismic/density.hpp"
#include "seismic/evaluation.hpp"
#include "seismic/model.hpp"
#include "seismic/partition.hpp"
#include "seismic/proposals.hpp"
#include "seismic/rng.hpp"
#include "seismic/samplers.hpp"
#include "seismic/worldgen.hpp"

#include "seis_oracle.h"

using namespace seismic;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& m) {
  g_err = m;
  return code;
}

ModelConfig to_config(const so_model* m) {
  ModelConfig c;
  c.lambda_rate = m->lambda_rate;
  c.T = m->T;
  c.x_max = m->x_max;
  c.v = m->v;
  c.sigma_arrival = m->sigma_arrival;
  c.t_s = m->t_s;
  c.var_noise = m->var_noise;
  c.var_event = m->var_event;
  c.sample_rate = m->sample_rate;
  c.stations.assign(m->stations, m->stations + m->n_stations);
  return c;
}

ObservedSignals to_signals(const ModelConfig& c, const double* sig) {
  ObservedSignals s;
  const std::size_t S = c.n_stations();
  const auto n = static_cast<std::size_t>(c.n_samples());
  s.station.resize(S);
  for (std::size_t j = 0; j < S; ++j) s.station[j].assign(sig + j * n, sig + (j + 1) * n);
  return s;
}

std::vector<Event> to_events(std::size_t S, int64_t N, const uint64_t* ids, const double* x,
                             const double* t, const double* arr) {
  std::vector<Event> ev(static_cast<std::size_t>(N));
  for (int64_t i = 0; i < N; ++i) {
    ev[i].id = ids[i];
    ev[i].x = x[i];
    ev[i].t = t[i];
    ev[i].arrivals.assign(arr + i * S, arr + (i + 1) * S);
  }
  return ev;
}

void from_world(const World& w, int64_t cap, int64_t* n_events, uint64_t* ids, double* x,
                double* t, double* arr, double* sig) {
  const std::size_t S = w.config.n_stations();
  const auto n = static_cast<std::size_t>(w.config.n_samples());
  *n_events = static_cast<int64_t>(w.events.size());
  if (*n_events > cap) throw std::runtime_error("event capacity too small");
  for (std::size_t i = 0; i < w.events.size(); ++i) {
    ids[i] = w.events[i].id;
    x[i] = w.events[i].x;
    t[i] = w.events[i].t;
    std::copy(w.events[i].arrivals.begin(), w.events[i].arrivals.end(), arr + i * S);
  }
  for (std::size_t j = 0; j < S; ++j)
    std::copy(w.signals.station[j].begin(), w.signals.station[j].end(), sig + j * n);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SO_OK;
  } catch (const std::invalid_argument& e) {
    return set_err(SO_EINVAL, e.what());
  } catch (const std::exception& e) {
    return set_err(SO_ERUNTIME, e.what());
  }
}

SamplerConfig to_sampler(const so_sampler* s) {
  SamplerConfig sc;
  sc.algorithm = s->dynamic ? Algorithm::ChromaticDynamic : Algorithm::ChromaticStatic;
  sc.steps_per_epoch = s->steps_per_epoch;
  sc.epochs = s->epochs;
  sc.n_regions = static_cast<int>(s->n_regions);
  sc.workers = 1;
  sc.seed = s->seed;
  sc.burn_in_fraction = s->burn_in_fraction;
  sc.record_every = s->record_every;
  for (int i = 0; i < 5; ++i) sc.moves.weights[static_cast<std::size_t>(i)] = s->weights[i];
  sc.step_sizes.location_x = s->step_location_x;
  sc.step_sizes.location_t = s->step_location_t;
  sc.step_sizes.arrival = s->step_arrival;
  sc.step_sizes.joint = s->step_joint;
  return sc;
}

}  // namespace

struct sr_run {
  int status = 0;
  std::size_t S = 0;
  std::vector<so_tape_rec> tape;
  std::vector<double> tarr;
  std::vector<int64_t> row_step, row_count;
  std::vector<double> row_lj;
  std::vector<Event> final;
  int64_t total_steps = 0, total_accepted = 0;
};

extern "C" {

const char* sr_last_error(void) { return g_err.c_str(); }

int sr_validate_model(const so_model* m) {
  return guarded([&] { to_config(m).validate(); });
}

int64_t sr_n_samples(const so_model* m) { return to_config(m).n_samples(); }

void sr_arrival_range(const so_model* m, double a, int64_t* lo, int64_t* hi) {
  const SampleRange r = arrival_sample_range(to_config(m), a);
  *lo = r.begin;
  *hi = r.end;
}

uint64_t sr_derive_u64(uint64_t seed, uint64_t purpose, uint64_t i0, uint64_t i1, uint64_t i2,
                       int64_t n, uint64_t* out) {
  Rng r = derive_stream(seed, purpose, i0, i1, i2);
  for (int64_t k = 0; k < n; ++k) out[k] = r.next_u64();
  return 0;
}

void sr_derive_draws(uint64_t seed, uint64_t purpose, uint64_t i0, uint64_t i1, uint64_t i2,
                     int64_t n, double* uniforms, double* normals, uint64_t idx_n,
                     uint64_t* indices) {
  Rng a = derive_stream(seed, purpose, i0, i1, i2);
  Rng b = a, c = a;
  for (int64_t k = 0; k < n; ++k) uniforms[k] = a.uniform();
  for (int64_t k = 0; k < n; ++k) normals[k] = b.normal();
  for (int64_t k = 0; k < n; ++k) indices[k] = c.uniform_index(idx_n);
}

uint64_t sr_poisson(uint64_t seed, uint64_t purpose, double mean) {
  Rng r = derive_stream(seed, purpose);
  return r.poisson(mean);
}

double sr_log_joint(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                    const double* x, const double* t, const double* arr) {
  const ModelConfig c = to_config(m);
  World w{c, to_events(c.n_stations(), N, ids, x, t, arr), to_signals(c, signals)};
  return log_joint(w);
}

double sr_delta(const so_model* m, const double* signals, int64_t N, const uint64_t* ids,
                const double* x, const double* t, const double* arr, int64_t n_removed,
                const int64_t* removed_idx, int64_t n_added, const uint64_t* added_ids,
                const double* added_x, const double* added_t, const double* added_arr,
                int64_t wlo, int64_t whi, double slo, double shi, int64_t sclosed) {
  const ModelConfig c = to_config(m);
  const std::size_t S = c.n_stations();
  World w{c, to_events(S, N, ids, x, t, arr), to_signals(c, signals)};
  Change ch;
  for (int64_t r = 0; r < n_removed; ++r)
    ch.removed.push_back(w.events[static_cast<std::size_t>(removed_idx[r])]);
  for (int64_t a = 0; a < n_added; ++a) {
    Event e;
    e.id = added_ids[a];
    e.x = added_x[a];
    e.t = added_t[a];
    e.arrivals.assign(added_arr + a * S, added_arr + (a + 1) * S);
    ch.added.push_back(e);
  }
  ScoreOptions opts{SampleRange{wlo, whi}, TimeRegion{{slo, shi}, sclosed != 0}};
  return delta_log_joint(w, ch, opts);
}

int sr_sample_world(const so_model* m, uint64_t seed, int64_t cap, int64_t* n_events,
                    uint64_t* ids, double* x, double* t, double* arr, double* signals) {
  return guarded([&] {
    const World w = sample_world(to_config(m), seed);
    from_world(w, cap, n_events, ids, x, t, arr, signals);
  });
}

// Thomas cluster process of BASELINE config[4]: the engine's
// host generator (worldgen.cpp seis_thomas_events) drawn here with the
// reference's own Rng/derive_stream under purpose ids 100-102 (outside the
// reference's 1..7), so the reference arm builds its world without the engine.
int sr_thomas_events(uint64_t seed, double x_max, double T, double parent_mean,
                     double child_mean, double sx, double st, int64_t cap, int64_t* n, double* cx,
                     double* ct) {
  return guarded([&] {
    Rng pc = derive_stream(seed, 100);
    const uint64_t np = pc.poisson(parent_mean);
    int64_t k = 0;
    for (uint64_t p = 0; p < np; ++p) {
      Rng pr = derive_stream(seed, 101, p);
      const double px = pr.uniform(0.0, x_max), pt = pr.uniform(0.0, T);
      Rng ch = derive_stream(seed, 102, p);
      const uint64_t nc = ch.poisson(child_mean);
      for (uint64_t c = 0; c < nc; ++c) {
        const double x = px + ch.normal(0.0, sx), t = pt + ch.normal(0.0, st);
        if (x < 0.0 || x > x_max || t < 0.0 || t >= T) continue;
        if (k < cap) {
          cx[k] = x;
          ct[k] = t;
        }
        ++k;
      }
    }
    *n = k;
    if (k > cap) throw std::runtime_error("capacity");
  });
}

int sr_make_world_with_events(const so_model* m, int64_t n, const double* cx, const double* ct,
                              uint64_t seed, uint64_t* ids, double* x, double* t, double* arr,
                              double* signals) {
  return guarded([&] {
    std::vector<std::pair<double, double>> coords;
    for (int64_t i = 0; i < n; ++i) coords.emplace_back(cx[i], ct[i]);
    const World w = make_world_with_events(to_config(m), coords, seed);
    int64_t got = 0;
    from_world(w, n, &got, ids, x, t, arr, signals);
  });
}

int sr_partition(double T, double l, double offset, double tau, int64_t cap, int64_t* n_regions,
                 double* boundaries, int32_t* colors, int32_t* n_colors) {
  return guarded([&] {
    Partition p = build_partition(T, l, offset);
    *n_regions = static_cast<int64_t>(p.n_regions());
    if (static_cast<int64_t>(p.boundaries.size()) > cap)
      throw std::runtime_error("partition capacity");
    std::copy(p.boundaries.begin(), p.boundaries.end(), boundaries);
    p = color_partition(p, tau);
    for (std::size_t i = 0; i < p.colors.size(); ++i) colors[i] = p.colors[i];
    *n_colors = p.n_colors;
  });
}

int64_t sr_region_of(const double* boundaries, int64_t n_regions, double t) {
  Partition p;
  p.boundaries.assign(boundaries, boundaries + n_regions + 1);
  for (int64_t i = 0; i < n_regions; ++i)
    p.regions.push_back(TimeInterval{boundaries[i], boundaries[i + 1]});
  return static_cast<int64_t>(p.region_of(t));
}

double sr_partition_offset(uint64_t seed, int64_t epoch, double l) {
  Rng r = derive_stream(seed, streams::kPartitionOffset, static_cast<uint64_t>(epoch));
  return r.uniform(0.0, l);
}

void sr_signal_window(double lo, double hi, double tau, double T, double rate, int64_t* wlo,
                      int64_t* whi) {
  const SampleRange r = signal_window(TimeInterval{lo, hi}, tau, T, rate);
  *wlo = r.begin;
  *whi = r.end;
}

// Tape-recording chromatic driver composed from reference functions; the
// control flow is run_chromatic (samplers.hpp:401-498) with run_region_steps
// (samplers.hpp:115-138) and mh_step (proposals.hpp:265-293) unrolled so the
// uniform drawn by mh_step and every proposal can be recorded.
sr_run* sr_run_chromatic(const so_model* mm, const double* signals, const so_sampler* s,
                         int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                         const double* arr, int64_t want_tape, int64_t want_rowlj) {
  auto* run = new sr_run;
  run->status = guarded([&] {
    if (s->rng_mode != 0) throw std::invalid_argument("reference supports rng_mode 0 only");
    const ModelConfig config = to_config(mm);
    const SamplerConfig sc = to_sampler(s);
    config.validate();
    sc.validate();
    const std::size_t S = config.n_stations();
    run->S = S;
    const ObservedSignals sig = to_signals(config, signals);
    const double tau = config.x_max / config.v;
    const double l = config.T / sc.n_regions;
    Partition partition = color_partition(build_partition(config.T, l, 0.0), tau);
    World global{config, to_events(S, n_init, ids, x, t, arr), sig};
    detail::sort_by_id(global.events);
    std::uint64_t next_base = 0;
    for (const Event& e : global.events) next_base = std::max(next_base, e.id + 1);
    const ScoreOptions opts = default_score_options(config);
    std::int64_t executed = 0, last_recorded = 0;
    auto record = [&](bool force) {
      if (!force && executed - last_recorded < sc.record_every) return;
      last_recorded = executed;
      run->row_step.push_back(executed);
      run->row_lj.push_back(want_rowlj ? log_joint(global) : 0.0);
      run->row_count.push_back(static_cast<int64_t>(global.events.size()));
    };
    run->row_step.push_back(0);
    run->row_lj.push_back(want_rowlj ? log_joint(global) : 0.0);
    run->row_count.push_back(static_cast<int64_t>(global.events.size()));
    for (std::int64_t epoch = 0; epoch < sc.epochs; ++epoch) {
      for (int color = 0; color < partition.n_colors; ++color) {
        std::vector<std::size_t> color_regions;
        for (std::size_t i = 0; i < partition.n_regions(); ++i)
          if (partition.colors[i] == color) color_regions.push_back(i);
        if (color_regions.empty()) continue;
        std::vector<std::vector<Event>> results(color_regions.size());
        for (std::size_t slot = 0; slot < color_regions.size(); ++slot) {
          const std::size_t region_index = color_regions[slot];
          const TimeRegion region = partition.region(region_index);
          World local{config, global.events, sig};
          Rng rng = derive_stream(sc.seed, streams::kChain, static_cast<uint64_t>(epoch),
                                  static_cast<uint64_t>(color), region_index);
          const std::uint64_t id_base =
              next_base + static_cast<std::uint64_t>(slot) *
                              static_cast<std::uint64_t>(sc.steps_per_epoch);
          std::int64_t births = 0;
          for (std::int64_t i = 0; i < sc.steps_per_epoch; ++i) {
            const MoveType type = sc.moves.sample(rng);
            const Proposal p =
                propose_move(type, region, local.events, config, sc.moves, sc.step_sizes,
                             id_base + static_cast<std::uint64_t>(births), rng);
            so_tape_rec rec{};
            rec.epoch = epoch;
            rec.color = color;
            rec.region = static_cast<int64_t>(region_index);
            rec.slot = static_cast<int64_t>(slot);
            rec.step = i;
            rec.type = static_cast<int64_t>(p.type);
            rec.is_null = p.null;
            rec.n_removed = static_cast<int64_t>(p.change.removed.size());
            rec.n_added = static_cast<int64_t>(p.change.added.size());
            for (std::size_t r = 0; r < p.change.removed.size(); ++r)
              rec.removed_id[r] = p.change.removed[r].id;
            for (std::size_t a = 0; a < p.change.added.size(); ++a) {
              rec.added_id[a] = p.change.added[a].id;
              rec.added_x[a] = p.change.added[a].x;
              rec.added_t[a] = p.change.added[a].t;
              if (want_tape) {
                if (a == 0) rec.added_arr_off = static_cast<int64_t>(run->tarr.size());
                run->tarr.insert(run->tarr.end(), p.change.added[a].arrivals.begin(),
                                 p.change.added[a].arrivals.end());
              }
            }
            rec.logq_f = p.log_q_forward;
            rec.logq_r = p.log_q_reverse;
            rec.delta = kLogZero;
            // mh_step (proposals.hpp:265-293)
            bool acc = false;
            if (!p.null) {
              bool constrained_out = false;
              for (const Event& e : p.change.added)
                if (!region.contains(e.t)) {
                  constrained_out = true;
                  break;
                }
              double log_r;
              if (constrained_out) {
                log_r = kLogZero;
              } else {
                rec.delta = delta_log_joint(local, p.change, opts);
                log_r = log_accept_ratio(rec.delta, p);
              }
              rec.constrained_out = constrained_out;
              rec.scored = !constrained_out;
              rec.log_r = log_r;
              if (log_r >= 0.0) {
                acc = true;
              } else {
                const double u = rng.uniform();
                rec.u_drawn = 1;
                rec.u = u;
                acc = std::log(u) < log_r;
              }
              if (acc) apply_change(local, p.change);
            }
            rec.accepted = acc;
            if (acc) {
              ++run->total_accepted;
              if (p.type == MoveType::Birth) ++births;
            }
            if (want_tape) run->tape.push_back(rec);
          }
          for (const Event& e : local.events)
            if (region.contains(e.t)) results[slot].push_back(e);
        }
        std::vector<Event> merged;
        for (const Event& e : global.events) {
          const std::size_t r = partition.region_of(e.t);
          if (partition.colors[r] != color) merged.push_back(e);
        }
        for (auto& res : results) merged.insert(merged.end(), res.begin(), res.end());
        detail::sort_by_id(merged);
        global.events = std::move(merged);
        next_base += static_cast<std::uint64_t>(color_regions.size()) *
                     static_cast<std::uint64_t>(sc.steps_per_epoch);
        executed += static_cast<std::int64_t>(color_regions.size()) * sc.steps_per_epoch;
        record(false);
      }
      if (s->dynamic && epoch + 1 < sc.epochs) {
        Rng offset_rng = derive_stream(sc.seed, streams::kPartitionOffset,
                                       static_cast<std::uint64_t>(epoch) + 1);
        const double u = offset_rng.uniform(0.0, l);
        partition = color_partition(build_partition(config.T, l, u), tau);
      }
    }
    if (last_recorded != executed) record(true);
    run->total_steps = executed;
    run->final = global.events;
  });
  return run;
}


// Tape-recording naive driver composed from reference functions: the control
// flow of run_naive_parallel (samplers.hpp:321-394) with run_region_steps and
// mh_step unrolled as in sr_run_chromatic.
sr_run* sr_run_naive(const so_model* mm, const double* signals, const so_sampler* s,
                     int64_t want_tape, int64_t want_rowlj) {
  auto* run = new sr_run;
  run->status = guarded([&] {
    if (s->rng_mode != 0) throw std::invalid_argument("reference supports rng_mode 0 only");
    const ModelConfig config = to_config(mm);
    SamplerConfig sc = to_sampler(s);
    sc.algorithm = Algorithm::NaiveParallel;
    config.validate();
    sc.validate();
    const std::size_t S = config.n_stations();
    run->S = S;
    const ObservedSignals sig = to_signals(config, signals);
    const double tau = config.x_max / config.v;
    const Partition partition = build_partition(config.T, config.T / sc.n_regions, 0.0);
    const std::size_t n_regions = partition.n_regions();
    const std::int64_t spr = sc.epochs * sc.steps_per_epoch;
    std::vector<std::vector<std::vector<Event>>> cps(n_regions);
    std::vector<std::int64_t> cp_steps{0};
    for (std::size_t m = 0; m < n_regions; ++m) {
      World local{config, {}, sig};
      const TimeRegion region = partition.region(m);
      ScoreOptions opts;
      opts.window = signal_window(partition.regions[m], tau, config.T, config.sample_rate);
      opts.prior_support = region;
      Rng rng = derive_stream(sc.seed, streams::kChain, 0, 0, m);
      std::uint64_t id_base = (static_cast<std::uint64_t>(m) + 1) << 32;
      cps[m].push_back(local.events);
      std::int64_t done = 0;
      while (done < spr) {
        const std::int64_t chunk = std::min(sc.record_every, spr - done);
        std::int64_t births = 0;
        for (std::int64_t i = 0; i < chunk; ++i) {
          const MoveType type = sc.moves.sample(rng);
          const Proposal p = propose_move(type, region, local.events, config, sc.moves,
                                          sc.step_sizes,
                                          id_base + static_cast<std::uint64_t>(births), rng);
          so_tape_rec rec{};
          rec.region = static_cast<int64_t>(m);
          rec.slot = static_cast<int64_t>(m);
          rec.step = done + i;
          rec.type = static_cast<int64_t>(p.type);
          rec.is_null = p.null;
          rec.n_removed = static_cast<int64_t>(p.change.removed.size());
          rec.n_added = static_cast<int64_t>(p.change.added.size());
          for (std::size_t r = 0; r < p.change.removed.size(); ++r)
            rec.removed_id[r] = p.change.removed[r].id;
          for (std::size_t a = 0; a < p.change.added.size(); ++a) {
            rec.added_id[a] = p.change.added[a].id;
            rec.added_x[a] = p.change.added[a].x;
            rec.added_t[a] = p.change.added[a].t;
            if (want_tape) {
              if (a == 0) rec.added_arr_off = static_cast<int64_t>(run->tarr.size());
              run->tarr.insert(run->tarr.end(), p.change.added[a].arrivals.begin(),
                               p.change.added[a].arrivals.end());
            }
          }
          rec.logq_f = p.log_q_forward;
          rec.logq_r = p.log_q_reverse;
          rec.delta = kLogZero;
          bool acc = false;
          if (!p.null) {
            bool constrained_out = false;
            for (const Event& e : p.change.added)
              if (!region.contains(e.t)) {
                constrained_out = true;
                break;
              }
            double log_r;
            if (constrained_out) {
              log_r = kLogZero;
            } else {
              rec.delta = delta_log_joint(local, p.change, opts);
              log_r = log_accept_ratio(rec.delta, p);
            }
            rec.constrained_out = constrained_out;
            rec.scored = !constrained_out;
            rec.log_r = log_r;
            if (log_r >= 0.0) {
              acc = true;
            } else {
              const double u = rng.uniform();
              rec.u_drawn = 1;
              rec.u = u;
              acc = std::log(u) < log_r;
            }
            if (acc) apply_change(local, p.change);
          }
          rec.accepted = acc;
          if (acc) {
            ++run->total_accepted;
            if (p.type == MoveType::Birth) ++births;
          }
          if (want_tape) run->tape.push_back(rec);
        }
        id_base += static_cast<std::uint64_t>(births);
        done += chunk;
        cps[m].push_back(local.events);
        if (m == 0) cp_steps.push_back(done);
      }
    }
    World scratch{config, {}, sig};
    for (std::size_t c = 0; c < cp_steps.size(); ++c) {
      std::vector<Event> merged;
      for (std::size_t m = 0; m < n_regions; ++m)
        merged.insert(merged.end(), cps[m][c].begin(), cps[m][c].end());
      detail::sort_by_id(merged);
      scratch.events = merged;
      run->row_step.push_back(cp_steps[c] * static_cast<std::int64_t>(n_regions));
      run->row_lj.push_back(want_rowlj ? log_joint(scratch) : 0.0);
      run->row_count.push_back(static_cast<int64_t>(merged.size()));
      if (c + 1 == cp_steps.size()) run->final = merged;
    }
    run->total_steps = spr * static_cast<std::int64_t>(n_regions);
  });
  return run;
}

// run_serial (samplers.hpp:282-315) with every step taped (mh_step without a
// constraint, proposals.hpp:265-293).
sr_run* sr_run_serial(const so_model* mm, const double* signals, const so_sampler* s,
                      int64_t n_init, const uint64_t* ids, const double* x, const double* t,
                      const double* arr, int64_t want_tape, int64_t want_rowlj) {
  auto* run = new sr_run;
  run->status = guarded([&] {
    if (s->rng_mode != 0) throw std::invalid_argument("reference supports rng_mode 0 only");
    const ModelConfig config = to_config(mm);
    SamplerConfig sc = to_sampler(s);
    sc.algorithm = Algorithm::Serial;
    config.validate();
    sc.validate();
    run->S = config.n_stations();
    const ObservedSignals sig = to_signals(config, signals);
    // the reference starts empty (samplers.hpp:291); an initial hypothesis
    // (the engine's resident one) starts in id order, births numbered above it
    World world{config, to_events(run->S, n_init, ids, x, t, arr), sig};
    detail::sort_by_id(world.events);
    const TimeRegion region = config.full_region();
    const ScoreOptions opts = default_score_options(config);
    const std::int64_t total = sc.epochs * sc.steps_per_epoch;
    Rng rng = derive_stream(sc.seed, streams::kChain, 0, 0, 0);
    run->row_step.push_back(0);
    run->row_lj.push_back(want_rowlj ? log_joint(world) : 0.0);
    run->row_count.push_back(static_cast<int64_t>(world.events.size()));
    std::uint64_t id_base = 0;
    for (const Event& e : world.events) id_base = std::max(id_base, e.id + 1);
    std::int64_t done = 0;
    while (done < total) {
      const std::int64_t chunk = std::min(sc.record_every, total - done);
      std::int64_t births = 0;
      for (std::int64_t i = 0; i < chunk; ++i) {
        const MoveType type = sc.moves.sample(rng);
        const Proposal p = propose_move(type, region, world.events, config, sc.moves,
                                        sc.step_sizes, id_base + static_cast<std::uint64_t>(births),
                                        rng);
        so_tape_rec rec{};
        rec.step = done + i;
        rec.type = static_cast<int64_t>(p.type);
        rec.is_null = p.null;
        rec.n_removed = static_cast<int64_t>(p.change.removed.size());
        rec.n_added = static_cast<int64_t>(p.change.added.size());
        for (std::size_t r = 0; r < p.change.removed.size(); ++r)
          rec.removed_id[r] = p.change.removed[r].id;
        for (std::size_t a = 0; a < p.change.added.size(); ++a) {
          rec.added_id[a] = p.change.added[a].id;
          rec.added_x[a] = p.change.added[a].x;
          rec.added_t[a] = p.change.added[a].t;
          if (want_tape) {
            if (a == 0) rec.added_arr_off = static_cast<int64_t>(run->tarr.size());
            run->tarr.insert(run->tarr.end(), p.change.added[a].arrivals.begin(),
                             p.change.added[a].arrivals.end());
          }
        }
        rec.logq_f = p.log_q_forward;
        rec.logq_r = p.log_q_reverse;
        rec.delta = kLogZero;
        bool acc = false;
        if (!p.null) {
          rec.delta = delta_log_joint(world, p.change, opts);
          const double log_r = log_accept_ratio(rec.delta, p);
          rec.scored = 1;
          rec.log_r = log_r;
          if (log_r >= 0.0) {
            acc = true;
          } else {
            const double u = rng.uniform();
            rec.u_drawn = 1;
            rec.u = u;
            acc = std::log(u) < log_r;
          }
          if (acc) apply_change(world, p.change);
        }
        rec.accepted = acc;
        if (acc) {
          ++run->total_accepted;
          if (p.type == MoveType::Birth) ++births;
        }
        if (want_tape) run->tape.push_back(rec);
      }
      id_base += static_cast<std::uint64_t>(births);
      done += chunk;
      run->row_step.push_back(done);
      run->row_lj.push_back(want_rowlj ? log_joint(world) : 0.0);
      run->row_count.push_back(static_cast<int64_t>(world.events.size()));
    }
    run->final = world.events;
    detail::sort_by_id(run->final);
    run->total_steps = total;
  });
  return run;
}

int sr_run_status(const sr_run* r) { return r->status; }

void sr_run_counts(const sr_run* r, int64_t* n_tape, int64_t* n_tape_arr, int64_t* n_rows,
                   int64_t* n_final, int64_t* total_steps, int64_t* total_accepted) {
  *n_tape = static_cast<int64_t>(r->tape.size());
  *n_tape_arr = static_cast<int64_t>(r->tarr.size());
  *n_rows = static_cast<int64_t>(r->row_step.size());
  *n_final = static_cast<int64_t>(r->final.size());
  *total_steps = r->total_steps;
  *total_accepted = r->total_accepted;
}

void sr_run_tape(const sr_run* r, so_tape_rec* recs, double* arr) {
  std::copy(r->tape.begin(), r->tape.end(), recs);
  std::copy(r->tarr.begin(), r->tarr.end(), arr);
}

void sr_run_rows(const sr_run* r, int64_t* step, double* lj, int64_t* count) {
  for (std::size_t i = 0; i < r->row_step.size(); ++i) {
    step[i] = r->row_step[i];
    lj[i] = r->row_lj[i];
    count[i] = r->row_count[i];
  }
}

void sr_run_final(const sr_run* r, uint64_t* ids, double* x, double* t, double* arr) {
  for (std::size_t i = 0; i < r->final.size(); ++i) {
    ids[i] = r->final[i].id;
    x[i] = r->final[i].x;
    t[i] = r->final[i].t;
    std::copy(r->final[i].arrivals.begin(), r->final[i].arrivals.end(), arr + i * r->S);
  }
}

void sr_run_free(sr_run* r) { delete r; }

// The reference's own run_sampler (chromatic static/dynamic from empty), for
// checking the composed driver above and for the CPU arm of bench.py.
int sr_run_sampler(const so_model* mm, const double* signals, const so_sampler* s,
                   int64_t workers, int64_t cap, int64_t* n_final, uint64_t* ids, double* x,
                   double* t, double* arr, int64_t* total_steps, int64_t* total_accepted,
                   double* wall_seconds) {
  return guarded([&] {
    const ModelConfig config = to_config(mm);
    SamplerConfig sc = to_sampler(s);
    if (s->dynamic == 2) sc.algorithm = Algorithm::NaiveParallel;
    if (s->dynamic == 3) sc.algorithm = Algorithm::Serial;
    sc.workers = static_cast<int>(workers);
    const ObservedSignals sig = to_signals(config, signals);
    const auto t0 = std::chrono::steady_clock::now();
    const Trace tr = run_sampler(config, sig, sc);
    *wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *total_steps = tr.total_steps;
    *total_accepted = tr.total_accepted;
    // final hypothesis = last snapshot (burn_in_fraction must let it be recorded)
    if (tr.snapshots.empty()) throw std::runtime_error("no snapshot recorded");
    const auto& ev = tr.snapshots.back().events;
    *n_final = static_cast<int64_t>(ev.size());
    if (*n_final > cap) throw std::runtime_error("capacity");
    const std::size_t S = config.n_stations();
    for (std::size_t i = 0; i < ev.size(); ++i) {
      ids[i] = ev[i].id;
      x[i] = ev[i].x;
      t[i] = ev[i].t;
      std::copy(ev[i].arrivals.begin(), ev[i].arrivals.end(), arr + i * S);
    }
  });
}

// CPU baseline (SURVEY §8(d) plan 2): `threads` OS threads, each running the
// reference run_region_steps on its own copy of a truth-initialised World in
// one chromatic region, until `seconds` elapse or `max_steps` are done.
// Returns total proposals and scored proposals through out-params.
int sr_bench_region_steps(const so_model* mm, const double* signals, int64_t N,
                          const uint64_t* ids, const double* x, const double* t,
                          const double* arr, const so_sampler* s, int64_t threads,
                          double seconds, int64_t max_steps, int64_t* proposals,
                          double* wall_seconds) {
  return guarded([&] {
    const ModelConfig config = to_config(mm);
    const SamplerConfig sc = to_sampler(s);
    const std::size_t S = config.n_stations();
    const ObservedSignals sig = to_signals(config, signals);
    const std::vector<Event> truth = to_events(S, N, ids, x, t, arr);
    const double tau = config.x_max / config.v;
    const double l = config.T / sc.n_regions;
    const Partition partition = color_partition(build_partition(config.T, l, 0.0), tau);
    const ScoreOptions opts = default_score_options(config);
    std::atomic<int64_t> total{0};
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    std::vector<std::thread> pool;
    for (int64_t th = 0; th < threads; ++th) {
      pool.emplace_back([&, th] {
        World local{config, truth, sig};
        const std::size_t region_index =
            static_cast<std::size_t>(th * 2) % partition.n_regions();
        const TimeRegion region = partition.region(region_index);
        Rng rng = derive_stream(sc.seed, streams::kChain, 0, 0, region_index);
        std::int64_t done = 0;
        std::uint64_t id_base = (static_cast<uint64_t>(th) + 1) << 40;
        while (done < max_steps && elapsed() < seconds) {
          const RegionStepResult r =
              run_region_steps(local, region, true, opts, sc.moves, sc.step_sizes, 1, id_base, rng);
          id_base += static_cast<std::uint64_t>(r.births);
          ++done;
        }
        total += done;
      });
    }
    for (auto& p : pool) p.join();
    *wall_seconds = elapsed();
    *proposals = total.load();
  });
}

int sr_match_events(int64_t nt, const uint64_t* tid, const double* tx, const double* tt,
                    int64_t ni, const uint64_t* iid, const double* ix, const double* it,
                    double threshold, double* out) {
  return guarded([&] {
    std::vector<EventPoint> a, b;
    for (int64_t i = 0; i < nt; ++i) a.push_back({tid[i], tx[i], tt[i]});
    for (int64_t i = 0; i < ni; ++i) b.push_back({iid[i], ix[i], it[i]});
    const MatchReport r = match_events(a, b, threshold);
    out[0] = r.precision;
    out[1] = r.recall;
    out[2] = r.location_error;
    out[3] = static_cast<double>(r.n_matched);
  });
}

int sr_bootstrap_ci(const double* values, int64_t n, double level, int32_t resamples,
                    uint64_t seed, double* out) {
  return guarded([&] {
    const std::vector<double> v(values, values + n);
    const BootstrapCI ci = bootstrap_ci(v, level, resamples, seed);
    out[0] = ci.mean;
    out[1] = ci.lo;
    out[2] = ci.hi;
    out[3] = ci.level;
  });
}

}  // extern "C"
