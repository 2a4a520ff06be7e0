// seis_b200.hpp — the binding a reference maintainer adds: the reference's own
// run_sampler seam (proj/include/seismic/samplers.hpp:500-509) forwarded to
// the B200 engine's C-ABI (include/seis_b200.h).
//
// Header-only C++20 next to the reference headers: it keeps the reference's
// types (ModelConfig, ObservedSignals, SamplerConfig, Trace with rows,
// snapshots and phases) and error behaviour (std::invalid_argument where the
// reference throws it, CLI exit 2; std::runtime_error otherwise, exit 3), so a
// caller switches with one line:
//
//     seismic::run_sampler(config, signals, sc)  ->  seismic::b200::run_sampler(...)
//
// (proj/tools/seismic_mcmc.cpp:82, proj/include/seismic/experiment.hpp:180).
// Build: -I<reference>/proj/include -I<repo>/include, link
// <repo>/paper_1612_00595_b200/_lib/libseis_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "seis_b200.h"
#include "seismic/samplers.hpp"

namespace seismic::b200 {

inline void check(int rc) {
  if (rc == SEIS_OK) return;
  if (rc == SEIS_EINVAL) throw std::invalid_argument(seis_last_error());
  throw std::runtime_error(seis_last_error());
}

// Owns one engine (device buffers, stream); not copyable.
class Engine {
 public:
  Engine(const ModelConfig& c, const ObservedSignals& sig, std::int64_t event_capacity = 1 << 16)
      : S_(c.n_stations()) {
    const std::size_t n = static_cast<std::size_t>(c.n_samples());
    if (sig.station.size() != S_)
      throw std::invalid_argument("ObservedSignals: one trace per station required");
    std::vector<double> flat(S_ * n);
    for (std::size_t j = 0; j < S_; ++j) {
      if (sig.station[j].size() != n)
        throw std::invalid_argument("ObservedSignals: trace length != n_samples");
      std::copy(sig.station[j].begin(), sig.station[j].end(), flat.begin() + j * n);
    }
    const seis_model_cfg mc{c.lambda_rate, c.T,         c.x_max,     c.v,          c.sigma_arrival,
                            c.t_s,         c.var_noise, c.var_event, c.sample_rate};
    check(seis_engine_create(&mc, c.stations.data(), static_cast<std::int64_t>(S_), flat.data(),
                             SEIS_F64, event_capacity, &eng_));
  }
  ~Engine() { seis_engine_destroy(eng_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // The drivers (samplers.hpp:282-498) from the engine's resident hypothesis
  // (empty after construction, as the reference starts, samplers.hpp:409).
  Trace run(const SamplerConfig& sc, std::int64_t snapshot_events = 1 << 20) {
    sc.validate();
    const auto fn = sc.algorithm == Algorithm::Serial          ? seis_run_serial
                    : sc.algorithm == Algorithm::NaiveParallel ? seis_run_naive
                                                               : seis_run_chromatic;
    const seis_sampler_cfg s{sc.steps_per_epoch,
                             sc.epochs,
                             sc.n_regions,
                             sc.seed,
                             sc.burn_in_fraction,
                             sc.record_every,
                             {sc.moves.weights[0], sc.moves.weights[1], sc.moves.weights[2],
                              sc.moves.weights[3], sc.moves.weights[4]},
                             sc.step_sizes.location_x,
                             sc.step_sizes.location_t,
                             sc.step_sizes.arrival,
                             sc.step_sizes.joint,
                             sc.algorithm == Algorithm::ChromaticDynamic ? 1 : 0,
                             /*record_log_joint=*/1};
    // rows: the initial one, one per record_every executed steps (checked at
    // phase ends), the final one
    const std::int64_t per_phase = sc.steps_per_epoch * std::max(1, sc.n_regions);
    const std::int64_t total = sc.epochs * per_phase;
    const std::int64_t cap = total / sc.record_every + 2 * sc.epochs * (sc.n_regions + 3) + 8;
    check(seis_set_snapshot_capacity(eng_, snapshot_events, cap));
    std::vector<std::int64_t> step(cap), count(cap);
    std::vector<double> lj(cap);
    seis_run_stats st{};
    check(fn(eng_, &s, 0, nullptr, 0, nullptr, 0, nullptr, cap, step.data(), lj.data(),
             count.data(), &st));
    Trace tr;
    const std::int64_t nr = std::min(cap, st.n_rows);
    std::vector<double> wall(std::max<std::int64_t>(nr, 1));
    std::int64_t nw = 0;
    check(seis_get_row_wall(eng_, nr, &nw, wall.data()));
    for (std::int64_t i = 0; i < nr; ++i)
      tr.rows.push_back({i < nw ? wall[i] : 0.0, step[i], lj[i], count[i]});
    // snapshots: id, x, t of every record point past burn-in (arrivals are
    // not kept per snapshot on the device; the last snapshot is the final
    // hypothesis, read with its arrivals)
    std::int64_t ns = 0;
    check(seis_get_snapshots(eng_, 0, &ns, nullptr, nullptr, 0, nullptr, nullptr, nullptr));
    if (ns > 0) {
      std::vector<std::int64_t> sstep(ns), scount(ns);
      std::int64_t total_ev = 0;
      check(seis_get_snapshots(eng_, ns, &ns, sstep.data(), scount.data(), 0, nullptr, nullptr,
                               nullptr));  // steps and counts only
      for (std::int64_t i = 0; i < ns; ++i) total_ev += scount[i];
      std::vector<std::uint64_t> ids(std::max<std::int64_t>(total_ev, 1));
      std::vector<double> x(ids.size()), t(ids.size());
      check(seis_get_snapshots(eng_, ns, &ns, sstep.data(), scount.data(), total_ev, ids.data(),
                               x.data(), t.data()));
      std::int64_t off = 0;
      for (std::int64_t i = 0; i < ns; ++i) {
        Snapshot sn;
        sn.id = i;
        sn.step = sstep[i];
        for (const TraceRow& r : tr.rows)
          if (r.step == sn.step) sn.wall_seconds = r.wall_seconds;
        for (std::int64_t k = 0; k < scount[i]; ++k)
          sn.events.push_back({ids[off + k], x[off + k], t[off + k], {}});
        off += scount[i];
        tr.snapshots.push_back(std::move(sn));
      }
    }
    std::int64_t np = 0;
    check(seis_get_phases(eng_, 0, &np, nullptr));
    std::vector<seis_phase_record> ph(std::max<std::int64_t>(np, 1));
    check(seis_get_phases(eng_, np, &np, ph.data()));
    for (std::int64_t i = 0; i < np; ++i)
      tr.phases.push_back({ph[i].epoch, ph[i].color, static_cast<std::size_t>(ph[i].region),
                           ph[i].steps});
    tr.total_steps = st.total_steps;
    tr.total_accepted = st.total_accepted;
    return tr;
  }

  // The resident hypothesis with arrivals (World::events, samplers.hpp:409).
  std::vector<Event> hypothesis() const {
    std::int64_t N = 0;
    check(seis_get_hypothesis(eng_, 0, &N, nullptr, nullptr, nullptr, nullptr));
    std::vector<std::uint64_t> ids(std::max<std::int64_t>(N, 1));
    std::vector<double> x(ids.size()), t(ids.size()), a(ids.size() * S_);
    check(seis_get_hypothesis(eng_, N, &N, ids.data(), x.data(), t.data(), a.data()));
    std::vector<Event> out;
    for (std::int64_t i = 0; i < N; ++i)
      out.push_back({ids[i], x[i], t[i],
                     std::vector<double>(a.begin() + i * S_, a.begin() + (i + 1) * S_)});
    return out;
  }

 private:
  std::size_t S_;
  seis_engine* eng_ = nullptr;
};

// Drop-in for run_sampler (samplers.hpp:500-509): every algorithm on the GPU.
// config.validate() / sc.validate() failures surface as std::invalid_argument,
// device failures (no sm_100 device, capacity) as std::runtime_error.
inline Trace run_sampler(const ModelConfig& config, const ObservedSignals& signals,
                         const SamplerConfig& sc) {
  config.validate();
  sc.validate();
  Engine eng(config, signals);
  Trace tr = eng.run(sc);
  if (!tr.snapshots.empty()) {  // the final snapshot carries the arrivals
    Snapshot& last = tr.snapshots.back();
    if (last.step == tr.total_steps) last.events = eng.hypothesis();
  }
  return tr;
}

}  // namespace seismic::b200
