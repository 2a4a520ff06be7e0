// evaluation.cpp — the evaluation bridge of the reference (arXiv 1612.00595
// reference, proj/include/seismic/evaluation.hpp:51-171): greedy event matching
// (precision / recall / mean location error) and the percentile bootstrap of
// the mean, over the engine's snapshots or final hypothesis. Host C++, not on
// the hot path; results are bit-exact with the reference (same sort keys, same
// fp64 expressions without contraction, same xoshiro256++ stream).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/seis_b200.h"

namespace {

thread_local std::string g_eerr;

int fail(int code, const char* m) {
  g_eerr = m;
  return code;
}

// splitmix64 / xoshiro256++ / derive_stream (rng.hpp:21-121)
struct Xoshiro {
  uint64_t s[4];
  static uint64_t mix(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  static Xoshiro derive(uint64_t seed, uint64_t purpose) {
    uint64_t key = seed;
    uint64_t k = mix(key);
    for (uint64_t w0 : {purpose, uint64_t{0}, uint64_t{0}, uint64_t{0}}) {
      uint64_t w = w0;
      k ^= mix(w);
      k = mix(k);
    }
    Xoshiro r;
    for (auto& w : r.s) w = mix(k);
    if ((r.s[0] | r.s[1] | r.s[2] | r.s[3]) == 0) r.s[0] = 1;
    return r;
  }
  uint64_t next() {
    const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  uint64_t index(uint64_t n) {  // uniform_index, rng.hpp:54-57
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
};

struct Point {
  uint64_t id;
  double x, t;
};

bool by_tx(const Point& a, const Point& b) {  // evaluation.hpp:55-59
  if (a.t != b.t) return a.t < b.t;
  if (a.x != b.x) return a.x < b.x;
  return a.id < b.id;
}

}  // namespace

extern "C" {

const char* seis_eval_last_error(void) { return g_eerr.c_str(); }

// match_events (evaluation.hpp:51-105): true events in (t, x) order each take
// the nearest untaken inferred event (Euclidean in (x, t), first in (t, x)
// order on ties); the pair counts when |dt| and |dx| are both below the
// threshold.
int seis_match_events(int64_t n_true, const uint64_t* true_id, const double* true_x,
                      const double* true_t, int64_t n_inf, const uint64_t* inf_id,
                      const double* inf_x, const double* inf_t, double threshold,
                      seis_match_report* report, uint64_t* pair_true_id,
                      uint64_t* pair_inf_id, double* pair_dist) {
  if (!(threshold > 0)) return fail(SEIS_EINVAL, "match_events: threshold must be > 0");
  if (n_true < 0 || n_inf < 0 || !report) return fail(SEIS_EINVAL, "match_events: bad arguments");
  std::vector<Point> tr(n_true), in(n_inf);
  for (int64_t i = 0; i < n_true; ++i) tr[i] = {true_id[i], true_x[i], true_t[i]};
  for (int64_t i = 0; i < n_inf; ++i) in[i] = {inf_id[i], inf_x[i], inf_t[i]};
  std::sort(tr.begin(), tr.end(), by_tx);
  std::sort(in.begin(), in.end(), by_tx);
  std::vector<char> taken(in.size(), 0);
  int64_t matched = 0;
  double sum = 0.0;
  for (const Point& p : tr) {
    size_t best = in.size();
    double best_dist = 0.0;
    for (size_t i = 0; i < in.size(); ++i) {
      if (taken[i]) continue;
      const double dx = p.x - in[i].x;
      const double dt = p.t - in[i].t;
      const double dist = std::sqrt(dx * dx + dt * dt);
      if (best == in.size() || dist < best_dist) {
        best = i;
        best_dist = dist;
      }
    }
    if (best == in.size()) continue;
    if (std::abs(p.t - in[best].t) < threshold && std::abs(p.x - in[best].x) < threshold) {
      taken[best] = 1;
      if (pair_true_id) pair_true_id[matched] = p.id;
      if (pair_inf_id) pair_inf_id[matched] = in[best].id;
      if (pair_dist) pair_dist[matched] = best_dist;
      sum += best_dist;
      ++matched;
    }
  }
  report->n_true = n_true;
  report->n_inferred = n_inf;
  report->n_matched = matched;
  report->precision = n_inf == 0 ? 1.0 : static_cast<double>(matched) / static_cast<double>(n_inf);
  report->recall = n_true == 0 ? 1.0 : static_cast<double>(matched) / static_cast<double>(n_true);
  report->location_error = matched ? sum / static_cast<double>(matched) : 0.0;
  return SEIS_OK;
}

// bootstrap_ci (evaluation.hpp:136-169): percentile bootstrap of the mean on
// the reference's kBootstrap stream.
int seis_bootstrap_ci(const double* values, int64_t n, double level, int32_t resamples,
                      uint64_t seed, seis_ci* out) {
  if (n <= 0) return fail(SEIS_EINVAL, "bootstrap_ci: no values");
  if (!(level > 0 && level < 1)) return fail(SEIS_EINVAL, "bootstrap_ci: level must be in (0, 1)");
  if (resamples < 1) return fail(SEIS_EINVAL, "bootstrap_ci: resamples must be >= 1");
  double mean = 0.0;
  for (int64_t i = 0; i < n; ++i) mean += values[i];
  mean /= static_cast<double>(n);
  Xoshiro rng = Xoshiro::derive(seed, 7);  // streams::kBootstrap
  std::vector<double> means(static_cast<size_t>(resamples));
  for (auto& m : means) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += values[rng.index(static_cast<uint64_t>(n))];
    m = acc / static_cast<double>(n);
  }
  std::sort(means.begin(), means.end());
  const auto quantile = [&](double q) {
    const double pos = q * static_cast<double>(means.size() - 1);
    const auto i = static_cast<size_t>(pos);
    if (i + 1 >= means.size()) return means.back();
    const double frac = pos - static_cast<double>(i);
    return means[i] * (1.0 - frac) + means[i + 1] * frac;
  };
  out->mean = mean;
  out->lo = quantile((1.0 - level) / 2.0);
  out->hi = quantile(1.0 - (1.0 - level) / 2.0);
  out->level = level;
  out->resamples = resamples;
  return SEIS_OK;
}

}  // extern "C"
