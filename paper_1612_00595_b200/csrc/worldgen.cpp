// worldgen.cpp — synthetic inputs for the engine, bit-exact with the
// reference generator (arXiv 1612.00595 reference,
// proj/include/seismic/worldgen.hpp:20-86; streams rng.hpp:21-121), so the
// engine and the CPU oracle see identical signals. Host C++ (glibc libm) on
// purpose: the signals come from fp64 log/sqrt/cos whose last bits must match
// the reference's. Stations are generated in parallel (one stream per station,
// worldgen.hpp:46).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/seis_b200.h"

namespace {

thread_local std::string g_werr;

struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& st) {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t key) {
    for (auto& w : s) w = splitmix(key);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal(double mean, double sd) {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    return mean + sd * r * std::cos(6.283185307179586476925286766559 * u2);
  }
  uint64_t poisson_small(double mean) {
    const double limit = std::exp(-mean);
    uint64_t k = 0;
    double p = 1.0;
    do {
      ++k;
      p *= uniform();
    } while (p > limit);
    return k - 1;
  }
  uint64_t poisson(double mean) {
    uint64_t total = 0;
    while (mean > 60.0) {
      total += poisson_small(60.0);
      mean -= 60.0;
    }
    return total + poisson_small(mean);
  }
  static Rng derive(uint64_t seed, uint64_t purpose, uint64_t i0 = 0, uint64_t i1 = 0,
                    uint64_t i2 = 0) {
    uint64_t key = seed;
    uint64_t k = splitmix(key);
    for (uint64_t w0 : {purpose, i0, i1, i2}) {
      uint64_t w = w0;
      k ^= splitmix(w);
      k = splitmix(k);
    }
    return Rng(k);
  }
};

struct Gen {
  const seis_model_cfg* c;
  const double* st;
  int64_t S, n;
  double mean(double x, double t, int64_t j) const { return t + std::abs(x - st[j]) / c->v; }
  void range(double a, int64_t& lo, int64_t& hi) const {  // density.hpp:29-36
    const double nn = static_cast<double>(n);
    lo = static_cast<int64_t>(std::clamp(std::ceil(a * c->sample_rate), 0.0, nn));
    hi = static_cast<int64_t>(std::clamp(std::ceil((a + c->t_s) * c->sample_rate), 0.0, nn));
  }
  void arrivals(uint64_t seed, uint64_t i, double x, double t, double* a) const {
    Rng r = Rng::derive(seed, 3, i);  // kEventArrivals, worldgen.hpp:34-38
    for (int64_t j = 0; j < S; ++j) a[j] = r.normal(mean(x, t, j), c->sigma_arrival);
  }
  // variance profile + noise, worldgen.hpp:42-51
  void signals(uint64_t seed, int64_t N, const double* arr, void* out, int dtype,
               int threads) const {
    auto work = [&](int64_t j0, int64_t j1) {
      std::vector<int32_t> cnt(static_cast<size_t>(n));
      for (int64_t j = j0; j < j1; ++j) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t e = 0; e < N; ++e) {
          int64_t lo, hi;
          range(arr[e * S + j], lo, hi);
          for (int64_t s = lo; s < hi; ++s) ++cnt[s];
        }
        Rng r = Rng::derive(seed, 4, static_cast<uint64_t>(j));
        for (int64_t s = 0; s < n; ++s) {
          const double var = c->var_noise + cnt[s] * c->var_event;
          const double y = r.normal(0.0, std::sqrt(var));
          if (dtype == SEIS_F64)
            static_cast<double*>(out)[j * n + s] = y;
          else
            static_cast<float*>(out)[j * n + s] = static_cast<float>(y);
        }
      }
    };
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, S));
    std::vector<std::thread> pool;
    for (int64_t k = 0; k < T; ++k)
      pool.emplace_back(work, S * k / T, S * (k + 1) / T);
    for (auto& th : pool) th.join();
  }
};

// Streaming variant: the coverage counts of
// worldgen.hpp:42-46 without materialising the N x S arrival matrix. Events
// are drawn in chunks of B (their per-event streams are independent,
// worldgen.hpp:34-38); each chunk's windows go into per-station difference
// arrays (+1 at lo, -1 at hi; stations split over threads, no atomics), the
// prefix sums are the reference's counts exactly (integer increments
// commute). Host memory: S (n + 1) int32 + B S fp64, independent of N.
struct StreamCounts {
  const Gen& g;
  int threads;
  std::vector<int32_t> diff;  // [S][n + 1]
  std::vector<double> buf;    // [B][S]
  int64_t B;
  StreamCounts(const Gen& g_, int threads_) : g(g_), threads(std::max(1, threads_)) {
    diff.assign(static_cast<size_t>(g.S) * (g.n + 1), 0);
    B = std::max<int64_t>(1, std::min<int64_t>(4096, ((int64_t)256 << 20) / (8 * g.S)));
    buf.resize(static_cast<size_t>(B) * g.S);
  }
  template <class F>
  void par(int64_t n, F&& f) {
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, n));
    std::vector<std::thread> pool;
    for (int64_t k = 0; k < T; ++k) pool.emplace_back([&, k] { f(n * k / T, n * (k + 1) / T); });
    for (auto& th : pool) th.join();
  }
  void add(uint64_t seed, int64_t N, const double* x, const double* t) {
    for (int64_t e0 = 0; e0 < N; e0 += B) {
      const int64_t nb = std::min(B, N - e0);
      par(nb, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i)
          g.arrivals(seed, (uint64_t)(e0 + i), x[e0 + i], t[e0 + i], buf.data() + i * g.S);
      });
      par(g.S, [&](int64_t j0, int64_t j1) {
        for (int64_t j = j0; j < j1; ++j) {
          int32_t* d = diff.data() + static_cast<size_t>(j) * (g.n + 1);
          for (int64_t i = 0; i < nb; ++i) {
            int64_t lo, hi;
            g.range(buf[i * g.S + j], lo, hi);
            if (lo < hi) {
              ++d[lo];
              --d[hi];
            }
          }
        }
      });
    }
  }
  // noise with the count-dependent variance (worldgen.hpp:46-51)
  void signals(uint64_t seed, void* out, int dtype) {
    par(g.S, [&](int64_t j0, int64_t j1) {
      for (int64_t j = j0; j < j1; ++j) {
        const int32_t* d = diff.data() + static_cast<size_t>(j) * (g.n + 1);
        Rng r = Rng::derive(seed, 4, static_cast<uint64_t>(j));
        int32_t cnt = 0;
        for (int64_t s2 = 0; s2 < g.n; ++s2) {
          cnt += d[s2];
          const double var = g.c->var_noise + cnt * g.c->var_event;
          const double y = r.normal(0.0, std::sqrt(var));
          if (dtype == SEIS_F64)
            static_cast<double*>(out)[j * g.n + s2] = y;
          else
            static_cast<float*>(out)[j * g.n + s2] = static_cast<float>(y);
        }
      }
    });
  }
};

int guard(int code, const std::string& m) {
  g_werr = m;
  return code;
}

}  // namespace

extern "C" {

const char* seis_world_last_error(void) { return g_werr.c_str(); }

// sample_world (worldgen.hpp:20-53). arrivals [cap][S] is required (the
// signals depend on them); signals [S][n] in dtype (fp32 signals are the fp64
// draws rounded once).
int seis_world_generate(const seis_model_cfg* cfg, const double* stations, int64_t S,
                        uint64_t seed, int64_t cap, int64_t* n_events, uint64_t* ids, double* x,
                        double* t, double* arrivals, void* signals, int32_t dtype,
                        int32_t threads) {
  try {
    Gen g{cfg, stations, S, static_cast<int64_t>(std::llround(cfg->sample_rate * cfg->T))};
    Rng count = Rng::derive(seed, 1);
    const uint64_t N = count.poisson(cfg->lambda_rate * cfg->T);
    *n_events = static_cast<int64_t>(N);
    if (static_cast<int64_t>(N) > cap) return guard(SEIS_ERUNTIME, "event capacity too small");
    for (uint64_t i = 0; i < N; ++i) {
      Rng cr = Rng::derive(seed, 2, i);
      ids[i] = i;
      x[i] = cr.uniform(0.0, cfg->x_max);
      t[i] = cr.uniform(0.0, cfg->T);
    }
    {
      const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, (int64_t)N));
      std::vector<std::thread> pool;
      for (int64_t k = 0; k < T; ++k)
        pool.emplace_back([&, k] {
          for (int64_t i = (int64_t)N * k / T; i < (int64_t)N * (k + 1) / T; ++i)
            g.arrivals(seed, (uint64_t)i, x[i], t[i], arrivals + i * S);
        });
      for (auto& th : pool) th.join();
    }
    g.signals(seed, (int64_t)N, arrivals, signals, dtype, threads);
    return SEIS_OK;
  } catch (const std::exception& e) {
    return guard(SEIS_ERUNTIME, e.what());
  }
}

// make_world_with_events (worldgen.hpp:57-86)
int seis_world_with_events(const seis_model_cfg* cfg, const double* stations, int64_t S,
                           int64_t N, const double* cx, const double* ct, uint64_t seed,
                           double* arrivals, void* signals, int32_t dtype, int32_t threads) {
  try {
    Gen g{cfg, stations, S, static_cast<int64_t>(std::llround(cfg->sample_rate * cfg->T))};
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, std::max<int64_t>(N, 1)));
    std::vector<std::thread> pool;
    for (int64_t k = 0; k < T; ++k)
      pool.emplace_back([&, k] {
        for (int64_t i = N * k / T; i < N * (k + 1) / T; ++i)
          g.arrivals(seed, (uint64_t)i, cx[i], ct[i], arrivals + i * S);
      });
    for (auto& th : pool) th.join();
    g.signals(seed, N, arrivals, signals, dtype, threads);
    return SEIS_OK;
  } catch (const std::exception& e) {
    return guard(SEIS_ERUNTIME, e.what());
  }
}

// sample_world (worldgen.hpp:20-53) without the N x S arrival matrix: the
// events (ids, x, t) and the signals, bit-exact with seis_world_generate;
// arrivals are regenerated on demand with seis_world_arrivals.
int seis_world_generate_events(const seis_model_cfg* cfg, const double* stations, int64_t S,
                               uint64_t seed, int64_t cap, int64_t* n_events, uint64_t* ids,
                               double* x, double* t, void* signals, int32_t dtype,
                               int32_t threads) {
  try {
    Gen g{cfg, stations, S, static_cast<int64_t>(std::llround(cfg->sample_rate * cfg->T))};
    Rng count = Rng::derive(seed, 1);
    const uint64_t N = count.poisson(cfg->lambda_rate * cfg->T);
    *n_events = static_cast<int64_t>(N);
    if (static_cast<int64_t>(N) > cap) return guard(SEIS_ERUNTIME, "event capacity too small");
    for (uint64_t i = 0; i < N; ++i) {
      Rng cr = Rng::derive(seed, 2, i);
      ids[i] = i;
      x[i] = cr.uniform(0.0, cfg->x_max);
      t[i] = cr.uniform(0.0, cfg->T);
    }
    StreamCounts sc(g, threads);
    sc.add(seed, (int64_t)N, x, t);
    sc.signals(seed, signals, dtype);
    return SEIS_OK;
  } catch (const std::exception& e) {
    return guard(SEIS_ERUNTIME, e.what());
  }
}

// make_world_with_events (worldgen.hpp:57-86) without the arrival matrix.
int seis_world_with_events_signals(const seis_model_cfg* cfg, const double* stations, int64_t S,
                                   int64_t N, const double* cx, const double* ct, uint64_t seed,
                                   void* signals, int32_t dtype, int32_t threads) {
  try {
    Gen g{cfg, stations, S, static_cast<int64_t>(std::llround(cfg->sample_rate * cfg->T))};
    StreamCounts sc(g, threads);
    sc.add(seed, N, cx, ct);
    sc.signals(seed, signals, dtype);
    return SEIS_OK;
  } catch (const std::exception& e) {
    return guard(SEIS_ERUNTIME, e.what());
  }
}

// Arrivals of events i0 .. i0 + n - 1 of a world (their per-event streams,
// worldgen.hpp:34-38): rows [n][S]; x, t hold those n events' coordinates.
int seis_world_arrivals(const seis_model_cfg* cfg, const double* stations, int64_t S,
                        uint64_t seed, int64_t i0, int64_t n, const double* x, const double* t,
                        double* arrivals, int32_t threads) {
  try {
    Gen g{cfg, stations, S, static_cast<int64_t>(std::llround(cfg->sample_rate * cfg->T))};
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(threads, std::max<int64_t>(n, 1)));
    std::vector<std::thread> pool;
    for (int64_t k = 0; k < T; ++k)
      pool.emplace_back([&, k] {
        for (int64_t i = n * k / T; i < n * (k + 1) / T; ++i)
          g.arrivals(seed, (uint64_t)(i0 + i), x[i], t[i], arrivals + i * S);
      });
    for (auto& th : pool) th.join();
    return SEIS_OK;
  } catch (const std::exception& e) {
    return guard(SEIS_ERUNTIME, e.what());
  }
}

// Thomas cluster process for config[4] (BASELINE.json): parents ~ Poisson,
// uniform on [0, x_max] x [0, T); children ~ Poisson(child_mean) around each
// parent with N(0, sx^2) / N(0, st^2) offsets; out-of-range children are
// rejected. Streams use purpose ids 100-102 (outside the reference's 1..7).
int seis_thomas_events(uint64_t seed, double x_max, double T, double parent_mean,
                       double child_mean, double sx, double st, int64_t cap, int64_t* n,
                       double* cx, double* ct) {
  Rng pc = Rng::derive(seed, 100);
  const uint64_t np = pc.poisson(parent_mean);
  int64_t k = 0;
  for (uint64_t p = 0; p < np; ++p) {
    Rng pr = Rng::derive(seed, 101, p);
    const double px = pr.uniform(0.0, x_max), pt = pr.uniform(0.0, T);
    Rng ch = Rng::derive(seed, 102, p);
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
  return k > cap ? guard(SEIS_ERUNTIME, "capacity") : SEIS_OK;
}

}  // extern "C"
