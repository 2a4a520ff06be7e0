// TEST INFRASTRUCTURE: compiles include/seis_b200.hpp (the binding a reference
// maintainer adds) against the unmodified reference headers and
// runs it next to the reference's own run_sampler.
//   binding_check cpu : without a GPU, validation errors surface as
//                       std::invalid_argument and engine creation as
//                       std::runtime_error (the engine has no CPU fallback)
//   binding_check gpu : seismic::b200::run_sampler for every algorithm against
//                       seismic::run_sampler on the same world: identical
//                       total_steps, trace-row steps, Trace::phases (the
//                       partition and its dynamic offsets are bit-exact) and
//                       snapshot steps; wall clocks increase; posterior
//                       precision/recall of both within reach of each other
// Built by oracle/oracle.py build_binding() into oracle/_ref/binding_check.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "seis_b200.hpp"
#include "seismic/evaluation.hpp"
#include "seismic/worldgen.hpp"

using namespace seismic;

static int fails = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                      \
    }                                                               \
  } while (0)

template <class Ex, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  ModelConfig c;
  const World w = sample_world(c, 5);
  SamplerConfig sc;
  sc.algorithm = Algorithm::ChromaticDynamic;
  sc.epochs = 6;
  sc.steps_per_epoch = 200;
  sc.n_regions = 4;
  sc.seed = 3;
  sc.record_every = 500;
  sc.burn_in_fraction = 0.5;
  ModelConfig bad = c;
  bad.var_event = 0.5;  // var_event must exceed var_noise (model.hpp:95-96)
  EXPECT(throws<std::invalid_argument>([&] { b200::run_sampler(bad, w.signals, sc); }));
  SamplerConfig bad_sc = sc;
  bad_sc.epochs = 0;
  EXPECT(throws<std::invalid_argument>([&] { b200::run_sampler(c, w.signals, bad_sc); }));
  if (!gpu) {
    EXPECT(throws<std::runtime_error>([&] { b200::run_sampler(c, w.signals, sc); }));
    std::printf("%s cpu\n", fails ? "FAILED" : "OK");
    return fails ? 1 : 0;
  }
  for (Algorithm alg : {Algorithm::ChromaticStatic, Algorithm::ChromaticDynamic,
                        Algorithm::NaiveParallel, Algorithm::Serial}) {
    SamplerConfig s = sc;
    s.algorithm = alg;
    const Trace r = run_sampler(c, w.signals, s);        // the reference, CPU
    const Trace b = b200::run_sampler(c, w.signals, s);  // the engine, GPU
    EXPECT(b.total_steps == r.total_steps);
    if (alg != Algorithm::NaiveParallel) {
      EXPECT(b.rows.size() == r.rows.size());
      for (std::size_t i = 0; i < std::min(b.rows.size(), r.rows.size()); ++i)
        EXPECT(b.rows[i].step == r.rows[i].step);
      EXPECT(b.snapshots.size() == r.snapshots.size());
      for (std::size_t i = 0; i < std::min(b.snapshots.size(), r.snapshots.size()); ++i)
        EXPECT(b.snapshots[i].step == r.snapshots[i].step);
    }
    // naive: the regions' chains run in one launch, so every checkpoint row
    // after the first carries the launch's end time
    for (std::size_t i = 1; i < b.rows.size(); ++i)
      EXPECT(alg == Algorithm::NaiveParallel ? b.rows[i].wall_seconds >= b.rows[i - 1].wall_seconds
                                             : b.rows[i].wall_seconds > b.rows[i - 1].wall_seconds);
    EXPECT(b.phases.size() == r.phases.size());
    for (std::size_t i = 0; i < std::min(b.phases.size(), r.phases.size()); ++i) {
      EXPECT(b.phases[i].epoch == r.phases[i].epoch);
      EXPECT(b.phases[i].color == r.phases[i].color);
      EXPECT(b.phases[i].region == r.phases[i].region);
      EXPECT(b.phases[i].steps == r.phases[i].steps);
    }
    EXPECT(!b.snapshots.empty());
    if (b.snapshots.empty()) continue;
    const auto& fb = b.snapshots.back().events;
    const auto& fr = r.snapshots.back().events;
    EXPECT(!fb.empty() && fb.front().arrivals.size() == c.n_stations());
    const MatchReport mb = match_events(event_points(w.events), event_points(fb), 12.0);
    const MatchReport mr = match_events(event_points(w.events), event_points(fr), 12.0);
    std::printf("%-18s steps %lld rows %zu phases %zu final %zu/%zu  precision %.3f/%.3f "
                "recall %.3f/%.3f\n",
                algorithm_name(alg).c_str(), (long long)b.total_steps, b.rows.size(),
                b.phases.size(), fb.size(), fr.size(), mb.precision, mr.precision, mb.recall,
                mr.recall);
    EXPECT(std::abs(mb.recall - mr.recall) <= 0.5);
  }
  std::printf("%s gpu\n", fails ? "FAILED" : "OK");
  return fails ? 1 : 0;
}
