// engine.cuh — device data layout and helpers of the B200 region-sweep engine.
//
// HBM layout:
//   y     [n][S_pad]   observed signals, time-major (fp32 for configs 1-4, fp64
//                      for config 0), so the ~20-sample arrival windows of a
//                      proposal at neighbouring stations fall in the same rows
//   cov   [n][S_pad/2] uint32 words packing two uint16 coverage counts
//                      (stations 2p, 2p+1): the reference's per-sample signal
//                      count, rebuilt there from all N events per proposal
//                      (density.hpp:263-278), kept resident here
//   pool  [P][S_pad]   fp64 arrival times, one slot per event version
//   table sorted-by-id event list {id, x, t, slot} (the reference's
//                      World::events after sort_by_id, samplers.hpp:481)
#pragma once

#include <cstdint>

#include "../../include/seis_b200.h"
#include "../../include/seis_philox.h"

namespace seis {

#ifndef SEIS_NT
#define SEIS_NT 512
#endif
constexpr int NT = SEIS_NT;      // threads per region CTA
#ifndef SEIS_MSPEC
#define SEIS_MSPEC 4
#endif
constexpr int MSPEC = SEIS_MSPEC;  // speculative proposals evaluated per round
// default depth at run time (<= MSPEC): at acceptance ~12 % a fourth proposal
// is discarded speculation more often than it saves a round (measured on
// configs 1 and 2: 3 beats 4 by 3-4 %, 2 and 1 lose); SEIS_SPEC overrides
constexpr int kSpecDefault = 3;
#ifndef SEIS_PROF_ITEMS
#define SEIS_PROF_ITEMS 0
#endif
constexpr bool kProfItems = SEIS_PROF_ITEMS;
#ifndef SEIS_MINB
#define SEIS_MINB 1  // k_phase CTAs per SM the register budget is cut for
#endif
constexpr int NW = NT / 32;
#ifndef SEIS_MAXOWN
#define SEIS_MAXOWN 64
#endif
constexpr int MAXOWN = SEIS_MAXOWN;  // events a region may hold during a phase (build.py passes the same)
constexpr int kMaxEvents = 1 << 22;  // event_capacity bound (table sizes; counts stay uint16)
constexpr int MAXDIFF = 2 * MAXOWN;  // diff pairs a region may hold
constexpr int MAXDOUT = 3 * MAXOWN;  // diff pairs + recycled slots per region
// run_serial's one chain holds every event of the world: its k_phase variant
// keeps up to kSerialCap events (and 2 / 3 x that in diff pairs / outputs) in
// dynamic shared memory instead of the static MAXOWN arrays
constexpr int kSerialCap = 1024;
template <int CAP>
struct ChainSmem {  // bytes of the chain arrays (own, st, pold, pnew, lfree, cur_of, log i)
  static constexpr int bytes = CAP * (32 + 24 + 4 + 4) + 2 * CAP * 8 + (CAP + 8) * 8;
};
constexpr int kRetryFree = 3 * MAXOWN;  // version slots a region chain can hand to its rerun
constexpr int kOvfRegions = 512;        // reruns per phase with outputs past MAXOWN / MAXDOUT (at least; Ovf::cap)

// Per-slot phase outputs (births alive at the end, diff entries): region
// slots at stride MAXOWN / MAXDOUT; a rerun region (whole-chain variant)
// writes to one of kOvfRegions overflow areas of kSerialCap / 3 kSerialCap
// after them, its index in slot[s] (-1: the regular area)
struct Ovf {
  int* slot;   // [n_slots] (null: no overflow areas, e.g. the serial chain)
  int* count;  // overflow areas handed out this phase (reset by the barrier)
  int cap;     // overflow areas allocated: kOvfRegions, or every region of a naive launch
};
__host__ __device__ __forceinline__ size_t births_off(const Ovf& o, int n_slots, int s) {
  const int k = o.slot ? o.slot[s] : -1;
  return k < 0 ? (size_t)s * MAXOWN : (size_t)n_slots * MAXOWN + (size_t)k * kSerialCap;
}
__host__ __device__ __forceinline__ size_t diff_off(const Ovf& o, int n_slots, int s) {
  const int k = o.slot ? o.slot[s] : -1;
  return k < 0 ? (size_t)s * MAXDOUT : (size_t)n_slots * MAXDOUT + (size_t)k * 3 * kSerialCap;
}
#ifndef SEIS_TBL
#define SEIS_TBL 512
#endif
constexpr int TBL = SEIS_TBL;    // coverage counts whose {dL, dI} rows live in smem
#ifndef SEIS_TM_TILES
#define SEIS_TM_TILES (4 * NW)
#endif
constexpr int kDiffCache = 2048;  // stations whose round diff windows k_phase caches in smem
constexpr int kTileFlags = 24576;  // station tiles whose diff flags the tile-major pass keeps
#ifndef SEIS_PAIR
#define SEIS_PAIR 1
#endif
constexpr bool kPairOn = SEIS_PAIR;  // tile pairs for births / deaths without own diff (phase.cuh)
constexpr int kRowPad = 32;      // zero rows appended to y and cov (unpredicated chunk loads)
#ifndef SEIS_LOGIWIN
#define SEIS_LOGIWIN 1024
#endif
constexpr int LOGIWIN = SEIS_LOGIWIN;  // log(i) window around the phase-start event count
constexpr int BANDMAX = 256;     // rows of the generic diff-correction scratch
constexpr double kLog2Pi = 1.8378770664093454835606594728112;

struct Win {
  int lo, hi;
};

// Signal and count layout ("station tiles"): the 32 stations of tile
// b = j >> 5 keep their rows contiguous, element (r, j) at
// ((j >> 5) * rows + r) * 32 + (j & 31) with rows = n + kRowPad. One row of a
// tile is one 128-byte line of y (fp32) / 64-byte line of counts, so a warp
// walking a station tile's rows reads coalesced lines at compile-time offsets.
// Counts are uint16; two neighbouring stations share a uint32 word (the
// commit's packed atomics): pair p = j >> 1 at ((p >> 4) * rows + r) * 16 + (p & 15).
// Compact arrival versions ("philox stream spec v2", include/seis_philox.h):
// an event version is either a stored row of the arrival pool (slot >= 0) or
// a generated version (slot = -2 - g, g indexing the GenV table): the arrival
// at station j is computed, arrival_mean(x, t, j) + sigma z_j with z_j the
// philox normal of the birth that created it, plus up to kGenOvr per-station
// overrides (accepted arrival moves). Slot -1 means "no version" (a birth's start, a death's end).
constexpr int kGenOvr = 8;  // per-station arrival overrides a generated version keeps
struct GenV {
  double x, t;                  // the version's location
  unsigned long long seed;      // the birth's philox key ...
  unsigned sweep, region, step; // ... and counter
  int n_ovr;                    // overrides, in the order the arrival moves were accepted
  int ovr_st[kGenOvr];
  double ovr_d[kGenOvr];
};
// (mean + sigma z) + the overrides at station j, in order
__device__ __forceinline__ double gen_apply_ovr(const GenV* g, int j, double a) {
  const int n = g->n_ovr;
  for (int k = 0; k < n; ++k)
    if (g->ovr_st[k] == j) a = a + g->ovr_d[k];
  return a;
}

struct Dev {
  int S, S_pad, P2, n;
  int rows;                        // n + kRowPad
  double rate, t_s, v, sigma, x_max, T;
  double c0_arr, inv_twovar_arr;   // log_gaussian constants for sigma_arrival
  double twovar_arr;               // 2 sigma^2
  double inv_v;                    // RN(1 / v): division by v as a reciprocal + one correction
  double log_lambda_T, lxa;        // log(lambda T), -log(x_max) - log(T)
  double log_xmax;
  const double* stations;          // [S_pad]
  const void* y;                   // [S_pad / 32][rows][32] (station tiles)
  uint32_t* cov;                   // [S_pad / 32][rows][16] uint16 pairs
  // per-sample term cache, same tiling as y: the likelihood change of one more
  // (tpos) / one fewer (tneg) event covering the sample at its committed count,
  // term(c, +-1) of density.hpp:286-301; rebuilt after every commit (k_terms),
  // read by the dense band of births and deaths where the region's own diff is
  // empty at the station
  const double* tpos;              // [S_pad / 32][rows][32]
  const double* tneg;
  double* pool;                    // [P][S_pad]
  GenV* gv;                        // [gv_cap] generated versions
  int* gv_free;                    // [gv_cap] free stack of GenV entries (top: Ctl::gv_top)
  const double* Lg;                // [tab_n] -0.5 (log 2pi + log var_c)
  const double* Ig;                // [tab_n] 0.5 / var_c
  const double2* Dg;               // [tab_n][4] {L[c+dc]-L[c], I[c+dc]-I[c]}, dc=-2,-1,1,2
  int tab_n;
  const double* logi;              // [logi_n] log((double) i)
  int logi_n;
  int pool_cap;
  int gv_cap;
  int dcache_on;  // proposal-major launches keep the round's diff windows in shared memory
};

struct Samp {
  int64_t k;
  uint64_t seed;
  double cumw[5];
  double logw[5];
  double step_lx, step_lt, step_arr, step_joint, joint_t_sd;
  int ncol;
  int mspec;  // speculative proposals per round, 1..MSPEC
  int first_scored;  // end every round at its first scored proposal (phase.cuh)
};

struct Table {
  unsigned long long* id;
  double* x;
  double* t;
  int* slot;
};

struct OutEv {
  unsigned long long id;
  double x, t;
  int slot, pad;
};

// One entry of a region's diff against the phase-start snapshot: the
// start version (old_slot, -1 for a birth) and the current version
// (new_slot, -1 for a death). kind 1 = slot to recycle only (a this-phase
// version that died).
struct DiffPair {
  int old_slot, new_slot, kind, pad;
};

struct Ctl {
  int n_events;
  int free_top;
  int err;
  int phase_stamp;
  int gv_top, gv_pad;  // free stack of generated-version entries
  unsigned long long scored, changed, arrvals, accepted, id_mismatch, speculative;
  unsigned long long prof[8];  // clock64 cycles per round section (thread 0 of every CTA)
  unsigned long long tprof[2][8];  // per move type: warp-cycles in items, items
};

struct PhaseArgs {
  int epoch, color, nreg, n_slots;
  const double* bnd;               // [nreg + 1]
  unsigned long long next_base;
  long long tape_base;
  Table tab;                       // phase-start table (sorted by id)
  int* fate_stamp;
  int* fate_alive;
  double* fate_x;
  double* fate_t;
  int* fate_slot;
  int* births_cnt;                 // [n_slots]
  OutEv* births;                   // [n_slots][MAXOWN]
  int* diff_cnt;                   // [n_slots]
  DiffPair* diff;                  // [n_slots][MAXDOUT]
  int* free_stack;
  int compact;                     // births (and their moves) make generated versions
  const seis_tape_step* tape;
  const double* tape_arr;
  seis_step_out* out;
  // naive mode (run_naive_parallel, samplers.hpp:321-394): all regions in one
  // launch from the empty hypothesis; per-region prior support and window
  int naive;
  const double* reg_llam;          // log(lambda * region length)
  const double* reg_lxa;           // -log(x_max) - log(region length)
  const int* reg_wlo;              // signal_window (partition.hpp:94-102)
  const int* reg_whi;
  int record_every;                // checkpoints every record_every local steps
  int* cp_counts;                  // [n_cp][nreg] own event count at checkpoint c
  // serial mode (run_serial, samplers.hpp:282-315): one chain over [0, T]
  // without the region constraint, run in chunks of record_every steps
  int serial;
  long long step_base;             // chain step of this launch's first step
  int* births_total;               // [n_slots] accepted births of the phase (may be null)
  unsigned long long* order_io;    // serial: [0] count, [1..] ids in list order (may be null)
  // regions outgrowing the MAXOWN chain arrays: the region kernel hands the
  // slot (and every version slot its chain took, retry_free[slot][0] = count)
  // to a second launch of the whole-chain variant (kSerialCap events), which
  // reruns the chain from the phase-start state (retry_pass = 1: only
  // flagged slots run); the counter-based stream makes the rerun identical
  int* retry;
  int* retry_free;
  int retry_pass;
  Ovf ovf;
  // dispatch order: CTA b runs region slot slot_order[b] (k_order: slots with
  // more phase-start events first, so the cheap event-free chains fill the
  // last wave); null = identity
  const int* slot_order;
};

enum : int {
  ERR_NONE = 0,
  ERR_OWN_OVERFLOW = 1,
  ERR_POOL_EXHAUSTED = 2,
  ERR_TAPE_UNKNOWN_ID = 3,
  ERR_TABLE_OVERFLOW = 4,
  ERR_COUNT_OVERFLOW = 5,
  ERR_GEN_EXHAUSTED = 6,
};

// the first device error of a run wins (later ones are consequences)
__device__ __forceinline__ void set_err(Ctl* ctl, int code) { atomicCAS(&ctl->err, 0, code); }

__device__ __forceinline__ Win make_win(const Dev& d, double a) {
  // arrival_sample_range, density.hpp:29-36: ceil in fp64 (no contraction:
  // --fmad=false), clamp to [0, n]. cvt.rpi.s32.f64 rounds up and saturates
  // out-of-range values, so clamping the int equals clamping the double.
  Win w;
  w.lo = min(max(__double2int_ru(a * d.rate), 0), d.n);
  w.hi = min(max(__double2int_ru((a + d.t_s) * d.rate), 0), d.n);
  return w;
}

// element (r, j) of y / uint16 counts; uint32 count pair (r, p = j >> 1)
__host__ __device__ __forceinline__ size_t yix(int rows, int r, int j) {
  return ((size_t)(j >> 5) * rows + r) * 32 + (j & 31);
}
__host__ __device__ __forceinline__ size_t pix(int rows, int r, int p) {
  return ((size_t)(p >> 4) * rows + r) * 16 + (p & 15);
}

__device__ __forceinline__ int inw(int r, Win w) {
  return (unsigned)(r - w.lo) < (unsigned)(w.hi - w.lo) ? 1 : 0;
}

// |x - s| / v correctly rounded without a division: q0 = a * RN(1/v), the
// exact remainder r = a - q0 v (one FMA), q = RN(q0 + r * RN(1/v)). With the
// correctly rounded reciprocal this final step yields the correctly rounded
// quotient (Markstein's theorem), i.e. the reference's IEEE division bit for
// bit; tests/test_oracle.py checks it against the host division on 10^7
// random operands per configuration.
__device__ __forceinline__ double div_v(const Dev& d, double a) {
  const double q0 = a * d.inv_v;
  return fma(fma(-q0, d.v, a), d.inv_v, q0);
}

__device__ __forceinline__ double arrival_mean(const Dev& d, double x, double t, double s) {
  return t + div_v(d, fabs(x - s));  // model.hpp:73-75
}

// generated version's arrival at station j (spec v2): (mean + sigma z) [+ override]
__device__ __forceinline__ double gen_arrival(const Dev& d, const GenV* g, int j, double mean) {
  double a =
      mean + d.sigma * (double)seis_normal(g->seed, g->sweep, g->region, g->step, (uint32_t)j);
  return gen_apply_ovr(g, j, a);
}
__device__ __forceinline__ const GenV* gv_of(const Dev& d, int slot) { return d.gv + (-2 - slot); }
// any version's arrival at station j (slot != -1)
__device__ __forceinline__ double arr_of(const Dev& d, int slot, int j) {
  if (slot >= 0) return __ldg(d.pool + (size_t)slot * d.S_pad + j);
  const GenV* g = gv_of(d, slot);
  return gen_arrival(d, g, j, arrival_mean(d, g->x, g->t, d.stations[j]));
}

// GEN = false: the kernel variant of runs that hold stored rows only (the
// default arrival storage): the plain pool load, as before spec v2
template <bool GEN>
__device__ __forceinline__ double ver_arr(const Dev& d, int slot, int j) {
  if constexpr (GEN) return arr_of(d, slot, j);
  return __ldg(d.pool + (size_t)slot * d.S_pad + j);
}

__device__ __forceinline__ double arr_logpdf(const Dev& d, double a, double mean) {
  // log_gaussian(a, mean, sigma^2), density.hpp:15-18 with host-computed
  // -0.5 (log 2pi + log sigma^2); the division d^2 / (2 sigma^2) is the
  // correctly rounded quotient by the reciprocal + one FMA correction, as in
  // div_v (bit-identical to the reference's division for every sigma_arrival;
  // exact in the first step already when 2 sigma^2 is a power of two)
  const double dd = a - mean;
  const double n2 = dd * dd;
  const double q0 = n2 * d.inv_twovar_arr;
  return d.c0_arr - fma(fma(-q0, d.twovar_arr, n2), d.inv_twovar_arr, q0);
}

}  // namespace seis
