// kernels.cuh — scoring core of the B200 region-sweep engine.
//
// Hot path (one launch per color phase): k_phase, one CTA per same-color
// region, runs that region's k MH steps against the phase-start snapshot
// (frozen-snapshot semantics of run_chromatic, samplers.hpp:445-463) and
// scores every proposal with the fused likelihood delta (density.hpp:214-305)
// over the resident coverage counts. A round evaluates up to M consecutive
// proposals of the chain against the same state and commits up to the first
// accepted one: with a counter-based stream a rejected step leaves the state
// and the next step's draws unchanged, so this is exactly the sequential
// chain. k_commit and k_rebuild are the color barrier (samplers.hpp:470-485).
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace seis {

template <typename YT>
struct Y2;
template <>
struct Y2<float> {
  using T = float2;
};
template <>
struct Y2<double> {
  using T = double2;
};

// per-item cycle counters of the profiling build (SEIS_PROF_ITEMS=1)
__shared__ unsigned long long s_tprof[2][8];

// Proposal descriptor (one per speculative slot, double-buffered by round).
struct Prop {
  int type, skip, scored, nr, na, bad;
  int rown[2], rslot[2], rsidx[2];
  double rx[2], rt[2];
  double ax[2], at[2];
  unsigned long long aid;
  int arr_st;
  double arr_da;
  long long tape_idx, tape_off;
  double logq_f, logq_r, u, logu;
  int u_drawn, tape_acc;
  int accept;
  int dslot[2], inplace[2];
  int dgen[2];  // the accepted version is a generated one (spec v2)
};

// sidx: the event's phase-start index i while its start version is current;
// -(i + 2) once a move replaced that version (the event keeps its start
// index); -1 for an event born this phase. sidx < 0 <=> a this-phase version.
struct OwnEv {
  unsigned long long id;
  double x, t;
  int slot, sidx;
};
__device__ __forceinline__ int own_src(int sidx) { return sidx >= 0 ? sidx : -sidx - 2; }

struct StartEv {
  unsigned long long id;
  int slot, tab, current, pad;
};

enum { SRC_NONE = 0, SRC_BIRTH = 1, SRC_SHIFT = 2, SRC_ROWS = 3 };

struct PassIn {
  int src;
  const double* rows[2];
  uint64_t seed;
  uint32_t sweep, region, step;
  int wlo, whi;
};

__device__ __forceinline__ Win empty_win() { return Win{0, 0}; }

__device__ __forceinline__ bool weq(Win a, Win b) { return a.lo == b.lo && a.hi == b.hi; }

__device__ __forceinline__ Win clampw(Win w, int wlo, int whi) {
  w.lo = max(w.lo, wlo);
  w.hi = min(w.hi, whi);
  if (w.hi < w.lo) w.hi = w.lo;
  return w;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-sample likelihood change for coverage c -> c + dc (density.hpp:286-301):
// (L[c+dc] - y^2 I[c+dc]) - (L[c] - y^2 I[c]) = dL - y^2 dI with the per-count
// differences precomputed on the host from glibc log (one 16-byte lookup).
__device__ __forceinline__ int dc_code(int dc) { return dc > 0 ? dc + 1 : dc + 2; }

// Shared copy of the table, code-major: entry (c, code) at code * (TBL + 1) + c,
// so the lanes of a warp (nearby counts, one code) read neighbouring 16-byte
// entries instead of entries 64 bytes apart on the same banks; kTsZero is an
// all-zero entry for masked rows. The global table Dg stays [count][code].
constexpr int kTsStride = TBL + 1;
constexpr int kTsZero = 4 * kTsStride;
constexpr int kTsSize = kTsZero + 1;
__device__ __forceinline__ int ts_idx(int c, int code) { return code * kTsStride + c; }

__device__ __forceinline__ void fill_ts(double2* Ts, const Dev& d, int tid, int nthreads) {
  for (int i = tid; i < kTsSize; i += nthreads) {
    const int code = i / kTsStride, c = i - code * kTsStride;
    Ts[i] = (code < 4 && c < TBL && c < d.tab_n) ? d.Dg[c * 4 + code] : make_double2(0, 0);
  }
}

__device__ __forceinline__ double term(const Dev& d, const double2* Ts, double y, int c, int dc) {
  const double2 e = c < TBL ? Ts[ts_idx(c, dc_code(dc))] : d.Dg[c * 4 + dc_code(dc)];
  const double y2 = y * y;
  return fma(-y2, e.y, e.x);
}

// shared-memory-only lookup; the caller guarantees c < TBL
__device__ __forceinline__ double term_fast(const double2* Ts, double y, int c, int dc) {
  const double2 e = Ts[ts_idx(c, dc_code(dc))];
  return fma(-(y * y), e.y, e.x);
}

template <int N>
struct Wins {
  Win w[N > 0 ? N : 1];
};

// Rows [blo, bhi) of one station (one lane), RU rows' loads in flight at a
// time, branch-free: dc = added - removed windows covering the row; c =
// phase-start count + own diff correction (the region's frozen view); only
// rows with dc != 0 load. Time-major layout: the warp's 32 stations of a row
// are contiguous. Counts at or above the shared table fall back to a slow
// pass over the whole item (rare: > TBL - 3 overlapping events).
template <int NR, int NA, int ND, typename YT>
__device__ __forceinline__ void band(const Dev& d, int j, int blo, int bhi, const Wins<NR>& R,
                                     const Wins<NA>& A, const Wins<ND>& D,
                                     const int (&sg)[ND > 0 ? ND : 1], const double2* Ts,
                                     double& sig, int& cnt) {
#ifndef SEIS_BANDG_RU
#define SEIS_BANDG_RU 4
#endif
  constexpr int RU = SEIS_BANDG_RU;
  constexpr int stride = 32;  // next row of the station tile
  const YT* __restrict__ y = reinterpret_cast<const YT*>(d.y) + yix(d.rows, 0, j);
  const uint16_t* __restrict__ c16 = reinterpret_cast<const uint16_t*>(d.cov) + yix(d.rows, 0, j);
  double s_loc = 0.0;
  int c_loc = 0;
  bool big = false;
  int off = blo * stride;
  for (int r0 = blo; r0 < bhi; r0 += RU, off += RU * stride) {
    int dc[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      const int r = r0 + k;  // rows past bhi lie outside every window: dc = 0
      int a = 0;
#pragma unroll
      for (int q = 0; q < NA; ++q) a += inw(r, A.w[q]);
#pragma unroll
      for (int q = 0; q < NR; ++q) a -= inw(r, R.w[q]);
      dc[k] = a;
    }
    int c[RU];
    float yv[RU];
    double yd[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      c[k] = dc[k] ? (int)__ldg(c16 + off + k * stride) : 0;
      if (sizeof(YT) == 4)
        yv[k] = dc[k] ? (float)__ldg(y + off + k * stride) : 0.0f;
      else
        yd[k] = dc[k] ? (double)__ldg(y + off + k * stride) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      int cc = c[k];
#pragma unroll
      for (int q = 0; q < ND; ++q) cc += sg[q] * inw(r0 + k, D.w[q]);
      big |= cc >= TBL - 2;
      const int ci = min(cc, TBL - 3) & (dc[k] ? 0x7fffffff : 0);
      const int dk = dc[k] ? dc[k] : 1;
      const double yy = sizeof(YT) == 4 ? (double)yv[k] : yd[k];
      const double t = term_fast(Ts, yy, ci, dk);
      s_loc += dc[k] ? t : 0.0;
      c_loc += dc[k] ? 1 : 0;
    }
  }
  if (__any_sync(0xffffffffu, big)) {
    // slow exact pass with the global table
    s_loc = 0.0;
    c_loc = 0;
    for (int r = blo; r < bhi; ++r) {
      int dcv = 0;
#pragma unroll
      for (int q = 0; q < NA; ++q) dcv += inw(r, A.w[q]);
#pragma unroll
      for (int q = 0; q < NR; ++q) dcv -= inw(r, R.w[q]);
      if (dcv) {
        const int o = r * stride;
        int cc = (int)__ldg(c16 + o);
#pragma unroll
        for (int q = 0; q < ND; ++q) cc += sg[q] * inw(r, D.w[q]);
        s_loc += term(d, Ts, (double)__ldg(y + o), cc, dcv);
        ++c_loc;
      }
    }
  }
  sig += s_loc;
  cnt += c_loc;
}

// Dense single-window moves (birth: SIGN +1, death: SIGN -1): every row of
// the lane's window changes. Each lane walks its own window down its station
// tile (rows 32 elements apart: compile-time load offsets, one 128-byte line
// per row for the warp when the lanes' windows align, as they do under the
// reference's geometry); the warp runs the longest window's trip count and
// rows past a lane's window index the zero row of the table. cnt is the
// window length (computed by the caller).
#ifndef SEIS_BAND_RU
#define SEIS_BAND_RU 20  // = t_s * rate of the reference default: a 20-row window is one unmasked batch
#endif
#ifndef SEIS_BAND_ACC
#define SEIS_BAND_ACC 1  // partial sums per lane in the dense band (more measured no faster)
#endif
static_assert(kRowPad >= SEIS_BAND_RU, "band1 reads up to RU - 1 rows past the longest window");
template <int SIGN, int ND, typename YT>
__device__ __forceinline__ void band1(const Dev& d, int j, Win W, const Wins<ND>& D,
                                      const int (&sg)[ND > 0 ? ND : 1], const double2* Ts,
                                      double& sig) {
  constexpr int RU = sizeof(YT) == 4 ? SEIS_BAND_RU : 4;
  constexpr int code = SIGN > 0 ? 2 : 1;  // dc_code(+1) / dc_code(-1)
  const int len = W.hi - W.lo;
  const int trips = (int)__reduce_max_sync(0xffffffffu, (unsigned)len);
  // the walk covers rows [base, base + ceil(trips / RU) * RU) of the tile;
  // base = W.lo unless that would run past the pad rows
  const int span = (trips + RU - 1) / RU * RU;
  const int base = min(W.lo, d.rows - span);
  const int sh = W.lo - base;
  const YT* __restrict__ yp = reinterpret_cast<const YT*>(d.y) + yix(d.rows, base, j);
  const uint16_t* __restrict__ cp =
      reinterpret_cast<const uint16_t*>(d.cov) + yix(d.rows, base, j);
  // independent partial sums: the rows' DADDs do not wait on each other
  constexpr int NACC = SEIS_BAND_ACC;
  double sa[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) sa[k] = 0.0;
  int mx = 0;
  for (int i0 = 0; i0 < trips; i0 += RU) {
    int c[RU];
    YT yv[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      c[k] = (int)__ldg(cp + k * 32);
      yv[k] = __ldg(yp + k * 32);
    }
    cp += RU * 32;
    yp += RU * 32;
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      int cc = c[k];
#pragma unroll
      for (int q = 0; q < ND; ++q) cc += sg[q] * inw(base + i0 + k, D.w[q]);
      mx = max(mx, cc);
      const bool in = (unsigned)(i0 + k - sh) < (unsigned)len;
      const int idx = in ? ts_idx(min(cc, TBL - 3), code) : kTsZero;
      const double2 e = Ts[idx];
      const double yy = (double)yv[k];
      sa[k % NACC] += fma(-(yy * yy), e.y, e.x);
    }
  }
  double s = sa[0];
#pragma unroll
  for (int k = 1; k < NACC; ++k) s += sa[k];
  if (__any_sync(0xffffffffu, mx >= TBL - 3)) {
    s = 0.0;  // slow exact pass with the global table
    const YT* y0 = reinterpret_cast<const YT*>(d.y) + yix(d.rows, 0, j);
    const uint16_t* c0 = reinterpret_cast<const uint16_t*>(d.cov) + yix(d.rows, 0, j);
    for (int r = W.lo; r < W.hi; ++r) {
      int cc = (int)__ldg(c0 + r * 32);
#pragma unroll
      for (int q = 0; q < ND; ++q) cc += sg[q] * inw(r, D.w[q]);
      s += term(d, Ts, (double)__ldg(y0 + r * 32), cc, SIGN);
    }
  }
  sig += s;
}

// The dense band where the region's own diff is empty at every station of the
// tile: the rows' terms at the committed counts were computed by k_terms
// (Dev::tpos / tneg, the same expression on the same table entries), so the
// lane sums its window's cached terms in band1's order (bit-identical sums):
// one 8-byte load and one add per row instead of two loads, a table lookup, a
// conversion and three fp64 operations.
template <int SIGN>
__device__ __forceinline__ void band1_terms(const Dev& d, int j, Win W, double& sig) {
  constexpr int RU = SEIS_BAND_RU;
  const int len = W.hi - W.lo;
  const int trips = (int)__reduce_max_sync(0xffffffffu, (unsigned)len);
  const int span = (trips + RU - 1) / RU * RU;
  const int base = min(W.lo, d.rows - span);
  const int sh = W.lo - base;
  const double* __restrict__ tp = (SIGN > 0 ? d.tpos : d.tneg) + yix(d.rows, base, j);
  double s = 0.0;
  if (trips == RU && __all_sync(0xffffffffu, len == RU && sh == 0)) {
    double v[RU];  // every lane's window is exactly one batch
#pragma unroll
    for (int k = 0; k < RU; ++k) v[k] = __ldg(tp + k * 32);
#pragma unroll
    for (int k = 0; k < RU; ++k) s += v[k];
  } else {
    for (int i0 = 0; i0 < trips; i0 += RU) {
      double v[RU];
#pragma unroll
      for (int k = 0; k < RU; ++k) v[k] = __ldg(tp + k * 32);
      tp += RU * 32;
#pragma unroll
      for (int k = 0; k < RU; ++k) s += (unsigned)(i0 + k - sh) < (unsigned)len ? v[k] : 0.0;
    }
  }
  sig += s;
}

// Two neighbouring station tiles (stations j0 .. j0 + 63, j0 a multiple of
// 64) of one production birth (BIRTH) or death, where the region's own diff
// has no window on either tile: station_item's setup (density.hpp:239-262:
// arrival of the added / removed version, its window, its log-density) and
// the cached-term band for both tiles side by side, so the two fp64 chains
// interleave and twice the rows are in flight. The 64 birth normals are the
// two normals of 32 Philox calls (draw 16 + (j >> 1), seis_philox.h): each
// lane makes one call and the lanes exchange the values by shuffle, where
// tile by tile every lane makes its own call per tile and neighbouring lanes
// repeat each other's. Per tile the values, operations and their order are
// station_item's + band1_terms': the sums are bit-identical to scoring the
// tiles one after the other. (Four tiles side by side, and a K-tile template
// of this function, measured slower: address arithmetic and spills at the
// 128-register budget.)
template <bool BIRTH>
__device__ __forceinline__ void dense_pair_terms(const Dev& d, const Prop& P, const PassIn& in,
                                                 int j0, double& sigA, double& sigB,
                                                 double& arrA, double& arrB, int& cnt) {
#ifndef SEIS_PAIR_H
#define SEIS_PAIR_H SEIS_BAND_RU  // rows per tile and batch: both windows' 40 rows in flight at once
                                  // (10 rows per tile and batch: -2.6 %, 5: the same)
#endif
  constexpr int H = SEIS_PAIR_H;
  constexpr int NB = SEIS_BAND_RU / H;
  static_assert(NB * H == SEIS_BAND_RU, "batches cover the window");
  const int lane = threadIdx.x & 31;
  const int jA = j0 + lane, jB = jA + 32;
  const bool vA = jA < d.S, vB = jB < d.S;
  const double sA = vA ? d.stations[jA] : 0.0, sB = vB ? d.stations[jB] : 0.0;
  const double ex = BIRTH ? P.ax[0] : P.rx[0], et = BIRTH ? P.at[0] : P.rt[0];
  const double mA = arrival_mean(d, ex, et, sA), mB = arrival_mean(d, ex, et, sB);
  double aA, aB;
  if (BIRTH) {
    // this lane's call: the normals of stations j0 + 2 lane and j0 + 2 lane + 1
    float z0, z1;
    seis_normal_pair(in.seed, in.sweep, in.region, in.step, (uint32_t)((j0 >> 1) + lane), &z0,
                     &z1);
    const int h = lane >> 1;
    const float a0 = __shfl_sync(0xffffffffu, z0, h), a1 = __shfl_sync(0xffffffffu, z1, h);
    const float b0 = __shfl_sync(0xffffffffu, z0, 16 + h),
                b1 = __shfl_sync(0xffffffffu, z1, 16 + h);
    aA = mA + d.sigma * (double)((lane & 1) ? a1 : a0);
    aB = mB + d.sigma * (double)((lane & 1) ? b1 : b0);
  } else {
    const double* row = d.pool + (size_t)P.rslot[0] * d.S_pad;
    aA = __ldg(row + jA);
    aB = __ldg(row + jB);
  }
  const Win WA = vA ? clampw(make_win(d, aA), in.wlo, in.whi) : empty_win();
  const Win WB = vB ? clampw(make_win(d, aB), in.wlo, in.whi) : empty_win();
  const double lA = vA ? arr_logpdf(d, aA, mA) : 0.0, lB = vB ? arr_logpdf(d, aB, mB) : 0.0;
  arrA = BIRTH ? lA : 0.0 - lA;
  arrB = BIRTH ? lB : 0.0 - lB;
  const int lenA = WA.hi - WA.lo, lenB = WB.hi - WB.lo;
  cnt += lenA + lenB;
  if (__all_sync(0xffffffffu, lenA == NB * H && lenB == NB * H)) {
    const double* __restrict__ tA = (BIRTH ? d.tpos : d.tneg) + yix(d.rows, WA.lo, jA);
    const double* __restrict__ tB = (BIRTH ? d.tpos : d.tneg) + yix(d.rows, WB.lo, jB);
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int h = 0; h < NB; ++h) {
      double v[2 * H];
#pragma unroll
      for (int k = 0; k < H; ++k) {
        v[k] = __ldg(tA + (h * H + k) * 32);
        v[H + k] = __ldg(tB + (h * H + k) * 32);
      }
#pragma unroll
      for (int k = 0; k < H; ++k) {
        a += v[k];
        b += v[H + k];
      }
    }
    sigA = a;
    sigB = b;
  } else {
    double a = 0.0, b = 0.0;
    band1_terms<BIRTH ? 1 : -1>(d, jA, WA, a);
    band1_terms<BIRTH ? 1 : -1>(d, jB, WB, b);
    sigA = a;
    sigB = b;
  }
}

// A one-event move (location / arrival, NR = NA = 1) whose windows overlap
// changes only the rows of their symmetric difference: each lane walks its own
// <= 2 edge intervals (a uniform trip count across the warp) instead of the
// warp's whole band. Loads are scattered over the ~10 distinct rows the warp's
// lanes sit on, which costs L1 wavefronts but saves most of the issue slots.
template <int ND, typename YT>
__device__ __forceinline__ void edges(const Dev& d, int j, Win A0, Win R0, const Wins<ND>& D,
                                      const int (&sg)[ND > 0 ? ND : 1], const double2* Ts,
                                      double& sig, int& cnt) {
  int lo1, n1, dc1, lo2, n2, dc2;
  if (A0.hi <= R0.lo || R0.hi <= A0.lo || A0.hi == A0.lo || R0.hi == R0.lo) {
    lo1 = A0.lo;
    n1 = A0.hi - A0.lo;
    dc1 = 1;
    lo2 = R0.lo;
    n2 = R0.hi - R0.lo;
    dc2 = -1;
  } else {
    lo1 = min(A0.lo, R0.lo);
    n1 = max(A0.lo, R0.lo) - lo1;
    dc1 = A0.lo < R0.lo ? 1 : -1;
    lo2 = min(A0.hi, R0.hi);
    n2 = max(A0.hi, R0.hi) - lo2;
    dc2 = A0.hi > R0.hi ? 1 : -1;
  }
  const int total = n1 + n2;
  const int trips = __reduce_max_sync(0xffffffffu, (unsigned)total);
  constexpr int stride = 32;  // next row of the station tile
  const YT* __restrict__ y = reinterpret_cast<const YT*>(d.y) + yix(d.rows, 0, j);
  const uint16_t* __restrict__ c16 = reinterpret_cast<const uint16_t*>(d.cov) + yix(d.rows, 0, j);
  double s_loc = 0.0;
  int c_loc = 0;
  bool big = false;
  constexpr int RU = 4;
  for (int i0 = 0; i0 < trips; i0 += RU) {
    int r[RU], dc[RU], c[RU];
    YT yv[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      const int i = i0 + k;
      // dead slots read the zero pad row n and index the zero table row
      r[k] = min(i < n1 ? lo1 + i : lo2 + (i - n1), d.n);
      dc[k] = i < total ? (i < n1 ? dc1 : dc2) : 0;
    }
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      const size_t o = (size_t)r[k] * stride;
      c[k] = (int)__ldg(c16 + o);
      yv[k] = __ldg(y + o);
    }
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      int cc = c[k];
#pragma unroll
      for (int q = 0; q < ND; ++q) cc += sg[q] * inw(r[k], D.w[q]);
      big |= cc >= TBL - 2;
      const int idx = dc[k] ? ts_idx(min(cc, TBL - 3), dc_code(dc[k])) : kTsZero;
      const double2 e = Ts[idx];
      const double yy = (double)yv[k];
      s_loc += fma(-(yy * yy), e.y, e.x);
    }
  }
  c_loc = total;
  if (__any_sync(0xffffffffu, big)) {
    s_loc = 0.0;
    c_loc = 0;
    for (int i = 0; i < total; ++i) {
      const int rr = i < n1 ? lo1 + i : lo2 + (i - n1);
      const size_t o = (size_t)rr * stride;
      int cc = (int)__ldg(c16 + o);
#pragma unroll
      for (int q = 0; q < ND; ++q) cc += sg[q] * inw(rr, D.w[q]);
      s_loc += term(d, Ts, (double)__ldg(y + o), cc, i < n1 ? dc1 : dc2);
      ++c_loc;
    }
  }
  sig += s_loc;
  cnt += c_loc;
}

// Many effective diff windows at a station (> 4): the correction of the band
// rows is accumulated in a per-thread scratch column first (rare).
template <int NR, int NA, typename YT, bool GEN>
__device__ __forceinline__ void band_generic(const Dev& d, int j, bool v, int blo, int bhi,
                                          const Wins<NR> R, const Wins<NA> A, int np,
                                          const int* pold, const int* pnew,
                                          const double2* Ts, double* out_sig, int* out_cnt) {
  const YT* __restrict__ y = reinterpret_cast<const YT*>(d.y);
  const uint16_t* __restrict__ c16 = reinterpret_cast<const uint16_t*>(d.cov);
  signed char corr[BANDMAX];
  double sig = 0.0;
  int cnt = 0;
  for (int c0 = blo; c0 < bhi; c0 += BANDMAX) {
    const int c1 = min(bhi, c0 + BANDMAX);
    for (int i = 0; i < c1 - c0; ++i) corr[i] = 0;
    for (int q = 0; q < np && v; ++q) {
      const Win wo = pold[q] != -1 ? make_win(d, ver_arr<GEN>(d, pold[q], j)) : empty_win();
      const Win wn = pnew[q] != -1 ? make_win(d, ver_arr<GEN>(d, pnew[q], j)) : empty_win();
      if (weq(wo, wn)) continue;
      for (int r = max(wo.lo, c0); r < min(wo.hi, c1); ++r) corr[r - c0] -= 1;
      for (int r = max(wn.lo, c0); r < min(wn.hi, c1); ++r) corr[r - c0] += 1;
    }
    for (int r = c0; r < c1; ++r) {
      int dc = 0;
      for (int q = 0; q < NA; ++q) dc += inw(r, A.w[q]);
      for (int q = 0; q < NR; ++q) dc -= inw(r, R.w[q]);
      if (dc) {
        const size_t off = yix(d.rows, r, j);
        const int co = (int)__ldg(c16 + off) + corr[r - c0];
        sig += term(d, Ts, (double)__ldg(y + off), co, dc);
        ++cnt;
      }
    }
  }
  *out_sig += sig;
  *out_cnt += cnt;
}

// Effective diff windows of the region's own changes at station j: (start,
// current) version pairs whose windows coincide here (an arrival move
// elsewhere) correct nothing. The same for every proposal of a round, so the
// tile-major pass computes them once per tile. nwmax (warp max) > 4 sends the
// station through band_generic, which walks the pairs itself.
struct DiffW {
  Wins<4> D;
  int sg[4];
  int nwmax;
};

// Walk the region's (start, current) pairs at station j with each batch of
// four pairs' pool loads issued together; first four effective windows kept.
template <int K, bool GEN>
__device__ __forceinline__ int diff_collect(const Dev& d, int j, int np, const int* pold,
                                            const int* pnew, Win (&w)[K], int (&sg)[K]) {
  int nw = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    w[k] = empty_win();
    sg[k] = 0;
  }
  if (j >= d.S) return 0;
  for (int q0 = 0; q0 < np; q0 += 4) {
    double vo[4], vn[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = q0 + k;
      const int so = q < np ? pold[q] : -1, sn = q < np ? pnew[q] : -1;
      vo[k] = so != -1 ? ver_arr<GEN>(d, so, j) : 0.0;
      vn[k] = sn != -1 ? ver_arr<GEN>(d, sn, j) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = q0 + k;
      if (q >= np) break;
      const Win wo = pold[q] != -1 ? make_win(d, vo[k]) : empty_win();
      const Win wn = pnew[q] != -1 ? make_win(d, vn[k]) : empty_win();
      if (weq(wo, wn)) continue;
      if (wo.hi > wo.lo) {
#pragma unroll
        for (int m = 0; m < K; ++m)
          if (m == nw) {
            w[m] = wo;
            sg[m] = -1;
          }
        ++nw;
      }
      if (wn.hi > wn.lo) {
#pragma unroll
        for (int m = 0; m < K; ++m)
          if (m == nw) {
            w[m] = wn;
            sg[m] = 1;
          }
        ++nw;
      }
    }
  }
  return nw;
}

template <bool GEN>
__device__ __forceinline__ void diff_windows(const Dev& d, int j, int np, const int* pold,
                                             const int* pnew, DiffW& X) {
  const int nw = diff_collect<4, GEN>(d, j, np, pold, pnew, X.D.w, X.sg);
  X.nwmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nw);
}

// Per-station diff windows cached in shared memory for a round (the
// proposal-major pass, few stations): windows as uint16 (n < 65535).
struct DiffS {
  uint16_t lo[4], hi[4];
  int8_t sg[4];
  int n;
};
// windows 5..8 of a station (a region that has accepted several births this
// phase, as during burn-in from an empty start), kept in a second array so
// the common four-window path reads what it did before
struct DiffS4x {
  uint16_t lo[4], hi[4];
  int8_t sg[4];
};

template <bool GEN>
__device__ __forceinline__ void diff_station(const Dev& d, int j, int np, const int* pold,
                                             const int* pnew, DiffS& o, DiffS4x& ov) {
  Win w[8];
  int sg[8];
  o.n = diff_collect<8, GEN>(d, j, np, pold, pnew, w, sg);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    o.lo[k] = (uint16_t)w[k].lo;
    o.hi[k] = (uint16_t)w[k].hi;
    o.sg[k] = (int8_t)sg[k];
    ov.lo[k] = (uint16_t)w[4 + k].lo;
    ov.hi[k] = (uint16_t)w[4 + k].hi;
    ov.sg[k] = (int8_t)sg[4 + k];
  }
}

// k_phase's per-round diff-window cache (proposal-major pass): active under
// the same condition k_phase builds it; the overflow windows follow the
// cache in dynamic shared memory
__device__ __forceinline__ bool diff_cache_active(const Dev& d, int np) {
  return np > 0 && d.dcache_on != 0;
}
__device__ __forceinline__ const DiffS4x* diff_cache_overflow() {
  extern __shared__ double s_dyn_diff[];
  return reinterpret_cast<const DiffS4x*>(
      reinterpret_cast<const char*>(s_dyn_diff + LOGIWIN + 2 * MSPEC * NT + MSPEC * NT / 2) +
      (size_t)kDiffCache * sizeof(DiffS));
}

__device__ __forceinline__ void diff_from_cache(const DiffS& c, DiffW& X) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    X.D.w[k].lo = c.lo[k];
    X.D.w[k].hi = c.hi[k];
    X.sg[k] = c.sg[k];
  }
  X.nwmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)c.n);
}

// One station of one proposal (density.hpp:239-301): arrival densities of
// the added/removed versions (arr += added - removed) and the per-sample
// terms where the coverage changes (sig). Called by a whole warp
// (j = tile base + lane) so the band reduction is warp-uniform.
template <int NR, int NA, typename YT, bool GEN>
__device__ __forceinline__ void station_item(const Dev& d, const Prop& P, const PassIn& in,
                                             int j, int np, const int* pold, const int* pnew,
                                             DiffW X, bool haveX, const double2* Ts, double& sig,
                                             double& arr, int& cnt) {
  const long long t_item = kProfItems ? clock64() : 0;
  const bool v = j < d.S;
  Wins<NR> R;
  Wins<NA> A;
  const double s = v ? d.stations[j] : 0.0;
  double ra[NR > 0 ? NR : 1];
  // a generated removed version (spec v2): its arrival and, for a location /
  // joint move, the moved version's arrival come from the same normal
  double rz[NR > 0 ? NR : 1];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    R.w[q] = empty_win();
    ra[q] = 0.0;
    rz[q] = 0.0;
    if (v && q < P.nr) {
      const double mo = arrival_mean(d, P.rx[q], P.rt[q], s);
      const int rs = P.rslot[q];
      if (!GEN || rs >= 0) {
        ra[q] = __ldg(d.pool + (size_t)rs * d.S_pad + j);
      } else {
        const GenV* g = gv_of(d, rs);
        rz[q] = d.sigma * (double)seis_normal(g->seed, g->sweep, g->region, g->step, (uint32_t)j);
        ra[q] = mo + rz[q];
        ra[q] = gen_apply_ovr(g, j, ra[q]);
      }
      R.w[q] = clampw(make_win(d, ra[q]), in.wlo, in.whi);
      arr -= arr_logpdf(d, ra[q], mo);
    }
  }
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    A.w[a] = empty_win();
    if (v && a < P.na) {
      double aa;
      const double m = arrival_mean(d, P.ax[a], P.at[a], s);
      if (in.src == SRC_BIRTH) {
        aa = m + d.sigma * (double)seis_normal(in.seed, in.sweep, in.region, in.step,
                                               (uint32_t)j);
      } else if (in.src == SRC_SHIFT) {
        const int q = a < NR ? a : 0;
        if (!GEN || P.rslot[q] >= 0) {  // stored row: shift by the mean (proposals.hpp:153-157)
          aa = ra[q] + (m - arrival_mean(d, P.rx[q], P.rt[q], s));
        } else {  // generated version (spec v2): residual kept exactly
          const GenV* g = gv_of(d, P.rslot[q]);
          aa = m + rz[q];
          aa = gen_apply_ovr(g, j, aa);
        }
      } else {
        aa = in.rows[a][j];
      }
      A.w[a] = clampw(make_win(d, aa), in.wlo, in.whi);
      arr += arr_logpdf(d, aa, m);
    }
  }
  // windows that do not move leave every count unchanged
  if (NR == NA && NR > 0 && P.nr == P.na) {
    bool same;
    if (NR == 1)
      same = weq(A.w[0], R.w[0]);
    else
      same = (weq(A.w[0], R.w[0]) && weq(A.w[NA - 1], R.w[NR - 1])) ||
             (weq(A.w[0], R.w[NR - 1]) && weq(A.w[NA - 1], R.w[0]));
    if (same) {
#pragma unroll
      for (int q = 0; q < NR; ++q) R.w[q] = empty_win();
#pragma unroll
      for (int a = 0; a < NA; ++a) A.w[a] = empty_win();
    }
  }
  int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
  for (int a = 0; a < NA; ++a)
    if (A.w[a].hi > A.w[a].lo) {
      lo = min(lo, A.w[a].lo);
      hi = max(hi, A.w[a].hi);
    }
#pragma unroll
  for (int q = 0; q < NR; ++q)
    if (R.w[q].hi > R.w[q].lo) {
      lo = min(lo, R.w[q].lo);
      hi = max(hi, R.w[q].hi);
    }
  const int blo = __reduce_min_sync(0xffffffffu, lo);
  const int bhi = __reduce_max_sync(0xffffffffu, hi);
  if (blo >= bhi) return;
  // the tile-major pass hands in the tile's diff windows; otherwise they are
  // built here, only for stations the proposal changes
  // (by value: a pointer or a reference selected between two DiffW objects
  // would put them in local memory)
  if (!haveX) diff_windows<GEN>(d, j, np, pold, pnew, X);
  const Wins<4>& D = X.D;
  const int(&sg)[4] = X.sg;
  const int nwmax = X.nwmax;
  long long t_band = 0;
  if (kProfItems && NR + NA == 1) {
    __syncwarp();
    t_band = clock64();
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&s_tprof[0][6], (unsigned long long)(t_band - t_item));
      atomicAdd(&s_tprof[1][6], 1ull);
    }
  }
  if (nwmax == 0) {
    Wins<0> D0;
    int sg0[1];
    if (NR + NA == 1) {
      const Win W = NA ? A.w[0] : R.w[0];
      if (d.tpos)
        band1_terms<NA ? 1 : -1>(d, j, W, sig);
      else
        band1<NA ? 1 : -1, 0, YT>(d, j, W, D0, sg0, Ts, sig);
      cnt += W.hi - W.lo;
    }
    else if (NR == 1 && NA == 1 && P.nr == 1 && P.na == 1)
      edges<0, YT>(d, j, A.w[0], R.w[0], D0, sg0, Ts, sig, cnt);
    else
      band<NR, NA, 0, YT>(d, j, blo, bhi, R, A, D0, sg0, Ts, sig, cnt);
  } else if (nwmax <= 2) {
    Wins<2> D2;
    int sg2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      D2.w[q] = D.w[q];
      sg2[q] = sg[q];
    }
    if (NR + NA == 1) {
      const Win W = NA ? A.w[0] : R.w[0];
      band1<NA ? 1 : -1, 2, YT>(d, j, W, D2, sg2, Ts, sig);
      cnt += W.hi - W.lo;
    }
    else if (NR == 1 && NA == 1 && P.nr == 1 && P.na == 1)
      edges<2, YT>(d, j, A.w[0], R.w[0], D2, sg2, Ts, sig, cnt);
    else
      band<NR, NA, 2, YT>(d, j, blo, bhi, R, A, D2, sg2, Ts, sig, cnt);
  } else if (nwmax <= 4) {
    if (NR + NA == 1) {  // a dense move: the whole window in one batch, as with two windows
      const Win W = NA ? A.w[0] : R.w[0];
      band1<NA ? 1 : -1, 4, YT>(d, j, W, D, sg, Ts, sig);
      cnt += W.hi - W.lo;
    } else {
      band<NR, NA, 4, YT>(d, j, blo, bhi, R, A, D, sg, Ts, sig, cnt);
    }
  } else if (nwmax <= 8 && haveX && diff_cache_active(d, np)) {
    // five to eight windows at some station of the tile (a region that has
    // accepted several births this phase, as during burn-in from an empty
    // start): the first four from the registers, the rest from the round
    // cache's overflow array (12x cheaper per item than band_generic)
    const DiffS4x& ov = diff_cache_overflow()[j];
    Wins<8> D8;
    int sg8[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      D8.w[q] = D.w[q];
      sg8[q] = sg[q];
      D8.w[4 + q].lo = ov.lo[q];
      D8.w[4 + q].hi = ov.hi[q];
      sg8[4 + q] = ov.sg[q];
    }
    band<NR, NA, 8, YT>(d, j, blo, bhi, R, A, D8, sg8, Ts, sig, cnt);
  } else {
    band_generic<NR, NA, YT, GEN>(d, j, v, blo, bhi, R, A, np, pold, pnew, Ts, &sig, &cnt);
  }
  if (kProfItems && NR + NA == 1) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&s_tprof[0][7], (unsigned long long)(clock64() - t_band));
      atomicAdd(&s_tprof[1][7], 1ull);
    }
  }
}

// Arrival move (proposals.hpp:161-174) in production: only station st moves;
// the warp's lanes take rows.
template <typename YT, bool GEN>
__device__ __forceinline__ void arrival_item(const Dev& d, const Prop& P, const PassIn& in,
                                             int np, const int* pold, const int* pnew,
                                             const double2* Ts, double& sig, double& arr,
                                             int& cnt) {
  const int lane = threadIdx.x & 31;
  const int st = P.arr_st;
  const double old_a = ver_arr<GEN>(d, P.rslot[0], st);
  const double new_a = old_a + P.arr_da;
  const double mean = arrival_mean(d, P.rx[0], P.rt[0], d.stations[st]);
  if (lane == 0) arr += arr_logpdf(d, new_a, mean) - arr_logpdf(d, old_a, mean);
  // likelihood window: [0, n) chromatic, signal_window naive (density.hpp:244-262)
  const Win wo = clampw(make_win(d, old_a), in.wlo, in.whi);
  const Win wn = clampw(make_win(d, new_a), in.wlo, in.whi);
  if (weq(wo, wn)) return;
  const int blo = min(wo.hi > wo.lo ? wo.lo : INT_MAX, wn.hi > wn.lo ? wn.lo : INT_MAX);
  const int bhi = max(wo.hi > wo.lo ? wo.hi : INT_MIN, wn.hi > wn.lo ? wn.hi : INT_MIN);
  const YT* y = reinterpret_cast<const YT*>(d.y);
  const uint16_t* c16 = reinterpret_cast<const uint16_t*>(d.cov);
  for (int r = blo + lane; r < bhi; r += 32) {
    const int dc = inw(r, wn) - inw(r, wo);
    if (!dc) continue;
    int co = (int)c16[yix(d.rows, r, st)];
    for (int q = 0; q < np; ++q) {
      if (pold[q] != -1) co -= inw(r, make_win(d, ver_arr<GEN>(d, pold[q], st)));
      if (pnew[q] != -1) co += inw(r, make_win(d, ver_arr<GEN>(d, pnew[q], st)));
    }
    sig += term(d, Ts, (double)y[yix(d.rows, r, st)], co, dc);
    ++cnt;
  }
}

// Dispatch one work item (tile of 32 stations) of proposal P.
template <int MODE, typename YT, bool GEN>
__device__ __forceinline__ void score_item(const Dev& d, const Prop& P, const PassIn& in,
                                           int tile, int np, const int* pold,
                                           const int* pnew, const DiffW& X, bool haveX,
                                           const double2* Ts,
                                           double& sig, double& arr, int& cnt) {
  if (P.skip) return;
  const int j = tile * 32 + (threadIdx.x & 31);
  if (MODE == 0 && P.type == 3) {
    if (tile == 0) arrival_item<YT, GEN>(d, P, in, np, pold, pnew, Ts, sig, arr, cnt);
    return;
  }
  const int shape = P.nr * 3 + P.na;
  if (shape == 1)  // birth
    station_item<0, 1, YT, GEN>(d, P, in, j, np, pold, pnew, X, haveX, Ts, sig, arr, cnt);
  else if (shape == 3)  // death
    station_item<1, 0, YT, GEN>(d, P, in, j, np, pold, pnew, X, haveX, Ts, sig, arr, cnt);
  else if (shape == 4)  // location / arrival
    station_item<1, 1, YT, GEN>(d, P, in, j, np, pold, pnew, X, haveX, Ts, sig, arr, cnt);
  else  // joint pair, and any other change of <= 2 removed / 2 added events
    station_item<2, 2, YT, GEN>(d, P, in, j, np, pold, pnew, X, haveX, Ts, sig, arr, cnt);
}

}  // namespace seis
