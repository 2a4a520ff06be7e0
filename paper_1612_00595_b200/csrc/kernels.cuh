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
  double logq_f, logq_r, u;
  int u_drawn, tape_acc;
  int accept;
  int dslot[2], inplace[2];
};

struct OwnEv {
  unsigned long long id;
  double x, t;
  int slot, sidx;
};

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
__device__ __forceinline__ double term(const Dev& d, const double2* Ts, double y, int c, int dc) {
  const int code = dc < 0 ? dc + 2 : dc + 1;  // dc in {-2,-1,1,2} -> 0..3
  const int idx = c * 4 + code;
  double2 e = Ts[min(idx, TBL * 4 - 1)];
  if (c >= TBL) e = d.Dg[idx];  // counts beyond the shared-memory table (rare)
  const double y2 = y * y;
  return fma(-y2, e.y, e.x);
}

template <int N>
struct Wins {
  Win w[N > 0 ? N : 1][2];
};

// Rows [blo, bhi) of one station pair, RU rows' loads in flight at a time.
// dc = added - removed windows covering the row; c = phase-start count + own
// diff correction (the region's frozen view); only rows with dc != 0 load.
template <int NR, int NA, int ND, typename YT>
__device__ __forceinline__ void band(const Dev& d, int p, int blo, int bhi, const Wins<NR>& R,
                                     const Wins<NA>& A, const Wins<ND>& D,
                                     const int (&sg)[ND > 0 ? ND : 1], const double2* Ts,
                                     double& sig, int& cnt) {
  using T2 = typename Y2<YT>::T;
  constexpr int RU = 4;
  const T2* __restrict__ yp = reinterpret_cast<const T2*>(d.y) + (size_t)blo * d.P2 + p;
  const uint32_t* __restrict__ cp = d.cov + (size_t)blo * d.P2 + p;
  const size_t stride = (size_t)d.P2;
  for (int r0 = blo; r0 < bhi; r0 += RU, yp += RU * stride, cp += RU * stride) {
    int dc0[RU], dc1[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k) {
      const int r = r0 + k;  // rows past bhi lie outside every window: dc = 0
      int a0 = 0, a1 = 0;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        a0 += inw(r, A.w[a][0]);
        a1 += inw(r, A.w[a][1]);
      }
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        a0 -= inw(r, R.w[q][0]);
        a1 -= inw(r, R.w[q][1]);
      }
      dc0[k] = a0;
      dc1[k] = a1;
    }
    uint32_t w[RU];
    T2 yy[RU];
#pragma unroll
    for (int k = 0; k < RU; ++k)
      if (dc0[k] | dc1[k]) {
        w[k] = __ldg(cp + k * stride);
        yy[k] = __ldg(yp + k * stride);
      }
#pragma unroll
    for (int k = 0; k < RU; ++k)
      if (dc0[k] | dc1[k]) {
        const int r = r0 + k;
        int c0 = (int)(w[k] & 0xffffu), c1 = (int)(w[k] >> 16);
#pragma unroll
        for (int q = 0; q < ND; ++q) {
          c0 += sg[q] * inw(r, D.w[q][0]);
          c1 += sg[q] * inw(r, D.w[q][1]);
        }
        if (dc0[k]) {
          sig += term(d, Ts, (double)yy[k].x, c0, dc0[k]);
          ++cnt;
        }
        if (dc1[k]) {
          sig += term(d, Ts, (double)yy[k].y, c1, dc1[k]);
          ++cnt;
        }
      }
  }
}

// Many own diff entries: the correction of the band rows is accumulated in a
// per-thread scratch column first (nd > 2).
template <int NR, int NA, typename YT>
__device__ __noinline__ void band_generic(const Dev& d, int p, int blo, int bhi,
                                          const Wins<NR> R, const Wins<NA> A, int nd,
                                          const int* dslot, const int* dsign,
                                          const double2* Ts, double& sig, int& cnt) {
  using T2 = typename Y2<YT>::T;
  const T2* __restrict__ y2 = reinterpret_cast<const T2*>(d.y);
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
  signed char corr[2][BANDMAX];
  for (int c0 = blo; c0 < bhi; c0 += BANDMAX) {
    const int c1 = min(bhi, c0 + BANDMAX);
    for (int i = 0; i < c1 - c0; ++i) corr[0][i] = corr[1][i] = 0;
    for (int q = 0; q < nd; ++q) {
      const double2 a = pool2[(size_t)dslot[q] * d.P2 + p];
      const Win w0 = 2 * p < d.S ? make_win(d, a.x) : empty_win();
      const Win w1 = 2 * p + 1 < d.S ? make_win(d, a.y) : empty_win();
      for (int r = max(w0.lo, c0); r < min(w0.hi, c1); ++r) corr[0][r - c0] += dsign[q];
      for (int r = max(w1.lo, c0); r < min(w1.hi, c1); ++r) corr[1][r - c0] += dsign[q];
    }
    for (int r = c0; r < c1; ++r) {
      int dc0 = 0, dc1 = 0;
      for (int a = 0; a < NA; ++a) {
        dc0 += inw(r, A.w[a][0]);
        dc1 += inw(r, A.w[a][1]);
      }
      for (int q = 0; q < NR; ++q) {
        dc0 -= inw(r, R.w[q][0]);
        dc1 -= inw(r, R.w[q][1]);
      }
      if (dc0 | dc1) {
        const size_t off = (size_t)r * d.P2 + p;
        const uint32_t w = __ldg(d.cov + off);
        const T2 yy = __ldg(y2 + off);
        const int co0 = (int)(w & 0xffffu) + corr[0][r - c0];
        const int co1 = (int)(w >> 16) + corr[1][r - c0];
        if (dc0) {
          sig += term(d, Ts, (double)yy.x, co0, dc0);
          ++cnt;
        }
        if (dc1) {
          sig += term(d, Ts, (double)yy.y, co1, dc1);
          ++cnt;
        }
      }
    }
  }
}

template <int NR, int NA, int ND, typename YT>
__device__ __forceinline__ void band_diff(const Dev& d, int p, bool v0, bool v1, int blo, int bhi,
                                          const Wins<NR>& R, const Wins<NA>& A, int nd,
                                          const int* dslot, const int* dsign, const double2* Ts,
                                          double& sig, int& cnt) {
  Wins<ND> D;
  int sg[ND > 0 ? ND : 1];
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
#pragma unroll
  for (int q = 0; q < ND; ++q) {
    D.w[q][0] = D.w[q][1] = empty_win();
    sg[q] = 0;
    if (q < nd) {
      const double2 a = pool2[(size_t)dslot[q] * d.P2 + p];
      if (v0) D.w[q][0] = make_win(d, a.x);
      if (v1) D.w[q][1] = make_win(d, a.y);
      sg[q] = dsign[q];
    }
  }
  band<NR, NA, ND, YT>(d, p, blo, bhi, R, A, D, sg, Ts, sig, cnt);
}

// One station pair of one proposal (density.hpp:239-301): arrival densities
// of the added/removed versions (arr += added - removed) and the per-sample
// terms where the coverage changes (sig). Called by a whole warp (p = tile
// base + lane), so the band reduction is warp-uniform.
template <int NR, int NA, typename YT>
__device__ __noinline__ void pair_item(const Dev& d, const Prop& P, const PassIn& in, int p,
                                          int nd, const int* dslot, const int* dsign,
                                          const double2* Ts, double& sig, double& arr,
                                          int& cnt) {
  const bool pv = p < d.P2;
  const bool v0 = pv && 2 * p < d.S, v1 = pv && 2 * p + 1 < d.S;
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
  Wins<NR> R;
  Wins<NA> A;
  double s0 = 0.0, s1 = 0.0;
  if (pv) {
    const double2 s = reinterpret_cast<const double2*>(d.stations)[p];
    s0 = s.x;
    s1 = s.y;
  }
  double ra[NR > 0 ? NR : 1][2];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    R.w[q][0] = R.w[q][1] = empty_win();
    ra[q][0] = ra[q][1] = 0.0;
    if (pv) {
      const double2 v = pool2[(size_t)P.rslot[q] * d.P2 + p];
      ra[q][0] = v.x;
      ra[q][1] = v.y;
      if (v0) {
        R.w[q][0] = clampw(make_win(d, v.x), in.wlo, in.whi);
        arr -= arr_logpdf(d, v.x, arrival_mean(d, P.rx[q], P.rt[q], s0));
      }
      if (v1) {
        R.w[q][1] = clampw(make_win(d, v.y), in.wlo, in.whi);
        arr -= arr_logpdf(d, v.y, arrival_mean(d, P.rx[q], P.rt[q], s1));
      }
    }
  }
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    A.w[a][0] = A.w[a][1] = empty_win();
    if (pv) {
      double a0 = 0.0, a1 = 0.0;
      const double m0 = arrival_mean(d, P.ax[a], P.at[a], s0);
      const double m1 = arrival_mean(d, P.ax[a], P.at[a], s1);
      if (in.src == SRC_BIRTH) {
        float z0, z1;
        seis_normal_pair(in.seed, in.sweep, in.region, in.step, (uint32_t)p, &z0, &z1);
        a0 = m0 + d.sigma * (double)z0;
        a1 = m1 + d.sigma * (double)z1;
      } else if (in.src == SRC_SHIFT) {
        const int q = a < NR ? a : 0;
        a0 = ra[q][0] + (m0 - arrival_mean(d, P.rx[q], P.rt[q], s0));
        a1 = ra[q][1] + (m1 - arrival_mean(d, P.rx[q], P.rt[q], s1));
      } else {
        if (v0) a0 = in.rows[a][2 * p];
        if (v1) a1 = in.rows[a][2 * p + 1];
      }
      if (v0) {
        A.w[a][0] = clampw(make_win(d, a0), in.wlo, in.whi);
        arr += arr_logpdf(d, a0, m0);
      }
      if (v1) {
        A.w[a][1] = clampw(make_win(d, a1), in.wlo, in.whi);
        arr += arr_logpdf(d, a1, m1);
      }
    }
  }
  // windows that do not move leave every count unchanged
  if (NR == NA && NR > 0) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      bool same;
      if (NR == 1)
        same = weq(A.w[0][s], R.w[0][s]);
      else
        same = (weq(A.w[0][s], R.w[0][s]) && weq(A.w[NA - 1][s], R.w[NR - 1][s])) ||
               (weq(A.w[0][s], R.w[NR - 1][s]) && weq(A.w[NA - 1][s], R.w[0][s]));
      if (same) {
#pragma unroll
        for (int q = 0; q < NR; ++q) R.w[q][s] = empty_win();
#pragma unroll
        for (int a = 0; a < NA; ++a) A.w[a][s] = empty_win();
      }
    }
  }
  int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
#pragma unroll
    for (int a = 0; a < NA; ++a)
      if (A.w[a][s].hi > A.w[a][s].lo) {
        lo = min(lo, A.w[a][s].lo);
        hi = max(hi, A.w[a][s].hi);
      }
#pragma unroll
    for (int q = 0; q < NR; ++q)
      if (R.w[q][s].hi > R.w[q][s].lo) {
        lo = min(lo, R.w[q][s].lo);
        hi = max(hi, R.w[q][s].hi);
      }
  }
  const int blo = __reduce_min_sync(0xffffffffu, lo);
  const int bhi = __reduce_max_sync(0xffffffffu, hi);
  if (blo >= bhi) return;
  if (nd == 0)
    band_diff<NR, NA, 0, YT>(d, p, v0, v1, blo, bhi, R, A, nd, dslot, dsign, Ts, sig, cnt);
  else if (nd <= 2)
    band_diff<NR, NA, 2, YT>(d, p, v0, v1, blo, bhi, R, A, nd, dslot, dsign, Ts, sig, cnt);
  else
    band_generic<NR, NA, YT>(d, p, blo, bhi, R, A, nd, dslot, dsign, Ts, sig, cnt);
}

// Arrival move (proposals.hpp:161-174) in production: only station st moves;
// the warp's lanes take rows.
template <typename YT>
__device__ __forceinline__ void arrival_item(const Dev& d, const Prop& P, int nd,
                                             const int* dslot, const int* dsign,
                                             const double2* Ts, double& sig, double& arr,
                                             int& cnt) {
  const int lane = threadIdx.x & 31;
  const int st = P.arr_st;
  const double old_a = d.pool[(size_t)P.rslot[0] * d.S_pad + st];
  const double new_a = old_a + P.arr_da;
  const double mean = arrival_mean(d, P.rx[0], P.rt[0], d.stations[st]);
  if (lane == 0) arr += arr_logpdf(d, new_a, mean) - arr_logpdf(d, old_a, mean);
  const Win wo = make_win(d, old_a), wn = make_win(d, new_a);
  if (weq(wo, wn)) return;
  const int blo = min(wo.hi > wo.lo ? wo.lo : INT_MAX, wn.hi > wn.lo ? wn.lo : INT_MAX);
  const int bhi = max(wo.hi > wo.lo ? wo.hi : INT_MIN, wn.hi > wn.lo ? wn.hi : INT_MIN);
  const YT* y = reinterpret_cast<const YT*>(d.y);
  const uint16_t* c16 = reinterpret_cast<const uint16_t*>(d.cov);
  for (int r = blo + lane; r < bhi; r += 32) {
    const int dc = inw(r, wn) - inw(r, wo);
    if (!dc) continue;
    int co = (int)c16[(size_t)r * d.S_pad + st];
    for (int q = 0; q < nd; ++q) {
      const Win w = make_win(d, d.pool[(size_t)dslot[q] * d.S_pad + st]);
      co += dsign[q] * inw(r, w);
    }
    sig += term(d, Ts, (double)y[(size_t)r * d.S_pad + st], co, dc);
    ++cnt;
  }
}

// Dispatch one work item (tile of 32 station pairs) of proposal P.
template <int MODE, typename YT>
__device__ __forceinline__ void score_item(const Dev& d, const Prop& P, const PassIn& in,
                                           int tile, int nd, const int* dslot,
                                           const int* dsign, const double2* Ts, double& sig,
                                           double& arr, int& cnt) {
  if (P.skip) return;
  const int p = tile * 32 + (threadIdx.x & 31);
  if (MODE == 0 && P.type == 3) {
    if (tile == 0) arrival_item<YT>(d, P, nd, dslot, dsign, Ts, sig, arr, cnt);
    return;
  }
  if (P.nr == 0 && P.na == 1)
    pair_item<0, 1, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 1 && P.na == 0)
    pair_item<1, 0, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 1 && P.na == 1)
    pair_item<1, 1, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 2 && P.na == 2)
    pair_item<2, 2, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 2 && P.na == 0)
    pair_item<2, 0, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 0 && P.na == 2)
    pair_item<0, 2, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 1 && P.na == 2)
    pair_item<1, 2, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
  else if (P.nr == 2 && P.na == 1)
    pair_item<2, 1, YT>(d, P, in, p, nd, dslot, dsign, Ts, sig, arr, cnt);
}

}  // namespace seis
