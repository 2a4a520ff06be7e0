// kernels.cuh — device kernels of the B200 region-sweep engine.
//
// Hot path (one launch per color phase): k_phase, one CTA per same-color
// region, runs that region's k MH steps against the phase-start snapshot
// (frozen-snapshot semantics of run_chromatic, samplers.hpp:445-463) and
// scores every proposal with the fused likelihood delta (density.hpp:214-305)
// over the resident coverage counts. k_commit and k_rebuild are the color
// barrier (samplers.hpp:470-485): coverage deltas are scattered with packed
// 32-bit atomics and the id-sorted event table is rebuilt without a sort.
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

// Proposal descriptor written by thread 0, read by the CTA (double-buffered).
struct Prop {
  int type, skip, scored, nr, na;
  int rown[2], rslot[2], rsidx[2];
  double rx[2], rt[2];
  double ax[2], at[2];
  unsigned long long aid;
  int arr_st;
  double arr_da;
  long long tape_idx, tape_off;
  double logq_f, logq_r, u;
  int u_drawn, tape_acc;
  int accept;        // apply the change
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

__device__ __forceinline__ double tabL(const Dev& d, const double* Ls, int c) {
  return c < TBL ? Ls[c] : d.Lg[c];
}
__device__ __forceinline__ double tabI(const Dev& d, const double* Is, int c) {
  return c < TBL ? Is[c] : d.Ig[c];
}

// Per-sample likelihood term exactly as the reference forms it
// (density.hpp:286-301): (new_log - y2 new_inv) - (old_log - y2 old_inv).
__device__ __forceinline__ double sample_term(const Dev& d, const double* Ls, const double* Is,
                                              double y, int co, int cn) {
  const double y2 = y * y;
  return (tabL(d, Ls, cn) - y2 * tabI(d, Is, cn)) - (tabL(d, Ls, co) - y2 * tabI(d, Is, co));
}

// Rows [blo, bhi) of one station pair: dc = (#added - #removed) windows
// covering the row; co = coverage seen by this region (phase-start count +
// own diff correction), cn = co + dc. Diff windows held in registers (ND).
template <int ND, typename YT>
__device__ __forceinline__ void band_rows(const Dev& d, int p, int blo, int bhi,
                                          const Win (&A)[2][2], const Win (&R)[2][2],
                                          const Win (&D)[ND > 0 ? ND : 1][2],
                                          const int (&sg)[ND > 0 ? ND : 1], const double* Ls,
                                          const double* Is, double& acc, int& cnt) {
  using T2 = typename Y2<YT>::T;
  const T2* __restrict__ y2 = reinterpret_cast<const T2*>(d.y);
  const uint32_t* __restrict__ cov = d.cov;
  for (int r = blo; r < bhi; ++r) {
    const int dc0 = inw(r, A[0][0]) + inw(r, A[1][0]) - inw(r, R[0][0]) - inw(r, R[1][0]);
    const int dc1 = inw(r, A[0][1]) + inw(r, A[1][1]) - inw(r, R[0][1]) - inw(r, R[1][1]);
    if (dc0 | dc1) {
      const size_t off = (size_t)r * d.P2 + p;
      const uint32_t w = __ldg(cov + off);
      const T2 yy = __ldg(y2 + off);
      int c0 = (int)(w & 0xffffu), c1 = (int)(w >> 16);
#pragma unroll
      for (int q = 0; q < ND; ++q) {
        c0 += sg[q] * inw(r, D[q][0]);
        c1 += sg[q] * inw(r, D[q][1]);
      }
      if (dc0) {
        acc += sample_term(d, Ls, Is, (double)yy.x, c0, c0 + dc0);
        ++cnt;
      }
      if (dc1) {
        acc += sample_term(d, Ls, Is, (double)yy.y, c1, c1 + dc1);
        ++cnt;
      }
    }
  }
}

// Generic diff correction for many own diff entries: the correction of the
// band rows is accumulated in a per-thread scratch column first.
template <typename YT>
__device__ __noinline__ void band_rows_generic(const Dev& d, int p, int blo, int bhi,
                                               const Win (&A)[2][2], const Win (&R)[2][2],
                                               int nd, const int* dslot, const int* dsign,
                                               const double* Ls, const double* Is, double& acc,
                                               int& cnt) {
  using T2 = typename Y2<YT>::T;
  const T2* __restrict__ y2 = reinterpret_cast<const T2*>(d.y);
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
  signed char corr[2][BANDMAX];
  for (int c0 = blo; c0 < bhi; c0 += BANDMAX) {
    const int c1 = min(bhi, c0 + BANDMAX);
    for (int i = 0; i < c1 - c0; ++i) corr[0][i] = corr[1][i] = 0;
    for (int q = 0; q < nd; ++q) {
      const double2 a = pool2[(size_t)dslot[q] * d.P2 + p];
      const Win w0 = make_win(d, a.x), w1 = make_win(d, a.y);
      for (int r = max(w0.lo, c0); r < min(w0.hi, c1); ++r) corr[0][r - c0] += dsign[q];
      for (int r = max(w1.lo, c0); r < min(w1.hi, c1); ++r) corr[1][r - c0] += dsign[q];
    }
    for (int r = c0; r < c1; ++r) {
      const int dc0 = inw(r, A[0][0]) + inw(r, A[1][0]) - inw(r, R[0][0]) - inw(r, R[1][0]);
      const int dc1 = inw(r, A[0][1]) + inw(r, A[1][1]) - inw(r, R[0][1]) - inw(r, R[1][1]);
      if (dc0 | dc1) {
        const size_t off = (size_t)r * d.P2 + p;
        const uint32_t w = __ldg(d.cov + off);
        const T2 yy = __ldg(y2 + off);
        const int co0 = (int)(w & 0xffffu) + corr[0][r - c0];
        const int co1 = (int)(w >> 16) + corr[1][r - c0];
        if (dc0) {
          acc += sample_term(d, Ls, Is, (double)yy.x, co0, co0 + dc0);
          ++cnt;
        }
        if (dc1) {
          acc += sample_term(d, Ls, Is, (double)yy.y, co1, co1 + dc1);
          ++cnt;
        }
      }
    }
  }
}

template <int ND, typename YT>
__device__ __forceinline__ void band_with_diff(const Dev& d, int p, bool v0, bool v1, int blo,
                                               int bhi, const Win (&A)[2][2],
                                               const Win (&R)[2][2], int nd, const int* dslot,
                                               const int* dsign, const double* Ls,
                                               const double* Is, double& acc, int& cnt) {
  Win D[ND > 0 ? ND : 1][2];
  int sg[ND > 0 ? ND : 1];
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
#pragma unroll
  for (int q = 0; q < (ND > 0 ? ND : 1); ++q) {
    D[q][0] = D[q][1] = empty_win();
    sg[q] = 0;
    if (q < nd && q < ND) {
      const double2 a = pool2[(size_t)dslot[q] * d.P2 + p];
      if (v0) D[q][0] = make_win(d, a.x);
      if (v1) D[q][1] = make_win(d, a.y);
      sg[q] = dsign[q];
    }
  }
  band_rows<ND, YT>(d, p, blo, bhi, A, R, D, sg, Ls, Is, acc, cnt);
}

}  // namespace seis
