// engine.cu — B200 chromatic region-sweep engine: kernels + C-ABI host.
//
// Replaces the reference's run_chromatic hot path (arXiv 1612.00595 reference,
// proj/include/seismic/samplers.hpp:401-498, proposals.hpp:84-293,
// density.hpp:214-305, partition.hpp:40-90) with one CTA per same-color
// region on sm_100a. See DESIGN.md for the layout and the roofline.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false ... (the
// reference's integer outputs come from fp64 expressions evaluated without
// contraction; FMA is used only where written explicitly).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.cuh"
#include "kernels.cuh"
#include "phase_api.h"

namespace seis {

// ----------------------------------------------------------------- device xoshiro
// derive_stream / Rng::uniform (reference rng.hpp:21-51, 110-121) for the
// partition offset stream; integer-exact on device.
__device__ __host__ inline uint64_t d_splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __host__ inline uint64_t d_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
__device__ __host__ inline double d_offset_uniform(uint64_t seed, uint64_t purpose, uint64_t i0,
                                                   double lo, double hi) {
  uint64_t key = seed;
  uint64_t k = d_splitmix(key);
  const uint64_t words[4] = {purpose, i0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    uint64_t w = words[i];
    k ^= d_splitmix(w);
    k = d_splitmix(k);
  }
  uint64_t s[4];
  for (int i = 0; i < 4; ++i) s[i] = d_splitmix(k);
  if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
  const uint64_t result = d_rotl(s[0] + s[3], 23) + s[0];
  const double u = (double)(result >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * u;
}

// ----------------------------------------------------------------- partition
// build_partition + color_partition (partition.hpp:40-90), one thread per
// epoch: boundaries by the reference's repeated fp64 addition, colors i % k,
// separation invariant checked against the nearest same-colored region
// (equivalent to the reference's all-pairs check since boundaries increase).
// One CTA per epoch: thread 0 places the boundaries (the reference's repeated
// fp64 addition is sequential), then the CTA fills colors and checks the
// separation invariant in parallel.
constexpr int kPartThreads = 128;
__global__ void __launch_bounds__(kPartThreads)
    k_partition(double T, double l, double tau, int ncol, int mode, uint64_t seed, int epoch0,
                int n_ep, double u_explicit, int bcap, double* bnd, int* nreg, int* err,
                int* colors) {
  const int e = blockIdx.x;
  if (e >= n_ep) return;
  const int epoch = epoch0 + e;
  double* b = bnd + (size_t)e * bcap;
  __shared__ int s_n;
  if (threadIdx.x == 0) {
    // mode 0 static (u = 0), 1 dynamic (u redrawn after every epoch,
    // samplers.hpp:488-493), 2 explicit offset
    double u = 0.0;
    if (mode == 1 && epoch > 0) u = d_offset_uniform(seed, 6, (uint64_t)epoch, 0.0, l);
    if (mode == 2) u = u_explicit;
    int nb = 0;
    b[nb++] = 0.0;
    double x = u > 0 ? u : l;
    while (x < T - 1e-9) {
      if (nb >= bcap - 1) {
        atomicExch(err, 2);
        nb = -1;
        break;
      }
      b[nb++] = x;
      x += l;
    }
    if (nb > 0) {
      b[nb++] = T;
      nreg[e] = nb - 1;
    }
    s_n = nb - 1;
  }
  __syncthreads();
  const int n = s_n;
  if (n < 0) return;
  if (colors)
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      colors[(size_t)e * bcap + i] = i % ncol;  // partition.hpp:81-82
  bool bad = false;
  for (int i = threadIdx.x; i + ncol < n; i += blockDim.x)
    bad |= b[i + ncol] - b[i + 1] < tau - 1e-9;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(err, 1);
}

__global__ void k_offsets(uint64_t seed, int64_t epoch, double l, double* out) {
  *out = d_offset_uniform(seed, 6, (uint64_t)epoch, 0.0, l);
}

// Partition::region_of (partition.hpp:33-37): first i < n-1 with t < b[i+1],
// else n-1; a binary search over the same boundary array.
__device__ __forceinline__ int region_of(const double* b, int n, double t) {
  int lo = 0, hi = n - 1;  // answer in [lo, hi]
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (t < b[mid + 1])
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__global__ void k_region_of(const double* b, int n, int64_t m, const double* t, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = region_of(b, n, t[i]);
}

// Dispatch order of a color phase's region chains (longest processing time
// first). A chain with no phase-start events proposes mostly null moves
// (death, location, arrival and joint need an event) and costs a fraction of
// one with events; CTAs are dispatched in blockIdx order, so slots with more
// events go first and the cheap chains fill the last wave instead of leaving
// SMs idle behind a late expensive chain. The order never changes results:
// each chain's draws, births' ids and outputs are keyed by its slot.
__device__ int block_scan_excl(int v, int* total);
constexpr int kOrderBuckets = 3;  // phase-start events >= 2, 1, 0
__global__ void __launch_bounds__(1024)
    k_order(const double* tab_t, const int* n_events, const double* bnd, int nreg, int color,
            int ncol, int ncr, int* cnt, int* order) {
  __shared__ int s_tot[kOrderBuckets], s_base[kOrderBuckets];
  const int tid = threadIdx.x;
  for (int i = tid; i < ncr; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int N = *n_events;
  for (int i = tid; i < N; i += blockDim.x) {
    const int r = region_of(bnd, nreg, tab_t[i]);
    if (r >= color && (r - color) % ncol == 0) atomicAdd(&cnt[(r - color) / ncol], 1);
  }
  __syncthreads();
  // stable counting sort: buckets in decreasing cost, slots (time order)
  // ascending inside a bucket, so concurrently running chains stay
  // neighbours in time and share signal rows in L2
  for (int b = tid; b < kOrderBuckets; b += blockDim.x) s_tot[b] = 0;
  __syncthreads();
  for (int s = tid; s < ncr; s += blockDim.x)
    atomicAdd(&s_tot[max(0, kOrderBuckets - 1 - min(cnt[s], kOrderBuckets - 1))], 1);
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int b = 0; b < kOrderBuckets; ++b) {
      s_base[b] = acc;
      acc += s_tot[b];
    }
  }
  __syncthreads();
  for (int c0 = 0; c0 < ncr; c0 += blockDim.x) {
    const int s = c0 + tid;
    const int b = s < ncr ? kOrderBuckets - 1 - min(cnt[s], kOrderBuckets - 1) : -1;
    int pos = 0;
#pragma unroll
    for (int q = 0; q < kOrderBuckets; ++q) {
      int tot;
      const int ex = block_scan_excl(b == q ? 1 : 0, &tot);
      if (b == q) pos = s_base[q] + ex;
      __syncthreads();
      if (tid == 0) s_base[q] += tot;
      __syncthreads();
    }
    if (s < ncr) order[pos] = s;
  }
}

// ----------------------------------------------------------------- signals
template <typename YT>
__global__ void k_transpose(const YT* __restrict__ src, YT* __restrict__ dst, int S, int S_pad,
                            int n, int rows) {
  __shared__ YT tile[32][33];
  const int s0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int j = j0 + k, s = s0 + threadIdx.x;
    tile[k][threadIdx.x] = (j < S && s < n) ? src[(size_t)j * n + s] : YT(0);
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int s = s0 + k, j = j0 + threadIdx.x;
    if (s < n && j < S_pad) dst[yix(rows, s, j)] = tile[threadIdx.x][k];
  }
}

// coverage of every event of the table (variance_profile, density.hpp:112-129)
__global__ void k_build_cov(Dev d, Table tab, Ctl* ctl) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= d.P2) return;
  for (int e = blockIdx.y; e < ctl->n_events; e += gridDim.y) {
    const int sl = tab.slot[e];
    double2 a;
    if (sl >= 0) {
      a = reinterpret_cast<const double2*>(d.pool)[(size_t)sl * d.P2 + p];
    } else {  // generated version
      a.x = 2 * p < d.S ? arr_of(d, sl, 2 * p) : 0.0;
      a.y = 2 * p + 1 < d.S ? arr_of(d, sl, 2 * p + 1) : 0.0;
    }
    const Win w0 = 2 * p < d.S ? make_win(d, a.x) : empty_win();
    const Win w1 = 2 * p + 1 < d.S ? make_win(d, a.y) : empty_win();
    const int lo = min(w0.lo < w0.hi ? w0.lo : INT_MAX, w1.lo < w1.hi ? w1.lo : INT_MAX);
    const int hi = max(w0.hi > w0.lo ? w0.hi : INT_MIN, w1.hi > w1.lo ? w1.hi : INT_MIN);
    for (int r = lo; r < hi; ++r) {
      const int i0 = inw(r, w0), i1 = inw(r, w1);
      const unsigned inc = (unsigned)i0 + ((unsigned)i1 << 16);
      if (inc) {
        const unsigned old = atomicAdd(d.cov + pix(d.rows, r, p), inc);
        if ((old & 0xffffu) + i0 > 0xffffu || (old >> 16) + i1 > 0xffffu)
          set_err(ctl, ERR_COUNT_OVERFLOW);
      }
    }
  }
}

// Per-sample term cache (Dev::tpos / tneg) from the committed counts: for
// every sample the likelihood change of one more / one fewer covering event,
// the same expression and table entries the dense band evaluates
// (density.hpp:286-301). One streaming pass over y and the counts.
template <typename YT>
__global__ void k_terms(Dev d, double* __restrict__ tpos, double* __restrict__ tneg) {
  const YT* __restrict__ y = reinterpret_cast<const YT*>(d.y);
  const uint16_t* __restrict__ c16 = reinterpret_cast<const uint16_t*>(d.cov);
  const size_t per_tile = (size_t)d.rows * 32, live = (size_t)d.n * 32;
  const size_t total = (size_t)(d.S_pad / 32) * per_tile;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    if (i % per_tile >= live) continue;  // pad rows stay zero
    const int c = (int)c16[i];
    const double yy = (double)y[i];
    const double w = -(yy * yy);
    const double2 ep = d.Dg[c * 4 + 2], em = d.Dg[c * 4 + 1];  // dc_code(+1), dc_code(-1)
    tpos[i] = fma(w, ep.y, ep.x);
    tneg[i] = fma(w, em.y, em.x);
  }
}

// ----------------------------------------------------------------- barrier
// Coverage commit: C += sum over regions of (own_now - own_start) windows;
// same-color footprints overlap, so packed 32-bit atomics.
#ifndef SEIS_COMMIT_THREADS
#define SEIS_COMMIT_THREADS 512
#endif
constexpr int kCommitThreads = SEIS_COMMIT_THREADS;
static_assert(kCommitThreads % 32 == 0 && kCommitThreads >= 64 && kCommitThreads <= 1024,
              "block_scan_excl needs whole warps, at most 32 of them");
// regions with few CTAs (config[1]: 128 per phase) split their items over
// blockIdx.y so the commit fills every SM several CTAs deep
inline dim3 commit_grid(int ncr, int n_sm) {
  const int split = std::max(1, std::min(8, (4 * n_sm + ncr - 1) / std::max(ncr, 1)));
  return dim3((unsigned)ncr, (unsigned)split);
}
__device__ __forceinline__ void commit_body(const Dev& d, int color, int ncol, int nreg,
                                            int n_slots, const int* diff_cnt,
                                            const DiffPair* diff, Ovf ovf, int* free_stack,
                                            Ctl* ctl) {
  const int slot_idx = blockIdx.x;
  const int region = color + slot_idx * ncol;
  if (region >= nreg) return;
  const int nd = diff_cnt[slot_idx];
  const DiffPair* de = diff + diff_off(ovf, n_slots, slot_idx);
  const double2* pool2 = reinterpret_cast<const double2*>(d.pool);
  // (diff entry, station pair) items over the whole CTA: a region's few
  // entries x P2 pairs, so every thread has work even when P2 is small
  const long long n_items = (long long)nd * d.P2;
  for (long long it = (long long)blockIdx.y * blockDim.x + threadIdx.x; it < n_items;
       it += (long long)gridDim.y * blockDim.x) {
    const int q = (int)(it / d.P2), p = (int)(it - (long long)q * d.P2);
    if (de[q].kind != 0) continue;
    const int so = de[q].old_slot, sn = de[q].new_slot;
    {
      Win o0 = empty_win(), o1 = empty_win(), n0 = empty_win(), n1 = empty_win();
      if (so >= 0) {
        const double2 a = pool2[(size_t)so * d.P2 + p];
        if (2 * p < d.S) o0 = make_win(d, a.x);
        if (2 * p + 1 < d.S) o1 = make_win(d, a.y);
      } else if (so != -1) {  // generated version
        if (2 * p < d.S) o0 = make_win(d, arr_of(d, so, 2 * p));
        if (2 * p + 1 < d.S) o1 = make_win(d, arr_of(d, so, 2 * p + 1));
      }
      if (sn >= 0) {
        const double2 a = pool2[(size_t)sn * d.P2 + p];
        if (2 * p < d.S) n0 = make_win(d, a.x);
        if (2 * p + 1 < d.S) n1 = make_win(d, a.y);
      } else if (sn != -1) {
        if (2 * p < d.S) n0 = make_win(d, arr_of(d, sn, 2 * p));
        if (2 * p + 1 < d.S) n1 = make_win(d, arr_of(d, sn, 2 * p + 1));
      }
      if (weq(o0, n0)) o0 = n0 = empty_win();  // unchanged at this station
      if (weq(o1, n1)) o1 = n1 = empty_win();
      int lo = INT_MAX, hi = INT_MIN;
      const Win ws[4] = {o0, o1, n0, n1};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ws[k].hi > ws[k].lo) {
          lo = min(lo, ws[k].lo);
          hi = max(hi, ws[k].hi);
        }
      for (int r = lo; r < hi; ++r) {
        const int d0 = inw(r, n0) - inw(r, o0), d1 = inw(r, n1) - inw(r, o1);
        const int inc = d0 + d1 * 65536;
        if (inc) {
          // true counts never go negative mid-commit (only counted start
          // versions are removed), so the halves never borrow: a half that
          // passes 0xffff is a real uint16 overflow
          const unsigned old = atomicAdd(d.cov + pix(d.rows, r, p), (unsigned)inc);
          if ((d0 > 0 && (int)(old & 0xffffu) + d0 > 0xffff) ||
              (d1 > 0 && (int)(old >> 16) + d1 > 0xffff))
            set_err(ctl, ERR_COUNT_OVERFLOW);
        }
      }
    }
  }
  // the freed slots are popped again only by the next phase's k_phase
  if (blockIdx.y == 0 && threadIdx.x == 0)
    for (int q = 0; q < nd; ++q) {
      const int slot = de[q].old_slot;
      if (slot >= 0) {  // replaced / dead start versions and recycled versions
        const int top = atomicAdd(&ctl->free_top, 1);
        if (top >= 0 && top < d.pool_cap)
          free_stack[top] = slot;
        else
          set_err(ctl, ERR_POOL_EXHAUSTED);  // never write outside the stack
      } else if (slot != -1) {  // a generated version's entry
        const int top = atomicAdd(&ctl->gv_top, 1);
        if (top >= 0 && top < d.gv_cap)
          d.gv_free[top] = -2 - slot;
        else
          set_err(ctl, ERR_GEN_EXHAUSTED);
      }
    }
}

__global__ void k_commit(Dev d, int color, int ncol, int nreg, int n_slots, const int* diff_cnt,
                         const DiffPair* diff, Ovf ovf, int* free_stack, Ctl* ctl) {
  commit_body(d, color, ncol, nreg, n_slots, diff_cnt, diff, ovf, free_stack, ctl);
}

// block-wide exclusive scan of one int per thread (any block size that is a
// multiple of 32, up to 1024 threads)
__device__ int block_scan_excl(int v, int* total) {
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int s = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  const int excl = x - v + (warp ? ws[warp - 1] : 0);
  *total = ws[(blockDim.x >> 5) - 1];
  __syncthreads();
  return excl;
}

// Event-table rebuild (merge + sort_by_id, samplers.hpp:471-482) without a
// sort: survivors keep their id order, births (ids above every old id,
// increasing with region slot) are appended region by region.
__device__ __forceinline__ void rebuild_body(Table in, Table out, int cap, int stamp,
                                             const int* fate_stamp, const int* fate_alive,
                                             const double* fate_x, const double* fate_t,
                                             const int* fate_slot, int n_slots,
                                             const int* births_cnt, const OutEv* births,
                                             Ovf ovf, Ctl* ctl) {
  const int N = ctl->n_events;
  int base = 0;
  for (int c0 = 0; c0 < N; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    int alive = 0;
    bool touched = false;
    if (i < N) {
      touched = fate_stamp[i] == stamp;
      alive = touched ? fate_alive[i] : 1;
    }
    int tot;
    const int pos = base + block_scan_excl(alive, &tot);
    if (alive) {
      if (pos < cap) {
        out.id[pos] = in.id[i];
        out.x[pos] = touched ? fate_x[i] : in.x[i];
        out.t[pos] = touched ? fate_t[i] : in.t[i];
        out.slot[pos] = touched ? fate_slot[i] : in.slot[i];
      }
    }
    base += tot;
  }
  for (int c0 = 0; c0 < n_slots; c0 += blockDim.x) {
    const int s = c0 + threadIdx.x;
    const int nb = s < n_slots ? births_cnt[s] : 0;
    int tot;
    const int pos = base + block_scan_excl(nb, &tot);
    for (int b = 0; b < nb; ++b) {
      const OutEv& e = births[births_off(ovf, n_slots, s) + b];
      if (pos + b < cap) {
        out.id[pos + b] = e.id;
        out.x[pos + b] = e.x;
        out.t[pos + b] = e.t;
        out.slot[pos + b] = e.slot;
      }
    }
    base += tot;
  }
  if (threadIdx.x == 0) {
    if (base > cap) set_err(ctl, ERR_TABLE_OVERFLOW);
    ctl->n_events = min(base, cap);
    if (ovf.count) *ovf.count = 0;  // the next phase's overflow areas
  }
}

__global__ void __launch_bounds__(1024) k_rebuild(Table in, Table out, int cap, int stamp,
                                                  const int* fate_stamp, const int* fate_alive,
                                                  const double* fate_x, const double* fate_t,
                                                  const int* fate_slot, int n_slots,
                                                  const int* births_cnt, const OutEv* births,
                                                  Ovf ovf, Ctl* ctl) {
  rebuild_body(in, out, cap, stamp, fate_stamp, fate_alive, fate_x, fate_t, fate_slot, n_slots,
               births_cnt, births, ovf, ctl);
}

// The color barrier in one launch: the commit CTAs (grid.x < ncr) and, in the
// last column, one table rebuild CTA. The two touch disjoint state (coverage,
// free stack / next table, n_events), so the rebuild runs beside the commit.
__global__ void __launch_bounds__(kCommitThreads) k_barrier(Dev d, int color, int ncol, int nreg, const int* diff_cnt,
                          const DiffPair* diff, int* free_stack, Ctl* ctl, Table in, Table out,
                          int cap, int stamp, const int* fate_stamp, const int* fate_alive,
                          const double* fate_x, const double* fate_t, const int* fate_slot,
                          int n_slots, const int* births_cnt, const OutEv* births, Ovf ovf) {
  if (blockIdx.x == gridDim.x - 1) {
    if (blockIdx.y == 0)
      rebuild_body(in, out, cap, stamp, fate_stamp, fate_alive, fate_x, fate_t, fate_slot,
                   n_slots, births_cnt, births, ovf, ctl);
    return;
  }
  commit_body(d, color, ncol, nreg, n_slots, diff_cnt, diff, ovf, free_stack, ctl);
}

// ----------------------------------------------------------------- score batch
struct ChangeDev {
  int nr, na;
  unsigned long long rid[2];
  double ax[2], at[2];
  long long arow[2];
  int wlo, whi;
  double slo, shi;
  int sclosed;
  double prior;  // host-computed prior part (reference order)
};

template <typename YT>
__global__ void __launch_bounds__(NT, 1)
    k_score_batch(const Dev d, Table tab, const Ctl* ctl, const ChangeDev* ch,
                  const double* rows, double* out) {
  __shared__ double2 Ts[kTsSize];
  __shared__ Prop P;
  __shared__ double rsig[NW], rarr[NW];
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ChangeDev c = ch[blockIdx.x];
  fill_ts(Ts, d, tid, NT);
  if (tid == 0) {
    s_bad = 0;
    P.type = -1;
    P.skip = 0;
    P.nr = c.nr;
    P.na = c.na;
    const int N = ctl->n_events;
    for (int q = 0; q < c.nr; ++q) {
      int lo = 0, hi = N;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (tab.id[mid] < c.rid[q])
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo >= N || tab.id[lo] != c.rid[q]) {
        s_bad = 2;
        break;
      }
      P.rslot[q] = tab.slot[lo];
      P.rx[q] = tab.x[lo];
      P.rt[q] = tab.t[lo];
    }
    for (int a = 0; a < c.na; ++a) {
      P.ax[a] = c.ax[a];
      P.at[a] = c.at[a];
      const double t = c.at[a];
      if (c.ax[a] < 0.0 || c.ax[a] > d.x_max ||
          !(t >= c.slo && (t < c.shi || (c.sclosed && t == c.shi))))
        s_bad = s_bad ? s_bad : 1;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) out[blockIdx.x] = s_bad == 1 ? -INFINITY : NAN;
    return;
  }
  PassIn in;
  in.src = SRC_ROWS;
  in.rows[0] = rows + (size_t)c.arow[0] * d.S;
  in.rows[1] = rows + (size_t)c.arow[1] * d.S;
  in.wlo = c.wlo;
  in.whi = c.whi;
  in.seed = 0;
  in.sweep = in.region = in.step = 0;
  double sig = 0.0, arr = 0.0;
  int cnt = 0;
  const int T_per = (d.S_pad + 31) / 32;
  DiffW X0;  // no own diff: the batch scores against the resident hypothesis
  X0.nwmax = 0;
  for (int t = warp; t < T_per; t += NW)
    score_item<1, YT, true>(d, P, in, t, 0, nullptr, nullptr, X0, true, Ts, sig, arr, cnt);
  sig = warp_sum(sig);
  arr = warp_sum(arr);
  if (lane == 0) {
    rsig[warp] = sig;
    rarr[warp] = arr;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, A = 0.0;
    for (int w = 0; w < NW; ++w) {
      s += rsig[w];
      A += rarr[w];
    }
    out[blockIdx.x] = c.prior + A + s;
  }
}

// ----------------------------------------------------------------- log_joint
// log_joint (density.hpp:146-154): full-window likelihood over [n][S] plus
// arrival densities; per-block partials reduced in a fixed order.
template <typename YT>
__global__ void k_lj_signal(const Dev d, double* part) {
  __shared__ double sred[32];
  using T2 = typename Y2<YT>::T;
  const T2* y2 = reinterpret_cast<const T2*>(d.y);
  const size_t total = (size_t)d.rows * d.P2;  // station tiles incl. pad rows
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t q = i >> 4;
    const int r = (int)(q % (size_t)d.rows);
    if (r >= d.n) continue;
    const int p = (int)((q / (size_t)d.rows) * 16 + (i & 15));
    const uint32_t w = d.cov[i];
    const T2 yy = y2[i];
    if (2 * p < d.S) {
      const int c = (int)(w & 0xffffu);
      const double y = (double)yy.x;
      acc += d.Lg[c] - y * y * d.Ig[c];
    }
    if (2 * p + 1 < d.S) {
      const int c = (int)(w >> 16);
      const double y = (double)yy.y;
      acc += d.Lg[c] - y * y * d.Ig[c];
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
    part[blockIdx.x] = s;
  }
}

__global__ void k_lj_arrivals(const Dev d, Table tab, const Ctl* ctl, double* part) {
  __shared__ double sred[32];
  const int N = ctl->n_events;
  const size_t total = (size_t)N * d.S;
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / d.S), j = (int)(i % d.S);
    const double a = arr_of(d, tab.slot[e], j);
    acc += arr_logpdf(d, a, arrival_mean(d, tab.x[e], tab.t[e], d.stations[j]));
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sred[w];
    part[blockIdx.x] = s;
  }
}

__global__ void k_lj_final(const Dev d, double lambdaT, const double* logfact, const Ctl* ctl,
                           const double* psig, int nsig, const double* parr, int narr,
                           double* out) {
  if (threadIdx.x != 0) return;
  const int N = ctl->n_events;
  double sig = 0.0, arr = 0.0;
  for (int i = 0; i < nsig; ++i) sig += psig[i];
  for (int i = 0; i < narr; ++i) arr += parr[i];
  // log_event_prior over [0, T] (density.hpp:45-61)
  const double prior =
      -lambdaT + (double)N * d.log_lambda_T - logfact[N] + (double)N * d.lxa;
  *out = prior + arr + sig;
}

__global__ void k_max_id(Table tab, const Ctl* ctl, unsigned long long* out) {
  const int N = ctl->n_events;
  unsigned long long m = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) m = max(m, tab.id[i] + 1);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ unsigned long long s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, s[w]);
    *out = m;
  }
}

__global__ void k_record(const Ctl* ctl, long long* count_out) { *count_out = ctl->n_events; }

// arrivals of hypothesis rows: pool slot rows <-> dense [m][S] (one launch,
// one copy, instead of one copy per event)
__global__ void k_gather_arrivals(const Dev d, const int* slot, int m, double* out) {
  const int e = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.S; j += gridDim.x * blockDim.x)
    out[(size_t)e * d.S + j] = arr_of(d, slot[e], j);  // stored row or generated version
}

// input rows [0, gridDim.y) of a chunk -> their pool slots
__global__ void k_scatter_arrivals(const double* in, const int* slot_of_row, int S, int S_pad,
                                   double* pool) {
  const int row = blockIdx.y;
  const double* src = in + (size_t)row * S;
  double* dst = pool + (size_t)slot_of_row[row] * S_pad;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S_pad; j += gridDim.x * blockDim.x)
    dst[j] = j < S ? src[j] : 0.0;
}

// Trace snapshot (samplers.hpp:430-433): append the event table to the arena
__global__ void k_snapshot(Table tab, const Ctl* ctl, unsigned long long* arena_id,
                           double* arena_x, double* arena_t, long long* arena_top,
                           long long arena_cap, long long* rec) {
  __shared__ long long base;
  const int N = ctl->n_events;
  if (threadIdx.x == 0) {
    base = *arena_top;
    const long long nb = base + N <= arena_cap ? base + N : base;
    *arena_top = nb;
    rec[0] = base;
    rec[1] = nb > base ? N : -1;  // -1: arena full
  }
  __syncthreads();
  if (base + N > arena_cap) return;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    arena_id[base + i] = tab.id[i];
    arena_x[base + i] = tab.x[i];
    arena_t[base + i] = tab.t[i];
  }
}

__global__ void k_reset_counters(Ctl* ctl) {
  ctl->scored = ctl->changed = ctl->arrvals = ctl->accepted = ctl->id_mismatch = 0ull;
  ctl->speculative = 0ull;
  for (int q = 0; q < 8; ++q) ctl->prof[q] = 0ull;
  for (int q = 0; q < 16; ++q) ctl->tprof[q >> 3][q & 7] = 0ull;
  ctl->err = 0;
}

}  // namespace seis

// =================================================================== host side
using namespace seis;

namespace {

thread_local std::string g_err;
// dynamic: the log(i) window + per-lane partial sums (2 double + 1 int per
// speculative slot and thread)
constexpr int kPhaseSmemTile = LOGIWIN * (int)sizeof(double) + MSPEC * NT * (2 * 8 + 4);
// + the per-round diff-window cache of the proposal-major pass (few stations)
constexpr int kPhaseSmem = kPhaseSmemTile + kDiffCache * (int)(sizeof(DiffS) + sizeof(DiffS4x));
// run_serial's chain: + its arrays in place of the diff-window cache (unused)
constexpr int kPhaseSmemSerial = kPhaseSmemTile + ChainSmem<kSerialCap>::bytes;
// tile-major launches: + per-tile flags
constexpr int kPhaseSmemTM = kPhaseSmemTile + kTileFlags;
static_assert(kPhaseSmemTM + 48 * 1024 <= 227 * 1024, "k_phase shared memory");
// The tile-major pass (S_pad >= 2048: 64 station tiles and more) never builds
// the diff-window cache, so its launches leave that shared memory to L1: the
// band rows a warp's proposals share on a tile stay resident between them.
// SEIS_SMEM_FULL=1 keeps the full allocation (A/B).
// The item order of a launch: tile-major (rounds that end at their first
// scored proposal, tile pairs on cached terms) from kTileMajorTiles station
// tiles on; below that the proposal-major pass with speculative rounds spreads
// the few (proposal, tile) items over the warps better. SEIS_TM_MIN_TILES
// overrides the threshold (A/B).
constexpr int kTileMajorTiles = SEIS_TM_TILES;
inline bool tile_major(const Dev& d) {
  static const int min_tiles =
      getenv("SEIS_TM_MIN_TILES") ? atoi(getenv("SEIS_TM_MIN_TILES")) : kTileMajorTiles;
  return (d.S_pad + 31) / 32 >= min_tiles;
}
inline int phase_smem(const Dev& d) {
  static const bool full = getenv("SEIS_SMEM_FULL") && atoi(getenv("SEIS_SMEM_FULL")) == 1;
  const bool dcache = d.dcache_on != 0;
  // tile-major: + one flag byte per station tile
  return (dcache || full) ? kPhaseSmem
                          : kPhaseSmemTile + std::min(kTileFlags, (d.S_pad / 32 + 15) & ~15);
}

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

struct ValidationError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SEIS_OK;
  } catch (const std::invalid_argument& e) {
    return fail(SEIS_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(SEIS_ERUNTIME, e.what());
  }
}

void check_device() {
  int dev = 0, n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw std::runtime_error("no CUDA device: the B200 engine has no CPU fallback");
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw std::runtime_error("engine is built for sm_100a (B200); device is sm_" +
                             std::to_string(prop.major) + std::to_string(prop.minor));
}

// ModelConfig::validate (model.hpp:79-103)
void validate_model(const seis_model_cfg* c, const double* st, int64_t S) {
  auto bad = [](const std::string& m) { throw std::invalid_argument("ModelConfig: " + m); };
  if (!(c->lambda_rate > 0)) bad("lambda_rate must be > 0");
  if (!(c->T > 0)) bad("T must be > 0");
  if (!(c->x_max > 0)) bad("x_max must be > 0");
  if (!(c->v > 0)) bad("v must be > 0");
  if (!(c->sigma_arrival > 0)) bad("sigma_arrival must be > 0");
  if (!(c->t_s > 0)) bad("t_s must be > 0");
  if (!(c->var_noise > 0)) bad("var_noise must be > 0");
  if (!(c->var_event > c->var_noise)) bad("var_event must exceed var_noise");
  if (!(c->sample_rate > 0)) bad("sample_rate must be > 0");
  const double n = c->sample_rate * c->T;
  if (std::abs(n - std::llround(n)) > 1e-9) bad("sample_rate * T must be an integer sample count");
  if (S < 2) bad("need at least 2 stations");
  for (int64_t j = 0; j < S; ++j) {
    if (st[j] < 0 || st[j] > c->x_max) bad("station " + std::to_string(j) + " outside [0, x_max]");
    if (j > 0 && !(st[j - 1] < st[j])) bad("stations must be sorted strictly ascending");
  }
}

}  // namespace

struct seis_engine {
  seis_model_cfg cfg{};
  int S = 0, S_pad = 0, P2 = 0, n = 0, dtype = 0, cap = 0;
  int pool_slots = 0;  // arrival versions: live events + this phase's retired ones
  GenV* gv = nullptr;  // generated versions (spec v2) and their free stack
  int* gv_free = nullptr;
  int gv_cap = 0;
  int compact = 0;     // production births make generated versions
  bool gen_present = false;  // generated versions may be live (cleared by a hypothesis load)
  // the last run's Trace::phases (samplers.hpp:87-95,370,479) and the device
  // time of its trace rows since the run started (TraceRow/Snapshot wall_seconds)
  std::vector<seis_phase_record> phases;
  std::vector<double> row_wall;
  // hypothesis load in pieces (seis_set_hypothesis_begin/_rows/_end)
  int64_t load_n = -1, load_chunk = 0;
  std::vector<int> load_slot_of_row;
  double* load_raw = nullptr;
  int* load_dslot = nullptr;
  cudaStream_t stream = nullptr;
  Dev d{};
  double* stations = nullptr;
  void* y = nullptr;
  uint32_t* cov = nullptr;
  double* tpos = nullptr;  // per-sample term cache (k_terms), valid while terms_valid
  double* tneg = nullptr;
  bool terms_valid = false;
  double* pool = nullptr;
  double* Lg = nullptr;
  double* Ig = nullptr;
  double2* Dg = nullptr;
  double* logi = nullptr;
  double* logfact = nullptr;
  std::vector<double> h_logi, h_logfact;
  Table tab[2]{};
  int cur = 0;
  int* free_stack = nullptr;
  Ctl* ctl = nullptr;
  int* fate_stamp = nullptr;
  int* fate_alive = nullptr;
  double* fate_x = nullptr;
  double* fate_t = nullptr;
  int* fate_slot = nullptr;
  int stamp = 0;
  int n_sm = 148;
  // trace snapshots of the last run (samplers.hpp:80-85,430-433)
  int64_t snap_cap = 0;
  unsigned long long* snap_id = nullptr;
  double* snap_x = nullptr;
  double* snap_t = nullptr;
  long long* snap_top = nullptr;
  long long* snap_rec = nullptr;  // [max_snaps][2] {offset, count}
  int64_t snap_rec_cap = 0;
  std::vector<int64_t> snap_steps;
  // per-call device scratch, kept between calls (one call at a time per
  // engine; every call ends with a stream sync): no cudaMalloc/cudaFree on
  // the run path
  std::vector<std::pair<void*, size_t>> scratch;
  size_t scratch_next = 0;

  ~seis_engine() {
    for (auto& b : scratch) cudaFree(b.first);
    cudaFree(stations);
    cudaFree(y);
    cudaFree(cov);
    cudaFree(tpos);
    cudaFree(tneg);
    cudaFree(pool);
    cudaFree(Lg);
    cudaFree(Ig);
    cudaFree(Dg);
    cudaFree(logi);
    cudaFree(logfact);
    for (auto& t : tab) {
      cudaFree(t.id);
      cudaFree(t.x);
      cudaFree(t.t);
      cudaFree(t.slot);
    }
    cudaFree(free_stack);
    cudaFree(ctl);
    cudaFree(fate_stamp);
    cudaFree(fate_alive);
    cudaFree(fate_x);
    cudaFree(fate_t);
    cudaFree(fate_slot);
    cudaFree(snap_id);
    cudaFree(snap_x);
    cudaFree(snap_t);
    cudaFree(snap_top);
    cudaFree(snap_rec);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

void scratch_reset(seis_engine* e) { e->scratch_next = 0; }

// the next scratch buffer of this call, grown when too small
void* scratch_get(seis_engine* e, size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  const size_t i = e->scratch_next++;
  if (i == e->scratch.size()) e->scratch.push_back({nullptr, 0});
  auto& b = e->scratch[i];
  if (b.second < bytes) {
    if (b.first) cudaFree(b.first);
    b.first = nullptr;
    b.second = 0;
    ck(cudaMalloc(&b.first, bytes), "cudaMalloc scratch");
    b.second = bytes;
  }
  return b.first;
}

template <typename T>
T* scratch_of(seis_engine* e, size_t n) {
  return static_cast<T*>(scratch_get(e, n * sizeof(T)));
}

void upload_signals(seis_engine* e, const void* signals) {
  const size_t esz = e->dtype == SEIS_F64 ? 8 : 4;
  e->terms_valid = false;
  scratch_reset(e);
  void* tmp = scratch_get(e, (size_t)e->S * e->n * esz);
  ck(cudaMemcpyAsync(tmp, signals, (size_t)e->S * e->n * esz, cudaMemcpyHostToDevice, e->stream),
     "H2D signals");
  dim3 grid((e->n + 31) / 32, (e->S_pad + 31) / 32), block(32, 8);
  if (e->dtype == SEIS_F64)
    k_transpose<double><<<grid, block, 0, e->stream>>>(static_cast<const double*>(tmp),
                                                       static_cast<double*>(e->y), e->S,
                                                       e->S_pad, e->n, e->n + kRowPad);
  else
    k_transpose<float><<<grid, block, 0, e->stream>>>(static_cast<const float*>(tmp),
                                                      static_cast<float*>(e->y), e->S, e->S_pad,
                                                      e->n, e->n + kRowPad);
  ck(cudaGetLastError(), "k_transpose");
  ck(cudaStreamSynchronize(e->stream), "sync");
}

Ctl read_ctl(seis_engine* e) {
  Ctl c;
  ck(cudaMemcpyAsync(&c, e->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, e->stream), "D2H ctl");
  ck(cudaStreamSynchronize(e->stream), "sync");
  return c;
}

const char* err_name(int e) {
  switch (e) {
    case ERR_OWN_OVERFLOW: return "a region chain exceeded 1024 events (the per-chain event limit)";
    case ERR_POOL_EXHAUSTED: return "arrival pool exhausted (live events + replaced versions > pool slots): raise event_capacity";
    case ERR_TAPE_UNKNOWN_ID: return "replay tape names an event the region does not hold";
    case ERR_TABLE_OVERFLOW: return "event table overflow: raise event_capacity";
    case ERR_GEN_EXHAUSTED: return "generated-version table exhausted (raise event_capacity)";
    case ERR_COUNT_OVERFLOW: return "more than 65535 events cover one (sample, station): uint16 coverage count overflow";
    default: return "device error";
  }
}

template <typename YT>
void launch_lj(seis_engine* e, double* out_dev, double* scratch) {
  const int nb = 296;
  k_lj_signal<YT><<<nb, 256, 0, e->stream>>>(e->d, scratch);
  k_lj_arrivals<<<nb, 256, 0, e->stream>>>(e->d, e->tab[e->cur], e->ctl, scratch + nb);
  k_lj_final<<<1, 32, 0, e->stream>>>(e->d, e->cfg.lambda_rate * e->cfg.T, e->logfact, e->ctl,
                                       scratch, nb, scratch + nb, nb, out_dev);
}

void launch_lj_any(seis_engine* e, double* out_dev, double* scratch) {
  if (e->dtype == SEIS_F64)
    launch_lj<double>(e, out_dev, scratch);
  else
    launch_lj<float>(e, out_dev, scratch);
}

}  // namespace

namespace {
// One 512-thread CTA per region. Measured on configs 1 and 2: 256-thread
// CTAs two or three per SM lose (1.44 M and 1.21 M vs 1.72 M proposals/s at
// config[2]): a chain's rounds slow down more than sharing an SM gains.
// Variants: the row-only production kernel (GEN = false) when the engine
// holds no generated versions and makes none (the default storage); every
// other launch (compact storage, replay, the serial chain) handles both kinds.
// the term cache follows every change of the counts or the signals: rebuilt
// before the first phase that reads them (returns the launches it made)
int refresh_terms(seis_engine* e) {
  if (!e->tpos || e->terms_valid) return 0;
  const int grid = e->n_sm * 8;
  if (e->dtype == SEIS_F64)
    k_terms<double><<<grid, 512, 0, e->stream>>>(e->d, e->tpos, e->tneg);
  else
    k_terms<float><<<grid, 512, 0, e->stream>>>(e->d, e->tpos, e->tneg);
  ck(cudaGetLastError(), "k_terms");
  e->terms_valid = true;
  return 1;
}

template <typename YT, int MODE, bool TM>
void launch_phase_tm(seis_engine* e, int ncr, const Samp& sp, const PhaseArgs& pa, int stamp) {
  const bool rows_only = MODE == 0 && !pa.serial && !e->compact && !e->gen_present;
#ifdef SEIS_FAST_BUILD  // development builds: the fp32 row-only production kernels alone
  if constexpr (std::is_same<YT, float>::value && MODE == 0) {
    if (rows_only && !pa.retry_pass)
      phase_launch<float, 0, MAXOWN, false, TM>(ncr, phase_smem(e->d), e->stream, e->d, sp, pa,
                                                e->ctl, stamp);
    else if (!pa.retry_pass)
      throw std::runtime_error("SEIS_FAST_BUILD: kernel variant not built");
  } else {
    throw std::runtime_error("SEIS_FAST_BUILD: kernel variant not built");
  }
#else
  if (pa.serial || pa.retry_pass)
    phase_launch<YT, MODE, kSerialCap, true, TM>(ncr, kPhaseSmemSerial, e->stream, e->d, sp, pa,
                                                 e->ctl, stamp);
  else if (MODE == 0 && rows_only)
    phase_launch<YT, 0, MAXOWN, false, TM>(ncr, phase_smem(e->d), e->stream, e->d, sp, pa, e->ctl,
                                           stamp);
  else
    phase_launch<YT, MODE, MAXOWN, true, TM>(ncr, phase_smem(e->d), e->stream, e->d, sp, pa,
                                             e->ctl, stamp);
#endif
  if (MODE == 0 && e->compact) e->gen_present = true;
}

template <typename YT, int MODE>
void launch_phase_t(seis_engine* e, int ncr, const Samp& sp, const PhaseArgs& pa, int stamp) {
  if (tile_major(e->d))
    launch_phase_tm<YT, MODE, true>(e, ncr, sp, pa, stamp);
  else
    launch_phase_tm<YT, MODE, false>(e, ncr, sp, pa, stamp);
}

void launch_phase(seis_engine* e, int mode, int ncr, const Samp& sp, const PhaseArgs& pa,
                  int stamp) {
  if (e->dtype == SEIS_F64) {
    if (mode == 0)
      launch_phase_t<double, 0>(e, ncr, sp, pa, stamp);
    else
      launch_phase_t<double, 1>(e, ncr, sp, pa, stamp);
  } else {
    if (mode == 0)
      launch_phase_t<float, 0>(e, ncr, sp, pa, stamp);
    else
      launch_phase_t<float, 1>(e, ncr, sp, pa, stamp);
  }
}

template <typename YT, int MODE, bool TM>
void set_phase_attrs_tm() {
#ifdef SEIS_FAST_BUILD
  if constexpr (std::is_same<YT, float>::value && MODE == 0)
    ck(phase_set_smem<float, 0, MAXOWN, false, TM>(TM ? std::max(kPhaseSmem, kPhaseSmemTM) : kPhaseSmem), "smem attribute");
#else
  ck(phase_set_smem<YT, MODE, MAXOWN, true, TM>(TM ? std::max(kPhaseSmem, kPhaseSmemTM) : kPhaseSmem), "smem attribute");
  if (MODE == 0) ck(phase_set_smem<YT, 0, MAXOWN, false, TM>(TM ? std::max(kPhaseSmem, kPhaseSmemTM) : kPhaseSmem), "smem attribute");
  ck(phase_set_smem<YT, MODE, kSerialCap, true, TM>(kPhaseSmemSerial), "smem attribute");
#endif
}
template <typename YT, int MODE>
void set_phase_attrs() {
  set_phase_attrs_tm<YT, MODE, true>();
  set_phase_attrs_tm<YT, MODE, false>();
}
}  // namespace

extern "C" {

const char* seis_last_error(void) { return g_err.c_str(); }

int seis_engine_create(const seis_model_cfg* cfg, const double* stations, int64_t n_stations,
                       const void* signals, int32_t dtype, int64_t event_capacity,
                       seis_engine** out) {
  *out = nullptr;
  seis_engine* e = nullptr;
  const int rc = guarded([&] {
    validate_model(cfg, stations, n_stations);
    if (dtype != SEIS_F32 && dtype != SEIS_F64) throw std::invalid_argument("dtype must be F32 or F64");
    if (event_capacity < 1 || event_capacity > kMaxEvents)
      throw std::invalid_argument("event_capacity must be in [1, 4194304]");
    check_device();
    e = new seis_engine;
    e->cfg = *cfg;
    e->S = (int)n_stations;
    e->S_pad = (int)((n_stations + 63) / 64 * 64);
    e->P2 = e->S_pad / 2;
    e->n = (int)std::llround(cfg->sample_rate * cfg->T);
    e->dtype = dtype;
    e->cap = (int)event_capacity;
    ck(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "stream");
    std::vector<double> st(e->S_pad, 0.0);
    std::copy(stations, stations + n_stations, st.begin());
    e->stations = dalloc<double>(e->S_pad);
    ck(cudaMemcpy(e->stations, st.data(), st.size() * 8, cudaMemcpyHostToDevice), "H2D");
    const size_t esz = dtype == SEIS_F64 ? 8 : 4;
    // kRowPad zero rows after the last sample: band loops load whole row
    // chunks without a bounds predicate
    ck(cudaMalloc(&e->y, (size_t)(e->n + kRowPad) * e->S_pad * esz), "cudaMalloc y");
    ck(cudaMemset(e->y, 0, (size_t)(e->n + kRowPad) * e->S_pad * esz), "memset");
    e->cov = dalloc<uint32_t>((size_t)(e->n + kRowPad) * e->P2);
    ck(cudaMemset(e->cov, 0, (size_t)(e->n + kRowPad) * e->P2 * 4), "memset");
    // SEIS_TERMS=0 runs without the term cache (A/B, and the parity suite's
    // second pass over the direct band)
    if (!(getenv("SEIS_TERMS") && atoi(getenv("SEIS_TERMS")) == 0)) {
      const size_t tn = (size_t)(e->n + kRowPad) * e->S_pad;
      e->tpos = dalloc<double>(tn);
      e->tneg = dalloc<double>(tn);
      ck(cudaMemset(e->tpos, 0, tn * 8), "memset");
      ck(cudaMemset(e->tneg, 0, tn * 8), "memset");
    }
    // arrival pool: a phase holds every live event plus the phase-start
    // versions it replaced or killed (freed at the barrier) -> about twice
    // the live events; bounded by what fits in HBM beside the other buffers
    {
      size_t free_b = 0, total_b = 0;
      ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      const size_t per = (size_t)e->S_pad * 8;
      // leave room for the tables, the per-launch scratch and other users
      const size_t reserve = std::max<size_t>((size_t)6 << 30, total_b / 16);
      const size_t fit = free_b > reserve ? (free_b - reserve) / per : 0;
      const size_t want = 2 * (size_t)e->cap + 2048;
      // may hold fewer rows than event_capacity: the engine then defaults to
      // the compact storage (generated versions need no row)
      size_t slots = std::max<size_t>(std::min<size_t>(want, fit), std::min<size_t>(want, 64));
      // SEIS_POOL_SLOTS (tests): a smaller pool, to exercise exhaustion
      if (const char* ov = getenv("SEIS_POOL_SLOTS"))
        slots = std::max<size_t>(1, std::min<size_t>(slots, (size_t)atoll(ov)));
      void* p = nullptr;
      while (cudaMalloc(&p, slots * per) != cudaSuccess) {
        (void)cudaGetLastError();
        if (slots <= 64) throw std::runtime_error("cudaMalloc: arrival pool out of memory");
        slots -= slots / 8;
      }
      e->pool_slots = (int)slots;
      e->pool = static_cast<double*>(p);
    }
    // per-count terms with glibc log, exactly as density.hpp:288-297; counts
    // are uint16 (<= 65535) plus at most 2 * MAXOWN in-phase own versions
    const int tab_n = std::min(e->cap, 65535) + 2 * kSerialCap + 8;
    std::vector<double> L(tab_n), I(tab_n);
    for (int c = 0; c < tab_n; ++c) {
      const double var = cfg->var_noise + c * cfg->var_event;
      L[c] = -0.5 * (kLog2Pi + std::log(var));
      I[c] = 0.5 / var;
    }
    std::vector<double2> Dt((size_t)tab_n * 4);
    const int dcs[4] = {-2, -1, 1, 2};
    for (int c = 0; c < tab_n; ++c)
      for (int k = 0; k < 4; ++k) {
        const int cn = c + dcs[k];
        Dt[(size_t)c * 4 + k] = (cn >= 0 && cn < tab_n)
                                    ? make_double2(L[cn] - L[c], I[cn] - I[c])
                                    : make_double2(0.0, 0.0);
      }
    e->Dg = dalloc<double2>((size_t)tab_n * 4);
    ck(cudaMemcpy(e->Dg, Dt.data(), Dt.size() * sizeof(double2), cudaMemcpyHostToDevice), "H2D");
    e->Lg = dalloc<double>(tab_n);
    e->Ig = dalloc<double>(tab_n);
    ck(cudaMemcpy(e->Lg, L.data(), tab_n * 8, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(e->Ig, I.data(), tab_n * 8, cudaMemcpyHostToDevice), "H2D");
    // log i and log i! for event counts: the live events plus a region's births
    const int logi_n = e->cap + 2 * kSerialCap + 8;
    e->h_logi.resize(logi_n);
    e->h_logfact.resize(logi_n);
    double acc = 0.0;
    for (int i = 0; i < logi_n; ++i) {
      e->h_logi[i] = i > 0 ? std::log(static_cast<double>(i)) : -INFINITY;
      if (i >= 2) acc += std::log(static_cast<double>(i));  // log_factorial, density.hpp:21-25
      e->h_logfact[i] = acc;
    }
    e->logi = dalloc<double>(logi_n);
    e->logfact = dalloc<double>(logi_n);
    ck(cudaMemcpy(e->logi, e->h_logi.data(), logi_n * 8, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(e->logfact, e->h_logfact.data(), logi_n * 8, cudaMemcpyHostToDevice), "H2D");
    for (auto& t : e->tab) {
      t.id = dalloc<unsigned long long>(e->cap);
      t.x = dalloc<double>(e->cap);
      t.t = dalloc<double>(e->cap);
      t.slot = dalloc<int>(e->cap);
    }
    e->free_stack = dalloc<int>(e->pool_slots);
    // generated versions (spec v2): four entries per event of capacity; the
    // compact storage is on by default when the pool cannot hold two stored
    // rows per event (seis_set_arrival_storage overrides)
    e->gv_cap = (int)std::min<int64_t>((int64_t)4 * e->cap + 4096, (int64_t)1 << 26);
    e->gv = dalloc<GenV>(e->gv_cap);
    e->gv_free = dalloc<int>(e->gv_cap);
    e->compact = e->pool_slots < 2 * e->cap ? 1 : 0;
    e->ctl = dalloc<Ctl>(1);
    e->fate_stamp = dalloc<int>(e->cap);
    ck(cudaMemset(e->fate_stamp, 0, e->cap * 4), "memset");
    e->fate_alive = dalloc<int>(e->cap);
    e->fate_x = dalloc<double>(e->cap);
    e->fate_t = dalloc<double>(e->cap);
    e->fate_slot = dalloc<int>(e->cap);
    Dev& d = e->d;
    d.S = e->S;
    d.S_pad = e->S_pad;
    d.rows = e->n + kRowPad;
    d.P2 = e->P2;
    d.n = e->n;
    d.rate = cfg->sample_rate;
    d.t_s = cfg->t_s;
    d.v = cfg->v;
    d.sigma = cfg->sigma_arrival;
    d.x_max = cfg->x_max;
    d.T = cfg->T;
    const double var_a = cfg->sigma_arrival * cfg->sigma_arrival;
    d.c0_arr = -0.5 * (kLog2Pi + std::log(var_a));
    d.inv_twovar_arr = 1.0 / (2.0 * var_a);
    d.twovar_arr = 2.0 * var_a;
    d.inv_v = 1.0 / cfg->v;
    d.log_lambda_T = std::log(cfg->lambda_rate * cfg->T);
    d.lxa = -std::log(cfg->x_max) - std::log(cfg->T);
    d.log_xmax = std::log(cfg->x_max);
    d.stations = e->stations;
    d.y = e->y;
    d.cov = e->cov;
    d.tpos = e->tpos;
    d.tneg = e->tneg;
    d.pool = e->pool;
    d.Lg = e->Lg;
    d.Ig = e->Ig;
    d.Dg = e->Dg;
    d.tab_n = tab_n;
    d.logi = e->logi;
    d.logi_n = logi_n;
    d.pool_cap = e->pool_slots;
    d.gv = e->gv;
    d.gv_free = e->gv_free;
    d.gv_cap = e->gv_cap;
    d.dcache_on = (!tile_major(d) && d.S_pad <= kDiffCache && d.n < 65535) ? 1 : 0;
    set_phase_attrs<float, 0>();
    set_phase_attrs<float, 1>();
    set_phase_attrs<double, 0>();
    set_phase_attrs<double, 1>();
    int dev = 0;
    ck(cudaGetDevice(&dev), "device");
    ck(cudaDeviceGetAttribute(&e->n_sm, cudaDevAttrMultiProcessorCount, dev), "sm count");
    upload_signals(e, signals);
  });
  if (rc) {
    delete e;
    return rc;
  }
  // start from the empty hypothesis (samplers.hpp:409)
  const int rc2 = seis_set_hypothesis(e, 0, nullptr, nullptr, nullptr, nullptr);
  if (rc2) {
    delete e;
    return rc2;
  }
  *out = e;
  return SEIS_OK;
}

void seis_engine_destroy(seis_engine* eng) { delete eng; }

int64_t seis_engine_pool_slots(const seis_engine* eng) { return eng ? eng->pool_slots : 0; }

int seis_upload_signals(seis_engine* e, const void* signals) {
  return guarded([&] { upload_signals(e, signals); });
}

// Hypothesis load in pieces (seis_set_hypothesis = begin + rows + end): the
// table in id order (the reference's World::events after sort_by_id), slot i
// for the i-th smallest id, arrival rows scattered to their slots through a
// <= 512 MiB device staging buffer, then the coverage counts.
namespace {
int hyp_begin(seis_engine* e, int64_t N, const uint64_t* ids, const double* x, const double* t) {
  return guarded([&] {
    e->load_n = -1;
    if (N < 0 || N > e->cap) throw std::invalid_argument("hypothesis larger than event_capacity");
    if (N > e->pool_slots)
      throw std::invalid_argument("hypothesis rows exceed the arrival pool (" +
                                  std::to_string(e->pool_slots) + " rows fit in HBM)");
    std::vector<int64_t> order(N);
    for (int64_t i = 0; i < N; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return ids[a] < ids[b]; });
    for (int64_t i = 1; i < N; ++i)
      if (ids[order[i]] == ids[order[i - 1]]) throw std::invalid_argument("duplicate event id");
    std::vector<unsigned long long> hid(N);
    std::vector<double> hx(N), ht(N);
    std::vector<int> hs(N), fs(e->pool_slots);
    e->load_slot_of_row.assign(N, 0);
    for (int64_t i = 0; i < N; ++i) {
      const int64_t k = order[i];
      hid[i] = ids[k];
      hx[i] = x[k];
      ht[i] = t[k];
      hs[i] = (int)i;
      e->load_slot_of_row[k] = (int)i;  // input row k goes to slot i
    }
    // free stack: slots N..pool_slots-1 (top of stack = lowest)
    int nf = 0;
    for (int s2 = e->pool_slots - 1; s2 >= (int)N; --s2) fs[nf++] = s2;
    e->cur = 0;
    Table& tb = e->tab[0];
    scratch_reset(e);
    e->load_chunk = std::max<int64_t>(
        1, std::min<int64_t>({std::max<int64_t>(N, 1), ((int64_t)512 << 20) / ((int64_t)e->S * 8),
                              65535}));
    e->load_raw = scratch_of<double>(e, (size_t)e->load_chunk * e->S);
    e->load_dslot = scratch_of<int>(e, std::max<int64_t>(N, 1));
    if (N) {
      // stream-ordered copies from pageable vectors (each returns once staged)
      ck(cudaMemcpyAsync(tb.id, hid.data(), N * 8, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(tb.x, hx.data(), N * 8, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(tb.t, ht.data(), N * 8, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(tb.slot, hs.data(), N * 4, cudaMemcpyHostToDevice, e->stream), "H2D");
      ck(cudaMemcpyAsync(e->load_dslot, e->load_slot_of_row.data(), (size_t)N * 4,
                         cudaMemcpyHostToDevice, e->stream),
         "H2D");
    }
    if (nf)
      ck(cudaMemcpyAsync(e->free_stack, fs.data(), (size_t)nf * 4, cudaMemcpyHostToDevice,
                         e->stream),
         "H2D");
    e->gen_present = false;
    e->terms_valid = false;
    // every generated-version entry free (a loaded hypothesis is stored rows)
    {
      std::vector<int> gf(e->gv_cap);
      for (int g = 0; g < e->gv_cap; ++g) gf[g] = e->gv_cap - 1 - g;  // top of stack = 0
      ck(cudaMemcpyAsync(e->gv_free, gf.data(), (size_t)e->gv_cap * 4, cudaMemcpyHostToDevice,
                         e->stream),
         "H2D");
    }
    Ctl c{};
    c.n_events = (int)N;
    c.free_top = nf;
    c.gv_top = e->gv_cap;
    ck(cudaMemcpyAsync(e->ctl, &c, sizeof c, cudaMemcpyHostToDevice, e->stream), "H2D");
    ck(cudaMemsetAsync(e->cov, 0, (size_t)(e->n + kRowPad) * e->P2 * 4, e->stream), "memset");
    // (pageable sources: each copy returned once its data was staged)
    e->load_n = N;
  });
}

int hyp_rows(seis_engine* e, int64_t i0, int64_t n, const double* arrivals, bool sync) {
  return guarded([&] {
    if (e->load_n < 0) throw std::invalid_argument("seis_set_hypothesis_rows without _begin");
    if (i0 < 0 || n < 0 || i0 + n > e->load_n)
      throw std::invalid_argument("arrival rows outside the hypothesis");
    for (int64_t r0 = 0; r0 < n; r0 += e->load_chunk) {
      const int64_t nr = std::min(e->load_chunk, n - r0);
      ck(cudaMemcpyAsync(e->load_raw, arrivals + (size_t)r0 * e->S, (size_t)nr * e->S * 8,
                         cudaMemcpyHostToDevice, e->stream),
         "H2D arrivals");
      dim3 grid((unsigned)std::min(64, (e->S_pad + 255) / 256), (unsigned)nr);
      k_scatter_arrivals<<<grid, 256, 0, e->stream>>>(e->load_raw, e->load_dslot + i0 + r0, e->S,
                                                      e->S_pad, e->pool);
      ck(cudaGetLastError(), "k_scatter_arrivals");
    }
    // the caller may reuse its (possibly pinned) buffer after the call
    if (sync) ck(cudaStreamSynchronize(e->stream), "sync");
  });
}
}  // namespace

int seis_set_hypothesis_begin(seis_engine* e, int64_t N, const uint64_t* ids, const double* x,
                              const double* t) {
  return hyp_begin(e, N, ids, x, t);
}

int seis_set_hypothesis_rows(seis_engine* e, int64_t i0, int64_t n, const double* arrivals) {
  return hyp_rows(e, i0, n, arrivals, true);
}

int seis_set_hypothesis_end(seis_engine* e) {
  bool cov_failed = false;
  const int rc = guarded([&] {
    if (e->load_n < 0) throw std::invalid_argument("seis_set_hypothesis_end without _begin");
    const int64_t N = e->load_n;
    e->load_n = -1;
    if (N) {
      dim3 grid((e->P2 + 127) / 128, (unsigned)std::min<int64_t>(N, 65535));
      k_build_cov<<<grid, 128, 0, e->stream>>>(e->d, e->tab[0], e->ctl);
      ck(cudaGetLastError(), "k_build_cov");
    }
    const Ctl after = read_ctl(e);  // the one synchronisation of the call
    if (after.err) {
      cov_failed = true;
      throw std::runtime_error(std::string("device: ") + err_name(after.err));
    }
  });
  if (rc && cov_failed) {  // leave the engine empty rather than half-loaded
    const std::string msg = g_err;
    seis_set_hypothesis(e, 0, nullptr, nullptr, nullptr, nullptr);
    g_err = msg;
  }
  return rc;
}

int seis_set_hypothesis(seis_engine* e, int64_t N, const uint64_t* ids, const double* x,
                        const double* t, const double* arrivals) {
  // one synchronisation for the whole call (in _end)
  int rc = hyp_begin(e, N, ids, x, t);
  if (rc == SEIS_OK && N > 0) rc = hyp_rows(e, 0, N, arrivals, false);
  if (rc == SEIS_OK) return seis_set_hypothesis_end(e);
  e->load_n = -1;
  return rc;
}

int seis_get_hypothesis(seis_engine* e, int64_t cap, int64_t* n, uint64_t* ids, double* x,
                        double* t, double* arrivals) {
  return guarded([&] {
    const Ctl c = read_ctl(e);
    *n = c.n_events;
    const int64_t m = std::min<int64_t>(cap, c.n_events);
    if (m <= 0) return;
    const Table& tb = e->tab[e->cur];
    ck(cudaMemcpyAsync(ids, tb.id, m * 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaMemcpyAsync(x, tb.x, m * 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaMemcpyAsync(t, tb.t, m * 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    if (arrivals) {  // in chunks of <= 512 MiB
      const int64_t chunk = std::max<int64_t>(
          1, std::min<int64_t>({m, ((int64_t)512 << 20) / ((int64_t)e->S * 8), 65535}));
      scratch_reset(e);
      double* buf = scratch_of<double>(e, (size_t)chunk * e->S);
      for (int64_t r0 = 0; r0 < m; r0 += chunk) {
        const int64_t nr = std::min(chunk, m - r0);
        dim3 grid((unsigned)std::min(64, (e->S + 255) / 256), (unsigned)nr);
        k_gather_arrivals<<<grid, 256, 0, e->stream>>>(e->d, tb.slot + r0,
                                                       (int)nr, buf);
        ck(cudaGetLastError(), "k_gather_arrivals");
        ck(cudaMemcpyAsync(arrivals + (size_t)r0 * e->S, buf, (size_t)nr * e->S * 8,
                           cudaMemcpyDeviceToHost, e->stream),
           "D2H arrivals");
      }
    }
    ck(cudaStreamSynchronize(e->stream), "sync");
  });
}

int seis_set_snapshot_capacity(seis_engine* e, int64_t max_events, int64_t max_snapshots) {
  return guarded([&] {
    if (max_events < 0 || max_snapshots < 0) throw std::invalid_argument("negative capacity");
    cudaFree(e->snap_id);
    cudaFree(e->snap_x);
    cudaFree(e->snap_t);
    cudaFree(e->snap_top);
    cudaFree(e->snap_rec);
    e->snap_id = nullptr;
    e->snap_x = e->snap_t = nullptr;
    e->snap_top = e->snap_rec = nullptr;
    e->snap_cap = max_events;
    e->snap_rec_cap = max_snapshots;
    e->snap_steps.clear();
    if (max_events == 0 || max_snapshots == 0) {
      e->snap_cap = 0;
      return;
    }
    e->snap_id = dalloc<unsigned long long>(max_events);
    e->snap_x = dalloc<double>(max_events);
    e->snap_t = dalloc<double>(max_events);
    e->snap_top = dalloc<long long>(1);
    e->snap_rec = dalloc<long long>(2 * max_snapshots);
  });
}

int seis_get_snapshots(seis_engine* e, int64_t cap_snap, int64_t* n_snap, int64_t* snap_step,
                       int64_t* snap_count, int64_t cap_ev, uint64_t* ids, double* x, double* t) {
  return guarded([&] {
    const int64_t ns = (int64_t)e->snap_steps.size();
    *n_snap = ns;
    if (ns == 0 || cap_snap <= 0) return;
    std::vector<long long> rec(2 * ns);
    ck(cudaMemcpy(rec.data(), e->snap_rec, rec.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    int64_t total = 0;
    for (int64_t i = 0; i < ns && i < cap_snap; ++i) {
      if (rec[2 * i + 1] < 0) throw std::runtime_error("snapshot arena full: raise max_events");
      snap_step[i] = e->snap_steps[i];
      snap_count[i] = rec[2 * i + 1];
      total = std::max<int64_t>(total, rec[2 * i] + rec[2 * i + 1]);
    }
    if (!ids) return;  // steps and counts only
    if (total > cap_ev) throw std::invalid_argument("event buffer too small for the snapshots");
    if (total > 0) {
      ck(cudaMemcpy(ids, e->snap_id, total * 8, cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(x, e->snap_x, total * 8, cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(t, e->snap_t, total * 8, cudaMemcpyDeviceToHost), "D2H");
    }
  });
}

int seis_set_arrival_storage(seis_engine* e, int32_t mode) {
  return guarded([&] {
    if (mode != SEIS_ARR_ROWS && mode != SEIS_ARR_COMPACT)
      throw std::invalid_argument("arrival storage must be SEIS_ARR_ROWS or SEIS_ARR_COMPACT");
    e->compact = mode == SEIS_ARR_COMPACT ? 1 : 0;
  });
}

int32_t seis_get_arrival_storage(const seis_engine* e) {
  return e && e->compact ? SEIS_ARR_COMPACT : SEIS_ARR_ROWS;
}

int seis_get_phases(seis_engine* e, int64_t cap, int64_t* n, seis_phase_record* out) {
  return guarded([&] {
    const int64_t np = (int64_t)e->phases.size();
    *n = np;
    for (int64_t i = 0; i < np && i < cap; ++i) out[i] = e->phases[i];
  });
}

int seis_get_row_wall(seis_engine* e, int64_t cap, int64_t* n, double* wall_seconds) {
  return guarded([&] {
    const int64_t nr = (int64_t)e->row_wall.size();
    *n = nr;
    for (int64_t i = 0; i < nr && i < cap; ++i) wall_seconds[i] = e->row_wall[i];
  });
}

int seis_partition(double T, double l, double offset, double tau, int64_t cap,
                   int64_t* n_regions, double* boundaries, int32_t* colors, int32_t* n_colors) {
  return guarded([&] {
    // argument validation of build_partition / color_partition (partition.hpp:41-46,67-78)
    if (!(T > 0)) throw std::invalid_argument("build_partition: T must be > 0");
    if (!(l > 0) || l > T) throw std::invalid_argument("build_partition: need 0 < l <= T");
    if (offset < 0 || offset >= l)
      throw std::invalid_argument("build_partition: need 0 <= offset < l");
    if (!(tau >= 0)) throw std::invalid_argument("color_partition: tau_max must be >= 0");
    int k;
    if (l >= tau)
      k = 2;
    else if (l >= tau / 2)
      k = 3;
    else
      throw std::invalid_argument("color_partition: region length is below tau_max/2");
    check_device();
    const int bcap = (int)std::min<int64_t>(cap, (int64_t)(T / l) + 8);
    double* b = dalloc<double>(bcap);
    int* nr = dalloc<int>(1);
    int* err = dalloc<int>(1);
    ck(cudaMemset(err, 0, 4), "memset");
    // offset passed explicitly: epoch-0 static path with the given u
    int* col = dalloc<int>(bcap);
    k_partition<<<1, kPartThreads>>>(T, l, tau, k, 2, 0, 0, 1, offset, bcap, b, nr, err, col);
    ck(cudaGetLastError(), "k_partition");
    int h_nr = 0, h_err = 0;
    ck(cudaMemcpy(&h_nr, nr, 4, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(&h_err, err, 4, cudaMemcpyDeviceToHost), "D2H");
    if (h_err == 2) throw std::runtime_error("partition capacity");
    *n_regions = h_nr;
    if (h_nr + 1 > cap) throw std::runtime_error("partition capacity");
    ck(cudaMemcpy(boundaries, b, (size_t)(h_nr + 1) * 8, cudaMemcpyDeviceToHost), "D2H");
    std::vector<int> hc(h_nr);
    ck(cudaMemcpy(hc.data(), col, (size_t)h_nr * 4, cudaMemcpyDeviceToHost), "D2H");
    for (int i = 0; i < h_nr; ++i) colors[i] = hc[i];
    *n_colors = k;
    cudaFree(col);
    cudaFree(b);
    cudaFree(nr);
    cudaFree(err);
    if (h_err == 1) throw std::logic_error("color_partition: separation invariant violated");
  });
}

int seis_assign_regions(const double* boundaries, int64_t n_regions, int64_t m, const double* t,
                        int64_t* region_out) {
  return guarded([&] {
    check_device();
    if (n_regions < 1) throw std::invalid_argument("need at least one region");
    double* b = dalloc<double>(n_regions + 1);
    double* dt = dalloc<double>(m);
    int64_t* o = dalloc<int64_t>(m);
    ck(cudaMemcpy(b, boundaries, (n_regions + 1) * 8, cudaMemcpyHostToDevice), "H2D");
    if (m) ck(cudaMemcpy(dt, t, m * 8, cudaMemcpyHostToDevice), "H2D");
    if (m) k_region_of<<<(unsigned)((m + 255) / 256), 256>>>(b, (int)n_regions, m, dt, o);
    ck(cudaGetLastError(), "k_region_of");
    if (m) ck(cudaMemcpy(region_out, o, m * 8, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(b);
    cudaFree(dt);
    cudaFree(o);
  });
}

int seis_partition_offset(uint64_t seed, int64_t epoch, double l, double* u_out) {
  return guarded([&] {
    check_device();
    double* o = dalloc<double>(1);
    k_offsets<<<1, 1>>>(seed, epoch, l, o);
    ck(cudaGetLastError(), "k_offsets");
    ck(cudaMemcpy(u_out, o, 8, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(o);
  });
}

int seis_score_batch(seis_engine* e, int64_t n_changes, const seis_change* changes,
                     const double* added_arrivals, int64_t n_rows, double* delta_out) {
  return guarded([&] {
    if (n_changes == 0) return;
    const Ctl c = read_ctl(e);
    const int64_t N = c.n_events;
    std::vector<ChangeDev> hc(n_changes);
    for (int64_t i = 0; i < n_changes; ++i) {
      const seis_change& s = changes[i];
      if (s.n_removed < 0 || s.n_removed > 2 || s.n_added < 0 || s.n_added > 2)
        throw std::invalid_argument("a change holds at most 2 removed and 2 added events");
      ChangeDev& h = hc[i];
      h.nr = s.n_removed;
      h.na = s.n_added;
      for (int q = 0; q < 2; ++q) {
        h.rid[q] = s.removed_id[q];
        h.ax[q] = s.added_x[q];
        h.at[q] = s.added_t[q];
        h.arow[q] = q < s.n_added ? s.added_row[q] : 0;
        if (q < s.n_added && (s.added_row[q] < 0 || s.added_row[q] >= n_rows))
          throw std::invalid_argument("added_row out of range");
      }
      h.wlo = (int)std::max<int64_t>(0, s.window_lo);
      h.whi = (int)std::min<int64_t>(e->n, s.window_hi);
      h.slo = s.support_lo;
      h.shi = s.support_hi;
      h.sclosed = s.support_closed;
      // prior part of delta_log_joint (density.hpp:223-237), glibc log
      const int64_t n0 = N, n1 = n0 - s.n_removed + s.n_added;
      const double area = s.support_hi - s.support_lo;
      const double lla = std::log(e->cfg.lambda_rate * area);
      double delta = 0.0;
      if (n1 > n0) {
        for (int64_t k = n0 + 1; k <= n1; ++k) delta += lla - std::log(static_cast<double>(k));
      } else if (n1 < n0) {
        for (int64_t k = n1 + 1; k <= n0; ++k) delta -= lla - std::log(static_cast<double>(k));
      }
      delta += static_cast<double>(n1 - n0) * (-std::log(e->cfg.x_max) - std::log(area));
      h.prior = delta;
    }
    ChangeDev* dc = dalloc<ChangeDev>(n_changes);
    double* rows = dalloc<double>(std::max<int64_t>(n_rows, 1) * e->S);
    double* o = dalloc<double>(n_changes);
    ck(cudaMemcpyAsync(dc, hc.data(), n_changes * sizeof(ChangeDev), cudaMemcpyHostToDevice,
                       e->stream),
       "H2D");
    if (n_rows)
      ck(cudaMemcpyAsync(rows, added_arrivals, (size_t)n_rows * e->S * 8,
                         cudaMemcpyHostToDevice, e->stream),
         "H2D");
    refresh_terms(e);
    if (e->dtype == SEIS_F64)
      k_score_batch<double><<<(unsigned)n_changes, NT, 0, e->stream>>>(e->d, e->tab[e->cur],
                                                                       e->ctl, dc, rows, o);
    else
      k_score_batch<float><<<(unsigned)n_changes, NT, 0, e->stream>>>(e->d, e->tab[e->cur],
                                                                      e->ctl, dc, rows, o);
    ck(cudaGetLastError(), "k_score_batch");
    ck(cudaMemcpyAsync(delta_out, o, n_changes * 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    cudaFree(dc);
    cudaFree(rows);
    cudaFree(o);
    for (int64_t i = 0; i < n_changes; ++i)
      if (std::isnan(delta_out[i]))
        throw std::invalid_argument("removed event id not in the hypothesis");
  });
}

int seis_log_joint(seis_engine* e, double* out) {
  return guarded([&] {
    double* scratch = dalloc<double>(2 * 296 + 1);
    launch_lj_any(e, scratch + 2 * 296, scratch);
    ck(cudaGetLastError(), "log_joint");
    ck(cudaMemcpyAsync(out, scratch + 2 * 296, 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    cudaFree(scratch);
  });
}

}  // extern "C"

// The chromatic driver (run_chromatic, samplers.hpp:401-498) and, with
// serial = true, run_serial (samplers.hpp:282-315): one region [0, T], no
// constraint, chunks of record_every steps.
// Speculative proposals per round (1..MSPEC); SEIS_SPEC overrides the
// default depth for A/B measurements.
// Rounds that score a prefix of their batch (first_scored) from 16 station
// tiles on; below that (config[0]: 4 tiles, rounds of a few microseconds)
// plain speculation over three proposals is faster (1.80 M against 1.48 M
// proposals/s at config[0]; config[1], 50 tiles: 9.74 M against 10.05 M).
static bool round_prefix(const seis_engine* e) { return (e->S_pad + 31) / 32 >= 16; }
static int spec_depth(const seis_engine* e) {
  const char* v = getenv("SEIS_SPEC");
  // proposals generated per round: 3 scored speculatively (proposal-major), 4
  // of which a tile-major round scores a prefix (first_scored)
  const int m = v ? atoi(v) : (round_prefix(e) ? MSPEC : kSpecDefault);
  return m < 1 ? 1 : (m > MSPEC ? MSPEC : m);
}
// Rounds that stop at their first scored proposal, births and deaths taking
// the next one along (unless the chain accepts them often, phase.cuh s_bd_hot):
// the default from 16 station tiles on (config[2], one
// B200: three proposals scored per round 3.70 M proposals/s, rounds ending at
// the first scored one 3.88 M; with tile pairs: 4.34 M, births / deaths taking
// one more along 4.57 M, as many as the batch of four holds 4.66 M);
// SEIS_FIRST = 0 / 1 / 2 / 3 overrides (A/B).
static int first_scored(const seis_engine* e) {
  if (const char* v = getenv("SEIS_FIRST")) return atoi(v);
  return round_prefix(e) ? 3 : 0;
}
static int run_driver(seis_engine* e, const seis_sampler_cfg* sc, int32_t mode,
                      const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                      int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                      int64_t* row_step, double* row_log_joint, int64_t* row_count,
                      seis_run_stats* stats, bool serial) {
  scratch_reset(e);
  std::vector<cudaEvent_t> evs;
  auto alloc = [&](size_t bytes) {
    return scratch_get(e, bytes);
  };
  const int rc = guarded([&] {
    // SamplerConfig::validate + MoveDistribution::validate (samplers.hpp:59-70,
    // proposals.hpp:23-31)
    if (sc->steps_per_epoch < 1)
      throw std::invalid_argument("SamplerConfig: steps_per_epoch must be >= 1");
    if (sc->epochs < 1) throw std::invalid_argument("SamplerConfig: epochs must be >= 1");
    if (sc->n_regions < 1) throw std::invalid_argument("SamplerConfig: n_regions must be >= 1");
    if (sc->burn_in_fraction < 0 || sc->burn_in_fraction >= 1)
      throw std::invalid_argument("SamplerConfig: burn_in_fraction must be in [0, 1)");
    if (sc->record_every < 1)
      throw std::invalid_argument("SamplerConfig: record_every must be >= 1");
    double wsum = 0.0;
    for (double w : sc->weights) {
      if (w < 0) throw std::invalid_argument("MoveDistribution: negative weight");
      wsum += w;
    }
    if (std::abs(wsum - 1.0) > 1e-12)
      throw std::invalid_argument("MoveDistribution: weights must sum to 1");
    if (mode != 0 && mode != 1) throw std::invalid_argument("mode must be 0 or 1");
    if (mode == 1 && (!tape || !step_out)) throw std::invalid_argument("replay needs a tape");
    // run_chromatic setup (samplers.hpp:405-407)
    const double tau = e->cfg.x_max / e->cfg.v;
    const double l = serial ? e->cfg.T : e->cfg.T / (double)sc->n_regions;
    if (l > e->cfg.T) throw std::invalid_argument("build_partition: need 0 < l <= T");
    int ncol = 1;
    if (serial)
      ncol = 1;
    else if (l >= tau)
      ncol = 2;
    else if (l >= tau / 2)
      ncol = 3;
    else
      throw std::invalid_argument("color_partition: region length " + std::to_string(l) +
                                  " is below tau_max/2 = " + std::to_string(tau / 2) +
                                  "; would need more than 3 colors");
    Samp sp{};
    sp.k = sc->steps_per_epoch;
    sp.seed = sc->seed;
    double cum = 0.0;
    for (int q = 0; q < 5; ++q) {
      cum += sc->weights[q];
      sp.cumw[q] = cum;
      sp.logw[q] = std::log(sc->weights[q]);
    }
    sp.step_lx = sc->step_location_x;
    sp.step_lt = sc->step_location_t;
    sp.step_arr = sc->step_arrival;
    sp.step_joint = sc->step_joint;
    sp.joint_t_sd = sc->step_joint / e->cfg.v;
    sp.ncol = ncol;
    sp.mspec = spec_depth(e);
    sp.first_scored = first_scored(e);
    const int bcap = (int)sc->n_regions + 4;
    // the timed region starts before the partition kernel: everything the run
    // launches (partition, id base, counters, phases, barriers, rows) is inside
    cudaEvent_t ev_start, ev_stop;
    ck(cudaEventCreate(&ev_start), "event");
    ck(cudaEventCreate(&ev_stop), "event");
    evs.push_back(ev_start);
    evs.push_back(ev_stop);
    ck(cudaEventRecord(ev_start, e->stream), "event");
    int64_t launches = 0;  // kernels launched inside the timed region
    e->phases.clear();
    e->row_wall.clear();
    std::vector<cudaEvent_t> row_ev;
    // every epoch's partition up front (one CTA per epoch), so the phases
    // hold no host round trip
    const int64_t n_ep = (sc->dynamic && !serial) ? sc->epochs : 1;
    double* bnd = static_cast<double*>(alloc((size_t)n_ep * bcap * 8));
    int* nreg_d = static_cast<int*>(alloc((size_t)n_ep * 4));
    int* perr = static_cast<int*>(alloc(4));
    std::vector<int> h_nreg(n_ep);
    int herr = 0;
    if (serial) {  // config.full_region() (model.hpp:109)
      const double hb[2] = {0.0, e->cfg.T};
      ck(cudaMemcpy(bnd, hb, sizeof hb, cudaMemcpyHostToDevice), "H2D");
      h_nreg[0] = 1;
    } else {
      ck(cudaMemsetAsync(perr, 0, 4, e->stream), "memset");
      k_partition<<<(unsigned)n_ep, kPartThreads, 0, e->stream>>>(
          e->cfg.T, l, tau, ncol, sc->dynamic ? 1 : 0, sc->seed, 0, (int)n_ep, 0.0, bcap, bnd,
          nreg_d, perr, nullptr);
      ck(cudaGetLastError(), "k_partition");
      ++launches;
      ck(cudaMemcpyAsync(h_nreg.data(), nreg_d, (size_t)n_ep * 4, cudaMemcpyDeviceToHost,
                         e->stream),
         "D2H nreg");
      ck(cudaMemcpyAsync(&herr, perr, 4, cudaMemcpyDeviceToHost, e->stream), "D2H");
      // checked after the synchronisation that also brings next_base back
    }
    const int n_slots = serial ? 1 : (int)((sc->n_regions + 1 + ncol - 1) / ncol) + 1;
    int* births_cnt = static_cast<int*>(alloc((size_t)n_slots * 4));
    int* births_total = static_cast<int*>(alloc((size_t)n_slots * 4));
    // serial: the chain's list order between chunks ([0] = count, -1 = none yet)
    unsigned long long* order_io = nullptr;
    if (serial) {
      order_io = static_cast<unsigned long long*>(alloc((kSerialCap + 1) * 8));
      const unsigned long long none = ~0ull;
      ck(cudaMemcpy(order_io, &none, 8, cudaMemcpyHostToDevice), "H2D");
    }
    // overflow areas (80 KB each) for region chains rerun past MAXOWN events:
    // the explosive phases of configs 3/4 rerun thousands of regions
    const int ovf_cap = serial ? 0 : std::max(kOvfRegions, std::min(n_slots, 8192));
    // per-slot outputs: MAXOWN births / MAXDOUT diff entries per region; the
    // serial chain's one slot holds kSerialCap / 3 kSerialCap
    // (region slots: + kOvfRegions overflow areas for chains rerun past MAXOWN)
    const size_t n_births =
        serial ? (size_t)kSerialCap : (size_t)n_slots * MAXOWN + (size_t)ovf_cap * kSerialCap;
    const size_t n_diff = serial ? (size_t)3 * kSerialCap
                                 : (size_t)n_slots * MAXDOUT + (size_t)ovf_cap * 3 * kSerialCap;
    OutEv* births = static_cast<OutEv*>(alloc(n_births * sizeof(OutEv)));
    int* diff_cnt = static_cast<int*>(alloc((size_t)n_slots * 4));
    DiffPair* diff = static_cast<DiffPair*>(alloc(n_diff * sizeof(DiffPair)));
    Ovf ovf{nullptr, nullptr, ovf_cap};
    if (!serial) {
      ovf.slot = static_cast<int*>(alloc((size_t)n_slots * 4));
      ovf.count = static_cast<int*>(alloc(4));
      ck(cudaMemsetAsync(ovf.count, 0, 4, e->stream), "memset");
    }
    // cost-ordered dispatch (k_order); SEIS_ORDER=0 disables it (A/B)
    const bool use_order = !serial && !(getenv("SEIS_ORDER") && atoi(getenv("SEIS_ORDER")) == 0);
    int* order_cnt = static_cast<int*>(alloc((size_t)n_slots * 4));
    int* order = static_cast<int*>(alloc((size_t)n_slots * 4));
    int* retry = nullptr;
    int* retry_free = nullptr;
    if (!serial) {
      retry = static_cast<int*>(alloc((size_t)n_slots * 4));
      retry_free = static_cast<int*>(alloc((size_t)n_slots * kRetryFree * 4));
      ck(cudaMemsetAsync(retry, 0, (size_t)n_slots * 4, e->stream), "memset");
    }
    seis_tape_step* d_tape = nullptr;
    double* d_tarr = nullptr;
    seis_step_out* d_out = nullptr;
    if (mode == 1) {
      d_tape = static_cast<seis_tape_step*>(alloc((size_t)n_tape * sizeof(seis_tape_step)));
      d_tarr = static_cast<double*>(alloc((size_t)std::max<int64_t>(n_tape_arr, 1) * 8));
      d_out = static_cast<seis_step_out*>(alloc((size_t)n_tape * sizeof(seis_step_out)));
      ck(cudaMemcpyAsync(d_tape, tape, (size_t)n_tape * sizeof(seis_tape_step),
                         cudaMemcpyHostToDevice, e->stream),
         "H2D tape");
      if (n_tape_arr)
        ck(cudaMemcpyAsync(d_tarr, tape_arr, (size_t)n_tape_arr * 8, cudaMemcpyHostToDevice,
                           e->stream),
           "H2D tape arrivals");
    } else if (step_out) {  // production run recording its per-step decisions
      if (n_tape < 1) throw std::invalid_argument("step_out needs n_tape >= 1 entries");
      d_out = static_cast<seis_step_out*>(alloc((size_t)n_tape * sizeof(seis_step_out)));
    }
    const int64_t rcap = std::max<int64_t>(row_cap, 1);
    double* lj_dev = static_cast<double*>(alloc((size_t)rcap * 8));
    long long* cnt_dev = static_cast<long long*>(alloc((size_t)rcap * 8));
    double* lj_scratch = static_cast<double*>(alloc((2 * 296 + 1) * 8));
    unsigned long long* maxid = static_cast<unsigned long long*>(alloc(8));
    // next_base: above every id already present (reference starts empty at 0)
    k_max_id<<<1, 1024, 0, e->stream>>>(e->tab[e->cur], e->ctl, maxid);
    k_reset_counters<<<1, 1, 0, e->stream>>>(e->ctl);
    launches += 2;
    unsigned long long next_base = 0;
    ck(cudaMemcpyAsync(&next_base, maxid, 8, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    if (herr == 1) throw std::logic_error("color_partition: separation invariant violated");
    if (herr == 2) throw std::runtime_error("partition capacity");
    const bool timing = stats != nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> phase_ev;
    int64_t n_rows = 0;
    std::vector<int64_t> h_row_step;
    // snapshots at record points once executed >= burn (samplers.hpp:411-413,430-433)
    const int64_t planned = sc->epochs * sc->steps_per_epoch * (serial ? 1 : sc->n_regions);
    const int64_t burn = (int64_t)(sc->burn_in_fraction * (double)planned);
    e->snap_steps.clear();
    if (e->snap_cap > 0) {
      const long long zero = 0;
      ck(cudaMemcpyAsync(e->snap_top, &zero, 8, cudaMemcpyHostToDevice, e->stream), "H2D");
    }
    auto take_snapshot = [&](int64_t executed) {
      if (e->snap_cap <= 0 || executed < burn) return;
      if ((int64_t)e->snap_steps.size() >= e->snap_rec_cap) return;
      k_snapshot<<<1, 256, 0, e->stream>>>(e->tab[e->cur], e->ctl, e->snap_id, e->snap_x,
                                            e->snap_t, e->snap_top, e->snap_cap,
                                            e->snap_rec + 2 * e->snap_steps.size());
      ++launches;
      e->snap_steps.push_back(executed);
    };
    auto record_row = [&](int64_t executed) {
      if (n_rows < row_cap) {
        if (sc->record_log_joint) {
          launch_lj_any(e, lj_dev + n_rows, lj_scratch);
          launches += 3;
        }
        k_record<<<1, 1, 0, e->stream>>>(e->ctl, cnt_dev + n_rows);
        ++launches;
        h_row_step.push_back(executed);
        cudaEvent_t rv = nullptr;
        ck(cudaEventCreate(&rv), "event");
        evs.push_back(rv);
        ck(cudaEventRecord(rv, e->stream), "event");
        row_ev.push_back(rv);
      }
      ++n_rows;
      if (executed > 0 || n_rows > 1) take_snapshot(executed);
    };
    record_row(0);
    int64_t executed = 0, last_recorded = 0;
    long long tape_base = 0;
    // one color phase: ncr same-colored regions x kk steps, then the barrier
    auto run_phase = [&](int epoch, int color, int nreg, int ncr, const double* bndp, int64_t kk,
                         long long step_base) {
      PhaseArgs pa{};
      pa.epoch = epoch;
      pa.color = color;
      pa.nreg = nreg;
      pa.n_slots = ncr;
      pa.bnd = bndp;
      pa.next_base = next_base;
      pa.tape_base = tape_base;
      pa.tab = e->tab[e->cur];
      pa.fate_stamp = e->fate_stamp;
      pa.fate_alive = e->fate_alive;
      pa.fate_x = e->fate_x;
      pa.fate_t = e->fate_t;
      pa.fate_slot = e->fate_slot;
      pa.births_cnt = births_cnt;
      pa.births = births;
      pa.diff_cnt = diff_cnt;
      pa.diff = diff;
      pa.free_stack = e->free_stack;
      pa.compact = e->compact;
      pa.tape = d_tape;
      pa.tape_arr = d_tarr;
      pa.out = d_out;
      pa.serial = serial ? 1 : 0;
      pa.step_base = step_base;
      pa.births_total = births_total;
      pa.order_io = serial ? order_io : nullptr;
      Samp spk = sp;
      spk.k = kk;
      const int stamp = ++e->stamp;
      if ((mode == 1 || d_out) && tape_base + (long long)ncr * kk > n_tape)
        throw std::invalid_argument(mode == 1 ? "replay tape shorter than the run"
                                              : "step_out shorter than the run");
      cudaEvent_t a = nullptr, b = nullptr;
      if (timing) {
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        evs.push_back(a);
        evs.push_back(b);
        ck(cudaEventRecord(a, e->stream), "event");
      }
      launches += refresh_terms(e);
      if (use_order && ncr > e->n_sm) {
        k_order<<<1, 1024, 0, e->stream>>>(e->tab[e->cur].t, &e->ctl->n_events, bndp, nreg,
                                           color, std::max(ncol, 1), ncr, order_cnt, order);
        ck(cudaGetLastError(), "k_order");
        pa.slot_order = order;
        ++launches;
      }
      pa.retry = retry;
      pa.retry_free = retry_free;
      pa.ovf = ovf;
      launch_phase(e, mode, ncr, spk, pa, stamp);
      if (retry) {  // regions that outgrew the region kernel's chain arrays
        PhaseArgs pr = pa;
        pr.retry_pass = 1;
        launch_phase(e, mode, ncr, spk, pr, stamp);
        ++launches;
      }
      if (timing) {
        ck(cudaEventRecord(b, e->stream), "event");
        phase_ev.emplace_back(a, b);
      }
      ck(cudaGetLastError(), "k_phase");
      const int nxt = e->cur ^ 1;
      dim3 bg = commit_grid(ncr, e->n_sm);
      bg.x += 1;  // + the table rebuild CTA
      k_barrier<<<bg, kCommitThreads, 0, e->stream>>>(
          e->d, color, std::max(ncol, 1), nreg, diff_cnt, diff, e->free_stack, e->ctl,
          e->tab[e->cur], e->tab[nxt], e->cap, stamp, e->fate_stamp, e->fate_alive, e->fate_x,
          e->fate_t, e->fate_slot, ncr, births_cnt, births, ovf);
      ck(cudaGetLastError(), "k_barrier");
      e->terms_valid = false;  // the commit changed the counts
      launches += 2;
      if (!serial)  // Trace::phases, one record per committed region (samplers.hpp:479)
        for (int slot = 0; slot < ncr; ++slot)
          e->phases.push_back({(int64_t)epoch, (int32_t)color, 0,
                               (int64_t)color + (int64_t)slot * ncol, (int64_t)kk});
      e->cur = nxt;
      tape_base += (long long)ncr * kk;
      executed += (int64_t)ncr * kk;
      if (serial) {
        // run_serial: id_base += births (samplers.hpp:302-303); births are the
        // chain's accepted births alive or not, counted by the kernel
        int nb = 0;
        ck(cudaMemcpyAsync(&nb, births_total, 4, cudaMemcpyDeviceToHost, e->stream), "D2H");
        ck(cudaStreamSynchronize(e->stream), "sync");
        next_base += (unsigned long long)nb;
      } else {
        next_base += (unsigned long long)ncr * (unsigned long long)kk;
      }
    };
    if (serial) {
      // run_serial (samplers.hpp:294-313): chunks of record_every steps, a
      // trace row (and snapshot past burn-in) after every chunk
      const int64_t total = sc->epochs * sc->steps_per_epoch;
      while (executed < total) {
        const int64_t chunk = std::min<int64_t>(sc->record_every, total - executed);
        run_phase(0, 0, 1, 1, bnd, chunk, (long long)executed);
        last_recorded = executed;
        record_row(executed);
      }
    } else {
      const int64_t k = sc->steps_per_epoch;
      for (int64_t i = 0; i < sc->epochs; ++i) {
        const int64_t pi = sc->dynamic ? i : 0;
        const int nreg = h_nreg[pi];
        for (int color = 0; color < ncol; ++color) {
          const int ncr = nreg > color ? (nreg - color + ncol - 1) / ncol : 0;
          if (ncr == 0) continue;
          run_phase((int)i, color, nreg, ncr, bnd + (size_t)pi * bcap, k, 0);
          // record(false), samplers.hpp:424-434
          if (executed - last_recorded >= sc->record_every) {
            last_recorded = executed;
            record_row(executed);
          }
        }
      }
    }
    if (last_recorded != executed) record_row(executed);
    ck(cudaEventRecord(ev_stop, e->stream), "event");
    ck(cudaStreamSynchronize(e->stream), "run");
    for (auto rv : row_ev) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, ev_start, rv), "elapsed");
      e->row_wall.push_back(1e-3 * (double)ms);
    }
    const Ctl c = read_ctl(e);
    if (c.err) throw std::runtime_error(std::string("device: ") + err_name(c.err));
    if (mode == 1 && tape_base != n_tape)
      throw std::invalid_argument("replay tape longer than the run");
    const int64_t nr_out = std::min<int64_t>(n_rows, row_cap);
    if (nr_out > 0) {
      std::vector<double> lj(nr_out);
      std::vector<long long> cn(nr_out);
      ck(cudaMemcpy(lj.data(), lj_dev, nr_out * 8, cudaMemcpyDeviceToHost), "D2H");
      ck(cudaMemcpy(cn.data(), cnt_dev, nr_out * 8, cudaMemcpyDeviceToHost), "D2H");
      for (int64_t i = 0; i < nr_out; ++i) {
        if (row_step) row_step[i] = h_row_step[i];
        if (row_log_joint) row_log_joint[i] = sc->record_log_joint ? lj[i] : 0.0;
        if (row_count) row_count[i] = cn[i];
      }
    }
    if (d_out)
      ck(cudaMemcpy(step_out, d_out, (size_t)std::min<long long>(n_tape, tape_base) *
                                         sizeof(seis_step_out),
                    cudaMemcpyDeviceToHost),
         "D2H out");
    if (getenv("SEIS_PROF"))
      fprintf(stderr, "[seis prof] cycles: gen %llu items %llu decide %llu (parallel part %llu) writeback %llu rounds %llu; region chains: max %llu sum %llu\n",
              c.prof[0], c.prof[1], c.prof[2], c.prof[5], c.prof[3], c.prof[4], c.prof[6], c.prof[7]);
    if (getenv("SEIS_PROF"))
      for (int q = 0; q < 8; ++q)
        fprintf(stderr, "[seis prof] type %d: items %llu warp-cycles/item %.0f\n", q,
                c.tprof[1][q], c.tprof[1][q] ? (double)c.tprof[0][q] / c.tprof[1][q] : 0.0);
    if (stats) {
      std::memset(stats, 0, sizeof *stats);
      stats->total_steps = executed;
      stats->total_accepted = (int64_t)c.accepted;
      stats->scored_proposals = (int64_t)c.scored;
      stats->changed_samples = (int64_t)c.changed;
      stats->arrival_values = (int64_t)c.arrvals;
      const double by = e->dtype == SEIS_F64 ? 8.0 : 4.0;
      stats->algorithmic_bytes = (double)c.changed * (by + 2.0) + 8.0 * (double)c.arrvals;
      float ms = 0.f;
      double tot = 0.0;
      for (auto& pr : phase_ev) {
        ck(cudaEventElapsedTime(&ms, pr.first, pr.second), "elapsed");
        tot += ms;
      }
      stats->sweep_kernel_ms = tot;
      ck(cudaEventElapsedTime(&ms, ev_start, ev_stop), "elapsed");
      stats->total_ms = ms;
      stats->kernel_launches = launches;
      stats->n_rows = n_rows;
      stats->final_events = c.n_events;
      stats->speculative_discarded = (int64_t)c.speculative;
      stats->phases = (int64_t)phase_ev.size();
      stats->generated_versions = (int64_t)e->gv_cap - c.gv_top;
    }
  });
  for (auto ev : evs) cudaEventDestroy(ev);
  return rc;
}

extern "C" int seis_run_chromatic(seis_engine* e, const seis_sampler_cfg* sc, int32_t mode,
                                  const seis_tape_step* tape, int64_t n_tape,
                                  const double* tape_arr, int64_t n_tape_arr,
                                  seis_step_out* step_out, int64_t row_cap, int64_t* row_step,
                                  double* row_log_joint, int64_t* row_count,
                                  seis_run_stats* stats) {
  return run_driver(e, sc, mode, tape, n_tape, tape_arr, n_tape_arr, step_out, row_cap, row_step,
                    row_log_joint, row_count, stats, false);
}

extern "C" int seis_run_serial(seis_engine* e, const seis_sampler_cfg* sc, int32_t mode,
                               const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                               int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                               int64_t* row_step, double* row_log_joint, int64_t* row_count,
                               seis_run_stats* stats) {
  return run_driver(e, sc, mode, tape, n_tape, tape_arr, n_tape_arr, step_out, row_cap, row_step,
                    row_log_joint, row_count, stats, true);
}

// run_naive_parallel (samplers.hpp:321-394): independent per-region chains
// from the empty hypothesis, no coloring, region prior support and signal
// window; one launch runs every region's whole chain. The final hypothesis
// (the union) is committed to the engine; trace rows carry the union's event
// count at every checkpoint and log_joint at the last row only.
extern "C" int seis_run_naive(seis_engine* e, const seis_sampler_cfg* sc, int32_t mode,
                              const seis_tape_step* tape, int64_t n_tape, const double* tape_arr,
                              int64_t n_tape_arr, seis_step_out* step_out, int64_t row_cap,
                              int64_t* row_step, double* row_log_joint, int64_t* row_count,
                              seis_run_stats* stats) {
  scratch_reset(e);
  auto alloc = [&](size_t bytes) {
    return scratch_get(e, bytes);
  };
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evp0 = nullptr, evp1 = nullptr;
  const int rc = guarded([&] {
    if (sc->steps_per_epoch < 1 || sc->epochs < 1 || sc->n_regions < 1 || sc->record_every < 1 ||
        sc->burn_in_fraction < 0 || sc->burn_in_fraction >= 1)
      throw std::invalid_argument("SamplerConfig: invalid");
    double wsum = 0.0;
    for (double w : sc->weights) {
      if (w < 0) throw std::invalid_argument("MoveDistribution: negative weight");
      wsum += w;
    }
    if (std::abs(wsum - 1.0) > 1e-12)
      throw std::invalid_argument("MoveDistribution: weights must sum to 1");
    if (mode != 0 && mode != 1) throw std::invalid_argument("mode must be 0 or 1");
    if (mode == 1 && (!tape || !step_out)) throw std::invalid_argument("replay needs a tape");
    if (read_ctl(e).n_events != 0)
      throw std::invalid_argument("the naive sampler starts from the empty hypothesis");
    const double tau = e->cfg.x_max / e->cfg.v;
    const double l = e->cfg.T / (double)sc->n_regions;
    if (!(l > 0) || l > e->cfg.T) throw std::invalid_argument("build_partition: need 0 < l <= T");
    const int bcap = (int)sc->n_regions + 4;
    double* bnd = static_cast<double*>(alloc((size_t)bcap * 8));
    int* nreg_d = static_cast<int*>(alloc(4));
    int* perr = static_cast<int*>(alloc(4));
    ck(cudaMemsetAsync(perr, 0, 4, e->stream), "memset");
    // build_partition only: no coloring, no separation check (tau = -inf)
    k_partition<<<1, kPartThreads, 0, e->stream>>>(e->cfg.T, l, -INFINITY, 1, 0, 0, 0, 1, 0.0, bcap, bnd,
                                         nreg_d, perr, nullptr);
    int nreg = 0, herr = 0;
    ck(cudaMemcpyAsync(&nreg, nreg_d, 4, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaMemcpyAsync(&herr, perr, 4, cudaMemcpyDeviceToHost, e->stream), "D2H");
    ck(cudaStreamSynchronize(e->stream), "sync");
    if (herr) throw std::runtime_error("partition capacity");
    std::vector<double> hb(nreg + 1);
    ck(cudaMemcpy(hb.data(), bnd, (size_t)(nreg + 1) * 8, cudaMemcpyDeviceToHost), "D2H");
    // per-region prior constants (glibc log, density.hpp:225-237) and
    // signal windows (partition.hpp:94-102)
    std::vector<double> llam(nreg), lxa(nreg);
    std::vector<int> wlo(nreg), whi(nreg);
    for (int r = 0; r < nreg; ++r) {
      const double area = hb[r + 1] - hb[r];
      llam[r] = std::log(e->cfg.lambda_rate * area);
      lxa[r] = -std::log(e->cfg.x_max) - std::log(area);
      const double h = std::min(hb[r + 1] + tau, e->cfg.T);
      wlo[r] = (int)std::max<int64_t>(0, (int64_t)std::ceil(hb[r] * e->cfg.sample_rate - 1e-9));
      whi[r] = (int)std::min<int64_t>(e->n, (int64_t)std::ceil(h * e->cfg.sample_rate - 1e-9));
    }
    double* d_llam = static_cast<double*>(alloc((size_t)nreg * 8));
    double* d_lxa = static_cast<double*>(alloc((size_t)nreg * 8));
    int* d_wlo = static_cast<int*>(alloc((size_t)nreg * 4));
    int* d_whi = static_cast<int*>(alloc((size_t)nreg * 4));
    ck(cudaMemcpy(d_llam, llam.data(), (size_t)nreg * 8, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_lxa, lxa.data(), (size_t)nreg * 8, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_wlo, wlo.data(), (size_t)nreg * 4, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_whi, whi.data(), (size_t)nreg * 4, cudaMemcpyHostToDevice), "H2D");
    const int64_t spr = sc->epochs * sc->steps_per_epoch;
    if (spr > INT32_MAX) throw std::invalid_argument("too many steps per region");
    const int64_t re = std::min<int64_t>(sc->record_every, spr);
    const int64_t n_cp = (spr + re - 1) / re + 1;
    int* cp = static_cast<int*>(alloc((size_t)n_cp * nreg * 4));
    ck(cudaMemsetAsync(cp, 0, (size_t)n_cp * nreg * 4, e->stream), "memset");
    Samp sp{};
    sp.k = spr;
    sp.seed = sc->seed;
    double cum = 0.0;
    for (int q = 0; q < 5; ++q) {
      cum += sc->weights[q];
      sp.cumw[q] = cum;
      sp.logw[q] = std::log(sc->weights[q]);
    }
    sp.step_lx = sc->step_location_x;
    sp.step_lt = sc->step_location_t;
    sp.step_arr = sc->step_arrival;
    sp.step_joint = sc->step_joint;
    sp.joint_t_sd = sc->step_joint / e->cfg.v;
    sp.ncol = 1;
    sp.mspec = spec_depth(e);
    sp.first_scored = first_scored(e);
    // every region of the one launch may outgrow MAXOWN events (long chains
    // from the empty start): an overflow area each, up to 32768 regions
    const int ovf_cap = std::max(kOvfRegions, std::min((int)nreg, 32768));
    int* births_cnt = static_cast<int*>(alloc((size_t)nreg * 4));
    OutEv* births = static_cast<OutEv*>(alloc(
        ((size_t)nreg * MAXOWN + (size_t)ovf_cap * kSerialCap) * sizeof(OutEv)));
    int* diff_cnt = static_cast<int*>(alloc((size_t)nreg * 4));
    DiffPair* diff = static_cast<DiffPair*>(alloc(
        ((size_t)nreg * MAXDOUT + (size_t)ovf_cap * 3 * kSerialCap) * sizeof(DiffPair)));
    Ovf ovf{static_cast<int*>(alloc((size_t)nreg * 4)), static_cast<int*>(alloc(4)), ovf_cap};
    ck(cudaMemsetAsync(ovf.count, 0, 4, e->stream), "memset");
    seis_tape_step* d_tape = nullptr;
    double* d_tarr = nullptr;
    seis_step_out* d_out = nullptr;
    if (mode == 1) {
      if (n_tape != spr * nreg) throw std::invalid_argument("replay tape length != steps x regions");
      d_tape = static_cast<seis_tape_step*>(alloc((size_t)n_tape * sizeof(seis_tape_step)));
      d_tarr = static_cast<double*>(alloc((size_t)std::max<int64_t>(n_tape_arr, 1) * 8));
      d_out = static_cast<seis_step_out*>(alloc((size_t)n_tape * sizeof(seis_step_out)));
      ck(cudaMemcpy(d_tape, tape, (size_t)n_tape * sizeof(seis_tape_step), cudaMemcpyHostToDevice),
         "H2D tape");
      if (n_tape_arr)
        ck(cudaMemcpy(d_tarr, tape_arr, (size_t)n_tape_arr * 8, cudaMemcpyHostToDevice), "H2D");
    } else if (step_out) {  // production run recording its per-step decisions
      if (n_tape < spr * nreg) throw std::invalid_argument("step_out shorter than the run");
      d_out = static_cast<seis_step_out*>(alloc((size_t)spr * nreg * sizeof(seis_step_out)));
    }
    k_reset_counters<<<1, 1, 0, e->stream>>>(e->ctl);
    PhaseArgs pa{};
    pa.epoch = 0;
    pa.color = 0;
    pa.nreg = nreg;
    pa.n_slots = nreg;
    pa.bnd = bnd;
    pa.next_base = 0;  // every event of a naive region is born in the run
    pa.tape_base = 0;
    pa.tab = e->tab[e->cur];
    pa.fate_stamp = e->fate_stamp;
    pa.fate_alive = e->fate_alive;
    pa.fate_x = e->fate_x;
    pa.fate_t = e->fate_t;
    pa.fate_slot = e->fate_slot;
    pa.births_cnt = births_cnt;
    pa.births = births;
    pa.diff_cnt = diff_cnt;
    pa.diff = diff;
    pa.free_stack = e->free_stack;
    pa.compact = e->compact;
    pa.tape = d_tape;
    pa.tape_arr = d_tarr;
    pa.out = d_out;
    pa.naive = 1;
    pa.reg_llam = d_llam;
    pa.reg_lxa = d_lxa;
    pa.reg_wlo = d_wlo;
    pa.reg_whi = d_whi;
    pa.record_every = (int)re;
    pa.cp_counts = cp;
    const int stamp = ++e->stamp;
    ck(cudaEventCreate(&ev0), "event");
    ck(cudaEventCreate(&ev1), "event");
    ck(cudaEventCreate(&evp0), "event");
    ck(cudaEventCreate(&evp1), "event");
    ck(cudaEventRecord(ev0, e->stream), "event");
    ck(cudaEventRecord(evp0, e->stream), "event");
    int* retry = static_cast<int*>(alloc((size_t)nreg * 4));
    int* retry_free = static_cast<int*>(alloc((size_t)nreg * kRetryFree * 4));
    ck(cudaMemsetAsync(retry, 0, (size_t)nreg * 4, e->stream), "memset");
    pa.retry = retry;
    pa.retry_free = retry_free;
    pa.ovf = ovf;
    refresh_terms(e);
    launch_phase(e, mode, nreg, sp, pa, stamp);
    {  // regions that outgrew the region kernel's chain arrays
      PhaseArgs pr = pa;
      pr.retry_pass = 1;
      launch_phase(e, mode, nreg, sp, pr, stamp);
    }
    ck(cudaEventRecord(evp1, e->stream), "event");
    ck(cudaGetLastError(), "k_phase (naive)");
    // the union: coverage of every region's events, table of all births
    k_commit<<<commit_grid(nreg, e->n_sm), kCommitThreads, 0, e->stream>>>(
        e->d, 0, 1, nreg, nreg, diff_cnt, diff, ovf, e->free_stack, e->ctl);
    const int nxt = e->cur ^ 1;
    k_rebuild<<<1, 1024, 0, e->stream>>>(e->tab[e->cur], e->tab[nxt], e->cap, stamp,
                                          e->fate_stamp, e->fate_alive, e->fate_x, e->fate_t,
                                          e->fate_slot, nreg, births_cnt, births, ovf, e->ctl);
    ck(cudaGetLastError(), "naive commit");
    e->terms_valid = false;
    e->cur = nxt;
    // the union's final snapshot (samplers.hpp:388-391 at the last checkpoint;
    // the intermediate checkpoints' event lists are not kept on the device)
    e->snap_steps.clear();
    if (e->snap_cap > 0) {
      const long long zero = 0;
      ck(cudaMemcpyAsync(e->snap_top, &zero, 8, cudaMemcpyHostToDevice, e->stream), "H2D");
      const int64_t total = spr * nreg;
      if (total >= (int64_t)(sc->burn_in_fraction * (double)total) && e->snap_rec_cap > 0) {
        k_snapshot<<<1, 256, 0, e->stream>>>(e->tab[e->cur], e->ctl, e->snap_id, e->snap_x,
                                              e->snap_t, e->snap_top, e->snap_cap, e->snap_rec);
        e->snap_steps.push_back(total);
      }
    }
    double* lj_dev = static_cast<double*>(alloc(8));
    double* lj_scratch = static_cast<double*>(alloc((2 * 296 + 1) * 8));
    if (sc->record_log_joint) launch_lj_any(e, lj_dev, lj_scratch);
    ck(cudaEventRecord(ev1, e->stream), "event");
    ck(cudaStreamSynchronize(e->stream), "run");
    // Trace::phases of run_naive_parallel: one record per region (samplers.hpp:370)
    e->phases.clear();
    for (int r = 0; r < nreg; ++r) e->phases.push_back({0, 0, 0, (int64_t)r, spr});
    e->row_wall.clear();
    {
      float ms = 0.f;  // checkpoints complete together, at the end of the launch
      ck(cudaEventElapsedTime(&ms, ev0, evp1), "elapsed");
      for (int64_t ci = 0; ci < n_cp; ++ci) e->row_wall.push_back(ci ? 1e-3 * (double)ms : 0.0);
    }
    const Ctl c = read_ctl(e);
    if (c.err) throw std::runtime_error(std::string("device: ") + err_name(c.err));
    std::vector<int> hcp((size_t)n_cp * nreg);
    ck(cudaMemcpy(hcp.data(), cp, hcp.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    double lj_last = 0.0;
    if (sc->record_log_joint) ck(cudaMemcpy(&lj_last, lj_dev, 8, cudaMemcpyDeviceToHost), "D2H");
    for (int64_t ci = 0; ci < n_cp && ci < row_cap; ++ci) {
      int64_t cnt = 0;
      for (int r = 0; r < nreg; ++r) cnt += hcp[(size_t)ci * nreg + r];
      if (row_step) row_step[ci] = std::min<int64_t>(ci * re, spr) * nreg;
      if (row_count) row_count[ci] = cnt;
      if (row_log_joint) row_log_joint[ci] = (ci + 1 == n_cp) ? lj_last : 0.0;
    }
    if (d_out)
      ck(cudaMemcpy(step_out, d_out, (size_t)spr * nreg * sizeof(seis_step_out),
                    cudaMemcpyDeviceToHost),
         "D2H out");
    if (stats) {
      std::memset(stats, 0, sizeof *stats);
      stats->total_steps = spr * nreg;
      stats->total_accepted = (int64_t)c.accepted;
      stats->scored_proposals = (int64_t)c.scored;
      stats->changed_samples = (int64_t)c.changed;
      stats->arrival_values = (int64_t)c.arrvals;
      const double by = e->dtype == SEIS_F64 ? 8.0 : 4.0;
      stats->algorithmic_bytes = (double)c.changed * (by + 2.0) + 8.0 * (double)c.arrvals;
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, evp0, evp1), "elapsed");
      stats->sweep_kernel_ms = ms;
      ck(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
      stats->total_ms = ms;
      stats->kernel_launches = 4 + (sc->record_log_joint ? 3 : 0);
      stats->n_rows = n_cp;
      stats->phases = 1;
      stats->generated_versions = (int64_t)e->gv_cap - c.gv_top;
      stats->final_events = c.n_events;
      stats->speculative_discarded = (int64_t)c.speculative;
    }
  });
  for (cudaEvent_t ev : {ev0, ev1, evp0, evp1})
    if (ev) cudaEventDestroy(ev);
  return rc;
}
