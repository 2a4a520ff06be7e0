// phase.cuh — the region-sweep kernel k_phase (one CTA per same-colored
// region: run_region_steps of samplers.hpp:115-138 with the fused likelihood
// delta) and its proposal generator. Compiled one instantiation per
// translation unit (phase_inst.cu), launched through phase_api.h.
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"
#include "kernels.cuh"
#include "phase_api.h"

namespace seis {

// ----------------------------------------------------------------- phase kernel
template <int MODE>
__device__ void gen_proposal(const Dev& d, const Samp& sp, const PhaseArgs& pa, Prop& P,
                             const OwnEv* own, int nown, int region, double rlo, double rhi,
                             bool rclosed, int step, long long tape_idx, unsigned long long id_next,
                             int* err) {
  P.skip = 0;
  P.bad = 0;
  P.scored = 0;
  P.nr = P.na = 0;
  P.accept = 0;
  P.u_drawn = 1;
  P.tape_acc = 0;
  P.logq_f = P.logq_r = 0.0;
  P.tape_idx = tape_idx;
  bool null_ = false;
  const int k = nown;
  if (MODE == 0) {
    // philox stream spec v1 (include/seis_philox.h); control flow of
    // MoveDistribution::sample + propose_move (proposals.hpp:33-41,236-253)
    const seis_u32x4 d0 = seis_draw(sp.seed, (uint32_t)pa.epoch, (uint32_t)region, (uint32_t)step,
                                    SEIS_DRAW_MOVE);
    const double um = seis_u53(d0.w[0], d0.w[1]);
    int type = 4;
    for (int q = 0; q < 5; ++q)
      if (um < sp.cumw[q]) {
        type = q;
        break;
      }
    P.type = type;
    P.u = seis_u53(d0.w[2], d0.w[3]);
    P.logu = log(P.u);
    const seis_u32x4 d1 = seis_draw(sp.seed, (uint32_t)pa.epoch, (uint32_t)region,
                                    (uint32_t)step, SEIS_DRAW_SCALAR);
    switch (type) {
      case 0: {  // birth, proposals.hpp:84-107
        P.na = 1;
        P.at[0] = rlo + (rhi - rlo) * seis_u53(d1.w[0], d1.w[1]);
        P.ax[0] = 0.0 + (d.x_max - 0.0) * seis_u53(d1.w[2], d1.w[3]);
        P.aid = id_next;
        break;
      }
      case 1: {  // death, proposals.hpp:111-138
        if (k == 0) {
          null_ = true;
          break;
        }
        const int pick = (int)seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        P.nr = 1;
        P.rown[0] = pick;
        break;
      }
      case 2: {  // location, proposals.hpp:143-159
        if (k == 0) {
          null_ = true;
          break;
        }
        const int pick = (int)seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        float z0, z1;
        seis_normal_pair(sp.seed, (uint32_t)pa.epoch, (uint32_t)region, (uint32_t)step, 0, &z0,
                         &z1);
        P.nr = P.na = 1;
        P.rown[0] = pick;
        P.ax[0] = own[pick].x + (0.0 + sp.step_lx * (double)z0);
        P.at[0] = own[pick].t + (0.0 + sp.step_lt * (double)z1);
        break;
      }
      case 3: {  // arrival, proposals.hpp:161-174
        if (k == 0) {
          null_ = true;
          break;
        }
        const int pick = (int)seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        P.arr_st = (int)seis_lemire(seis_u64(d1.w[2], d1.w[3]), (uint64_t)d.S);
        const float z0 = seis_normal(sp.seed, (uint32_t)pa.epoch, (uint32_t)region,
                                     (uint32_t)step, 0);
        P.arr_da = 0.0 + sp.step_arr * (double)z0;
        P.nr = P.na = 1;
        P.rown[0] = pick;
        P.ax[0] = own[pick].x;
        P.at[0] = own[pick].t;
        break;
      }
      default: {  // joint pair, proposals.hpp:182-234
        if (k < 2) {
          null_ = true;
          break;
        }
        const int i1 = (int)seis_lemire(seis_u64(d1.w[0], d1.w[1]), (uint64_t)k);
        int i2 = (int)seis_lemire(seis_u64(d1.w[2], d1.w[3]), (uint64_t)(k - 1));
        if (i2 >= i1) ++i2;
        const seis_u32x4 d2 = seis_draw(sp.seed, (uint32_t)pa.epoch, (uint32_t)region,
                                        (uint32_t)step, SEIS_DRAW_PAIR);
        const int pair = (int)seis_lemire(seis_u64(d2.w[0], d2.w[1]), (uint64_t)(d.S - 1));
        const double xl = d.stations[pair], xr = d.stations[pair + 1], v = d.v;
        const double x1 = own[i1].x, t1 = own[i1].t, x2 = own[i2].x, t2 = own[i2].t;
        const double al1 = t1 + fabs(x1 - xl) / v;
        const double ar1 = t1 + fabs(x1 - xr) / v;
        const double al2 = t2 + fabs(x2 - xl) / v;
        const double ar2 = t2 + fabs(x2 - xr) / v;
        double n1x = 0.5 * (xl + xr) + 0.5 * v * (al1 - ar2);
        double n1t = 0.5 * (al1 + ar2) - (xr - xl) / (2.0 * v);
        double n2x = 0.5 * (xl + xr) + 0.5 * v * (al2 - ar1);
        double n2t = 0.5 * (al2 + ar1) - (xr - xl) / (2.0 * v);
        float z0, z1, z2, z3;
        seis_normal_pair(sp.seed, (uint32_t)pa.epoch, (uint32_t)region, (uint32_t)step, 0, &z0,
                         &z1);
        seis_normal_pair(sp.seed, (uint32_t)pa.epoch, (uint32_t)region, (uint32_t)step, 1, &z2,
                         &z3);
        n1x += 0.0 + sp.step_joint * (double)z0;
        n1t += 0.0 + sp.joint_t_sd * (double)z1;
        n2x += 0.0 + sp.step_joint * (double)z2;
        n2t += 0.0 + sp.joint_t_sd * (double)z3;
        P.nr = P.na = 2;
        P.rown[0] = i1;
        P.rown[1] = i2;
        P.ax[0] = n1x;
        P.at[0] = n1t;
        P.ax[1] = n2x;
        P.at[1] = n2t;
        break;
      }
    }
  } else {
    // replay: the proposal comes from the host tape (reference draws)
    const seis_tape_step& ts = pa.tape[tape_idx];
    P.type = (int)ts.type;
    null_ = ts.is_null != 0;
    P.u = ts.u;
    P.logu = log(ts.u);
    P.u_drawn = (int)ts.u_drawn;
    P.tape_acc = (int)ts.accepted;
    P.logq_f = ts.logq_f;
    P.logq_r = ts.logq_r;
    P.tape_off = ts.added_arr_off;
    if (!null_) {
      P.nr = (int)ts.n_removed;
      P.na = (int)ts.n_added;
      for (int q = 0; q < P.nr; ++q) {
        int f = -1;
        for (int i = 0; i < nown; ++i)
          if (own[i].id == ts.removed_id[q]) {
            f = i;
            break;
          }
        if (f < 0) {
          // may name an event born by an earlier step of this speculative
          // round; only an error if this proposal is actually reached
          P.bad = 1;
          null_ = true;
          break;
        }
        P.rown[q] = f;
      }
      for (int a = 0; a < P.na; ++a) {
        P.ax[a] = ts.added_x[a];
        P.at[a] = ts.added_t[a];
      }
      P.aid = P.type == 0 ? ts.added_id[0] : 0;
    }
  }
  if (null_) {
    P.skip = 1;
    P.nr = P.na = 0;
    P.u_drawn = 0;
    return;
  }
  for (int q = 0; q < P.nr; ++q) {
    const OwnEv& e = own[P.rown[q]];
    P.rslot[q] = e.slot;
    P.rsidx[q] = e.sidx;
    P.rx[q] = e.x;
    P.rt[q] = e.t;
  }
  // mh_step constraint (proposals.hpp:269-282; none in run_serial,
  // samplers.hpp:300), then delta_log_joint's support check (density.hpp:218-221)
  if (!pa.serial)
    for (int a = 0; a < P.na; ++a) {
      const double t = P.at[a];
      if (!(t >= rlo && (t < rhi || (rclosed && t == rhi)))) P.skip = 1;
    }
  if (P.skip) return;
  P.scored = 1;
  // support: [0, T] closed in chromatic mode, the region in naive mode
  // (density.hpp:218-221); naive support == the constraint already checked
  for (int a = 0; a < P.na; ++a) {
    const double t = P.at[a], x = P.ax[a];
    if (x < 0.0 || x > d.x_max || !(t >= 0.0 && t <= d.T)) P.skip = 1;
  }
}

template <typename YT, int MODE, int NTT, int MINB, int CAP, bool GEN, bool TM>
__global__ void __launch_bounds__(NTT, MINB)
    k_phase(const Dev d, const Samp sp, const PhaseArgs pa, Ctl* ctl, int stamp) {
  constexpr int NWT = NTT / 32;
  static_assert(NTT == NT, "diff_cache_overflow() places the cache for NT threads");
  constexpr bool kBig = CAP > MAXOWN;  // run_serial's whole-world chain
  __shared__ double2 Ts[kTsSize];  // {dL, dI} per (dc, count) + a zero entry
  // the chain's arrays: static for a region chain, dynamic (after the
  // partial sums, in place of the diff-window cache) for the serial chain
  __shared__ OwnEv own_s[kBig ? 1 : CAP];
  __shared__ StartEv st_s[kBig ? 1 : CAP];
  __shared__ int pold_s[kBig ? 1 : 2 * CAP], pnew_s[kBig ? 1 : 2 * CAP];
  __shared__ int lfree_s[kBig ? 1 : CAP], cur_of_s[kBig ? 1 : CAP];
  __shared__ double s_logi_k_s[kBig ? 1 : CAP + 2];  // log(i), i <= CAP + 1 (proposal terms)
  __shared__ Prop prop[2][MSPEC];
  __shared__ double red_sig[NWT][MSPEC], red_arr[NWT][MSPEC];

  __shared__ int red_cnt[NWT][MSPEC];
  __shared__ int s_w[NWT];
  __shared__ int s_nown, s_np, s_abort, s_tmp, s_adv, s_accq, s_dc_dirty, s_tw_dirty;
  __shared__ int s_bd_hot, s_bd_scored, s_bd_acc;  // this chain's scored / accepted births + deaths
  __shared__ int s_specok;  // this round's proposals were generated during the last decision
  __shared__ unsigned long long s_births;
  __shared__ double s_delta[MSPEC], s_logr[MSPEC], s_prior[2];
  // dynamic: [LOGIWIN] log(i), i in [N - LOGIWIN/2, N + LOGIWIN/2), then the
  // per-lane partial sums of the tile-major pass
  extern __shared__ double s_logi_n[];
  double(*acc_sig)[NTT] = reinterpret_cast<double(*)[NTT]>(s_logi_n + LOGIWIN);
  double(*acc_arr)[NTT] = reinterpret_cast<double(*)[NTT]>(s_logi_n + LOGIWIN + MSPEC * NTT);
  int(*acc_cnt)[NTT] = reinterpret_cast<int(*)[NTT]>(s_logi_n + LOGIWIN + 2 * MSPEC * NTT);
  DiffS* dcache =
      reinterpret_cast<DiffS*>(s_logi_n + LOGIWIN + 2 * MSPEC * NTT + MSPEC * NTT / 2);
  // tile-major pass (never together with the diff-window cache): one flag per
  // station tile in its place (region chains only)
  unsigned char* const tile_nw = reinterpret_cast<unsigned char*>(dcache);
  // serial layout in dynamic smem: own | st | log i | pold | pnew | lfree | cur_of
  char* const big = reinterpret_cast<char*>(dcache);
  constexpr size_t kOffSt = CAP * sizeof(OwnEv), kOffLogi = kOffSt + CAP * sizeof(StartEv);
  constexpr size_t kOffPold = kOffLogi + (CAP + 8) * sizeof(double);
  OwnEv* const own = kBig ? reinterpret_cast<OwnEv*>(big) : own_s;
  StartEv* const st = kBig ? reinterpret_cast<StartEv*>(big + kOffSt) : st_s;
  double* const s_logi_k = kBig ? reinterpret_cast<double*>(big + kOffLogi) : s_logi_k_s;
  int* const pold = kBig ? reinterpret_cast<int*>(big + kOffPold) : pold_s;
  int* const pnew = kBig ? pold + 2 * CAP : pnew_s;
  int* const lfree = kBig ? pold + 4 * CAP : lfree_s;
  int* const cur_of = kBig ? pold + 5 * CAP : cur_of_s;
  __shared__ int s_accg[MSPEC], s_cnt[MSPEC];
  __shared__ long long s_nlocal;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot_idx = pa.slot_order ? pa.slot_order[blockIdx.x] : (int)blockIdx.x;
  if (pa.retry_pass && pa.retry[slot_idx] == 0) return;  // not handed over: done
  if (tid == 0) {  // a CTA that stops on an error leaves nothing for the barrier
    pa.births_cnt[slot_idx] = 0;
    pa.diff_cnt[slot_idx] = 0;
    if (pa.ovf.slot) pa.ovf.slot[slot_idx] = -1;
    if (pa.births_total) pa.births_total[slot_idx] = 0;
  }
  const int region = pa.naive ? slot_idx : pa.color + slot_idx * sp.ncol;
  if (region >= pa.nreg) return;
  const double rlo = pa.bnd[region], rhi = pa.bnd[region + 1];
  const bool rclosed = region + 1 == pa.nreg;
  const int N = ctl->n_events;
  const double log_len = log(rhi - rlo);  // std::log(region.length()), proposals.hpp:102
  // prior constants: area T in chromatic mode (samplers.hpp:410), the region
  // in naive mode (samplers.hpp:347); likelihood window likewise
  const double llam = pa.naive ? pa.reg_llam[region] : d.log_lambda_T;
  const double lxa_r = pa.naive ? pa.reg_lxa[region] : d.lxa;
  const int win_lo = pa.naive ? pa.reg_wlo[region] : 0;
  const int win_hi = pa.naive ? pa.reg_whi[region] : d.n;

  fill_ts(Ts, d, tid, NTT);
  const int logi_base = N - LOGIWIN / 2;
  for (int i = tid; i < CAP + 2; i += NTT) s_logi_k[i] = i < d.logi_n ? d.logi[i] : 0.0;
  for (int i = tid; i < LOGIWIN; i += NTT) {
    const int g = logi_base + i;
    s_logi_n[i] = (g >= 0 && g < d.logi_n) ? d.logi[g] : 0.0;
  }
  if (tid == 0) {
    s_nown = 0;
    s_abort = 0;
    s_dc_dirty = 1;
    s_tw_dirty = 1;
    s_specok = 0;
    s_bd_hot = 0;
    s_bd_scored = 0;
    s_bd_acc = 0;
  }
  if (tid < 16) s_tprof[tid >> 3][tid & 7] = 0ull;  // kernels.cuh
  __syncthreads();
  // own events: table entries (id order) inside the region
  // (events_in_region, proposals.hpp:65-71, on the local copy of samplers.hpp:448)
  for (int base = 0; base < N; base += NTT) {
    const int i = base + tid;
    bool inr = false;
    if (i < N) {
      const double t = pa.tab.t[i];
      inr = t >= rlo && (t < rhi || (rclosed && t == rhi));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, inr);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    if (tid == 0) {
      int acc = s_nown;
      for (int w = 0; w < NWT; ++w) {
        const int c = s_w[w];
        s_w[w] = acc;
        acc += c;
      }
      s_tmp = acc;
    }
    __syncthreads();
    if (inr) {
      const int pos = s_w[warp] + __popc(bal & ((1u << lane) - 1u));
      if (pos < CAP) {
        own[pos].id = pa.tab.id[i];
        own[pos].x = pa.tab.x[i];
        own[pos].t = pa.tab.t[i];
        own[pos].slot = pa.tab.slot[i];
        own[pos].sidx = pos;
        st[pos].id = pa.tab.id[i];
        st[pos].slot = pa.tab.slot[i];
        st[pos].tab = i;
        st[pos].current = 1;
      }
    }
    __syncthreads();
    if (tid == 0) s_nown = s_tmp;
    __syncthreads();
  }
  if (s_nown > CAP) {
    if (!kBig && pa.retry) {  // rerun by the whole-chain variant
      if (tid == 0) {
        pa.retry_free[(size_t)slot_idx * kRetryFree] = 0;
        pa.retry[slot_idx] = 1;
      }
      return;
    }
    if (tid == 0) set_err(ctl, ERR_OWN_OVERFLOW);
    return;
  }
  // run_serial keeps the chain's list order (erase + push_back) across its
  // chunks (samplers.hpp:299-303); the table is in id order, so the previous
  // chunk's order is restored here
  if (pa.order_io && tid == 0) {
    const long long cnt = (long long)pa.order_io[0];
    if (cnt >= 0 && cnt == s_nown) {
      for (int i = 0; i < cnt; ++i) {
        const unsigned long long want = pa.order_io[1 + i];
        int f = i;
        while (f < s_nown && own[f].id != want) ++f;
        if (f < s_nown && f != i) {
          const OwnEv tmp = own[f];
          own[f] = own[i];
          own[i] = tmp;
        }
      }
    }
  }
  __syncthreads();
  const int nstart = s_nown;
  // thread-0 chain state (mirrored in shared memory for the generators)
  // thread-0 chain state lives in shared memory: registers are allocated for
  // every thread, and the scoring passes need them more
  __shared__ struct {
    long long n_local, tc, t0, tprof[6];
    unsigned long long births, n_acc, n_scored, n_arr, n_changed, n_spec;
    int nown, np, nlfree;
  } z;
  int& nown = z.nown;
  int& np = z.np;
  int& nlfree = z.nlfree;
  long long& n_local = z.n_local;
  unsigned long long& births = z.births;
  unsigned long long& n_acc = z.n_acc;
  unsigned long long& n_scored = z.n_scored;
  unsigned long long& n_arr = z.n_arr;
  unsigned long long& n_changed = z.n_changed;
  unsigned long long& n_spec = z.n_spec;
  long long(&tprof)[6] = z.tprof;
  long long& tc = z.tc;
  if (tid == 0) {
    nown = nstart;
    np = nlfree = 0;
    if (pa.retry_pass) {  // the slots the region kernel's attempt took
      const int* rf = pa.retry_free + (size_t)slot_idx * kRetryFree;
      for (int k2 = 0; k2 < rf[0]; ++k2) lfree[nlfree++] = rf[1 + k2];
      pa.retry[slot_idx] = 0;
    }
    n_local = N;
    births = n_acc = n_scored = n_arr = n_changed = n_spec = 0;
    for (int q = 0; q < 6; ++q) tprof[q] = 0;
    tc = clock64();
    z.t0 = tc;
  }
  const unsigned long long id_base =
      pa.naive ? ((unsigned long long)region + 1ull) << 32  // samplers.hpp:349
               : pa.next_base + (unsigned long long)slot_idx * sp.k;
  if (tid == 0) {
    s_np = 0;
    s_births = 0;
    s_nlocal = N;
  }
  const int T_per = (d.S_pad + 31) / 32;  // tiles of 32 stations
  int round = 0;
  for (int i0 = 0; i0 < (int)sp.k; ++round) {
    int m = min(sp.mspec, (int)sp.k - i0);
    const int buf = round & 1;
    __syncthreads();  // S0: previous round's write-back and state are visible
    if (tid == 0) {
      const long long now = clock64();
      tprof[3] += now - tc;
      tc = now;
    }
    if (tid == 0) {
      const long long n0 = s_nlocal;
      const long long wb = n0 + 1 - logi_base, wd = n0 - logi_base;
      const double lb = (wb >= 0 && wb < LOGIWIN) ? s_logi_n[wb] : d.logi[n0 + 1];
      const double ld = (wd >= 0 && wd < LOGIWIN) ? s_logi_n[wd] : d.logi[n0];
      double pb = 0.0, pdth = 0.0;
      pb += llam - lb;
      pb += 1.0 * lxa_r;
      pdth -= llam - ld;
      pdth += -1.0 * lxa_r;
      s_prior[0] = pb;
      s_prior[1] = pdth;
    }
    // the round's diff windows per station (proposal-major pass): rebuilt only
    // after an accept changed the region's diff, alongside generation
    const bool use_dcache =
        !TM && !kBig && d.dcache_on != 0;
    const bool dc_build = use_dcache && s_np > 0 && s_dc_dirty;
    const bool tw_dirty = s_tw_dirty != 0;  // per-tile diff flags of the tile-major pass
    if (warp < m && lane == 0 && !(MODE == 0 && s_specok)) {  // one lane per warp: move types do not diverge
      const int step = i0 + warp;
      gen_proposal<MODE>(d, sp, pa, prop[buf][warp], own, s_nown, region, rlo, rhi, rclosed,
                         (int)(pa.step_base + step),
                         pa.tape_base + (long long)slot_idx * sp.k + step, id_base + s_births,
                         &ctl->err);
    }
    if (lane < MSPEC) {
      red_sig[warp][lane] = 0.0;
      red_arr[warp][lane] = 0.0;
      red_cnt[warp][lane] = 0;
    }
#pragma unroll
    for (int q = 0; q < MSPEC; ++q) {
      acc_sig[q][tid] = 0.0;
      acc_arr[q][tid] = 0.0;
      acc_cnt[q][tid] = 0;
    }
    if (dc_build) {
      const int np_c = s_np;
      DiffS4x* ovf = const_cast<DiffS4x*>(diff_cache_overflow());
      for (int j = tid; j < d.S_pad; j += NTT)
        diff_station<GEN>(d, j, np_c, pold, pnew, dcache[j], ovf[j]);
    }
    __syncthreads();  // S1: proposals (and diff windows) ready
    // first_scored: the round ends with its first proposal that needs scoring
    // (the skipped ones before it are rejected for free, the ones after it
    // are regenerated), except that births and deaths, which are rarely
    // accepted, take the batch's next scored proposal along (2: one more, 3:
    // as long as they are births or deaths). Almost nothing scored is
    // discarded (config[2]: 1 % of the steps), generation stays parallel, and
    // a round's fixed cost (barriers, decision) is shared where that is
    // safe. Pays where a round's items are long (tile-major launches);
    // plain speculation pays where they are short.
    if (sp.first_scored) {
      int f = 0;
      while (f < m - 1 && prop[buf][f].skip) ++f;
      // first_scored = 2: a birth or death (rarely accepted) takes the next
      // scored proposal of the batch along. Not where this chain does accept
      // them often (s_bd_hot: more than one in eight of its scored births /
      // deaths this phase, e.g. configs 3 / 4, whose hypothesis swings by
      // 400 k events per phase): there the round ends at its first scored one.
      int more = s_bd_hot ? 0 : sp.first_scored - 1;  // 2: one more, 3: while births / deaths
      while (more > 0 && f < m - 1 && !prop[buf][f].skip && prop[buf][f].type <= 1) {
        ++f;
        while (f < m - 1 && prop[buf][f].skip) ++f;
        if (sp.first_scored == 2) --more;
      }
      m = f + 1;
    }
    if (tid == 0) {
      const long long now = clock64();
      tprof[0] += now - tc;
      tc = now;
      s_dc_dirty = 0;
      if (TM && s_np > 0) {  // a dense round rebuilds every tile's flag
        bool dense = false;
        for (int q = 0; q < m; ++q)
          dense |= !prop[buf][q].skip && !(MODE == 0 && prop[buf][q].type == 3);
        if (dense) s_tw_dirty = 0;
      }
    }
    {
      const int np_now = s_np;
      // Two item orders. Many tiles per warp (configs 2-4): one item = one
      // tile, the warp scores every proposal of the round on it back to back,
      // so the later proposals (same region, overlapping rows) hit the lines
      // the first brought into L1. Few tiles (config 1): items (proposal,
      // tile) proposal-major, which balances the warps better.
      if constexpr (TM) {
        // a round whose proposals are all skipped (null, constrained out)
        // visits no tile; production arrival moves alone visit only tile 0
        bool any_dense = false, any_arr = false;
        // every scored proposal a production birth or death of a stored /
        // generated version whose arrivals a lane can compute: tile pairs
        bool pair_round = kPairOn && MODE == 0 && d.tpos != nullptr;
        for (int q = 0; q < m; ++q) {
          const Prop& P = prop[buf][q];
          if (P.skip) continue;
          if (MODE == 0 && P.type == 3)
            any_arr = true;
          else
            any_dense = true;
          if (!(P.type == 0 || (P.type == 1 && (!GEN || P.rslot[0] >= 0)))) pair_round = false;
        }
        pair_round = pair_round && any_dense;
        const int tile_end = any_dense ? T_per : (any_arr ? 1 : 0);
        const bool tw_ok = !kBig && T_per <= kTileFlags;
        const bool tw_fresh = tw_ok && any_dense && !tw_dirty;
        // A warp owns pairs of neighbouring station tiles (2u, 2u + 1), u =
        // warp, warp + NWT, ...: 64 consecutive stations, whose birth normals
        // come from 32 Philox calls, one per lane (dense_pair_terms).
        for (int u = warp; 2 * u < tile_end; u += NWT) {
          const int t0 = 2 * u;
          // Tile pairs: when every scored proposal of the round is a production
          // birth or death and the region's diff has no window on either tile,
          // both are scored together: two independent setup chains and twice
          // the cached-term rows in flight
          if (pair_round && t0 + 1 < tile_end &&
              (np_now == 0 || (tw_fresh && tile_nw[t0] == 0 && tile_nw[t0 + 1] == 0))) {
#pragma unroll 1
            for (int q = 0; q < m; ++q) {
              const Prop& P = prop[buf][q];
              if (P.skip) continue;
              PassIn in;
              in.seed = sp.seed;
              in.sweep = (uint32_t)pa.epoch;
              in.region = (uint32_t)region;
              in.step = (uint32_t)(pa.step_base + i0 + q);
              in.wlo = win_lo;
              in.whi = win_hi;
              double sA = 0.0, sB = 0.0, aA = 0.0, aB = 0.0;
              int cnt = 0;
              if (P.type == 0)
                dense_pair_terms<true>(d, P, in, t0 * 32, sA, sB, aA, aB, cnt);
              else
                dense_pair_terms<false>(d, P, in, t0 * 32, sA, sB, aA, aB, cnt);
              acc_sig[q][tid] = (acc_sig[q][tid] + sA) + sB;  // tile order
              acc_arr[q][tid] = (acc_arr[q][tid] + aA) + aB;
              acc_cnt[q][tid] += cnt;
            }
            continue;
          }
          const int t1 = min(t0 + 2, tile_end);
#pragma unroll 1
          for (int tile = t0; tile < t1; ++tile) {
            DiffW X;
            long long tq = kProfItems ? clock64() : 0;
            // tiles where the region's diff has no effective window (e.g. only
            // arrival moves at other stations were accepted) stay so until the
            // next accept: remembered per tile, the pair walk is skipped
            if (np_now == 0 || (tw_fresh && tile_nw[tile] == 0)) {
              X.nwmax = 0;
            } else {
              diff_windows<GEN>(d, tile * 32 + lane, np_now, pold, pnew, X);
              if (tw_ok && any_dense && lane == 0)
                tile_nw[tile] = (unsigned char)min(X.nwmax, 255);
            }
            if (kProfItems) {
              __syncwarp();
              const long long now = clock64();
              if (lane == 0) {
                atomicAdd(&s_tprof[0][5], (unsigned long long)(now - tq));
                atomicAdd(&s_tprof[1][5], 1ull);
              }
              tq = now;
            }
#pragma unroll 1
            for (int q = 0; q < m; ++q) {
              const Prop& P = prop[buf][q];
              if (P.skip) continue;
              if (MODE == 0 && P.type == 3 && tile != 0) continue;
              PassIn in;
              in.src = P.na == 0 ? SRC_NONE
                                 : (MODE == 1 ? SRC_ROWS : (P.type == 0 ? SRC_BIRTH : SRC_SHIFT));
              in.rows[0] = pa.tape_arr + (MODE == 1 ? P.tape_off : 0);
              in.rows[1] = in.rows[0] + d.S;
              in.seed = sp.seed;
              in.sweep = (uint32_t)pa.epoch;
              in.region = (uint32_t)region;
              in.step = (uint32_t)(pa.step_base + i0 + q);
              in.wlo = win_lo;
              in.whi = win_hi;
              double sig = 0.0, arr = 0.0;
              int cnt = 0;
              score_item<MODE, YT, GEN>(d, P, in, tile, np_now, pold, pnew, X, true, Ts, sig, arr,
                                        cnt);
              // per-lane partial sums; the warp reduces them once per round
              acc_sig[q][tid] += sig;
              acc_arr[q][tid] += arr;
              acc_cnt[q][tid] += cnt;
              if (kProfItems) {
                const long long now = clock64();
                if (lane == 0) {
                  atomicAdd(&s_tprof[0][P.type], (unsigned long long)(now - tq));
                  atomicAdd(&s_tprof[1][P.type], 1ull);
                }
                tq = now;
              }
            }
          }
        }
        for (int q = 0; q < m; ++q) {
          const double sg = warp_sum(acc_sig[q][tid]);
          const double ar = warp_sum(acc_arr[q][tid]);
          const int cn = (int)__reduce_add_sync(0xffffffffu, (unsigned)acc_cnt[q][tid]);
          if (lane == 0) {
            red_sig[warp][q] = sg;
            red_arr[warp][q] = ar;
            red_cnt[warp][q] = cn;
          }
        }
      } else {
        int cur_q = -1;
        double sig = 0.0, arr = 0.0;
        int cnt = 0;
        const int n_items = m * T_per;
        int q = 0, tile = warp;  // t = q * T_per + tile, advanced without division
        while (tile >= T_per) {
          tile -= T_per;
          ++q;
        }
        for (int t = warp; t < n_items; t += NWT, tile += NWT) {
          while (tile >= T_per) {
            tile -= T_per;
            ++q;
          }
          if (q != cur_q) {
            if (cur_q >= 0) {
              sig = warp_sum(sig);
              arr = warp_sum(arr);
              cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
              if (lane == 0) {
                red_sig[warp][cur_q] += sig;
                red_arr[warp][cur_q] += arr;
                red_cnt[warp][cur_q] += cnt;
              }
              sig = arr = 0.0;
              cnt = 0;
            }
            cur_q = q;
          }
          const Prop& P = prop[buf][q];
          // nothing to score: a skipped proposal, or a production arrival
          // move outside the tile of its one station (before the cache read)
          if (P.skip || (MODE == 0 && P.type == 3 && tile != 0)) continue;
          PassIn in;
          in.src = P.na == 0 ? SRC_NONE
                             : (MODE == 1 ? SRC_ROWS : (P.type == 0 ? SRC_BIRTH : SRC_SHIFT));
          in.rows[0] = pa.tape_arr + (MODE == 1 ? P.tape_off : 0);
          in.rows[1] = in.rows[0] + d.S;
          in.seed = sp.seed;
          in.sweep = (uint32_t)pa.epoch;
          in.region = (uint32_t)region;
          in.step = (uint32_t)(pa.step_base + i0 + q);
          in.wlo = win_lo;
          in.whi = win_hi;
          DiffW X;
          if (use_dcache) {
            if (np_now > 0) {
              diff_from_cache(dcache[tile * 32 + lane], X);
            } else {
              X.nwmax = 0;
            }
          }
          score_item<MODE, YT, GEN>(d, P, in, tile, np_now, pold, pnew, X, use_dcache, Ts, sig, arr,
                               cnt);
        }
        if (cur_q >= 0) {
          sig = warp_sum(sig);
          arr = warp_sum(arr);
          cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
          if (lane == 0) {
            red_sig[warp][cur_q] += sig;
            red_arr[warp][cur_q] += arr;
            red_cnt[warp][cur_q] += cnt;
          }
        }
      }
    }
    __syncthreads();  // S2: partial sums ready
    if (tid == 0) {
      const long long now = clock64();
      tprof[1] += now - tc;
      tc = now;
    }
    // Production mode: while warp 0 decides, lanes 0 of warps 1..m generate
    // the next round's proposals assuming this round accepts nothing (the
    // common case: the state, and so every draw, is then unchanged). They are
    // used only if that holds; after an accept they are regenerated.
    const int i_next = i0 + m;
    const int m_next = MODE == 0 ? min(sp.mspec, (int)sp.k - i_next) : 0;
    if (MODE == 0 && warp >= 1 && warp <= m_next && lane == 0) {
      const int step = i_next + warp - 1;
      gen_proposal<MODE>(d, sp, pa, prop[buf ^ 1][warp - 1], own, s_nown, region, rlo, rhi,
                         rclosed, (int)(pa.step_base + step),
                         pa.tape_base + (long long)slot_idx * sp.k + step, id_base + s_births,
                         &ctl->err);
    }
    if (warp == 0) {
      // per-proposal delta / log_r / decision against the round's state, in
      // parallel lanes (delta_log_joint density.hpp:223-240; log_accept_ratio
      // and mh_step proposals.hpp:255-291). Lanes 8q..8q+7 reduce proposal q's
      // per-warp partials (fixed order, deterministic).
      // (kLPQ lanes per proposal: 8 with up to four proposals per round)
      constexpr int kLPQ = MSPEC <= 4 ? 8 : (MSPEC <= 8 ? 4 : 2);
      static_assert(MSPEC * kLPQ <= 32 && MSPEC <= 16, "reduction layout");
      const int q = lane / kLPQ, g = lane % kLPQ;
      double sig = 0.0, A = 0.0;
      int c = 0;
      if (q < m)
        for (int w = g; w < NWT; w += kLPQ) {
          sig += red_sig[w][q];
          A += red_arr[w][q];
          c += red_cnt[w][q];
        }
#pragma unroll
      for (int o = kLPQ / 2; o; o >>= 1) {
        sig += __shfl_down_sync(0xffffffffu, sig, o, kLPQ);
        A += __shfl_down_sync(0xffffffffu, A, o, kLPQ);
        c += __shfl_down_sync(0xffffffffu, c, o, kLPQ);
      }
      Prop& P = prop[buf][q < m ? q : 0];
      if (g == 0 && q < m && !P.skip) {
        const long long n0 = s_nlocal, n1 = n0 - P.nr + P.na;
        double delta = 0.0;
        // every move changes the count by -1, 0 or +1; thread 0 prepared the
        // two prior deltas of this round (density.hpp:223-237)
        if (n1 == n0 + 1) {
          delta = s_prior[0];
        } else if (n1 == n0 - 1) {
          delta = s_prior[1];
        } else if (n1 != n0) {
          if (n1 > n0) {
            for (long long i = n0 + 1; i <= n1; ++i) delta += llam - d.logi[i];
          } else {
            for (long long i = n1 + 1; i <= n0; ++i) delta -= llam - d.logi[i];
          }
          delta += (double)(n1 - n0) * lxa_r;
        }
        delta += A;
        delta += sig;
        if (MODE == 0) {  // proposal log densities (proposals.hpp:100-104,120-126)
          const int k = s_nown;
          if (P.type == 0) {
            P.logq_f = sp.logw[0] - log_len - d.log_xmax + A;
            P.logq_r = sp.logw[1] - s_logi_k[k + 1];
          } else if (P.type == 1) {
            P.logq_f = sp.logw[1] - s_logi_k[k];
            P.logq_r = sp.logw[0] - log_len - d.log_xmax - A;
          }
        }
        const double log_r = delta + P.logq_r - P.logq_f;
        bool acc_gpu = log_r >= 0.0;
        if (!acc_gpu) acc_gpu = P.logu < log_r;
        s_delta[q] = delta;
        s_logr[q] = log_r;
        s_accg[q] = acc_gpu ? 1 : 0;
        s_cnt[q] = c;
      }
    }
    __syncwarp();
    if (tid == 0) {
      const long long now = clock64();
      tprof[5] += now - tc;
    }
    if (tid == 0) {
      int adv = m, accq = -1;
      for (int q = 0; q < m; ++q) {
        Prop& P = prop[buf][q];
        if (MODE == 1 && P.bad) {
          set_err(ctl, ERR_TAPE_UNKNOWN_ID);
          s_abort = 1;
          adv = q + 1;
          break;
        }
        if (P.scored) ++n_scored;
        if (P.skip) {
          // null (no draw), constrained out, or out of support: log_r = -inf
          // -> reject (proposals.hpp:268-291)
          if (pa.out) {
            seis_step_out o;
            o.delta = -INFINITY;
            o.log_r = -INFINITY;
            o.scored = P.scored;
            o.accepted = 0;
            pa.out[P.tape_idx] = o;
          }
          continue;
        }
        if (P.type <= 1) ++s_bd_scored;
        n_changed += (unsigned long long)s_cnt[q];
        n_arr += (P.type == 3) ? 2ull : (unsigned long long)d.S * (P.nr + P.na);
        const double delta = s_delta[q], log_r = s_logr[q];
        const bool acc_gpu = s_accg[q] != 0;
        bool apply = acc_gpu;
        if (pa.out) {  // replay, or a production run asked for its decisions
          seis_step_out o;
          o.delta = delta;
          o.log_r = log_r;
          o.scored = 1;
          o.accepted = acc_gpu ? 1 : 0;
          pa.out[P.tape_idx] = o;
        }
        if (MODE == 1) apply = P.tape_acc != 0;  // keep the state on the tape's trajectory
        P.accept = 0;
        if (!apply) continue;
        // allocate destination slots; modify this-phase versions in place
        bool ok = true;
        for (int a = 0; a < P.na; ++a) {
          // the new version's kind (spec v2): a birth of a compact run, and a
          // location / joint move or a first arrival override of a generated
          // version, stay generated; everything else is a stored row
          int gen = 0;
          if (MODE == 0 && GEN) {
            if (P.type == 0) {
              gen = pa.compact;
            } else {
              const int rs = P.rslot[a < P.nr ? a : 0];
              if (rs < -1) gen = P.type == 3 ? (d.gv[-2 - rs].n_ovr < kGenOvr ? 1 : 0) : 1;
            }
          }
          P.dgen[a] = gen;
          if (a < P.nr && P.rsidx[a] < 0 && (!GEN || (P.rslot[a] < -1) == (gen != 0))) {
            P.dslot[a] = P.rslot[a];
            P.inplace[a] = 1;
          } else {
            P.inplace[a] = 0;
            int got = -1;  // a slot of the same kind freed earlier this phase
            if (!GEN) {
              if (nlfree > 0) got = lfree[--nlfree];
            } else {
              for (int k2 = nlfree - 1; k2 >= 0; --k2)
                if ((lfree[k2] < -1) == (gen != 0)) {
                  got = lfree[k2];
                  lfree[k2] = lfree[--nlfree];
                  break;
                }
            }
            if (got != -1) {
              P.dslot[a] = got;
            } else if (gen) {
              const int top = atomicSub(&ctl->gv_top, 1) - 1;
              if (top < 0) {
                atomicAdd(&ctl->gv_top, 1);
                set_err(ctl, ERR_GEN_EXHAUSTED);
                ok = false;
                break;
              }
              P.dslot[a] = -2 - d.gv_free[top];
            } else {
              const int top = atomicSub(&ctl->free_top, 1) - 1;
              if (top < 0) {
                atomicAdd(&ctl->free_top, 1);  // undo the failed pop: the stack stays valid
                set_err(ctl, ERR_POOL_EXHAUSTED);
                ok = false;
                break;
              }
              P.dslot[a] = pa.free_stack[top];
            }
          }
        }
        if (ok && P.na >= 1 && nown - P.nr + P.na > CAP) {
          if (!kBig && pa.retry) {
            // hand the region to the whole-chain variant, with every version
            // slot this chain took (the rerun reuses them first)
            int* rf = pa.retry_free + (size_t)slot_idx * kRetryFree;
            int nrf = 0;
            for (int a = 0; a < P.na; ++a)
              if (!P.inplace[a]) rf[1 + nrf++] = P.dslot[a];
            for (int j = 0; j < nown; ++j)
              if (own[j].sidx < 0) rf[1 + nrf++] = own[j].slot;
            for (int k2 = 0; k2 < nlfree; ++k2) rf[1 + nrf++] = lfree[k2];
            rf[0] = nrf;
            pa.retry[slot_idx] = 1;
            s_abort = 1;
            adv = q + 1;
            break;
          }
          set_err(ctl, ERR_OWN_OVERFLOW);
          ok = false;
        }
        if (!ok) {
          s_abort = 1;
          adv = q + 1;
          break;
        }
        P.accept = 1;
        ++n_acc;
        if (P.type <= 1) ++s_bd_acc;
        if (P.type == 0) ++births;
        // retire removed versions; deaths of this-phase versions free slots
        for (int r = 0; r < P.nr; ++r) {
          const int sidx = P.rsidx[r];
          if (sidx >= 0)
            st[sidx].current = 0;
          else if (!(r < P.na && P.inplace[r]))
            lfree[nlfree++] = P.rslot[r];
        }
        // apply_change (density.hpp:171-180): erase by id, push_back added
        unsigned long long rid[2];
        int rsrc[2] = {-1, -1};
        for (int r = 0; r < P.nr; ++r) {
          rid[r] = own[P.rown[r]].id;
          if constexpr (kBig) rsrc[r] = own_src(own[P.rown[r]].sidx);
        }
        for (int r = 0; r < P.nr; ++r) {
          int i = 0;
          while (i < nown && own[i].id != rid[r]) ++i;
          for (int j = i; j + 1 < nown; ++j) own[j] = own[j + 1];
          --nown;
        }
        for (int a = 0; a < P.na; ++a) {
          OwnEv e;
          e.id = P.type == 0 ? P.aid : rid[a];
          e.x = P.ax[a];
          e.t = P.at[a];
          e.slot = P.dslot[a];
          // serial chain: a modified start event keeps its start index, encoded
          e.sidx = (!kBig || P.type == 0 || rsrc[a] < 0) ? -1 : -rsrc[a] - 2;
          own[nown++] = e;
        }
        n_local += P.na - P.nr;
        // own diff vs the phase-start snapshot (frozen-snapshot view) as
        // (start version, current version) pairs, in start order, then the
        // births; O(nstart + nown) through each event's start index
        np = 0;
        if constexpr (kBig) {
          for (int i = 0; i < nstart; ++i) cur_of[i] = -1;
          for (int j = 0; j < nown; ++j)
            if (own_src(own[j].sidx) >= 0) cur_of[own_src(own[j].sidx)] = j;
        }
        for (int i = 0; i < nstart; ++i)
          if (!st[i].current) {
            int f = -1;
            if constexpr (kBig) {
              f = cur_of[i];
            } else {  // a region chain holds few events: search by id
              for (int j = 0; j < nown; ++j)
                if (own[j].id == st[i].id) {
                  f = j;
                  break;
                }
            }
            pold[np] = st[i].slot;
            pnew[np++] = f >= 0 ? own[f].slot : -1;
          }
        for (int i = 0; i < nown; ++i)
          if (own[i].sidx < 0 && own[i].id >= pa.next_base) {
            pold[np] = -1;
            pnew[np++] = own[i].slot;
          }
        if (MODE == 1 && P.type == 0 && P.aid != id_base + births - 1)
          atomicAdd(&ctl->id_mismatch, 1ull);
        accq = q;
        adv = q + 1;
        s_dc_dirty = 1;
        s_tw_dirty = 1;
        break;
      }
      n_spec += (unsigned long long)(m - adv);
      if (pa.naive && pa.record_every > 0) {
        // checkpoints at local steps c * record_every (and the end) inside
        // (i0, i0 + adv]: every step before the round's accept was rejected
        const int hi_step = i0 + adv;
        int c = i0 / pa.record_every + 1;
        for (int cb = c * pa.record_every; ; cb += pa.record_every, ++c) {
          const int at = cb < (int)sp.k ? cb : (int)sp.k;
          if (at > hi_step) break;
          pa.cp_counts[(size_t)c * pa.nreg + region] = at == hi_step ? nown : s_nown;
          if (at == (int)sp.k) break;
        }
      }
      s_bd_hot = (s_bd_scored >= 4 && 8 * s_bd_acc > s_bd_scored) ? 1 : 0;
      s_adv = adv;
      s_accq = accq;
      s_specok = (MODE == 0 && accq < 0 && m_next > 0) ? 1 : 0;
      s_nown = nown;
      s_np = np;
      s_births = births;
      s_nlocal = n_local;
    }
    __syncthreads();  // S3: decision
    if (tid == 0) {
      const long long now = clock64();
      tprof[2] += now - tc;
      tc = now;
      tprof[4] += 1;
    }
    if (s_abort) return;
    const int accq = s_accq;
    if (accq >= 0) {
      // write the accepted version's arrivals (recomputed exactly as scored)
      const Prop& P = prop[buf][accq];
      const int step = (int)(pa.step_base + i0 + accq);  // chain step (philox counter)
      double2* pool2 = reinterpret_cast<double2*>(d.pool);
      const double2* st2 = reinterpret_cast<const double2*>(d.stations);
      if (MODE == 0 && GEN && tid == 0) {  // generated versions: their descriptors (spec v2)
        for (int a = 0; a < P.na; ++a) {
          if (!P.dgen[a]) continue;
          GenV g;
          if (P.type == 0) {
            g.seed = sp.seed;
            g.sweep = (unsigned)pa.epoch;
            g.region = (unsigned)region;
            g.step = (unsigned)step;
            g.n_ovr = 0;
          } else {
            g = *gv_of(d, P.rslot[a]);  // (read before an in-place write)
            if (P.type == 3) {
              g.ovr_st[g.n_ovr] = P.arr_st;
              g.ovr_d[g.n_ovr] = P.arr_da;
              ++g.n_ovr;
            }
          }
          g.x = P.ax[a];
          g.t = P.at[a];
          d.gv[-2 - P.dslot[a]] = g;
        }
      }
      if (MODE == 0 && P.type == 3) {
        if (GEN && P.dgen[0]) {
          // nothing to write: the override lives in the descriptor
        } else if (P.inplace[0]) {
          if (tid == 0) {
            double& a = d.pool[(size_t)P.dslot[0] * d.S_pad + P.arr_st];
            a = a + P.arr_da;
          }
        } else {
          const int rs = P.rslot[0];
          for (int p = tid; p < d.P2; p += NTT) {
            double2 v;
            if (!GEN || rs >= 0) {
              v = pool2[(size_t)rs * d.P2 + p];
            } else {  // a generated version with an override: materialised
              v.x = 2 * p < d.S ? arr_of(d, rs, 2 * p) : 0.0;
              v.y = 2 * p + 1 < d.S ? arr_of(d, rs, 2 * p + 1) : 0.0;
            }
            if (2 * p == P.arr_st) v.x = v.x + P.arr_da;
            if (2 * p + 1 == P.arr_st) v.y = v.y + P.arr_da;
            pool2[(size_t)P.dslot[0] * d.P2 + p] = v;
          }
        }
      } else {
        for (int a = 0; a < P.na; ++a) {
          if (MODE == 0 && GEN && P.dgen[a]) continue;
          for (int p = tid; p < d.P2; p += NTT) {
            const double2 s = st2[p];
            const double m0 = arrival_mean(d, P.ax[a], P.at[a], s.x);
            const double m1 = arrival_mean(d, P.ax[a], P.at[a], s.y);
            double2 v;
            if (MODE == 1) {
              const double* row = pa.tape_arr + P.tape_off + (size_t)a * d.S;
              v.x = 2 * p < d.S ? row[2 * p] : 0.0;
              v.y = 2 * p + 1 < d.S ? row[2 * p + 1] : 0.0;
            } else if (P.type == 0) {
              float z0, z1;
              seis_normal_pair(sp.seed, (uint32_t)pa.epoch, (uint32_t)region, (uint32_t)step,
                               (uint32_t)p, &z0, &z1);
              v.x = m0 + d.sigma * (double)z0;
              v.y = m1 + d.sigma * (double)z1;
            } else {
              const double2 o = pool2[(size_t)P.rslot[a] * d.P2 + p];
              v.x = o.x + (m0 - arrival_mean(d, P.rx[a], P.rt[a], s.x));
              v.y = o.y + (m1 - arrival_mean(d, P.rx[a], P.rt[a], s.y));
            }
            pool2[(size_t)P.dslot[a] * d.P2 + p] = v;
          }
        }
      }
    }
    i0 += s_adv;
  }
  __syncthreads();
  // ---- phase outputs (the barrier merge, samplers.hpp:459-462,471-482)
  if (tid == 0) {
    // fates of the phase-start versions
    if constexpr (kBig) {
      for (int i = 0; i < nstart; ++i) cur_of[i] = -1;
      for (int j = 0; j < nown; ++j)
        if (own_src(own[j].sidx) >= 0) cur_of[own_src(own[j].sidx)] = j;
    }
    for (int i = 0; i < nstart; ++i) {
      const int tab = st[i].tab;
      pa.fate_stamp[tab] = stamp;
      int f = -1;
      if constexpr (kBig) {
        f = cur_of[i];
      } else {
        for (int j = 0; j < nown; ++j)
          if (own[j].id == st[i].id) {
            f = j;
            break;
          }
      }
      pa.fate_alive[tab] = f >= 0;
      if (f >= 0) {
        pa.fate_x[tab] = own[f].x;
        pa.fate_t[tab] = own[f].t;
        pa.fate_slot[tab] = own[f].slot;
      }
    }
    // births alive at phase end, sorted by id
    // a rerun region writes past MAXOWN / MAXDOUT: an overflow area
    if (kBig && pa.retry_pass && pa.ovf.slot) {
      const int k = atomicAdd(pa.ovf.count, 1);
      if (k >= pa.ovf.cap) {
        set_err(ctl, ERR_OWN_OVERFLOW);
        pa.births_cnt[slot_idx] = 0;
        pa.diff_cnt[slot_idx] = 0;
        return;  // (thread 0 alone from here on)
      }
      pa.ovf.slot[slot_idx] = k;
    }
    OutEv* bo = pa.births + births_off(pa.ovf, pa.n_slots, slot_idx);
    int nb = 0;
    for (int j = 0; j < nown; ++j)
      if (own[j].id >= pa.next_base) {
        OutEv e;
        e.id = own[j].id;
        e.x = own[j].x;
        e.t = own[j].t;
        e.slot = own[j].slot;
        e.pad = 0;
        int q = nb++;
        while (q > 0 && bo[q - 1].id > e.id) {
          bo[q] = bo[q - 1];
          --q;
        }
        bo[q] = e;
      }
    pa.births_cnt[slot_idx] = nb;
    if (pa.births_total) pa.births_total[slot_idx] = (int)births;
    if (pa.order_io) {
      pa.order_io[0] = (unsigned long long)nown;
      for (int j = 0; j < nown; ++j) pa.order_io[1 + j] = own[j].id;
    }
    // coverage diff for the commit, then this-phase versions that died (sign
    // 0): k_commit returns those slots to the pool, after every CTA of this
    // phase has stopped popping from it
    DiffPair* dout = pa.diff + diff_off(pa.ovf, pa.n_slots, slot_idx);
    for (int q = 0; q < np; ++q) {
      dout[q].old_slot = pold[q];
      dout[q].new_slot = pnew[q];
      dout[q].kind = 0;
    }
    for (int q = 0; q < nlfree; ++q) {
      dout[np + q].old_slot = lfree[q];
      dout[np + q].new_slot = -1;
      dout[np + q].kind = 1;
    }
    pa.diff_cnt[slot_idx] = np + nlfree;
    atomicAdd(&ctl->scored, n_scored);
    atomicAdd(&ctl->changed, n_changed);
    atomicAdd(&ctl->arrvals, n_arr);
    atomicAdd(&ctl->accepted, n_acc);
    atomicAdd(&ctl->speculative, n_spec);
    for (int q = 0; q < 6; ++q) atomicAdd(&ctl->prof[q], (unsigned long long)tprof[q]);
    const unsigned long long dur = (unsigned long long)(clock64() - z.t0);
    atomicMax(&ctl->prof[6], dur);  // slowest region chain of the run
    atomicAdd(&ctl->prof[7], dur);
    for (int q = 0; q < 16; ++q) atomicAdd(&ctl->tprof[q >> 3][q & 7], s_tprof[q >> 3][q & 7]);
  }
}

// host entry points of one instantiation (declared in phase_api.h)
template <typename YT, int MODE, int CAP, bool GEN, bool TM>
void phase_launch(int grid, int smem, cudaStream_t st, const Dev& d, const Samp& sp,
                  const PhaseArgs& pa, Ctl* ctl, int stamp) {
  k_phase<YT, MODE, NT, SEIS_MINB, CAP, GEN, TM><<<grid, NT, smem, st>>>(d, sp, pa, ctl, stamp);
}
template <typename YT, int MODE, int CAP, bool GEN, bool TM>
cudaError_t phase_set_smem(int bytes) {
  return cudaFuncSetAttribute(k_phase<YT, MODE, NT, SEIS_MINB, CAP, GEN, TM>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace seis
