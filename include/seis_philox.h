/*
 * seis_philox.h — the production-mode random stream of the B200 region-sweep
 * engine ("philox stream spec v1").
 *
 * The reference draws every chain step from one sequential xoshiro256++ stream
 * per (seed, kChain, epoch, color, region) (reference
 * proj/include/seismic/rng.hpp:28-121, proj/include/seismic/samplers.hpp:449-451).
 * A sequential stream serialises the S station normals of a birth, so the GPU
 * engine instead keys a counter-based Philox4x32-10 generator by
 * (seed, sweep, region, step) and a per-step draw index, which lets every
 * thread of a CTA draw its own station's normal independently.
 *
 * Everything here is integer arithmetic or IEEE-754 fp32 operations written
 * with explicit fmaf(), so a host build with -ffp-contract=off and a device
 * build with --fmad=false produce bit-identical draws. The CPU oracle
 * (oracle/seis_oracle.c) includes this header to replay GPU production
 * trajectories exactly.
 *
 * Draw layout per step (counter = {draw, step, region, sweep}, key = seed):
 *   draw 0 : w0w1 -> move-type uniform, w2w3 -> acceptance uniform
 *   draw 1 : w0w1 / w2w3 -> the two scalar draws of the move (birth t and x
 *            uniforms; event / station / partner indices by Lemire reduction)
 *   draw 2 : w0w1 -> joint-pair station-pair index
 *   draw 16+(i>>1) : i-th standard normal of the step from words w0w1 (i
 *            even) or w2w3 (i odd), so one Philox call feeds a station pair
 *            (birth: i = station j; location: 0 = x, 1 = t; arrival: 0;
 *            joint: 0..3)
 *
 * Arrival storage ("philox stream spec v2", seis_set_arrival_storage
 * SEIS_ARR_COMPACT; spec v1 = SEIS_ARR_ROWS stores every version's S fp64
 * arrivals and follows the reference's arithmetic, proposals.hpp:143-174):
 *   birth at (x, t), step key (seed, sweep, region, step): a generated
 *     version; arrival_j = arrival_mean(x, t, j) + sigma * (double) z_j with
 *     z_j = seis_normal(seed, sweep, region, step, j) (the v1 birth values)
 *   location / joint move of a generated version to (x', t'): generated,
 *     same key and override; arrival_j = arrival_mean(x', t', j) + sigma z_j
 *     (+ override): the residual is kept exactly instead of the reference's
 *     a + (m' - m), which differs from it only by rounding
 *   arrival move (station s, delta d) of a generated version with fewer
 *     than 8 overrides: generated, override (s, d) appended; arrival_j =
 *     (mean_j + sigma z_j) + the deltas of the overrides at j in acceptance
 *     order (the v1 values a_s + d); with 8 overrides already: the version
 *     becomes a stored row (its current arrivals, a_s + d at s), v1 rules
 *     from then on
 *   stored rows (a loaded hypothesis, materialised versions): v1 rules
 * The CPU oracle (oracle/seis_oracle.c, so_sampler.compact) implements the
 * same rules; tests/test_gpu_compact.py checks production runs bit-exactly.
 */
#ifndef SEIS_PHILOX_H
#define SEIS_PHILOX_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SEIS_HD __host__ __device__ __forceinline__
#else
#define SEIS_HD static inline
#endif

#define SEIS_DRAW_MOVE 0u
#define SEIS_DRAW_SCALAR 1u
#define SEIS_DRAW_PAIR 2u
#define SEIS_DRAW_NORMAL0 16u

typedef struct {
  uint32_t w[4];
} seis_u32x4;

SEIS_HD uint32_t seis_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi) {
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

/* Philox4x32 with 10 rounds (Salmon et al., SC'11; constants of Random123). */
SEIS_HD seis_u32x4 seis_philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                      uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    const uint32_t lo0 = seis_mulhilo32(0xD2511F53u, c0, &hi0);
    const uint32_t lo1 = seis_mulhilo32(0xCD9E8D57u, c2, &hi1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  seis_u32x4 out;
  out.w[0] = c0;
  out.w[1] = c1;
  out.w[2] = c2;
  out.w[3] = c3;
  return out;
}

SEIS_HD seis_u32x4 seis_draw(uint64_t seed, uint32_t sweep, uint32_t region, uint32_t step,
                             uint32_t draw) {
  return seis_philox4x32_10(draw, step, region, sweep, (uint32_t)seed,
                            (uint32_t)(seed >> 32));
}

SEIS_HD uint64_t seis_u64(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; }

/* [0, 1) with 53-bit resolution, same transform as the reference's
 * Rng::uniform (rng.hpp:49) applied to a Philox 64-bit word. */
SEIS_HD double seis_u53(uint32_t hi, uint32_t lo) {
  return (double)(seis_u64(hi, lo) >> 11) * 0x1.0p-53;
}

/* [0, n) by Lemire multiply-shift, as the reference's uniform_index
 * (rng.hpp:54-57). */
SEIS_HD uint64_t seis_lemire(uint64_t v, uint64_t n) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(v, n);
#else
  return (uint64_t)(((unsigned __int128)v * n) >> 64);
#endif
}

SEIS_HD float seis_fmaf(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
  return __fmaf_rn(a, b, c);
#else
  return __builtin_fmaf(a, b, c);
#endif
}

SEIS_HD uint32_t seis_f2u(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  union {
    float f;
    uint32_t u;
  } v;
  v.f = f;
  return v.u;
#endif
}

SEIS_HD float seis_u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  union {
    float f;
    uint32_t u;
  } v;
  v.u = u;
  return v.f;
#endif
}

/* Natural log for u in [2^-24, 1], fp32, reproducible: u = m 2^e with
 * m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh((m-1)/(m+1)) by odd series. */
SEIS_HD float seis_lnf(float u) {
  const uint32_t bits = seis_f2u(u);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float m = seis_u2f((bits & 0x7fffffu) | 0x3f800000u);
  if (m > 0x1.6a09e6p+0f) {
    m = m * 0.5f;
    e += 1;
  }
#if defined(__CUDA_ARCH__)
  const float s = __fdiv_rn(m - 1.0f, m + 1.0f);
#else
  const float s = (m - 1.0f) / (m + 1.0f);
#endif
  const float s2 = s * s;
  float p = seis_fmaf(s2, 0x1.c71c72p-4f, 0x1.24924ap-3f);
  p = seis_fmaf(s2, p, 0x1.99999ap-3f);
  p = seis_fmaf(s2, p, 0x1.555556p-2f);
  p = seis_fmaf(s2, p, 1.0f);
  const float lnm = (2.0f * s) * p;
  return seis_fmaf((float)e, 0x1.62e430p-1f, lnm);
}

/* cos(2 pi u) for u in [0, 1), fp32, reproducible quadrant reduction. */
SEIS_HD float seis_cos2pif(float u) {
  const float q = u * 4.0f;
  const int k = (int)q;
  const float f = q - (float)k;
  const float th = f * 0x1.921fb6p+0f;
  const float t2 = th * th;
  float c = seis_fmaf(t2, 0x1.1eed8ep-29f, -0x1.27e4fcp-22f);
  c = seis_fmaf(t2, c, 0x1.a01a02p-16f);
  c = seis_fmaf(t2, c, -0x1.6c16c2p-10f);
  c = seis_fmaf(t2, c, 0x1.555556p-5f);
  c = seis_fmaf(t2, c, -0.5f);
  c = seis_fmaf(t2, c, 1.0f);
  float s = seis_fmaf(t2, -0x1.ae6456p-26f, 0x1.71de3ap-19f);
  s = seis_fmaf(t2, s, -0x1.a01a02p-13f);
  s = seis_fmaf(t2, s, 0x1.111112p-7f);
  s = seis_fmaf(t2, s, -0x1.555556p-3f);
  s = seis_fmaf(t2, s, 1.0f);
  s = s * th;
  /* quadrant k & 3 -> c, -s, -c, s: selects, not a switch (lanes of a warp
   * sit in different quadrants) */
  const float v = (k & 1) ? s : c;
  return ((k + 1) & 2) ? -v : v;
}

/* Standard normal from two 32-bit words: Box-Muller, cosine branch (as the
 * reference's Rng::normal, rng.hpp:60-65), in reproducible fp32. */
SEIS_HD float seis_bm(uint32_t w0, uint32_t w1) {
  const float u1 = (float)((w0 >> 8) + 1u) * 0x1.0p-24f; /* (0, 1] */
  const float u2 = (float)(w1 >> 8) * 0x1.0p-24f;        /* [0, 1) */
#if defined(__CUDA_ARCH__)
  const float r = __fsqrt_rn(-2.0f * seis_lnf(u1));
#else
  const float r = __builtin_sqrtf(-2.0f * seis_lnf(u1));
#endif
  return r * seis_cos2pif(u2);
}

SEIS_HD float seis_normal(uint64_t seed, uint32_t sweep, uint32_t region, uint32_t step,
                          uint32_t i) {
  const seis_u32x4 d = seis_draw(seed, sweep, region, step, SEIS_DRAW_NORMAL0 + (i >> 1));
  /* pick the words first: neighbouring lanes (stations) have opposite parity */
  const uint32_t a = (i & 1u) ? d.w[2] : d.w[0];
  const uint32_t b = (i & 1u) ? d.w[3] : d.w[1];
  return seis_bm(a, b);
}

/* normals 2i and 2i+1 of a step from one Philox call */
SEIS_HD void seis_normal_pair(uint64_t seed, uint32_t sweep, uint32_t region, uint32_t step,
                              uint32_t i2, float* z0, float* z1) {
  const seis_u32x4 d = seis_draw(seed, sweep, region, step, SEIS_DRAW_NORMAL0 + i2);
  *z0 = seis_bm(d.w[0], d.w[1]);
  *z1 = seis_bm(d.w[2], d.w[3]);
}

#endif /* SEIS_PHILOX_H */
