/*
 * hs_oracle_rng.c -- TEST INFRASTRUCTURE ONLY (see hs_oracle.h).
 *
 * A plain-C restatement of the seeded streams the reference draws from
 * numpy.random.default_rng(seed).  numpy is a third-party dependency of the
 * reference (pinned here: numpy 2.3.5) and is not vendored under
 * /root/reference, so this file restates numpy's published algorithms and
 * parity is anchored on the reference's own call sites:
 *
 *   cli.py:160-193        _sample_lengths: rng.lognormal(mu, sigma, size=n) or
 *                         rng.integers(lo, hi + 1, size=n).astype(float), then
 *                         int(min(max(round(v), 1), upper)); cmd_gen_trace draws
 *                         inputs then outputs from ONE generator
 *   simulator.py:112-124  generate_arrivals: np.cumsum(rng.exponential(1/rate, n))
 *   scheduling.py:87-95   OutputLengthPredictor: round(rng.normal(mean, sd)),
 *                         clamped to [1, max_output_len]
 *
 * numpy pieces restated (numpy/random/src/...):
 *   pcg64/pcg64.h            XSL-RR 128/64 step + output, next32 buffering
 *   distributions.c          random_standard_normal / _exponential (256-layer
 *                            ziggurat, tables in include/hs_ziggurat_tables.h),
 *                            random_normal, random_lognormal, random_exponential,
 *                            random_bounded_uint64_fill (Lemire, next32 path
 *                            for ranges below 2^32)
 *   libm                     exp and log1p as glibc 2.39 evaluates them on an
 *                            FMA x86-64 host (hs_oracle_exp; hs_oracle_log1p
 *                            below restates sysdeps/ieee754/dbl-64/s_log1p.c
 *                            with the contractions of the FMA ifunc variant).
 *
 * Pinned by tests/test_oracle_rng.py against numpy itself.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "hs_oracle.h"
#include "../include/hs_ziggurat_tables.h"

typedef unsigned __int128 u128;

static const double kNorR = 3.6541528853610087963519472518;
static const double kNorInvR = 0.27366123732975827203338247596;
static const double kExpR = 7.6971174701310497140446280481;

/* ---------------------------------------------------------------- log1p */
static inline int32_t hi_word(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (int32_t)(u >> 32);
}
static inline double with_hi_word(double x, uint32_t hi) {
  uint64_t u;
  memcpy(&u, &x, 8);
  u = ((uint64_t)hi << 32) | (u & 0xffffffffull);
  memcpy(&x, &u, 8);
  return x;
}

/* glibc 2.39 log1p (fdlibm s_log1p.c) as its FMA ifunc variant evaluates it:
 * the polynomial's products fold into fused multiply-adds, as do k*ln2_lo + c
 * and the final k*ln2_hi - (...).  The small-negative window that takes the
 * u = 1 + x path is 0xbfd2bec4 <= hx <= 0 (as the compiled code tests it). */
double hs_oracle_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  int32_t hx = hi_word(x), ax = hx & 0x7fffffff, hu = 0, k = 1;
  double f = 0.0, c = 0.0;
  if (hx < 0x3fda827a) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return fma(-(x * x), 0.5, x);
    }
    if (hx > 0 || hx < (int32_t)0xbfd2bec4) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, (uint32_t)hu | 0x3ff00000u);
    } else {
      k += 1;
      u = with_hi_word(u, (uint32_t)hu | 0x3fe00000u);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  double hfsq = (0.5 * f) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      double dk = (double)k;
      return fma(dk, ln2_hi, fma(dk, ln2_lo, c));
    }
    double R = fma(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    double dk = (double)k;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  double s = f / (2.0 + f);
  double z = s * s;
  double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
  double z2 = z * z;
  double z4 = z2 * z2;
  double z6 = z2 * z4;
  double R = fma(z, Lp1, z2 * R2);
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  double t = s * (R + hfsq);
  if (k == 0) return f - (hfsq - t);
  double dk = (double)k;
  return fma(dk, ln2_hi, -((hfsq - (fma(dk, ln2_lo, c) + t)) - f));
}

/* ---------------------------------------------------------------- PCG64 */
static const u128 kPcgMult = ((u128)2549297995355413924ull << 64) | 4865540595714422341ull;

uint64_t hs_oracle_pcg64_next64(hs_pcg64_state* g) {
  u128 st = ((u128)g->state_hi << 64) | g->state_lo;
  u128 inc = ((u128)g->inc_hi << 64) | g->inc_lo;
  st = st * kPcgMult + inc;
  g->state_hi = (uint64_t)(st >> 64);
  g->state_lo = (uint64_t)st;
  uint64_t x = g->state_hi ^ g->state_lo;
  unsigned rot = (unsigned)(g->state_hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t next32(hs_pcg64_state* g) {
  if (g->has_uint32) {
    g->has_uint32 = 0;
    return g->uinteger;
  }
  uint64_t n = hs_oracle_pcg64_next64(g);
  g->has_uint32 = 1;
  g->uinteger = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

static double next_double(hs_pcg64_state* g) {
  return (double)(hs_oracle_pcg64_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------- ziggurat */
double hs_oracle_std_normal(hs_pcg64_state* g) {
  int of;
  for (;;) {
    uint64_t r = hs_oracle_pcg64_next64(g);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * kZig_wi[idx];
    if (sign) x = -x;
    if (rabs < kZig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -kNorInvR * hs_oracle_log1p(-next_double(g));
        double yy = -hs_oracle_log1p(-next_double(g));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(kNorR + xx) : kNorR + xx;
      }
    }
    double u = next_double(g);
    if ((kZig_fi[idx - 1] - kZig_fi[idx]) * u + kZig_fi[idx] < hs_oracle_exp(-0.5 * x * x, &of)) return x;
  }
}

double hs_oracle_std_exp(hs_pcg64_state* g) {
  int of;
  for (;;) {
    uint64_t ri = hs_oracle_pcg64_next64(g) >> 3;
    int idx = (int)(ri & 0xff);
    ri >>= 8;
    double x = (double)ri * kZig_we[idx];
    if (ri < kZig_ke[idx]) return x;
    if (idx == 0) return kExpR - hs_oracle_log1p(-next_double(g));
    double u = next_double(g);
    if ((kZig_fe[idx - 1] - kZig_fe[idx]) * u + kZig_fe[idx] < hs_oracle_exp(-x, &of)) return x;
  }
}

/* random_bounded_uint64_fill, one value (Lemire; next32 below 2^32). */
static uint64_t bounded(hs_pcg64_state* g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng <= 0xffffffffull) {
    if (rng == 0xffffffffull) return next32(g);
    uint32_t rx = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)next32(g) * rx;
    uint32_t left = (uint32_t)m;
    if (left < rx) {
      uint32_t th = (UINT32_MAX - (uint32_t)rng) % rx;
      while (left < th) {
        m = (uint64_t)next32(g) * rx;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
  if (rng == UINT64_MAX) return hs_oracle_pcg64_next64(g);
  uint64_t rx = rng + 1;
  u128 m = (u128)hs_oracle_pcg64_next64(g) * rx;
  uint64_t left = (uint64_t)m;
  if (left < rx) {
    uint64_t th = (UINT64_MAX - rng) % rx;
    while (left < th) {
      m = (u128)hs_oracle_pcg64_next64(g) * rx;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

/* int(min(max(round(v), 1), cap)); -1 when round() would raise. */
static int64_t clamp_len(double v, int32_t cap) {
  if (!isfinite(v)) return -1;
  double r = rint(v);
  if (r < 1.0) return 1;
  if (r > (double)cap) return cap;
  return (int64_t)r;
}

int64_t hs_oracle_rng_fill(hs_pcg64_state* g, const hs_dist* d, int64_t n, void* out) {
  int64_t bad = -1;
  int32_t* oi = (int32_t*)out;
  double* od = (double*)out;
  int of;
  switch (d->kind) {
    case HS_DIST_LOGNORMAL_LEN:
    case HS_DIST_NORMAL_LEN:
      for (int64_t i = 0; i < n; ++i) {
        double v = d->p0 + d->p1 * hs_oracle_std_normal(g);
        if (d->kind == HS_DIST_LOGNORMAL_LEN) v = hs_oracle_exp(v, &of);
        int64_t L = clamp_len(v, d->cap);
        if (L < 0 && bad < 0) bad = i;
        oi[i] = L < 0 ? 0 : (int32_t)L;
      }
      break;
    case HS_DIST_UNIFORM_LEN: {
      uint64_t rng = (uint64_t)d->hi - (uint64_t)d->lo;
      for (int64_t i = 0; i < n; ++i) {
        int64_t v = (int64_t)((uint64_t)d->lo + bounded(g, rng));
        oi[i] = v < 1 ? 1 : (v > d->cap ? d->cap : (int32_t)v);
      }
      break;
    }
    case HS_DIST_EXP_CUMSUM: {
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double gap = d->p0 * hs_oracle_std_exp(g);
        acc = i == 0 ? gap : acc + gap;
        od[i] = acc;
      }
      break;
    }
    default:
      return -2;
  }
  return bad;
}

/* Batch: stream t fills dists[0..n_dists) in order over its own slice. */
int hs_oracle_rng_generate(hs_pcg64_state* states, int32_t n_streams, const int64_t* offsets,
                           const hs_dist* dists, int32_t n_dists, void* const* out, int64_t* bad_index) {
  for (int32_t t = 0; t < n_streams; ++t) {
    int64_t a = offsets[t], n = offsets[t + 1] - a, bad = -1;
    for (int32_t j = 0; j < n_dists; ++j) {
      size_t w = dists[j].kind == HS_DIST_EXP_CUMSUM ? 8 : 4;
      int64_t b = hs_oracle_rng_fill(&states[t], &dists[j], n, (char*)out[j] + (size_t)a * w);
      if (b == -2) return HS_ERR_ARG;
      if (b >= 0 && bad < 0) bad = b;
    }
    if (bad_index) bad_index[t] = bad;
  }
  return HS_OK;
}
