// hs_device.cuh -- device-side fp64 semantics of the reference (CPython 3.12
// on glibc 2.39), shared by the search and replay kernels.
//
// Everything is evaluated exactly as CPython evaluates the reference
// expressions: left to right, one rounding per operation (the library is
// compiled with -fmad=false so nvcc never contracts a*b+c; the only fused
// operations are the explicit __fma_rn calls of the exp port, which mirror
// the vfmadd instructions of glibc's FMA exp body).
#pragma once
#include <stdint.h>

#define HS_TABLE __device__ const
#include "../../include/hs_exp_table.h"

namespace hs {

__device__ __forceinline__ double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }

// Python float(int) for |v| < 2^63: correctly rounded (PyLong_AsDouble).
__device__ __forceinline__ double i2d(int64_t v) { return __ll2double_rn(v); }

// Saturating int64 helpers (values are non-negative byte/token counts; a
// saturated value compares greater than any budget below 2^63).
__device__ __forceinline__ int64_t sat_mul(int64_t a, int64_t b) {
  if (a == 0 || b == 0) return 0;
  if (a > INT64_MAX / b) return INT64_MAX;
  return a * b;
}
__device__ __forceinline__ int64_t sat_add(int64_t a, int64_t b) {
  return (a > INT64_MAX - b) ? INT64_MAX : a + b;
}

// latency.py:90-92  p1*b*I + p2*b + p3*I + p4
__device__ __forceinline__ double prefill_time(const double* p, int64_t b, int64_t I) {
  double db = i2d(b), dI = i2d(I);
  double x = __dmul_rn(__dmul_rn(p[0], db), dI);
  x = __dadd_rn(x, __dmul_rn(p[1], db));
  x = __dadd_rn(x, __dmul_rn(p[2], dI));
  return __dadd_rn(x, p[3]);
}

// latency.py:95-97  p5*b*c + p6*b + p7*c + p8
__device__ __forceinline__ double decode_iteration_time(const double* p, int64_t cached, int64_t b) {
  double db = i2d(b), dc = i2d(cached);
  double x = __dmul_rn(__dmul_rn(p[4], db), dc);
  x = __dadd_rn(x, __dmul_rn(p[5], db));
  x = __dadd_rn(x, __dmul_rn(p[6], dc));
  return __dadd_rn(x, p[7]);
}

// latency.py:100-109 closed form: S = O*I + O*(O+1)/2.0;
// (p5*b + p7)*S + (p6*b + p8)*O
__device__ __forceinline__ double decode_time(const double* p, int64_t b, int64_t I, int64_t O) {
  double S = __dadd_rn(i2d(O * I), __ddiv_rn(i2d(O * (O + 1)), 2.0));
  double db = i2d(b);
  double a = __dmul_rn(__dadd_rn(__dmul_rn(p[4], db), p[6]), S);
  double c = __dmul_rn(__dadd_rn(__dmul_rn(p[5], db), p[7]), i2d(O));
  return __dadd_rn(a, c);
}

// CPython float floor division (Objects/floatobject.c _float_div_mod); here
// both operands are positive (scheduling.py:128: budget > 0, bytes > 0).
// fmod(x, y) for x >= 0, 0 < y < inf: x - n*y with n = trunc(x/y) is exactly
// representable, q = trunc(fl(x/y)) is n or n +- 1 below 2^52, and one FMA
// with the right q yields that remainder exactly (the library fmod is a
// bit-serial loop); anything else takes the library path.
__device__ __forceinline__ double exact_fmod(double vx, double wx) {
  const double q = trunc(__ddiv_rn(vx, wx));
  if (!(vx >= 0.0 && wx > 0.0 && wx < INFINITY && q < 4503599627370496.0)) return fmod(vx, wx);
  double r = __fma_rn(-q, wx, vx);
  if (r < 0.0) r = __fma_rn(-(q - 1.0), wx, vx);
  else if (r >= wx) r = __fma_rn(-(q + 1.0), wx, vx);
  return r;
}

// x / b rounded to nearest from r = RN(1 / b), for finite positive b and
// finite x: q0 = RN(x r) lies within an ulp of x / b, the FMA residual
// x - q0 b is then exact, and one correction RN(q0 + r (x - q0 b)) is the
// correctly rounded quotient (Markstein's theorem for round-to-nearest) -- the
// IEEE quotient CPython's `/` gives, without the reciprocal refinement of a
// full division.  Pinned against numpy's x / b by tests/test_gpu_floordiv.py.
__device__ __forceinline__ double div_rn_by(double x, double b, double r) {
  const double q0 = __dmul_rn(x, r);
  const double e = __fma_rn(-q0, b, x);
  return __fma_rn(e, r, q0);
}

#ifndef HS_RECIP_DIV
#define HS_RECIP_DIV 1
#endif

__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  {
    // x >= 0, 0 < w < inf, integer quotient n < 2^50: CPython's result is n.
    // Its steps: mod = x - n*w (exact), div = fl(fl(x - mod) / w) with x - mod
    // = n*w, so |div - n| <= n * (2u + u^2) <= 1/4 + 2^-56 (u = 2^-53), and
    // floor(div) (+1 when div - floor(div) > 0.5) lands on n; n itself is
    // trunc(fl(x/w)) corrected by the sign of one exact FMA remainder.
    double q = trunc(__ddiv_rn(vx, wx));
    if (vx >= 0.0 && wx > 0.0 && wx < INFINITY && q < 1125899906842624.0) {
      const double r = __fma_rn(-q, wx, vx);
      if (r < 0.0) q -= 1.0;
      else if (r >= wx) q += 1.0;
      return q;
    }
  }
  double mod = exact_fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) {
      mod = __dadd_rn(mod, wx);
      div = __dsub_rn(div, 1.0);
    }
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
  } else {
    fl = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fl;
}

// CPython 3.12 builtin sum() over floats with int start 0 (Neumaier).
struct PySum {
  double f, c;
  int64_t n;
  __device__ __forceinline__ void init() { f = 0.0; c = 0.0; n = 0; }
  __device__ __forceinline__ void add(double x) {
    if (n++ == 0) { f = __dadd_rn(0.0, x); return; }
    double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
  }
  __device__ __forceinline__ double result() const {
    double r = f;
    if (c != 0.0 && isfinite(c)) r = __dadd_rn(r, c);
    return r;
  }
};

// glibc 2.39 exp, FMA variant (sysdeps/ieee754/dbl-64/e_exp.c compiled with
// FMA contraction; CPython's math.exp on an FMA x86-64 host).  `tab` is the
// 256-entry table (shared or global memory).  *overflow set when CPython
// raises OverflowError.
__device__ __forceinline__ double py_exp(double x, const uint64_t* tab, bool* overflow) {
  const double kInvLn2N = 0x1.71547652b82fep+7;
  const double kShift = 0x1.8p52;
  const double kNegLn2HiN = -0x1.62e42fefa0000p-8;
  const double kNegLn2LoN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  *overflow = false;
  uint64_t ix = d2u(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 969u >= 63u) {
    if ((int32_t)(abstop - 969u) < 0) return __dadd_rn(1.0, x);
    if (abstop >= 1033u) {
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return __dadd_rn(1.0, x);
      if (ix >> 63) return 0.0;
      *overflow = true;
      return __longlong_as_double(0x7ff0000000000000ll);
    }
    abstop = 0;
  }
  double kd = __fma_rn(x, kInvLn2N, kShift);
  uint64_t ki = d2u(kd);
  kd = __dsub_rn(kd, kShift);
  double r = __fma_rn(kd, kNegLn2HiN, x);
  r = __fma_rn(kd, kNegLn2LoN, r);
  uint32_t idx = 2u * (uint32_t)(ki & 127u);
  uint64_t top = ki << 45;
  double tail = u2d(tab[idx]);
  uint64_t sbits = tab[idx + 1] + top;
  double a = __fma_rn(r, C3, C2);
  double t1 = __dadd_rn(r, tail);
  double r2 = __dmul_rn(r, r);
  double b = __fma_rn(r, C5, C4);
  double tmp = __fma_rn(a, r2, t1);
  double r4 = __dmul_rn(r2, r2);
  tmp = __fma_rn(r4, b, tmp);
  if (abstop == 0) {
    if ((ki & 0x80000000u) == 0) {
      double scale = u2d(sbits - (1009ull << 52));
      double y = __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
      if (isinf(y)) *overflow = true;
      return y;
    }
    double scale = u2d(sbits + (1022ull << 52));
    double st = __dmul_rn(scale, tmp);
    double y = __dadd_rn(scale, st);
    if (y < 1.0) {
      double lo = __dadd_rn(__dsub_rn(scale, y), st);
      double hi = __dadd_rn(1.0, y);
      lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
      y = __dsub_rn(__dadd_rn(lo, hi), 1.0);
      if (y == 0.0) y = 0.0;
    }
    return __dmul_rn(0x1p-1022, y);
  }
  double scale = u2d(sbits);
  return __fma_rn(scale, tmp, scale);
}

// glibc 2.39 log1p, FMA variant (sysdeps/ieee754/dbl-64/s_log1p.c compiled
// with FMA contraction; what numpy's ziggurat tails call on an FMA x86-64
// host).  Restated from the compiled variant's operation order: the
// polynomial and the k*ln2 reconstruction are fused exactly where its
// vfmadd/vfmsub instructions are.
__device__ __forceinline__ double py_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  int32_t hx = __double2hiint(x), ax = hx & 0x7fffffff, hu = 0, k = 1;
  double f = 0.0, c = 0.0;
  if (hx < 0x3fda827a) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -__longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double(0x7ff8000000000000ll);
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx < (int32_t)0xbfd2bec4) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return __dadd_rn(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      double dk = (double)k;
      return __fma_rn(dk, ln2_hi, __fma_rn(dk, ln2_lo, c));
    }
    double R = __dmul_rn(__fma_rn(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    double dk = (double)k;
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  double z = __dmul_rn(s, s);
  double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  double z2 = __dmul_rn(z, z);
  double z4 = __dmul_rn(z2, z2);
  double z6 = __dmul_rn(z2, z4);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  double t = __dmul_rn(s, __dadd_rn(R, hfsq));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  double dk = (double)k;
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(dk, ln2_lo, c), t)), f));
}

// warp helpers --------------------------------------------------------------
__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

}  // namespace hs
