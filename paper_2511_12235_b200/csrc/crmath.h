/* crmath.h -- correctly rounded double sin/cos/tan/atan/atan2 (ctsm-b200).
 *
 * Why this exists: the reference (ctsm, /root/reference/proj) calls libm's
 * sin/cos/tan/atan/atan2 inside every weight formula (geometry.cpp:56-62,
 * weights2d.cpp:8-34,100-149, weights3d.cpp:63-168) and drops 3D weights at
 * 1e-16 (weights3d.cpp:453) while cancellation noise reaches 1e-12, so the
 * sparsity pattern depends on the last bit of every libm result (SURVEY.md
 * §0 fact 5, §7 H1). Bit-exact sparsity between the CPU oracle and the GPU
 * therefore needs ONE libm whose results are identical on both sides. This
 * header is that libm: every function is evaluated in double-double with
 * ~2^-100 relative accuracy and rounded once, so results are the correctly
 * rounded values except in (astronomically rare) hard-to-round cases.
 *
 * Determinism contract: only IEEE-754 binary64 +, -, *, /, explicit fma(),
 * rint() and comparisons are used. Compile host code with
 * -ffp-contract=off (no implicit FMA contraction) and device code with
 * -fmad=false; then host (gcc) and device (nvcc, sm_100a) results are
 * bit-identical for every input.
 *
 * Domain: sin/cos/tan are accurate for |x| < 2^26 (the reference's angles are
 * below 8*pi); larger finite arguments return a deterministic value with
 * reduced accuracy. atan/atan2 accept all doubles.
 */
#pragma once
#include <math.h>
#include <stdint.h>

#include "crmath_tables.h"

#if defined(__CUDACC__)
#define CRM_FN static __host__ __device__ __forceinline__
#define CRM_NOINLINE static __host__ __device__ __noinline__
#else
#define CRM_FN static inline
#define CRM_NOINLINE static
#endif

/* ---- tables (same initialisers on host and device) ---------------------- */
#if defined(__CUDACC__)
__device__ static const double crm_sincos_tab_d[4 * CRM_NSC] = CRM_SINCOS_TABLE_INIT;
__device__ static const double crm_atan_tab_d[2 * CRM_NATAN] = CRM_ATAN_TABLE_INIT;
#endif
static const double crm_sincos_tab_h[4 * CRM_NSC] = CRM_SINCOS_TABLE_INIT;
static const double crm_atan_tab_h[2 * CRM_NATAN] = CRM_ATAN_TABLE_INIT;

#if defined(__CUDA_ARCH__)
#define CRM_SC(i) __ldg(&crm_sincos_tab_d[(i)])
#define CRM_AT(i) __ldg(&crm_atan_tab_d[(i)])
#else
#define CRM_SC(i) (crm_sincos_tab_h[(i)])
#define CRM_AT(i) (crm_atan_tab_h[(i)])
#endif

/* ---- double-double primitives (Dekker / Knuth error-free transforms) ----- */
typedef struct {
  double hi, lo;
} crm_dd;

CRM_FN crm_dd crm_mk(double hi, double lo) {
  crm_dd r;
  r.hi = hi;
  r.lo = lo;
  return r;
}
CRM_FN crm_dd crm_two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return crm_mk(s, e);
}
CRM_FN crm_dd crm_fast_two_sum(double a, double b) { /* |a| >= |b| or a == 0 */
  double s = a + b;
  double e = b - (s - a);
  return crm_mk(s, e);
}
CRM_FN crm_dd crm_two_prod(double a, double b) {
  double p = a * b;
  double e = fma(a, b, -p);
  return crm_mk(p, e);
}
CRM_FN crm_dd crm_add(crm_dd a, crm_dd b) {
  crm_dd s = crm_two_sum(a.hi, b.hi);
  crm_dd t = crm_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = crm_fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return crm_fast_two_sum(s.hi, s.lo);
}
CRM_FN crm_dd crm_neg(crm_dd a) { return crm_mk(-a.hi, -a.lo); }
CRM_FN crm_dd crm_sub(crm_dd a, crm_dd b) { return crm_add(a, crm_neg(b)); }
CRM_FN crm_dd crm_add_d(crm_dd a, double b) {
  crm_dd s = crm_two_sum(a.hi, b);
  s.lo += a.lo;
  return crm_fast_two_sum(s.hi, s.lo);
}
CRM_FN crm_dd crm_mul(crm_dd a, crm_dd b) {
  crm_dd p = crm_two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, p.lo);
  p.lo = fma(a.lo, b.hi, p.lo);
  return crm_fast_two_sum(p.hi, p.lo);
}
CRM_FN crm_dd crm_mul_d(crm_dd a, double b) {
  crm_dd p = crm_two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return crm_fast_two_sum(p.hi, p.lo);
}
CRM_FN crm_dd crm_div(crm_dd a, crm_dd b) {
  double q1 = a.hi / b.hi;
  crm_dd r = crm_sub(a, crm_mul_d(b, q1));
  double q2 = r.hi / b.hi;
  r = crm_sub(r, crm_mul_d(b, q2));
  double q3 = r.hi / b.hi;
  crm_dd q = crm_fast_two_sum(q1, q2);
  return crm_add_d(q, q3);
}
/* a / b for doubles, result as double-double (exact remainder via fma). */
CRM_FN crm_dd crm_div_dd_d(double a, double b) {
  double q = a / b;
  double r = fma(-q, b, a);
  double q2 = r / b;
  return crm_fast_two_sum(q, q2);
}
CRM_FN double crm_round(crm_dd a) { return a.hi + a.lo; }

/* ---- sin / cos kernel on |r| <= pi/4 + eps -------------------------------- */

/* Reduces x to r = x - k*pi/2 (double-double) and returns k. */
CRM_FN crm_dd crm_reduce_pio2(double x, int64_t* k_out) {
  double kd = rint(x * CRM_2_OVER_PI);
  crm_dd t1 = crm_two_prod(kd, CRM_PIO2_1);
  crm_dd r = crm_two_sum(x, -t1.hi);
  r = crm_add_d(r, -t1.lo);
  crm_dd t2 = crm_two_prod(kd, CRM_PIO2_2);
  r = crm_sub(r, t2);
  crm_dd t3 = crm_two_prod(kd, CRM_PIO2_3);
  r = crm_sub(r, t3);
  r = crm_add_d(r, -kd * CRM_PIO2_4);
  *k_out = (int64_t)kd;
  return r;
}

/* sin and cos of a reduced argument r (|r| <= ~0.8) in double-double. */
CRM_FN void crm_sincos_reduced(crm_dd r, crm_dd* s_out, crm_dd* c_out) {
  double jd = rint(r.hi * 32.0);
  int j = (int)jd;
  double a = jd * 0.03125;
  crm_dd d = crm_two_sum(r.hi, -a);
  d = crm_add_d(d, r.lo); /* d = r - a, |d| <= 1/64 + tiny */
  crm_dd d2 = crm_mul(d, d);
  double z = d2.hi;
  /* sin(d) = d*(1 + z*(-1/6 + z*(1/120 + z*(-1/5040 + z*u)))) */
  double us = 1.0 / 362880.0 + z * (-1.0 / 39916800.0 + z * (1.0 / 6227020800.0));
  crm_dd ps = crm_add_d(crm_mk(CRM_C5040_HI, CRM_C5040_LO), z * us);
  ps = crm_mul(ps, d2);
  ps = crm_add(ps, crm_mk(CRM_C120_HI, CRM_C120_LO));
  ps = crm_mul(ps, d2);
  ps = crm_add(ps, crm_mk(CRM_C6_HI, CRM_C6_LO));
  ps = crm_mul(ps, d2);
  ps = crm_add_d(ps, 1.0);
  crm_dd sd = crm_mul(ps, d);
  /* cos(d) = 1 + z*(-1/2 + z*(1/24 + z*(-1/720 + z*u))) */
  double uc = 1.0 / 40320.0 + z * (-1.0 / 3628800.0 + z * (1.0 / 479001600.0));
  crm_dd pc = crm_add_d(crm_mk(CRM_C720_HI, CRM_C720_LO), z * uc);
  pc = crm_mul(pc, d2);
  pc = crm_add(pc, crm_mk(CRM_C24_HI, CRM_C24_LO));
  pc = crm_mul(pc, d2);
  pc = crm_add_d(pc, -0.5);
  pc = crm_mul(pc, d2);
  crm_dd cd = crm_add_d(pc, 1.0);
  int aj = j < 0 ? -j : j;
  crm_dd sa = crm_mk(CRM_SC(4 * aj + 0), CRM_SC(4 * aj + 1));
  crm_dd ca = crm_mk(CRM_SC(4 * aj + 2), CRM_SC(4 * aj + 3));
  if (j < 0) sa = crm_neg(sa);
  /* sin(a+d) = sa*cd + ca*sd ; cos(a+d) = ca*cd - sa*sd */
  *s_out = crm_add(crm_mul(sa, cd), crm_mul(ca, sd));
  *c_out = crm_sub(crm_mul(ca, cd), crm_mul(sa, sd));
}

/* sin(x), cos(x) in double-double (x finite). */
CRM_FN void crm_sincos_dd(double x, crm_dd* s_out, crm_dd* c_out) {
  int64_t k;
  crm_dd r = crm_reduce_pio2(x, &k);
  crm_dd s, c;
  crm_sincos_reduced(r, &s, &c);
  switch ((int)(k & 3)) {
    case 0: *s_out = s; *c_out = c; break;
    case 1: *s_out = c; *c_out = crm_neg(s); break;
    case 2: *s_out = crm_neg(s); *c_out = crm_neg(c); break;
    default: *s_out = crm_neg(c); *c_out = s; break;
  }
}

CRM_NOINLINE double crm_sin(double x) {
  double ax = fabs(x);
  if (!(ax < 0x1p1023)) return x - x; /* inf / nan -> nan */
  if (ax < 0x1p-27) return x;
  crm_dd s, c;
  crm_sincos_dd(x, &s, &c);
  return crm_round(s);
}

CRM_NOINLINE double crm_cos(double x) {
  double ax = fabs(x);
  if (!(ax < 0x1p1023)) return x - x;
  if (ax < 0x1p-27) return 1.0;
  crm_dd s, c;
  crm_sincos_dd(x, &s, &c);
  return crm_round(c);
}

CRM_NOINLINE double crm_tan(double x) {
  double ax = fabs(x);
  if (!(ax < 0x1p1023)) return x - x;
  if (ax < 0x1p-27) return x;
  crm_dd s, c;
  crm_sincos_dd(x, &s, &c);
  return crm_round(crm_div(s, c));
}

/* ---- atan ---------------------------------------------------------------- */

/* atan(z) for a double-double 0 <= z <= 1. */
CRM_FN crm_dd crm_atan_unit(crm_dd z) {
  double jd = rint(z.hi * 64.0);
  int j = (int)jd;
  double c = jd * 0.015625;
  crm_dd num = crm_add_d(z, -c);
  crm_dd den = crm_add_d(crm_mul_d(z, c), 1.0);
  crm_dd d = crm_div(num, den); /* |d| <= 1/128 */
  crm_dd d2 = crm_mul(d, d);
  double w = d2.hi;
  /* atan(d) = d*(1 + w*(-1/3 + w*(1/5 + w*(-1/7 + w*u)))) */
  double u = 1.0 / 9.0 + w * (-1.0 / 11.0 + w * (1.0 / 13.0 + w * (-1.0 / 15.0)));
  crm_dd p = crm_add_d(crm_mk(CRM_C7_HI, CRM_C7_LO), w * u);
  p = crm_mul(p, d2);
  p = crm_add(p, crm_mk(CRM_C5_HI, CRM_C5_LO));
  p = crm_mul(p, d2);
  p = crm_add(p, crm_mk(CRM_C3_HI, CRM_C3_LO));
  p = crm_mul(p, d2);
  p = crm_add_d(p, 1.0);
  crm_dd at = crm_mul(p, d);
  return crm_add(crm_mk(CRM_AT(2 * j), CRM_AT(2 * j + 1)), at);
}

CRM_NOINLINE double crm_atan(double x) {
  if (x != x) return x + x;
  double ax = fabs(x);
  if (ax < 0x1p-27) return x;
  crm_dd r;
  if (ax <= 1.0) {
    r = crm_atan_unit(crm_mk(ax, 0.0));
  } else if (ax < 0x1p100) {
    r = crm_sub(crm_mk(CRM_PIO2_HI, CRM_PIO2_LO), crm_atan_unit(crm_div_dd_d(1.0, ax)));
  } else {
    r = crm_mk(CRM_PIO2_HI, CRM_PIO2_LO);
  }
  double v = crm_round(r);
  return x < 0 ? -v : v;
}

CRM_NOINLINE double crm_atan2(double y, double x) {
  if (x != x || y != y) return x + y;
  const double pi_r = CRM_PI_HI;     /* RN(pi) */
  const double pio2_r = CRM_PIO2_HI; /* RN(pi/2) */
  if (y == 0.0) {
    if (x > 0.0 || (x == 0.0 && !signbit(x))) return y;
    return copysign(pi_r, y);
  }
  if (x == 0.0) return copysign(pio2_r, y);
  double ax = fabs(x), ay = fabs(y);
  if (isinf(ax) || isinf(ay)) {
    if (isinf(ax) && isinf(ay)) {
      double v = x > 0 ? 0.78539816339744828 : 2.3561944901923448; /* RN(pi/4), RN(3pi/4) */
      return copysign(v, y);
    }
    if (isinf(ax)) return x > 0 ? copysign(0.0, y) : copysign(pi_r, y);
    return copysign(pio2_r, y);
  }
  crm_dd t;
  if (ay <= ax) {
    t = crm_atan_unit(crm_div_dd_d(ay, ax));
  } else {
    t = crm_sub(crm_mk(CRM_PIO2_HI, CRM_PIO2_LO), crm_atan_unit(crm_div_dd_d(ax, ay)));
  }
  if (x < 0.0) t = crm_sub(crm_mk(CRM_PI_HI, CRM_PI_LO), t);
  double v = crm_round(t);
  return y < 0 ? -v : v;
}
