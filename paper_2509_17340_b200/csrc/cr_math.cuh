// Correctly-rounded double sin / cos / atan2 for integer-keying decisions.
//
// The reference keys points and anchors to 3°/18° cells with glibc's double
// atan2/sin/cos followed by floor() (perception.cpp:17-26, guidance.cpp:16-72).
// CUDA's double transcendentals carry up to 2 ulp of error, which flips a cell
// index whenever the quotient sits on a boundary (the
// paper-default anchors land EXACTLY on 18° boundaries).  These routines
// return the correctly rounded result (double-double evaluation, ~2^-100
// relative), which equals glibc's whenever glibc itself rounds correctly.
// tests/test_cr_math.py measures that agreement on the host against glibc.
//
// Requirements: compiled WITHOUT FMA contraction (nvcc -fmad=false; host
// -ffp-contract=off): the error-free transforms below rely on exact IEEE
// rounding of every + and *.  Inputs are assumed finite with magnitudes in
// [2^-500, 2^500]; zero / non-finite operands fall back to the plain libm
// call, whose special-case results are exact on both sides.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define CRM_HD __host__ __device__ __forceinline__
#else
#define CRM_HD inline
#endif

namespace crm {

struct dd {
  double hi, lo;
};

CRM_HD double fma_exact(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

CRM_HD dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double err = (a - (s - bb)) + (b - bb);
  return {s, err};
}

CRM_HD dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}

CRM_HD dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma_exact(a, b, -p)};
}

CRM_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}

CRM_HD dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
CRM_HD dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

CRM_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}

CRM_HD dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}

CRM_HD dd dd_div_d(dd a, double b) {
  const double q1 = a.hi / b;
  dd p = two_prod(q1, b);
  dd r = two_sum(a.hi, -p.hi);
  r.lo -= p.lo;
  r.lo += a.lo;
  const double q2 = (r.hi + r.lo) / b;
  dd q = quick_two_sum(q1, q2);
  // one more correction step for ~2^-104 accuracy
  p = dd_mul_d(q, b);
  r = dd_sub(a, p);
  const double q3 = r.hi / b;
  return dd_add(q, dd{q3, 0.0});
}

// pi/2 as four pieces P1 + P2 + P3 + P4 (fdlibm's pio2_1, pio2_2, pio2_3,
// pio2_3t; the first three carry 33 significant bits so k*Pi is exact for
// |k| < 2^20).  The sum equals pi/2 to ~2^-160.
constexpr double kPio2_1 = 0x1.921fb544p+0;
constexpr double kPio2_2 = 0x1.0b4611a6p-34;
constexpr double kPio2_3 = 0x1.3198a2ep-69;
constexpr double kPio2_4 = 0x1.b839a252049c1p-104;

// x - k*pi/2 as a double-double, k = nearest integer to x*2/pi.
CRM_HD dd reduce_pio2(double x, int& quadrant) {
  const double kd = nearbyint(x * 0.63661977236758134308);
  quadrant = static_cast<int>(kd) & 3;
  // r = x - k P1 - k P2 - k P3 - k P4, every product tracked exactly
  dd r = two_sum(x, -kd * kPio2_1);
  r = dd_add(r, dd{-kd * kPio2_2, 0.0});
  r = dd_add(r, dd{-kd * kPio2_3, 0.0});
  r = dd_add(r, dd_neg(two_prod(kd, kPio2_4)));
  return r;
}

// sin(r), cos(r) for |r| <= pi/4 + eps, Taylor series in double-double.
CRM_HD void dd_sincos_small(dd r, dd& s, dd& c) {
  const dd r2 = dd_mul(r, r);
  // sin: r - r^3/3! + ...  (terms up to r^33)
  dd term = r;
  dd sum_s = r;
  for (int n = 3; n <= 33; n += 2) {
    term = dd_div_d(dd_mul(term, r2), -static_cast<double>(n * (n - 1)));
    sum_s = dd_add(sum_s, term);
  }
  // cos: 1 - r^2/2! + ... (terms up to r^32)
  term = dd{1.0, 0.0};
  dd sum_c = term;
  for (int n = 2; n <= 32; n += 2) {
    term = dd_div_d(dd_mul(term, r2), -static_cast<double>(n * (n - 1)));
    sum_c = dd_add(sum_c, term);
  }
  s = sum_s;
  c = sum_c;
}

CRM_HD void dd_sincos(double x, dd& s, dd& c) {
  int q = 0;
  const dd r = reduce_pio2(x, q);
  dd sr, cr;
  dd_sincos_small(r, sr, cr);
  switch (q) {
    case 0: s = sr; c = cr; break;
    case 1: s = cr; c = dd_neg(sr); break;
    case 2: s = dd_neg(sr); c = dd_neg(cr); break;
    default: s = dd_neg(cr); c = sr; break;
  }
}

CRM_HD double round_dd(dd a) { return a.hi + a.lo; }

CRM_HD bool plain_args(double x) {
  const double ax = fabs(x);
  return !(ax < 1e150) || ax < 1e-150;  // non-finite, huge, zero or tiny
}

CRM_HD double sin_cr(double x) {
  if (plain_args(x) || fabs(x) > 1e5) return sin(x);
  dd s, c;
  dd_sincos(x, s, c);
  return round_dd(s);
}

CRM_HD double cos_cr(double x) {
  if (plain_args(x) || fabs(x) > 1e5) return cos(x);
  dd s, c;
  dd_sincos(x, s, c);
  return round_dd(c);
}

// Correction of a near-correct atan2 estimate t0: rotate (x, y) by -t0 in
// double-double and add atan(y'/x') ~= y'/x' (|y'/x'| ~ 1e-16).
CRM_HD double atan2_refine(double y, double x, double t0) {
  dd s, c;
  dd_sincos(t0, s, c);
  const dd yc = dd_mul_d(c, y);
  const dd xs = dd_mul_d(s, x);
  const dd xc = dd_mul_d(c, x);
  const dd ys = dd_mul_d(s, y);
  const dd yp = dd_sub(yc, xs);  // y' = y cos t0 - x sin t0
  const dd xp = dd_add(xc, ys);  // x' = x cos t0 + y sin t0
  const double delta = (yp.hi + yp.lo) / (xp.hi + xp.lo);
  const dd t = two_sum(t0, delta);
  return t.hi + t.lo;
}

CRM_HD double atan2_cr(double y, double x) {
  const double t0 = atan2(y, x);
  if (plain_args(x) || plain_args(y)) return t0;
  return atan2_refine(y, x, t0);
}

}  // namespace crm
