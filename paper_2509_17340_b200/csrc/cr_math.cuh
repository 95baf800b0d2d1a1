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

// 1/n! as double-doubles (hi + lo, generated with mpmath at 400 bits).
#ifdef __CUDACC__
__device__ __constant__
#endif
static const dd kInvFact[36] = {
    {0x1.0000000000000p+0, 0x0.0p+0},  // 1/0!
    {0x1.0000000000000p+0, 0x0.0p+0},  // 1/1!
    {0x1.0000000000000p-1, 0x0.0p+0},  // 1/2!
    {0x1.5555555555555p-3, 0x1.5555555555555p-57},  // 1/3!
    {0x1.5555555555555p-5, 0x1.5555555555555p-59},  // 1/4!
    {0x1.1111111111111p-7, 0x1.1111111111111p-63},  // 1/5!
    {0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65},  // 1/6!
    {0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73},  // 1/7!
    {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76},  // 1/8!
    {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},  // 1/9!
    {0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76},  // 1/10!
    {0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80},  // 1/11!
    {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83},  // 1/12!
    {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87},  // 1/13!
    {0x1.93974a8c07c9dp-37, 0x1.05d6f8a2efd1fp-92},  // 1/14!
    {0x1.ae7f3e733b81fp-41, 0x1.1d8656b0ee8cbp-97},  // 1/15!
    {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101},  // 1/16!
    {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103},  // 1/17!
    {0x1.6827863b97d97p-53, 0x1.eec01221a8b0bp-107},  // 1/18!
    {0x1.2f49b46814157p-57, 0x1.2650f61dbdcb4p-112},  // 1/19!
    {0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120},  // 1/20!
    {0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120},  // 1/21!
    {0x1.0ce396db7f853p-70, -0x1.aebcdbd20331cp-124},  // 1/22!
    {0x1.761b41316381ap-75, -0x1.3423c7d91404fp-130},  // 1/23!
    {0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135},  // 1/24!
    {0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139},  // 1/25!
    {0x1.88e85fc6a4e5ap-89, -0x1.71c37ebd16540p-143},  // 1/26!
    {0x1.d1ab1c2dccea3p-94, 0x1.054d0c78aea14p-149},  // 1/27!
    {0x1.0a18a2635085dp-98, 0x1.b9e2e28e1aa54p-153},  // 1/28!
    {0x1.259f98b4358adp-103, 0x1.eaf8c39dd9bc5p-157},  // 1/29!
    {0x1.3932c5047d60ep-108, 0x1.832b7b530a627p-162},  // 1/30!
    {0x1.434d2e783f5bcp-113, 0x1.0b87b91be9affp-167},  // 1/31!
    {0x1.434d2e783f5bcp-118, 0x1.0b87b91be9affp-172},  // 1/32!
    {0x1.3981254dd0d52p-123, -0x1.2b1f4c8015a2fp-177},  // 1/33!
    {0x1.2710231c0fd7ap-128, 0x1.3f8a2b4af9d6bp-184},  // 1/34!
    {0x1.0dc59c716d91fp-133, 0x1.419e3fad3f031p-188},  // 1/35!
};

CRM_HD dd inv_fact(int n) {
#ifdef __CUDA_ARCH__
  return kInvFact[n];
#else
  return kInvFact[n];
#endif
}

// sin(r), cos(r) for |r| <= pi/4 + eps: Horner in r^2 over double-double
// Taylor coefficients (terms through r^33 / r^32, truncation < 2^-110).
//   sin r = r * sum_i (-1)^i r^2i / (2i+1)!,   cos r = sum_i (-1)^i r^2i / (2i)!
CRM_HD void dd_sincos_small(dd r, dd& s, dd& c) {
  const dd r2 = dd_mul(r, r);
  dd ps = inv_fact(33);  // i = 16: positive
  for (int i = 15; i >= 0; --i) {
    const dd a = (i & 1) ? dd_neg(inv_fact(2 * i + 1)) : inv_fact(2 * i + 1);
    ps = dd_add(a, dd_mul(r2, ps));
  }
  s = dd_mul(ps, r);
  dd pc = inv_fact(32);  // i = 16: positive
  for (int i = 15; i >= 0; --i) {
    const dd b = (i & 1) ? dd_neg(inv_fact(2 * i)) : inv_fact(2 * i);
    pc = dd_add(b, dd_mul(r2, pc));
  }
  c = pc;
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

CRM_HD void sincos_cr(double x, double& sn, double& cs) {
  if (plain_args(x) || fabs(x) > 1e5) {
    sn = sin(x);
    cs = cos(x);
    return;
  }
  dd s, c;
  dd_sincos(x, s, c);
  sn = round_dd(s);
  cs = round_dd(c);
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
