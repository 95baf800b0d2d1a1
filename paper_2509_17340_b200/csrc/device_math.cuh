// Device math for the plan-cycle kernels, templated on the arithmetic type.
//
// Real = double is compiled in translation units built with -fmad=false and
// follows the reference's Eigen operation order exactly (SURVEY.md Appendix
// A.1; the same convention the CPU oracle fixes), so FP64 results differ from
// the oracle only through libm last-ulp differences (exp/log/sin/cos).
// Real = float is the throughput path (FMA contraction on, fast forms for the
// attitude term and quaternion normalisation); it is used for stage-I
// screening only, never for a returned value.
#pragma once

#include <cstdint>
#include <type_traits>

#include "layout.h"

namespace amppi_dev {

#ifdef AMPPI_STATS
// Query statistics (stats builds only): [0] queries, [1] queries with a
// non-empty neighbourhood, [2] cell records tested, [3] cells scanned,
// [4] points scanned, [5]/[6] queries ending with / without a point within
// reach, [7] points scanned by queries without one; [8 + j] live screening
// lanes at step j.
constexpr int kStatSlots = 8 + 64 + 8;  // query counters, live samples by step, d_max band
__device__ unsigned long long g_query_stats[kStatSlots];
#define AMPPI_STAT(i, v) atomicAdd(&g_query_stats[i], static_cast<unsigned long long>(v))
#else
#define AMPPI_STAT(i, v) ((void)0)
#endif

template <typename R>
struct V3 {
  R x, y, z;
};
template <typename R>
struct Q4 {
  R w, x, y, z;
};

template <typename R>
__device__ __forceinline__ V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <typename R>
__device__ __forceinline__ V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <typename R>
__device__ __forceinline__ V3<R> operator*(R s, V3<R> a) { return {s * a.x, s * a.y, s * a.z}; }

template <typename R>
__device__ __forceinline__ R sqnorm(V3<R> a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }

// FP32 screening square root: the hardware approximation (MUFU.SQRT,
// relative error < 2^-22; +inf -> +inf).  FP32 is only ever the screening
// arithmetic; every FP64 path uses sqrt().
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <typename R>
__device__ __forceinline__ R dsqrt(R x) {
  if constexpr (std::is_same_v<R, double>) return sqrt(x); else return sqrt_approx(x);
}

template <typename R>
__device__ __forceinline__ R norm3(V3<R> a) { return dsqrt(sqnorm(a)); }

template <typename R>
__device__ __forceinline__ V3<R> cross(V3<R> a, V3<R> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// std::clamp semantics (NaN passes through), ensemble of types.hpp:70-78.
template <typename R>
__device__ __forceinline__ R clampv(R v, R lo, R hi) { return v < lo ? lo : (hi < v ? hi : v); }

template <typename R>
__device__ __forceinline__ bool finite3(V3<R> a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

template <typename R>
__device__ __forceinline__ Q4<R> qmul(Q4<R> a, Q4<R> b) {  // Hamilton, left to right
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}

template <typename R>
__device__ __forceinline__ R qsqnorm(Q4<R> q) { return ((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w; }

// Eigen normalized(): divide by sqrt(squaredNorm) when positive.
template <typename R>
__device__ __forceinline__ Q4<R> qnormalized(Q4<R> q) {
  const R n2 = qsqnorm(q);
  if constexpr (std::is_same_v<R, double>) {
    if (!(n2 > 0.0)) return q;
    const double n = sqrt(n2);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
  } else {
    if (!(n2 > 0.0f)) return q;
    const float r = rsqrtf(n2);
    return {q.w * r, q.x * r, q.y * r, q.z * r};
  }
}

template <typename R>
__device__ __forceinline__ bool qfinite(Q4<R> q) {
  return isfinite(q.w) && isfinite(q.x) && isfinite(q.y) && isfinite(q.z);
}

// Eigen _transformVector: uv = 2 (q.vec x v); v + w uv + q.vec x uv.
template <typename R>
__device__ __forceinline__ V3<R> qrot(Q4<R> q, V3<R> v) {
  const V3<R> qv{q.x, q.y, q.z};
  V3<R> uv = cross(qv, v);
  uv = uv + uv;
  return (v + q.w * uv) + cross(qv, uv);
}

// Third column of R(q) for a unit q == q * e_z; FP32 shortcut only.
__device__ __forceinline__ V3<float> qrot_ez_fast(Q4<float> q) {
  return {2.f * (q.w * q.y + q.x * q.z), 2.f * (q.y * q.z - q.w * q.x), 1.f - 2.f * (q.x * q.x + q.y * q.y)};
}

struct M3 {
  double m[3][3];
};

// Eigen QuaternionBase::toRotationMatrix.
__device__ __forceinline__ M3 rotmat(Q4<double> q) {
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  M3 r;
  r.m[0][0] = 1.0 - (tyy + tzz);
  r.m[0][1] = txy - twz;
  r.m[0][2] = txz + twy;
  r.m[1][0] = txy + twz;
  r.m[1][1] = 1.0 - (txx + tzz);
  r.m[1][2] = tyz - twx;
  r.m[2][0] = txz - twy;
  r.m[2][1] = tyz + twx;
  r.m[2][2] = 1.0 - (txx + tyy);
  return r;
}

__device__ __forceinline__ V3<double> mat_vec(const M3& a, V3<double> v) {
  return {(a.m[0][0] * v.x + a.m[0][1] * v.y) + a.m[0][2] * v.z,
          (a.m[1][0] * v.x + a.m[1][1] * v.y) + a.m[1][2] * v.z,
          (a.m[2][0] * v.x + a.m[2][1] * v.y) + a.m[2][2] * v.z};
}

__device__ __forceinline__ V3<double> mat_t_vec(const M3& a, V3<double> v) {  // a^T v
  return {(a.m[0][0] * v.x + a.m[1][0] * v.y) + a.m[2][0] * v.z,
          (a.m[0][1] * v.x + a.m[1][1] * v.y) + a.m[2][1] * v.z,
          (a.m[0][2] * v.x + a.m[1][2] * v.y) + a.m[2][2] * v.z};
}

// ||R(q) G^T - I||_F with the oracle's column-major summation (costs.hpp:100-104).
// gt = R(q_goal)^T.
__device__ __forceinline__ double attitude_err_exact(Q4<double> q, const M3& gt) {
  const M3 r = rotmat(q);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double e = (r.m[i][0] * gt.m[0][j] + r.m[i][1] * gt.m[1][j]) + r.m[i][2] * gt.m[2][j];
      e = e - (i == j ? 1.0 : 0.0);
      s = s + e * e;
    }
  return sqrt(s);
}

// Closed form for unit quaternions: ||R(q)R(g)^T - I||_F = 2 sqrt(2) |vec(q (x) g*)|.
__device__ __forceinline__ float attitude_err_fast(Q4<float> q, Q4<float> g) {
  const float ex = g.w * q.x - q.w * g.x - (q.y * g.z - q.z * g.y);
  const float ey = g.w * q.y - q.w * g.y - (q.z * g.x - q.x * g.z);
  const float ez = g.w * q.z - q.w * g.z - (q.x * g.y - q.y * g.x);
  return 2.8284271247461903f * sqrt_approx(ex * ex + ey * ey + ez * ez);
}

// ---------------------------------------------------------------------------
// SplitMix64 counter RNG (rng.hpp:10-66)
// ---------------------------------------------------------------------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// RandomStream::derive(seed, a, b, c) followed by the constructor's mix.
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t k = mix64(seed + kGamma);
  k = mix64(k ^ (a + kGamma));
  k = mix64(k ^ (b + kGamma));
  k = mix64(k ^ (c + kGamma));
  return mix64(k ^ kGamma);
}

// Normal pair p of the stream (normals 2p -> cos, 2p+1 -> sin) drawn from
// counters 2p+1 (u1 = 1 - U) and 2p+2 (u2), Box-Muller as rng.hpp:43-55.
__device__ __forceinline__ void normal_pair(uint64_t key, uint32_t p, double& n0, double& n1) {
  const uint64_t a = mix64(key + (2ull * p + 1ull) * kGamma);
  const uint64_t b = mix64(key + (2ull * p + 2ull) * kGamma);
  const double u1 = 1.0 - static_cast<double>(a >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586 * u2;  // (2.0 * pi) * u2, 2.0*pi exact
  double s, c;
  sincos(ang, &s, &c);
  n0 = r * c;
  n1 = r * s;
}

// FP32 screening draw: same integers, float arithmetic.  log(1 - U): for
// U >= 1/16 the hardware log of 1 - U (from the integer complement, so U near
// 1 keeps its tail; relative error < 6e-6 there); for U < 1/16 the series
// -U (1 + U/2 + ... + U^5/6) on U itself (relative error < 1e-7) -- the float
// 1 - U would lose U below 2^-24, and the hardware log's absolute error
// (~4e-7) would dominate log(1 - U) ~ -U, turning a rare draw with U ~ 1e-6
// into a normal off by ~1e-3 (an FP32 rollout 1e-4 m from its FP64 twin;
// tools/screen_drift.py).  Both forms are evaluated and one selected, so the
// lanes of a warp stay converged.
#ifndef AMPPI_F32_BOX
#define AMPPI_F32_BOX 1  // nearest_sq_exact prunes boxes in FP32 with a rounding margin (0: FP64 box test)
#endif
#ifndef AMPPI_F32_PRESCREEN
#define AMPPI_F32_PRESCREEN 1  // nearest_sq_exact prescreens points in FP32 (needs AMPPI_F32_BOX)
#endif
#ifndef AMPPI_LOG_SERIES
#define AMPPI_LOG_SERIES 1
#endif
__device__ __forceinline__ void normal_pair_f(uint64_t key, uint32_t p, float& n0, float& n1) {
  const uint64_t a = mix64(key + (2ull * p + 1ull) * kGamma);
  const uint64_t b = mix64(key + (2ull * p + 2ull) * kGamma);
  const uint64_t ma = a >> 11;
  const float lhw = __logf(static_cast<float>((1ull << 53) - ma) * 0x1.0p-53f);
#if AMPPI_LOG_SERIES
  const float u = static_cast<float>(ma) * 0x1.0p-53f;
  const float ser =
      -u * (1.0f + u * (0.5f + u * (0.333333343f + u * (0.25f + u * (0.200000003f + u * 0.166666672f)))));
  const float lg = u < 0.0625f ? ser : lhw;
#else
  const float lg = lhw;
#endif
  const float r = sqrt_approx(fmaxf(-2.0f * lg, 0.0f));  // (the approximate log may round above 0 next to 1)
  // angle 2*pi*u2 in [0, 2pi): hardware sin/cos after reduction to [-pi, pi)
  // (abs error ~1e-6, far inside the screening window)
  const float u2 = static_cast<float>(b >> 11) * 0x1.0p-53f;
  const float ang = 6.28318530717958647f * (u2 < 0.5f ? u2 : u2 - 1.0f);
  float s, c;
  __sincosf(ang, &s, &c);
  n0 = r * c;
  n1 = r * s;
}

// ---------------------------------------------------------------------------
// dynamics (dynamics.hpp:13-78)
// ---------------------------------------------------------------------------
template <typename R>
struct Dyn {
  R mass, inv_mass, gx, gy, gz, dt, half_dt, dt6;
  R tmin, tmax, wxy, wz;
};

template <typename R>
__device__ __forceinline__ Dyn<R> make_dyn(const DevConfig& c) {
  Dyn<R> d;
  d.mass = static_cast<R>(c.mass);
  d.inv_mass = static_cast<R>(1.0 / c.mass);
  d.gx = static_cast<R>(c.gravity[0]);
  d.gy = static_cast<R>(c.gravity[1]);
  d.gz = static_cast<R>(c.gravity[2]);
  d.dt = static_cast<R>(c.dyn_dt);
  d.half_dt = static_cast<R>(0.5 * c.dyn_dt);
  d.dt6 = static_cast<R>(c.dyn_dt / 6.0);
  d.tmin = static_cast<R>(c.thrust_min);
  d.tmax = static_cast<R>(c.thrust_max);
  d.wxy = static_cast<R>(c.omega_xy_max);
  d.wz = static_cast<R>(c.omega_z_max);
  return d;
}

template <typename R>
struct St {
  V3<R> p;
  Q4<R> q;
  V3<R> v;
};

template <typename R>
struct Deriv {
  V3<R> dp;
  Q4<R> dq;
  V3<R> dv;
};

template <typename R>
__device__ __forceinline__ Deriv<R> derivative(const St<R>& x, R thrust, V3<R> om, const Dyn<R>& d) {
  Deriv<R> k;
  k.dp = x.v;
  const Q4<R> qd = qmul(x.q, Q4<R>{R(0), om.x, om.y, om.z});
  k.dq = {R(0.5) * qd.w, R(0.5) * qd.x, R(0.5) * qd.y, R(0.5) * qd.z};
  if constexpr (std::is_same_v<R, double>) {
    const V3<double> dir = qrot(qnormalized(x.q), V3<double>{0.0, 0.0, 1.0});
    const double a = thrust / d.mass;
    k.dv = V3<double>{a * dir.x, a * dir.y, a * dir.z} + V3<double>{d.gx, d.gy, d.gz};
  } else {
    // R(q/|q|) e_z = R_raw(q) e_z / |q|^2: one reciprocal instead of a
    // normalisation (screening arithmetic; the FP64 branch keeps Eigen's)
    const Q4<float>& q = x.q;
    const float n2 = ((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w;
    const float a = __fdividef(thrust * d.inv_mass, n2);
    k.dv = {a * (2.f * (q.w * q.y + q.x * q.z)) + d.gx, a * (2.f * (q.y * q.z - q.w * q.x)) + d.gy,
            a * ((q.w * q.w + q.z * q.z) - (q.x * q.x + q.y * q.y)) + d.gz};
  }
  return k;
}

template <typename R>
__device__ __forceinline__ St<R> advance(const St<R>& s, const Deriv<R>& k, R h) {
  St<R> o;
  o.p = s.p + h * k.dp;
  o.v = s.v + h * k.dv;
  o.q = {s.q.w + h * k.dq.w, s.q.x + h * k.dq.x, s.q.y + h * k.dq.y, s.q.z + h * k.dq.z};
  return o;
}

template <typename R>
__device__ __forceinline__ R rk_comb(R a, R b, R c, R e) { return ((a + R(2) * b) + R(2) * c) + e; }

// rk4_step_raw followed by q.normalize() (mppi.cpp:48-49).
template <typename R>
__device__ __forceinline__ St<R> rk4_normalized(const St<R>& x, R thrust, V3<R> om, const Dyn<R>& d) {
  const Deriv<R> k1 = derivative(x, thrust, om, d);
  const Deriv<R> k2 = derivative(advance(x, k1, d.half_dt), thrust, om, d);
  const Deriv<R> k3 = derivative(advance(x, k2, d.half_dt), thrust, om, d);
  const Deriv<R> k4 = derivative(advance(x, k3, d.dt), thrust, om, d);
  const R h6 = d.dt6;
  St<R> n;
  n.p = {x.p.x + h6 * rk_comb(k1.dp.x, k2.dp.x, k3.dp.x, k4.dp.x),
         x.p.y + h6 * rk_comb(k1.dp.y, k2.dp.y, k3.dp.y, k4.dp.y),
         x.p.z + h6 * rk_comb(k1.dp.z, k2.dp.z, k3.dp.z, k4.dp.z)};
  n.v = {x.v.x + h6 * rk_comb(k1.dv.x, k2.dv.x, k3.dv.x, k4.dv.x),
         x.v.y + h6 * rk_comb(k1.dv.y, k2.dv.y, k3.dv.y, k4.dv.y),
         x.v.z + h6 * rk_comb(k1.dv.z, k2.dv.z, k3.dv.z, k4.dv.z)};
  n.q = {x.q.w + h6 * rk_comb(k1.dq.w, k2.dq.w, k3.dq.w, k4.dq.w),
         x.q.x + h6 * rk_comb(k1.dq.x, k2.dq.x, k3.dq.x, k4.dq.x),
         x.q.y + h6 * rk_comb(k1.dq.y, k2.dq.y, k3.dq.y, k4.dq.y),
         x.q.z + h6 * rk_comb(k1.dq.z, k2.dq.z, k3.dq.z, k4.dq.z)};
  n.q = qnormalized(n.q);
  return n;
}

template <typename R>
__device__ __forceinline__ bool state_finite(const St<R>& s) {
  return finite3(s.p) && finite3(s.v) && qfinite(s.q);
}

// ---------------------------------------------------------------------------
// collision (costs.hpp:113-118, perception.cpp:191-235)
// ---------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ R collision_term(R d, R scale, R slope, R dmin, R dmax) {
  if (d < dmin) return scale;
  if (d < dmax) {
    if constexpr (std::is_same_v<R, double>) return scale * exp(-slope * (d - dmin));
    else return scale * __expf(-slope * (d - dmin));
  }
  return R(0);
}

// Bulk asynchronous copy (the non-tensor TMA path: cp.async.bulk with an
// mbarrier transaction count) of a CTA's per-instance tables into shared
// memory.  One thread arms the barrier and issues the copies; every thread
// waits on the barrier's phase before reading the tables.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bytes: a multiple of 16; src and dst 16-byte aligned
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(__cvta_generic_to_global(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// FP32 screening collision term with the d_max jump guarded.  The term
// falls from C exp(-a (d_max - d_min)) (~5e4 with the paper's weights) to 0
// at d_max, so a screening distance on the other side of d_max than the
// FP64 one would move the sample's FP32 cost far outside the softmin window.
// Within kAmbBand of d_max the screening adds 0 -- a lower bound of either
// branch -- and flags the sample (*amb): its screening cost is then a lower
// bound, k_support admits it by that bound and leaves it out of the FP32
// minimum.  The band covers the FP32 distance error
// (coordinates and RK4 in float) with a wide margin; queries reach
// d_max + band so a point just past d_max is seen.
__device__ __forceinline__ float amb_band(float dmax) { return 1e-4f * dmax + 1e-4f; }
__device__ __forceinline__ float screen_reach2(float dmax) {
  const float r = dmax + amb_band(dmax);
  return r * r * 1.0001f;
}
__device__ __forceinline__ float screen_collision(float d2, float cs, float ca, float dmin, float dmax, bool& amb) {
  const float d = sqrt_approx(d2);
  if (fabsf(d - dmax) < amb_band(dmax)) {
    AMPPI_STAT(72, 1);
    amb = true;
    return 0.f;
  }
  return collision_term(d, cs, ca, dmin, dmax);
}
// The same with the band precomputed (ScreenConsts).
__device__ __forceinline__ float screen_collision_b(float d2, float cs, float ca, float dmin, float dmax, float band,
                                                    bool& amb) {
  const float d = sqrt_approx(d2);
  if (fabsf(d - dmax) < band) {
    AMPPI_STAT(72, 1);
    amb = true;
    return 0.f;
  }
  return collision_term(d, cs, ca, dmin, dmax);
}
// Stored screening cost: a flagged (lower-bound) cost carries the sign bit.
__device__ __forceinline__ float screen_store(float cost, bool amb) { return amb ? -cost : cost; }

// The FP32 data and the FP32 screening live in the scene's local frame:
// x_f = float(x - g.org), the difference taken in FP64 before the one
// rounding, with org the snapshot pose.  Positions then stay within metres of
// 0 whatever the world coordinates, so the FP32 rollout drift does not grow
// with them (DESIGN.md §2 "The d_max jump"; tools/screen_drift.py).
__device__ __forceinline__ V3<float> to_local_f(const GridMeta& g, const double* v) {
  return {static_cast<float>(v[0] - g.org[0]), static_cast<float>(v[1] - g.org[1]),
          static_cast<float>(v[2] - g.org[2])};
}

// Collision-grid queries (replacing ClearanceIndex::nearest,
// perception.cpp:191-235).  The squared distance to the nearest filtered point
// is exact whenever the true nearest distance is below d_max: every such point
// lies in the 27 cells (size h >= d_max) around p, and the padded neighbour
// mask lists the non-empty ones.  Branch and bound over their float boxes
// (outward-rounded, so box distance <= point distance in the same arithmetic):
// own cell first, then the 6 face neighbours, then the rest; a cell is skipped
// when its box is farther than the best so far or than d_max (its points
// cannot change the cost); the scan stops once a point is closer than d_min
// (cost = C for any such d).  Returns +inf when no point is within reach.

// Neighbour bit b = i*9 + j*3 + k -> record index offset relative to
// cbase = ((cx-1)*D1 + (cy-1))*D2 + (cz-1).
__device__ __forceinline__ int nbr_offset(int b, int d12, int d2) {
  const int i = (b * 57) >> 9;  // b / 9 for b < 27
  const int r = b - 9 * i;
  const int j = (r * 11) >> 5;  // r / 3 for r < 9
  return i * d12 + j * d2 + (r - 3 * j);
}

// Padded-lattice mask of the query cell (cx, cy, cz); 0 when outside.
__device__ __forceinline__ uint32_t nbr_mask(const GridMeta& g, const uint32_t* __restrict__ nbr, int cx, int cy,
                                             int cz) {
  if (static_cast<unsigned>(cx + 1) > static_cast<unsigned>(g.dims[0] + 1) ||
      static_cast<unsigned>(cy + 1) > static_cast<unsigned>(g.dims[1] + 1) ||
      static_cast<unsigned>(cz + 1) > static_cast<unsigned>(g.dims[2] + 1))
    return 0u;
  return __ldg(nbr + ((cx + 1) * (g.dims[1] + 2) + (cy + 1)) * (g.dims[2] + 2) + (cz + 1));
}

__device__ __forceinline__ uint32_t nbr_phase(uint32_t m, int phase) {
  return m & (phase == 0 ? kNbrCenter : (phase == 1 ? kNbrFaces : ~(kNbrCenter | kNbrFaces)));
}

// Squared norm with a pinned evaluation shape, fma(z, z, fma(y, y, x * x)):
// the FP32 box bounds and the packed point distances below both use it, and
// it is monotone in each |component|, so a box distance never exceeds the
// distance of a point inside the box.
__device__ __forceinline__ float sq3f(float x, float y, float z) {
  return __fmaf_rn(z, z, __fmaf_rn(y, y, __fmul_rn(x, x)));
}

// Squared distance from p to a float box given as per-axis (lo, hi) pairs
// (the cell record / leaf box layout): per axis one packed FADD2 gives
// (lo - p, hi - p); gap = max(lo - p, p - hi, 0) in the same rounding as
// the point differences, squared in the sq3f shape.
__device__ __forceinline__ float box_gap_sq(uint32_t lx, uint32_t hx, uint32_t ly, uint32_t hy, uint32_t lz,
                                           uint32_t hz, V3<float> p) {
  const float2 dx = __fadd2_rn(make_float2(__uint_as_float(lx), __uint_as_float(hx)), make_float2(-p.x, -p.x));
  const float2 dy = __fadd2_rn(make_float2(__uint_as_float(ly), __uint_as_float(hy)), make_float2(-p.y, -p.y));
  const float2 dz = __fadd2_rn(make_float2(__uint_as_float(lz), __uint_as_float(hz)), make_float2(-p.z, -p.z));
  return sq3f(fmaxf(fmaxf(dx.x, -dx.y), 0.f), fmaxf(fmaxf(dy.x, -dy.y), 0.f), fmaxf(fmaxf(dz.x, -dz.y), 0.f));
}

// Squared distances from p to the 4 points of one FP32 point block
// ({x0..x3}, {y0..y3}, {z0..z3}), as two packed FP32x2 pairs: per pair one
// FADD2 per axis, FMUL2, two FFMA2 (sm_100 packed FP32) -- the sq3f shape.
__device__ __forceinline__ void block_d2(const float4* __restrict__ blk, V3<float> p, float2& d01, float2& d23) {
  const float4 X = __ldg(blk), Y = __ldg(blk + 1), Z = __ldg(blk + 2);
  const float2 npx = make_float2(-p.x, -p.x), npy = make_float2(-p.y, -p.y), npz = make_float2(-p.z, -p.z);
  float2 dx = __fadd2_rn(make_float2(X.x, X.y), npx), dy = __fadd2_rn(make_float2(Y.x, Y.y), npy),
         dz = __fadd2_rn(make_float2(Z.x, Z.y), npz);
  d01 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
  dx = __fadd2_rn(make_float2(X.z, X.w), npx);
  dy = __fadd2_rn(make_float2(Y.z, Y.w), npy);
  dz = __fadd2_rn(make_float2(Z.z, Z.w), npz);
  d23 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
}

__device__ __forceinline__ float block_min_d2(const float4* __restrict__ pts, uint32_t blk, V3<float> p) {
  float2 a, b;
  block_d2(pts + 3 * blk, p, a, b);
  return fminf(fminf(a.x, a.y), fminf(b.x, b.y));
}

template <bool kPrescreen = (AMPPI_F32_BOX && AMPPI_F32_PRESCREEN)>
__device__ __forceinline__ double nearest_sq_exact(const GridMeta& g, const uint4* __restrict__ rec,
                                                   const uint32_t* __restrict__ nbr, const uint4* __restrict__ leaves,
                                                   const double* __restrict__ pts, const float4* __restrict__ pts32,
                                                   V3<double> p, double lim2, double stop2, uint32_t* hint) {
  double best = __longlong_as_double(0x7ff0000000000000ll);
  if (g.dims[0] == 0) return best;
  uint32_t bi = *hint;
  if (bi != kNoHint) {
    best = sqnorm(p - V3<double>{pts[3 * bi], pts[3 * bi + 1], pts[3 * bi + 2]});
    if (best < stop2) return best;
  }
  const int cx = static_cast<int>(floor((p.x - g.origin[0]) * g.inv_h));
  const int cy = static_cast<int>(floor((p.y - g.origin[1]) * g.inv_h));
  const int cz = static_cast<int>(floor((p.z - g.origin[2]) * g.inv_h));
  const uint32_t m = nbr_mask(g, nbr, cx, cy, cz);
  if (!m) return best;
  const int d2 = g.dims[2], d12 = g.dims[1] * g.dims[2];
  const int cbase = ((cx - 1) * g.dims[1] + (cy - 1)) * d2 + (cz - 1);
#if AMPPI_F32_BOX
  // Box pruning in FP32, in the local frame of the float boxes (the
  // screening's box_gap_sq on pf = float(p - org)), with a margin that covers
  // its rounding: per axis the FP32 gap is off by at most
  // E = 2^-23 (|p - org|max + 2h + 1) (the rounding of pf plus the FADD's,
  // for boxes within the 27 cells around p), so the float box distance exceeds the true one
  // by at most 3.5 E sqrt(lim2) + 4 E^2 for any threshold <= lim2 -- plus the
  // relative rounding of the three squares and of the threshold.  A box is
  // skipped only when that slack still leaves it farther than the best point
  // so far (or than sqrt(lim2)): the same boxes as an exact test can keep,
  // never fewer, so the FP64 minimum is unchanged.
  const V3<float> pf{static_cast<float>(p.x - g.org[0]), static_cast<float>(p.y - g.org[1]),
                     static_cast<float>(p.z - g.org[2])};  // to_local_f
  const float e_ax = 0x1.0p-23f * (fmaxf(fmaxf(fabsf(pf.x), fabsf(pf.y)), fabsf(pf.z)) + 2.0f * g.h_f + 1.0f);
  const float slack = 3.5f * e_ax * __double2float_ru(sqrt(lim2)) + 4.0f * e_ax * e_ax;
  // (a float squared distance above cut cannot be within fmin(best, lim2))
  auto cut_of = [&](double b) { return __double2float_ru(fmin(b, lim2)) * (1.0f + 1e-6f) + slack; };
  float cut = cut_of(best);
  auto rec_far = [&](const uint4& ra, const uint4& rb) {
    return box_gap_sq(ra.z, ra.w, rb.x, rb.y, rb.z, rb.w, pf) > cut;
  };
  auto leaf_far = [&](const uint4& la, const uint4& lb) {
    return box_gap_sq(la.x, la.y, la.z, la.w, lb.x, lb.y, pf) > cut;
  };
#else
  // box lower bounds in the same arithmetic as the point distances (sqnorm of
  // a difference), so box distance <= point distance; the 1e-12 slack only
  // guards the lim2 comparison
  // (the float boxes are in the local frame of the FP32 data: pl = p - org,
  // off by at most an FP64 rounding, far inside the slack for any d > 1e-3)
  const V3<double> pl{p.x - g.org[0], p.y - g.org[1], p.z - g.org[2]};
  auto box_d2 = [&](uint32_t lx, uint32_t ly, uint32_t lz, uint32_t hx, uint32_t hy, uint32_t hz) {
    const V3<double> lo{__uint_as_float(lx), __uint_as_float(ly), __uint_as_float(lz)};
    const V3<double> hi{__uint_as_float(hx), __uint_as_float(hy), __uint_as_float(hz)};
    return sqnorm(V3<double>{fmax(fmax(lo.x - pl.x, pl.x - hi.x), 0.0), fmax(fmax(lo.y - pl.y, pl.y - hi.y), 0.0),
                             fmax(fmax(lo.z - pl.z, pl.z - hi.z), 0.0)});
  };
  auto rec_far = [&](const uint4& ra, const uint4& rb) {
    return box_d2(ra.z, rb.x, rb.z, ra.w, rb.y, rb.w) > fmin(best, lim2) * (1.0 + 1e-12);
  };
  auto leaf_far = [&](const uint4& la, const uint4& lb) {
    return box_d2(la.x, la.z, lb.x, la.y, la.w, lb.y) > fmin(best, lim2) * (1.0 + 1e-12);
  };
#endif
  for (int phase = 0; phase < 3; ++phase) {
    uint32_t mm = nbr_phase(m, phase);
    while (mm) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1;
      const int c = cbase + nbr_offset(b, d12, d2);
      const uint4 ra = rec[2 * c], rb = rec[2 * c + 1];
      if (rec_far(ra, rb)) continue;
      const uint32_t k0 = ra.x & 0xFFFFu, k1 = k0 + (ra.x >> 16);
      const uint4* lf = leaves + 2 * ra.y;
      for (uint32_t t = k0; t < k1; t += kLeafSize, lf += 2) {
        const uint4 la = lf[0], lb = lf[1];
        if (leaf_far(la, lb)) continue;
        const uint32_t te = min(t + kLeafSize, k1);
#if AMPPI_F32_BOX
        if constexpr (kPrescreen) {
        // FP32 prescreen: the leaf's 4-point float blocks (the screening's,
        // same local frame) in packed FP32x2; a point's FP32 squared distance
        // is off from the true one by no more than a box's, so FP64 is
        // evaluated only for points that can still beat best (or reach
        // lim2).  The blocks may hold a few real points of the neighbouring
        // leaves (harmless: real points) and +inf padding (never evaluated).
        for (uint32_t u = t / kPointBlock; u <= (te - 1) / kPointBlock; ++u) {
          float2 a01, a23;
          block_d2(pts32 + 3 * u, pf, a01, a23);
          const float dq[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (!(dq[i] <= cut)) continue;
            const uint32_t k = u * kPointBlock + i;
            const double dd = sqnorm(p - V3<double>{pts[3 * k], pts[3 * k + 1], pts[3 * k + 2]});
            if (dd < best) {
              best = dd;
              bi = k;
              cut = cut_of(best);
            }
          }
        }
        } else {
        for (uint32_t k = t; k < te; ++k) {
          const double dd = sqnorm(p - V3<double>{pts[3 * k], pts[3 * k + 1], pts[3 * k + 2]});
          if (dd < best) {
            best = dd;
            bi = k;
            cut = cut_of(best);
          }
        }
        }
#else
        for (uint32_t k = t; k < te; ++k) {
          const double dd = sqnorm(p - V3<double>{pts[3 * k], pts[3 * k + 1], pts[3 * k + 2]});
          if (dd < best) {
            best = dd;
            bi = k;
#if AMPPI_F32_BOX
            cut = cut_of(best);
#endif
          }
        }
#endif
        if (best < stop2) {
          *hint = bi;
          return best;
        }
      }
    }
  }
  *hint = bi;
  return best;
}

// FP32 screening query: as nearest_sq_exact, plus a second branch-and-bound
// level over each scanned cell's 16-point leaves (float leaf boxes).  Points
// are stored in blocks of 4 (kPointBlock, struct-of-arrays x4 / y4 / z4,
// +inf padding past the last point) and scanned a block at a time with
// packed FP32x2 arithmetic; a leaf's blocks may include a few points of the
// neighbouring leaves -- real points, so the minimum is unchanged.  Returns
// the exact squared distance when it lies in [stop2, lim2); any value below
// stop2 once a point closer than sqrt(stop2) is found (with stop2 = lim2 this
// is an existence test for a point within reach); >= lim2 (or +inf) when no
// point is closer than sqrt(lim2).  *hint (a block index, kNoHint for none)
// seeds the search with that block's nearest distance -- an upper bound on
// the minimum, so every box at least that far is pruned from the start --
// and receives the block of the nearest point found (the previous step's
// nearest block is a good seed for the next step of the same rollout).
__device__ __forceinline__ float nearest_sq_fast(const GridMeta& g, const uint4* __restrict__ rec,
                                                 const uint32_t* __restrict__ nbr, const uint4* __restrict__ leaves,
                                                 const float4* __restrict__ pts, V3<float> p, float lim2, float stop2,
                                                 uint32_t* hint) {
  float best = __int_as_float(0x7f800000);
  if (g.dims[0] == 0) return best;
  uint32_t bi = *hint;
  if (bi != kNoHint) {
    best = block_min_d2(pts, bi, p);
    if (best < stop2) return best;
  }
  const int cx = __float2int_rd((p.x - g.origin_f[0]) * g.inv_h_f);
  const int cy = __float2int_rd((p.y - g.origin_f[1]) * g.inv_h_f);
  const int cz = __float2int_rd((p.z - g.origin_f[2]) * g.inv_h_f);
  AMPPI_STAT(0, 1);
  const uint32_t m = nbr_mask(g, nbr, cx, cy, cz);
  if (!m) return best;
  AMPPI_STAT(1, 1);
#ifdef AMPPI_STATS
  uint32_t q_scanned = 0;
#define AMPPI_QEND(v) (AMPPI_STAT((v) < lim2 ? 5 : 6, 1), AMPPI_STAT(7, (v) < lim2 ? 0u : q_scanned), (v))
#else
#define AMPPI_QEND(v) (v)
#endif
  const int d2 = g.dims[2], d12 = g.dims[1] * g.dims[2];
  const int cbase = ((cx - 1) * g.dims[1] + (cy - 1)) * d2 + (cz - 1);
#pragma unroll 1
  for (int phase = 0; phase < 3; ++phase) {
    uint32_t mm = nbr_phase(m, phase);
    while (mm) {
      const int b = __ffs(mm) - 1;
      mm &= mm - 1;
      const int c = cbase + nbr_offset(b, d12, d2);
      const uint4 ra = __ldg(rec + 2 * c), rb = __ldg(rec + 2 * c + 1);
      AMPPI_STAT(2, 1);
      if (box_gap_sq(ra.z, ra.w, rb.x, rb.y, rb.z, rb.w, p) >= fminf(best, lim2)) continue;
      AMPPI_STAT(3, 1);
      const uint32_t k0 = ra.x & 0xFFFFu, k1 = k0 + (ra.x >> 16);
      const uint4* lf = leaves + 2 * ra.y;
      for (uint32_t t = k0; t < k1; t += kLeafSize, lf += 2) {
        const uint4 la = __ldg(lf), lb = __ldg(lf + 1);
        if (box_gap_sq(la.x, la.y, la.z, la.w, lb.x, lb.y, p) >= fminf(best, lim2)) continue;
        const uint32_t te = min(t + kLeafSize, k1);
        AMPPI_STAT(4, te - t);
#ifdef AMPPI_STATS
        q_scanned += te - t;
#endif
        for (uint32_t u = t / kPointBlock; u <= (te - 1) / kPointBlock; ++u) {
          const float dd = block_min_d2(pts, u, p);
          if (dd < best) {
            best = dd;
            bi = u;
          }
        }
        if (best < stop2) {
          *hint = bi;
          return AMPPI_QEND(best);
        }
      }
    }
  }
  *hint = bi;
  return AMPPI_QEND(best);
#undef AMPPI_QEND
}

}  // namespace amppi_dev
