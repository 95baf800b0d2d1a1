// LiDAR ray casting of the synthetic input generator,
// shared verbatim by the GPU kernel (k_lidar.cu, built with -fmad=false) and
// the host generator (api_sim.cpp, -ffp-contract=off): every operation is an
// IEEE single-precision +, -, *, /, sqrt, floor or rint, and the
// transcendentals are the polynomial forms below, so the two produce the same
// bits.  Mirrors lidar_scan (sim_world.cpp:248-328): near-set by AABB
// distance, azimuth-column culling, one jittered ray per 3° cell inside the
// elevation mask, nearest hit within r_max, truncated Gaussian range noise.
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define AMPPI_HD __host__ __device__ __forceinline__
#else
#define AMPPI_HD inline
#endif

namespace amppi_sim {

constexpr int kLidarAz = 120;
constexpr int kLidarEl = 60;
constexpr float kPiF = 3.14159265358979323846f;
constexpr float kInfF = __builtin_huge_valf();

// Device form of one primitive (FP32), with the culling bounds precomputed.
struct DevPrim {
  float w2l[9];  // world -> local rotation (row-major)
  float base[3];
  float radius, height;
  float half[3];
  float lo[3], hi[3];  // world AABB
  float cx, cy, rad;   // azimuth-culling disc (sim_world.cpp:271-283)
  int kind;            // 0 vertical cylinder, 1 tilted cylinder, 2 box
};

struct Frame {
  int scene;
  float p[3];
  float q[4];  // w, x, y, z
  unsigned long long seed;
};

// IEEE square root / floor / round-to-nearest-even on either side
AMPPI_HD float sim_sqrt(float x) {
#ifdef __CUDA_ARCH__
  return __fsqrt_rn(x);
#else
  return __builtin_sqrtf(x);
#endif
}
AMPPI_HD float sim_floor(float x) {
#ifdef __CUDA_ARCH__
  return floorf(x);
#else
  return __builtin_floorf(x);
#endif
}
AMPPI_HD float sim_rint(float x) {
#ifdef __CUDA_ARCH__
  return rintf(x);
#else
  return __builtin_rintf(x);
#endif
}

AMPPI_HD uint32_t f2u(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
AMPPI_HD float u2f(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
AMPPI_HD float fmin_d(float a, float b) { return b < a ? b : a; }
AMPPI_HD float fmax_d(float a, float b) { return a < b ? b : a; }
AMPPI_HD float fabs_d(float a) { return u2f(f2u(a) & 0x7FFFFFFFu); }

// SplitMix64 (rng.hpp:10-36)
AMPPI_HD uint64_t sim_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
constexpr uint64_t kSimGamma = 0x9e3779b97f4a7c15ull;
AMPPI_HD uint64_t sim_stream_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t k = sim_mix64(seed + kSimGamma);
  k = sim_mix64(k ^ (a + kSimGamma));
  k = sim_mix64(k ^ (b + kSimGamma));
  k = sim_mix64(k ^ (c + kSimGamma));
  return sim_mix64(k ^ kSimGamma);
}
// RandomStream::uniform() of draw `ctr` (1-based), rounded to float
AMPPI_HD float uniform_at(uint64_t key, uint64_t ctr) {
  return static_cast<float>(static_cast<double>(sim_mix64(key + ctr * kSimGamma) >> 11) * 0x1.0p-53);
}

// sin and cos: reduction by the nearest multiple of pi/2 (three-part
// Cody-Waite), Taylor polynomials on [-pi/4, pi/4] (error < 3e-8).
AMPPI_HD void det_sincos(float x, float* s, float* c) {
  const float kf = sim_rint(x * 0.636619772f);
  float r = x - kf * 1.5703125f;
  r = r - kf * 4.83751297e-4f;
  r = r - kf * 7.54978995e-8f;
  const float r2 = r * r;
  const float sn = r + r * r2 * (-0.166666667f + r2 * (8.33333333e-3f + r2 * (-1.98412698e-4f + r2 * 2.75573192e-6f)));
  const float cs = 1.0f + r2 * (-0.5f + r2 * (4.16666667e-2f + r2 * (-1.38888889e-3f + r2 * 2.48015873e-5f)));
  const int q = static_cast<int>(kf) & 3;
  *s = q == 0 ? sn : (q == 1 ? cs : (q == 2 ? -sn : -cs));
  *c = q == 0 ? cs : (q == 1 ? -sn : (q == 2 ? -cs : sn));
}

// atan2: odd degree-11 polynomial for atan on [0, 1] (error < 2e-6 rad) and
// the octant fold.
AMPPI_HD float det_atan2(float y, float x) {
  const float ax = fabs_d(x), ay = fabs_d(y);
  const float mx = fmax_d(ax, ay);
  if (mx == 0.0f) return 0.0f;
  const float a = fmin_d(ax, ay) / mx;
  const float s = a * a;
  float r = -0.01172120f;
  r = r * s + 0.05265332f;
  r = r * s - 0.11643287f;
  r = r * s + 0.19354346f;
  r = r * s - 0.33262347f;
  r = r * s + 0.99997726f;
  r = r * a;
  if (ay > ax) r = 1.57079632679f - r;
  if (x < 0.f) r = 3.14159265359f - r;
  return y < 0.f ? -r : r;
}

AMPPI_HD float det_asin(float v) {  // v in [0, 1]
  float c = 1.0f - v * v;
  c = c > 0.0f ? c : 0.0f;
  return det_atan2(v, sim_sqrt(c));
}

// natural log of a positive normal float: exponent split, atanh series on
// [sqrt(1/2), sqrt(2)) (error < 1e-7 relative)
AMPPI_HD float det_log(float u) {
  const uint32_t b = f2u(u);
  int e = static_cast<int>((b >> 23) & 0xFFu) - 127;
  float m = u2f((b & 0x7FFFFFu) | 0x3F800000u);
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e += 1;
  }
  const float t = (m - 1.0f) / (m + 1.0f);
  const float t2 = t * t;
  const float lm = 2.0f * t * (1.0f + t2 * (0.333333333f + t2 * (0.2f + t2 * (0.142857143f + t2 * 0.111111111f))));
  const float fe = static_cast<float>(e);
  return fe * 0.693145752f + (fe * 1.42860677e-6f + lm);
}


AMPPI_HD float ray_cylinder(const float* o, const float* d, float radius, float height, float t_max) {
  if (o[0] * o[0] + o[1] * o[1] <= radius * radius && o[2] >= 0.f && o[2] <= height) return kInfF;
  float best = kInfF;
  const float a = d[0] * d[0] + d[1] * d[1];
  const float c = o[0] * o[0] + o[1] * o[1] - radius * radius;
  if (a > 1e-14f) {
    const float b = 2.f * (o[0] * d[0] + o[1] * d[1]);
    const float disc = b * b - 4.f * a * c;
    if (disc >= 0.f) {
      const float root = sim_sqrt(disc);
      const float ts[2] = {(-b - root) / (2.f * a), (-b + root) / (2.f * a)};
      for (float t : ts)
        if (t > 1e-9f && t < best) {
          const float z = o[2] + t * d[2];
          if (z >= 0.f && z <= height) best = t;
        }
    }
  }
  if (fabs_d(d[2]) > 1e-14f) {
    const float planes[2] = {0.f, height};
    for (float pl : planes) {
      const float t = (pl - o[2]) / d[2];
      if (t > 1e-9f && t < best) {
        const float x = o[0] + t * d[0], y = o[1] + t * d[1];
        if (x * x + y * y <= radius * radius) best = t;
      }
    }
  }
  return best <= t_max ? best : kInfF;
}

AMPPI_HD float ray_box(const float* o, const float* d, const DevPrim& b, float t_max) {
  float tmin = -kInfF, tmax = kInfF;
  for (int a = 0; a < 3; ++a) {
    const float lo = b.base[a] - b.half[a], hi = b.base[a] + b.half[a];
    if (fabs_d(d[a]) < 1e-14f) {
      if (o[a] < lo || o[a] > hi) return kInfF;
      continue;
    }
    float t0 = (lo - o[a]) / d[a], t1 = (hi - o[a]) / d[a];
    if (t0 > t1) {
      const float t = t0;
      t0 = t1;
      t1 = t;
    }
    tmin = fmax_d(tmin, t0);
    tmax = fmin_d(tmax, t1);
    if (tmin > tmax) return kInfF;
  }
  if (tmin <= 1e-9f) return kInfF;
  return tmin <= t_max ? tmin : kInfF;
}

AMPPI_HD float ray_hit(const DevPrim& p, const float* o, const float* d, float t_max) {
  if (p.kind == 2) return ray_box(o, d, p, t_max);
  const float rel[3] = {o[0] - p.base[0], o[1] - p.base[1], o[2] - p.base[2]};
  float lo[3], ld[3];
  for (int i = 0; i < 3; ++i) {
    lo[i] = p.w2l[3 * i] * rel[0] + p.w2l[3 * i + 1] * rel[1] + p.w2l[3 * i + 2] * rel[2];
    ld[i] = p.w2l[3 * i] * d[0] + p.w2l[3 * i + 1] * d[1] + p.w2l[3 * i + 2] * d[2];
  }
  return ray_cylinder(lo, ld, p.radius, p.height, t_max);
}

// AABB distance test of the near set (sim_world.cpp:255-259)
AMPPI_HD bool prim_near(const DevPrim& p, const Frame& fr, float r_max) {
  float d2 = 0.f;
  for (int a = 0; a < 3; ++a) {
    const float dd = fmax_d(fmax_d(p.lo[a] - fr.p[a], fr.p[a] - p.hi[a]), 0.f);
    d2 = d2 + dd * dd;
  }
  return sim_sqrt(d2) <= r_max;
}

// Azimuth columns [i0, i1] (mod kLidarAz) a near primitive can be hit in
// (sim_world.cpp:271-286); all columns when the vehicle is inside its disc.
AMPPI_HD void prim_columns(const DevPrim& p, const Frame& fr, int* i0, int* i1) {
  const float az_step = 2.f * kPiF / kLidarAz;
  const float rx = p.cx - fr.p[0], ry = p.cy - fr.p[1];
  const float dist = sim_sqrt(rx * rx + ry * ry);
  *i0 = 0;
  *i1 = kLidarAz - 1;
  if (dist > p.rad + 1e-9f) {
    const float half = det_asin(fmin_d(1.f, p.rad / dist)) + az_step;
    const float bearing = det_atan2(ry, rx);
    *i0 = static_cast<int>(sim_floor((bearing - half + kPiF) / az_step));
    *i1 = static_cast<int>(sim_floor((bearing + half + kPiF) / az_step));
  }
}

// Direction of ray (i, j) of a frame (RandomStream::derive(frame_seed,
// 0x11DA2, i*60+j): draws 1, 2 jitter the cell, lidar_scan's pose.q * dir).
AMPPI_HD uint64_t ray_key(const Frame& fr, int i, int j) {
  return sim_stream_key(fr.seed, 0x11DA2u, static_cast<uint64_t>(i * kLidarEl + j), 0);
}
AMPPI_HD void ray_dir(const Frame& fr, uint64_t key, int i, int j, float* dir) {
  const float az_step = 2.f * kPiF / kLidarAz, el_step = kPiF / kLidarEl;
  const float az = -kPiF + (static_cast<float>(i) + uniform_at(key, 1)) * az_step;
  const float el = -0.5f * kPiF + (static_cast<float>(j) + uniform_at(key, 2)) * el_step;
  float se, ce, sa, ca;
  det_sincos(el, &se, &ce);
  det_sincos(az, &sa, &ca);
  const float v[3] = {ce * ca, ce * sa, se};
  const float qw = fr.q[0], qx = fr.q[1], qy = fr.q[2], qz = fr.q[3];
  float uv[3] = {qy * v[2] - qz * v[1], qz * v[0] - qx * v[2], qx * v[1] - qy * v[0]};
  uv[0] = uv[0] + uv[0];
  uv[1] = uv[1] + uv[1];
  uv[2] = uv[2] + uv[2];
  dir[0] = (v[0] + qw * uv[0]) + (qy * uv[2] - qz * uv[1]);
  dir[1] = (v[1] + qw * uv[1]) + (qz * uv[0] - qx * uv[2]);
  dir[2] = (v[2] + qw * uv[2]) + (qx * uv[1] - qy * uv[0]);
}

// Column of a ray direction (azimuth_cell of atan2(dir.y, dir.x)), or -1 for
// a vertical ray (every near primitive is a candidate).
AMPPI_HD int ray_column(const float* dir) {
  const float dxy = sim_sqrt(dir[0] * dir[0] + dir[1] * dir[1]);
  if (dxy < 1e-12f) return -1;
  int c = static_cast<int>(sim_floor((det_atan2(dir[1], dir[0]) + kPiF) / (2.f * kPiF / kLidarAz)));
  if (c >= kLidarAz) c -= kLidarAz;
  return c < 0 ? 0 : c;
}

// The return of a ray whose nearest hit is at `best` (finite): truncated
// Gaussian range noise from draws 3, 4 (RandomStream::normal, Box-Muller cos
// branch), clamped to +-4 sigma.
AMPPI_HD void ray_return(const Frame& fr, uint64_t key, const float* dir, float best, float sigma, float* out) {
  const float u1 = 1.f - uniform_at(key, 3), u2 = uniform_at(key, 4);
  float s, c;
  det_sincos(2.f * kPiF * u2, &s, &c);
  const float n0 = sim_sqrt(-2.f * det_log(fmax_d(u1, 1e-30f))) * c;
  const float noise = fmin_d(fmax_d(sigma * n0, -4.f * sigma), 4.f * sigma);
  const float range = fmax_d(best + noise, 1e-3f);
  out[0] = fr.p[0] + range * dir[0];
  out[1] = fr.p[1] + range * dir[1];
  out[2] = fr.p[2] + range * dir[2];
}

// Rows of the elevation mask (ray rows whose centre lies inside it,
// sim_world.cpp:291-295): first row and row count.
inline void lidar_rows(float el_min, float el_max, int* j0, int* n_rows) {
  *j0 = -1;
  *n_rows = 0;
  for (int j = 0; j < kLidarEl; ++j) {
    const double c = -0.5 * 3.141592653589793 + (j + 0.5) * (3.141592653589793 / kLidarEl);
    if (c < el_min || c > el_max) continue;
    if (*j0 < 0) *j0 = j;
    ++*n_rows;
  }
}

}  // namespace amppi_sim
