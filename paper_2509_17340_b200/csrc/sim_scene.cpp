// Host side of the synthetic input generator: scenario families with the
// reference's parameters and seeded rejection placement
// (proj/src/sim_world.cpp:174-246), converted to FP32 device primitives.
#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>

#include "sim.h"

namespace amppi_sim {

namespace {

constexpr double kPi = std::numbers::pi;
constexpr uint64_t kG = 0x9e3779b97f4a7c15ull;

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Stream {  // counter RNG, uniform draws (rng.hpp:19-38)
  uint64_t key;
  uint64_t ctr = 0;
  explicit Stream(uint64_t seed, uint64_t a) {
    uint64_t k = mix64(seed + kG);
    k = mix64(k ^ (a + kG));
    k = mix64(k ^ (0 + kG));
    k = mix64(k ^ (0 + kG));
    key = mix64(k ^ kG);
  }
  double uniform() { return static_cast<double>(mix64(key + (++ctr) * kG) >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

struct Rot {
  double m[3][3];  // local -> world
};

Rot rotation(const Prim& p) {
  Rot r{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  if (p.kind != 1 || p.tilt_angle == 0.0) return r;
  double ax = p.tilt_axis[0], ay = p.tilt_axis[1], az = p.tilt_axis[2];
  const double n = std::sqrt(ax * ax + ay * ay + az * az);
  ax /= n;
  ay /= n;
  az /= n;
  const double h = 0.5 * p.tilt_angle, s = std::sin(h);
  const double w = std::cos(h), x = s * ax, y = s * ay, z = s * az;
  r.m[0][0] = 1 - 2 * (y * y + z * z);
  r.m[0][1] = 2 * (x * y - w * z);
  r.m[0][2] = 2 * (x * z + w * y);
  r.m[1][0] = 2 * (x * y + w * z);
  r.m[1][1] = 1 - 2 * (x * x + z * z);
  r.m[1][2] = 2 * (y * z - w * x);
  r.m[2][0] = 2 * (x * z - w * y);
  r.m[2][1] = 2 * (y * z + w * x);
  r.m[2][2] = 1 - 2 * (x * x + y * y);
  return r;
}

double cylinder_surface_distance(const Prim& p, const double* q) {
  const Rot r = rotation(p);
  double d[3] = {q[0] - p.base[0], q[1] - p.base[1], q[2] - p.base[2]};
  double l[3];
  for (int i = 0; i < 3; ++i) l[i] = r.m[0][i] * d[0] + r.m[1][i] * d[1] + r.m[2][i] * d[2];
  const double radial = std::sqrt(l[0] * l[0] + l[1] * l[1]);
  const double dx = radial - p.radius;
  const double dz = std::abs(l[2] - 0.5 * p.height) - 0.5 * p.height;
  const double ox = std::max(dx, 0.0), oz = std::max(dz, 0.0);
  return std::abs(std::sqrt(ox * ox + oz * oz) + std::min(std::max(dx, dz), 0.0));
}

std::vector<Prim> cylinder_field(int count, double rmin, double rmax, double hmin, double hmax, double tilt_max,
                                 uint64_t seed) {
  std::vector<Prim> out;
  Stream rs(seed, 0x5CE9A210u);
  const double start[3] = {0.0, 0.0, 2.0}, goal[3] = {45.0, 0.0, 2.0};
  for (int i = 0; i < count; ++i) {
    Prim p{};
    bool placed = false;
    for (int attempt = 0; attempt < 10000 && !placed; ++attempt) {
      p = Prim{};
      p.kind = tilt_max > 0.0 ? 1 : 0;
      p.base[0] = rs.uniform(2.5, 42.5);
      p.base[1] = rs.uniform(-20.0, 20.0);
      p.base[2] = 0.0;
      p.radius = rs.uniform(rmin, rmax);
      p.height = hmin == hmax ? hmin : rs.uniform(hmin, hmax);
      p.tilt_axis[0] = 1.0;
      if (tilt_max > 0.0) {
        p.tilt_angle = rs.uniform(0.0, tilt_max);
        const double a = rs.uniform(0.0, 2.0 * kPi);
        p.tilt_axis[0] = std::cos(a);
        p.tilt_axis[1] = std::sin(a);
      }
      placed = cylinder_surface_distance(p, start) >= 1.0 && cylinder_surface_distance(p, goal) >= 1.0;
    }
    if (!placed) throw std::runtime_error("cannot place obstacle clear of start/goal");
    out.push_back(p);
  }
  return out;
}

}  // namespace

std::vector<Prim> generate_scenario(int kind, uint64_t seed) {
  switch (kind) {
    case kForest: return cylinder_field(100, 0.1, 0.5, 3.0, 8.0, 30.0 * kPi / 180.0, seed);
    case kVerticals: return cylinder_field(1000, 0.4, 1.1, 6.0, 6.0, 0.0, seed);
    case kInclines: return cylinder_field(800, 0.06, 0.3, 10.0, 10.0, 30.0 * kPi / 180.0, seed);
    case kTwoGap: {
      std::vector<Prim> out;
      for (auto [lo, hi] : {std::pair{-20.0, -5.0}, std::pair{-2.0, 2.0}, std::pair{5.0, 20.0}}) {
        Prim p{};
        p.kind = 2;
        p.base[0] = 20.0;
        p.base[1] = 0.5 * (lo + hi);
        p.base[2] = 4.0;
        p.half[0] = 0.2;
        p.half[1] = 0.5 * (hi - lo);
        p.half[2] = 4.0;
        out.push_back(p);
      }
      return out;
    }
    default: return {};
  }
}

DevPrim to_device(const Prim& p) {
  DevPrim d{};
  d.kind = p.kind;
  const Rot r = rotation(p);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) d.w2l[3 * i + j] = static_cast<float>(r.m[j][i]);
  for (int i = 0; i < 3; ++i) {
    d.base[i] = static_cast<float>(p.base[i]);
    d.half[i] = static_cast<float>(p.half[i]);
  }
  d.radius = static_cast<float>(p.radius);
  d.height = static_cast<float>(p.height);
  if (p.kind == 2) {
    for (int i = 0; i < 3; ++i) {
      d.lo[i] = static_cast<float>(p.base[i] - p.half[i]);
      d.hi[i] = static_cast<float>(p.base[i] + p.half[i]);
    }
    d.cx = static_cast<float>(p.base[0]);
    d.cy = static_cast<float>(p.base[1]);
    d.rad = static_cast<float>(std::sqrt(p.half[0] * p.half[0] + p.half[1] * p.half[1]));
  } else {
    const double tip[3] = {p.base[0] + r.m[0][2] * p.height, p.base[1] + r.m[1][2] * p.height,
                           p.base[2] + r.m[2][2] * p.height};
    for (int i = 0; i < 3; ++i) {
      d.lo[i] = static_cast<float>(std::min(p.base[i], tip[i]) - p.radius);
      d.hi[i] = static_cast<float>(std::max(p.base[i], tip[i]) + p.radius);
    }
    d.cx = static_cast<float>(0.5 * (p.base[0] + tip[0]));
    d.cy = static_cast<float>(0.5 * (p.base[1] + tip[1]));
    const double hx = p.base[0] - tip[0], hy = p.base[1] - tip[1];
    d.rad = static_cast<float>(0.5 * std::sqrt(hx * hx + hy * hy) + p.radius);
  }
  return d;
}

}  // namespace amppi_sim

namespace amppi_sim {

// Host twin of k_lidar + k_compact (same sim_ray.h arithmetic, built with
// -ffp-contract=off): frames in order, rays row-major, hits kept up to cap.
int64_t scan_host(const DevPrim* prims, int n_prims, const Frame* frames, int n_frames, float r_max, float el_min,
                  float el_max, float range_sigma, int64_t cap, float* xyz) {
  int j0 = -1, n_rows = 0;
  lidar_rows(el_min, el_max, &j0, &n_rows);
  int64_t n = 0;
  std::vector<int> near;
  std::vector<std::vector<int>> cols(kLidarAz);
  for (int f = 0; f < n_frames && n < cap; ++f) {
    const Frame& fr = frames[f];
    near.clear();
    for (int i = 0; i < n_prims; ++i)
      if (prim_near(prims[i], fr, r_max)) near.push_back(i);
    for (auto& c : cols) c.clear();
    for (int k = 0; k < static_cast<int>(near.size()); ++k) {
      int i0, i1;
      prim_columns(prims[near[k]], fr, &i0, &i1);
      for (int ii = i0; ii <= i1 && ii - i0 < kLidarAz; ++ii) cols[((ii % kLidarAz) + kLidarAz) % kLidarAz].push_back(k);
    }
    for (int j = j0; j < j0 + n_rows && n < cap; ++j)
      for (int i = 0; i < kLidarAz && n < cap; ++i) {
        const uint64_t key = ray_key(fr, i, j);
        float dir[3];
        ray_dir(fr, key, i, j, dir);
        float best = kInfF;
        const int c = ray_column(dir);
        if (c >= 0) {
          for (int k : cols[c]) best = fmin_d(best, ray_hit(prims[near[k]], fr.p, dir, r_max));
        } else {
          for (int idx : near) best = fmin_d(best, ray_hit(prims[idx], fr.p, dir, r_max));
        }
        if (best < kInfF) {
          ray_return(fr, key, dir, best, range_sigma, xyz + 3 * n);
          ++n;
        }
      }
  }
  return n;
}

}  // namespace amppi_sim
