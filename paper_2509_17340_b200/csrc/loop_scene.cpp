// Host side of the GPU closed loop: the reference's scenario families
// (proj/src/sim_world.cpp:174-246) in FP64 with its operation order, so the
// obstacle set (seeded rejection placement against the start and goal) is the
// reference's exactly, plus the per-obstacle values the device LiDAR and
// collision check need (sim_world.cpp:17-46, :107-122, :271-283).
#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>

#include "loop.h"

namespace amppi_dev {

namespace {

constexpr double kPi = std::numbers::pi;
constexpr uint64_t kG = 0x9e3779b97f4a7c15ull;

uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Stream {  // RandomStream::derive(seed, a) + uniform (rng.hpp:19-38)
  uint64_t key, ctr = 0;
  Stream(uint64_t seed, uint64_t a) {
    uint64_t k = mix(seed + kG);
    k = mix(k ^ (a + kG));
    k = mix(k ^ (0 + kG));
    k = mix(k ^ (0 + kG));
    key = mix(k ^ kG);
  }
  double uniform() { return static_cast<double>(mix(key + (++ctr) * kG) >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

struct V {
  double x, y, z;
};
V sub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V add(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V scale(double s, V a) { return {s * a.x, s * a.y, s * a.z}; }
V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double sqn(V a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }

struct Q {
  double w, x, y, z;
};

// ObstaclePrimitive::rotation (sim_world.hpp:24-28): AngleAxis(tilt, axis.normalized())
Q rotation(const LoopPrim& p, V axis, double tilt) {
  if (p.kind != 1 || tilt == 0.0) return {1.0, 0.0, 0.0, 0.0};
  const double n2 = sqn(axis);
  if (n2 > 0.0) {
    const double n = std::sqrt(n2);
    axis = {axis.x / n, axis.y / n, axis.z / n};
  }
  const double ha = 0.5 * tilt, s = std::sin(ha);
  return {std::cos(ha), s * axis.x, s * axis.y, s * axis.z};
}

V qrot(Q q, V v) {  // Eigen _transformVector
  const V qv{q.x, q.y, q.z};
  V uv = cross(qv, v);
  uv = add(uv, uv);
  return add(add(v, scale(q.w, uv)), cross(qv, uv));
}

void world_to_local(Q q, double* m) {  // toRotationMatrix().transpose(), row-major
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  const double r[3][3] = {{1.0 - (tyy + tzz), txy - twz, txz + twy},
                          {txy + twz, 1.0 - (txx + tzz), tyz - twx},
                          {txz - twy, tyz + twx, 1.0 - (txx + tyy)}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = r[j][i];
}

V mat_vec(const double* m, V v) {
  return {(m[0] * v.x + m[1] * v.y) + m[2] * v.z, (m[3] * v.x + m[4] * v.y) + m[5] * v.z,
          (m[6] * v.x + m[7] * v.y) + m[8] * v.z};
}

double cylinder_sdf(V q, double radius, double height) {  // sim_world.cpp:31-39
  const double radial = std::sqrt(q.x * q.x + q.y * q.y);
  const double dx = radial - radius;
  const double dz = std::abs(q.z - 0.5 * height) - 0.5 * height;
  const double ox = std::max(dx, 0.0), oz = std::max(dz, 0.0);
  return std::sqrt(ox * ox + oz * oz) + std::min(std::max(dx, dz), 0.0);
}

double surface_distance(const LoopPrim& p, V q) {  // sim_world.cpp:145-151 (cylinders)
  return std::abs(cylinder_sdf(mat_vec(p.w2l, sub(q, V{p.base[0], p.base[1], p.base[2]})), p.radius, p.height));
}

void finish(LoopPrim& p, Q rot) {  // AABB + culling disc (sim_world.cpp:107-117, :271-283)
  if (p.kind == 2) {
    for (int a = 0; a < 9; ++a) p.w2l[a] = (a % 4 == 0) ? 1.0 : 0.0;
    for (int a = 0; a < 3; ++a) {
      p.lo[a] = p.base[a] - p.half[a];
      p.hi[a] = p.base[a] + p.half[a];
    }
    p.cx = p.base[0];
    p.cy = p.base[1];
    p.rad = std::sqrt(p.half[0] * p.half[0] + p.half[1] * p.half[1]);
    return;
  }
  world_to_local(rot, p.w2l);
  const V base{p.base[0], p.base[1], p.base[2]};
  const V tip = add(base, qrot(rot, V{0.0, 0.0, p.height}));
  const double b[3] = {base.x, base.y, base.z}, t[3] = {tip.x, tip.y, tip.z};
  for (int a = 0; a < 3; ++a) {
    p.lo[a] = std::min(b[a], t[a]) - p.radius;
    p.hi[a] = std::max(b[a], t[a]) + p.radius;
  }
  p.cx = 0.5 * (base.x + tip.x);
  p.cy = 0.5 * (base.y + tip.y);
  const double hx = base.x - tip.x, hy = base.y - tip.y;
  p.rad = 0.5 * std::sqrt(hx * hx + hy * hy) + p.radius;
}

std::vector<LoopPrim> cylinder_field(int count, double rmin, double rmax, double hmin, double hmax, double tilt_max,
                                     uint64_t seed) {  // generate_cylinder_field (sim_world.cpp:174-207)
  std::vector<LoopPrim> out;
  Stream rs(seed, 0x5CE9A210u);
  const V start{0.0, 0.0, 2.0}, goal{45.0, 0.0, 2.0};
  for (int i = 0; i < count; ++i) {
    LoopPrim p{};
    bool placed = false;
    for (int attempt = 0; attempt < 10000 && !placed; ++attempt) {
      p = LoopPrim{};
      p.kind = tilt_max > 0.0 ? 1 : 0;
      p.base[0] = rs.uniform(2.5, 42.5);
      p.base[1] = rs.uniform(-20.0, 20.0);
      p.base[2] = 0.0;
      p.radius = rs.uniform(rmin, rmax);
      p.height = hmin == hmax ? hmin : rs.uniform(hmin, hmax);
      V axis{1.0, 0.0, 0.0};
      double tilt = 0.0;
      if (tilt_max > 0.0) {
        tilt = rs.uniform(0.0, tilt_max);
        const double az = rs.uniform(0.0, 2.0 * kPi);
        axis = {std::cos(az), std::sin(az), 0.0};
      }
      finish(p, rotation(p, axis, tilt));
      placed = surface_distance(p, start) >= 1.0 && surface_distance(p, goal) >= 1.0;
    }
    if (!placed) throw std::runtime_error("cannot place obstacle clear of start/goal");
    out.push_back(p);
  }
  return out;
}

}  // namespace

std::vector<LoopPrim> loop_scenario(int kind, uint64_t seed) {  // generate_scenario (sim_world.cpp:209-246)
  switch (kind) {
    case 0: return {};
    case 1: return cylinder_field(100, 0.1, 0.5, 3.0, 8.0, 30.0 * kPi / 180.0, seed);
    case 2: return cylinder_field(1000, 0.4, 1.1, 6.0, 6.0, 0.0, seed);
    case 3: return cylinder_field(800, 0.06, 0.3, 10.0, 10.0, 30.0 * kPi / 180.0, seed);
    case 4: {
      std::vector<LoopPrim> out;
      for (auto [lo, hi] : {std::pair{-20.0, -5.0}, std::pair{-2.0, 2.0}, std::pair{5.0, 20.0}}) {
        LoopPrim p{};
        p.kind = 2;
        p.base[0] = 20.0;
        p.base[1] = 0.5 * (lo + hi);
        p.base[2] = 4.0;
        p.half[0] = 0.2;
        p.half[1] = 0.5 * (hi - lo);
        p.half[2] = 4.0;
        finish(p, Q{1.0, 0.0, 0.0, 0.0});
        out.push_back(p);
      }
      return out;
    }
    default: throw std::invalid_argument("unknown scenario kind");
  }
}

}  // namespace amppi_dev
