// GPU closed loop kernels: per cycle the LiDAR scan
// into the PointCloudBuffer ring, then (after the regular snapshot + plan
// launches) the vehicle step, episode bookkeeping and the cycle record --
// execute_cycle (proj/src/ensemble.cpp:245-305) without leaving the device.
//
// FP64 with the reference's operation order (built with -fmad=false); the
// transcendentals (sin/cos/atan2/asin/log) are CUDA's.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "device_math.cuh"
#include "loop.h"

namespace amppi_dev {

namespace {

constexpr double kPiD = 0x1.921fb54442d18p+1;
constexpr double kAzStepD = 2.0 * kPiD / kAz;
constexpr double kElStepD = kPiD / kEl;
constexpr double kRayEps = 1e-9;
constexpr int kScanThreads = 1024;
constexpr int kMaxPrims = 1024;  // obstacle bitsets (the reference's families hold <= 1000)
constexpr int kPrimWords = kMaxPrims / 32;
constexpr int kRowsMax = kEl;

struct V {
  double x, y, z;
};
__device__ __forceinline__ V vsub(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V vadd(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V vscale(double s, V a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V vcross(V a, V b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ V mat3(const double* m, V v) {
  return {(m[0] * v.x + m[1] * v.y) + m[2] * v.z, (m[3] * v.x + m[4] * v.y) + m[5] * v.z,
          (m[6] * v.x + m[7] * v.y) + m[8] * v.z};
}
__device__ __forceinline__ V qrotv(const double* q, V v) {  // q = (w, x, y, z), Eigen _transformVector
  const V qv{q[1], q[2], q[3]};
  V uv = vcross(qv, v);
  uv = vadd(uv, uv);
  return vadd(vadd(v, vscale(q[0], uv)), vcross(qv, uv));
}

// RandomStream::derive(seed, a, b) and its counter draws (rng.hpp:10-66)
__device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t k = mix64(seed + kGamma);
  k = mix64(k ^ (a + kGamma));
  k = mix64(k ^ (b + kGamma));
  k = mix64(k ^ (0 + kGamma));
  return mix64(k ^ kGamma);
}
__device__ __forceinline__ double uniform_at(uint64_t key, uint64_t ctr) {
  return static_cast<double>(mix64(key + ctr * kGamma) >> 11) * 0x1.0p-53;
}

__device__ double ray_capped_cylinder(V o, V d, double radius, double height, double t_max) {  // sim_world.cpp:48-85
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (o.x * o.x + o.y * o.y <= radius * radius && o.z >= 0.0 && o.z <= height) return kInf;
  double best = kInf;
  const double a = d.x * d.x + d.y * d.y;
  const double c = o.x * o.x + o.y * o.y - radius * radius;
  if (a > 1e-14) {
    const double b = 2.0 * (o.x * d.x + o.y * d.y);
    const double disc = b * b - 4.0 * a * c;
    if (disc >= 0.0) {
      const double root = sqrt(disc);
      const double ts[2] = {(-b - root) / (2.0 * a), (-b + root) / (2.0 * a)};
      for (int k = 0; k < 2; ++k) {
        const double t = ts[k];
        if (t > kRayEps && t < best) {
          const double z = o.z + t * d.z;
          if (z >= 0.0 && z <= height) best = t;
        }
      }
    }
  }
  if (fabs(d.z) > 1e-14) {
    const double planes[2] = {0.0, height};
    for (int k = 0; k < 2; ++k) {
      const double t = (planes[k] - o.z) / d.z;
      if (t > kRayEps && t < best) {
        const double x = o.x + t * d.x;
        const double y = o.y + t * d.y;
        if (x * x + y * y <= radius * radius) best = t;
      }
    }
  }
  return best <= t_max ? best : kInf;
}

__device__ double ray_box(V o, V d, const double* center, const double* half, double t_max) {  // sim_world.cpp:87-105
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  double tmin = -kInf, tmax = kInf;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
  for (int axis = 0; axis < 3; ++axis) {
    const double lo = center[axis] - half[axis];
    const double hi = center[axis] + half[axis];
    if (fabs(dd[axis]) < 1e-14) {
      if (oo[axis] < lo || oo[axis] > hi) return kInf;
      continue;
    }
    double t0 = (lo - oo[axis]) / dd[axis];
    double t1 = (hi - oo[axis]) / dd[axis];
    if (t0 > t1) {
      const double tt = t0;
      t0 = t1;
      t1 = tt;
    }
    tmin = fmax(tmin, t0);
    tmax = fmin(tmax, t1);
    if (tmin > tmax) return kInf;
  }
  if (tmin <= kRayEps) return kInf;
  return tmin <= t_max ? tmin : kInf;
}

__device__ double ray_hit(const LoopPrim& p, V origin, V dir, double t_max) {  // sim_world.cpp:164-172
  if (p.kind == 2) return ray_box(origin, dir, p.base, p.half, t_max);
  return ray_capped_cylinder(mat3(p.w2l, vsub(origin, V{p.base[0], p.base[1], p.base[2]})), mat3(p.w2l, dir),
                             p.radius, p.height, t_max);
}

__device__ double surface_distance(const LoopPrim& p, V q) {  // sim_world.cpp:145-151
  if (p.kind == 2) {
    const V d{fabs(q.x - p.base[0]) - p.half[0], fabs(q.y - p.base[1]) - p.half[1], fabs(q.z - p.base[2]) - p.half[2]};
    const V o{fmax(d.x, 0.0), fmax(d.y, 0.0), fmax(d.z, 0.0)};
    const double outside = sqrt((o.x * o.x + o.y * o.y) + o.z * o.z);
    const double inside = fmin(fmax(fmax(d.x, d.y), d.z), 0.0);
    return fabs(outside + inside);
  }
  const V l = mat3(p.w2l, vsub(q, V{p.base[0], p.base[1], p.base[2]}));
  const double radial = sqrt(l.x * l.x + l.y * l.y);
  const double dx = radial - p.radius;
  const double dz = fabs(l.z - 0.5 * p.height) - 0.5 * p.height;
  const double ox = fmax(dx, 0.0), oz = fmax(dz, 0.0);
  return fabs(sqrt(ox * ox + oz * oz) + fmin(fmax(dx, dz), 0.0));
}

__device__ __forceinline__ int azimuth_cell_d(double az) {  // perception.cpp:17-21
  int i = static_cast<int>(floor((az + kPiD) / kAzStepD));
  if (i >= kAz) i -= kAz;
  return i < 0 ? 0 : (i > kAz - 1 ? kAz - 1 : i);
}

struct ScanSmem {
  uint32_t near[kPrimWords];
  uint32_t cols[kAz][kPrimWords];
  uint32_t warp_sums[kScanThreads / 32];
  uint32_t total;
};

__device__ uint32_t scan_exclusive(uint32_t v, ScanSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm.warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < static_cast<int>(blockDim.x >> 5) ? sm.warp_sums[lane] : 0u;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sm.warp_sums[lane] = w;
    if (lane == 31) sm.total = w;
  }
  __syncthreads();
  const uint32_t out = (warp > 0 ? sm.warp_sums[warp - 1] : 0u) + x - v;
  __syncthreads();
  return out;
}

// lidar_scan (sim_world.cpp:248-328) into the ring + PointCloudBuffer::push and
// all_points (perception.cpp:44-62): one CTA.
__global__ void __launch_bounds__(kScanThreads, 1) k_loop_scan(LoopDev L, LoopParams prm) {
  __shared__ ScanSmem sm;
  LoopState* st = L.st;
  if (st->status != 0) return;
  const int tid = threadIdx.x;
  const V pp{st->x[0], st->x[1], st->x[2]};
  const double q[4] = {st->x[3], st->x[4], st->x[5], st->x[6]};
  const uint64_t frame_seed = mix64(prm.seed) + st->cycle;
  for (int w = tid; w < kPrimWords; w += blockDim.x) sm.near[w] = 0u;
  for (int w = tid; w < kAz * kPrimWords; w += blockDim.x) (&sm.cols[0][0])[w] = 0u;
  __syncthreads();
  // near obstacles and their azimuth columns
  for (int i = tid; i < prm.n_prims; i += blockDim.x) {
    const LoopPrim& pr = L.prims[i];
    const V a{pr.lo[0] - pp.x, pr.lo[1] - pp.y, pr.lo[2] - pp.z}, b{pp.x - pr.hi[0], pp.y - pr.hi[1], pp.z - pr.hi[2]};
    const V d{fmax(fmax(a.x, b.x), 0.0), fmax(fmax(a.y, b.y), 0.0), fmax(fmax(a.z, b.z), 0.0)};
    if (!(sqrt((d.x * d.x + d.y * d.y) + d.z * d.z) <= prm.r_max)) continue;
    atomicOr(&sm.near[i >> 5], 1u << (i & 31));
    const double rx = pr.cx - pp.x, ry = pr.cy - pp.y;
    const double dist = sqrt(rx * rx + ry * ry);
    if (dist <= pr.rad + 1e-9) {
      for (int c = 0; c < kAz; ++c) atomicOr(&sm.cols[c][i >> 5], 1u << (i & 31));
      continue;
    }
    const double half = asin(fmin(1.0, pr.rad / dist)) + kAzStepD;
    const double bearing = atan2(ry, rx);
    const int i0 = static_cast<int>(floor((bearing - half + kPiD) / kAzStepD));
    const int i1 = static_cast<int>(floor((bearing + half + kPiD) / kAzStepD));
    for (int ii = i0; ii <= i1 && ii - i0 < kAz; ++ii)
      atomicOr(&sm.cols[((ii % kAz) + kAz) % kAz][i >> 5], 1u << (i & 31));
  }
  __syncthreads();
  // rays: slot = j * 120 + i (elevation outer, azimuth inner: the push order)
  const int slot_ring = (st->ring_head + 1) % prm.capacity;
  double* __restrict__ frame = L.frames + static_cast<int64_t>(slot_ring) * kLidarRays * 3;
  constexpr int kPer = (kLidarRays + kScanThreads - 1) / kScanThreads;  // 8 consecutive slots per thread
  double hx[kPer], hy[kPer], hz[kPer];
  uint32_t mine = 0;
  for (int u = 0; u < kPer; ++u) {
    const int slot = tid * kPer + u;
    hx[u] = __longlong_as_double(0x7ff8000000000000ll);
    if (slot >= kLidarRays) continue;
    const int j = slot / kAz, i = slot % kAz;
    const double el_center = -0.5 * kPiD + (j + 0.5) * kElStepD;
    if (el_center < prm.el_min || el_center > prm.el_max) continue;
    const uint64_t key = derive_key(frame_seed, 0x11DA2u, static_cast<uint64_t>(i * kEl + j));
    const double az = -kPiD + (i + uniform_at(key, 1)) * kAzStepD;
    const double el = -0.5 * kPiD + (j + uniform_at(key, 2)) * kElStepD;
    double sa, ca, se, ce;
    sincos(az, &sa, &ca);
    sincos(el, &se, &ce);
    const V dir = qrotv(q, V{ce * ca, ce * sa, se});
    double best = __longlong_as_double(0x7ff0000000000000ll);
    const double dir_xy = sqrt(dir.x * dir.x + dir.y * dir.y);
    const uint32_t* set = dir_xy < 1e-12 ? sm.near : sm.cols[azimuth_cell_d(atan2(dir.y, dir.x))];
    for (int w = 0; w < kPrimWords; ++w) {
      uint32_t bits = set[w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        best = fmin(best, ray_hit(L.prims[w * 32 + b], pp, dir, prm.r_max));
      }
    }
    if (!isfinite(best)) continue;
    // RandomStream::normal (counters 3, 4), clamped at 4 sigma
    const double u1 = 1.0 - uniform_at(key, 3);
    const double u2 = uniform_at(key, 4);
    const double r = sqrt(-2.0 * log(u1));
    const double noise0 = r * cos(2.0 * kPiD * u2);
    const double noise = fmin(fmax(0.0 + prm.range_sigma * noise0, -4.0 * prm.range_sigma), 4.0 * prm.range_sigma);
    const double range = fmax(best + noise, 1e-3);
    hx[u] = pp.x + range * dir.x;
    hy[u] = pp.y + range * dir.y;
    hz[u] = pp.z + range * dir.z;
    ++mine;
  }
  const uint32_t base = scan_exclusive(mine, sm);
  uint32_t o = base;
  for (int u = 0; u < kPer; ++u) {
    if (isnan(hx[u])) continue;
    frame[3 * o] = hx[u];
    frame[3 * o + 1] = hy[u];
    frame[3 * o + 2] = hz[u];
    ++o;
  }
  const uint32_t n_frame = sm.total;
  __syncthreads();
  __threadfence_block();
  // PointCloudBuffer push: the new frame becomes the newest, the oldest drops
  const int size = min(st->ring_size + 1, prm.capacity);
  if (tid == 0) L.frame_n[slot_ring] = static_cast<int32_t>(n_frame);
  __syncthreads();
  // all_points: frames oldest -> newest into the contiguous cloud
  int64_t out = 0;
  for (int f = size - 1; f >= 0; --f) {
    const int sl = ((slot_ring - f) % prm.capacity + prm.capacity) % prm.capacity;
    const int n = L.frame_n[sl];
    const double* src = L.frames + static_cast<int64_t>(sl) * kLidarRays * 3;
    for (int k = tid; k < 3 * n; k += blockDim.x) L.cloud[3 * out + k] = src[k];
    out += n;
  }
  __syncthreads();
  if (tid == 0) {
    st->ring_head = slot_ring;
    st->ring_size = size;
    L.offsets[0] = 0;
    L.offsets[1] = out;
    L.cycles[0] = st->cycle;
  }
}

// After the plan: apply the control (hover on "planning failed"), step the
// vehicle at 1/replan_hz, update the episode (ensemble.cpp:316-349), record.
__global__ void __launch_bounds__(256) k_loop_step(LoopDev L, LoopParams prm, Plan pl, DevConfig cfg) {
  __shared__ double s_min[8];
  __shared__ double s_u[4];
  __shared__ int s_planned, s_winner;
  LoopState* st = L.st;
  if (st->status != 0) return;
  const int tid = threadIdx.x, N = cfg.N;
  if (tid == 0) {
    s_planned = pl.status[0] == 0;
    s_winner = pl.winner[0];
    for (int c = 0; c < 4; ++c) s_u[c] = s_planned ? pl.control[c] : L.hover[c];
  }
  __syncthreads();
  const bool planned = s_planned;
  const int winner = s_winner;
  if (planned)
    for (int k = tid; k < 4 * N; k += blockDim.x) L.nominal[k] = pl.nominal[static_cast<int64_t>(winner) * N * 4 + k];
  __syncthreads();
  __shared__ double s_x[10];
  if (tid == 0) {
    const int64_t rc = static_cast<int64_t>(st->cycle);
    if (rc < L.max_records) {
      LoopRecord& r = L.records[rc];
      r.cycle = st->cycle;
      r.planned = planned ? 1 : 0;
      r.winner = planned ? winner : -1;
      for (int i = 0; i < 10; ++i) r.x[i] = st->x[i];
      for (int c = 0; c < 4; ++c) r.control[c] = s_u[c];
      r.stage2 = planned ? pl.stage2[winner] : __longlong_as_double(0x7ff0000000000000ll);
      r.n_points = static_cast<int32_t>(L.offsets[1]);
    }
    // es.x = rk4_step(es.x, u, dt = 1/replan_hz) (dynamics.hpp:70-78)
    Dyn<double> dy = make_dyn<double>(cfg);
    dy.dt = prm.step_dt;
    dy.half_dt = 0.5 * prm.step_dt;
    dy.dt6 = prm.step_dt / 6.0;
    St<double> x;
    x.p = {st->x[0], st->x[1], st->x[2]};
    x.q = {st->x[3], st->x[4], st->x[5], st->x[6]};
    x.v = {st->x[7], st->x[8], st->x[9]};
    const St<double> nx = rk4_normalized(x, s_u[0], V3<double>{s_u[1], s_u[2], s_u[3]}, dy);
    s_x[0] = nx.p.x; s_x[1] = nx.p.y; s_x[2] = nx.p.z;
    s_x[3] = nx.q.w; s_x[4] = nx.q.x; s_x[5] = nx.q.y; s_x[6] = nx.q.z;
    s_x[7] = nx.v.x; s_x[8] = nx.v.y; s_x[9] = nx.v.z;
  }
  __syncthreads();
  // true_clearance of the new position (sim_world.cpp:153-162): min over obstacles
  const V p{s_x[0], s_x[1], s_x[2]};
  double m = __longlong_as_double(0x7ff0000000000000ll);
  for (int i = tid; i < prm.n_prims; i += blockDim.x) m = fmin(m, surface_distance(L.prims[i], p));
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) s_min[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    double clearance = s_min[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) clearance = fmin(clearance, s_min[w]);
    for (int i = 0; i < 10; ++i) st->x[i] = s_x[i];
    st->t += prm.step_dt;
    for (int c = 0; c < 4; ++c) st->last[c] = s_u[c];
    const uint64_t rc = st->cycle;
    st->cycle += 1;
    if (planned) {
      st->prev_len = N;
      st->failures = 0;
    } else {
      st->failures += 1;
    }
    const double gx = s_x[0] - L.goal[0], gy = s_x[1] - L.goal[1], gz = s_x[2] - L.goal[2];
    int status = 0;
    if (clearance < prm.drone_radius) {
      status = 2;  // collision
    } else if (prm.goal_radius > 0.0 && sqrt((gx * gx + gy * gy) + gz * gz) <= prm.goal_radius) {
      status = 1;  // success
    } else if (st->failures >= prm.max_failures) {
      status = 4;  // planner_failure
    } else if (st->t >= prm.timeout) {
      status = 3;  // timeout
    }
    st->status = status;
    if (static_cast<int64_t>(rc) < L.max_records) {
      LoopRecord& r = L.records[rc];
      r.status = status;
      r.t = st->t;
      for (int i = 0; i < 10; ++i) r.x_after[i] = s_x[i];
      r.clearance = clearance;
      for (int i = 0; i < 5; ++i) r.breakdown[i] = planned ? pl.breakdown[static_cast<int64_t>(winner) * 5 + i] : 0.0;
    }
  }
}

// compute_metrics (metrics.cpp:12-49) on the device log, in the reference's
// summation order (one thread; a log is a few thousand records).
__global__ void k_loop_metrics(LoopDev L, int64_t n, LoopMetrics* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const LoopRecord* rec = L.records;
  auto vel = [&](int64_t i) { return V{rec[i].x_after[7], rec[i].x_after[8], rec[i].x_after[9]}; };
  auto pos = [&](int64_t i) { return V{rec[i].x_after[0], rec[i].x_after[1], rec[i].x_after[2]}; };
  auto norm = [](V a) { return sqrt((a.x * a.x + a.y * a.y) + a.z * a.z); };
  const double dt = rec[1].t - rec[0].t;
  LoopMetrics m{0.0, 0.0, 0.0, 0.0, 0.0, __longlong_as_double(0x7ff0000000000000ll)};
  double speed_sum = 0.0, clearance_sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double speed = norm(vel(i));
    speed_sum += speed;
    m.max_vel = fmax(m.max_vel, speed);
    if (i + 1 < n) m.path_length += norm(vsub(pos(i + 1), pos(i)));
    const double c = rec[i].clearance;
    clearance_sum += c;
    m.min_clearance = fmin(m.min_clearance, c);
  }
  m.avg_vel = speed_sum / static_cast<double>(n);
  m.avg_clearance = clearance_sum / static_cast<double>(n);
  auto second_diff = [&](int64_t a, int64_t b, int64_t c) {  // (v_c - 2 v_b + v_a) / dt^2
    const V va = vel(a), vb = vel(b), vc = vel(c);
    const double d2 = dt * dt;
    return V{((vc.x - 2.0 * vb.x) + va.x) / d2, ((vc.y - 2.0 * vb.y) + va.y) / d2, ((vc.z - 2.0 * vb.z) + va.z) / d2};
  };
  for (int64_t i = 0; i < n; ++i) {
    const V j = i == 0 ? second_diff(0, 1, 2) : (i == n - 1 ? second_diff(n - 3, n - 2, n - 1) : second_diff(i - 1, i, i + 1));
    m.smoothness += ((j.x * j.x + j.y * j.y) + j.z * j.z) * dt;
  }
  *out = m;
}

}  // namespace

cudaError_t launch_loop_scan(const LoopDev& L, const LoopParams& prm, cudaStream_t st) {
  if (prm.n_prims > kMaxPrims) return cudaErrorInvalidValue;
  k_loop_scan<<<1, kScanThreads, 0, st>>>(L, prm);
  return cudaGetLastError();
}

cudaError_t launch_loop_step(const LoopDev& L, const LoopParams& prm, const Plan& pl, const DevConfig& cfg,
                             cudaStream_t st) {
  k_loop_step<<<1, 256, 0, st>>>(L, prm, pl, cfg);
  return cudaGetLastError();
}

cudaError_t launch_loop_metrics(const LoopDev& L, int64_t n, LoopMetrics* out, cudaStream_t st) {
  k_loop_metrics<<<1, 32, 0, st>>>(L, n, out);
  return cudaGetLastError();
}

}  // namespace amppi_dev
