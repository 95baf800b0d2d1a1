// GPU LiDAR simulator (input generator): one CTA per
// frame, one thread per ray slot.  Mirrors lidar_scan (sim_world.cpp:248-328):
// near-set filter by AABB distance, azimuth-column culling, one jittered ray
// per 3° cell inside the elevation mask, nearest hit within r_max, truncated
// Gaussian range noise; FP32 geometry.
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "sim.h"

namespace amppi_sim {

using amppi_dev::mix64;
using amppi_dev::stream_key;

namespace {

constexpr int kAz = 120;
constexpr int kEl = 60;
constexpr int kNearCap = 1024;
constexpr int kColCap = 32;
constexpr float kPiF = 3.14159265358979323846f;

__device__ __forceinline__ float uniform_at(uint64_t key, uint64_t ctr) {
  return static_cast<float>(static_cast<double>(mix64(key + ctr * amppi_dev::kGamma) >> 11) * 0x1.0p-53);
}

__device__ float ray_cylinder(const float* o, const float* d, float radius, float height, float t_max) {
  if (o[0] * o[0] + o[1] * o[1] <= radius * radius && o[2] >= 0.f && o[2] <= height) return INFINITY;
  float best = INFINITY;
  const float a = d[0] * d[0] + d[1] * d[1];
  const float c = o[0] * o[0] + o[1] * o[1] - radius * radius;
  if (a > 1e-14f) {
    const float b = 2.f * (o[0] * d[0] + o[1] * d[1]);
    const float disc = b * b - 4.f * a * c;
    if (disc >= 0.f) {
      const float root = sqrtf(disc);
      const float ts[2] = {(-b - root) / (2.f * a), (-b + root) / (2.f * a)};
      for (float t : ts)
        if (t > 1e-9f && t < best) {
          const float z = o[2] + t * d[2];
          if (z >= 0.f && z <= height) best = t;
        }
    }
  }
  if (fabsf(d[2]) > 1e-14f) {
    const float planes[2] = {0.f, height};
    for (float pl : planes) {
      const float t = (pl - o[2]) / d[2];
      if (t > 1e-9f && t < best) {
        const float x = o[0] + t * d[0], y = o[1] + t * d[1];
        if (x * x + y * y <= radius * radius) best = t;
      }
    }
  }
  return best <= t_max ? best : INFINITY;
}

__device__ float ray_box(const float* o, const float* d, const DevPrim& b, float t_max) {
  float tmin = -INFINITY, tmax = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const float lo = b.base[a] - b.half[a], hi = b.base[a] + b.half[a];
    if (fabsf(d[a]) < 1e-14f) {
      if (o[a] < lo || o[a] > hi) return INFINITY;
      continue;
    }
    float t0 = (lo - o[a]) / d[a], t1 = (hi - o[a]) / d[a];
    if (t0 > t1) {
      const float t = t0;
      t0 = t1;
      t1 = t;
    }
    tmin = fmaxf(tmin, t0);
    tmax = fminf(tmax, t1);
    if (tmin > tmax) return INFINITY;
  }
  if (tmin <= 1e-9f) return INFINITY;
  return tmin <= t_max ? tmin : INFINITY;
}

__device__ float ray_hit(const DevPrim& p, const float* o, const float* d, float t_max) {
  if (p.kind == 2) return ray_box(o, d, p, t_max);
  const float rel[3] = {o[0] - p.base[0], o[1] - p.base[1], o[2] - p.base[2]};
  float lo[3], ld[3];
  for (int i = 0; i < 3; ++i) {
    lo[i] = p.w2l[3 * i] * rel[0] + p.w2l[3 * i + 1] * rel[1] + p.w2l[3 * i + 2] * rel[2];
    ld[i] = p.w2l[3 * i] * d[0] + p.w2l[3 * i + 1] * d[1] + p.w2l[3 * i + 2] * d[2];
  }
  return ray_cylinder(lo, ld, p.radius, p.height, t_max);
}

__global__ void __launch_bounds__(256) k_lidar(const DevPrim* __restrict__ prims, const int* __restrict__ prim_off,
                                               const Frame* __restrict__ frames, float r_max, int j0, int n_rows,
                                               float range_sigma, float4* __restrict__ slots, int* __restrict__ hits) {
  __shared__ int near[kNearCap];
  __shared__ int n_near;
  __shared__ unsigned short cols[kAz][kColCap];
  __shared__ int col_n[kAz];
  __shared__ int s_hits;
  const Frame fr = frames[blockIdx.x];
  const int b = prim_off[fr.scene], e = prim_off[fr.scene + 1];
  const float az_step = 2.f * kPiF / kAz, el_step = kPiF / kEl;
  if (threadIdx.x == 0) {
    n_near = 0;
    s_hits = 0;
  }
  for (int c = threadIdx.x; c < kAz; c += blockDim.x) col_n[c] = 0;
  __syncthreads();
  for (int i = b + threadIdx.x; i < e; i += blockDim.x) {
    const DevPrim& p = prims[i];
    float d2 = 0.f;
    for (int a = 0; a < 3; ++a) {
      const float dd = fmaxf(fmaxf(p.lo[a] - fr.p[a], fr.p[a] - p.hi[a]), 0.f);
      d2 += dd * dd;
    }
    if (sqrtf(d2) <= r_max) {
      const int slot = atomicAdd(&n_near, 1);
      if (slot < kNearCap) near[slot] = i;
    }
  }
  __syncthreads();
  const int nn = min(n_near, kNearCap);
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    const DevPrim& p = prims[near[k]];
    const float rx = p.cx - fr.p[0], ry = p.cy - fr.p[1];
    const float dist = sqrtf(rx * rx + ry * ry);
    int i0 = 0, i1 = kAz - 1;
    if (dist > p.rad + 1e-9f) {
      const float half = asinf(fminf(1.f, p.rad / dist)) + az_step;
      const float bearing = atan2f(ry, rx);
      i0 = static_cast<int>(floorf((bearing - half + kPiF) / az_step));
      i1 = static_cast<int>(floorf((bearing + half + kPiF) / az_step));
    }
    for (int ii = i0; ii <= i1 && ii - i0 < kAz; ++ii) {
      const int c = ((ii % kAz) + kAz) % kAz;
      const int s = atomicAdd(&col_n[c], 1);
      if (s < kColCap) cols[c][s] = static_cast<unsigned short>(k);
    }
  }
  __syncthreads();
  const float qw = fr.q[0], qx = fr.q[1], qy = fr.q[2], qz = fr.q[3];
  int my_hits = 0;
  const int n_rays = n_rows * kAz;
  for (int r = threadIdx.x; r < n_rays; r += blockDim.x) {
    const int j = j0 + r / kAz, i = r % kAz;
    const uint64_t key = stream_key(fr.seed, 0x11DA2u, static_cast<uint64_t>(i * kEl + j), 0);
    const float az = -kPiF + (static_cast<float>(i) + uniform_at(key, 1)) * az_step;
    const float el = -0.5f * kPiF + (static_cast<float>(j) + uniform_at(key, 2)) * el_step;
    float se, ce, sa, ca;
    __sincosf(el, &se, &ce);
    __sincosf(az, &sa, &ca);
    const float v[3] = {ce * ca, ce * sa, se};
    // q * v (Eigen transform)
    float uv[3] = {qy * v[2] - qz * v[1], qz * v[0] - qx * v[2], qx * v[1] - qy * v[0]};
    uv[0] += uv[0];
    uv[1] += uv[1];
    uv[2] += uv[2];
    const float dir[3] = {v[0] + qw * uv[0] + (qy * uv[2] - qz * uv[1]),
                          v[1] + qw * uv[1] + (qz * uv[0] - qx * uv[2]),
                          v[2] + qw * uv[2] + (qx * uv[1] - qy * uv[0])};
    float best = INFINITY;
    const float dxy = sqrtf(dir[0] * dir[0] + dir[1] * dir[1]);
    if (dxy < 1e-12f) {
      for (int k = 0; k < nn; ++k) best = fminf(best, ray_hit(prims[near[k]], fr.p, dir, r_max));
    } else {
      int c = static_cast<int>(floorf((atan2f(dir[1], dir[0]) + kPiF) / az_step));
      if (c >= kAz) c -= kAz;
      c = c < 0 ? 0 : c;
      const int cn = col_n[c];
      if (cn <= kColCap && n_near <= kNearCap) {
        for (int k = 0; k < cn; ++k) best = fminf(best, ray_hit(prims[near[cols[c][k]]], fr.p, dir, r_max));
      } else {
        for (int k = 0; k < nn; ++k) best = fminf(best, ray_hit(prims[near[k]], fr.p, dir, r_max));
      }
    }
    float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (best < INFINITY) {
      // truncated Gaussian range noise (normal() draws counters 3, 4)
      const float u1 = 1.f - uniform_at(key, 3), u2 = uniform_at(key, 4);
      const float n0 = sqrtf(-2.f * logf(fmaxf(u1, 1e-30f))) * cosf(2.f * kPiF * u2);
      const float noise = fminf(fmaxf(range_sigma * n0, -4.f * range_sigma), 4.f * range_sigma);
      const float range = fmaxf(best + noise, 1e-3f);
      out = make_float4(fr.p[0] + range * dir[0], fr.p[1] + range * dir[1], fr.p[2] + range * dir[2], 1.f);
      ++my_hits;
    }
    slots[static_cast<int64_t>(blockIdx.x) * n_rays + r] = out;
  }
  atomicAdd(&s_hits, my_hits);
  __syncthreads();
  if (threadIdx.x == 0) hits[blockIdx.x] = s_hits;
}

// Ordered compaction of one frame's hits (ray order) into its output range.
__global__ void __launch_bounds__(256) k_compact(const float4* __restrict__ slots, int n_rays,
                                                 const int* __restrict__ out_off, const int* __restrict__ take,
                                                 float* __restrict__ xyz) {
  __shared__ int warp_tot[8];
  __shared__ int base;
  const int f = blockIdx.x;
  const int lim = take[f];
  if (lim <= 0) return;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r0 = 0; r0 < n_rays; r0 += blockDim.x) {
    const int r = r0 + threadIdx.x;
    const float4 s = r < n_rays ? slots[static_cast<int64_t>(f) * n_rays + r] : make_float4(0, 0, 0, 0);
    const int v = s.w > 0.f;
    const unsigned m = __ballot_sync(0xffffffffu, v);
    const int pre = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    const int pos = off + pre;
    if (v && pos < lim) {
      float* o = xyz + 3 * (static_cast<int64_t>(out_off[f]) + pos);
      o[0] = s.x;
      o[1] = s.y;
      o[2] = s.z;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 8; ++w) base += warp_tot[w];
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_lidar(const DevPrim* prims, const int* prim_offsets, const Frame* frames, int n_frames, float r_max,
                         float el_min, float el_max, float range_sigma, float4* slots, int* frame_hits,
                         cudaStream_t st) {
  // rows whose centre lies inside the elevation mask (sim_world.cpp:291-295)
  int j0 = -1, n_rows = 0;
  for (int j = 0; j < kEl; ++j) {
    const double c = -0.5 * 3.141592653589793 + (j + 0.5) * (3.141592653589793 / kEl);
    if (c < el_min || c > el_max) continue;
    if (j0 < 0) j0 = j;
    ++n_rows;
  }
  if (n_rows == 0) return cudaErrorInvalidValue;
  k_lidar<<<n_frames, 256, 0, st>>>(prims, prim_offsets, frames, r_max, j0, n_rows, range_sigma, slots, frame_hits);
  return cudaGetLastError();
}

int lidar_rays(float el_min, float el_max) {
  int n_rows = 0;
  for (int j = 0; j < kEl; ++j) {
    const double c = -0.5 * 3.141592653589793 + (j + 0.5) * (3.141592653589793 / kEl);
    if (!(c < el_min || c > el_max)) ++n_rows;
  }
  return n_rows * kAz;
}

cudaError_t launch_compact(const float4* slots, int n_rays, const int* frame_out_offset, const int* frame_take,
                           int n_frames, float* xyz, cudaStream_t st) {
  k_compact<<<n_frames, 256, 0, st>>>(slots, n_rays, frame_out_offset, frame_take, xyz);
  return cudaGetLastError();
}

}  // namespace amppi_sim
