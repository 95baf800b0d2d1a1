// GPU LiDAR simulator (input generator): one CTA per
// frame, one thread per ray slot.  The per-ray arithmetic is sim_ray.h,
// shared with the host generator (scan_host in sim_scene.cpp); this TU is
// built with -fmad=false so both produce the same bits.
#include <cuda_runtime.h>

#include "sim.h"

namespace amppi_sim {

namespace {

constexpr int kNearCap = 1024;
constexpr int kColCap = 32;

__global__ void __launch_bounds__(256) k_lidar(const DevPrim* __restrict__ prims, const int* __restrict__ prim_off,
                                               const Frame* __restrict__ frames, float r_max, int j0, int n_rows,
                                               float range_sigma, float4* __restrict__ slots, int* __restrict__ hits) {
  __shared__ int near[kNearCap];
  __shared__ int n_near;
  __shared__ unsigned short cols[kLidarAz][kColCap];
  __shared__ int col_n[kLidarAz];
  __shared__ int s_hits;
  const Frame fr = frames[blockIdx.x];
  const int b = prim_off[fr.scene], e = prim_off[fr.scene + 1];
  if (threadIdx.x == 0) {
    n_near = 0;
    s_hits = 0;
  }
  for (int c = threadIdx.x; c < kLidarAz; c += blockDim.x) col_n[c] = 0;
  __syncthreads();
  // near set (any order: every ray takes the minimum over its candidates)
  for (int i = b + threadIdx.x; i < e; i += blockDim.x)
    if (prim_near(prims[i], fr, r_max)) {
      const int slot = atomicAdd(&n_near, 1);
      if (slot < kNearCap) near[slot] = i;
    }
  __syncthreads();
  const int nn = min(n_near, kNearCap);
  for (int k = threadIdx.x; k < nn; k += blockDim.x) {
    int i0, i1;
    prim_columns(prims[near[k]], fr, &i0, &i1);
    for (int ii = i0; ii <= i1 && ii - i0 < kLidarAz; ++ii) {
      const int c = ((ii % kLidarAz) + kLidarAz) % kLidarAz;
      const int s = atomicAdd(&col_n[c], 1);
      if (s < kColCap) cols[c][s] = static_cast<unsigned short>(k);
    }
  }
  __syncthreads();
  int my_hits = 0;
  const int n_rays = n_rows * kLidarAz;
  for (int r = threadIdx.x; r < n_rays; r += blockDim.x) {
    const int j = j0 + r / kLidarAz, i = r % kLidarAz;
    const uint64_t key = ray_key(fr, i, j);
    float dir[3];
    ray_dir(fr, key, i, j, dir);
    float best = kInfF;
    const int c = ray_column(dir);
    if (c >= 0 && col_n[c] <= kColCap && n_near <= kNearCap) {
      for (int k = 0; k < col_n[c]; ++k) best = fmin_d(best, ray_hit(prims[near[cols[c][k]]], fr.p, dir, r_max));
    } else {
      for (int k = 0; k < nn; ++k) best = fmin_d(best, ray_hit(prims[near[k]], fr.p, dir, r_max));
    }
    float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (best < kInfF) {
      float o[3];
      ray_return(fr, key, dir, best, range_sigma, o);
      out = make_float4(o[0], o[1], o[2], 1.f);
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
  int j0 = -1, n_rows = 0;
  lidar_rows(el_min, el_max, &j0, &n_rows);
  if (n_rows == 0) return cudaErrorInvalidValue;
  k_lidar<<<n_frames, 256, 0, st>>>(prims, prim_offsets, frames, r_max, j0, n_rows, range_sigma, slots, frame_hits);
  return cudaGetLastError();
}

int lidar_rays(float el_min, float el_max) {
  int j0 = -1, n_rows = 0;
  lidar_rows(el_min, el_max, &j0, &n_rows);
  return n_rows * kLidarAz;
}

cudaError_t launch_compact(const float4* slots, int n_rays, const int* frame_out_offset, const int* frame_take,
                           int n_frames, float* xyz, cudaStream_t st) {
  k_compact<<<n_frames, 256, 0, st>>>(slots, n_rays, frame_out_offset, frame_take, xyz);
  return cudaGetLastError();
}

}  // namespace amppi_sim
