// Synthetic input generator: the reference's scenario
// families (proj/src/sim_world.cpp:174-246) placed on the host and its
// per-cell jittered LiDAR (sim_world.cpp:248-328) ray-cast on the GPU.
// Feeds bench.py / tests with forest / verticals / inclines scans; not part of
// the plan path and not bit-matched to the oracle's simulator (FP32 casts).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace amppi_sim {

enum Kind { kEmpty = 0, kForest = 1, kVerticals = 2, kInclines = 3, kTwoGap = 4 };

struct Prim {
  int kind;  // 0 vertical cylinder, 1 tilted cylinder, 2 box
  double base[3];
  double radius, height;
  double half[3];
  double tilt_axis[3];
  double tilt_angle;
};

std::vector<Prim> generate_scenario(int kind, uint64_t seed);

// Device form of one primitive (FP32), with the culling bounds precomputed.
struct DevPrim {
  float w2l[9];  // world -> local rotation (row-major)
  float base[3];
  float radius, height;
  float half[3];
  float lo[3], hi[3];  // world AABB
  float cx, cy, rad;   // azimuth-culling disc (sim_world.cpp:271-283)
  int kind;
};

DevPrim to_device(const Prim& p);

struct Frame {
  int scene;
  float p[3];
  float q[4];  // w, x, y, z
  unsigned long long seed;
};

// One CTA per frame; writes 3600 (ray) slots of xyz (NaN = miss).
cudaError_t launch_lidar(const DevPrim* prims, const int* prim_offsets, const Frame* frames, int n_frames,
                         float r_max, float el_min, float el_max, float range_sigma, float4* slots, int* frame_hits,
                         cudaStream_t st);
int lidar_rays(float el_min, float el_max);  // ray slots per frame
// Compact hits frame-major into per-scene packed points, capped per scene.
cudaError_t launch_compact(const float4* slots, int n_rays, const int* frame_out_offset, const int* frame_take,
                           int n_frames, float* xyz, cudaStream_t st);

}  // namespace amppi_sim
