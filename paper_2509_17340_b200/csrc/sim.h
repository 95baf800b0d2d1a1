// Synthetic input generator: the reference's scenario
// families (proj/src/sim_world.cpp:174-246) placed on the host and its
// per-cell jittered LiDAR (sim_world.cpp:248-328) ray-cast on the GPU.
// Feeds bench.py / tests with forest / verticals / inclines scans; not part of
// the plan path.  FP32 ray casting (sim_ray.h) whose host and device forms
// give the same bits; it follows the oracle's FP64 simulator to FP32
// accuracy (tests/test_lidar.py).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "sim_ray.h"

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

DevPrim to_device(const Prim& p);

// One CTA per frame; writes 3600 (ray) slots of xyz (NaN = miss).
cudaError_t launch_lidar(const DevPrim* prims, const int* prim_offsets, const Frame* frames, int n_frames,
                         float r_max, float el_min, float el_max, float range_sigma, float4* slots, int* frame_hits,
                         cudaStream_t st);
int lidar_rays(float el_min, float el_max);  // ray slots per frame
// Compact hits frame-major into per-scene packed points, capped per scene.
// (Host twin: scan_host, same Frame / DevPrim inputs, same output.)
cudaError_t launch_compact(const float4* slots, int n_rays, const int* frame_out_offset, const int* frame_take,
                           int n_frames, float* xyz, cudaStream_t st);

// Host form of launch_lidar + launch_compact for one scene's frames: the
// frames' hits in frame-then-ray order, at most `cap` points.
int64_t scan_host(const DevPrim* prims, int n_prims, const Frame* frames, int n_frames, float r_max, float el_min,
                  float el_max, float range_sigma, int64_t cap, float* xyz);

}  // namespace amppi_sim
