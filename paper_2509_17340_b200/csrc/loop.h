// GPU-resident closed loop: the reference's
// execute_cycle (proj/src/ensemble.cpp:245-305) with the vehicle, its
// PointCloudBuffer ring (perception.cpp:44-62) and its LiDAR
// (sim_world.cpp:248-328) kept on the device, so a C2-style episode runs with
// no per-cycle host traffic.  FP64 throughout, with the reference's operation
// order; the transcendentals are CUDA's (<= 2 ulp from glibc), so a long
// episode tracks the CPU loop closely rather than bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "layout.h"

namespace amppi_dev {

constexpr int kLidarRays = kAz * kEl;  // ray slots per frame (rows outside the FOV stay empty)

// One obstacle in world coordinates (sim_world.hpp:16-28) with the values the
// reference derives from it: world -> local rotation (transpose of the
// Eigen toRotationMatrix of the tilt quaternion), world AABB, azimuth-culling
// disc (sim_world.cpp:107-117, :271-283).
struct LoopPrim {
  int kind;  // 0 vertical cylinder, 1 tilted cylinder, 2 box
  double base[3];
  double radius, height;
  double half[3];
  double w2l[9];  // row-major world_to_local
  double lo[3], hi[3];
  double cx, cy, rad;
};

// Episode state on the device (ensemble.cpp:238-243 EpisodeState).
struct LoopState {
  double x[10];         // p, q (w x y z), v
  double last[4];       // last applied control
  double t;             // episode time
  uint64_t cycle;
  int32_t prev_len;     // 0 (no previous plan) or N
  int32_t failures;     // consecutive planner failures
  int32_t status;       // 0 running, 1 success, 2 collision, 3 timeout, 4 planner_failure
  int32_t ring_head;    // slot of the newest frame
  int32_t ring_size;    // frames held
};

// Per-cycle record (the CPU loop's CycleRecord minus the cloud); the same
// layout as amppi_loop_record.
struct LoopRecord {
  uint64_t cycle;
  int32_t planned, winner;
  double x[10];         // state the plan saw
  double control[4];    // applied control (hover on failure)
  double stage2;        // winner's stage-II cost
  int32_t status;       // episode status after this cycle
  int32_t n_points;     // points in the buffer the plan saw
  // TrajectoryLog LogRecord (ensemble.hpp:84-94, ensemble.cpp:280-290): after the step
  double t;             // episode time
  double x_after[10];   // p, q, v after the vehicle step
  double clearance;     // true_clearance of the new position
  double breakdown[5];  // winner's cost breakdown (zeros when not planned)
};

// EpisodeMetrics (metrics.hpp:11-18), same layout as amppi_episode_metrics.
struct LoopMetrics {
  double avg_vel, max_vel, smoothness, path_length, avg_clearance, min_clearance;
};

struct LoopParams {
  int n_prims;
  int capacity;         // PointCloudBuffer frames
  uint64_t seed;        // plan seed; frame seed = mix64(seed) + cycle
  double r_max, el_min, el_max, range_sigma;
  double goal_radius, timeout, drone_radius;
  int max_failures;
  double step_dt;       // 1 / replan_hz
};

struct LoopDev {
  const LoopPrim* prims;
  LoopState* st;
  double* frames;       // [capacity][kLidarRays][3] ring of world-frame scans
  int32_t* frame_n;     // [capacity]
  double* cloud;        // [capacity*kLidarRays*3] buffer contents, oldest frame first
  int64_t* offsets;     // [2] = {0, n}
  double* goal;         // [10] p v q
  double* nominal;      // [N*4] previous winner nominal
  double* hover;        // [4]
  uint64_t* cycles;     // [1] plan cycle counter (BatchIn view)
  uint64_t* seeds;      // [1]
  LoopRecord* records;  // [max_records]
  int64_t max_records;
};

std::vector<LoopPrim> loop_scenario(int kind, uint64_t seed);  // generate_scenario (sim_world.cpp:174-246)

// One cycle's kernels before / after the plan (the plan itself is the normal
// snapshot + plan launch on the BatchIn view of the loop state).
cudaError_t launch_loop_scan(const LoopDev& L, const LoopParams& prm, cudaStream_t st);
cudaError_t launch_loop_step(const LoopDev& L, const LoopParams& prm, const Plan& pl, const DevConfig& cfg,
                             cudaStream_t st);
// compute_metrics (metrics.cpp:12-49) over records [0, n); n >= 4.
cudaError_t launch_loop_metrics(const LoopDev& L, int64_t n, LoopMetrics* out, cudaStream_t st);

}  // namespace amppi_dev
