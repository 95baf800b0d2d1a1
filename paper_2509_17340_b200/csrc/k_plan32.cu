// FP32 stage-I screening rollouts: the throughput kernel of the plan cycle.
//
// One thread per (scene, anchor, sample): counter-RNG draws, clamp, RK4 and
// every stage-I cost term fused in registers over the horizon
// (sample_rollout_perturbations + rollout_into + stage1_cost,
// mppi.cpp:16-61, costs.hpp:150-162).  The instance's nominal sequence and
// guide table are staged once per CTA in shared memory; the collision query
// reads the scene's grid (dilated occupancy bit first, then <= 9 contiguous
// cell ranges).  Its FP32 costs only select the softmin support; k_update
// re-evaluates that support in FP64.
#include <cuda_runtime.h>

#include "kernels.h"
#include "rollout.cuh"

namespace amppi_dev {

namespace {

constexpr int kMaxN = 64;

__global__ void __launch_bounds__(128) k_stage1_f32(BatchIn in, Perception P, Plan pl, DevConfig cfg, int iter) {
  __shared__ float s_unom[4 * kMaxN];
  __shared__ float4 s_guide[kMaxN];
  const int tiles = (cfg.K + blockDim.x - 1) / blockDim.x;
  int b = blockIdx.x;
  const int tile = b % tiles;
  b /= tiles;
  const int m = b % cfg.M;
  const int s = b / cfg.M;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) s_unom[i] = static_cast<float>(pl.nominal[smi * N * 4 + i]);
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_guide[i] = pl.guide32[smi * N + i];
  __syncthreads();
  const int k = tile * blockDim.x + threadIdx.x;
  if (k >= cfg.K) return;
  float* out = pl.cost32 + smi * cfg.K + k;
  if (!pl.alive[smi]) {
    *out = __int_as_float(0x7f800000);
    return;
  }
  RolloutEnv<float> env;
  env.unom = s_unom;
  env.guide = s_guide;
  env.N = N;
  env.dyn = make_dyn<float>(cfg);
  const double* gl = in.goals + 10 * s;
  env.pg = {static_cast<float>(gl[0]), static_cast<float>(gl[1]), static_cast<float>(gl[2])};
  env.vg = {static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  env.qg = {static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]), static_cast<float>(gl[9])};
  env.q_p = static_cast<float>(cfg.q_p);
  env.q_v = static_cast<float>(cfg.q_v);
  env.q_q = static_cast<float>(cfg.q_q);
  env.cs = static_cast<float>(cfg.col_scale);
  env.ca = static_cast<float>(cfg.col_slope);
  env.cdmin = static_cast<float>(cfg.col_d_min);
  env.cdmax = static_cast<float>(cfg.col_d_max);
  env.grid = P.grid[s];
  env.gstart = P.grid_start + static_cast<int64_t>(s) * (kGridCells + 1);
  env.gocc = P.grid_occ + static_cast<int64_t>(s) * kOccWords;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;

  const double* xs = in.states + 10 * s;
  St<float> x0;
  x0.p = {static_cast<float>(xs[0]), static_cast<float>(xs[1]), static_cast<float>(xs[2])};
  x0.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x0.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};

  CostSums<float> cs;
  if (in.injected) {
    const int64_t row = (((static_cast<int64_t>(s) * cfg.iterations + iter) * cfg.M + m) * cfg.K + k);
    cs = rollout_costs(x0, env, PertInjected<float>{in.injected + row * N * 4});
  } else {
    const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
    const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                      static_cast<float>(cfg.sigma[0]), static_cast<float>(cfg.sigma[1]),
                      static_cast<float>(cfg.sigma[2]), static_cast<float>(cfg.sigma[3])};
    cs = rollout_costs(x0, env, pr);
  }
  *out = cs.valid ? stage1_total(cs, static_cast<float>(cfg.q_track), static_cast<float>(cfg.q_vnorm),
                                 static_cast<float>(cfg.q_c), static_cast<float>(cfg.q_c_delta))
                  : __int_as_float(0x7f800000);
}

}  // namespace

cudaError_t launch_stage1_f32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                              cudaStream_t st, KernelTimer* timer) {
  const int64_t total = static_cast<int64_t>(in.S) * cfg.M * cfg.K;
  // latency mode (few rollouts): spread warps over SMs; throughput mode: 128
  const int threads = total < 148 * 128 ? 32 : 128;
  const int tiles = (cfg.K + threads - 1) / threads;
  TimedRegion t(timer, "k_stage1_f32", st);
  k_stage1_f32<<<static_cast<unsigned>(static_cast<int64_t>(in.S) * cfg.M * tiles), threads, 0, st>>>(in, P, pl, cfg,
                                                                                                       iter);
  return cudaGetLastError();
}

}  // namespace amppi_dev
