// FP32 stage-I screening rollouts: the throughput kernel of the plan cycle.
//
// One thread per (scene, anchor, sample): counter-RNG draws, clamp, RK4 and
// every stage-I cost term fused in registers over the horizon
// (sample_rollout_perturbations + rollout_into + stage1_cost,
// mppi.cpp:16-61, costs.hpp:150-162).  The instance's nominal sequence and
// guide table are staged once per CTA in shared memory; the collision query
// reads the scene's grid (dilated occupancy bit, then branch and bound over
// the 27 neighbour cells' point boxes).  Its FP32 costs only select the
// softmin support; k_refine re-evaluates that support in FP64 (DESIGN.md
// "Precision").
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "rollout.cuh"

namespace amppi_dev {

namespace {

constexpr int kMaxN = 64;

// mode 0: every sample, no bound.  mode 1: samples [0, k1) without bound.
// mode 2: samples [k1, K) aborted once their partial cost exceeds
// U + 2 window, U = min cost of samples [0, k1) -- an actual sample cost, so
// the instance minimum rho <= U and no softmin-support member (cost <= rho +
// 64 lambda) can abort.  Aborted samples report FLT_MAX.
template <int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) k_stage1_f32(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                                int iter, int mode, int k1) {
  __shared__ float s_unom[4 * kMaxN];
  __shared__ float4 s_guide[kMaxN];
  __shared__ float s_bound;
  const int k_lo = mode == 2 ? k1 : 0;
  const int k_n = mode == 0 ? cfg.K : (mode == 1 ? k1 : cfg.K - k1);
  const int tiles = (k_n + blockDim.x - 1) / blockDim.x;
  int b = blockIdx.x;
  const int tile = b % tiles;
  b /= tiles;
  const int m = b % cfg.M;
  const int s = b / cfg.M;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) s_unom[i] = static_cast<float>(pl.nominal[smi * N * 4 + i]);
  for (int i = threadIdx.x; i < N; i += blockDim.x) s_guide[i] = pl.guide32[smi * N + i];
  if (threadIdx.x < 32) {
    float u = __int_as_float(0x7f800000);
    if (mode == 2)
      for (int k = threadIdx.x; k < k1; k += 32) u = fminf(u, pl.cost32[smi * cfg.K + k]);
    for (int o = 16; o > 0; o >>= 1) u = fminf(u, __shfl_xor_sync(0xffffffffu, u, o));
    if (threadIdx.x == 0) {
      const float window = static_cast<float>(64.0 * cfg.lambda) + 1e-4f * fabsf(u) + 1e-2f;
      s_bound = (mode == 2 && u < 3.0e38f) ? u + 2.0f * window : __int_as_float(0x7f800000);
    }
  }
  __syncthreads();
  const int k = k_lo + tile * blockDim.x + threadIdx.x;
  if (k >= k_lo + k_n) return;
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
  env.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;

  env.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;
  env.abort_above = s_bound;
  env.wq_track = static_cast<float>(cfg.q_track);
  env.wq_vnorm = static_cast<float>(cfg.q_vnorm);
  env.wq_c = static_cast<float>(cfg.q_c);
  env.wq_cd = static_cast<float>(cfg.q_c_delta);

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
  *out = cs.aborted ? 3.4028234663852886e38f
                    : cs.valid ? stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd)
                               : __int_as_float(0x7f800000);
}

// Latency path, pass 1: one thread per rollout, everything but collision;
// positions to pl.pos32, partial cost to cost32.
__global__ void __launch_bounds__(32) k_stage1_traj32(BatchIn in, Perception P, Plan pl, DevConfig cfg, int iter) {
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
  const int64_t r = smi * cfg.K + k;
  float* out = pl.cost32 + r;
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
  env.has_guide = true;
  env.abort_above = __int_as_float(0x7f800000);
  env.wq_track = static_cast<float>(cfg.q_track);
  env.wq_vnorm = static_cast<float>(cfg.q_vnorm);
  env.wq_c = static_cast<float>(cfg.q_c);
  env.wq_cd = static_cast<float>(cfg.q_c_delta);
  const double* xs = in.states + 10 * s;
  St<float> x0;
  x0.p = {static_cast<float>(xs[0]), static_cast<float>(xs[1]), static_cast<float>(xs[2])};
  x0.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x0.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};
  float* pos = pl.pos32 + r * N * 4;
  CostSums<float> cs;
  if (in.injected) {
    const int64_t row = (((static_cast<int64_t>(s) * cfg.iterations + iter) * cfg.M + m) * cfg.K + k);
    cs = rollout_costs<float, PertInjected<float>, true>(x0, env, PertInjected<float>{in.injected + row * N * 4},
                                                         nullptr, nullptr, pos);
  } else {
    const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
    const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                      static_cast<float>(cfg.sigma[0]), static_cast<float>(cfg.sigma[1]),
                      static_cast<float>(cfg.sigma[2]), static_cast<float>(cfg.sigma[3])};
    cs = rollout_costs<float, PertRngF, true>(x0, env, pr, nullptr, nullptr, pos);
  }
  *out = cs.valid ? stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd) : __int_as_float(0x7f800000);
}

// Latency path, pass 2: one warp per rollout, lane j -> collision term of step j.
__global__ void __launch_bounds__(128) k_stage1_col32(Perception P, Plan pl, DevConfig cfg, int64_t n_rollouts) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n_rollouts) return;
  const float base = pl.cost32[r];
  if (!isfinite(base)) return;  // invalid rollout or dead instance
  const int s = static_cast<int>(r / (static_cast<int64_t>(cfg.M) * cfg.K));
  const GridMeta g = P.grid[s];
  const uint4* cells = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;

  const uint32_t* occ = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  const float4* pts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  const float cs = static_cast<float>(cfg.col_scale), ca = static_cast<float>(cfg.col_slope);
  const float dmin = static_cast<float>(cfg.col_d_min), dmax = static_cast<float>(cfg.col_d_max);
  const float* pos = pl.pos32 + r * cfg.N * 4;
  float col = 0.f;
  for (int j = lane; j < cfg.N; j += 32) {
    const V3<float> p{pos[4 * j], pos[4 * j + 1], pos[4 * j + 2]};
    const float d2 = nearest_sq_fast(g, cells, occ, pts, p, dmax * dmax * 1.0001f, dmin * dmin);
    col += collision_term(sqrtf(d2), cs, ca, dmin, dmax);
  }
  for (int o = 16; o > 0; o >>= 1) col += __shfl_xor_sync(0xffffffffu, col, o);
  if (lane == 0) pl.cost32[r] = base + col;
}

}  // namespace

cudaError_t launch_stage1_f32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                              cudaStream_t st, KernelTimer* timer) {
  const int64_t total = static_cast<int64_t>(in.S) * cfg.M * cfg.K;
  const int64_t SM = static_cast<int64_t>(in.S) * cfg.M;
  static const char* sched = std::getenv("AMPPI_SCREEN");  // experiment switch: "single" disables the bound
  const bool single = sched && std::strcmp(sched, "single") == 0;
  // throughput mode: 64 registers (8 CTAs = 32 warps per SM, a few bytes of
  // L1-resident spill); latency mode: no cap (fastest single rollout)
  auto kern = k_stage1_f32<8>;
  if (single || total < 148 * 128 * 4 || cfg.K <= 64) {
    // latency mode (few rollouts): one pass, warps spread over the SMs
    const int threads = total < 148 * 128 ? 32 : 128;
    const int tiles = (cfg.K + threads - 1) / threads;
    if (total < kLatencyRollouts) {
      {
        TimedRegion t(timer, "k_stage1_traj32", st);
        k_stage1_traj32<<<static_cast<unsigned>(SM * ((cfg.K + 31) / 32)), 32, 0, st>>>(in, P, pl, cfg, iter);
      }
      TimedRegion t(timer, "k_stage1_col32", st);
      k_stage1_col32<<<static_cast<unsigned>((total * 32 + 127) / 128), 128, 0, st>>>(P, pl, cfg, total);
      return cudaGetLastError();
    }
    TimedRegion t(timer, "k_stage1_f32", st);
    kern<<<static_cast<unsigned>(SM * tiles), threads, 0, st>>>(in, P, pl, cfg, iter, 0, 0);
    return cudaGetLastError();
  }
  const int k1 = 32;
  {
    TimedRegion t(timer, "k_stage1_f32_bound", st);
    kern<<<static_cast<unsigned>(SM), 32, 0, st>>>(in, P, pl, cfg, iter, 1, k1);
  }
  const int tiles = (cfg.K - k1 + 127) / 128;
  TimedRegion t(timer, "k_stage1_f32", st);
  kern<<<static_cast<unsigned>(SM * tiles), 128, 0, st>>>(in, P, pl, cfg, iter, 2, k1);
  return cudaGetLastError();
}

#ifdef AMPPI_STATS
extern "C" int amppi_query_stats(unsigned long long* out5, int reset) {
  cudaMemcpyFromSymbol(out5, g_query_stats, sizeof(unsigned long long) * 5);
  if (reset) {
    unsigned long long z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_query_stats, z, sizeof(z));
  }
  return 0;
}
#endif

}  // namespace amppi_dev
