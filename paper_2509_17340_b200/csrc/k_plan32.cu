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

#include <algorithm>
#include <cstdlib>
#include <cstring>


#include "kernels.h"
#include "rollout.cuh"

namespace amppi_dev {

namespace {

constexpr int kMaxN = 64;

// The screening kernels' float constants, converted once on the host and passed by
// value: kernel parameters live in the constant bank, so the FP32 code reads
// them as operands instead of re-converting the FP64 config (F2F) inside its
// loops.
struct ScreenConsts {
  Dyn<float> dyn;
  float q_p, q_v, q_q, cs, ca, cdmin, cdmax;
  float wq_track, wq_vnorm, wq_c, wq_cd;
  float sigma[4];
  float reach2, band, dthr_cap;
};

ScreenConsts screen_consts(const DevConfig& c) {
  ScreenConsts k{};
  k.dyn.mass = static_cast<float>(c.mass);
  k.dyn.inv_mass = static_cast<float>(1.0 / c.mass);
  k.dyn.gx = static_cast<float>(c.gravity[0]);
  k.dyn.gy = static_cast<float>(c.gravity[1]);
  k.dyn.gz = static_cast<float>(c.gravity[2]);
  k.dyn.dt = static_cast<float>(c.dyn_dt);
  k.dyn.half_dt = static_cast<float>(0.5 * c.dyn_dt);
  k.dyn.dt6 = static_cast<float>(c.dyn_dt / 6.0);
  k.dyn.tmin = static_cast<float>(c.thrust_min);
  k.dyn.tmax = static_cast<float>(c.thrust_max);
  k.dyn.wxy = static_cast<float>(c.omega_xy_max);
  k.dyn.wz = static_cast<float>(c.omega_z_max);
  k.q_p = static_cast<float>(c.q_p);
  k.q_v = static_cast<float>(c.q_v);
  k.q_q = static_cast<float>(c.q_q);
  k.cs = static_cast<float>(c.col_scale);
  k.ca = static_cast<float>(c.col_slope);
  k.cdmin = static_cast<float>(c.col_d_min);
  k.cdmax = static_cast<float>(c.col_d_max);
  k.wq_track = static_cast<float>(c.q_track);
  k.wq_vnorm = static_cast<float>(c.q_vnorm);
  k.wq_c = static_cast<float>(c.q_c);
  k.wq_cd = static_cast<float>(c.q_c_delta);
  for (int i = 0; i < 4; ++i) k.sigma[i] = static_cast<float>(c.sigma[i]);
  // screen_reach2 / amb_band (device_math.cuh) with the same float operations
  k.band = 1e-4f * k.cdmax + 1e-4f;
  const float r = k.cdmax + k.band;
  k.reach2 = r * r * 1.0001f;
  k.dthr_cap = (k.cdmax - k.band) * 0.9999995f;
  return k;
}

// The current nominal in float (one thread per instance step), the table the
// screening kernels bulk-copy into shared memory.
__global__ void k_unom32(Plan pl, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* u = pl.nominal + 4 * i;
  pl.unom32[i] = make_float4(static_cast<float>(u[0]), static_cast<float>(u[1]), static_cast<float>(u[2]),
                             static_cast<float>(u[3]));
}

// mode 0: every sample, no bound.  mode 1: samples [0, k1) without bound.
// mode 2: samples [k1, K) aborted once their partial cost exceeds
// U + window(U), U = min cost of samples [0, k1) -- an actual sample cost,
// so the instance minimum rho <= U.  The FP32 partial sums only grow towards
// the final FP32 cost (non-negative terms, monotone rounding), so an aborted
// sample ends above rho + window(rho) (window(U) >= window(rho)): outside the
// support k_support selects.  Aborted samples report FLT_MAX.
template <int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) k_stage1_f32(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                                const ScreenConsts sc, int iter, int mode, int k1) {
  __shared__ float4 s_unom[kMaxN];
  __shared__ float4 s_guide[kMaxN];
  __shared__ float s_bound;
  __shared__ uint64_t s_bar;
  const int k_lo = mode == 2 ? cfg.k_lo + k1 : cfg.k_lo;
  const int k_n = mode == 0 ? cfg.k_hi - cfg.k_lo : (mode == 1 ? k1 : cfg.k_hi - cfg.k_lo - k1);
  const int tiles = (k_n + blockDim.x - 1) / blockDim.x;
  int b = blockIdx.x;
  const int tile = b % tiles;
  b /= tiles;
  const int m = b % cfg.M;
  const int s = b / cfg.M;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  if (threadIdx.x == 0) {  // the instance's nominal and guide tables: bulk async copies into smem
    mbar_init(&s_bar, 1);
    mbar_expect_tx(&s_bar, 2u * 16u * static_cast<uint32_t>(N));
    bulk_copy_g2s(s_unom, pl.unom32 + smi * N, 16u * N, &s_bar);
    bulk_copy_g2s(s_guide, pl.guide32 + smi * N, 16u * N, &s_bar);
  }
  if (threadIdx.x < 32) {
    float u = __int_as_float(0x7f800000);
    if (mode == 2)
      for (int k = cfg.k_lo + threadIdx.x; k < cfg.k_lo + k1; k += 32) {
        const float c = pl.cost32[smi * cfg.K + k];
        if (!signbit(c)) u = fminf(u, c);  // U is an unflagged sample's cost
      }
    for (int o = 16; o > 0; o >>= 1) u = fminf(u, __shfl_xor_sync(0xffffffffu, u, o));
    if (threadIdx.x == 0) {
      const float window = static_cast<float>(kWindowLambdas * cfg.lambda) + 1e-4f * fabsf(u) + 1e-2f;
      // + 1e-6 |u| covers the float rounding of the threshold itself
      s_bound = (mode == 2 && u < 3.0e38f) ? u + window + (1e-6f * fabsf(u) + 1e-5f) : __int_as_float(0x7f800000);
    }
  }
  __syncthreads();
  mbar_wait(&s_bar, 0);
  const int k = k_lo + tile * blockDim.x + threadIdx.x;
  if (k >= k_lo + k_n) return;
  float* out = pl.cost32 + smi * cfg.K + k;
  if (!pl.alive[smi]) {
    *out = __int_as_float(0x7f800000);
    return;
  }
  RolloutEnv<float> env;
  env.unom = reinterpret_cast<const float*>(s_unom);
  env.guide = s_guide;
  env.N = N;
  env.dyn = sc.dyn;
  const double* gl = in.goals + 10 * s;
  env.pg = to_local_f(P.grid[s], gl);
  env.vg = {static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  env.qg = {static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]), static_cast<float>(gl[9])};
  env.q_p = sc.q_p;
  env.q_v = sc.q_v;
  env.q_q = sc.q_q;
  env.cs = sc.cs;
  env.ca = sc.ca;
  env.cdmin = sc.cdmin;
  env.cdmax = sc.cdmax;
  env.grid = P.grid[s];
  env.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;

  env.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  env.gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;
  env.abort_above = s_bound;
  env.wq_track = sc.wq_track;
  env.wq_vnorm = sc.wq_vnorm;
  env.wq_c = sc.wq_c;
  env.wq_cd = sc.wq_cd;
  env.reach2 = sc.reach2;
  env.band = sc.band;

  const double* xs = in.states + 10 * s;
  St<float> x0;
  x0.p = to_local_f(P.grid[s], xs);
  x0.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x0.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};

  CostSums<float> cs;
  if (in.injected) {
    const int64_t row = (((static_cast<int64_t>(s) * cfg.iterations + iter) * cfg.M + m) * cfg.K + k);
    cs = rollout_costs(x0, env, PertInjected<float>{in.injected + row * N * 4});
  } else {
    const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
    const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                      sc.sigma[0], sc.sigma[1], sc.sigma[2], sc.sigma[3]};
    cs = rollout_costs(x0, env, pr);
  }
  *out = cs.aborted ? 3.4028234663852886e38f
                    : cs.valid ? screen_store(stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd), cs.amb)
                               : __int_as_float(0x7f800000);
}

// Bound pass: samples [k_lo, k_lo + B) of G instances per warp (B = 32 / G
// lanes each), full horizon, no abort -- their minimum is the abort bound of
// the main pass.  Packing several instances into a warp cuts the warps of the
// pass by G: every lane's collision queries diverge anyway (each lane walks
// its own cells and leaves), so a warp's time hardly depends on whether its
// lanes share an instance.
template <int G>
__global__ void __launch_bounds__(32) k_stage1_bound(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                     const ScreenConsts sc, int iter) {
  constexpr int B = 32 / G;
  __shared__ float4 s_unom[G][kMaxN];
  __shared__ float4 s_guide[G][kMaxN];
  __shared__ uint64_t s_bar;
  const int lane = threadIdx.x, g = lane / B;
  const int64_t SMn = static_cast<int64_t>(in.S) * cfg.M;
  const int64_t smi0 = static_cast<int64_t>(blockIdx.x) * G;
  const int n_inst = static_cast<int>(SMn - smi0 < G ? SMn - smi0 : G);
  const int N = cfg.N;
  if (lane == 0) {  // the instances' nominal and guide tables: bulk async copies into smem
    mbar_init(&s_bar, 1);
    mbar_expect_tx(&s_bar, 2u * 16u * static_cast<uint32_t>(N) * static_cast<uint32_t>(n_inst));
    for (int i = 0; i < n_inst; ++i) {
      bulk_copy_g2s(s_unom[i], pl.unom32 + (smi0 + i) * N, 16u * N, &s_bar);
      bulk_copy_g2s(s_guide[i], pl.guide32 + (smi0 + i) * N, 16u * N, &s_bar);
    }
  }
  __syncwarp();
  mbar_wait(&s_bar, 0);
  if (g >= n_inst) return;
  const int64_t smi = smi0 + g;
  const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
  const int k = cfg.k_lo + lane % B;
  float* out = pl.cost32 + smi * cfg.K + k;
  if (!pl.alive[smi]) {
    *out = __int_as_float(0x7f800000);
    return;
  }
  RolloutEnv<float> env;
  env.unom = reinterpret_cast<const float*>(s_unom[g]);
  env.guide = s_guide[g];
  env.N = N;
  env.dyn = sc.dyn;
  const double* gl = in.goals + 10 * s;
  env.pg = to_local_f(P.grid[s], gl);
  env.vg = {static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  env.qg = {static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]), static_cast<float>(gl[9])};
  env.q_p = sc.q_p;
  env.q_v = sc.q_v;
  env.q_q = sc.q_q;
  env.cs = sc.cs;
  env.ca = sc.ca;
  env.cdmin = sc.cdmin;
  env.cdmax = sc.cdmax;
  env.grid = P.grid[s];
  env.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  env.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  env.gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;
  env.abort_above = __int_as_float(0x7f800000);
  env.wq_track = sc.wq_track;
  env.wq_vnorm = sc.wq_vnorm;
  env.wq_c = sc.wq_c;
  env.wq_cd = sc.wq_cd;
  env.reach2 = sc.reach2;
  env.band = sc.band;
  const double* xs = in.states + 10 * s;
  St<float> x0;
  x0.p = to_local_f(P.grid[s], xs);
  x0.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x0.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};
  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                    sc.sigma[0], sc.sigma[1], sc.sigma[2], sc.sigma[3]};
  const CostSums<float> cs = rollout_costs(x0, env, pr);
  *out = cs.valid ? screen_store(stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd), cs.amb)
                  : __int_as_float(0x7f800000);
}

// One screening step j of a rollout (the loop body of rollout_costs<float>):
// costs on states[j], perturbed clamped control, control costs, the
// partial-cost bound, RK4.  Returns 0 (continue), 1 (aborted), 2 (invalid).
// The collision query runs last and knows the partial cost, so it only has
// to find one point inside the radius whose collision term would exhaust the
// remaining budget (then the sample aborts); otherwise it returns the exact
// distance.  Same sums in the same order as rollout_costs for every sample
// that is not aborted.  Split in two around the query (screen_pre /
// screen_post) so a warp can answer its lanes' queries together.
struct StepCtl {
  float u[4];      // the step's clamped control
  float stop2;     // the query may stop below this squared distance
  bool abortable;  // a point closer than sqrt(stop2) aborts the sample
};

template <typename Pert>
__device__ __forceinline__ int screen_pre(const St<float>& x, CostSums<float>& s, float (&up)[4], int j,
                                          const RolloutEnv<float>& env, const Pert& pert, StepCtl& c) {
  const Dyn<float>& dy = env.dyn;
  const int N = env.N;
  AMPPI_STAT(8 + j, 1);
  s.trk = s.trk + norm3(x.p - env.guide_at(j));
  s.vn = s.vn + sqnorm(x.v);
  s.goal = s.goal + env.q_p * norm3(x.p - env.pg);
  s.goal = s.goal + env.q_v * norm3(x.v - env.vg);
  s.goal = s.goal + env.q_q * env.attitude(x.q);
  float d[4];
  pert(j, d);
  // one 16-byte shared load of the step's nominal; min/max clamps (the
  // screening's controls are finite, so std::clamp's NaN pass-through is moot)
  const float4 un = reinterpret_cast<const float4*>(env.unom)[j];
  const float u0 = fminf(fmaxf(un.x + d[0], dy.tmin), dy.tmax);
  const float u1 = fminf(fmaxf(un.y + d[1], -dy.wxy), dy.wxy);
  const float u2 = fminf(fmaxf(un.z + d[2], -dy.wxy), dy.wxy);
  const float u3 = fminf(fmaxf(un.w + d[3], -dy.wz), dy.wz);
  if (j + 1 < N) {
    s.mag = s.mag + (((u0 * u0 + u1 * u1) + u2 * u2) + u3 * u3);
    if (j >= 1) {
      const float e0 = u0 - up[0], e1 = u1 - up[1], e2 = u2 - up[2], e3 = u3 - up[3];
      s.rate = s.rate + (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3);
    }
  }
  up[0] = u0; up[1] = u1; up[2] = u2; up[3] = u3;
  c.u[0] = u0; c.u[1] = u1; c.u[2] = u2; c.u[3] = u3;
  const float part =
      ((env.wq_track * s.trk + env.wq_vnorm * s.vn) + (env.wq_c * s.mag + env.wq_cd * s.rate)) + (s.goal + s.col);
  if (part > env.abort_above) return 1;
  // Abort radius: a point closer than d_thr adds more than the remaining
  // budget (C exp(-a (d_thr - d_min)) = budget e^0.001), so finding one ends
  // the sample; otherwise the query returns the exact distance (>= d_thr).
  c.stop2 = env.cdmin * env.cdmin;
  c.abortable = false;
  const float budget = env.abort_above - part;
  if (budget < env.cs) {
    // (approximate division and log: their errors are far inside the 1e-3 slack)
    float d_thr = env.cdmin + __fdividef(__logf(__fdividef(env.cs, budget)) - 1e-3f, env.ca);
    d_thr = fminf(d_thr, env.dthr_cap);  // (d_max - band)(1 - 5e-7): d < d_thr is a counted term
    if (d_thr > env.cdmin) {
      c.stop2 = d_thr * d_thr;
      c.abortable = true;
    }
  }
  return 0;
}

// The rest of the step once the query answered d2: collision term, bound, RK4.
__device__ __forceinline__ int screen_post(St<float>& x, CostSums<float>& s, const StepCtl& c, float d2,
                                           const RolloutEnv<float>& env) {
  if (c.abortable && d2 < c.stop2) return 1;
  s.col = s.col + screen_collision_b(d2, env.cs, env.ca, env.cdmin, env.cdmax, env.band, s.amb);
  if (((env.wq_track * s.trk + env.wq_vnorm * s.vn) + (env.wq_c * s.mag + env.wq_cd * s.rate)) + (s.goal + s.col) >
      env.abort_above)
    return 1;
  const St<float> nx = rk4_normalized(x, c.u[0], V3<float>{c.u[1], c.u[2], c.u[3]}, env.dyn);
  if (!state_finite(nx)) return 2;
  x = nx;
  return 0;
}

template <typename Pert>
__device__ __forceinline__ int screen_step(St<float>& x, CostSums<float>& s, float (&up)[4], int j,
                                           const RolloutEnv<float>& env, const Pert& pert, float* last_d2 = nullptr) {
  StepCtl c;
  if (screen_pre(x, s, up, j, env, pert, c)) return 1;
  // step 0 is x0 for every sample: its query was answered once per CTA
  const float d2 = j == 0 ? env.d2_x0
                          : nearest_sq_fast(env.grid, env.grec, env.gnbr, env.gleaf, env.gpts, x.p, env.reach2,
                                            c.stop2, &env.hint);
  if (last_d2) *last_d2 = d2;
  return screen_post(x, s, c, d2, env);
}


// Main screening pass with lane compaction: samples [k1, K) of one instance
// per CTA, stepped in lockstep; every kCompact steps the live samples (not
// yet past the abort bound) are packed into the lowest threads through shared
// memory, so warps whose lanes all aborted stop issuing.  Same per-sample
// arithmetic as k_stage1_f32 mode 2.
constexpr int kScreenThreads = 128;
#ifndef AMPPI_MAIN_THREADS  // experiment switches (make variant DEFS=...)
#define AMPPI_MAIN_THREADS 224
#endif
#ifndef AMPPI_MAIN_MINBLOCKS
#define AMPPI_MAIN_MINBLOCKS 5
#endif
#ifndef AMPPI_MAIN_COMPACT
#define AMPPI_MAIN_COMPACT 10
#endif
constexpr int kMainThreads = AMPPI_MAIN_THREADS, kMainMinBlocks = AMPPI_MAIN_MINBLOCKS;
#ifndef AMPPI_MAIN_GROUPS
#define AMPPI_MAIN_GROUPS 1
#endif
constexpr int kMainGroups = AMPPI_MAIN_GROUPS;
#ifndef AMPPI_BOUND_SAMPLES
#define AMPPI_BOUND_SAMPLES 32
#endif
constexpr int kBoundSamples = AMPPI_BOUND_SAMPLES;  // 32, 16, 8 or 4
#ifndef AMPPI_BOUND_LARGE
#define AMPPI_BOUND_LARGE 1024
#endif
constexpr int kBoundLarge = AMPPI_BOUND_LARGE;  // bound-sample cap when K >= 2048 (K / 8 below it)
static_assert(kBoundLarge % 32 == 0, "whole warps of bound samples");
static_assert(32 % kBoundSamples == 0, "bound samples divide a warp");
constexpr int kMainCompact = AMPPI_MAIN_COMPACT;
constexpr int kStateWords = 22;  // p(3) q(4) v(3) trk vn mag rate goal col up(4) hint amb

// Samples [k_lo + kb0, k_lo + kend) of every instance, aborted against the
// minimum of samples [k_lo, k_lo + nb) (main pass: kb0 = nb = 32; bound
// pass: kb0 = nb = 1, kend = 32).
template <int kMinBlocks, int kCompact, int kT = kScreenThreads>
__global__ void __launch_bounds__(kT, kMinBlocks)
    k_stage1_f32c(BatchIn in, Perception P, Plan pl, DevConfig cfg, const ScreenConsts sc, int iter, int kb0, int kend,
                  int nb) {
  __shared__ float4 s_unom[kMaxN];
  __shared__ float4 s_guide[kMaxN];
  __shared__ float s_bound;
  __shared__ uint64_t s_bar;
  __shared__ float s_state[kStateWords][kT];
  __shared__ int s_k[kT];
  __shared__ int s_wcount[2][kT / 32];
  __shared__ uint32_t s_bcnt[64], s_boff[64];  // cell-order buckets of the repack
  if (threadIdx.x < 64) s_bcnt[threadIdx.x] = 0u;
  const int k_n = kend - kb0;
  const int tiles = (k_n + kT - 1) / kT;
  int b = blockIdx.x;
  const int tile = b % tiles;
  b /= tiles;
  const int m = b % cfg.M;
  const int s = b / cfg.M;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* __restrict__ out = pl.cost32 + smi * cfg.K;
  if (!pl.alive[smi]) {
    const int k = cfg.k_lo + kb0 + tile * kT + tid;
    if (k < cfg.k_lo + kend) out[k] = __int_as_float(0x7f800000);
    return;
  }
  if (tid == 0) {  // the instance's nominal and guide tables: bulk async copies into smem
    mbar_init(&s_bar, 1);
    mbar_expect_tx(&s_bar, 2u * 16u * static_cast<uint32_t>(N));
    bulk_copy_g2s(s_unom, pl.unom32 + smi * N, 16u * N, &s_bar);
    bulk_copy_g2s(s_guide, pl.guide32 + smi * N, 16u * N, &s_bar);
  }
  if (tid < 32) {
    float u = __int_as_float(0x7f800000);
    for (int k = cfg.k_lo + tid; k < cfg.k_lo + nb; k += 32)
      if (!signbit(out[k])) u = fminf(u, out[k]);  // U is an unflagged sample's cost
    for (int o = 16; o > 0; o >>= 1) u = fminf(u, __shfl_xor_sync(0xffffffffu, u, o));
    if (tid == 0) {
      const float window = static_cast<float>(kWindowLambdas * cfg.lambda) + 1e-4f * fabsf(u) + 1e-2f;
      // + 1e-6 |u| covers the float rounding of the threshold itself
      s_bound = u < 3.0e38f ? u + window + (1e-6f * fabsf(u) + 1e-5f) : __int_as_float(0x7f800000);
    }
  }
  __syncthreads();
  mbar_wait(&s_bar, 0);
  RolloutEnv<float> env;
  env.unom = reinterpret_cast<const float*>(s_unom);
  env.guide = s_guide;
  env.N = N;
  env.dyn = sc.dyn;
  const double* gl = in.goals + 10 * s;
  env.pg = to_local_f(P.grid[s], gl);
  env.vg = {static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  env.qg = {static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]), static_cast<float>(gl[9])};
  env.q_p = sc.q_p;
  env.q_v = sc.q_v;
  env.q_q = sc.q_q;
  env.cs = sc.cs;
  env.ca = sc.ca;
  env.cdmin = sc.cdmin;
  env.cdmax = sc.cdmax;
  env.grid = P.grid[s];
  env.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  env.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  env.gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;
  env.abort_above = s_bound;
  env.wq_track = sc.wq_track;
  env.wq_vnorm = sc.wq_vnorm;
  env.wq_c = sc.wq_c;
  env.wq_cd = sc.wq_cd;
  env.reach2 = sc.reach2;
  env.band = sc.band;
  env.dthr_cap = sc.dthr_cap;

  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  const uint64_t seed = in.seeds[s];
  PertRngF pr{0ull, sc.sigma[0], sc.sigma[1], sc.sigma[2], sc.sigma[3]};
  int k = cfg.k_lo + kb0 + tile * kT + tid;
  bool live = k < cfg.k_lo + kend;
  pr.key = stream_key(seed, static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k));
  const double* xs = in.states + 10 * s;
  St<float> x;
  x.p = to_local_f(P.grid[s], xs);
  x.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};
  CostSums<float> cs{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, true, false, false};
  float up[4] = {0.f, 0.f, 0.f, 0.f};
  {  // the step-0 collision query (exact; every sample starts at x0)
    __shared__ float s_d2;
    __shared__ uint32_t s_hint;
    if (tid == 0) {
      uint32_t h = kNoHint;
      s_d2 = nearest_sq_fast(env.grid, env.grec, env.gnbr, env.gleaf, env.gpts, x.p, env.reach2,
                             env.cdmin * env.cdmin, &h);
      s_hint = h;
    }
    __syncthreads();
    env.d2_x0 = s_d2;
    env.hint = s_hint;
  }
  int round = 0;
  for (int j0 = 0; j0 < N; j0 += kCompact, ++round) {
    const int j1 = min(j0 + kCompact, N);
    if (live) {
      for (int j = j0; j < j1; ++j) {
        const int st = screen_step(x, cs, up, j, env, pr);
        if (st) {
          out[k] = st == 1 ? 3.4028234663852886e38f : __int_as_float(0x7f800000);
          live = false;
          break;
        }
      }
    }
    if (j1 >= N) break;
    const unsigned bal = __ballot_sync(0xffffffffu, live);
    int* wc = s_wcount[round & 1];
    if (lane == 0) wc[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0, live_warps = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) {
      const int c = wc[w];
      before += w < warp ? c : 0;
      total += c;
      live_warps += c > 0;
    }
    if (total == 0) return;
    // Repack when it retires a warp or the live samples span more than one
    // warp; in the latter case the samples are also ordered by grid cell
    // (counting sort over 64 hash buckets), so spatially close samples share
    // a warp and walk the same cells and leaves in their collision queries
    // (C5 main pass -2%, measured; the order does not change any result).
    const bool sorted = total > 32;
    if (sorted || (total + 31) / 32 < live_warps) {
      int slot = before + __popc(bal & ((1u << lane) - 1u));
      if (sorted) {
        int bkt = 0;
        uint32_t rank = 0;
        if (live) {
          const int cx = __float2int_rd((x.p.x - env.grid.origin_f[0]) * env.grid.inv_h_f);
          const int cy = __float2int_rd((x.p.y - env.grid.origin_f[1]) * env.grid.inv_h_f);
          const int cz = __float2int_rd((x.p.z - env.grid.origin_f[2]) * env.grid.inv_h_f);
          bkt = static_cast<int>((static_cast<uint32_t>(cx) * 73856093u ^ static_cast<uint32_t>(cy) * 19349663u ^
                                  static_cast<uint32_t>(cz) * 83492791u) >> 26);
          rank = atomicAdd(&s_bcnt[bkt], 1u);
        }
        __syncthreads();
        if (warp == 0) {
          const uint32_t c0 = s_bcnt[2 * lane], c1 = s_bcnt[2 * lane + 1];
          uint32_t v = c0 + c1;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
          }
          const uint32_t ex = v - (c0 + c1);
          s_boff[2 * lane] = ex;
          s_boff[2 * lane + 1] = ex + c0;
          s_bcnt[2 * lane] = 0u;
          s_bcnt[2 * lane + 1] = 0u;
        }
        __syncthreads();
        if (live) slot = static_cast<int>(s_boff[bkt] + rank);
      }
      if (live) {
        float* st = &s_state[0][slot];
        st[0 * kT] = x.p.x; st[1 * kT] = x.p.y; st[2 * kT] = x.p.z;
        st[3 * kT] = x.q.w; st[4 * kT] = x.q.x; st[5 * kT] = x.q.y;
        st[6 * kT] = x.q.z;
        st[7 * kT] = x.v.x; st[8 * kT] = x.v.y; st[9 * kT] = x.v.z;
        st[10 * kT] = cs.trk; st[11 * kT] = cs.vn; st[12 * kT] = cs.mag;
        st[13 * kT] = cs.rate; st[14 * kT] = cs.goal; st[15 * kT] = cs.col;
        st[16 * kT] = up[0]; st[17 * kT] = up[1]; st[18 * kT] = up[2];
        st[19 * kT] = up[3];
        st[20 * kT] = __uint_as_float(env.hint);
        st[21 * kT] = cs.amb ? 1.f : 0.f;
        s_k[slot] = k;
      }
      __syncthreads();
      live = tid < total;
      if (live) {
        const float* st = &s_state[0][tid];
        x.p = {st[0 * kT], st[1 * kT], st[2 * kT]};
        x.q = {st[3 * kT], st[4 * kT], st[5 * kT], st[6 * kT]};
        x.v = {st[7 * kT], st[8 * kT], st[9 * kT]};
        cs.trk = st[10 * kT]; cs.vn = st[11 * kT]; cs.mag = st[12 * kT];
        cs.rate = st[13 * kT]; cs.goal = st[14 * kT]; cs.col = st[15 * kT];
        up[0] = st[16 * kT]; up[1] = st[17 * kT]; up[2] = st[18 * kT];
        up[3] = st[19 * kT];
        env.hint = __float_as_uint(st[20 * kT]);
        cs.amb = st[21 * kT] != 0.f;
        k = s_k[tid];
        pr.key = stream_key(seed, static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k));
      }
      __syncthreads();
    }
  }
  if (live) {
    AMPPI_STAT(73, cs.amb ? 1 : 0);
    AMPPI_STAT(74, 1);
    out[k] = screen_store(stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd), cs.amb);
  }
}

// Latency path (few rollouts), one warp per rollout: the draws, clamps and
// control costs of all steps in parallel (lane = step), the RK4 recursion by
// the whole warp (quaternion chain in every lane, one stage acceleration per
// lane), then per-state cost terms and collision terms in parallel (lane =
// step; no abort here), summed in step order by lane 0.
__device__ __forceinline__ St<float> rk4_normalized_warp32(const St<float>& x, float thrust, V3<float> om,
                                                           const Dyn<float>& d) {
  const int lane = threadIdx.x & 31;
  const Q4<float> w0{0.f, om.x, om.y, om.z};
  auto dq_of = [&](Q4<float> q) {
    const Q4<float> qd = qmul(q, w0);
    return Q4<float>{0.5f * qd.w, 0.5f * qd.x, 0.5f * qd.y, 0.5f * qd.z};
  };
  auto adv = [](Q4<float> q, Q4<float> dq, float h) {
    return Q4<float>{q.w + h * dq.w, q.x + h * dq.x, q.y + h * dq.y, q.z + h * dq.z};
  };
  const Q4<float> dq1 = dq_of(x.q);
  const Q4<float> q2 = adv(x.q, dq1, d.half_dt);
  const Q4<float> dq2 = dq_of(q2);
  const Q4<float> q3 = adv(x.q, dq2, d.half_dt);
  const Q4<float> dq3 = dq_of(q3);
  const Q4<float> q4 = adv(x.q, dq3, d.dt);
  const Q4<float> dq4 = dq_of(q4);
  const Q4<float> qs = lane == 0 ? x.q : (lane == 1 ? q2 : (lane == 2 ? q3 : q4));
  const V3<float> dir = qrot_ez_fast(qnormalized(qs));
  const float a = thrust * d.inv_mass;
  const V3<float> dvl{a * dir.x + d.gx, a * dir.y + d.gy, a * dir.z + d.gz};
  V3<float> dv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    dv[i] = {__shfl_sync(0xffffffffu, dvl.x, i), __shfl_sync(0xffffffffu, dvl.y, i),
             __shfl_sync(0xffffffffu, dvl.z, i)};
  const V3<float> v2 = x.v + d.half_dt * dv[0];
  const V3<float> v3 = x.v + d.half_dt * dv[1];
  const V3<float> v4 = x.v + d.dt * dv[2];
  const float h6 = d.dt6;
  St<float> n;
  n.p = {x.p.x + h6 * rk_comb(x.v.x, v2.x, v3.x, v4.x), x.p.y + h6 * rk_comb(x.v.y, v2.y, v3.y, v4.y),
         x.p.z + h6 * rk_comb(x.v.z, v2.z, v3.z, v4.z)};
  n.v = {x.v.x + h6 * rk_comb(dv[0].x, dv[1].x, dv[2].x, dv[3].x),
         x.v.y + h6 * rk_comb(dv[0].y, dv[1].y, dv[2].y, dv[3].y),
         x.v.z + h6 * rk_comb(dv[0].z, dv[1].z, dv[2].z, dv[3].z)};
  n.q = {x.q.w + h6 * rk_comb(dq1.w, dq2.w, dq3.w, dq4.w), x.q.x + h6 * rk_comb(dq1.x, dq2.x, dq3.x, dq4.x),
         x.q.y + h6 * rk_comb(dq1.y, dq2.y, dq3.y, dq4.y), x.q.z + h6 * rk_comb(dq1.z, dq2.z, dq3.z, dq4.z)};
  n.q = qnormalized(n.q);
  return n;
}

constexpr int kWarpsPerCta32 = 4;

__global__ void __launch_bounds__(32 * kWarpsPerCta32) k_stage1_warp32(BatchIn in, Perception P, Plan pl,
                                                                       DevConfig cfg, int iter) {
  __shared__ float s_u[kWarpsPerCta32][4 * kMaxN];
  __shared__ float s_x[kWarpsPerCta32][10 * (kMaxN + 1)];
  __shared__ float s_t[kWarpsPerCta32][8 * kMaxN];  // trk vn g1 g2 g3 mag rate col
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta32 + wid;  // rollout (smi*K + k)
  const int kr = cfg.k_hi - cfg.k_lo;
  if (r >= static_cast<int64_t>(in.S) * cfg.M * kr) return;
  const int64_t smi = r / kr;
  const int k = cfg.k_lo + static_cast<int>(r % kr);
  const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
  float* out = pl.cost32 + smi * cfg.K + k;
  if (!pl.alive[smi]) {
    if (lane == 0) *out = __int_as_float(0x7f800000);
    return;
  }
  const int N = cfg.N;
  const Dyn<float> dy = make_dyn<float>(cfg);
  float* su = s_u[wid];
  float* sx = s_x[wid];
  float* st = s_t[wid];
  const double* unom = pl.nominal + smi * N * 4;
  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                    static_cast<float>(cfg.sigma[0]), static_cast<float>(cfg.sigma[1]),
                    static_cast<float>(cfg.sigma[2]), static_cast<float>(cfg.sigma[3])};
  const double* inj =
      in.injected ? in.injected + ((((static_cast<int64_t>(s) * cfg.iterations + iter) * cfg.M + m) * cfg.K + k) * N * 4)
                  : nullptr;
  for (int j = lane; j < N; j += 32) {
    float d[4];
    if (inj) {
      PertInjected<float>{inj}(j, d);
    } else {
      pr(j, d);
    }
    su[4 * j] = clampv(static_cast<float>(unom[4 * j]) + d[0], dy.tmin, dy.tmax);
    su[4 * j + 1] = clampv(static_cast<float>(unom[4 * j + 1]) + d[1], -dy.wxy, dy.wxy);
    su[4 * j + 2] = clampv(static_cast<float>(unom[4 * j + 2]) + d[2], -dy.wxy, dy.wxy);
    su[4 * j + 3] = clampv(static_cast<float>(unom[4 * j + 3]) + d[3], -dy.wz, dy.wz);
  }
  __syncwarp();
  for (int j = lane; j < N; j += 32) {
    const float u0 = su[4 * j], u1 = su[4 * j + 1], u2 = su[4 * j + 2], u3 = su[4 * j + 3];
    st[5 * N + j] = (((u0 * u0 + u1 * u1) + u2 * u2) + u3 * u3);
    if (j >= 1) {
      const float e0 = u0 - su[4 * j - 4], e1 = u1 - su[4 * j - 3], e2 = u2 - su[4 * j - 2], e3 = u3 - su[4 * j - 1];
      st[6 * N + j] = (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3);
    }
  }
  const double* xs = in.states + 10 * s;
  St<float> x;
  x.p = to_local_f(P.grid[s], xs);
  x.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};
  int n_ok = N;
  __syncwarp();
  for (int j = 0; j < N; ++j) {
    if (lane == 0) {
      float* o = sx + 10 * j;
      o[0] = x.p.x; o[1] = x.p.y; o[2] = x.p.z;
      o[3] = x.q.w; o[4] = x.q.x; o[5] = x.q.y; o[6] = x.q.z;
      o[7] = x.v.x; o[8] = x.v.y; o[9] = x.v.z;
    }
    const St<float> nx = rk4_normalized_warp32(x, su[4 * j], V3<float>{su[4 * j + 1], su[4 * j + 2], su[4 * j + 3]}, dy);
    if (!state_finite(nx)) {
      n_ok = j + 1;
      break;
    }
    x = nx;
  }
  __syncwarp();
  // per-state terms + collision, lane = step
  const double* gl = in.goals + 10 * s;
  const V3<float> pg = to_local_f(P.grid[s], gl);
  const V3<float> vg{static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  const Q4<float> qg{static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]),
                     static_cast<float>(gl[9])};
  const GridMeta g = P.grid[s];
  const uint4* grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  const uint32_t* gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  const uint4* gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  const float4* gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  const float cs = static_cast<float>(cfg.col_scale), ca = static_cast<float>(cfg.col_slope);
  const float dmin = static_cast<float>(cfg.col_d_min), dmax = static_cast<float>(cfg.col_d_max);
  const float4* guide = pl.guide32 + smi * N;
  bool amb = false;
  for (int j = lane; j < n_ok; j += 32) {
    const float* o = sx + 10 * j;
    const V3<float> p{o[0], o[1], o[2]}, v{o[7], o[8], o[9]};
    const Q4<float> q{o[3], o[4], o[5], o[6]};
    const float4 gd = guide[j];
    st[j] = norm3(p - V3<float>{gd.x, gd.y, gd.z});
    st[N + j] = sqnorm(v);
    st[2 * N + j] = static_cast<float>(cfg.q_p) * norm3(p - pg);
    st[3 * N + j] = static_cast<float>(cfg.q_v) * norm3(v - vg);
    st[4 * N + j] = static_cast<float>(cfg.q_q) * attitude_err_fast(q, qg);
    uint32_t hint = kNoHint;
    const float d2 = nearest_sq_fast(g, grec, gnbr, gleaf, gpts, p, screen_reach2(dmax), dmin * dmin, &hint);
    st[7 * N + j] = screen_collision(d2, cs, ca, dmin, dmax, amb);
  }
  amb = __any_sync(0xffffffffu, amb);
  __syncwarp();
  if (lane == 0) {
    float trk = 0.f, vn = 0.f, goal = 0.f, mag = 0.f, rate = 0.f, col = 0.f;
    for (int j = 0; j < n_ok; ++j) {
      trk = trk + st[j];
      vn = vn + st[N + j];
      goal = goal + st[2 * N + j];
      goal = goal + st[3 * N + j];
      goal = goal + st[4 * N + j];
      col = col + st[7 * N + j];
      if (j + 1 < N) {
        mag = mag + st[5 * N + j];
        if (j >= 1) rate = rate + st[6 * N + j];
      }
    }
    const float wt = static_cast<float>(cfg.q_track), wv = static_cast<float>(cfg.q_vnorm);
    const float wc = static_cast<float>(cfg.q_c), wd = static_cast<float>(cfg.q_c_delta);
    *out = n_ok == N ? screen_store(((wt * trk + wv * vn) + (wc * mag + wd * rate)) + (goal + col), amb)
                     : __int_as_float(0x7f800000);
  }
}

// ---------------------------------------------------------------------------
// Screening-drift diagnostic, FP32 half (amppi_screen_drift; DESIGN.md §2
// "The d_max jump"): sampled rollouts of scenes [s0, s0 + S) integrated as
// the screening integrates them (FP32 draws, clamp, RK4; rollout_costs<float>
// has the screening's sums and order for every sample it does not abort),
// with no abort bound.  Per step it stores the FP32 position and the exact
// FP32 squared clearance (reach: the grid cell h, no early stop); per rollout the
// screening cost (sign bit = flagged, +inf = invalid).  k_drift64 (k_plan64.cu)
// integrates the same rollouts in FP64 and compares.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_drift32(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                 const ScreenConsts sc, int iter, int s0, int S, int kstride,
                                                 float4* steps, float* cost) {
  const int kn = (cfg.k_hi - cfg.k_lo + kstride - 1) / kstride;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= static_cast<int64_t>(S) * cfg.M * kn) return;
  const int kk = static_cast<int>(r % kn);
  const int m = static_cast<int>((r / kn) % cfg.M);
  const int s = s0 + static_cast<int>(r / (static_cast<int64_t>(kn) * cfg.M));
  const int k = cfg.k_lo + kk * kstride;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  float4* st = steps + r * N;
  if (!pl.alive[smi]) {
    cost[r] = __int_as_float(0x7fc00000);  // NaN: instance not planned
    return;
  }
  float unom[4 * kMaxN];
  for (int i = 0; i < 4 * N; ++i) unom[i] = static_cast<float>(pl.nominal[smi * N * 4 + i]);  // as k_unom32
  RolloutEnv<float> env;
  env.unom = unom;
  env.guide = pl.guide32 + smi * N;
  env.N = N;
  env.dyn = sc.dyn;
  const double* gl = in.goals + 10 * s;
  env.pg = to_local_f(P.grid[s], gl);
  env.vg = {static_cast<float>(gl[3]), static_cast<float>(gl[4]), static_cast<float>(gl[5])};
  env.qg = {static_cast<float>(gl[6]), static_cast<float>(gl[7]), static_cast<float>(gl[8]), static_cast<float>(gl[9])};
  env.q_p = sc.q_p;
  env.q_v = sc.q_v;
  env.q_q = sc.q_q;
  env.cs = sc.cs;
  env.ca = sc.ca;
  env.cdmin = sc.cdmin;
  env.cdmax = sc.cdmax;
  env.grid = P.grid[s];
  env.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  env.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  env.gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  env.gpts = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  env.has_guide = true;
  env.abort_above = __int_as_float(0x7f800000);
  env.wq_track = sc.wq_track;
  env.wq_vnorm = sc.wq_vnorm;
  env.wq_c = sc.wq_c;
  env.wq_cd = sc.wq_cd;
  env.reach2 = sc.reach2;
  env.band = sc.band;
  const double* xs = in.states + 10 * s;
  St<float> x0;
  x0.p = to_local_f(P.grid[s], xs);
  x0.q = {static_cast<float>(xs[3]), static_cast<float>(xs[4]), static_cast<float>(xs[5]), static_cast<float>(xs[6])};
  x0.v = {static_cast<float>(xs[7]), static_cast<float>(xs[8]), static_cast<float>(xs[9])};
  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  const PertRngF pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                    sc.sigma[0], sc.sigma[1], sc.sigma[2], sc.sigma[3]};
  const CostSums<float> cs = rollout_costs(x0, env, pr);
  cost[r] = cs.valid ? screen_store(stage1_total(cs, env.wq_track, env.wq_vnorm, env.wq_c, env.wq_cd), cs.amb)
                     : __int_as_float(0x7f800000);
  float pos[4 * kMaxN];
  for (int j = 0; j < N; ++j) pos[4 * j] = pos[4 * j + 1] = pos[4 * j + 2] = __int_as_float(0x7fc00000);
  rollout_costs<float, PertRngF, true>(x0, env, pr, nullptr, nullptr, pos);
  const float lim = env.grid.h_f;  // exact below the cell size (k_drift64)
  uint32_t hint = kNoHint;
  for (int j = 0; j < N; ++j) {
    const V3<float> p{pos[4 * j], pos[4 * j + 1], pos[4 * j + 2]};
    const float d2 = isfinite(p.x) ? nearest_sq_fast(env.grid, env.grec, env.gnbr, env.gleaf, env.gpts, p, lim * lim,
                                                     0.f, &hint)
                                   : __int_as_float(0x7fc00000);
    st[j] = make_float4(p.x, p.y, p.z, d2);
  }
}

}  // namespace

cudaError_t launch_drift32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                           int s0, int S, int kstride, float4* steps, float* cost, cudaStream_t st) {
  const int kn = (cfg.k_hi - cfg.k_lo + kstride - 1) / kstride;
  const int64_t rows = static_cast<int64_t>(S) * cfg.M * kn;
  k_drift32<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, st>>>(in, P, pl, cfg, screen_consts(cfg), iter, s0, S,
                                                                      kstride, steps, cost);
  return cudaGetLastError();
}

cudaError_t launch_stage1_f32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                              cudaStream_t st, KernelTimer* timer) {
  const int kr = cfg.k_hi - cfg.k_lo;  // samples per instance screened here
  const int64_t total = static_cast<int64_t>(in.S) * cfg.M * kr;
  const int64_t SM = static_cast<int64_t>(in.S) * cfg.M;
  // throughput mode: 64 registers (8 CTAs = 32 warps per SM, a few bytes of
  // L1-resident spill); latency mode: no cap (fastest single rollout)
  auto kern = k_stage1_f32<8>;
  const ScreenConsts sc = screen_consts(cfg);
  auto unom32 = [&] {  // float nominal table for the bulk smem copies of k_stage1_f32 / k_stage1_f32c
    const int64_t n = SM * cfg.N;
    k_unom32<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pl, n);
  };
  if (total < 148 * 128 * 4 || kr <= 64) {
    // latency mode (few rollouts): one pass, warps spread over the SMs
    const int threads = total < 148 * 128 ? 32 : 128;
    const int tiles = (kr + threads - 1) / threads;
    if (total < kLatencyRollouts) {
      TimedRegion t(timer, "k_stage1_warp32", st);
      k_stage1_warp32<<<static_cast<unsigned>((total + kWarpsPerCta32 - 1) / kWarpsPerCta32), 32 * kWarpsPerCta32, 0,
                        st>>>(in, P, pl, cfg, iter);
      return cudaGetLastError();
    }
    unom32();
    TimedRegion t(timer, "k_stage1_f32", st);
    kern<<<static_cast<unsigned>(SM * tiles), threads, 0, st>>>(in, P, pl, cfg, sc, iter, 0, 0);
    return cudaGetLastError();
  }
  unom32();
  // bound samples per instance: AMPPI_BOUND_SAMPLES of every instance, 32 / that
  // instances per warp (injected perturbations: 32, one instance per warp)
  // Large ensembles (K >= 2048 samples on this context) take an eighth of
  // their samples, up to AMPPI_BOUND_LARGE, as bound samples: with 8192
  // samples per instance a 32-sample minimum is a weak bound, and the bound
  // pass is a small share of the screening (C4 64 x 8192 x 50: 32 bound
  // samples 1.95 ms per cycle, 256: 1.84, 1024: 1.80; gpurun_out/r49, r50)
  const int k1 = in.injected ? 32
                             : (kr >= 2048 && kBoundSamples == 32 ? std::min(kBoundLarge, (kr / 8) & ~31)
                                                                   : kBoundSamples);
  {
    TimedRegion t(timer, "k_stage1_f32_bound", st);
    if (in.injected || kBoundSamples == 32) {
      kern<<<static_cast<unsigned>(SM * (k1 / 32)), 32, 0, st>>>(in, P, pl, cfg, sc, iter, 1, k1);
    } else {
      constexpr int G = 32 / kBoundSamples;
      k_stage1_bound<G><<<static_cast<unsigned>((SM + G - 1) / G), 32, 0, st>>>(in, P, pl, cfg, sc, iter);
    }
  }
  TimedRegion t(timer, "k_stage1_f32", st);
  if (in.injected) {
    const int tiles = (kr - k1 + kScreenThreads - 1) / kScreenThreads;
    kern<<<static_cast<unsigned>(SM * tiles), kScreenThreads, 0, st>>>(in, P, pl, cfg, sc, iter, 2, k1);
  } else {
    // Lane compaction every 10 steps at 56 registers.  The larger the CTA,
    // the better live samples pack: 224 threads (5 CTAs per SM; the whole
    // K = 256 main pass of an instance in one CTA) beat 128 (9 per SM) by 4%,
    // 64 threads lose 15% (C5, measured); 128 when that covers the samples.
    if (kMainGroups > 1 && kr - k1 > 128) {
      // (experiment builds) the main pass in kMainGroups sequential launches
      // of 128-sample CTAs; each group aborts against the minimum of every
      // sample screened before it, a tighter bound than the 32 bound samples
      const int per = (kr - k1 + kMainGroups - 1) / kMainGroups;
      for (int g0 = k1; g0 < kr; g0 += per) {
        const int g1 = min(kr, g0 + per);
        const int tiles = (g1 - g0 + kScreenThreads - 1) / kScreenThreads;
        k_stage1_f32c<9, kMainCompact, kScreenThreads>
            <<<static_cast<unsigned>(SM * tiles), kScreenThreads, 0, st>>>(in, P, pl, cfg, sc, iter, g0, g1, g0);
      }
    } else if (kBoundSamples < 32 && kr - k1 > kMainThreads && kr - k1 <= 256) {  // (experiment builds) one 256-thread CTA
      k_stage1_f32c<4, kMainCompact, 256><<<static_cast<unsigned>(SM), 256, 0, st>>>(in, P, pl, cfg, sc, iter, k1,
                                                                                    kr, k1);
    } else if (kr - k1 > 128) {
      const int tiles = (kr - k1 + kMainThreads - 1) / kMainThreads;
      k_stage1_f32c<kMainMinBlocks, kMainCompact, kMainThreads>
          <<<static_cast<unsigned>(SM * tiles), kMainThreads, 0, st>>>(in, P, pl, cfg, sc, iter, k1, kr, k1);
    } else {
      const int tiles = (kr - k1 + kScreenThreads - 1) / kScreenThreads;
      k_stage1_f32c<9, kMainCompact, kScreenThreads>
          <<<static_cast<unsigned>(SM * tiles), kScreenThreads, 0, st>>>(in, P, pl, cfg, sc, iter, k1, kr, k1);
    }
  }
  return cudaGetLastError();
}

#ifdef AMPPI_STATS
extern "C" int amppi_query_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_query_stats, sizeof(unsigned long long) * kStatSlots);
  if (reset) {
    unsigned long long z[kStatSlots] = {};
    cudaMemcpyToSymbol(g_query_stats, z, sizeof(z));
  }
  return 0;
}
#endif

}  // namespace amppi_dev
