// Plan kernels in FP64 (built with -fmad=false): anchors + guides, the FP64
// stage-I rollouts (precision 64), the per-instance MPPI update with exact
// softmin support, stage II and the per-scene winner selection.  Replaces
// plan_step (proj/src/ensemble.cpp:29-169) end to end together with the FP32
// screening kernel in k_plan32.cu.
//
//   K4  k_anchors       one thread per (scene, anchor): near-goal logic
//                       (ensemble.cpp:42-66), sample_initial_endpoints /
//                       refine_endpoints (guidance.cpp:16-72) with
//                       correctly-rounded atan2/sin/cos, quintic guide
//                       (guidance.cpp:74-140), guide table g(t*dt), warm
//                       start (ensemble.cpp:68-77)
//   K3d k_stage1_f64    one thread per (scene, anchor, sample), FP64 stage I
//   K4b k_update        one CTA per (scene, anchor): min / softmin support,
//                       FP64 re-evaluation of the support (after FP32
//                       screening), weights, weighted perturbation sum and
//                       clamp (mppi.cpp:70-101), stage-II re-rollout
//                       (ensemble.cpp:132-149); the last CTA of a scene picks
//                       the winner (ensemble.cpp:151-168)
#include <cuda_runtime.h>

#include <algorithm>

#include "cr_math.cuh"
#include "kernels.h"
#include "rollout.cuh"

#ifndef AMPPI_COL_MINB
#define AMPPI_COL_MINB 8  // FP64 collision-term kernels at 64 registers (8 CTAs per SM): measured best of 1-16
#endif

namespace amppi_dev {

namespace {

constexpr double kPiD = 0x1.921fb54442d18p+1;
constexpr double kHalfPi = 0x1.921fb54442d18p+0;
constexpr double kAzStep = 0x1.acee9f37bebd5p-5;
constexpr double kMaxElevation = 0x1.8da7e39bae2a4p+0;  // 89*pi/180

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

__device__ __forceinline__ St<double> load_state(const double* s) {
  St<double> x;
  x.p = {s[0], s[1], s[2]};
  x.q = {s[3], s[4], s[5], s[6]};
  x.v = {s[7], s[8], s[9]};
  return x;
}

// cell of an exactly computed angle (atan2 already correctly rounded)
__device__ __forceinline__ int az_cell_exact(double az) {
  int i = static_cast<int>(floor((az + kPiD) / kAzStep));
  if (i >= kAz) i -= kAz;
  return i < 0 ? 0 : (i > kAz - 1 ? kAz - 1 : i);
}
__device__ __forceinline__ int el_cell_exact(double el) {
  const int j = static_cast<int>(floor((el + kHalfPi) / kAzStep));
  return j < 0 ? 0 : (j > kEl - 1 ? kEl - 1 : j);
}

__device__ __forceinline__ V3<double> direction_from_angles(double az, double el, bool cr) {
  if (cr) {
    double se, ce, sa, ca;
    crm::sincos_cr(el, se, ce);
    crm::sincos_cr(az, sa, ca);
    return {ce * ca, ce * sa, se};
  }
  const double ce = cos(el);
  return {ce * cos(az), ce * sin(az), sin(el)};
}

__device__ __forceinline__ bool near_integer(double v) {
  const double fl = floor(v);
  return (v - fl) < 1e-9 || ((fl + 1.0) - v) < 1e-9;
}

// ---------------------------------------------------------------------------
// K4: anchors, guides, warm start
// ---------------------------------------------------------------------------
// kL lanes per (scene, instance): lane 0 places the anchor and solves the
// quintic; the guide table and the warm start are filled lane-parallel.
// kL = 32 (one warp) for few instances (latency), 1 for many (throughput).
template <int kL>
__global__ void __launch_bounds__(64) k_anchors(BatchIn in, Perception P, Plan pl, DevConfig cfg) {
  __shared__ double s_c[64 / kL][18];
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / kL;
  const int lane = static_cast<int>(threadIdx.x % kL), wid = static_cast<int>(threadIdx.x / kL);
  const int M = cfg.M, N = cfg.N;
  if (gid >= in.S * M) return;
  const int s = gid / M, m = gid % M;
  const int64_t sm = static_cast<int64_t>(s) * M + m;
  const double T = static_cast<double>(N) * cfg.mppi_dt;
  // Every lane of an instance's warp computes the inputs (identical values);
  // the correctly rounded pass, when needed, splits its independent atan2 /
  // sincos pairs over lanes 0 and 1 (the C1 anchors straight at the goal sit
  // on cell boundaries, so this pass is on the latency path).
  const St<double> x = load_state(in.states + 10 * s);
  const double* gl = in.goals + 10 * s;
  const V3<double> goal_p{gl[0], gl[1], gl[2]};
  const double* ps = in.poses + 10 * s;
  const V3<double> pose_p{ps[0], ps[1], ps[2]};
  const M3 body_to_world = rotmat(Q4<double>{ps[3], ps[4], ps[5], ps[6]});
  const double horizon_s = static_cast<double>(N) * cfg.mppi_dt;

  V3<double> initial, refined, safe_dir;
  double safe_range, terminal_speed = 0.0, lookahead = 0.0;
  int ci = 0, cj = 0;
  const double goal_dist = norm3(goal_p - x.p);
  const bool far_goal = goal_dist > cfg.min_anchor_distance;
  if (far_goal) {
    lookahead = dmin(cfg.lookahead, goal_dist);
    terminal_speed = dmin(cfg.terminal_speed, goal_dist / horizon_s);
    // sample_initial_endpoints (index m = v*m_h + h) + refine_endpoints.
    // Pass 0 uses CUDA's libm (<= 2 ulp); if either refined-direction
    // quotient lands within 1e-9 of a cell boundary the anchor is recomputed
    // with correctly-rounded atan2/sin/cos (pass 1) so its cell equals the
    // glibc-based reference's.
    const int v = m / cfg.m_h, h = m % cfg.m_h;
    const V3<double> tg = goal_p - x.p;
    const double spacing = cfg.spacing_deg * kPiD / 180.0;
    // a pair of independent correctly rounded evaluations: lanes 0 and 1 in
    // parallel for a warp per instance, in turn for a thread per instance
    auto cr_pair = [&](auto f0, auto f1, double& r0, double& r1) {
      if constexpr (kL > 1) {
        const double mine = lane == 1 ? f1() : (lane == 0 ? f0() : 0.0);
        r0 = __shfl_sync(0xffffffffu, mine, 0);
        r1 = __shfl_sync(0xffffffffu, mine, 1);
      } else {
        r0 = f0();
        r1 = f1();
      }
    };
    for (int pass = 0; pass < 2; ++pass) {
      const bool cr = pass == 1;
      double az0, el0;
      if (!cr) {
        az0 = atan2(tg.y, tg.x);
        el0 = atan2(tg.z, sqrt(tg.x * tg.x + tg.y * tg.y));
      } else {
        cr_pair([&] { return crm::atan2_cr(tg.y, tg.x); },
                [&] { return crm::atan2_cr(tg.z, sqrt(tg.x * tg.x + tg.y * tg.y)); }, az0, el0);
      }
      const double el_off = (static_cast<double>(v) - 0.5 * static_cast<double>(cfg.m_v - 1)) * spacing;
      const double el = clampv(el0 + el_off, -kMaxElevation, kMaxElevation);
      const double az = az0 + (static_cast<double>(h) - 0.5 * static_cast<double>(cfg.m_h - 1)) * spacing;
      V3<double> dir_unit;
      if (!cr) {
        dir_unit = direction_from_angles(az, el, false);
      } else {  // direction_from_angles(az, el, true): sincos_cr(el) and sincos_cr(az) in parallel
        double se, ce, sa, ca;
        if constexpr (kL > 1) {
          double sn = 0.0, cs = 0.0;
          if (lane < 2) crm::sincos_cr(lane == 0 ? el : az, sn, cs);
          se = __shfl_sync(0xffffffffu, sn, 0);
          ce = __shfl_sync(0xffffffffu, cs, 0);
          sa = __shfl_sync(0xffffffffu, sn, 1);
          ca = __shfl_sync(0xffffffffu, cs, 1);
        } else {
          crm::sincos_cr(el, se, ce);
          crm::sincos_cr(az, sa, ca);
        }
        dir_unit = {ce * ca, ce * sa, se};
      }
      initial = x.p + lookahead * dir_unit;
      V3<double> dir_world = initial - pose_p;
      if (sqnorm(dir_world) < 1e-18) dir_world = {1.0, 0.0, 0.0};
      const double n2 = sqnorm(dir_world);
      if (n2 > 0.0) {
        const double n = sqrt(n2);
        dir_world = {dir_world.x / n, dir_world.y / n, dir_world.z / n};
      }
      const V3<double> db = mat_t_vec(body_to_world, dir_world);
      double azb, elb;
      if (!cr) {
        azb = atan2(db.y, db.x);
        elb = atan2(db.z, sqrt(db.x * db.x + db.y * db.y));
      } else {
        cr_pair([&] { return crm::atan2_cr(db.y, db.x); },
                [&] { return crm::atan2_cr(db.z, sqrt(db.x * db.x + db.y * db.y)); }, azb, elb);
      }
      const double qa = (azb + kPiD) / kAzStep, qe = (elb + kHalfPi) / kAzStep;
      if (!cr && (near_integer(qa) || near_integer(qe))) continue;
      ci = az_cell_exact(azb) / kPool;
      cj = el_cell_exact(elb) / kPool;
      break;
    }
  }
  if (lane == 0) {
  if (far_goal) {
    const int64_t f = static_cast<int64_t>(s) * kCoarse + ci * kCEl + cj;
    safe_range = P.safe_range[f];
    safe_dir = mat_vec(body_to_world, V3<double>{P.safe_dir[3 * f], P.safe_dir[3 * f + 1], P.safe_dir[3 * f + 2]});
    const double reach = dmin(lookahead, dmax(safe_range - cfg.col_d_max, cfg.min_anchor_distance));
    refined = pose_p + reach * safe_dir;
  } else {
    // inside the anchor floor every guide settles on the goal at rest
    initial = goal_p;
    refined = goal_p;
    safe_dir = qrot(x.q, V3<double>{1.0, 0.0, 0.0});
    safe_range = in.r_max;
    terminal_speed = 0.0;
  }
  double* ai = pl.anchor_init + 3 * sm;
  double* ar = pl.anchor_ref + 3 * sm;
  double* ad = pl.anchor_dir + 3 * sm;
  ai[0] = initial.x; ai[1] = initial.y; ai[2] = initial.z;
  ar[0] = refined.x; ar[1] = refined.y; ar[2] = refined.z;
  ad[0] = safe_dir.x; ad[1] = safe_dir.y; ad[2] = safe_dir.z;
  pl.anchor_range[sm] = safe_range;
  pl.anchor_ij[2 * sm] = ci;
  pl.anchor_ij[2 * sm + 1] = cj;

  // build_guides: start acceleration from the clamped last control
  const Dyn<double> dy = make_dyn<double>(cfg);
  const double* la = in.last_applied + 4 * s;
  const double lt = clampv(la[0], dy.tmin, dy.tmax);
  const V3<double> lw{clampv(la[1], -dy.wxy, dy.wxy), clampv(la[2], -dy.wxy, dy.wxy), clampv(la[3], -dy.wz, dy.wz)};
  const V3<double> a0 = derivative(x, lt, lw, dy).dv;
  const V3<double> end_v = terminal_speed * safe_dir;
  // solve_quintic (guidance.cpp:74-94)
  const double T2 = T * T, T3 = T2 * T, T4 = T3 * T, T5 = T4 * T;
  const V3<double> half_a = 0.5 * a0;
  const V3<double> dp = refined - ((x.p + T * x.v) + T2 * half_a);
  const V3<double> dv = end_v - (x.v + T * a0);
  const V3<double> da = V3<double>{0.0, 0.0, 0.0} - a0;
  V3<double> c[6];
  c[0] = x.p;
  c[1] = x.v;
  c[2] = half_a;
  const double e3 = 2.0 * T3, e4 = 2.0 * T4, e5 = 2.0 * T5;
  const double t8 = 8.0 * T, t14 = 14.0 * T, t6 = 6.0 * T, t2 = 2.0 * T2;
  {
    const V3<double> num = ((20.0 * dp - t8 * dv) + T2 * da);
    c[3] = {num.x / e3, num.y / e3, num.z / e3};
  }
  {
    const V3<double> num = ((-30.0 * dp + t14 * dv) - t2 * da);
    c[4] = {num.x / e4, num.y / e4, num.z / e4};
  }
  {
    const V3<double> num = ((12.0 * dp - t6 * dv) + T2 * da);
    c[5] = {num.x / e5, num.y / e5, num.z / e5};
  }
  double* gc = pl.guide_coef + 18 * sm;
  for (int k = 0; k < 6; ++k) {
    gc[k] = c[k].x;
    gc[6 + k] = c[k].y;
    gc[12 + k] = c[k].z;
    s_c[wid][3 * k] = c[k].x;
    s_c[wid][3 * k + 1] = c[k].y;
    s_c[wid][3 * k + 2] = c[k].z;
  }
  }  // lane 0
  if (kL > 1) __syncwarp();
  V3<double> c[6];
  for (int k = 0; k < 6; ++k) c[k] = {s_c[wid][3 * k], s_c[wid][3 * k + 1], s_c[wid][3 * k + 2]};
  // guide table g(t * dt) for t < N (tracking cost, costs.hpp:59-66)
  for (int t = lane; t < N; t += kL) {
    double tt = static_cast<double>(t) * cfg.dyn_dt;
    tt = clampv(tt, 0.0, T);
    V3<double> o = c[5];
    for (int k = 4; k >= 0; --k) o = V3<double>{o.x * tt, o.y * tt, o.z * tt} + c[k];
    const int64_t gi = sm * N + t;
    pl.guide64[3 * gi] = o.x;
    pl.guide64[3 * gi + 1] = o.y;
    pl.guide64[3 * gi + 2] = o.z;
    const V3<float> of = to_local_f(P.grid[s], &pl.guide64[3 * gi]);  // the screening's local frame
    pl.guide32[gi] = make_float4(of.x, of.y, of.z, 0.f);
  }
  // warm start: shifted previous winner, or hover (ensemble.cpp:68-77)
  const int plen = in.prev ? (in.prev_len ? in.prev_len[s] : N) : 0;
  double* nom = pl.nominal + sm * N * 4;
  if (plen == N) {
    const double* pv = in.prev + static_cast<int64_t>(s) * N * 4;
    for (int j = lane; j < N; j += kL) {
      const int src = j + 1 < N ? j + 1 : N - 1;
      for (int cc = 0; cc < 4; ++cc) nom[4 * j + cc] = pv[4 * src + cc];
    }
  } else {
    const double hover = cfg.mass * sqrt((cfg.gravity[0] * cfg.gravity[0] + cfg.gravity[1] * cfg.gravity[1]) +
                                         cfg.gravity[2] * cfg.gravity[2]);
    for (int j = lane; j < N; j += kL) {
      nom[4 * j] = hover;
      nom[4 * j + 1] = 0.0;
      nom[4 * j + 2] = 0.0;
      nom[4 * j + 3] = 0.0;
    }
  }
  if (lane == 0) {
    pl.alive[sm] = 1;
    pl.stage1[sm] = 0.0;
    pl.ess[sm] = 0.0;
  }
}

// Fill an FP64 rollout environment for (scene, instance); unom may point to
// shared or global memory.
__device__ __forceinline__ RolloutEnv<double> make_env64(const BatchIn& in, const Perception& P, const Plan& pl,
                                                        const DevConfig& cfg, int s, int m, const double* unom) {
  RolloutEnv<double> e;
  const int64_t sm = static_cast<int64_t>(s) * cfg.M + m;
  e.unom = unom;
  e.guide = pl.guide64 + sm * cfg.N * 3;
  e.N = cfg.N;
  e.dyn = make_dyn<double>(cfg);
  const double* gl = in.goals + 10 * s;
  e.pg = {gl[0], gl[1], gl[2]};
  e.vg = {gl[3], gl[4], gl[5]};
  const M3 g = rotmat(Q4<double>{gl[6], gl[7], gl[8], gl[9]});
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) e.gt.m[i][j] = g.m[j][i];
  e.q_p = cfg.q_p;
  e.q_v = cfg.q_v;
  e.q_q = cfg.q_q;
  e.cs = cfg.col_scale;
  e.ca = cfg.col_slope;
  e.cdmin = cfg.col_d_min;
  e.cdmax = cfg.col_d_max;
  e.grid = P.grid[s];
  e.grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;

  e.gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  e.gleaf = P.grid_leaf + static_cast<int64_t>(s) * kCells * 2;
  e.gpts = P.grid_pts64 + static_cast<int64_t>(s) * kCells * 3;
  e.gpts32 = P.grid_pts32 + static_cast<int64_t>(s) * kCells;
  e.has_guide = true;
  e.abort_above = __longlong_as_double(0x7ff0000000000000ll);
  return e;
}

__device__ __forceinline__ const double* injected_row(const BatchIn& in, const DevConfig& cfg, int s, int iter, int m,
                                                      int k) {
  const int64_t row = (((static_cast<int64_t>(s) * cfg.iterations + iter) * cfg.M + m) * cfg.K + k);
  return in.injected + row * cfg.N * 4;
}

// ---------------------------------------------------------------------------
// K3d: FP64 stage I (precision 64)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_stage1_f64(BatchIn in, Perception P, Plan pl, DevConfig cfg, int iter) {
  extern __shared__ double sm_unom[];
  const int tiles = (cfg.K + blockDim.x - 1) / blockDim.x;
  int b = blockIdx.x;
  const int tile = b % tiles;
  b /= tiles;
  const int m = b % cfg.M;
  const int s = b / cfg.M;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
  const int N = cfg.N;
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x) sm_unom[i] = pl.nominal[smi * N * 4 + i];
  __syncthreads();
  const int k = tile * blockDim.x + threadIdx.x;
  if (k >= cfg.K) return;
  double* out = pl.cost64 + smi * cfg.K + k;
  if (!pl.alive[smi]) {
    *out = __longlong_as_double(0x7ff0000000000000ll);
    return;
  }
  const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, sm_unom);
  const St<double> x0 = load_state(in.states + 10 * s);
  CostSums<double> cs;
  if (in.injected) {
    cs = rollout_costs(x0, env, PertInjected<double>{injected_row(in, cfg, s, iter, m, k)});
  } else {
    const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
    const PertRngD pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                      cfg.sigma[0], cfg.sigma[1], cfg.sigma[2], cfg.sigma[3]};
    cs = rollout_costs(x0, env, pr);
  }
  *out = cs.valid ? stage1_total(cs, cfg.q_track, cfg.q_vnorm, cfg.q_c, cfg.q_c_delta)
                  : __longlong_as_double(0x7ff0000000000000ll);
}

// ---------------------------------------------------------------------------
// K4b: MPPI update (compute_weights + update_nominal, mppi.cpp:70-101) as
//   k_support  one CTA per instance: screening minimum, softmin support
//              (samples whose weight can exceed e^-64 of the maximum) in k order
//   k_refine   one warp per instance: exact FP64 stage-I cost of the support
//              (FP32 screening only)
//   k_nominal  one CTA per instance: rho / weights / eta / ess in k order,
//              weighted perturbation sum, clamp
// K5: k_stage2 one thread per instance (noise-free re-rollout, stage-II cost,
//     breakdown); k_select one thread per scene (first minimum wins).
// ---------------------------------------------------------------------------
constexpr int kSupportThreads = 128;

#ifndef AMPPI_COL_PASSES
#define AMPPI_COL_PASSES 1
#endif
constexpr bool kColPasses = AMPPI_COL_PASSES != 0;  // classify / query / sum form of the FP64 collision terms

struct UpdateScratch {  // global, per (scene, instance): [K] each
  uint32_t* cand_k;
  double* cand_s;
  double* cand_w;
  uint2* pairs;                     // [S*M*K] (instance, support slot) work list for k_refine
  unsigned long long* pair_count;
};

__device__ __forceinline__ double load_cost(const Plan& pl, int precision, int64_t i) {
  return precision == 32 ? static_cast<double>(fabsf(pl.cost32[i])) : pl.cost64[i];
}
// FP32 screening cost flagged as a lower bound (d_max band, screen_collision)
__device__ __forceinline__ bool cost_flagged(const Plan& pl, int precision, int64_t i) {
  return precision == 32 && signbit(pl.cost32[i]);
}

// Softmin support of each instance over samples [k_lo, k_hi): every sample
// within the window of rho, the screening minimum -- computed here, or the
// global minimum over all sample shards when rho_ext is given.
__global__ void __launch_bounds__(kSupportThreads) k_support(Plan pl, DevConfig cfg, UpdateScratch us, int precision,
                                                            const float* rho_ext) {
  __shared__ double s_red[kSupportThreads / 32];
  __shared__ uint32_t s_cnt[kSupportThreads / 32];
  __shared__ double s_rho;
  const int64_t smi = blockIdx.x;
  const int K = cfg.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (!pl.alive[smi]) {
    if (tid == 0) pl.n_support[smi] = 0;
    return;
  }
  const int64_t base = smi * K;
  const int k_lo = cfg.k_lo, kr = cfg.k_hi - cfg.k_lo;
  if (rho_ext) {
    if (tid == 0) s_rho = static_cast<double>(rho_ext[smi]);
  } else {
    // rho over the unflagged costs; flagged ones only bound their sample from
    // below.  With finite costs that are all flagged, every one is admitted
    // (rho = -FLT_MAX, "admit all").
    double lmin = kInf;
    bool any_flagged = false;
    for (int k = k_lo + tid; k < cfg.k_hi; k += blockDim.x) {
      const double c = load_cost(pl, precision, base + k);
      if (!isfinite(c)) continue;
      if (cost_flagged(pl, precision, base + k)) any_flagged = true;
      else lmin = fmin(lmin, c);
    }
    for (int o = 16; o > 0; o >>= 1) lmin = fmin(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
    any_flagged = __any_sync(0xffffffffu, any_flagged);
    if (lane == 0) s_red[warp] = any_flagged && !isfinite(lmin) ? -1.0 : lmin;
    __syncthreads();
    if (tid == 0) {
      double r = kInf;
      bool flagged_only = false;
      for (int w = 0; w < kSupportThreads / 32; ++w) {
        if (s_red[w] == -1.0) flagged_only = true;
        else r = fmin(r, s_red[w]);
      }
      s_rho = (!isfinite(r) && flagged_only) ? -3.4028234663852886e38 : r;
    }
  }
  __syncthreads();
  const double rho_s = s_rho;
  if (!isfinite(rho_s)) {  // "no valid rollout": the instance dies
    if (tid == 0) {
      pl.alive[smi] = 0;
      pl.n_support[smi] = 0;
    }
    return;
  }
  const bool admit_all = rho_s <= -3.0e38;
  const double window = precision == 32 ? kWindowLambdas * cfg.lambda + 1e-4 * fabs(rho_s) + 1e-2 : 746.0 * cfg.lambda;
  const int per = (kr + blockDim.x - 1) / blockDim.x;
  const int k0 = k_lo + min(tid * per, kr), k1 = min(k0 + per, cfg.k_hi);
  uint32_t mine = 0;
  for (int k = k0; k < k1; ++k) {
    const double c = load_cost(pl, precision, base + k);
    mine += (isfinite(c) && (admit_all || c - rho_s <= window));
  }
  uint32_t x = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_cnt[warp] = x;
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (int w = 0; w < kSupportThreads / 32; ++w) {
      const uint32_t t = s_cnt[w];
      s_cnt[w] = run;
      run += t;
    }
    pl.n_support[smi] = run;
    if (precision == 32 && run > 0) {  // reserve this instance's refine work items
      const unsigned long long at = atomicAdd(us.pair_count, static_cast<unsigned long long>(run));
      for (uint32_t c = 0; c < run; ++c) us.pairs[at + c] = make_uint2(static_cast<uint32_t>(smi), c);
    }
  }
  __syncthreads();
  uint32_t pos = s_cnt[warp] + x - mine;
  for (int k = k0; k < k1; ++k) {
    const double c = load_cost(pl, precision, base + k);
    if (isfinite(c) && (admit_all || c - rho_s <= window)) {
      us.cand_k[base + pos] = static_cast<uint32_t>(k);
      us.cand_s[base + pos] = c;
      ++pos;
    }
  }
}

// One thread per (instance, support slot) over the flattened work list:
// full warps regardless of how the support sizes are distributed.
// Fused FP64 re-rollout of support pairs [first, pair_count) (the pairs the
// split traj/col kernels had no scratch for).
__global__ void __launch_bounds__(64) k_refine(BatchIn in, Perception P, Plan pl, DevConfig cfg, UpdateScratch us,
                                               int iter, unsigned long long first) {
  const unsigned long long n = *us.pair_count;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  for (unsigned long long w = first + static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < n;
       w += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const uint2 pr = us.pairs[w];
    const int64_t smi = pr.x;
    const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
    const int64_t slot = smi * cfg.K + pr.y;
    const int k = static_cast<int>(us.cand_k[slot]);
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    const St<double> x0 = load_state(in.states + 10 * s);
    CostSums<double> cs;
    if (in.injected) {
      cs = rollout_costs(x0, env, PertInjected<double>{injected_row(in, cfg, s, iter, m, k)});
    } else {
      const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
      const PertRngD prng{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                          cfg.sigma[0], cfg.sigma[1], cfg.sigma[2], cfg.sigma[3]};
      cs = rollout_costs(x0, env, prng);
    }
    us.cand_s[slot] = cs.valid ? stage1_total(cs, cfg.q_track, cfg.q_vnorm, cfg.q_c, cfg.q_c_delta) : kInf;
  }
}

__global__ void __launch_bounds__(128) k_nominal(BatchIn in, Plan pl, DevConfig cfg, UpdateScratch us, int iter) {
  __shared__ int s_dead;
  const int64_t smi = blockIdx.x;
  const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
  const uint32_t n = pl.n_support[smi];
  if (n == 0) return;  // dead (or died this iteration)
  const int N = cfg.N, tid = threadIdx.x;
  const int64_t base = smi * cfg.K;
  const uint32_t* cand_k = us.cand_k + base;
  const double* cand_s = us.cand_s + base;
  double* cand_w = us.cand_w + base;
  if (tid == 0) {
    // compute_weights (mppi.cpp:70-87): rho, e_k, eta, w_k = e_k / eta, ess
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double rho = kInf;
    for (uint32_t c = 0; c < n; ++c)
      if (isfinite(cand_s[c])) rho = dmin(rho, cand_s[c]);
    s_dead = !isfinite(rho);
    if (!s_dead) {
      double eta = 0.0;
      for (uint32_t c = 0; c < n; ++c) {
        const double e = isfinite(cand_s[c]) ? exp(-(cand_s[c] - rho) / cfg.lambda) : 0.0;
        cand_w[c] = e;
        eta += e;
      }
      double w2 = 0.0;
      for (uint32_t c = 0; c < n; ++c) {
        const double w = cand_w[c] / eta;
        cand_w[c] = w;
        w2 += w * w;
      }
      pl.stage1[smi] = rho;
      pl.ess[smi] = w2 > 0.0 ? 1.0 / w2 : 0.0;
    } else {
      pl.alive[smi] = 0;
    }
  }
  __syncthreads();
  if (s_dead) return;
  // update_nominal (mppi.cpp:89-101): deltas regenerated from the counter RNG
  // and clamped against u_j exactly as rollout_into rewrote them
  const Dyn<double> dy = make_dyn<double>(cfg);
  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  // One thread per Box-Muller pair (components jc = 2p, 2p+1 share one
  // normal_pair): the same per-component sums in support order, half the
  // FP64 draws.
  double* nom = pl.nominal + smi * N * 4;
  for (int pj = tid; pj < 2 * N; pj += blockDim.x) {
    const int jc0 = 2 * pj, c0 = jc0 & 3, c1 = c0 + 1;
    const double ua = nom[jc0], ub = nom[jc0 + 1];
    const double lo0 = c0 == 0 ? dy.tmin : -dy.wxy, hi0 = c0 == 0 ? dy.tmax : dy.wxy;
    const double lo1 = c1 == 3 ? -dy.wz : -dy.wxy, hi1 = c1 == 3 ? dy.wz : dy.wxy;
    double da = 0.0, db = 0.0;
    for (uint32_t ci = 0; ci < n; ++ci) {
      const double w = cand_w[ci];
      if (w == 0.0) continue;  // 0 * delta adds exactly nothing
      const int k = static_cast<int>(cand_k[ci]);
      double d0, d1;
      if (in.injected) {
        const double* row = injected_row(in, cfg, s, iter, m, k);
        d0 = row[jc0];
        d1 = row[jc0 + 1];
      } else {
        const uint64_t key = stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k));
        double n0, n1;
        normal_pair(key, static_cast<uint32_t>(pj), n0, n1);
        d0 = cfg.sigma[c0] * n0;
        d1 = cfg.sigma[c1] * n1;
      }
      da = da + w * (clampv(ua + d0, lo0, hi0) - ua);
      db = db + w * (clampv(ub + d1, lo1, hi1) - ub);
    }
    nom[jc0] = clampv(ua + da, lo0, hi0);
    nom[jc0 + 1] = clampv(ub + db, lo1, hi1);
  }
}

// ---------------------------------------------------------------------------
// Sample sharding (config C4).  A shard screens samples
// [k_lo, k_hi) of every instance (global k in the RNG key, so its draws are
// the single-GPU draws), the shards agree on the global screening minimum
// (all-reduce MIN of k_local_min), each refines its part of the softmin
// support and reduces it to per-instance partials, and after one all-gather
// every shard merges the partials in shard order (k_merge) -- the same
// nominal on every shard, so stage II and the winner are replicated.
// Partials per instance: {m_g, eta_g, w2_g, ed_g[4N]} with e_k =
// exp(-(S_k - m_g)/lambda), eta_g = sum e_k, w2_g = sum e_k^2, ed_g[jc] =
// sum e_k * applied_k[jc] (mppi.cpp:70-101 split by shard).
// ---------------------------------------------------------------------------
__global__ void k_local_min(Plan pl, DevConfig cfg, float* out) {
  // minimum over the unflagged screening costs; a shard whose finite costs
  // are all flagged reports -FLT_MAX, so the global minimum admits every
  // flagged sample (k_support "admit all")
  const int64_t smi = blockIdx.x;
  float v = __int_as_float(0x7f800000);
  bool flagged = false;
  if (pl.alive[smi])
    for (int k = cfg.k_lo + threadIdx.x; k < cfg.k_hi; k += blockDim.x) {
      const float c = pl.cost32[smi * cfg.K + k];
      if (!isfinite(c)) continue;
      if (signbit(c)) flagged = true;
      else v = fminf(v, c);
    }
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  flagged = __any_sync(0xffffffffu, flagged);
  if (threadIdx.x == 0) out[smi] = (flagged && !isfinite(v)) ? -3.4028234663852886e38f : v;
}

__global__ void __launch_bounds__(128) k_partials(BatchIn in, Plan pl, DevConfig cfg, UpdateScratch us, int iter,
                                                 double* out) {
  __shared__ double s_m;
  const int64_t smi = blockIdx.x;
  const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
  const int N = cfg.N, tid = threadIdx.x;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  double* o = out + smi * (3 + 4 * N);
  const uint32_t n = pl.alive[smi] ? pl.n_support[smi] : 0u;
  const int64_t base = smi * cfg.K;
  const uint32_t* cand_k = us.cand_k + base;
  const double* cand_s = us.cand_s + base;
  double* cand_w = us.cand_w + base;
  if (tid == 0) {
    double mg = kInf;
    for (uint32_t c = 0; c < n; ++c)
      if (isfinite(cand_s[c])) mg = dmin(mg, cand_s[c]);
    double eta = 0.0, w2 = 0.0;
    if (isfinite(mg))
      for (uint32_t c = 0; c < n; ++c) {
        const double e = isfinite(cand_s[c]) ? exp(-(cand_s[c] - mg) / cfg.lambda) : 0.0;
        cand_w[c] = e;
        eta += e;
        w2 += e * e;
      }
    o[0] = mg;
    o[1] = eta;
    o[2] = w2;
    s_m = mg;
  }
  __syncthreads();
  const bool live = isfinite(s_m);
  const Dyn<double> dy = make_dyn<double>(cfg);
  const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
  const double* nom = pl.nominal + smi * N * 4;
  for (int jc = tid; jc < 4 * N; jc += blockDim.x) {
    double ed = 0.0;
    if (live) {
      const int c = jc & 3;
      const double u = nom[jc];
      const double lo = c == 0 ? dy.tmin : (c == 3 ? -dy.wz : -dy.wxy);
      const double hi = c == 0 ? dy.tmax : (c == 3 ? dy.wz : dy.wxy);
      for (uint32_t ci = 0; ci < n; ++ci) {
        const double e = cand_w[ci];
        if (e == 0.0) continue;
        const int k = static_cast<int>(cand_k[ci]);
        double draw;
        if (in.injected) {
          draw = injected_row(in, cfg, s, iter, m, k)[jc];
        } else {
          const uint64_t key = stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k));
          double n0, n1;
          normal_pair(key, static_cast<uint32_t>(jc >> 1), n0, n1);
          draw = cfg.sigma[c] * ((jc & 1) ? n1 : n0);
        }
        ed = ed + e * (clampv(u + draw, lo, hi) - u);
      }
    }
    o[3 + jc] = ed;
  }
}

constexpr int kMaxShards = 64;

__global__ void __launch_bounds__(128) k_merge(Plan pl, DevConfig cfg, const double* parts, int n_shards) {
  __shared__ double s_a[kMaxShards];
  __shared__ double s_eta;
  __shared__ int s_dead;
  const int64_t smi = blockIdx.x;
  const int N = cfg.N, tid = threadIdx.x, stride = 3 + 4 * N;
  const int64_t inst = static_cast<int64_t>(gridDim.x);  // S*M
  if (tid == 0) {
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double rho = kInf;
    for (int g = 0; g < n_shards; ++g) rho = dmin(rho, parts[(g * inst + smi) * stride]);
    s_dead = !isfinite(rho);
    if (s_dead) {
      pl.alive[smi] = 0;  // "no valid rollout" on every shard (ensemble.cpp:126)
      pl.n_support[smi] = 0;
    } else {
      double eta = 0.0, w2 = 0.0;
      for (int g = 0; g < n_shards; ++g) {
        const double* p = parts + (g * inst + smi) * stride;
        const double a = isfinite(p[0]) ? exp(-(p[0] - rho) / cfg.lambda) : 0.0;
        s_a[g] = a;
        eta += a * p[1];
        w2 += (a * a) * p[2];
      }
      s_eta = eta;
      pl.stage1[smi] = rho;
      pl.ess[smi] = w2 > 0.0 ? (eta * eta) / w2 : 0.0;
    }
  }
  __syncthreads();
  if (s_dead) return;
  const Dyn<double> dy = make_dyn<double>(cfg);
  double* nom = pl.nominal + smi * N * 4;
  for (int jc = tid; jc < 4 * N; jc += blockDim.x) {
    const int c = jc & 3;
    const double lo = c == 0 ? dy.tmin : (c == 3 ? -dy.wz : -dy.wxy);
    const double hi = c == 0 ? dy.tmax : (c == 3 ? dy.wz : dy.wxy);
    double acc = 0.0;
    for (int g = 0; g < n_shards; ++g)
      if (s_a[g] != 0.0) acc = acc + s_a[g] * parts[(g * inst + smi) * stride + 3 + jc];
    nom[jc] = clampv(nom[jc] + acc / s_eta, lo, hi);
  }
}

// Stage II (ensemble.cpp:132-149) in two passes: a sequential FP64 trajectory
// per instance with the collision queries deferred, then one warp per
// instance evaluating the N collision terms in parallel and summing them in
// step order (costs.hpp:121-127).
// Warp-cooperative deferred-collision FP64 rollout (latency-critical paths:
// support refine and stage II).  Only the RK4 recursion is sequential (lane
// 0); the perturbation draws, clamps and control costs are computed for all
// steps in parallel before it, and the per-state cost terms in parallel after
// it, then lane 0 adds every term in rollout_costs' order -- the same FP64
// values and sums as rollout_costs<double, Pert, true>.  sm: per-warp scratch
// of kWarpRolloutDoubles(N) doubles.
constexpr int kRolloutMaxN = 64;
constexpr int kRolloutDone = 1 << 20;  // ready-word marker: trajectory finished (+ number of finite states)
__host__ __device__ constexpr int warp_rollout_doubles(int N) { return 4 * N + 10 * (N + 1) + 7 * N; }

// rk4_normalized<double> evaluated by a whole warp: every lane runs the
// quaternion chain (it does not depend on the thrust direction), lanes 0..3
// then normalise and rotate one RK stage each in parallel, and the
// velocity / position combination uses the gathered stage accelerations.
// Same IEEE operations as rk4_normalized, so the same bits; the latency per
// step is the quaternion chain plus one stage instead of four.
__device__ __forceinline__ St<double> rk4_normalized_warp(const St<double>& x, double thrust, V3<double> om,
                                                          const Dyn<double>& d) {
  const int lane = threadIdx.x & 31;
  const Q4<double> w0{0.0, om.x, om.y, om.z};
  auto dq_of = [&](Q4<double> q) {
    const Q4<double> qd = qmul(q, w0);
    return Q4<double>{0.5 * qd.w, 0.5 * qd.x, 0.5 * qd.y, 0.5 * qd.z};
  };
  auto adv = [](Q4<double> q, Q4<double> dq, double h) {
    return Q4<double>{q.w + h * dq.w, q.x + h * dq.x, q.y + h * dq.y, q.z + h * dq.z};
  };
  const Q4<double> dq1 = dq_of(x.q);
  const Q4<double> q2 = adv(x.q, dq1, d.half_dt);
  const Q4<double> dq2 = dq_of(q2);
  const Q4<double> q3 = adv(x.q, dq2, d.half_dt);
  const Q4<double> dq3 = dq_of(q3);
  const Q4<double> q4 = adv(x.q, dq3, d.dt);
  const Q4<double> dq4 = dq_of(q4);
  // stage accelerations, one stage per lane
  const Q4<double> qs = lane == 0 ? x.q : (lane == 1 ? q2 : (lane == 2 ? q3 : q4));
  const V3<double> dir = qrot(qnormalized(qs), V3<double>{0.0, 0.0, 1.0});
  const double a = thrust / d.mass;
  const V3<double> dvl = V3<double>{a * dir.x, a * dir.y, a * dir.z} + V3<double>{d.gx, d.gy, d.gz};
  V3<double> dv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    dv[i] = {__shfl_sync(0xffffffffu, dvl.x, i), __shfl_sync(0xffffffffu, dvl.y, i),
             __shfl_sync(0xffffffffu, dvl.z, i)};
  const V3<double> v2 = x.v + d.half_dt * dv[0];
  const V3<double> v3 = x.v + d.half_dt * dv[1];
  const V3<double> v4 = x.v + d.dt * dv[2];
  const double h6 = d.dt6;
  St<double> n;
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

template <typename Pert>
__device__ TrajSums rollout_warp64(St<double> x0, const RolloutEnv<double>& env, const Pert& pert, double* pos_out,
                                   double* sm, volatile int* ready = nullptr) {
  const int lane = threadIdx.x & 31, N = env.N;
  double* su = sm;                  // [N*4] applied controls
  double* sx = su + 4 * N;          // [(N+1)*10] states p q v
  double* st = sx + 10 * (N + 1);   // [7][N]: trk vn g1 g2 g3 mag rate
  const Dyn<double>& dy = env.dyn;
  for (int j = lane; j < N; j += 32) {
    double d[4];
    pert(j, d);
    su[4 * j] = clampv(env.unom_at(j, 0) + d[0], dy.tmin, dy.tmax);
    su[4 * j + 1] = clampv(env.unom_at(j, 1) + d[1], -dy.wxy, dy.wxy);
    su[4 * j + 2] = clampv(env.unom_at(j, 2) + d[2], -dy.wxy, dy.wxy);
    su[4 * j + 3] = clampv(env.unom_at(j, 3) + d[3], -dy.wz, dy.wz);
  }
  __syncwarp();
  for (int j = lane; j < N; j += 32) {
    const double u0 = su[4 * j], u1 = su[4 * j + 1], u2 = su[4 * j + 2], u3 = su[4 * j + 3];
    st[5 * N + j] = (((u0 * u0 + u1 * u1) + u2 * u2) + u3 * u3);
    if (j >= 1) {
      const double e0 = u0 - su[4 * j - 4], e1 = u1 - su[4 * j - 3], e2 = u2 - su[4 * j - 2], e3 = u3 - su[4 * j - 1];
      st[6 * N + j] = (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3);
    }
  }
  __syncwarp();
  int n_ok = N;  // states 0..n_ok-1 are costed; n_ok < N: the rollout went non-finite
  {
    St<double> x = x0;  // identical in every lane
    for (int j = 0; j < N; ++j) {
      if (lane == 0) {
        double* o = sx + 10 * j;
        o[0] = x.p.x; o[1] = x.p.y; o[2] = x.p.z;
        o[3] = x.q.w; o[4] = x.q.x; o[5] = x.q.y; o[6] = x.q.z;
        o[7] = x.v.x; o[8] = x.v.y; o[9] = x.v.z;
        if (ready) {  // state j is visible to the consumer warp of the CTA
          __threadfence_block();
          *ready = j + 1;
        }
      }
      const St<double> nx =
          rk4_normalized_warp(x, su[4 * j], V3<double>{su[4 * j + 1], su[4 * j + 2], su[4 * j + 3]}, dy);
      if (!state_finite(nx)) {  // warp-uniform
        n_ok = j + 1;  // state j was costed, then the rollout stopped
        break;
      }
      x = nx;
    }
  }
  const bool valid = n_ok == N;
  if (ready && lane == 0) {
    __threadfence_block();
    *ready = kRolloutDone + n_ok;  // the chain is over: n_ok states exist
  }
  __syncwarp();
  for (int j = lane; j < n_ok; j += 32) {
    const double* o = sx + 10 * j;
    const V3<double> p{o[0], o[1], o[2]}, v{o[7], o[8], o[9]};
    const Q4<double> q{o[3], o[4], o[5], o[6]};
    if (env.has_guide) st[j] = norm3(p - env.guide_at(j));
    st[N + j] = sqnorm(v);
    st[2 * N + j] = env.q_p * norm3(p - env.pg);
    st[3 * N + j] = env.q_v * norm3(v - env.vg);
    st[4 * N + j] = env.q_q * env.attitude(q);
    pos_out[4 * j] = p.x;
    pos_out[4 * j + 1] = p.y;
    pos_out[4 * j + 2] = p.z;
  }
  __syncwarp();
  TrajSums t{0, 0, 0, 0, 0, valid ? 1 : 0};
  if (lane == 0) {
    double trk = 0.0, vn = 0.0, goal = 0.0, mag = 0.0, rate = 0.0;
    for (int j = 0; j < n_ok; ++j) {  // rollout_costs' order, step by step
      if (env.has_guide) trk = trk + st[j];
      vn = vn + st[N + j];
      goal = goal + st[2 * N + j];
      goal = goal + st[3 * N + j];
      goal = goal + st[4 * N + j];
      if (j + 1 < N) {
        mag = mag + st[5 * N + j];
        if (j >= 1) rate = rate + st[6 * N + j];
      }
    }
    t = TrajSums{trk, vn, mag, rate, goal, valid ? 1 : 0};
  }
  return t;
}

// Throughput form: one thread per instance.
__global__ void __launch_bounds__(64) k_stage2_traj(BatchIn in, Perception P, Plan pl, DevConfig cfg) {
  const int64_t smi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (smi >= static_cast<int64_t>(in.S) * cfg.M) return;
  TrajSums t{0, 0, 0, 0, 0, 0};
  if (pl.alive[smi]) {
    const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    const CostSums<double> cs = rollout_costs<double, PertZero<double>, true>(
        load_state(in.states + 10 * s), env, PertZero<double>{}, nullptr, nullptr, pl.pos64 + smi * cfg.N * 4);
    t = TrajSums{cs.trk, cs.vn, cs.mag, cs.rate, cs.goal, cs.valid ? 1 : 0};
  }
  pl.tsum[smi] = t;
}

// Latency path, fused: one 64-thread CTA per trajectory.  Warp 0 runs the
// FP64 trajectory (rollout_warp64) and publishes each state as soon as the
// RK4 chain reaches it; warp 1 answers the exact collision query of step j
// (lane j) as soon as state j is published, so the queries overlap the chain
// instead of following it in a second kernel.  Same terms, summed in step
// order: the results equal the two-kernel form.
__device__ __forceinline__ void consume_collisions(const RolloutEnv<double>& env, const double* sx, int N,
                                                   volatile int* ready, double* terms) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < N; j += 32) {
    int r;
    while ((r = *ready) <= j) {
    }
    __threadfence_block();
    const int n_ok = r >= kRolloutDone ? r - kRolloutDone : N;
    terms[j] = j < n_ok ? env.collision(V3<double>{sx[10 * j], sx[10 * j + 1], sx[10 * j + 2]}) : 0.0;
  }
}

__global__ void __launch_bounds__(64) k_stage2_fused_w(BatchIn in, Perception P, Plan pl, DevConfig cfg) {
  __shared__ double s_scr[warp_rollout_doubles(kRolloutMaxN)];
  __shared__ double s_terms[kRolloutMaxN];
  __shared__ int s_ready;
  __shared__ TrajSums s_t;
  const int64_t smi = blockIdx.x;
  if (smi >= static_cast<int64_t>(in.S) * cfg.M) return;
  if (threadIdx.x == 0) s_ready = 0;
  __syncthreads();
  const bool alive = pl.alive[smi];
  const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
  if (alive) {
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    double* sx = s_scr + 4 * cfg.N;  // rollout_warp64's state table
    if (threadIdx.x < 32) {
      const TrajSums t = rollout_warp64(load_state(in.states + 10 * s), env, PertZero<double>{},
                                        pl.pos64 + smi * cfg.N * 4, s_scr, &s_ready);
      if (threadIdx.x == 0) s_t = t;
    } else {
      consume_collisions(env, sx, cfg.N, &s_ready, s_terms);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double st2 = __longlong_as_double(0x7ff0000000000000ll);
    bool valid = false;
    double bd[5] = {0, 0, 0, 0, 0};
    if (alive && s_t.valid) {
      double col = 0.0;
      for (int j = 0; j < cfg.N; ++j) col = col + s_terms[j];
      const TrajSums t = s_t;
      st2 = t.goal + col;  // stage2_cost (costs.hpp:139-147)
      valid = isfinite(st2);
      bd[0] = cfg.q_track * t.trk;
      bd[1] = cfg.q_vnorm * t.vn;
      bd[2] = cfg.q_c * t.mag + cfg.q_c_delta * t.rate;
      bd[3] = t.goal;
      bd[4] = col;
    }
    pl.stage2[smi] = st2;
    pl.valid[smi] = valid ? 1 : 0;
    for (int i = 0; i < 5; ++i) pl.breakdown[smi * 5 + i] = bd[i];
  }
}

__global__ void __launch_bounds__(64) k_refine_fused_w(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                       UpdateScratch us, int iter) {
  __shared__ double s_scr[warp_rollout_doubles(kRolloutMaxN)];
  __shared__ double s_terms[kRolloutMaxN];
  __shared__ int s_ready;
  __shared__ TrajSums s_t;
  const unsigned long long n = min(*us.pair_count, static_cast<unsigned long long>(pl.pos_cap));
  for (unsigned long long w = blockIdx.x; w < n; w += gridDim.x) {
    if (threadIdx.x == 0) s_ready = 0;
    __syncthreads();
    const uint2 pr = us.pairs[w];
    const int64_t smi = pr.x;
    const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
    const int k = static_cast<int>(us.cand_k[smi * cfg.K + pr.y]);
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    double* pos = pl.pos64 + static_cast<int64_t>(w) * cfg.N * 4;
    if (threadIdx.x < 32) {
      const St<double> x0 = load_state(in.states + 10 * s);
      TrajSums t;
      if (in.injected) {
        t = rollout_warp64(x0, env, PertInjected<double>{injected_row(in, cfg, s, iter, m, k)}, pos, s_scr, &s_ready);
      } else {
        const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
        const PertRngD prng{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                            cfg.sigma[0], cfg.sigma[1], cfg.sigma[2], cfg.sigma[3]};
        t = rollout_warp64(x0, env, prng, pos, s_scr, &s_ready);
      }
      if (threadIdx.x == 0) s_t = t;
    } else {
      consume_collisions(env, s_scr + 4 * cfg.N, cfg.N, &s_ready, s_terms);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const TrajSums t = s_t;
      double val = __longlong_as_double(0x7ff0000000000000ll);
      if (t.valid) {
        double col = 0.0;
        for (int j = 0; j < cfg.N; ++j) col = col + s_terms[j];
        val = ((cfg.q_track * t.trk + cfg.q_vnorm * t.vn) + (cfg.q_c * t.mag + cfg.q_c_delta * t.rate)) + (t.goal + col);
      }
      pl.tsum[w] = t;
      us.cand_s[smi * cfg.K + pr.y] = val;
    }
    __syncthreads();  // s_ready / s_terms are reused by the next trajectory
  }
}

// Sum of the N collision terms of one deferred trajectory, in step order
// (warp-cooperative; the result is valid in every lane).
__device__ __forceinline__ double collision_sum_warp(const RolloutEnv<double>& env, const double* pos, int N,
                                                     double* sm_terms) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < N; j += 32)
    sm_terms[j] = env.collision(V3<double>{pos[4 * j], pos[4 * j + 1], pos[4 * j + 2]});
  __syncwarp();
  double col = 0.0;
  if (lane == 0)
    for (int j = 0; j < N; ++j) col = col + sm_terms[j];
  return __shfl_sync(0xffffffffu, col, 0);
}

__global__ void __launch_bounds__(128, AMPPI_COL_MINB) k_stage2_col(BatchIn in, Perception P, Plan pl, DevConfig cfg) {
  __shared__ double s_terms[4][64];
  const int64_t smi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (smi >= static_cast<int64_t>(in.S) * cfg.M) return;
  const TrajSums t = pl.tsum[smi];
  double st2 = __longlong_as_double(0x7ff0000000000000ll);
  bool valid = false;
  double bd[5] = {0, 0, 0, 0, 0};
  if (pl.alive[smi] && t.valid) {
    const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    const double col = collision_sum_warp(env, pl.pos64 + smi * cfg.N * 4, cfg.N, s_terms[wid]);
    st2 = t.goal + col;  // stage2_cost (costs.hpp:139-147)
    valid = isfinite(st2);
    bd[0] = cfg.q_track * t.trk;
    bd[1] = cfg.q_vnorm * t.vn;
    bd[2] = cfg.q_c * t.mag + cfg.q_c_delta * t.rate;
    bd[3] = t.goal;
    bd[4] = col;
  }
  if (lane == 0) {
    pl.stage2[smi] = st2;
    pl.valid[smi] = valid ? 1 : 0;
    for (int i = 0; i < 5; ++i) pl.breakdown[smi * 5 + i] = bd[i];
  }
}

// Latency-path refine: deferred-collision FP64 trajectory per support slot,
// then a warp per slot for the collision terms.
// Throughput form: one thread per support pair.
__global__ void __launch_bounds__(64) k_refine_traj(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                    UpdateScratch us, int iter) {
  const unsigned long long n = min(*us.pair_count, static_cast<unsigned long long>(pl.pos_cap));
  for (unsigned long long w = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; w < n;
       w += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const uint2 pr = us.pairs[w];
    const int64_t smi = pr.x;
    const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
    const int k = static_cast<int>(us.cand_k[smi * cfg.K + pr.y]);
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
    const St<double> x0 = load_state(in.states + 10 * s);
    double* pos = pl.pos64 + static_cast<int64_t>(w) * cfg.N * 4;
    CostSums<double> cs;
    if (in.injected) {
      cs = rollout_costs<double, PertInjected<double>, true>(
          x0, env, PertInjected<double>{injected_row(in, cfg, s, iter, m, k)}, nullptr, nullptr, pos);
    } else {
      const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
      const PertRngD prng{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                          cfg.sigma[0], cfg.sigma[1], cfg.sigma[2], cfg.sigma[3]};
      cs = rollout_costs<double, PertRngD, true>(x0, env, prng, nullptr, nullptr, pos);
    }
    pl.tsum[w] = TrajSums{cs.trk, cs.vn, cs.mag, cs.rate, cs.goal, cs.valid ? 1 : 0};
  }
}

__global__ void __launch_bounds__(128, AMPPI_COL_MINB) k_refine_col(BatchIn in, Perception P, Plan pl, DevConfig cfg,
                                                    UpdateScratch us) {
  __shared__ double s_terms[4][64];
  const unsigned long long n = min(*us.pair_count, static_cast<unsigned long long>(pl.pos_cap));
  const int wid = threadIdx.x >> 5;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  for (unsigned long long w = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n;
       w += (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5) {
    const uint2 pr = us.pairs[w];
    const int64_t smi = pr.x;
    const TrajSums t = pl.tsum[w];
    double val = kInf;
    if (t.valid) {
      const int s = static_cast<int>(smi / cfg.M), m = static_cast<int>(smi % cfg.M);
      const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * cfg.N * 4);
      const double col = collision_sum_warp(env, pl.pos64 + static_cast<int64_t>(w) * cfg.N * 4, cfg.N, s_terms[wid]);
      val = ((cfg.q_track * t.trk + cfg.q_vnorm * t.vn) + (cfg.q_c * t.mag + cfg.q_c_delta * t.rate)) + (t.goal + col);
    }
    if ((threadIdx.x & 31) == 0) us.cand_s[smi * cfg.K + pr.y] = val;
  }
}

// ---------------------------------------------------------------------------
// Collision terms of deferred FP64 trajectories (the refined support and the
// stage-II re-rollouts), as three passes over (trajectory, step) queries:
//   k_col_classify  one thread per query: a step whose padded neighbour mask
//                   is empty has nothing within d_max (term 0); the others
//                   join a work list;
//   k_col_query     one thread per listed query: the exact FP64 nearest
//                   distance (nearest_sq_exact) and the collision term;
//   k_*_col_sum     one thread per trajectory: the N terms summed in step
//                   order (the reference's sum over states[0..N-1]).
// Every lane of the query pass carries a real query; the former warp per
// trajectory (lane = step) idled beside the trajectory's empty steps and ran
// 4.4 of 32 lanes per instruction.  Terms and sums are the same FP64 values.
struct ColJobs {
  const uint2* pairs;                    // refine: (instance, slot) per trajectory; stage II: null (w = instance)
  const unsigned long long* pair_count;  // refine: trajectories listed
  int64_t cap;                           // trajectories with deferred positions
};

__device__ __forceinline__ bool col_traj(const ColJobs& J, const Plan& pl, int64_t w, int64_t* smi) {
  if (J.pairs) {
    if (w >= static_cast<int64_t>(min(*J.pair_count, static_cast<unsigned long long>(J.cap)))) return false;
    *smi = J.pairs[w].x;
    return pl.tsum[w].valid != 0;
  }
  if (w >= J.cap) return false;
  *smi = w;
  return pl.alive[w] && pl.tsum[w].valid;
}

__global__ void __launch_bounds__(256) k_col_classify(Perception P, Plan pl, DevConfig cfg, ColJobs J,
                                                      uint32_t* __restrict__ work, unsigned int* __restrict__ count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t w = i / cfg.N;
  int64_t smi;
  if (!col_traj(J, pl, w, &smi)) return;
  const int s = static_cast<int>(smi / cfg.M);
  const GridMeta g = P.grid[s];
  bool near = false;
  if (g.dims[0] != 0) {  // the cell test of nearest_sq_exact
    const double* q = pl.pos64 + 4 * i;
    const int cx = static_cast<int>(floor((q[0] - g.origin[0]) * g.inv_h));
    const int cy = static_cast<int>(floor((q[1] - g.origin[1]) * g.inv_h));
    const int cz = static_cast<int>(floor((q[2] - g.origin[2]) * g.inv_h));
    near = nbr_mask(g, P.grid_nbr + static_cast<int64_t>(s) * kPadCells, cx, cy, cz) != 0u;
  }
  if (near)
    work[atomicAdd(count, 1u)] = static_cast<uint32_t>(i);
  else
    pl.col_terms[i] = 0.0;  // no point within d_max: collision_term(+inf) = 0
}

// Bucketed work list (AMPPI_COL_BUCKETS): a query's cost grows with the
// number of non-empty cells around it, and a warp of the query pass runs as
// long as its slowest lane, so the list is ordered by that count (most cells
// first): lanes of a warp get queries of similar cost.  Two passes over the
// queries: k_col_count histograms the counts (term 0 for empty
// neighbourhoods, as k_col_classify), k_col_place writes each listed query
// into its bucket's range.  counters: [0] list length, [1 + b] bucket count,
// [65 + b] bucket fill, for b = 27 - popcount(mask) in 0..26 (or, with
// AMPPI_COL_BUCKETS=2, 63 - (points in those cells) / 16 in 0..63).
#ifndef AMPPI_COL_BUCKETS
#define AMPPI_COL_BUCKETS 1
#endif
constexpr int kColBuckets = AMPPI_COL_BUCKETS == 2 ? 64 : 27;
constexpr int kColBucketSlots = 2 * 64 + 1;  // [0] length, [1 + b] counts, [65 + b] fills
static_assert(kColBucketSlots <= kColCountStride, "Plan::col_count stride");

__device__ __forceinline__ int col_bucket(const Perception& P, const Plan& pl, const ColJobs& J, const DevConfig& cfg,
                                          int64_t i, bool* valid) {
  const int64_t w = i / cfg.N;
  int64_t smi;
  *valid = col_traj(J, pl, w, &smi);
  if (!*valid) return -1;
  const int s = static_cast<int>(smi / cfg.M);
  const GridMeta g = P.grid[s];
  if (g.dims[0] == 0) return -1;
  const double* q = pl.pos64 + 4 * i;
  const int cx = static_cast<int>(floor((q[0] - g.origin[0]) * g.inv_h));
  const int cy = static_cast<int>(floor((q[1] - g.origin[1]) * g.inv_h));
  const int cz = static_cast<int>(floor((q[2] - g.origin[2]) * g.inv_h));
  const uint32_t m = nbr_mask(g, P.grid_nbr + static_cast<int64_t>(s) * kPadCells, cx, cy, cz);
#if AMPPI_COL_BUCKETS == 2
  // finer: the points in the non-empty cells around the query, 16 per bucket
  if (!m) return -1;
  const uint4* rec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  const int d2 = g.dims[2], d12 = g.dims[1] * g.dims[2];
  const int cbase = ((cx - 1) * g.dims[1] + (cy - 1)) * d2 + (cz - 1);
  uint32_t pts = 0, mm = m;
  while (mm) {
    const int b = __ffs(mm) - 1;
    mm &= mm - 1;
    pts += rec[2 * (cbase + nbr_offset(b, d12, d2))].x >> 16;
  }
  return kColBuckets - 1 - static_cast<int>(min(pts >> 4, static_cast<uint32_t>(kColBuckets - 1)));
#else
  return m ? 27 - __popc(m) : -1;
#endif
}

__global__ void __launch_bounds__(256) k_col_count(Perception P, Plan pl, DevConfig cfg, ColJobs J, int64_t q,
                                                   unsigned int* __restrict__ counters) {
  __shared__ unsigned int h[kColBuckets];
  if (threadIdx.x < kColBuckets) h[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < q) {
    bool valid;
    const int b = col_bucket(P, pl, J, cfg, i, &valid);
    if (b >= 0) atomicAdd(&h[b], 1u);
    else if (valid) pl.col_terms[i] = 0.0;  // no point within d_max: collision_term(+inf) = 0
  }
  __syncthreads();
  if (threadIdx.x < kColBuckets && h[threadIdx.x]) atomicAdd(&counters[1 + threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_col_place(Perception P, Plan pl, DevConfig cfg, ColJobs J, int64_t q,
                                                   uint32_t* __restrict__ work, unsigned int* __restrict__ counters) {
  __shared__ unsigned int h[kColBuckets], base[kColBuckets], start[kColBuckets];
  if (threadIdx.x < kColBuckets) h[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {  // bucket starts: exclusive prefix of the counts
    unsigned int run = 0;
    for (int b = 0; b < kColBuckets; ++b) {
      start[b] = run;
      run += counters[1 + b];
    }
    if (blockIdx.x == 0) counters[0] = run;
  }
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int b = -1;
  unsigned int r = 0;
  if (i < q) {
    bool valid;
    b = col_bucket(P, pl, J, cfg, i, &valid);
    if (b >= 0) r = atomicAdd(&h[b], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kColBuckets && h[threadIdx.x])
    base[threadIdx.x] = start[threadIdx.x] + atomicAdd(&counters[65 + threadIdx.x], h[threadIdx.x]);
  __syncthreads();
  if (b >= 0) work[base[b] + r] = static_cast<uint32_t>(i);
}

__global__ void __launch_bounds__(128) k_col_query(Perception P, Plan pl, DevConfig cfg, ColJobs J,
                                                   const uint32_t* __restrict__ work,
                                                   const unsigned int* __restrict__ count) {
  const unsigned int n = *count;
  for (unsigned int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const uint32_t i = work[q];
    const int64_t w = i / cfg.N;
    const int64_t smi = J.pairs ? static_cast<int64_t>(J.pairs[w].x) : w;
    const int s = static_cast<int>(smi / cfg.M);
    const double* pp = pl.pos64 + 4 * static_cast<int64_t>(i);
    uint32_t hint = kNoHint;
    const double d2 = nearest_sq_exact(P.grid[s], P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2,
                                       P.grid_nbr + static_cast<int64_t>(s) * kPadCells,
                                       P.grid_leaf + static_cast<int64_t>(s) * kCells * 2,
                                       P.grid_pts64 + static_cast<int64_t>(s) * kCells * 3,
                                       P.grid_pts32 + static_cast<int64_t>(s) * kCells,
                                       V3<double>{pp[0], pp[1], pp[2]}, cfg.col_d_max * cfg.col_d_max,
                                       cfg.col_d_min * cfg.col_d_min, &hint);
    pl.col_terms[i] = collision_term(sqrt(d2), cfg.col_scale, cfg.col_slope, cfg.col_d_min, cfg.col_d_max);
  }
}

__device__ __forceinline__ double col_sum(const Plan& pl, int64_t w, int N) {
  double col = 0.0;
  for (int j = 0; j < N; ++j) col = col + pl.col_terms[w * N + j];
  return col;
}

__global__ void __launch_bounds__(128) k_refine_col_sum(Plan pl, DevConfig cfg, UpdateScratch us, int64_t cap) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= static_cast<int64_t>(min(*us.pair_count, static_cast<unsigned long long>(cap)))) return;
  const uint2 pr = us.pairs[w];
  const TrajSums t = pl.tsum[w];
  double val = __longlong_as_double(0x7ff0000000000000ll);
  if (t.valid) {
    const double col = col_sum(pl, w, cfg.N);
    val = ((cfg.q_track * t.trk + cfg.q_vnorm * t.vn) + (cfg.q_c * t.mag + cfg.q_c_delta * t.rate)) + (t.goal + col);
  }
  us.cand_s[static_cast<int64_t>(pr.x) * cfg.K + pr.y] = val;
}

__global__ void __launch_bounds__(128) k_stage2_col_sum(BatchIn in, Plan pl, DevConfig cfg) {
  const int64_t smi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (smi >= static_cast<int64_t>(in.S) * cfg.M) return;
  const TrajSums t = pl.tsum[smi];
  double st2 = __longlong_as_double(0x7ff0000000000000ll);
  bool valid = false;
  double bd[5] = {0, 0, 0, 0, 0};
  if (pl.alive[smi] && t.valid) {
    const double col = col_sum(pl, smi, cfg.N);
    st2 = t.goal + col;  // stage2_cost (costs.hpp:139-147)
    valid = isfinite(st2);
    bd[0] = cfg.q_track * t.trk;
    bd[1] = cfg.q_vnorm * t.vn;
    bd[2] = cfg.q_c * t.mag + cfg.q_c_delta * t.rate;
    bd[3] = t.goal;
    bd[4] = col;
  }
  pl.stage2[smi] = st2;
  pl.valid[smi] = valid ? 1 : 0;
  for (int i = 0; i < 5; ++i) pl.breakdown[smi * 5 + i] = bd[i];
}

// classify + query passes for `jobs` (an upper bound of the) trajectories
void launch_col_queries(const Perception& P, const Plan& pl, const DevConfig& cfg, const ColJobs& J, int64_t jobs,
                        cudaStream_t st) {
  cudaMemsetAsync(pl.col_count, 0, (AMPPI_COL_BUCKETS ? kColBucketSlots : 1) * sizeof(unsigned int), st);
  const int64_t q = jobs * cfg.N;
  if (q == 0) return;
#if AMPPI_COL_BUCKETS
  k_col_count<<<static_cast<unsigned>((q + 255) / 256), 256, 0, st>>>(P, pl, cfg, J, q, pl.col_count);
  k_col_place<<<static_cast<unsigned>((q + 255) / 256), 256, 0, st>>>(P, pl, cfg, J, q, pl.col_work, pl.col_count);
#else
  k_col_classify<<<static_cast<unsigned>((q + 255) / 256), 256, 0, st>>>(P, pl, cfg, J, pl.col_work, pl.col_count);
#endif
  const int64_t b = std::min<int64_t>((q + 127) / 128, static_cast<int64_t>(device_sms()) * 16);
  k_col_query<<<static_cast<unsigned>(b), 128, 0, st>>>(P, pl, cfg, J, pl.col_work, pl.col_count);
}

__global__ void k_select(Plan pl, DevConfig cfg, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  int winner = -1;
  const int64_t base = static_cast<int64_t>(s) * cfg.M;
  for (int mm = 0; mm < cfg.M; ++mm) {
    if (!pl.valid[base + mm]) continue;
    if (winner < 0 || pl.stage2[base + mm] < pl.stage2[base + winner]) winner = mm;
  }
  pl.winner[s] = winner;
  pl.status[s] = winner < 0 ? 1 : 0;
  if (winner >= 0) {
    const Dyn<double> dy = make_dyn<double>(cfg);
    const double* u = pl.nominal + (base + winner) * cfg.N * 4;
    pl.control[4 * s] = clampv(u[0], dy.tmin, dy.tmax);
    pl.control[4 * s + 1] = clampv(u[1], -dy.wxy, dy.wxy);
    pl.control[4 * s + 2] = clampv(u[2], -dy.wxy, dy.wxy);
    pl.control[4 * s + 3] = clampv(u[3], -dy.wz, dy.wz);
  }
}

// Winner re-rollout states/controls (PlanResult::winner_rollout) on request.
__global__ void k_winner_rollout(BatchIn in, Perception P, Plan pl, DevConfig cfg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= in.S) return;
  const int w = pl.winner[s];
  if (w < 0) return;
  const int64_t smi = static_cast<int64_t>(s) * cfg.M + w;
  const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, w, pl.nominal + smi * cfg.N * 4);
  rollout_costs(load_state(in.states + 10 * s), env, PertZero<double>{}, pl.winner_states + static_cast<int64_t>(s) * (cfg.N + 1) * 10,
                pl.winner_controls + static_cast<int64_t>(s) * cfg.N * 4);
}

__global__ void k_gather(Plan pl, DevConfig cfg, int S, GatherOut g) {
  const int s = blockIdx.x;
  if (s >= S) return;
  const int w = pl.winner[s];
  const int M = cfg.M, N = cfg.N;
  const int64_t base = static_cast<int64_t>(s) * M;
  for (int i = threadIdx.x; i < 4 * N; i += blockDim.x)
    if (g.winner_nominal) g.winner_nominal[static_cast<int64_t>(s) * N * 4 + i] = w >= 0 ? pl.nominal[(base + w) * N * 4 + i] : 0.0;
  for (int m = threadIdx.x; m < M; m += blockDim.x)
    if (g.stage2) g.stage2[base + m] = pl.stage2[base + m];
  if (threadIdx.x < 5 && g.breakdown) g.breakdown[5 * s + threadIdx.x] = w >= 0 ? pl.breakdown[(base + w) * 5 + threadIdx.x] : 0.0;
  if (threadIdx.x < 4 && g.control) g.control[4 * s + threadIdx.x] = w >= 0 ? pl.control[4 * s + threadIdx.x] : 0.0;
  if (threadIdx.x == 0) {
    if (g.status) g.status[s] = pl.status[s];
    if (g.winner) g.winner[s] = w;
  }
}

// ---------------------------------------------------------------------------
// Screening-drift diagnostic, FP64 half (amppi_screen_drift): the rollouts
// k_drift32 integrated in FP32, integrated again as the refine does (FP64
// draws, oracle op order), with the exact FP64 clearance per step.  Reduced
// into acc[kDriftSlots] (non-negative doubles as ordered bits for the maxima):
//   0 rollouts compared (valid in both)      1 max |p32 - p64| (m)
//   2 max |d32 - d64| where min(d) < h - 1e-4 (m; h = grid cell > d_max + band)   3 steps in slot 2
//   4 steps on opposite sides of d_max outside the band (soundness: 0)
//   5 steps the screening flags (|d32 - d_max| < band)
//   6 max |S32 - S64| / |S64| over unflagged rollouts
//   7 rollouts valid in one precision only
// d32 is the screening's own distance: sqrt.approx of the FP32 squared
// clearance; band = 1e-4 d_max + 1e-4 as amb_band.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_max_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u(unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(128) k_drift64(BatchIn in, Perception P, Plan pl, DevConfig cfg, int iter, int s0,
                                                 int S, int kstride, const float4* steps, const float* cost,
                                                 unsigned long long* acc) {
  const int kn = (cfg.k_hi - cfg.k_lo + kstride - 1) / kstride;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t rows = static_cast<int64_t>(S) * cfg.M * kn;
  double dp_max = 0.0, dd_max = 0.0, rel_max = 0.0;
  unsigned long long n_roll = 0, n_cmp = 0, n_viol = 0, n_amb = 0, n_mis = 0;
  const float c32 = r < rows ? cost[r] : __int_as_float(0x7fc00000);
  if (r < rows && !isnan(c32)) {
    const int kk = static_cast<int>(r % kn);
    const int m = static_cast<int>((r / kn) % cfg.M);
    const int s = s0 + static_cast<int>(r / (static_cast<int64_t>(kn) * cfg.M));
    const int k = cfg.k_lo + kk * kstride;
    const int64_t smi = static_cast<int64_t>(s) * cfg.M + m;
    const int N = cfg.N;
    const RolloutEnv<double> env = make_env64(in, P, pl, cfg, s, m, pl.nominal + smi * N * 4);
    const St<double> x0 = load_state(in.states + 10 * s);
    const uint64_t iter_cycle = in.cycles[s] * static_cast<uint64_t>(cfg.iterations) + static_cast<uint64_t>(iter);
    const PertRngD pr{stream_key(in.seeds[s], static_cast<uint64_t>(m), iter_cycle, static_cast<uint64_t>(k)),
                      cfg.sigma[0], cfg.sigma[1], cfg.sigma[2], cfg.sigma[3]};
    const CostSums<double> cs = rollout_costs(x0, env, pr);
    const bool v32 = isfinite(c32);
    if (cs.valid != v32) {
      n_mis = 1;
    } else if (cs.valid) {
      n_roll = 1;
      const double c64 = stage1_total(cs, cfg.q_track, cfg.q_vnorm, cfg.q_c, cfg.q_c_delta);
      if (!signbit(c32)) rel_max = fabs(static_cast<double>(c32) - c64) / fmax(fabs(c64), 1e-300);
      double pos[4 * 64];
      rollout_costs<double, PertRngD, true>(x0, env, pr, nullptr, nullptr, pos);
      const float dmaxf = static_cast<float>(cfg.col_d_max);
      const float band = 1e-4f * dmaxf + 1e-4f;
      // both queries are exact below the grid cell h (>= d_max + band): the
      // 27 cells around a position hold every point that close
      const double lim = env.grid.h;
      uint32_t hint = kNoHint;
      const float4* st = steps + r * N;
      for (int j = 0; j < N; ++j) {
        const float4 q = st[j];
        const V3<double> p{pos[4 * j], pos[4 * j + 1], pos[4 * j + 2]};
        // q is in the screening's local frame (to_local_f)
        const V3<double> e{static_cast<double>(q.x) - (p.x - env.grid.org[0]),
                           static_cast<double>(q.y) - (p.y - env.grid.org[1]),
                           static_cast<double>(q.z) - (p.z - env.grid.org[2])};
        dp_max = fmax(dp_max, sqrt(sqnorm(e)));
        const double d64 = sqrt(nearest_sq_exact(env.grid, env.grec, env.gnbr, env.gleaf, env.gpts, env.gpts32, p, lim * lim, 0.0,
                                                 &hint));
        const float d32f = sqrt_approx(q.w);
        const double d32 = d32f;  // +inf past the reach in both
        if (fmin(d32, d64) < lim - 1e-4) {
          dd_max = fmax(dd_max, fabs(d32 - d64));
          ++n_cmp;
#ifdef AMPPI_DRIFT_DEBUG
          if (fabs(d32 - d64) > 1e-3 && atomicAdd(acc + 8, 1ull) < 12)
            printf("drift s=%d m=%d k=%d j=%d d32=%.9g d64=%.9g p64=(%.9g %.9g %.9g) p32=(%.9g %.9g %.9g) "
                   "grid origin=(%.9g %.9g %.9g) h=%.9g dims=(%d %d %d)\n",
                   s, m, k, j, d32, d64, p.x, p.y, p.z, q.x, q.y, q.z, env.grid.origin[0], env.grid.origin[1],
                   env.grid.origin[2], env.grid.h, env.grid.dims[0], env.grid.dims[1], env.grid.dims[2]);
#endif
        }
        if (fabsf(d32f - dmaxf) < band) {
          ++n_amb;
        } else if ((d32f < dmaxf) != (d64 < cfg.col_d_max)) {
          ++n_viol;
        }
      }
    }
  }
  dp_max = warp_max_d(dp_max);
  dd_max = warp_max_d(dd_max);
  rel_max = warp_max_d(rel_max);
  n_roll = warp_sum_u(n_roll);
  n_cmp = warp_sum_u(n_cmp);
  n_viol = warp_sum_u(n_viol);
  n_amb = warp_sum_u(n_amb);
  n_mis = warp_sum_u(n_mis);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc + 0, n_roll);
    atomicMax(acc + 1, static_cast<unsigned long long>(__double_as_longlong(dp_max)));
    atomicMax(acc + 2, static_cast<unsigned long long>(__double_as_longlong(dd_max)));
    atomicAdd(acc + 3, n_cmp);
    atomicAdd(acc + 4, n_viol);
    atomicAdd(acc + 5, n_amb);
    atomicMax(acc + 6, static_cast<unsigned long long>(__double_as_longlong(rel_max)));
    atomicAdd(acc + 7, n_mis);
  }
}

}  // namespace

cudaError_t launch_drift64(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                           int s0, int S, int kstride, const float4* steps, const float* cost,
                           unsigned long long* acc, cudaStream_t st) {
  const int kn = (cfg.k_hi - cfg.k_lo + kstride - 1) / kstride;
  const int64_t rows = static_cast<int64_t>(S) * cfg.M * kn;
  k_drift64<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, st>>>(in, P, pl, cfg, iter, s0, S, kstride, steps,
                                                                      cost, acc);
  return cudaGetLastError();
}

cudaError_t launch_gather(const Plan& pl, const DevConfig& cfg, int S, const GatherOut& g, cudaStream_t st) {
  k_gather<<<S, 128, 0, st>>>(pl, cfg, S, g);
  return cudaGetLastError();
}

int device_sms() {
  static int sms = [] {
    int v = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

cudaError_t launch_plan_begin(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                              cudaStream_t st, KernelTimer* timer) {
  const int SM = in.S * cfg.M;
  TimedRegion t(timer, "k_anchors", st);
  if (SM < device_sms() * 16)
    k_anchors<32><<<(SM * 32 + 63) / 64, 64, 0, st>>>(in, P, pl, cfg);
  else
    k_anchors<1><<<(SM + 63) / 64, 64, 0, st>>>(in, P, pl, cfg);
  return cudaGetLastError();
}

// Support + FP64 re-rollout of the support (FP32 screening): fills cand_s.
static void launch_support_refine(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                                  const UpdateScratch& us, int iter, const float* rho_ext, cudaStream_t st,
                                  KernelTimer* timer) {
  const int SM = in.S * cfg.M;
  const int sms = device_sms();
  cudaMemsetAsync(us.pair_count, 0, sizeof(unsigned long long), st);
  {
    TimedRegion t(timer, "k_support", st);
    k_support<<<SM, kSupportThreads, 0, st>>>(pl, cfg, us, 32, rho_ext);
  }
  // FP64 re-rollout of the support: trajectories first (collision deferred,
  // positions to pos64), then one warp per rollout for the collision terms --
  // a rollout's latency is its trajectory, not N sequential exact queries.
  // Pairs beyond pos_cap take the fused kernel.
  const int64_t total = static_cast<int64_t>(SM) * (cfg.k_hi - cfg.k_lo);
  const int64_t jobs = std::min<int64_t>(total, pl.pos_cap);
  {
    TimedRegion t(timer, "k_refine_traj", st);
    if (jobs < static_cast<int64_t>(sms) * 64) {  // too few rollouts to fill the GPU: cut the latency instead
      // trajectory and collision terms in one CTA per pair (queries overlap the RK4 chain)
      k_refine_fused_w<<<static_cast<int>(std::min<int64_t>(jobs, sms * 16)), 64, 0, st>>>(in, P, pl, cfg, us, iter);
    } else {
      const int64_t b = (jobs + 63) / 64;
      k_refine_traj<<<static_cast<int>(std::min<int64_t>(b, sms * 16)), 64, 0, st>>>(in, P, pl, cfg, us, iter);
    }
  }
  if (jobs >= static_cast<int64_t>(sms) * 64) {  // (the latency path's fused kernel produced the costs)
    TimedRegion t(timer, "k_refine_col", st);
    if (kColPasses) {
      launch_col_queries(P, pl, cfg, ColJobs{us.pairs, us.pair_count, pl.pos_cap}, jobs, st);
      k_refine_col_sum<<<static_cast<unsigned>((jobs + 127) / 128), 128, 0, st>>>(pl, cfg, us, pl.pos_cap);
    } else {
      const int64_t b = (jobs * 32 + 127) / 128;
      k_refine_col<<<static_cast<int>(std::min<int64_t>(b, sms * 32)), 128, 0, st>>>(in, P, pl, cfg, us);
    }
  }
  if (total > pl.pos_cap) {
    TimedRegion t(timer, "k_refine", st);
    const int64_t b = (total - pl.pos_cap + 63) / 64;
    k_refine<<<static_cast<int>(std::min<int64_t>(b, sms * 16)), 64, 0, st>>>(
        in, P, pl, cfg, us, iter, static_cast<unsigned long long>(pl.pos_cap));
  }
}

cudaError_t launch_plan_finish(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                               bool want_winner_rollout, cudaStream_t st, KernelTimer* timer) {
  const int SM = in.S * cfg.M;
  const bool latency = SM < device_sms() * 64;
  if (latency) {  // trajectory and collision terms in one CTA per instance
    TimedRegion t(timer, "k_stage2_fused_w", st);
    k_stage2_fused_w<<<SM, 64, 0, st>>>(in, P, pl, cfg);
  } else {
    TimedRegion t(timer, "k_stage2_traj", st);
    k_stage2_traj<<<(SM + 63) / 64, 64, 0, st>>>(in, P, pl, cfg);
  }
  if (!latency) {
    TimedRegion t(timer, "k_stage2_col", st);
    if (kColPasses) {
      launch_col_queries(P, pl, cfg, ColJobs{nullptr, nullptr, SM}, SM, st);
      k_stage2_col_sum<<<(SM + 127) / 128, 128, 0, st>>>(in, pl, cfg);
    } else {
      k_stage2_col<<<(SM * 32 + 127) / 128, 128, 0, st>>>(in, P, pl, cfg);
    }
  }
  {
    TimedRegion t(timer, "k_select", st);
    k_select<<<(in.S + 127) / 128, 128, 0, st>>>(pl, cfg, in.S);
  }
  if (want_winner_rollout) {
    TimedRegion t(timer, "k_winner_rollout", st);
    k_winner_rollout<<<(in.S + 31) / 32, 32, 0, st>>>(in, P, pl, cfg);
  }
  return cudaGetLastError();
}

cudaError_t launch_plan_impl(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                             int precision, bool want_winner_rollout, uint32_t* cand_k, double* cand_s, double* cand_w,
                             uint2* pairs, unsigned long long* pair_count, cudaStream_t st, KernelTimer* timer) {
  const int SM = in.S * cfg.M;
  if (cudaError_t e = launch_plan_begin(in, P, pl, cfg, st, timer); e != cudaSuccess) return e;
  const UpdateScratch us{cand_k, cand_s, cand_w, pairs, pair_count};
  for (int iter = 0; iter < cfg.iterations; ++iter) {
    if (precision == 32) {
      cudaError_t e = launch_stage1_f32(in, P, pl, cfg, iter, st, timer);
      if (e != cudaSuccess) return e;
      launch_support_refine(in, P, pl, cfg, us, iter, nullptr, st, timer);
    } else {
      const int threads = 128;
      const int tiles = (cfg.K + threads - 1) / threads;
      {
        TimedRegion t(timer, "k_stage1_f64", st);
        k_stage1_f64<<<SM * tiles, threads, 4 * cfg.N * sizeof(double), st>>>(in, P, pl, cfg, iter);
      }
      cudaMemsetAsync(pair_count, 0, sizeof(unsigned long long), st);
      TimedRegion t(timer, "k_support", st);
      k_support<<<SM, kSupportThreads, 0, st>>>(pl, cfg, us, precision, nullptr);
    }
    {
      TimedRegion t(timer, "k_nominal", st);
      k_nominal<<<SM, 128, 0, st>>>(in, pl, cfg, us, iter);
    }
  }
  return launch_plan_finish(in, P, pl, cfg, want_winner_rollout, st, timer);
}

cudaError_t launch_shard_screen(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                                float* local_min, cudaStream_t st, KernelTimer* timer) {
  if (cudaError_t e = launch_stage1_f32(in, P, pl, cfg, iter, st, timer); e != cudaSuccess) return e;
  k_local_min<<<in.S * cfg.M, 32, 0, st>>>(pl, cfg, local_min);
  return cudaGetLastError();
}

cudaError_t launch_shard_partials(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                                  uint32_t* cand_k, double* cand_s, double* cand_w, uint2* pairs,
                                  unsigned long long* pair_count, int iter, const float* global_min, double* partials,
                                  cudaStream_t st, KernelTimer* timer) {
  const UpdateScratch us{cand_k, cand_s, cand_w, pairs, pair_count};
  launch_support_refine(in, P, pl, cfg, us, iter, global_min, st, timer);
  TimedRegion t(timer, "k_partials", st);
  k_partials<<<in.S * cfg.M, 128, 0, st>>>(in, pl, cfg, us, iter, partials);
  return cudaGetLastError();
}

cudaError_t launch_shard_merge(const BatchIn& in, const Plan& pl, const DevConfig& cfg, const double* all_partials,
                               int n_shards, cudaStream_t st, KernelTimer* timer) {
  if (n_shards < 1 || n_shards > kMaxShards) return cudaErrorInvalidValue;
  TimedRegion t(timer, "k_merge", st);
  k_merge<<<in.S * cfg.M, 128, 0, st>>>(pl, cfg, all_partials, n_shards);
  return cudaGetLastError();
}

}  // namespace amppi_dev
