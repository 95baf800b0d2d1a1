// Fused rollout + stage-I/II cost evaluation, shared by the FP32 screening
// kernel (k_plan32.cu) and the FP64 exact paths (k_plan64.cu).
//
// One call = one rollout: N x (perturb -> clamp -> RK4 -> renormalise) with
// every cost term accumulated on the fly in registers (the reference
// materialises N+1 states per rollout and then walks them five times,
// mppi.cpp:33-61 + costs.hpp:59-162).  Accumulation order per term matches
// the reference's separate sums, so the FP64 instantiation reproduces the
// oracle's op sequence.
#pragma once

#include "device_math.cuh"

namespace amppi_dev {

#ifndef AMPPI_ENV_PRESCREEN
#define AMPPI_ENV_PRESCREEN (AMPPI_F32_BOX && AMPPI_F32_PRESCREEN)
#endif

template <typename R>
struct CostSums {
  R trk, vn, mag, rate, goal, col;
  bool valid;
  bool aborted;  // partial stage-I cost passed RolloutEnv::abort_above (FP32 screening only)
  bool amb;      // a step's FP32 distance fell within amb_band of d_max (FP32 screening only)
};

// Read-only per-(scene, instance) environment of a rollout.
template <typename R>
struct RolloutEnv;

template <>
struct RolloutEnv<double> {
  const double* unom;   // [N*4]
  const double* guide;  // [N*3]
  int N;
  Dyn<double> dyn;
  V3<double> pg, vg;
  M3 gt;  // R(q_goal)^T
  double q_p, q_v, q_q;
  double cs, ca, cdmin, cdmax;
  GridMeta grid;
  const uint4* grec;
  const uint32_t* gnbr;
  const uint4* gleaf;
  const double* gpts;
  const float4* gpts32;  // the FP32 point blocks (local frame): the exact query's prescreen
  bool has_guide;
  double abort_above;
  mutable uint32_t hint = kNoHint;  // nearest point of the previous query (per rollout)

  __device__ __forceinline__ V3<double> guide_at(int j) const {
    return {guide[3 * j], guide[3 * j + 1], guide[3 * j + 2]};
  }
  __device__ __forceinline__ double unom_at(int j, int c) const { return unom[4 * j + c]; }
  __device__ __forceinline__ double attitude(Q4<double> q) const { return attitude_err_exact(q, gt); }
  __device__ __forceinline__ double collision(V3<double> p) const {
    // (the latency kernels' lane-per-step queries: AMPPI_ENV_PRESCREEN)
    const double d2 =
        nearest_sq_exact<AMPPI_ENV_PRESCREEN>(grid, grec, gnbr, gleaf, gpts, gpts32, p, cdmax * cdmax, cdmin * cdmin, &hint);
    return collision_term(sqrt(d2), cs, ca, cdmin, cdmax);
  }
};

template <>
struct RolloutEnv<float> {
  const float* unom;     // [N*4] (shared memory)
  const float4* guide;   // [N]   (shared memory)
  int N;
  Dyn<float> dyn;
  V3<float> pg, vg;
  Q4<float> qg;
  float q_p, q_v, q_q;
  float cs, ca, cdmin, cdmax;
  GridMeta grid;
  const uint4* grec;
  const uint32_t* gnbr;
  const uint4* gleaf;
  const float4* gpts;
  bool has_guide;
  float abort_above;
  float wq_track, wq_vnorm, wq_c, wq_cd;  // stage-I weights for the partial-cost bound
  mutable uint32_t hint = kNoHint;        // nearest point of the previous query (per rollout)
  float d2_x0 = 0.f;                      // squared clearance of x0 (screening kernels share it per CTA)
  float reach2 = 0.f, band = 0.f, dthr_cap = 0.f;  // main pass: query reach, d_max band, abort-radius cap

  __device__ __forceinline__ V3<float> guide_at(int j) const {
    const float4 g = guide[j];
    return {g.x, g.y, g.z};
  }
  __device__ __forceinline__ float unom_at(int j, int c) const { return unom[4 * j + c]; }
  __device__ __forceinline__ float attitude(Q4<float> q) const { return attitude_err_fast(q, qg); }
  __device__ __forceinline__ float collision(V3<float> p, bool& amb) const {  // needs reach2 / band set
    const float d2 = nearest_sq_fast(grid, grec, gnbr, gleaf, gpts, p, reach2, cdmin * cdmin, &hint);
    return screen_collision_b(d2, cs, ca, cdmin, cdmax, band, amb);
  }
};

// Perturbation sources.  operator()(j, d) writes the 4 sampled deltas of step j.
struct PertRngD {
  uint64_t key;
  double s0, s1, s2, s3;
  __device__ __forceinline__ void operator()(int j, double* d) const {
    double a, b, c, e;
    normal_pair(key, 2u * j, a, b);
    normal_pair(key, 2u * j + 1u, c, e);
    d[0] = s0 * a;
    d[1] = s1 * b;
    d[2] = s2 * c;
    d[3] = s3 * e;
  }
};

struct PertRngF {
  uint64_t key;
  float s0, s1, s2, s3;
  __device__ __forceinline__ void operator()(int j, float* d) const {
    float a, b, c, e;
    normal_pair_f(key, 2u * j, a, b);
    normal_pair_f(key, 2u * j + 1u, c, e);
    d[0] = s0 * a;
    d[1] = s1 * b;
    d[2] = s2 * c;
    d[3] = s3 * e;
  }
};

template <typename R>
struct PertInjected {
  const double* base;  // [N*4]
  __device__ __forceinline__ void operator()(int j, R* d) const {
    d[0] = static_cast<R>(base[4 * j]);
    d[1] = static_cast<R>(base[4 * j + 1]);
    d[2] = static_cast<R>(base[4 * j + 2]);
    d[3] = static_cast<R>(base[4 * j + 3]);
  }
};

template <typename R>
struct PertZero {
  __device__ __forceinline__ void operator()(int, R* d) const { d[0] = d[1] = d[2] = d[3] = R(0); }
};

// Rollout with all cost sums.  If states/controls are given the trajectory is
// written out (winner_rollout); on a non-finite step the remaining entries
// repeat the last finite state / applied control as rollout_into does.
// kDeferCol: skip the collision queries and store the positions p_0..p_{N-1}
// (stride 4) to pos_out instead; a collision pass evaluates them in parallel.
template <typename R, typename Pert, bool kDeferCol = false>
__device__ __forceinline__ CostSums<R> rollout_costs(St<R> x, const RolloutEnv<R>& env, const Pert& pert,
                                                      R* states_out = nullptr, R* controls_out = nullptr,
                                                      R* pos_out = nullptr) {
  CostSums<R> s{R(0), R(0), R(0), R(0), R(0), R(0), true, false, false};
  const Dyn<R>& dy = env.dyn;
  R up0 = R(0), up1 = R(0), up2 = R(0), up3 = R(0);
  const int N = env.N;
  auto put_state = [&](int t, const St<R>& st) {
    if (states_out) {
      R* o = states_out + 10 * t;
      o[0] = st.p.x; o[1] = st.p.y; o[2] = st.p.z;
      o[3] = st.q.w; o[4] = st.q.x; o[5] = st.q.y; o[6] = st.q.z;
      o[7] = st.v.x; o[8] = st.v.y; o[9] = st.v.z;
    }
  };
  put_state(0, x);
  for (int j = 0; j < N; ++j) {
    // costs on states[j] (t = j < N)
    if (env.has_guide) s.trk = s.trk + norm3(x.p - env.guide_at(j));
    s.vn = s.vn + sqnorm(x.v);
    s.goal = s.goal + env.q_p * norm3(x.p - env.pg);
    s.goal = s.goal + env.q_v * norm3(x.v - env.vg);
    s.goal = s.goal + env.q_q * env.attitude(x.q);
    if constexpr (kDeferCol) {
      pos_out[4 * j] = x.p.x;
      pos_out[4 * j + 1] = x.p.y;
      pos_out[4 * j + 2] = x.p.z;
    } else {
      if constexpr (std::is_same_v<R, float>) s.col = s.col + env.collision(x.p, s.amb);
      else s.col = s.col + env.collision(x.p);
    }
    // perturbed, clamped control (mppi.cpp:40-45)
    R d[4];
    pert(j, d);
    const R u0 = clampv(env.unom_at(j, 0) + d[0], dy.tmin, dy.tmax);
    const R u1 = clampv(env.unom_at(j, 1) + d[1], -dy.wxy, dy.wxy);
    const R u2 = clampv(env.unom_at(j, 2) + d[2], -dy.wxy, dy.wxy);
    const R u3 = clampv(env.unom_at(j, 3) + d[3], -dy.wz, dy.wz);
    if (controls_out) {
      controls_out[4 * j] = u0; controls_out[4 * j + 1] = u1;
      controls_out[4 * j + 2] = u2; controls_out[4 * j + 3] = u3;
    }
    // control cost over t <= N-2 (costs.hpp:80-92)
    if (j + 1 < N) {
      s.mag = s.mag + (((u0 * u0 + u1 * u1) + u2 * u2) + u3 * u3);
      if (j >= 1) {
        const R e0 = u0 - up0, e1 = u1 - up1, e2 = u2 - up2, e3 = u3 - up3;
        s.rate = s.rate + (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3);
      }
    }
    up0 = u0; up1 = u1; up2 = u2; up3 = u3;
    if constexpr (std::is_same_v<R, float>) {
      // every stage-I term is >= 0, so the partial sum bounds the final cost
      // from below: past the bound the sample cannot be in the softmin support
      if (((env.wq_track * s.trk + env.wq_vnorm * s.vn) + (env.wq_c * s.mag + env.wq_cd * s.rate)) +
              (s.goal + s.col) > env.abort_above) {
        s.aborted = true;
        return s;
      }
    }
    const St<R> nx = rk4_normalized(x, u0, V3<R>{u1, u2, u3}, dy);
    if (!state_finite(nx)) {
      s.valid = false;
      if (states_out || controls_out)
        for (int rest = j; rest < N; ++rest) {
          put_state(rest + 1, x);
          if (controls_out) {
            controls_out[4 * rest] = u0; controls_out[4 * rest + 1] = u1;
            controls_out[4 * rest + 2] = u2; controls_out[4 * rest + 3] = u3;
          }
        }
      return s;
    }
    x = nx;
    put_state(j + 1, x);
  }
  return s;
}

template <typename R>
__device__ __forceinline__ R stage1_total(const CostSums<R>& s, R q_track, R q_vnorm, R q_c, R q_cd) {
  return ((q_track * s.trk + q_vnorm * s.vn) + (q_c * s.mag + q_cd * s.rate)) + (s.goal + s.col);
}

}  // namespace amppi_dev
