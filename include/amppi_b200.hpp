// amppi_b200.hpp — C++ shim over the C ABI (amppi_b200.h) that restores the
// reference planner's hot-path signatures and error behaviour:
//
//   PerceptionSnapshot build_snapshot(const PointCloudBuffer&, const State& pose,
//                                     double r_max = 10.0);        // perception.hpp:142-143
//   PlanResult plan_step(const State& x, const GoalSpec& goal,
//                        const PerceptionSnapshot& snap, const EnsembleConfig& cfg,
//                        const NominalSequence& previous,
//                        const ControlInput& last_applied, std::uint64_t cycle,
//                        std::uint64_t seed);                     // ensemble.hpp:65-69
//
// Differences a caller sees: value types use std::array instead of Eigen
// (conversion helpers for Eigen are provided when <Eigen/Dense> is present),
// and a Planner (one amppi_ctx: device arenas + stream) must exist; the
// snapshot lives on that planner's device.  plan_step throws
// std::runtime_error("planning failed") exactly where the reference does
// (ensemble.cpp:158); CUDA failures throw amppi_b200::CudaError.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "amppi_b200.h"

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#include <Eigen/Geometry>
#define AMPPI_B200_HAVE_EIGEN 1
#endif
#endif

namespace amppi_b200 {

using Vec3 = std::array<double, 3>;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// types.hpp:18-53
struct State {
  Vec3 p{0, 0, 0};
  std::array<double, 4> q{1, 0, 0, 0};  // w, x, y, z
  Vec3 v{0, 0, 0};
};

struct ControlInput {
  double thrust{0.0};
  Vec3 omega{0, 0, 0};
};

struct DynamicsParams {
  double mass{1.0};
  Vec3 gravity{0.0, 0.0, -9.81};
  double dt{0.05};
  double thrust_min{0.3};
  double thrust_max{16.35};
  double omega_xy_max{3.0};
  double omega_z_max{2.0};
  ControlInput hover() const {
    return {mass * std::sqrt((gravity[0] * gravity[0] + gravity[1] * gravity[1]) + gravity[2] * gravity[2]),
            {0, 0, 0}};
  }
};

// guidance.hpp:10-19, mppi.hpp:14-21, costs.hpp:13-29, ensemble.hpp:16-23
struct AnchorGrid {
  int m_h{5}, m_v{3};
  double lookahead{5.0}, spacing_deg{18.0}, terminal_speed{3.0}, min_anchor_distance{0.5};
  int count() const { return m_h * m_v; }
};
struct MppiConfig {
  int rollouts{128}, horizon{25};
  double lambda{0.1};
  std::array<double, 4> sigma{1.0, 1.0, 1.0, 0.5};
  double dt{0.05};
  int iterations{1};
};
struct CollisionParams {
  double scale{1.0e6}, slope{5.0}, d_min{0.4}, d_max{1.0};
};
struct CostWeights {
  double q_track{15.0}, q_vnorm{0.15}, q_c{0.5}, q_c_delta{0.5}, q_p{3.0}, q_v{0.25}, q_q{1.0};
  CollisionParams collision;
};
struct EnsembleConfig {
  AnchorGrid grid;
  MppiConfig mppi;
  CostWeights weights;
  DynamicsParams dynamics;
  double replan_hz{50.0};
  double r_max{10.0};

  amppi_config to_c() const {
    amppi_config c{};
    c.m_h = grid.m_h;
    c.m_v = grid.m_v;
    c.lookahead = grid.lookahead;
    c.spacing_deg = grid.spacing_deg;
    c.terminal_speed = grid.terminal_speed;
    c.min_anchor_distance = grid.min_anchor_distance;
    c.rollouts = mppi.rollouts;
    c.horizon = mppi.horizon;
    c.lambda = mppi.lambda;
    for (int i = 0; i < 4; ++i) c.sigma[i] = mppi.sigma[i];
    c.mppi_dt = mppi.dt;
    c.iterations = mppi.iterations;
    c.q_track = weights.q_track;
    c.q_vnorm = weights.q_vnorm;
    c.q_c = weights.q_c;
    c.q_c_delta = weights.q_c_delta;
    c.q_p = weights.q_p;
    c.q_v = weights.q_v;
    c.q_q = weights.q_q;
    c.col_scale = weights.collision.scale;
    c.col_slope = weights.collision.slope;
    c.col_d_min = weights.collision.d_min;
    c.col_d_max = weights.collision.d_max;
    c.mass = dynamics.mass;
    for (int i = 0; i < 3; ++i) c.gravity[i] = dynamics.gravity[i];
    c.dyn_dt = dynamics.dt;
    c.thrust_min = dynamics.thrust_min;
    c.thrust_max = dynamics.thrust_max;
    c.omega_xy_max = dynamics.omega_xy_max;
    c.omega_z_max = dynamics.omega_z_max;
    c.replan_hz = replan_hz;
    c.r_max = r_max;
    return c;
  }
};

// costs.hpp:42-56
struct GoalSpec {
  Vec3 p_goal{0, 0, 0};
  Vec3 v_goal{0, 0, 0};
  std::array<double, 4> q_goal{1, 0, 0, 0};
  static GoalSpec facing(const Vec3& from, const Vec3& target) {
    GoalSpec g;
    g.p_goal = target;
    const double dx = target[0] - from[0], dy = target[1] - from[1];
    if (dx * dx + dy * dy > 1e-12) {
      const double ha = 0.5 * std::atan2(dy, dx);
      const double s = std::sin(ha);
      g.q_goal = {std::cos(ha), s * 0.0, s * 0.0, s * 1.0};
    }
    return g;
  }
};

struct NominalSequence {
  std::vector<ControlInput> controls;
};

// perception.hpp:39-55: ring of world-frame frames, oldest evicted first
class PointCloudBuffer {
 public:
  explicit PointCloudBuffer(std::size_t capacity = 10) : capacity_(capacity) {}
  void push(std::vector<Vec3> world_frame_points) {
    frames_.push_back(std::move(world_frame_points));
    while (frames_.size() > capacity_) frames_.pop_front();
  }
  std::size_t frames() const { return frames_.size(); }
  std::size_t capacity() const { return capacity_; }
  std::size_t total_points() const {
    std::size_t n = 0;
    for (const auto& f : frames_) n += f.size();
    return n;
  }
  // frames concatenated oldest first (the order body_points projects them in)
  std::vector<double> flat_xyz() const {
    std::vector<double> out;
    out.reserve(3 * total_points());
    for (const auto& f : frames_)
      for (const auto& p : f) out.insert(out.end(), p.begin(), p.end());
    return out;
  }

 private:
  std::deque<std::vector<Vec3>> frames_;
  std::size_t capacity_;
};

struct Anchor {
  Vec3 initial_endpoint, refined_endpoint, safe_dir;
  double safe_range{0.0};
  int coarse_i{0}, coarse_j{0};
};

struct InstanceRecord {
  double stage1{0.0}, stage2{0.0}, ess{0.0};
  bool valid{false};
  NominalSequence nominal;
};

struct CostBreakdown {
  double track{0}, vnorm{0}, ctrl{0}, goal{0}, collision{0};
  double stage2() const { return goal + collision; }
  double stage1() const { return track + vnorm + ctrl + stage2(); }
};

struct PlanResult {
  int winner{-1};
  ControlInput control;
  std::vector<State> winner_states;  // winner_rollout.states (N+1)
  std::vector<ControlInput> winner_controls;
  std::vector<InstanceRecord> per_instance;
  std::vector<Anchor> anchors;
  std::vector<std::array<double, 18>> guide_coeffs;  // [axis][power]
  CostBreakdown breakdown;
};

class Planner;

// Device-resident snapshot: valid until the planner's next build_snapshot.
struct PerceptionSnapshot {
  Planner* planner{nullptr};
  State pose;
  double r_max{10.0};
  std::uint64_t generation{0};
};

class Planner {
 public:
  explicit Planner(const EnsembleConfig& cfg, int device = 0, int precision = 32, std::int64_t max_points = 1 << 20)
      : cfg_(cfg) {
    amppi_config c = cfg.to_c();
    amppi_options o;
    amppi_options_default(&o);
    o.device = device;
    o.precision = precision;
    o.max_points = max_points;
    amppi_ctx* h = nullptr;
    const int rc = amppi_create(&c, &o, &h);
    if (rc == AMPPI_INVALID_ARGUMENT) throw std::invalid_argument("invalid EnsembleConfig");
    if (rc != AMPPI_OK) throw CudaError("amppi_create failed (no CUDA device?)");
    ctx_.reset(h);
  }

  const EnsembleConfig& config() const { return cfg_; }

  PerceptionSnapshot build_snapshot(const PointCloudBuffer& buffer, const State& pose, double r_max = 10.0) {
    const std::vector<double> xyz = buffer.flat_xyz();
    amppi_state ps = to_c(pose);
    check(amppi_snapshot_f64(ctx_.get(), xyz.data(), static_cast<std::int64_t>(xyz.size() / 3), &ps, r_max));
    return PerceptionSnapshot{this, pose, r_max, ++generation_};
  }

  PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                       const NominalSequence& previous, const ControlInput& last_applied, std::uint64_t cycle,
                       std::uint64_t seed) {
    if (snap.planner != this || snap.generation != generation_)
      throw std::invalid_argument("snapshot is not this planner's current device snapshot");
    const int M = cfg_.grid.count(), N = cfg_.mppi.horizon;
    std::vector<double> prev;
    for (const auto& u : previous.controls) prev.insert(prev.end(), {u.thrust, u.omega[0], u.omega[1], u.omega[2]});
    std::vector<double> st1(M), st2(M), ess(M), nom(static_cast<std::size_t>(M) * N * 4), ai(3 * M), ar(3 * M),
        ad(3 * M), rng(M), gc(18 * M), ws(10 * (N + 1)), wc(4 * N);
    std::vector<std::uint8_t> valid(M);
    std::vector<std::int32_t> ij(2 * M);
    amppi_plan_result r{};
    r.stage1 = st1.data();
    r.stage2 = st2.data();
    r.ess = ess.data();
    r.valid = valid.data();
    r.nominal = nom.data();
    r.winner_states = ws.data();
    r.winner_controls = wc.data();
    r.anchor_initial = ai.data();
    r.anchor_refined = ar.data();
    r.anchor_safe_dir = ad.data();
    r.anchor_safe_range = rng.data();
    r.anchor_ij = ij.data();
    r.guide_coeffs = gc.data();
    amppi_state xs = to_c(x);
    amppi_goal g{};
    for (int i = 0; i < 3; ++i) {
      g.p_goal[i] = goal.p_goal[i];
      g.v_goal[i] = goal.v_goal[i];
    }
    for (int i = 0; i < 4; ++i) g.q_goal[i] = goal.q_goal[i];
    amppi_control la{last_applied.thrust, {last_applied.omega[0], last_applied.omega[1], last_applied.omega[2]}};
    const int rc = amppi_plan(ctx_.get(), &xs, &g, prev.empty() ? nullptr : prev.data(),
                              static_cast<std::int32_t>(previous.controls.size()), &la, cycle, seed, nullptr, &r);
    if (rc == AMPPI_PLANNING_FAILED) throw std::runtime_error("planning failed");
    check(rc);
    PlanResult out;
    out.winner = r.winner;
    out.control = {r.control.thrust, {r.control.omega[0], r.control.omega[1], r.control.omega[2]}};
    out.breakdown = {r.breakdown[0], r.breakdown[1], r.breakdown[2], r.breakdown[3], r.breakdown[4]};
    for (int m = 0; m < M; ++m) {
      InstanceRecord rec;
      rec.stage1 = st1[m];
      rec.stage2 = st2[m];
      rec.ess = ess[m];
      rec.valid = valid[m] != 0;
      if (rec.valid)
        for (int j = 0; j < N; ++j) {
          const double* u = &nom[(static_cast<std::size_t>(m) * N + j) * 4];
          rec.nominal.controls.push_back({u[0], {u[1], u[2], u[3]}});
        }
      out.per_instance.push_back(std::move(rec));
      Anchor a;
      for (int i = 0; i < 3; ++i) {
        a.initial_endpoint[i] = ai[3 * m + i];
        a.refined_endpoint[i] = ar[3 * m + i];
        a.safe_dir[i] = ad[3 * m + i];
      }
      a.safe_range = rng[m];
      a.coarse_i = ij[2 * m];
      a.coarse_j = ij[2 * m + 1];
      out.anchors.push_back(a);
      std::array<double, 18> c{};
      for (int i = 0; i < 18; ++i) c[i] = gc[18 * m + i];
      out.guide_coeffs.push_back(c);
    }
    for (int t = 0; t <= N; ++t) {
      const double* s = &ws[10 * t];
      out.winner_states.push_back({{s[0], s[1], s[2]}, {s[3], s[4], s[5], s[6]}, {s[7], s[8], s[9]}});
    }
    for (int j = 0; j < N; ++j) out.winner_controls.push_back({wc[4 * j], {wc[4 * j + 1], wc[4 * j + 2], wc[4 * j + 3]}});
    return out;
  }

 private:
  struct Deleter {
    void operator()(amppi_ctx* c) const { amppi_destroy(c); }
  };
  static amppi_state to_c(const State& s) {
    amppi_state o{};
    for (int i = 0; i < 3; ++i) {
      o.p[i] = s.p[i];
      o.v[i] = s.v[i];
    }
    for (int i = 0; i < 4; ++i) o.q[i] = s.q[i];
    return o;
  }
  void check(int rc) const {
    if (rc == AMPPI_OK) return;
    const std::string msg = amppi_last_error(ctx_.get());
    if (rc == AMPPI_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw CudaError(msg);
  }

  EnsembleConfig cfg_;
  std::unique_ptr<amppi_ctx, Deleter> ctx_;
  std::uint64_t generation_{0};
};

// Free functions with the reference's names (the planner stands in for the
// process-global worker pool of the reference).
inline PerceptionSnapshot build_snapshot(Planner& planner, const PointCloudBuffer& buffer, const State& pose,
                                         double r_max = 10.0) {
  return planner.build_snapshot(buffer, pose, r_max);
}

inline PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                            const EnsembleConfig& cfg, const NominalSequence& previous,
                            const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed) {
  if (!snap.planner) throw std::invalid_argument("snapshot without planner");
  (void)cfg;  // the planner was created with the configuration (device arenas are sized from it)
  return snap.planner->plan_step(x, goal, snap, previous, last_applied, cycle, seed);
}

#ifdef AMPPI_B200_HAVE_EIGEN
// Conversions from the reference's Eigen-based value types.
inline Vec3 from_eigen(const Eigen::Vector3d& v) { return {v.x(), v.y(), v.z()}; }
inline State state_from_eigen(const Eigen::Vector3d& p, const Eigen::Quaterniond& q, const Eigen::Vector3d& v) {
  return State{from_eigen(p), {q.w(), q.x(), q.y(), q.z()}, from_eigen(v)};
}
#endif

}  // namespace amppi_b200
