// amppi_b200.hpp — C++ shim over the C ABI (amppi_b200.h) that restores the
// reference planner's hot-path signatures and error behaviour:
//
//   PerceptionSnapshot build_snapshot(const PointCloudBuffer&, const State& pose,
//                                     double r_max = 10.0);        // perception.hpp:142-143
//   PlanResult plan_step(const State& x, const GoalSpec& goal,
//                        const PerceptionSnapshot& snap, const EnsembleConfig& cfg,
//                        const NominalSequence& previous,
//                        const ControlInput& last_applied, std::uint64_t cycle,
//                        std::uint64_t seed, PlanScratch& scratch);  // ensemble.hpp:59-63
//   PlanResult plan_step(..., std::uint64_t seed);                  // ensemble.hpp:65-69
//   State rk4_step(const State&, const ControlInput&, const DynamicsParams&);  // dynamics.hpp:64-70
//   EnsembleConfig apply_velocity_cap(const EnsembleConfig&, double cap);     // metrics.cpp:74-81
//
// Semantics follow the reference:
// - a PerceptionSnapshot is an immutable value (perception.hpp:132-133): it
//   keeps its input frames, so any snapshot can be planned on at any time;
//   the device copy of the most recent one is reused and an older one is
//   rebuilt on demand (identical result: the build is deterministic);
// - plan_step honours the cfg of every call: each host thread keeps one
//   device context per plan size (anchor grid, rollouts, horizon,
//   iterations); weights, dynamics and sampling parameters are re-applied per
//   call (amppi_set_config), so per-job configs such as apply_velocity_cap
//   (metrics.cpp:145) plan with their own weights;
// - PlanScratch is a caller-owned reusable workspace (the host result
//   buffers); output is identical with or without reuse (ensemble.hpp:43);
// - plan_step throws std::runtime_error("planning failed") exactly where the
//   reference does (ensemble.cpp:158); invalid arguments throw
//   std::invalid_argument; CUDA failures throw amppi_b200::CudaError.
// Differences a caller sees: value types use std::array instead of Eigen
// (conversion helpers for Eigen are provided when <Eigen/Dense> is present),
// and contexts live on device 0 unless set_default_device() says otherwise.
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
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

// dynamics.hpp:13-70: rigid-body CTBR model, classic RK4 over prm.dt with the
// quaternion as a plain R^4 block, renormalised afterwards (the vehicle step of
// execute_cycle, ensemble.cpp:274-276).  Host FP64 in the reference's Eigen
// operation order.
namespace detail {
struct Deriv {
  Vec3 dp;
  std::array<double, 4> dq;
  Vec3 dv;
};
inline Deriv derivative_raw(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  const auto& q = x.q;  // w, x, y, z
  const double ox = u.omega[0], oy = u.omega[1], oz = u.omega[2];
  // q (x) [0, omega], left to right (dynamics.hpp:18)
  const double qw = q[0] * 0.0 - q[1] * ox - q[2] * oy - q[3] * oz;
  const double qx = q[0] * ox + q[1] * 0.0 + q[2] * oz - q[3] * oy;
  const double qy = q[0] * oy + q[2] * 0.0 + q[3] * ox - q[1] * oz;
  const double qz = q[0] * oz + q[3] * 0.0 + q[1] * oy - q[2] * ox;
  Deriv d;
  d.dp = x.v;
  d.dq = {0.5 * qw, 0.5 * qx, 0.5 * qy, 0.5 * qz};
  // q.normalized() * e_z (Eigen _transformVector: uv = 2 (q.vec x v); v + w uv + q.vec x uv)
  double n[4] = {q[0], q[1], q[2], q[3]};
  const double n2 = ((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3]) + q[0] * q[0];
  if (n2 > 0.0) {
    const double nn = std::sqrt(n2);
    for (double& c : n) c = c / nn;
  }
  double uv[3] = {n[2] * 1.0 - n[3] * 0.0, n[3] * 0.0 - n[1] * 1.0, n[1] * 0.0 - n[2] * 0.0};
  for (double& c : uv) c = c + c;
  const double t0 = 0.0 + n[0] * uv[0], t1 = 0.0 + n[0] * uv[1], t2 = 1.0 + n[0] * uv[2];
  const double dir[3] = {t0 + (n[2] * uv[2] - n[3] * uv[1]), t1 + (n[3] * uv[0] - n[1] * uv[2]),
                         t2 + (n[1] * uv[1] - n[2] * uv[0])};
  const double a = u.thrust / prm.mass;
  for (int i = 0; i < 3; ++i) d.dv[i] = a * dir[i] + prm.gravity[i];
  return d;
}
}  // namespace detail

inline bool finite(const State& s) {
  for (double v : s.p) if (!std::isfinite(v)) return false;
  for (double v : s.q) if (!std::isfinite(v)) return false;
  for (double v : s.v) if (!std::isfinite(v)) return false;
  return true;
}

inline State rk4_step(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  if (!finite(x) || !std::isfinite(u.thrust) || !std::isfinite(u.omega[0]) || !std::isfinite(u.omega[1]) ||
      !std::isfinite(u.omega[2]))
    throw std::invalid_argument("invalid state");
  const double dt = prm.dt;
  auto advance = [](const State& s, const detail::Deriv& d, double h) {
    State o;
    for (int i = 0; i < 3; ++i) {
      o.p[i] = s.p[i] + h * d.dp[i];
      o.v[i] = s.v[i] + h * d.dv[i];
    }
    for (int i = 0; i < 4; ++i) o.q[i] = s.q[i] + h * d.dq[i];
    return o;
  };
  const detail::Deriv k1 = detail::derivative_raw(x, u, prm);
  const detail::Deriv k2 = detail::derivative_raw(advance(x, k1, 0.5 * dt), u, prm);
  const detail::Deriv k3 = detail::derivative_raw(advance(x, k2, 0.5 * dt), u, prm);
  const detail::Deriv k4 = detail::derivative_raw(advance(x, k3, dt), u, prm);
  const double h6 = dt / 6.0;
  State n;
  for (int i = 0; i < 3; ++i) {
    n.p[i] = x.p[i] + h6 * (((k1.dp[i] + 2.0 * k2.dp[i]) + 2.0 * k3.dp[i]) + k4.dp[i]);
    n.v[i] = x.v[i] + h6 * (((k1.dv[i] + 2.0 * k2.dv[i]) + 2.0 * k3.dv[i]) + k4.dv[i]);
  }
  for (int i = 0; i < 4; ++i) n.q[i] = x.q[i] + h6 * (((k1.dq[i] + 2.0 * k2.dq[i]) + 2.0 * k3.dq[i]) + k4.dq[i]);
  const double n2 = ((n.q[1] * n.q[1] + n.q[2] * n.q[2]) + n.q[3] * n.q[3]) + n.q[0] * n.q[0];
  if (n2 > 0.0) {
    const double nn = std::sqrt(n2);
    for (double& c : n.q) c = c / nn;
  }
  return n;
}

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

  bool same_sizes(const EnsembleConfig& o) const {
    return grid.m_h == o.grid.m_h && grid.m_v == o.grid.m_v && mppi.rollouts == o.mppi.rollouts &&
           mppi.horizon == o.mppi.horizon && mppi.iterations == o.mppi.iterations;
  }

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

// metrics.cpp:74-81: rescale Q_vnorm by (reference / cap)^2, retarget the terminal speed.
inline EnsembleConfig apply_velocity_cap(const EnsembleConfig& cfg, double cap) {
  if (!(cap > 0.0)) return cfg;
  EnsembleConfig out = cfg;
  const double reference = cfg.grid.terminal_speed;
  out.weights.collision = cfg.weights.collision;
  out.weights.q_vnorm = cfg.weights.q_vnorm * (reference / cap) * (reference / cap);
  out.grid.terminal_speed = cap;
  return out;
}

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

// ensemble.hpp:43-53: caller-owned reusable workspace.  Here it holds the host
// buffers the device results are copied into; plan_step output is identical
// with or without reuse.
struct PlanScratch {
  std::vector<double> stage1, stage2, ess, nominal, anchor_initial, anchor_refined, anchor_safe_dir,
      anchor_safe_range, guide_coeffs, winner_states, winner_controls, previous;
  std::vector<std::uint8_t> valid;
  std::vector<std::int32_t> anchor_ij;

  void resize(int instances, int horizon) {
    const std::size_t M = static_cast<std::size_t>(instances), N = static_cast<std::size_t>(horizon);
    stage1.resize(M);
    stage2.resize(M);
    ess.resize(M);
    valid.resize(M);
    nominal.resize(M * N * 4);
    anchor_initial.resize(3 * M);
    anchor_refined.resize(3 * M);
    anchor_safe_dir.resize(3 * M);
    anchor_safe_range.resize(M);
    anchor_ij.resize(2 * M);
    guide_coeffs.resize(18 * M);
    winner_states.resize(10 * (N + 1));
    winner_controls.resize(4 * N);
    previous.reserve(4 * N);
  }
};

namespace detail {
// The snapshot's inputs: the buffer's frames concatenated oldest first
// (PointCloudBuffer::body_points order), the pose and r_max.
struct SnapshotData {
  std::vector<double> xyz;
  State pose;
  double r_max{10.0};
  std::uint64_t id{0};
};
inline std::uint64_t next_snapshot_id() {
  static std::atomic<std::uint64_t> n{0};
  return ++n;
}
}  // namespace detail

// Immutable, shareable value (perception.hpp:132-143).  The device copy is
// built by build_snapshot on the calling thread's current context and rebuilt
// from the kept inputs by any context that plans on a snapshot it does not
// hold.
struct PerceptionSnapshot {
  State pose;
  double r_max{10.0};
  std::shared_ptr<const detail::SnapshotData> data;
  std::size_t point_count() const { return data ? data->xyz.size() / 3 : 0; }
};

class Planner;

namespace detail {
inline int& default_device() {
  static int dev = 0;
  return dev;
}
inline Planner*& current_planner() {
  thread_local Planner* p = nullptr;
  return p;
}
}  // namespace detail

inline void set_default_device(int device) { detail::default_device() = device; }

// One device context (amppi_ctx: device arenas + stream) of a fixed plan size.
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
  ~Planner() {
    if (detail::current_planner() == this) detail::current_planner() = nullptr;
  }
  Planner(const Planner&) = delete;
  Planner& operator=(const Planner&) = delete;

  const EnsembleConfig& config() const { return cfg_; }
  amppi_ctx* handle() const { return ctx_.get(); }

  // build_snapshot on this context (perception.cpp:237-246).
  PerceptionSnapshot build_snapshot(const PointCloudBuffer& buffer, const State& pose, double r_max = 10.0) {
    auto d = std::make_shared<detail::SnapshotData>();
    d->xyz = buffer.flat_xyz();
    d->pose = pose;
    d->r_max = r_max;
    d->id = detail::next_snapshot_id();
    upload(*d);
    return PerceptionSnapshot{pose, r_max, std::move(d)};
  }

  // plan_step (ensemble.hpp:59-63) on this context; cfg must have this
  // context's sizes (m_h, m_v, rollouts, horizon, iterations).
  PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                       const EnsembleConfig& cfg, const NominalSequence& previous, const ControlInput& last_applied,
                       std::uint64_t cycle, std::uint64_t seed, PlanScratch& scratch) {
    if (!snap.data) throw std::invalid_argument("empty PerceptionSnapshot");
    apply_config(cfg);
    ensure_snapshot(*snap.data);
    const int M = cfg_.grid.count(), N = cfg_.mppi.horizon;
    scratch.resize(M, N);
    scratch.previous.clear();
    for (const auto& u : previous.controls)
      scratch.previous.insert(scratch.previous.end(), {u.thrust, u.omega[0], u.omega[1], u.omega[2]});
    amppi_plan_result r{};
    r.stage1 = scratch.stage1.data();
    r.stage2 = scratch.stage2.data();
    r.ess = scratch.ess.data();
    r.valid = scratch.valid.data();
    r.nominal = scratch.nominal.data();
    r.winner_states = scratch.winner_states.data();
    r.winner_controls = scratch.winner_controls.data();
    r.anchor_initial = scratch.anchor_initial.data();
    r.anchor_refined = scratch.anchor_refined.data();
    r.anchor_safe_dir = scratch.anchor_safe_dir.data();
    r.anchor_safe_range = scratch.anchor_safe_range.data();
    r.anchor_ij = scratch.anchor_ij.data();
    r.guide_coeffs = scratch.guide_coeffs.data();
    amppi_state xs = to_c(x);
    amppi_goal g{};
    for (int i = 0; i < 3; ++i) {
      g.p_goal[i] = goal.p_goal[i];
      g.v_goal[i] = goal.v_goal[i];
    }
    for (int i = 0; i < 4; ++i) g.q_goal[i] = goal.q_goal[i];
    amppi_control la{last_applied.thrust, {last_applied.omega[0], last_applied.omega[1], last_applied.omega[2]}};
    const int rc = amppi_plan(ctx_.get(), &xs, &g, scratch.previous.empty() ? nullptr : scratch.previous.data(),
                              static_cast<std::int32_t>(previous.controls.size()), &la, cycle, seed, nullptr, &r);
    if (rc == AMPPI_PLANNING_FAILED) throw std::runtime_error("planning failed");
    check(rc);
    PlanResult out;
    out.winner = r.winner;
    out.control = {r.control.thrust, {r.control.omega[0], r.control.omega[1], r.control.omega[2]}};
    out.breakdown = {r.breakdown[0], r.breakdown[1], r.breakdown[2], r.breakdown[3], r.breakdown[4]};
    out.per_instance.reserve(M);
    out.anchors.reserve(M);
    out.guide_coeffs.reserve(M);
    for (int m = 0; m < M; ++m) {
      InstanceRecord rec;
      rec.stage1 = scratch.stage1[m];
      rec.stage2 = scratch.stage2[m];
      rec.ess = scratch.ess[m];
      rec.valid = scratch.valid[m] != 0;
      if (rec.valid)
        for (int j = 0; j < N; ++j) {
          const double* u = &scratch.nominal[(static_cast<std::size_t>(m) * N + j) * 4];
          rec.nominal.controls.push_back({u[0], {u[1], u[2], u[3]}});
        }
      out.per_instance.push_back(std::move(rec));
      Anchor a;
      for (int i = 0; i < 3; ++i) {
        a.initial_endpoint[i] = scratch.anchor_initial[3 * m + i];
        a.refined_endpoint[i] = scratch.anchor_refined[3 * m + i];
        a.safe_dir[i] = scratch.anchor_safe_dir[3 * m + i];
      }
      a.safe_range = scratch.anchor_safe_range[m];
      a.coarse_i = scratch.anchor_ij[2 * m];
      a.coarse_j = scratch.anchor_ij[2 * m + 1];
      out.anchors.push_back(a);
      std::array<double, 18> c{};
      for (int i = 0; i < 18; ++i) c[i] = scratch.guide_coeffs[18 * m + i];
      out.guide_coeffs.push_back(c);
    }
    for (int t = 0; t <= N; ++t) {
      const double* s = &scratch.winner_states[10 * t];
      out.winner_states.push_back({{s[0], s[1], s[2]}, {s[3], s[4], s[5], s[6]}, {s[7], s[8], s[9]}});
    }
    for (int j = 0; j < N; ++j)
      out.winner_controls.push_back({scratch.winner_controls[4 * j],
                                     {scratch.winner_controls[4 * j + 1], scratch.winner_controls[4 * j + 2],
                                      scratch.winner_controls[4 * j + 3]}});
    return out;
  }

  PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                       const EnsembleConfig& cfg, const NominalSequence& previous, const ControlInput& last_applied,
                       std::uint64_t cycle, std::uint64_t seed) {
    PlanScratch scratch;
    return plan_step(x, goal, snap, cfg, previous, last_applied, cycle, seed, scratch);
  }

  // Make cfg this context's configuration (same sizes required).
  void apply_config(const EnsembleConfig& cfg) {
    if (!cfg.same_sizes(cfg_))
      throw std::invalid_argument("EnsembleConfig sizes differ from this planner's (create another Planner)");
    const amppi_config c = cfg.to_c(), cur = cfg_.to_c();
    if (std::memcmp(&c, &cur, sizeof(c)) == 0) return;
    check(amppi_set_config(ctx_.get(), &c));
    if (cfg.weights.collision.d_max != cfg_.weights.collision.d_max) device_snapshot_ = 0;  // grid sized by d_max
    cfg_ = cfg;
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
    if (rc == AMPPI_PLANNING_FAILED) throw std::runtime_error("planning failed");
    throw CudaError(msg);
  }
  void upload(const detail::SnapshotData& d) {
    amppi_state ps = to_c(d.pose);
    check(amppi_snapshot_f64(ctx_.get(), d.xyz.data(), static_cast<std::int64_t>(d.xyz.size() / 3), &ps, d.r_max));
    device_snapshot_ = d.id;
  }
  void ensure_snapshot(const detail::SnapshotData& d) {
    if (device_snapshot_ != d.id) upload(d);
  }

  EnsembleConfig cfg_;
  std::unique_ptr<amppi_ctx, Deleter> ctx_;
  std::uint64_t device_snapshot_{0};  // id of the snapshot the context's device slot holds
};

namespace detail {
// The calling thread's contexts, one per plan size (the reference's
// plan_step is reentrant across threads; contexts are never shared).
inline Planner& planner_for(const EnsembleConfig& cfg) {
  using Key = std::tuple<int, int, int, int, int, int>;
  thread_local std::map<Key, std::unique_ptr<Planner>> planners;
  const Key key{default_device(), cfg.grid.m_h, cfg.grid.m_v, cfg.mppi.rollouts, cfg.mppi.horizon,
                cfg.mppi.iterations};
  auto it = planners.find(key);
  if (it == planners.end()) it = planners.emplace(key, std::make_unique<Planner>(cfg, default_device())).first;
  current_planner() = it->second.get();
  return *it->second;
}
}  // namespace detail

// build_snapshot(buffer, pose, r_max) (perception.hpp:142-143): builds the
// device snapshot on the thread's current context (the one its last plan_step
// used; a default-config context before the first plan).
inline PerceptionSnapshot build_snapshot(const PointCloudBuffer& buffer, const State& pose, double r_max = 10.0) {
  Planner* p = detail::current_planner();
  if (!p) p = &detail::planner_for(EnsembleConfig{});
  return p->build_snapshot(buffer, pose, r_max);
}

// plan_step (ensemble.hpp:59-69).
inline PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                            const EnsembleConfig& cfg, const NominalSequence& previous,
                            const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed,
                            PlanScratch& scratch) {
  return detail::planner_for(cfg).plan_step(x, goal, snap, cfg, previous, last_applied, cycle, seed, scratch);
}

inline PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                            const EnsembleConfig& cfg, const NominalSequence& previous,
                            const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed) {
  PlanScratch scratch;
  return plan_step(x, goal, snap, cfg, previous, last_applied, cycle, seed, scratch);
}

#ifdef AMPPI_B200_HAVE_EIGEN
// Conversions from the reference's Eigen-based value types.
inline Vec3 from_eigen(const Eigen::Vector3d& v) { return {v.x(), v.y(), v.z()}; }
inline State state_from_eigen(const Eigen::Vector3d& p, const Eigen::Quaterniond& q, const Eigen::Vector3d& v) {
  return State{from_eigen(p), {q.w(), q.x(), q.y(), q.z()}, from_eigen(v)};
}
#endif

}  // namespace amppi_b200
