// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ restatement of the AERO-MPPI reference planner's hot path
// (build_snapshot + plan_step) and of the scenario/LiDAR generator and the
// closed-loop driver that feed it.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it, and only as the
// checker or the timed CPU baseline.  The product path never links it.
//
// Parity status: pinned against every known-answer test the reference's own
// suites hold for this path (oracle/kat_runner.cpp ports them, tests/
// test_oracle_kat.py runs it).  The reference itself cannot be compiled here
// (Eigen3 and vendor/ are absent), so bit-level Eigen operation
// order is fixed by convention:
//   * Vec3 squared norm  = (x*x + y*y) + z*z
//   * quaternion squared norm = ((x*x + y*y) + z*z) + w*w   (Eigen storage order)
//   * matrix * vector row  = (m0*v0 + m1*v1) + m2*v2
//   * Frobenius norm       = sequential over column-major storage
//   * no FMA contraction (-ffp-contract=off), glibc libm transcendentals.
//
// Every function cites the reference file:line it restates (paths relative
// to the reference's proj/ directory).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <functional>
#include <limits>
#include <numbers>
#include <span>
#include <string>
#include <vector>

namespace oracle {

constexpr double kPi = std::numbers::pi;
constexpr double kInf = std::numeric_limits<double>::infinity();

// ---------------------------------------------------------------------------
// small linear algebra with the fixed operation order above
// ---------------------------------------------------------------------------
struct Vec3 {
  double x{0}, y{0}, z{0};
  constexpr Vec3() = default;
  constexpr Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double squared_norm() const { return (x * x + y * y) + z * z; }
  double norm() const { return std::sqrt(squared_norm()); }
  bool finite() const { return std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
  Vec3 normalized() const {
    const double n2 = squared_norm();
    if (!(n2 > 0.0)) return *this;
    const double n = std::sqrt(n2);
    return {x / n, y / n, z / n};
  }
  double dot(const Vec3& o) const { return (x * o.x + y * o.y) + z * o.z; }
  Vec3 cross(const Vec3& o) const {
    return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x};
  }
  double max_coeff() const { return std::max(std::max(x, y), z); }
  static constexpr Vec3 unit_x() { return {1, 0, 0}; }
  static constexpr Vec3 unit_z() { return {0, 0, 1}; }
};
inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline Vec3 operator*(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline Vec3 cwise_min(const Vec3& a, const Vec3& b) {
  return {std::min(a.x, b.x), std::min(a.y, b.y), std::min(a.z, b.z)};
}
inline Vec3 cwise_max(const Vec3& a, const Vec3& b) {
  return {std::max(a.x, b.x), std::max(a.y, b.y), std::max(a.z, b.z)};
}

// (w, x, y, z) as a plain 4-vector; also used for ControlInput::vec().
struct Vec4 {
  double v[4]{0, 0, 0, 0};
  constexpr Vec4() = default;
  constexpr Vec4(double a, double b, double c, double d) : v{a, b, c, d} {}
  double operator[](int i) const { return v[i]; }
  double& operator[](int i) { return v[i]; }
  double squared_norm() const { return ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]) + v[3] * v[3]; }
  double norm() const { return std::sqrt(squared_norm()); }
  static Vec4 zero() { return {}; }
};
inline Vec4 operator+(const Vec4& a, const Vec4& b) {
  return {a[0] + b[0], a[1] + b[1], a[2] + b[2], a[3] + b[3]};
}
inline Vec4 operator-(const Vec4& a, const Vec4& b) {
  return {a[0] - b[0], a[1] - b[1], a[2] - b[2], a[3] - b[3]};
}
inline Vec4 operator*(double s, const Vec4& a) { return {s * a[0], s * a[1], s * a[2], s * a[3]}; }

struct Mat3 {
  double m[3][3]{{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // m[row][col]
  static Mat3 identity() {
    Mat3 r;
    r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
    return r;
  }
  Mat3 transpose() const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[j][i];
    return r;
  }
  Vec3 operator*(const Vec3& v) const {
    return {(m[0][0] * v.x + m[0][1] * v.y) + m[0][2] * v.z,
            (m[1][0] * v.x + m[1][1] * v.y) + m[1][2] * v.z,
            (m[2][0] * v.x + m[2][1] * v.y) + m[2][2] * v.z};
  }
  Mat3 operator*(const Mat3& b) const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        r.m[i][j] = (m[i][0] * b.m[0][j] + m[i][1] * b.m[1][j]) + m[i][2] * b.m[2][j];
    return r;
  }
  // Frobenius norm, column-major sequential summation.
  double norm() const {
    double s = 0.0;
    bool first = true;
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) {
        const double e2 = m[i][j] * m[i][j];
        s = first ? e2 : s + e2;
        first = false;
      }
    return std::sqrt(s);
  }
};

// Unit quaternion, scalar-first in the API (types.hpp:13-14).
struct Quat {
  double w{1}, x{0}, y{0}, z{0};
  constexpr Quat() = default;
  constexpr Quat(double w_, double x_, double y_, double z_) : w(w_), x(x_), y(y_), z(z_) {}
  static Quat identity() { return {}; }
  // Eigen::AngleAxisd -> Quaterniond (half-angle construction).
  static Quat from_angle_axis(double angle, const Vec3& axis) {
    const double ha = 0.5 * angle;
    const double s = std::sin(ha);
    return {std::cos(ha), s * axis.x, s * axis.y, s * axis.z};
  }
  Vec3 vec() const { return {x, y, z}; }
  double squared_norm() const { return ((x * x + y * y) + z * z) + w * w; }
  double norm() const { return std::sqrt(squared_norm()); }
  Quat normalized() const {
    const double n2 = squared_norm();
    if (!(n2 > 0.0)) return *this;
    const double n = std::sqrt(n2);
    return {w / n, x / n, y / n, z / n};
  }
  void normalize() { *this = normalized(); }
  bool finite() const {
    return std::isfinite(w) && std::isfinite(x) && std::isfinite(y) && std::isfinite(z);
  }
  // Hamilton product, left-to-right evaluation (dynamics.hpp:18).
  Quat operator*(const Quat& b) const {
    return {w * b.w - x * b.x - y * b.y - z * b.z,
            w * b.x + x * b.w + y * b.z - z * b.y,
            w * b.y + y * b.w + z * b.x - x * b.z,
            w * b.z + z * b.w + x * b.y - y * b.x};
  }
  // Eigen _transformVector: uv = 2 (q.vec x v); v + w uv + q.vec x uv.
  Vec3 operator*(const Vec3& v) const {
    Vec3 uv = vec().cross(v);
    uv = uv + uv;
    return (v + w * uv) + vec().cross(uv);
  }
  // Eigen QuaternionBase::toRotationMatrix.
  Mat3 to_rotation_matrix() const {
    const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    Mat3 r;
    r.m[0][0] = 1.0 - (tyy + tzz);
    r.m[0][1] = txy - twz;
    r.m[0][2] = txz + twy;
    r.m[1][0] = txy + twz;
    r.m[1][1] = 1.0 - (txx + tzz);
    r.m[1][2] = tyz - twx;
    r.m[2][0] = txz - twy;
    r.m[2][1] = tyz + twx;
    r.m[2][2] = 1.0 - (txx + tyy);
    return r;
  }
};
inline Vec4 quat_vec(const Quat& q) { return {q.w, q.x, q.y, q.z}; }
inline Quat vec_quat(const Vec4& v) { return {v[0], v[1], v[2], v[3]}; }

// ---------------------------------------------------------------------------
// rng.hpp:10-66
// ---------------------------------------------------------------------------
constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ull;
constexpr std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

class RandomStream {
 public:
  explicit RandomStream(std::uint64_t key) : key_(mix64(key ^ kGamma)) {}
  static RandomStream derive(std::uint64_t seed, std::uint64_t a = 0, std::uint64_t b = 0,
                             std::uint64_t c = 0) {
    std::uint64_t k = mix64(seed + kGamma);
    k = mix64(k ^ (a + kGamma));
    k = mix64(k ^ (b + kGamma));
    k = mix64(k ^ (c + kGamma));
    return RandomStream(k);
  }
  std::uint64_t next_u64() { return mix64(key_ + (++counter_) * kGamma); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * kPi * u2;
    spare_ = r * std::sin(a);
    has_spare_ = true;
    return r * std::cos(a);
  }
  double normal(double mean, double stddev) { return mean + stddev * normal(); }

 private:
  std::uint64_t key_;
  std::uint64_t counter_ = 0;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ---------------------------------------------------------------------------
// types.hpp:18-59
// ---------------------------------------------------------------------------
struct State {
  Vec3 p{};
  Quat q{};
  Vec3 v{};
  bool finite() const { return p.finite() && v.finite() && q.finite(); }
};

struct ControlInput {
  double thrust{0.0};
  Vec3 omega{};
  Vec4 vec() const { return {thrust, omega.x, omega.y, omega.z}; }
  static ControlInput from_vec(const Vec4& u) { return {u[0], Vec3(u[1], u[2], u[3])}; }
  bool finite() const { return std::isfinite(thrust) && omega.finite(); }
};

struct DynamicsParams {
  double mass{1.0};
  Vec3 gravity{0.0, 0.0, -9.81};
  double dt{0.05};
  double thrust_min{0.3};
  double thrust_max{16.35};
  double omega_xy_max{3.0};
  double omega_z_max{2.0};
  ControlInput hover() const { return {mass * gravity.norm(), Vec3()}; }
};

struct StateDerivative {
  Vec3 dp{};
  Vec4 dq{};  // scalar-first
  Vec3 dv{};
};

// dynamics.hpp:13-78
StateDerivative derivative_raw(const State& x, const ControlInput& u, const DynamicsParams& prm);
State rk4_step_raw(const State& x, const ControlInput& u, const DynamicsParams& prm);
StateDerivative state_derivative(const State& x, const ControlInput& u, const DynamicsParams& prm);
State rk4_step(const State& x, const ControlInput& u, const DynamicsParams& prm);
ControlInput clamp_control(const ControlInput& u, const DynamicsParams& prm);

// ---------------------------------------------------------------------------
// parallel.hpp / parallel.cpp:14-63
// ---------------------------------------------------------------------------
void set_worker_count(unsigned n);
unsigned worker_count();
void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn);

// ---------------------------------------------------------------------------
// perception.hpp:12-143, perception.cpp
// ---------------------------------------------------------------------------
constexpr int kAzimuthCells = 120;
constexpr int kElevationCells = 60;
constexpr int kPoolFactor = 6;
constexpr int kCoarseAzimuthCells = kAzimuthCells / kPoolFactor;
constexpr int kCoarseElevationCells = kElevationCells / kPoolFactor;
constexpr int kCells = kAzimuthCells * kElevationCells;
constexpr int kCoarseCells = kCoarseAzimuthCells * kCoarseElevationCells;
constexpr double kMinPointRange = 0.05;
constexpr double kHorizonReach = 25.0;
constexpr double kAzStep = 2.0 * kPi / kAzimuthCells;
constexpr double kElStep = kPi / kElevationCells;

Vec3 direction_from_angles(double azimuth, double elevation);
int azimuth_cell(double azimuth);
int elevation_cell(double elevation);
int coarse_azimuth_cell(double azimuth);
int coarse_elevation_cell(double elevation);
Vec3 cell_direction(int i, int j);  // throws std::out_of_range

class PointCloudBuffer {
 public:
  explicit PointCloudBuffer(std::size_t capacity = 10) : capacity_(capacity) {}
  void push(std::vector<Vec3> world_frame_points);
  std::size_t frames() const { return frames_.size(); }
  std::size_t capacity() const { return capacity_; }
  std::size_t total_points() const;
  std::vector<Vec3> body_points(const State& pose) const;
  std::vector<Vec3> all_points() const;  // world frame, oldest frame first

 private:
  std::deque<std::vector<Vec3>> frames_;
  std::size_t capacity_;
};

struct SphericalPartition {
  double r_max{10.0};
  std::vector<double> ranges;            // flat(i, j), empty cells = r_max
  std::vector<Vec3> nearest;             // body frame
  std::vector<std::uint8_t> has_point;
  static int flat(int i, int j) { return i * kElevationCells + j; }
  double range(int i, int j) const { return ranges[flat(i, j)]; }
  double& range(int i, int j) { return ranges[flat(i, j)]; }
};

struct CoarsePartition {
  double r_max{10.0};
  std::vector<double> safe_range;  // flat(I, J)
  std::vector<Vec3> safe_dir;
  std::vector<Vec3> safe_point;
  static int flat(int I, int J) { return I * kCoarseElevationCells + J; }
};

struct FilteredCloud {
  enum class Frame { body, world };
  Frame frame{Frame::body};
  double r_max{10.0};
  std::vector<Vec3> points;
  double far_clearance() const { return r_max + kHorizonReach; }
};

SphericalPartition build_partition(const std::vector<Vec3>& body_cloud, double r_max = 10.0);
CoarsePartition pool_coarse(const SphericalPartition& part);
FilteredCloud filtered_cloud(const SphericalPartition& part);
FilteredCloud to_world_frame(const FilteredCloud& fc, const State& pose);
double clearance(const FilteredCloud& fc, const Vec3& p);

class ClearanceIndex {
 public:
  ClearanceIndex() = default;
  explicit ClearanceIndex(const FilteredCloud& fc, double cell_size = 1.0);
  double nearest(const Vec3& p) const;
  bool empty() const { return points_.empty(); }
  double far_clearance() const { return far_; }

 private:
  int cell_of(const Vec3& p, int axis) const;
  double cell_{1.0};
  double far_{35.0};
  Vec3 origin_{};
  int dims_[3]{0, 0, 0};
  std::vector<std::int32_t> cell_start_;
  std::vector<Vec3> points_;
};

struct PerceptionSnapshot {
  State pose;
  SphericalPartition partition;
  CoarsePartition coarse;
  FilteredCloud filtered;
  ClearanceIndex clearance_index;
};

PerceptionSnapshot build_snapshot(const PointCloudBuffer& buffer, const State& pose,
                                  double r_max = 10.0);
// Same, from an explicit world-frame point list (a one-frame buffer).
PerceptionSnapshot build_snapshot_points(const std::vector<Vec3>& world_points,
                                         const State& pose, double r_max = 10.0);

// ---------------------------------------------------------------------------
// guidance.hpp:10-75, guidance.cpp
// ---------------------------------------------------------------------------
struct AnchorGrid {
  int m_h{5};
  int m_v{3};
  double lookahead{5.0};
  double spacing_deg{18.0};
  double terminal_speed{3.0};
  double min_anchor_distance{0.5};
  int count() const { return m_h * m_v; }
};

struct Anchor {
  Vec3 initial_endpoint{};
  Vec3 refined_endpoint{};
  Vec3 safe_dir{1, 0, 0};
  double safe_range{0.0};
  int coarse_i{0};
  int coarse_j{0};
};

struct BoundaryCondition {
  Vec3 p{}, v{}, a{};
};

struct GuidingTrajectory {
  Vec3 coeffs[6]{};  // coeffs[k] = column k (per-axis coefficient of t^k)
  double horizon{0.0};
};

std::vector<Vec3> sample_initial_endpoints(const Vec3& p0, const Vec3& goal, const AnchorGrid& grid);
std::vector<Anchor> refine_endpoints(const std::vector<Vec3>& endpoints, const CoarsePartition& coarse,
                                     const State& pose, double lookahead, double obstacle_shell,
                                     double min_distance = 0.5);
GuidingTrajectory solve_quintic(const BoundaryCondition& start, const BoundaryCondition& end,
                                double horizon);
Vec3 eval_guide(const GuidingTrajectory& g, double t);
Vec3 eval_guide_velocity(const GuidingTrajectory& g, double t);
Vec3 eval_guide_acceleration(const GuidingTrajectory& g, double t);
std::vector<GuidingTrajectory> build_guides(const std::vector<Anchor>& anchors, const State& x,
                                            const ControlInput& last_control,
                                            const DynamicsParams& prm, double terminal_speed,
                                            double horizon);

// ---------------------------------------------------------------------------
// costs.hpp:13-187
// ---------------------------------------------------------------------------
struct CollisionParams {
  double scale{1.0e6};
  double slope{5.0};
  double d_min{0.4};
  double d_max{1.0};
};

struct CostWeights {
  double q_track{15.0};
  double q_vnorm{0.15};
  double q_c{0.5};
  double q_c_delta{0.5};
  double q_p{3.0};
  double q_v{0.25};
  double q_q{1.0};
  CollisionParams collision;
};

struct Rollout {
  std::vector<State> states;
  std::vector<ControlInput> controls;
  const GuidingTrajectory* guide{nullptr};
  double dt{0.05};
  bool valid{true};
  int horizon() const { return static_cast<int>(controls.size()); }
};

struct GoalSpec {
  Vec3 p_goal{};
  Vec3 v_goal{};
  Quat q_goal{};
  static GoalSpec facing(const Vec3& from, const Vec3& target);
};

double tracking_cost(const Rollout& r, const CostWeights& w);
double vnorm_cost(const Rollout& r, const CostWeights& w);
double control_cost(const Rollout& r, const CostWeights& w, const ControlInput& u_prev);
double goal_cost(const Rollout& r, const GoalSpec& goal, const CostWeights& w);
double collision_term(double d, const CostWeights& w);
double collision_cost(const Rollout& r, const FilteredCloud& filtered, const CostWeights& w);
double collision_cost(const Rollout& r, const ClearanceIndex& index, const CostWeights& w);
double stage2_cost(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                   const CostWeights& w);
double stage2_cost(const Rollout& r, const GoalSpec& goal, const FilteredCloud& filtered,
                   const CostWeights& w);
double stage1_cost(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                   const CostWeights& w, const ControlInput& u_prev);
double stage1_cost(const Rollout& r, const GoalSpec& goal, const FilteredCloud& filtered,
                   const CostWeights& w, const ControlInput& u_prev);

struct CostBreakdown {
  double track{0}, vnorm{0}, ctrl{0}, goal{0}, collision{0};
  double stage2() const { return goal + collision; }
  double stage1() const { return track + vnorm + ctrl + stage2(); }
};
CostBreakdown cost_breakdown(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                             const CostWeights& w, const ControlInput& u_prev);

// ---------------------------------------------------------------------------
// mppi.hpp:14-128, mppi.cpp
// ---------------------------------------------------------------------------
struct MppiConfig {
  int rollouts{128};
  int horizon{25};
  double lambda{0.1};
  Vec4 sigma{1.0, 1.0, 1.0, 0.5};
  double dt{0.05};
  int iterations{1};
};

struct NominalSequence {
  std::vector<ControlInput> controls;
  static NominalSequence constant(const ControlInput& u, int horizon) {
    NominalSequence n;
    n.controls.assign(horizon, u);
    return n;
  }
};

struct StreamKey {
  std::uint64_t seed{0}, instance{0}, cycle{0};
};

struct RolloutBatch {
  std::vector<Vec4> perturbations;
  std::vector<Rollout> trajectories;
  std::vector<double> costs;
  std::vector<double> weights;
  void resize(const MppiConfig& cfg);
};

void sample_rollout_perturbations(const MppiConfig& cfg, const StreamKey& key, int k,
                                  std::span<Vec4> out);
std::vector<Vec4> sample_perturbations(const MppiConfig& cfg, const StreamKey& key);
void rollout_into(Rollout& r, const State& x0, const NominalSequence& nominal,
                  std::span<Vec4> delta, const DynamicsParams& prm);
Rollout rollout(const State& x0, const NominalSequence& nominal, std::span<Vec4> delta,
                const DynamicsParams& prm);
std::vector<double> compute_weights(const std::vector<double>& costs, double lambda);
void update_nominal(NominalSequence& nominal, std::span<const Vec4> deltas,
                    const std::vector<double>& weights, const DynamicsParams& prm);
NominalSequence shift_nominal(const NominalSequence& nominal);

struct MppiDiagnostics {
  double min_cost{0}, mean_cost{0}, ess{0};
};

MppiDiagnostics mppi_step(NominalSequence& nominal, const State& x0, const MppiConfig& cfg,
                          const DynamicsParams& prm, const StreamKey& key,
                          const std::function<double(const Rollout&)>& cost, RolloutBatch& batch);

// ---------------------------------------------------------------------------
// ensemble.hpp:16-69, ensemble.cpp:19-179
// ---------------------------------------------------------------------------
struct EnsembleConfig {
  AnchorGrid grid;
  MppiConfig mppi;
  CostWeights weights;
  DynamicsParams dynamics;
  double replan_hz{50.0};
  double r_max{10.0};
};

struct InstanceRecord {
  double stage1{0.0};
  double stage2{0.0};
  double ess{0.0};
  bool valid{false};
  NominalSequence nominal;
};

struct PlanResult {
  int winner{-1};
  ControlInput control;
  Rollout winner_rollout;
  std::vector<InstanceRecord> per_instance;
  std::vector<Anchor> anchors;
  std::vector<GuidingTrajectory> guides;
  CostBreakdown breakdown;
};

struct PlanScratch {
  std::vector<Vec4> perturbations;
  std::vector<Rollout> trajectories;
  std::vector<double> costs;
  std::vector<double> slice_weights;
  std::vector<Vec4> zero_deltas;
  std::vector<Rollout> re_rollouts;
  void resize(int instances, const MppiConfig& cfg);
};

// Verification hooks (not part of the reference interface): per-sample
// stage-I costs of the last iteration, and host-injected perturbations that
// replace the RNG draws ([iteration][m][k][j] rows).
struct PlanDebug {
  const std::vector<Vec4>* injected_delta{nullptr};
  std::vector<double> stage1_costs;     // M*K, last iteration
  std::vector<double> collision_margin; // M*K: min over costed steps of |d - d_min|, |d - d_max|
};

PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                     const EnsembleConfig& cfg, const NominalSequence& previous,
                     const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed,
                     PlanScratch& scratch, PlanDebug* debug = nullptr);
PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                     const EnsembleConfig& cfg, const NominalSequence& previous,
                     const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed);

// ---------------------------------------------------------------------------
// sim_world.hpp / sim_world.cpp (input generator for the oracle's own loops)
// ---------------------------------------------------------------------------
enum class PrimitiveKind { vertical_cylinder, tilted_cylinder, box };

struct ObstaclePrimitive {
  PrimitiveKind kind{PrimitiveKind::vertical_cylinder};
  Vec3 base{};
  double radius{0.5};
  double height{6.0};
  Vec3 half_extents{1, 1, 1};
  Vec3 tilt_axis{1, 0, 0};
  double tilt_angle{0.0};
  Quat rotation() const;
};

struct Scenario {
  std::string kind{"empty"};
  std::uint64_t seed{0};
  Vec3 placement_min{2.5, -20.0, 0.0};
  Vec3 placement_max{42.5, 20.0, 0.0};
  Vec3 start{0.0, 0.0, 2.0};
  Vec3 goal{45.0, 0.0, 2.0};
  std::vector<ObstaclePrimitive> obstacles;
};

enum class ScenarioKind { empty = 0, forest = 1, verticals = 2, inclines = 3, two_gap = 4 };

struct CylinderFieldParams {
  int count{0};
  double radius_min{0.4}, radius_max{1.1};
  double height_min{6.0}, height_max{6.0};
  double tilt_max{0.0};
};

Scenario generate_cylinder_field(const CylinderFieldParams& params, std::uint64_t seed,
                                 const std::string& label);
Scenario generate_scenario(ScenarioKind kind, std::uint64_t seed);
double surface_distance(const ObstaclePrimitive& prim, const Vec3& p);
double true_clearance(const Scenario& scene, const Vec3& p);
bool check_collision(const Scenario& scene, const Vec3& p, double drone_radius = 0.2);
double ray_hit(const ObstaclePrimitive& prim, const Vec3& origin, const Vec3& dir, double t_max);

struct LidarModel {
  double r_max{10.0};
  double elevation_min_deg{-45.0};
  double elevation_max_deg{45.0};
  double range_sigma{0.01};
};

std::vector<Vec3> lidar_scan(const Scenario& scene, const State& pose, const LidarModel& model,
                             std::uint64_t frame_seed);

// ---------------------------------------------------------------------------
// closed-loop driver: ensemble.cpp:238-305, metrics.cpp:74-81
// ---------------------------------------------------------------------------
enum class EpisodeStatus { running, success, collision, timeout, planner_failure };

struct World {
  Scenario scene;
  LidarModel lidar;
};

struct EpisodeParams {
  double goal_radius{1.0};
  double timeout{60.0};
  double drone_radius{0.2};
  int max_planner_failures{50};
};

// One recorded cycle of the loop: the exact inputs plan_step saw, plus its
// outputs, so a device planner can replay the cycle.
struct CycleRecord {
  std::vector<Vec3> cloud;      // buffer contents, oldest frame first (world)
  State x;
  NominalSequence previous;
  ControlInput last_applied;
  std::uint64_t cycle{0};
  bool planned{false};           // false -> "planning failed"
  int winner{-1};
  ControlInput control;
  double stage2{kInf};
  NominalSequence winner_nominal;
};

struct EpisodeState {
  State x;
  PointCloudBuffer buffer{10};
  NominalSequence nominal;
  ControlInput last_applied;
  std::uint64_t cycle{0};
  double t{0.0};
  int consecutive_failures{0};
  EpisodeStatus status{EpisodeStatus::running};
  std::vector<CycleRecord>* recorder{nullptr};
};

EpisodeState make_episode_state(const World& world, const EnsembleConfig& cfg);
void execute_cycle(EpisodeState& es, const World& world, const GoalSpec& goal,
                   const EnsembleConfig& cfg, const EpisodeParams& params, std::uint64_t seed,
                   PlanScratch& scratch);
EnsembleConfig apply_velocity_cap(const EnsembleConfig& cfg, double cap);

}  // namespace oracle
