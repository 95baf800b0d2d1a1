// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/include/amppi/dynamics.hpp, proj/src/{parallel,perception,
// guidance,mppi,ensemble}.cpp and proj/include/amppi/costs.hpp.
#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <thread>

namespace oracle {

// ===========================================================================
// dynamics.hpp:13-78
// ===========================================================================
StateDerivative derivative_raw(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  StateDerivative d;
  d.dp = x.v;
  const Quat omega_q(0.0, u.omega.x, u.omega.y, u.omega.z);
  const Quat qdot = x.q * omega_q;                 // dynamics.hpp:18
  d.dq = 0.5 * quat_vec(qdot);                     // dynamics.hpp:19
  const Vec3 thrust_dir = x.q.normalized() * Vec3::unit_z();
  d.dv = (u.thrust / prm.mass) * thrust_dir + prm.gravity;  // dynamics.hpp:20
  return d;
}

State rk4_step_raw(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  const double dt = prm.dt;
  auto advance = [](const State& s, const StateDerivative& d, double h) {
    State out;
    out.p = s.p + h * d.dp;
    out.v = s.v + h * d.dv;
    out.q = vec_quat(quat_vec(s.q) + h * d.dq);
    return out;
  };
  const StateDerivative k1 = derivative_raw(x, u, prm);
  const StateDerivative k2 = derivative_raw(advance(x, k1, 0.5 * dt), u, prm);
  const StateDerivative k3 = derivative_raw(advance(x, k2, 0.5 * dt), u, prm);
  const StateDerivative k4 = derivative_raw(advance(x, k3, dt), u, prm);
  const double h6 = dt / 6.0;
  State next;
  next.p = x.p + h6 * (((k1.dp + 2.0 * k2.dp) + 2.0 * k3.dp) + k4.dp);
  next.v = x.v + h6 * (((k1.dv + 2.0 * k2.dv) + 2.0 * k3.dv) + k4.dv);
  next.q = vec_quat(quat_vec(x.q) + h6 * (((k1.dq + 2.0 * k2.dq) + 2.0 * k3.dq) + k4.dq));
  return next;
}

StateDerivative state_derivative(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  if (!x.finite() || !u.finite()) throw std::invalid_argument("invalid state");
  return derivative_raw(x, u, prm);
}

State rk4_step(const State& x, const ControlInput& u, const DynamicsParams& prm) {
  if (!x.finite() || !u.finite()) throw std::invalid_argument("invalid state");
  State next = rk4_step_raw(x, u, prm);
  next.q.normalize();
  return next;
}

ControlInput clamp_control(const ControlInput& u, const DynamicsParams& prm) {
  ControlInput c;
  c.thrust = std::clamp(u.thrust, prm.thrust_min, prm.thrust_max);
  c.omega.x = std::clamp(u.omega.x, -prm.omega_xy_max, prm.omega_xy_max);
  c.omega.y = std::clamp(u.omega.y, -prm.omega_xy_max, prm.omega_xy_max);
  c.omega.z = std::clamp(u.omega.z, -prm.omega_z_max, prm.omega_z_max);
  return c;
}

// ===========================================================================
// parallel.cpp:14-63 — fresh threads per call, static chunks, nested calls
// serial, first exception rethrown.
// ===========================================================================
namespace {
std::atomic<unsigned> g_workers{0};
thread_local bool t_inside_parallel = false;
}  // namespace

void set_worker_count(unsigned n) { g_workers.store(n, std::memory_order_relaxed); }

unsigned worker_count() {
  unsigned n = g_workers.load(std::memory_order_relaxed);
  if (n == 0) {
    n = std::thread::hardware_concurrency();
    if (n == 0) n = 1;
  }
  return n;
}

void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn) {
  if (n == 0) return;
  const std::size_t workers = t_inside_parallel ? 1 : std::min<std::size_t>(worker_count(), n);
  if (workers <= 1) {
    fn(0, n);
    return;
  }
  const std::size_t chunk = (n + workers - 1) / workers;
  std::exception_ptr error;
  std::mutex error_mutex;
  auto run = [&](std::size_t begin, std::size_t end) {
    t_inside_parallel = true;
    try {
      fn(begin, end);
    } catch (...) {
      std::lock_guard<std::mutex> lock(error_mutex);
      if (!error) error = std::current_exception();
    }
    t_inside_parallel = false;
  };
  std::vector<std::thread> pool;
  pool.reserve(workers - 1);
  for (std::size_t w = 1; w < workers; ++w) {
    const std::size_t begin = w * chunk;
    const std::size_t end = std::min(n, begin + chunk);
    if (begin >= end) break;
    pool.emplace_back(run, begin, end);
  }
  run(0, std::min(n, chunk));
  for (auto& t : pool) t.join();
  if (error) std::rethrow_exception(error);
}

// ===========================================================================
// perception.cpp
// ===========================================================================
Vec3 direction_from_angles(double azimuth, double elevation) {  // perception.hpp:27-31
  const double ce = std::cos(elevation);
  return {ce * std::cos(azimuth), ce * std::sin(azimuth), std::sin(elevation)};
}

int azimuth_cell(double azimuth) {  // perception.cpp:17-21
  int i = static_cast<int>(std::floor((azimuth + kPi) / kAzStep));
  if (i >= kAzimuthCells) i -= kAzimuthCells;
  return std::clamp(i, 0, kAzimuthCells - 1);
}

int elevation_cell(double elevation) {  // perception.cpp:23-26
  int j = static_cast<int>(std::floor((elevation + 0.5 * kPi) / kElStep));
  return std::clamp(j, 0, kElevationCells - 1);
}

int coarse_azimuth_cell(double azimuth) { return azimuth_cell(azimuth) / kPoolFactor; }
int coarse_elevation_cell(double elevation) { return elevation_cell(elevation) / kPoolFactor; }

Vec3 cell_direction(int i, int j) {  // perception.cpp:36-42
  if (i < 0 || i >= kAzimuthCells || j < 0 || j >= kElevationCells)
    throw std::out_of_range("cell index out of range");
  const double az = -kPi + (i + 0.5) * kAzStep;
  const double el = -0.5 * kPi + (j + 0.5) * kElStep;
  return direction_from_angles(az, el);
}

void PointCloudBuffer::push(std::vector<Vec3> world_frame_points) {  // perception.cpp:44-47
  frames_.push_back(std::move(world_frame_points));
  while (frames_.size() > capacity_) frames_.pop_front();
}

std::size_t PointCloudBuffer::total_points() const {
  std::size_t n = 0;
  for (const auto& f : frames_) n += f.size();
  return n;
}

std::vector<Vec3> PointCloudBuffer::body_points(const State& pose) const {  // perception.cpp:55-62
  std::vector<Vec3> out;
  out.reserve(total_points());
  const Mat3 world_to_body = pose.q.to_rotation_matrix().transpose();
  for (const auto& frame : frames_)
    for (const auto& p : frame) out.push_back(world_to_body * (p - pose.p));
  return out;
}

std::vector<Vec3> PointCloudBuffer::all_points() const {
  std::vector<Vec3> out;
  out.reserve(total_points());
  for (const auto& frame : frames_) out.insert(out.end(), frame.begin(), frame.end());
  return out;
}

SphericalPartition build_partition(const std::vector<Vec3>& body_cloud, double r_max) {
  // perception.cpp:64-89: strict < keeps the first point on exact range ties;
  // a point at exactly r_max still occupies its cell.
  SphericalPartition part;
  part.r_max = r_max;
  part.ranges.assign(kCells, r_max);
  part.nearest.assign(kCells, Vec3());
  part.has_point.assign(kCells, 0);
  for (const auto& p : body_cloud) {
    const double r = p.norm();
    if (!(r > kMinPointRange) || r > r_max) continue;
    const double az = std::atan2(p.y, p.x);
    const double el = std::atan2(p.z, std::sqrt(p.x * p.x + p.y * p.y));
    const int i = azimuth_cell(az);
    const int j = elevation_cell(el);
    const int f = SphericalPartition::flat(i, j);
    if (!part.has_point[f] || r < part.ranges[f]) {
      if (r < part.ranges[f]) part.ranges[f] = r;
      part.nearest[f] = p;
      part.has_point[f] = 1;
    }
  }
  return part;
}

CoarsePartition pool_coarse(const SphericalPartition& part) {  // perception.cpp:91-122
  CoarsePartition coarse;
  coarse.r_max = part.r_max;
  coarse.safe_range.assign(kCoarseCells, 0.0);
  coarse.safe_dir.assign(kCoarseCells, Vec3());
  coarse.safe_point.assign(kCoarseCells, Vec3());
  for (int I = 0; I < kCoarseAzimuthCells; ++I) {
    for (int J = 0; J < kCoarseElevationCells; ++J) {
      int best_i = I * kPoolFactor, best_j = J * kPoolFactor;
      double best_r = -1.0;
      for (int i = I * kPoolFactor; i < (I + 1) * kPoolFactor; ++i)
        for (int j = J * kPoolFactor; j < (J + 1) * kPoolFactor; ++j)
          if (part.range(i, j) > best_r) {
            best_r = part.range(i, j);
            best_i = i;
            best_j = j;
          }
      const int f = CoarsePartition::flat(I, J);
      coarse.safe_range[f] = best_r;
      coarse.safe_dir[f] = cell_direction(best_i, best_j);
      coarse.safe_point[f] = best_r * coarse.safe_dir[f];
    }
  }
  return coarse;
}

FilteredCloud filtered_cloud(const SphericalPartition& part) {  // perception.cpp:124-133
  FilteredCloud fc;
  fc.frame = FilteredCloud::Frame::body;
  fc.r_max = part.r_max;
  for (int f = 0; f < kCells; ++f)
    if (part.has_point[f]) fc.points.push_back(part.nearest[f]);
  return fc;
}

FilteredCloud to_world_frame(const FilteredCloud& fc, const State& pose) {  // perception.cpp:135-144
  if (fc.frame == FilteredCloud::Frame::world) return fc;
  FilteredCloud out;
  out.frame = FilteredCloud::Frame::world;
  out.r_max = fc.r_max;
  out.points.reserve(fc.points.size());
  const Mat3 body_to_world = pose.q.to_rotation_matrix();
  for (const auto& p : fc.points) out.points.push_back(pose.p + body_to_world * p);
  return out;
}

double clearance(const FilteredCloud& fc, const Vec3& p) {  // perception.cpp:146-151
  if (fc.points.empty()) return fc.far_clearance();
  double best2 = kInf;
  for (const auto& q : fc.points) best2 = std::min(best2, (p - q).squared_norm());
  return std::sqrt(best2);
}

ClearanceIndex::ClearanceIndex(const FilteredCloud& fc, double cell_size) {  // perception.cpp:153-185
  far_ = fc.far_clearance();
  if (fc.points.empty()) return;
  Vec3 lo = fc.points.front(), hi = fc.points.front();
  for (const auto& p : fc.points) {
    lo = cwise_min(lo, p);
    hi = cwise_max(hi, p);
  }
  const Vec3 extent = hi - lo;
  cell_ = std::max(cell_size, extent.max_coeff() / 96.0);
  origin_ = lo;
  for (int a = 0; a < 3; ++a)
    dims_[a] = std::max(1, static_cast<int>(std::floor(extent[a] / cell_)) + 1);
  const int n_cells = dims_[0] * dims_[1] * dims_[2];
  std::vector<std::int32_t> counts(n_cells, 0);
  auto flat_cell = [&](const Vec3& p) {
    int c[3];
    for (int a = 0; a < 3; ++a)
      c[a] = std::clamp(static_cast<int>(std::floor((p[a] - origin_[a]) / cell_)), 0, dims_[a] - 1);
    return (c[0] * dims_[1] + c[1]) * dims_[2] + c[2];
  };
  for (const auto& p : fc.points) ++counts[flat_cell(p)];
  cell_start_.assign(n_cells + 1, 0);
  for (int c = 0; c < n_cells; ++c) cell_start_[c + 1] = cell_start_[c] + counts[c];
  points_.resize(fc.points.size());
  std::vector<std::int32_t> cursor(cell_start_.begin(), cell_start_.end() - 1);
  for (const auto& p : fc.points) points_[cursor[flat_cell(p)]++] = p;
}

int ClearanceIndex::cell_of(const Vec3& p, int axis) const {
  return static_cast<int>(std::floor((p[axis] - origin_[axis]) / cell_));
}

double ClearanceIndex::nearest(const Vec3& p) const {  // perception.cpp:191-235
  if (points_.empty()) return far_;
  const int c[3] = {cell_of(p, 0), cell_of(p, 1), cell_of(p, 2)};
  auto ring_to_box = [](int cc, int dim) { return std::max({0, -cc, cc - (dim - 1)}); };
  auto ring_from_box = [](int cc, int dim) { return std::max(std::abs(cc), std::abs(cc - (dim - 1))); };
  const int first_ring = std::max({ring_to_box(c[0], dims_[0]), ring_to_box(c[1], dims_[1]),
                                   ring_to_box(c[2], dims_[2])});
  const int last_ring = std::max({ring_from_box(c[0], dims_[0]), ring_from_box(c[1], dims_[1]),
                                  ring_from_box(c[2], dims_[2])});
  double best2 = kInf;
  for (int r = first_ring; r <= last_ring; ++r) {
    if (r > first_ring) {
      const double bound = (r - 1) * cell_;
      if (best2 <= bound * bound) break;
    }
    const int x0 = std::max(c[0] - r, 0), x1 = std::min(c[0] + r, dims_[0] - 1);
    const int y0 = std::max(c[1] - r, 0), y1 = std::min(c[1] + r, dims_[1] - 1);
    const int z0 = std::max(c[2] - r, 0), z1 = std::min(c[2] + r, dims_[2] - 1);
    for (int x = x0; x <= x1; ++x)
      for (int y = y0; y <= y1; ++y) {
        const bool face_xy = (std::abs(x - c[0]) == r) || (std::abs(y - c[1]) == r);
        for (int z = z0; z <= z1; ++z) {
          if (!face_xy && std::abs(z - c[2]) != r) continue;
          const int cell = (x * dims_[1] + y) * dims_[2] + z;
          for (std::int32_t k = cell_start_[cell]; k < cell_start_[cell + 1]; ++k)
            best2 = std::min(best2, (p - points_[k]).squared_norm());
        }
      }
  }
  return std::sqrt(best2);
}

PerceptionSnapshot build_snapshot(const PointCloudBuffer& buffer, const State& pose, double r_max) {
  // perception.cpp:237-246
  PerceptionSnapshot snap;
  snap.pose = pose;
  snap.partition = build_partition(buffer.body_points(pose), r_max);
  snap.coarse = pool_coarse(snap.partition);
  snap.filtered = to_world_frame(filtered_cloud(snap.partition), pose);
  snap.clearance_index = ClearanceIndex(snap.filtered);
  return snap;
}

PerceptionSnapshot build_snapshot_points(const std::vector<Vec3>& world_points, const State& pose,
                                         double r_max) {
  PointCloudBuffer buf(1);
  buf.push(world_points);
  return build_snapshot(buf, pose, r_max);
}

// ===========================================================================
// guidance.cpp
// ===========================================================================
namespace {
constexpr double kMaxElevation = 89.0 * kPi / 180.0;
}

std::vector<Vec3> sample_initial_endpoints(const Vec3& p0, const Vec3& goal, const AnchorGrid& grid) {
  // guidance.cpp:16-38: index v*m_h + h (v outer, h inner)
  const Vec3 to_goal = goal - p0;
  const double dist = to_goal.norm();
  if (!(dist > 1e-9)) throw std::invalid_argument("degenerate goal direction");
  const double az0 = std::atan2(to_goal.y, to_goal.x);
  const double el0 = std::atan2(to_goal.z, std::sqrt(to_goal.x * to_goal.x + to_goal.y * to_goal.y));
  const double spacing = grid.spacing_deg * kPi / 180.0;
  std::vector<Vec3> endpoints;
  endpoints.reserve(grid.count());
  for (int v = 0; v < grid.m_v; ++v) {
    const double el_off = (v - 0.5 * (grid.m_v - 1)) * spacing;
    const double el = std::clamp(el0 + el_off, -kMaxElevation, kMaxElevation);
    for (int h = 0; h < grid.m_h; ++h) {
      const double az = az0 + (h - 0.5 * (grid.m_h - 1)) * spacing;
      endpoints.push_back(p0 + grid.lookahead * direction_from_angles(az, el));
    }
  }
  return endpoints;
}

std::vector<Anchor> refine_endpoints(const std::vector<Vec3>& endpoints, const CoarsePartition& coarse,
                                     const State& pose, double lookahead, double obstacle_shell,
                                     double min_distance) {
  // guidance.cpp:40-72
  std::vector<Anchor> anchors;
  anchors.reserve(endpoints.size());
  const Mat3 body_to_world = pose.q.to_rotation_matrix();
  const Mat3 world_to_body = body_to_world.transpose();
  for (const auto& endpoint : endpoints) {
    Vec3 dir_world = endpoint - pose.p;
    if (dir_world.squared_norm() < 1e-18) dir_world = Vec3::unit_x();
    const Vec3 dir_body = world_to_body * dir_world.normalized();
    const double az = std::atan2(dir_body.y, dir_body.x);
    const double el = std::atan2(dir_body.z, std::sqrt(dir_body.x * dir_body.x + dir_body.y * dir_body.y));
    Anchor a;
    a.initial_endpoint = endpoint;
    a.coarse_i = coarse_azimuth_cell(az);
    a.coarse_j = coarse_elevation_cell(el);
    const int f = CoarsePartition::flat(a.coarse_i, a.coarse_j);
    a.safe_range = coarse.safe_range[f];
    a.safe_dir = body_to_world * coarse.safe_dir[f];
    const double reach = std::min(lookahead, std::max(a.safe_range - obstacle_shell, min_distance));
    a.refined_endpoint = pose.p + reach * a.safe_dir;
    anchors.push_back(a);
  }
  return anchors;
}

GuidingTrajectory solve_quintic(const BoundaryCondition& start, const BoundaryCondition& end,
                                double horizon) {
  // guidance.cpp:74-94
  if (!(horizon > 0.0)) throw std::invalid_argument("horizon must be positive");
  const double T = horizon;
  const double T2 = T * T, T3 = T2 * T, T4 = T3 * T, T5 = T4 * T;
  const Vec3 dp = end.p - ((start.p + start.v * T) + (0.5 * start.a) * T2);
  const Vec3 dv = end.v - (start.v + start.a * T);
  const Vec3 da = end.a - start.a;
  GuidingTrajectory g;
  g.horizon = T;
  g.coeffs[0] = start.p;
  g.coeffs[1] = start.v;
  g.coeffs[2] = 0.5 * start.a;
  g.coeffs[3] = ((20.0 * dp - (8.0 * T) * dv) + T2 * da) / (2.0 * T3);
  g.coeffs[4] = ((-30.0 * dp + (14.0 * T) * dv) - (2.0 * T2) * da) / (2.0 * T4);
  g.coeffs[5] = ((12.0 * dp - (6.0 * T) * dv) + T2 * da) / (2.0 * T5);
  return g;
}

Vec3 eval_guide(const GuidingTrajectory& g, double t) {  // guidance.cpp:96-101
  t = std::clamp(t, 0.0, g.horizon);
  Vec3 out = g.coeffs[5];
  for (int k = 4; k >= 0; --k) out = out * t + g.coeffs[k];
  return out;
}

Vec3 eval_guide_velocity(const GuidingTrajectory& g, double t) {
  t = std::clamp(t, 0.0, g.horizon);
  Vec3 out = 5.0 * g.coeffs[5];
  for (int k = 4; k >= 1; --k) out = out * t + static_cast<double>(k) * g.coeffs[k];
  return out;
}

Vec3 eval_guide_acceleration(const GuidingTrajectory& g, double t) {
  t = std::clamp(t, 0.0, g.horizon);
  Vec3 out = 20.0 * g.coeffs[5];
  out = out * t + 12.0 * g.coeffs[4];
  out = out * t + 6.0 * g.coeffs[3];
  out = out * t + 2.0 * g.coeffs[2];
  return out;
}

std::vector<GuidingTrajectory> build_guides(const std::vector<Anchor>& anchors, const State& x,
                                            const ControlInput& last_control,
                                            const DynamicsParams& prm, double terminal_speed,
                                            double horizon) {
  // guidance.cpp:119-140
  BoundaryCondition start;
  start.p = x.p;
  start.v = x.v;
  start.a = derivative_raw(x, clamp_control(last_control, prm), prm).dv;
  std::vector<GuidingTrajectory> guides;
  guides.reserve(anchors.size());
  for (const auto& anchor : anchors) {
    BoundaryCondition end;
    end.p = anchor.refined_endpoint;
    end.v = terminal_speed * anchor.safe_dir;
    end.a = Vec3();
    guides.push_back(solve_quintic(start, end, horizon));
  }
  return guides;
}

// ===========================================================================
// costs.hpp:42-187
// ===========================================================================
GoalSpec GoalSpec::facing(const Vec3& from, const Vec3& target) {  // costs.hpp:47-55
  GoalSpec g;
  g.p_goal = target;
  const Vec3 d = target - from;
  if (d.x * d.x + d.y * d.y > 1e-12)
    g.q_goal = Quat::from_angle_axis(std::atan2(d.y, d.x), Vec3::unit_z());
  return g;
}

double tracking_cost(const Rollout& r, const CostWeights& w) {  // costs.hpp:59-66
  if (r.guide == nullptr) return 0.0;
  double sum = 0.0;
  for (int t = 0; t < r.horizon(); ++t) sum += (r.states[t].p - eval_guide(*r.guide, t * r.dt)).norm();
  return w.q_track * sum;
}

double vnorm_cost(const Rollout& r, const CostWeights& w) {  // costs.hpp:69-74
  double sum = 0.0;
  for (int t = 0; t < r.horizon(); ++t) sum += r.states[t].v.squared_norm();
  return w.q_vnorm * sum;
}

double control_cost(const Rollout& r, const CostWeights& w, const ControlInput& u_prev) {
  // costs.hpp:80-92: u_{N-1} and u_prev do not enter the stated ranges
  (void)u_prev;
  double magnitude = 0.0, rate = 0.0;
  const int n = r.horizon();
  for (int t = 0; t + 1 < n; ++t) {
    magnitude += r.controls[t].vec().squared_norm();
    if (t >= 1) rate += (r.controls[t].vec() - r.controls[t - 1].vec()).squared_norm();
  }
  return w.q_c * magnitude + w.q_c_delta * rate;
}

double goal_cost(const Rollout& r, const GoalSpec& goal, const CostWeights& w) {  // costs.hpp:96-110
  const Mat3 goal_rot_t = goal.q_goal.to_rotation_matrix().transpose();
  const Mat3 eye = Mat3::identity();
  double sum = 0.0;
  for (int t = 0; t < r.horizon(); ++t) {
    const State& x = r.states[t];
    sum += w.q_p * (x.p - goal.p_goal).norm();
    sum += w.q_v * (x.v - goal.v_goal).norm();
    Mat3 err = x.q.to_rotation_matrix() * goal_rot_t;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) err.m[i][j] = err.m[i][j] - eye.m[i][j];
    sum += w.q_q * err.norm();
  }
  return sum;
}

double collision_term(double d, const CostWeights& w) {  // costs.hpp:113-118
  const CollisionParams& c = w.collision;
  if (d < c.d_min) return c.scale;
  if (d < c.d_max) return c.scale * std::exp(-c.slope * (d - c.d_min));
  return 0.0;
}

double collision_cost(const Rollout& r, const FilteredCloud& filtered, const CostWeights& w) {
  double sum = 0.0;
  for (int t = 0; t < r.horizon(); ++t) sum += collision_term(clearance(filtered, r.states[t].p), w);
  return sum;
}

double collision_cost(const Rollout& r, const ClearanceIndex& index, const CostWeights& w) {
  double sum = 0.0;
  for (int t = 0; t < r.horizon(); ++t) sum += collision_term(index.nearest(r.states[t].p), w);
  return sum;
}

double stage2_cost(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                   const CostWeights& w) {
  return goal_cost(r, goal, w) + collision_cost(r, index, w);
}

double stage2_cost(const Rollout& r, const GoalSpec& goal, const FilteredCloud& filtered,
                   const CostWeights& w) {
  return goal_cost(r, goal, w) + collision_cost(r, filtered, w);
}

double stage1_cost(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                   const CostWeights& w, const ControlInput& u_prev) {
  return ((tracking_cost(r, w) + vnorm_cost(r, w)) + control_cost(r, w, u_prev)) +
         stage2_cost(r, goal, index, w);
}

double stage1_cost(const Rollout& r, const GoalSpec& goal, const FilteredCloud& filtered,
                   const CostWeights& w, const ControlInput& u_prev) {
  return ((tracking_cost(r, w) + vnorm_cost(r, w)) + control_cost(r, w, u_prev)) +
         stage2_cost(r, goal, filtered, w);
}

CostBreakdown cost_breakdown(const Rollout& r, const GoalSpec& goal, const ClearanceIndex& index,
                             const CostWeights& w, const ControlInput& u_prev) {
  CostBreakdown b;
  b.track = tracking_cost(r, w);
  b.vnorm = vnorm_cost(r, w);
  b.ctrl = control_cost(r, w, u_prev);
  b.goal = goal_cost(r, goal, w);
  b.collision = collision_cost(r, index, w);
  return b;
}

// ===========================================================================
// mppi.cpp
// ===========================================================================
void RolloutBatch::resize(const MppiConfig& cfg) {
  perturbations.resize(static_cast<std::size_t>(cfg.rollouts) * cfg.horizon);
  trajectories.resize(cfg.rollouts);
  costs.resize(cfg.rollouts);
  weights.resize(cfg.rollouts);
}

void sample_rollout_perturbations(const MppiConfig& cfg, const StreamKey& key, int k,
                                  std::span<Vec4> out) {  // mppi.cpp:16-22
  RandomStream rs = RandomStream::derive(key.seed, key.instance, key.cycle, static_cast<std::uint64_t>(k));
  for (int j = 0; j < cfg.horizon; ++j)
    for (int c = 0; c < 4; ++c) out[j][c] = cfg.sigma[c] * rs.normal();
}

std::vector<Vec4> sample_perturbations(const MppiConfig& cfg, const StreamKey& key) {
  std::vector<Vec4> all(static_cast<std::size_t>(cfg.rollouts) * cfg.horizon);
  for (int k = 0; k < cfg.rollouts; ++k)
    sample_rollout_perturbations(cfg, key, k,
                                 std::span<Vec4>(all.data() + static_cast<std::size_t>(k) * cfg.horizon, cfg.horizon));
  return all;
}

void rollout_into(Rollout& r, const State& x0, const NominalSequence& nominal, std::span<Vec4> delta,
                  const DynamicsParams& prm) {  // mppi.cpp:33-61
  const int n = static_cast<int>(delta.size());
  r.dt = prm.dt;
  r.valid = true;
  r.states.resize(n + 1);
  r.controls.resize(n);
  r.states[0] = x0;
  for (int j = 0; j < n; ++j) {
    const Vec4 nominal_u = nominal.controls[j].vec();
    const ControlInput applied = clamp_control(ControlInput::from_vec(nominal_u + delta[j]), prm);
    delta[j] = applied.vec() - nominal_u;
    r.controls[j] = applied;
    State next = rk4_step_raw(r.states[j], applied, prm);
    next.q.normalize();
    if (!next.finite()) {
      r.valid = false;
      for (int rest = j; rest < n; ++rest) {
        r.states[rest + 1] = r.states[j];
        r.controls[rest] = applied;
      }
      return;
    }
    r.states[j + 1] = next;
  }
}

Rollout rollout(const State& x0, const NominalSequence& nominal, std::span<Vec4> delta,
                const DynamicsParams& prm) {
  Rollout r;
  rollout_into(r, x0, nominal, delta, prm);
  return r;
}

std::vector<double> compute_weights(const std::vector<double>& costs, double lambda) {
  // mppi.cpp:70-87
  double rho = kInf;
  for (double c : costs)
    if (std::isfinite(c)) rho = std::min(rho, c);
  if (!std::isfinite(rho)) throw std::runtime_error("no valid rollout");
  std::vector<double> weights(costs.size(), 0.0);
  double eta = 0.0;
  for (std::size_t k = 0; k < costs.size(); ++k)
    if (std::isfinite(costs[k])) {
      weights[k] = std::exp(-(costs[k] - rho) / lambda);
      eta += weights[k];
    }
  for (double& w : weights) w /= eta;
  return weights;
}

void update_nominal(NominalSequence& nominal, std::span<const Vec4> deltas,
                    const std::vector<double>& weights, const DynamicsParams& prm) {
  // mppi.cpp:89-101
  const int n = static_cast<int>(nominal.controls.size());
  const int k_count = static_cast<int>(weights.size());
  for (int j = 0; j < n; ++j) {
    Vec4 du = Vec4::zero();
    for (int k = 0; k < k_count; ++k)
      du = du + weights[k] * deltas[static_cast<std::size_t>(k) * n + j];
    nominal.controls[j] = clamp_control(ControlInput::from_vec(nominal.controls[j].vec() + du), prm);
  }
}

NominalSequence shift_nominal(const NominalSequence& nominal) {  // mppi.cpp:103-109
  NominalSequence out;
  if (nominal.controls.empty()) return out;
  out.controls.assign(nominal.controls.begin() + 1, nominal.controls.end());
  out.controls.push_back(nominal.controls.back());
  return out;
}

MppiDiagnostics mppi_step(NominalSequence& nominal, const State& x0, const MppiConfig& cfg,
                          const DynamicsParams& prm, const StreamKey& key,
                          const std::function<double(const Rollout&)>& cost, RolloutBatch& batch) {
  // mppi.hpp:92-128
  batch.resize(cfg);
  const int n = cfg.horizon;
  parallel_for(cfg.rollouts, [&](std::size_t begin, std::size_t end) {
    for (std::size_t k = begin; k < end; ++k) {
      std::span<Vec4> delta(batch.perturbations.data() + k * n, n);
      sample_rollout_perturbations(cfg, key, static_cast<int>(k), delta);
      rollout_into(batch.trajectories[k], x0, nominal, delta, prm);
      batch.costs[k] = batch.trajectories[k].valid ? cost(batch.trajectories[k]) : kInf;
    }
  });
  batch.weights = compute_weights(batch.costs, cfg.lambda);
  update_nominal(nominal, batch.perturbations, batch.weights, prm);
  MppiDiagnostics diag;
  diag.min_cost = kInf;
  double sum = 0.0, w2 = 0.0;
  int finite = 0;
  for (int k = 0; k < cfg.rollouts; ++k) {
    if (std::isfinite(batch.costs[k])) {
      diag.min_cost = std::min(diag.min_cost, batch.costs[k]);
      sum += batch.costs[k];
      ++finite;
    }
    w2 += batch.weights[k] * batch.weights[k];
  }
  diag.mean_cost = finite > 0 ? sum / finite : diag.min_cost;
  diag.ess = w2 > 0.0 ? 1.0 / w2 : 0.0;
  return diag;
}

// ===========================================================================
// ensemble.cpp:19-179
// ===========================================================================
void PlanScratch::resize(int instances, const MppiConfig& cfg) {
  const std::size_t mk = static_cast<std::size_t>(instances) * cfg.rollouts;
  perturbations.resize(mk * cfg.horizon);
  trajectories.resize(mk);
  costs.resize(mk);
  slice_weights.resize(cfg.rollouts);
  zero_deltas.resize(static_cast<std::size_t>(instances) * cfg.horizon);
  re_rollouts.resize(instances);
}

namespace {
// Verification-only: distance of the rollout's clearances from the collision
// branch boundaries (an FP32 device path may legitimately land on the other
// side of d_min / d_max when this margin is ~1e-6).
double collision_margin(const Rollout& r, const ClearanceIndex& index, const CostWeights& w) {
  double m = kInf;
  for (int t = 0; t < r.horizon(); ++t) {
    const double d = index.nearest(r.states[t].p);
    m = std::min(m, std::min(std::abs(d - w.collision.d_min), std::abs(d - w.collision.d_max)));
  }
  return m;
}
}  // namespace

PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                     const EnsembleConfig& cfg, const NominalSequence& previous,
                     const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed,
                     PlanScratch& scratch, PlanDebug* debug) {
  const int m_count = cfg.grid.count();
  const int k_count = cfg.mppi.rollouts;
  const int n = cfg.mppi.horizon;
  const double horizon_s = n * cfg.mppi.dt;
  scratch.resize(m_count, cfg.mppi);
  PlanResult result;

  // anchors and guides (ensemble.cpp:42-66)
  AnchorGrid grid = cfg.grid;
  const double goal_dist = (goal.p_goal - x.p).norm();
  if (goal_dist > grid.min_anchor_distance) {
    grid.lookahead = std::min(grid.lookahead, goal_dist);
    const double terminal_speed = std::min(grid.terminal_speed, goal_dist / horizon_s);
    result.anchors = refine_endpoints(sample_initial_endpoints(x.p, goal.p_goal, grid), snap.coarse,
                                      snap.pose, grid.lookahead, cfg.weights.collision.d_max,
                                      grid.min_anchor_distance);
    result.guides = build_guides(result.anchors, x, last_applied, cfg.dynamics, terminal_speed, horizon_s);
  } else {
    Anchor hold;
    hold.initial_endpoint = goal.p_goal;
    hold.refined_endpoint = goal.p_goal;
    hold.safe_dir = x.q * Vec3::unit_x();
    hold.safe_range = snap.partition.r_max;
    result.anchors.assign(m_count, hold);
    result.guides = build_guides(result.anchors, x, last_applied, cfg.dynamics, 0.0, horizon_s);
  }

  // warm start (ensemble.cpp:68-77)
  NominalSequence warm;
  if (static_cast<int>(previous.controls.size()) == n)
    warm = shift_nominal(previous);
  else
    warm = NominalSequence::constant(cfg.dynamics.hover(), n);

  result.per_instance.assign(m_count, InstanceRecord{});
  std::vector<NominalSequence> nominals(m_count, warm);
  std::vector<std::uint8_t> alive(m_count, 1);
  if (debug) {
    debug->stage1_costs.assign(static_cast<std::size_t>(m_count) * k_count, kInf);
    debug->collision_margin.assign(static_cast<std::size_t>(m_count) * k_count, kInf);
  }

  // stage I (ensemble.cpp:80-130)
  for (int iter = 0; iter < cfg.mppi.iterations; ++iter) {
    const std::uint64_t iter_cycle = cycle * static_cast<std::uint64_t>(cfg.mppi.iterations) + iter;
    const bool last_iter = iter + 1 == cfg.mppi.iterations;
    parallel_for(static_cast<std::size_t>(m_count) * k_count, [&](std::size_t begin, std::size_t end) {
      for (std::size_t idx = begin; idx < end; ++idx) {
        const int m = static_cast<int>(idx / k_count);
        const int k = static_cast<int>(idx % k_count);
        if (!alive[m]) {
          scratch.costs[idx] = kInf;
          continue;
        }
        std::span<Vec4> delta(scratch.perturbations.data() + idx * n, n);
        if (debug && debug->injected_delta) {
          const std::size_t base = (static_cast<std::size_t>(iter) * m_count * k_count + idx) * n;
          for (int j = 0; j < n; ++j) delta[j] = (*debug->injected_delta)[base + j];
        } else {
          sample_rollout_perturbations(cfg.mppi, StreamKey{seed, static_cast<std::uint64_t>(m), iter_cycle},
                                       k, delta);
        }
        Rollout& r = scratch.trajectories[idx];
        rollout_into(r, x, nominals[m], delta, cfg.dynamics);
        r.guide = &result.guides[m];
        scratch.costs[idx] = r.valid ? stage1_cost(r, goal, snap.clearance_index, cfg.weights, last_applied) : kInf;
        if (debug && last_iter) {
          debug->stage1_costs[idx] = scratch.costs[idx];
          if (r.valid) debug->collision_margin[idx] = collision_margin(r, snap.clearance_index, cfg.weights);
        }
      }
    });

    for (int m = 0; m < m_count; ++m) {
      if (!alive[m]) continue;
      const std::size_t base = static_cast<std::size_t>(m) * k_count;
      std::vector<double> slice(scratch.costs.begin() + base, scratch.costs.begin() + base + k_count);
      try {
        auto weights = compute_weights(slice, cfg.mppi.lambda);
        update_nominal(nominals[m],
                       std::span<const Vec4>(scratch.perturbations.data() + base * n,
                                             static_cast<std::size_t>(k_count) * n),
                       weights, cfg.dynamics);
        InstanceRecord& rec = result.per_instance[m];
        rec.stage1 = *std::min_element(slice.begin(), slice.end());
        double w2 = 0.0;
        for (double w : weights) w2 += w * w;
        rec.ess = w2 > 0.0 ? 1.0 / w2 : 0.0;
      } catch (const std::runtime_error&) {
        alive[m] = 0;
      }
    }
  }

  // stage II (ensemble.cpp:132-149)
  parallel_for(m_count, [&](std::size_t begin, std::size_t end) {
    for (std::size_t m = begin; m < end; ++m) {
      InstanceRecord& rec = result.per_instance[m];
      rec.valid = false;
      rec.stage2 = kInf;
      if (!alive[m]) continue;
      std::span<Vec4> zeros(scratch.zero_deltas.data() + m * n, n);
      for (auto& z : zeros) z = Vec4::zero();
      Rollout& r = scratch.re_rollouts[m];
      rollout_into(r, x, nominals[m], zeros, cfg.dynamics);
      r.guide = &result.guides[m];
      if (!r.valid) continue;
      rec.stage2 = stage2_cost(r, goal, snap.clearance_index, cfg.weights);
      rec.valid = std::isfinite(rec.stage2);
      rec.nominal = nominals[m];
    }
  });

  // selection (ensemble.cpp:151-168): first minimum wins
  int winner = -1;
  for (int m = 0; m < m_count; ++m) {
    const InstanceRecord& rec = result.per_instance[m];
    if (!rec.valid) continue;
    if (winner < 0 || rec.stage2 < result.per_instance[winner].stage2) winner = m;
  }
  if (winner < 0) throw std::runtime_error("planning failed");
  result.winner = winner;
  result.winner_rollout = scratch.re_rollouts[winner];
  result.control = clamp_control(result.per_instance[winner].nominal.controls.front(), cfg.dynamics);
  result.breakdown = cost_breakdown(result.winner_rollout, goal, snap.clearance_index, cfg.weights, last_applied);
  return result;
}

PlanResult plan_step(const State& x, const GoalSpec& goal, const PerceptionSnapshot& snap,
                     const EnsembleConfig& cfg, const NominalSequence& previous,
                     const ControlInput& last_applied, std::uint64_t cycle, std::uint64_t seed) {
  PlanScratch scratch;
  return plan_step(x, goal, snap, cfg, previous, last_applied, cycle, seed, scratch);
}

}  // namespace oracle
