// CPU ORACLE KNOWN-ANSWER RUNNER — TEST INFRASTRUCTURE ONLY.
//
// Pins the oracle restatement to the reference's own test suites for the hot
// path: every case below re-runs a doctest case (same seeds, same inputs,
// same expected values / tolerances) from proj/tests/test_{dynamics,
// perception,guidance,costs,mppi,ensemble}.cpp and the hot-path criteria of
// proj/tests/acceptance.cpp.  Usage: kat_runner [--slow] [filter].
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "oracle.hpp"

using namespace oracle;

namespace {

struct Case {
  const char* name;
  const char* origin;
  bool slow;
  std::function<void()> fn;
};
std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
int g_checks = 0, g_failures = 0;
const char* g_current = "";

struct Reg {
  Reg(const char* n, const char* o, bool slow, std::function<void()> f) {
    registry().push_back({n, o, slow, std::move(f)});
  }
};

#define KAT_CAT2(a, b) a##b
#define KAT_CAT(a, b) KAT_CAT2(a, b)
#define KAT(name, origin) KAT_IMPL(name, origin, false)
#define KAT_SLOW(name, origin) KAT_IMPL(name, origin, true)
#define KAT_IMPL(name, origin, slow)                                              \
  static void KAT_CAT(kat_fn_, __LINE__)();                                       \
  static Reg KAT_CAT(kat_reg_, __LINE__)(name, origin, slow, KAT_CAT(kat_fn_, __LINE__)); \
  static void KAT_CAT(kat_fn_, __LINE__)()

#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_failures;                                                              \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_current, __FILE__, __LINE__, #cond); \
    }                                                                            \
  } while (0)

#define CHECK_THROWS(expr, type)             \
  do {                                       \
    bool thrown = false;                     \
    try {                                    \
      (void)(expr);                          \
    } catch (const type&) {                  \
      thrown = true;                         \
    }                                        \
    CHECK(thrown && #expr " throws " #type); \
  } while (0)

// doctest::Approx semantics: |a-b| < eps * (scale + max(|a|,|b|)), scale 1.
bool approx(double a, double b, double eps = FLT_EPSILON * 100) {
  return std::abs(a - b) < eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

State random_state(RandomStream& rs) {
  State x;
  x.p = Vec3(rs.uniform(-5, 5), rs.uniform(-5, 5), rs.uniform(-5, 5));
  x.v = Vec3(rs.uniform(-3, 3), rs.uniform(-3, 3), rs.uniform(-3, 3));
  Vec4 q(rs.normal(), rs.normal(), rs.normal(), rs.normal());
  const double n = q.norm();
  x.q = Quat(q[0] / n, q[1] / n, q[2] / n, q[3] / n);
  return x;
}

Vec4 quat_mul_oracle(const Vec4& a, const Vec4& b) {
  return Vec4(a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
              a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
              a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
              a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]);
}

double state_error(const State& a, const State& b) {
  return (a.p - b.p).norm() + (a.v - b.v).norm() + (quat_vec(a.q) - quat_vec(b.q)).norm();
}

State propagate(State x, const ControlInput& u, DynamicsParams prm, double dt, int steps) {
  prm.dt = dt;
  for (int i = 0; i < steps; ++i) x = rk4_step(x, u, prm);
  return x;
}

Quat yaw(double a) { return Quat::from_angle_axis(a, Vec3::unit_z()); }

}  // namespace

// ===========================================================================
// test_dynamics.cpp
// ===========================================================================
KAT("hover input cancels gravity", "test_dynamics.cpp:34") {
  DynamicsParams prm;
  State x;
  StateDerivative d = state_derivative(x, ControlInput{9.81, Vec3()}, prm);
  CHECK(approx(d.dv.norm(), 0.0, 1e-12));
  CHECK(approx(d.dq.norm(), 0.0, 1e-12));
  CHECK(approx(d.dp.norm(), 0.0, 1e-12));
}

KAT("zero thrust free fall", "test_dynamics.cpp:44") {
  DynamicsParams prm;
  StateDerivative d = state_derivative(State{}, ControlInput{0.0, Vec3()}, prm);
  CHECK(approx(d.dv.x, 0.0));
  CHECK(approx(d.dv.y, 0.0));
  CHECK(approx(d.dv.z, -9.81));
}

KAT("quaternion derivative matches hand-expanded product", "test_dynamics.cpp:54") {
  DynamicsParams prm;
  StateDerivative d = state_derivative(State{}, ControlInput{9.81, Vec3(0, 0, 1)}, prm);
  CHECK(approx(d.dq[0], 0.0) && approx(d.dq[1], 0.0) && approx(d.dq[2], 0.0));
  CHECK(approx(d.dq[3], 0.5));
  RandomStream rs(7);
  for (int i = 0; i < 200; ++i) {
    State xr = random_state(rs);
    ControlInput ur{rs.uniform(0, 16), Vec3(rs.uniform(-3, 3), rs.uniform(-3, 3), rs.uniform(-2, 2))};
    Vec4 expect = 0.5 * quat_mul_oracle(quat_vec(xr.q), Vec4(0, ur.omega.x, ur.omega.y, ur.omega.z));
    Vec4 got = state_derivative(xr, ur, prm).dq;
    CHECK((got - expect).norm() < 1e-12);
  }
}

KAT("non-finite input is rejected", "test_dynamics.cpp:78") {
  DynamicsParams prm;
  State x;
  x.p.x = std::nan("");
  CHECK_THROWS(state_derivative(x, ControlInput{9.81, Vec3()}, prm), std::invalid_argument);
  CHECK_THROWS(rk4_step(State{}, ControlInput{INFINITY, Vec3()}, prm), std::invalid_argument);
}

KAT("rk4 hover step leaves the state unchanged", "test_dynamics.cpp:90") {
  DynamicsParams prm;
  State x;
  x.p = Vec3(1, 2, 3);
  State next = rk4_step(x, prm.hover(), prm);
  CHECK((next.p - x.p).norm() < 1e-9);
  CHECK((next.v - x.v).norm() < 1e-9);
  CHECK((quat_vec(next.q) - quat_vec(x.q)).norm() < 1e-9);
}

KAT("ballistic drop matches the closed form", "test_dynamics.cpp:100") {
  DynamicsParams prm;
  State next = rk4_step(State{}, ControlInput{0.0, Vec3()}, prm);
  CHECK(approx(next.p.z, -0.5 * 9.81 * 0.05 * 0.05, 1e-12));
  CHECK(approx(next.p.z, -0.0122625, 1e-9));
  CHECK(approx(next.v.z, -9.81 * 0.05, 1e-12));
}

KAT("rk4 self-convergence is fourth order", "test_dynamics.cpp:127") {
  DynamicsParams prm;
  ControlInput u{12.0, Vec3(0.7, -0.4, 0.3)};
  State ref = propagate(State{}, u, prm, 0.05 / 1000.0, 20 * 1000);
  const double ratio = state_error(propagate(State{}, u, prm, 0.05, 20), ref) /
                       state_error(propagate(State{}, u, prm, 0.025, 40), ref);
  CHECK(ratio > 10.0);
  CHECK(ratio < 24.0);
}

KAT("clamp_control saturates to the actuation limits", "test_dynamics.cpp:143") {
  DynamicsParams prm;
  CHECK(approx(clamp_control({20.0, Vec3()}, prm).thrust, 16.35));
  ControlInput boundary{0.3, Vec3(3.0, -3.0, 2.0)};
  ControlInput c = clamp_control(boundary, prm);
  CHECK(approx(c.thrust, 0.3));
  CHECK((c.omega - boundary.omega).norm() == 0.0);
  c = clamp_control({9.0, Vec3(5.0, 0.0, -4.0)}, prm);
  CHECK(approx(c.omega.x, 3.0) && approx(c.omega.y, 0.0) && approx(c.omega.z, -2.0));
}

KAT("quaternion norm is preserved by stepping", "test_dynamics.cpp:156") {
  DynamicsParams prm;
  State x;
  ControlInput u{11.0, Vec3(2.9, -2.5, 1.9)};
  for (int i = 0; i < 200; ++i) {
    x = rk4_step(x, u, prm);
    CHECK(std::abs(x.q.norm() - 1.0) < 1e-9);
  }
  State raw = rk4_step_raw(x, u, prm);
  CHECK(std::abs(raw.q.norm() - 1.0) < 1e-6);
}

KAT("horizontal velocity is conserved in free fall", "test_dynamics.cpp:170") {
  DynamicsParams prm;
  State x;
  x.v = Vec3(1.25, -0.75, 0.5);
  State end = propagate(x, ControlInput{0.0, Vec3()}, prm, 0.05, 100);
  CHECK(std::abs(end.v.x - 1.25) < 1e-12);
  CHECK(std::abs(end.v.y + 0.75) < 1e-12);
}

// ===========================================================================
// test_perception.cpp
// ===========================================================================
namespace {
struct BinOracle {  // test_perception.cpp:19-44
  std::vector<double> ranges;
  std::vector<int> counts;
  BinOracle(const std::vector<Vec3>& cloud, double r_max) {
    ranges.assign(kCells, r_max);
    counts.assign(kCells, 0);
    const double az_step = 2.0 * kPi / kAzimuthCells, el_step = kPi / kElevationCells;
    for (const auto& p : cloud) {
      const double r = std::sqrt(p.x * p.x + p.y * p.y + p.z * p.z);
      if (!(r > kMinPointRange) || r > r_max) continue;
      const double az = std::atan2(p.y, p.x);
      const double el = std::atan2(p.z, std::sqrt(p.x * p.x + p.y * p.y));
      int i = static_cast<int>(std::floor((az + kPi) / az_step));
      if (i >= kAzimuthCells) i -= kAzimuthCells;
      int j = static_cast<int>(std::floor((el + 0.5 * kPi) / el_step));
      if (j >= kElevationCells) j = kElevationCells - 1;
      if (j < 0) j = 0;
      if (i < 0) i = 0;
      ++counts[i * kElevationCells + j];
      if (r < ranges[i * kElevationCells + j]) ranges[i * kElevationCells + j] = r;
    }
  }
};

std::vector<Vec3> random_cloud(RandomStream& rs, int n, double spread) {
  std::vector<Vec3> cloud;
  cloud.reserve(n);
  for (int k = 0; k < n; ++k) {
    const double x = rs.uniform(-spread, spread);
    const double y = rs.uniform(-spread, spread);
    const double z = rs.uniform(-spread, spread);
    cloud.emplace_back(x, y, z);
  }
  return cloud;
}
}  // namespace

KAT("ring buffer keeps the most recent frames", "test_perception.cpp:58") {
  PointCloudBuffer buf(10);
  for (int f = 0; f < 11; ++f) buf.push({Vec3(static_cast<double>(f), 0.0, 0.0)});
  CHECK(buf.frames() == 10);
  auto pts = buf.body_points(State{});
  CHECK(pts.size() == 10);
  for (const auto& p : pts) CHECK(p.x > 0.5);
}

KAT("body projection for identity and translated poses", "test_perception.cpp:67") {
  PointCloudBuffer buf;
  buf.push({Vec3(1, 0, 0)});
  CHECK((buf.body_points(State{})[0] - Vec3(1, 0, 0)).norm() < 1e-12);
  PointCloudBuffer buf2;
  buf2.push({Vec3(2, 0, 0)});
  State pose;
  pose.p = Vec3(1, 0, 0);
  CHECK((buf2.body_points(pose)[0] - Vec3(1, 0, 0)).norm() < 1e-12);
}

KAT("body projection undoes attitude", "test_perception.cpp:81") {
  PointCloudBuffer buf;
  buf.push({Vec3(0, 3, 2)});
  State pose;
  pose.q = yaw(0.5 * kPi);
  CHECK((buf.body_points(pose)[0] - Vec3(3, 0, 2)).norm() < 1e-9);
}

KAT("cell directions at the cardinal angles", "test_perception.cpp:90") {
  const double lim = std::cos(2.2 * kPi / 180.0);
  CHECK(cell_direction(azimuth_cell(0.0), elevation_cell(0.0)).dot(Vec3(1, 0, 0)) > lim);
  CHECK(cell_direction(azimuth_cell(0.5 * kPi), elevation_cell(0.0)).dot(Vec3(0, 1, 0)) > lim);
  CHECK(cell_direction(azimuth_cell(0.0), elevation_cell(0.5 * kPi)).dot(Vec3(0, 0, 1)) > lim);
  CHECK_THROWS(cell_direction(-1, 0), std::out_of_range);
  CHECK_THROWS(cell_direction(0, kElevationCells), std::out_of_range);
}

KAT("empty cloud gives a uniform open partition", "test_perception.cpp:102") {
  auto part = build_partition({}, 10.0);
  for (double r : part.ranges) CHECK(r == 10.0);
  CHECK(filtered_cloud(part).points.empty());
}

KAT("single point occupies exactly one cell", "test_perception.cpp:108") {
  const Vec3 p = 4.0 * direction_from_angles(0.01, 0.01);
  auto part = build_partition({p}, 10.0);
  int occupied = 0;
  for (auto h : part.has_point) occupied += h;
  CHECK(occupied == 1);
  CHECK(approx(part.range(azimuth_cell(0.01), elevation_cell(0.01)), 4.0, 1e-12));
  CHECK(filtered_cloud(part).points.size() == 1);
}

KAT("random clouds match the brute-force binning oracle exactly", "test_perception.cpp:122") {
  RandomStream rs(101);
  for (int trial = 0; trial < 5; ++trial) {
    auto cloud = random_cloud(rs, 10000, 12.0);
    auto part = build_partition(cloud, 10.0);
    BinOracle oracle(cloud, 10.0);
    for (int f = 0; f < kCells; ++f) CHECK(part.ranges[f] == oracle.ranges[f]);
  }
}

KAT("binning is partition-complete", "test_perception.cpp:134") {
  RandomStream rs(202);
  auto cloud = random_cloud(rs, 20000, 12.0);
  BinOracle oracle(cloud, 10.0);
  int in_range = 0, binned = 0;
  for (const auto& p : cloud) {
    const double r = p.norm();
    if (r > kMinPointRange && r <= 10.0) ++in_range;
  }
  for (int c : oracle.counts) binned += c;
  CHECK(binned == in_range);
}

KAT("pooling an empty partition keeps r_max everywhere", "test_perception.cpp:148") {
  auto coarse = pool_coarse(build_partition({}, 10.0));
  for (double r : coarse.safe_range) CHECK(r == 10.0);
  for (const auto& d : coarse.safe_dir) CHECK(std::abs(d.norm() - 1.0) < 1e-9);
}

KAT("pooling breaks argmax ties toward the lowest index", "test_perception.cpp:154") {
  auto part = build_partition({}, 10.0);
  part.range(2, 2) = 3.0;
  auto coarse = pool_coarse(part);
  CHECK(approx(coarse.safe_range[0], 10.0));
  CHECK((coarse.safe_dir[0] - cell_direction(0, 0)).norm() < 1e-12);
  CHECK((coarse.safe_point[0] - 10.0 * cell_direction(0, 0)).norm() < 1e-12);
}

KAT("pooling matches an exhaustive per-block scan", "test_perception.cpp:168") {
  RandomStream rs(303);
  for (int trial = 0; trial < 20; ++trial) {
    auto part = build_partition({}, 10.0);
    for (int i = 0; i < kAzimuthCells; ++i)
      for (int j = 0; j < kElevationCells; ++j) part.range(i, j) = rs.uniform(0.5, 10.0);
    auto coarse = pool_coarse(part);
    for (int I = 0; I < kCoarseAzimuthCells; ++I)
      for (int J = 0; J < kCoarseElevationCells; ++J) {
        double best = -1.0;
        int bi = 0, bj = 0;
        for (int i = I * kPoolFactor; i < (I + 1) * kPoolFactor; ++i)
          for (int j = J * kPoolFactor; j < (J + 1) * kPoolFactor; ++j)
            if (part.range(i, j) > best) {
              best = part.range(i, j);
              bi = i;
              bj = j;
            }
        CHECK(coarse.safe_range[CoarsePartition::flat(I, J)] == best);
        CHECK((coarse.safe_dir[CoarsePartition::flat(I, J)] - cell_direction(bi, bj)).norm() == 0.0);
      }
  }
}

KAT("clearance sentinel and trivial cases", "test_perception.cpp:196") {
  FilteredCloud empty;
  CHECK(clearance(empty, Vec3()) == empty.far_clearance());
  CHECK(ClearanceIndex(empty).nearest(Vec3()) == empty.far_clearance());
  CHECK(empty.far_clearance() == 35.0);
  FilteredCloud one;
  one.points = {Vec3(1, 0, 0)};
  CHECK(approx(clearance(one, Vec3()), 1.0, 1e-12));
}

KAT("clearance index equals the linear-scan oracle exactly", "test_perception.cpp:206") {
  RandomStream rs(404);
  auto cloud = random_cloud(rs, 30000, 11.0);
  FilteredCloud fc = filtered_cloud(build_partition(cloud, 10.0));
  CHECK(fc.points.size() <= static_cast<std::size_t>(kCells));
  ClearanceIndex index(fc);
  for (int k = 0; k < 2000; ++k) {
    const double x = rs.uniform(-15, 15), y = rs.uniform(-15, 15), z = rs.uniform(-15, 15);
    const Vec3 p(x, y, z);
    CHECK(index.nearest(p) == clearance(fc, p));
  }
}

KAT("clearance is 1-Lipschitz", "test_perception.cpp:219") {
  RandomStream rs(505);
  auto cloud = random_cloud(rs, 5000, 11.0);
  FilteredCloud fc = filtered_cloud(build_partition(cloud, 10.0));
  for (int k = 0; k < 500; ++k) {
    const double ax = rs.uniform(-12, 12), ay = rs.uniform(-12, 12), az = rs.uniform(-12, 12);
    const double bx = rs.uniform(-12, 12), by = rs.uniform(-12, 12), bz = rs.uniform(-12, 12);
    const Vec3 a(ax, ay, az), b(bx, by, bz);
    CHECK(std::abs(clearance(fc, a) - clearance(fc, b)) <= (a - b).norm() + 1e-12);
  }
}

KAT("partition rebuild is bit-identical", "test_perception.cpp:231") {
  RandomStream rs(606);
  auto cloud = random_cloud(rs, 8000, 11.0);
  auto a = build_partition(cloud, 10.0);
  auto b = build_partition(cloud, 10.0);
  for (int c = 0; c < kCells; ++c) {
    CHECK(a.ranges[c] == b.ranges[c]);
    CHECK(a.has_point[c] == b.has_point[c]);
    CHECK((a.nearest[c] - b.nearest[c]).norm() == 0.0);
  }
}

KAT("snapshot projects the filtered cloud to world frame", "test_perception.cpp:243") {
  PointCloudBuffer buf;
  buf.push({Vec3(3, 1, 2)});
  State pose;
  pose.p = Vec3(1, 1, 2);
  auto snap = build_snapshot(buf, pose);
  CHECK(snap.filtered.points.size() == 1);
  CHECK(snap.filtered.frame == FilteredCloud::Frame::world);
  CHECK((snap.filtered.points[0] - Vec3(3, 1, 2)).norm() < 1e-12);
  CHECK(snap.clearance_index.nearest(Vec3(3, 1, 2)) < 1e-12);
}

// ===========================================================================
// test_guidance.cpp
// ===========================================================================
namespace {
// Vandermonde 6x6 solve (test_guidance.cpp:17-32); partial-pivot Gaussian
// elimination stands in for Eigen's colPivHouseholderQr.
void quintic_oracle(double p0, double v0, double a0, double pT, double vT, double aT, double T,
                    double out[6]) {
  double A[6][7] = {};
  A[0][0] = 1.0;
  A[1][1] = 1.0;
  A[2][2] = 2.0;
  for (int k = 0; k < 6; ++k) {
    A[3][k] = std::pow(T, k);
    if (k >= 1) A[4][k] = k * std::pow(T, k - 1);
    if (k >= 2) A[5][k] = k * (k - 1) * std::pow(T, k - 2);
  }
  const double b[6] = {p0, v0, a0, pT, vT, aT};
  for (int i = 0; i < 6; ++i) A[i][6] = b[i];
  for (int c = 0; c < 6; ++c) {
    int piv = c;
    for (int r = c + 1; r < 6; ++r)
      if (std::abs(A[r][c]) > std::abs(A[piv][c])) piv = r;
    for (int k = 0; k < 7; ++k) std::swap(A[c][k], A[piv][k]);
    for (int r = 0; r < 6; ++r) {
      if (r == c) continue;
      const double f = A[r][c] / A[c][c];
      for (int k = c; k < 7; ++k) A[r][k] -= f * A[c][k];
    }
  }
  for (int i = 0; i < 6; ++i) out[i] = A[i][6] / A[i][i];
}
}  // namespace

KAT("single anchor straight ahead", "test_guidance.cpp:36") {
  AnchorGrid grid;
  grid.m_h = grid.m_v = 1;
  auto eps = sample_initial_endpoints(Vec3(), Vec3(10, 0, 0), grid);
  CHECK(eps.size() == 1);
  CHECK((eps[0] - Vec3(5, 0, 0)).norm() < 1e-12);
}

KAT("flank endpoints sit at the spacing offsets", "test_guidance.cpp:45") {
  AnchorGrid grid;
  grid.m_h = 3;
  grid.m_v = 1;
  auto eps = sample_initial_endpoints(Vec3(), Vec3(20, 0, 0), grid);
  CHECK(eps.size() == 3);
  const double s = 18.0 * kPi / 180.0;
  CHECK((eps[0] - 5.0 * Vec3(std::cos(-s), std::sin(-s), 0)).norm() < 1e-12);
  CHECK((eps[1] - Vec3(5, 0, 0)).norm() < 1e-12);
  CHECK((eps[2] - 5.0 * Vec3(std::cos(s), std::sin(s), 0)).norm() < 1e-12);
  for (const auto& e : eps) CHECK(approx(e.norm(), 5.0));
}

KAT("grid center tracks the goal azimuth", "test_guidance.cpp:58") {
  AnchorGrid grid;
  const Vec3 goal = 20.0 * Vec3(std::cos(kPi / 4), std::sin(kPi / 4), 0);
  auto eps = sample_initial_endpoints(Vec3(), goal, grid);
  CHECK((eps[1 * 5 + 2].normalized() - goal.normalized()).norm() < 1e-12);
  double az_sum = 0;
  for (const auto& e : eps) az_sum += std::atan2(e.y, e.x) - kPi / 4;
  CHECK(std::abs(az_sum) < 1e-9);
}

KAT("degenerate goal direction is rejected", "test_guidance.cpp:73") {
  AnchorGrid grid;
  CHECK_THROWS(sample_initial_endpoints(Vec3(1, 1, 1), Vec3(1, 1, 1), grid), std::invalid_argument);
}

KAT("refinement distances follow the clamp rule", "test_guidance.cpp:80") {
  auto coarse = pool_coarse(build_partition({}, 10.0));
  State pose;
  AnchorGrid grid;
  auto eps = sample_initial_endpoints(pose.p, Vec3(10, 0, 0), grid);
  auto anchors = refine_endpoints(eps, coarse, pose, 5.0, 1.0);
  CHECK(anchors.size() == 15);
  for (const auto& a : anchors) {
    CHECK(approx((a.refined_endpoint - pose.p).norm(), 5.0, 1e-12));
    CHECK(std::abs(a.safe_dir.norm() - 1.0) < 1e-9);
  }
  CoarsePartition tight = coarse;
  for (auto& r : tight.safe_range) r = 3.0;
  for (const auto& a : refine_endpoints(eps, tight, pose, 5.0, 1.0))
    CHECK(approx((a.refined_endpoint - pose.p).norm(), 2.0, 1e-12));
  CoarsePartition blocked = coarse;
  for (auto& r : blocked.safe_range) r = 1.0;
  for (const auto& a : refine_endpoints(eps, blocked, pose, 5.0, 1.0))
    CHECK(approx((a.refined_endpoint - pose.p).norm(), 0.5, 1e-12));
}

KAT("refinement maps endpoints through the body frame", "test_guidance.cpp:112") {
  State pose;
  pose.q = yaw(0.5 * kPi);
  auto coarse = pool_coarse(build_partition({}, 10.0));
  auto anchors = refine_endpoints({Vec3(5, 0, 0)}, coarse, pose, 5.0, 1.0);
  CHECK(anchors.size() == 1);
  CHECK(anchors[0].coarse_i == coarse_azimuth_cell(-0.5 * kPi));
  const int f = CoarsePartition::flat(anchors[0].coarse_i, anchors[0].coarse_j);
  CHECK((anchors[0].safe_dir - pose.q * coarse.safe_dir[f]).norm() < 1e-12);
}

KAT("anchor endpoints stay within the lookahead ball", "test_guidance.cpp:127") {
  RandomStream rs(42);
  AnchorGrid grid;
  for (int trial = 0; trial < 50; ++trial) {
    std::vector<Vec3> cloud;
    for (int k = 0; k < 500; ++k) {
      const double x = rs.uniform(-9, 9), y = rs.uniform(-9, 9), z = rs.uniform(-9, 9);
      cloud.emplace_back(x, y, z);
    }
    auto coarse = pool_coarse(build_partition(cloud, 10.0));
    State pose;
    const double px = rs.uniform(-2, 2), py = rs.uniform(-2, 2), pz = rs.uniform(1, 3);
    pose.p = Vec3(px, py, pz);
    const double gx = rs.uniform(5, 30), gy = rs.uniform(-10, 10);
    const Vec3 goal(gx, gy, 2.0);
    auto eps = sample_initial_endpoints(pose.p, goal, grid);
    for (const auto& a : refine_endpoints(eps, coarse, pose, grid.lookahead, 1.0))
      CHECK((a.refined_endpoint - pose.p).norm() <= grid.lookahead + 1e-9);
  }
}

KAT("anchor diversity in the open", "test_guidance.cpp:145") {
  AnchorGrid grid;
  State pose;
  pose.p = Vec3(0, 0, 2);
  auto coarse = pool_coarse(build_partition({}, 10.0));
  auto anchors = refine_endpoints(sample_initial_endpoints(pose.p, Vec3(45, 0, 2), grid), coarse, pose, 5.0, 1.0);
  for (std::size_t a = 0; a < anchors.size(); ++a)
    for (std::size_t b = a + 1; b < anchors.size(); ++b)
      CHECK((anchors[a].refined_endpoint - anchors[b].refined_endpoint).norm() > 1e-3);
}

KAT("refinement does not reduce clearance in a one-wall scene", "test_guidance.cpp:157") {
  std::vector<Vec3> cloud;
  for (double y = -0.4; y <= 0.4; y += 0.1)
    for (double z = -0.4; z <= 0.4; z += 0.1) cloud.emplace_back(4.0, y, z);
  auto part = build_partition(cloud, 10.0);
  auto coarse = pool_coarse(part);
  FilteredCloud fc = filtered_cloud(part);
  State pose;
  AnchorGrid grid;
  grid.m_h = grid.m_v = 1;
  auto anchors = refine_endpoints(sample_initial_endpoints(pose.p, Vec3(10, 0, 0), grid), coarse, pose, 5.0, 1.0);
  CHECK(clearance(fc, anchors[0].refined_endpoint) >= clearance(fc, anchors[0].initial_endpoint) - 1e-9);
}

KAT("constant quintic for identical rest boundary conditions", "test_guidance.cpp:176") {
  BoundaryCondition rest;
  rest.p = Vec3(1, 2, 3);
  auto g = solve_quintic(rest, rest, 1.25);
  CHECK((g.coeffs[0] - rest.p).norm() < 1e-12);
  for (int k = 1; k < 6; ++k) CHECK(g.coeffs[k].norm() < 1e-12);
  CHECK((eval_guide(g, 0.7) - rest.p).norm() < 1e-12);
}

KAT("classic rest-to-rest quintic 10t^3 - 15t^4 + 6t^5", "test_guidance.cpp:185") {
  BoundaryCondition start, end;
  end.p = Vec3(1, 1, 1);
  auto g = solve_quintic(start, end, 1.0);
  for (int axis = 0; axis < 3; ++axis) {
    CHECK(approx(g.coeffs[0][axis], 0.0) && approx(g.coeffs[1][axis], 0.0) && approx(g.coeffs[2][axis], 0.0));
    CHECK(approx(g.coeffs[3][axis], 10.0, 1e-12));
    CHECK(approx(g.coeffs[4][axis], -15.0, 1e-12));
    CHECK(approx(g.coeffs[5][axis], 6.0, 1e-12));
  }
}

KAT("quintic reproduces random boundary conditions", "test_guidance.cpp:199") {
  RandomStream rs(9);
  for (int trial = 0; trial < 1000; ++trial) {
    BoundaryCondition s, e;
    for (int axis = 0; axis < 3; ++axis) {
      s.p[axis] = rs.uniform(-10, 10);
      s.v[axis] = rs.uniform(-5, 5);
      s.a[axis] = rs.uniform(-10, 10);
      e.p[axis] = rs.uniform(-10, 10);
      e.v[axis] = rs.uniform(-5, 5);
      e.a[axis] = rs.uniform(-10, 10);
    }
    const double T = rs.uniform(0.5, 3.0);
    auto g = solve_quintic(s, e, T);
    CHECK((eval_guide(g, 0.0) - s.p).norm() < 1e-9);
    CHECK((eval_guide_velocity(g, 0.0) - s.v).norm() < 1e-9);
    CHECK((eval_guide_acceleration(g, 0.0) - s.a).norm() < 1e-9);
    CHECK((eval_guide(g, T) - e.p).norm() < 1e-9);
    CHECK((eval_guide_velocity(g, T) - e.v).norm() < 1e-9);
    CHECK((eval_guide_acceleration(g, T) - e.a).norm() < 1e-9);
  }
}

KAT("quintic matches the linear-solve oracle", "test_guidance.cpp:224") {
  RandomStream rs(19);
  for (int trial = 0; trial < 50; ++trial) {
    BoundaryCondition s, e;
    s.p = Vec3(rs.uniform(-5, 5), 0, 0);
    s.v = Vec3(rs.uniform(-3, 3), 0, 0);
    s.a = Vec3(rs.uniform(-5, 5), 0, 0);
    e.p = Vec3(rs.uniform(-5, 5), 0, 0);
    e.v = Vec3(rs.uniform(-3, 3), 0, 0);
    e.a = Vec3(rs.uniform(-5, 5), 0, 0);
    const double T = rs.uniform(0.4, 2.5);
    auto g = solve_quintic(s, e, T);
    double o[6];
    quintic_oracle(s.p.x, s.v.x, s.a.x, e.p.x, e.v.x, e.a.x, T, o);
    for (int k = 0; k < 6; ++k) CHECK(approx(g.coeffs[k].x, o[k], 1e-8));
  }
}

KAT("eval clamps outside the horizon and rejects bad horizons", "test_guidance.cpp:244") {
  BoundaryCondition s, e;
  e.p = Vec3(1, 0, 0);
  auto g = solve_quintic(s, e, 1.0);
  CHECK((eval_guide(g, -1.0) - s.p).norm() < 1e-12);
  CHECK((eval_guide(g, 5.0) - e.p).norm() < 1e-12);
  CHECK_THROWS(solve_quintic(s, e, 0.0), std::invalid_argument);
  CHECK_THROWS(solve_quintic(s, e, -1.0), std::invalid_argument);
}

KAT("build_guides applies the dynamics start acceleration", "test_guidance.cpp:254") {
  DynamicsParams prm;
  State x;
  x.p = Vec3(0, 0, 2);
  x.v = Vec3(1, 0, 0);
  Anchor a;
  a.refined_endpoint = Vec3(5, 0, 2);
  a.safe_dir = Vec3(1, 0, 0);
  auto guides = build_guides({a}, x, prm.hover(), prm, 3.0, 1.25);
  CHECK(guides.size() == 1);
  CHECK((eval_guide(guides[0], 0.0) - x.p).norm() < 1e-12);
  CHECK((eval_guide_velocity(guides[0], 0.0) - x.v).norm() < 1e-12);
  CHECK(eval_guide_acceleration(guides[0], 0.0).norm() < 1e-9);
  CHECK((eval_guide(guides[0], 1.25) - a.refined_endpoint).norm() < 1e-9);
  CHECK((eval_guide_velocity(guides[0], 1.25) - Vec3(3, 0, 0)).norm() < 1e-9);
}

// ===========================================================================
// test_costs.cpp
// ===========================================================================
namespace {
Rollout make_rollout(int n, const Vec3& p, const Vec3& v) {
  Rollout r;
  r.states.assign(n + 1, State{});
  r.controls.assign(n, ControlInput{});
  for (auto& s : r.states) {
    s.p = p;
    s.v = v;
  }
  return r;
}

Rollout random_rollout(RandomStream& rs, int n) {
  Rollout r;
  r.dt = 0.05;
  r.states.resize(n + 1);
  r.controls.resize(n);
  for (auto& s : r.states) {
    const double px = rs.uniform(-5, 5), py = rs.uniform(-5, 5), pz = rs.uniform(-5, 5);
    s.p = Vec3(px, py, pz);
    const double vx = rs.uniform(-3, 3), vy = rs.uniform(-3, 3), vz = rs.uniform(-3, 3);
    s.v = Vec3(vx, vy, vz);
    const double a = rs.normal(), b = rs.normal(), c = rs.normal(), d = rs.normal();
    Vec4 q(a, b, c, d);
    const double n4 = q.norm();
    s.q = Quat(q[0] / n4, q[1] / n4, q[2] / n4, q[3] / n4);
  }
  for (auto& u : r.controls) {
    u.thrust = rs.uniform(0, 16);
    const double wx = rs.uniform(-3, 3), wy = rs.uniform(-3, 3), wz = rs.uniform(-2, 2);
    u.omega = Vec3(wx, wy, wz);
  }
  return r;
}
}  // namespace

KAT("tracking cost on and off the guide", "test_costs.cpp:44") {
  CostWeights w;
  BoundaryCondition rest;
  rest.p = Vec3(1, 1, 1);
  GuidingTrajectory guide = solve_quintic(rest, rest, 1.25);
  Rollout on = make_rollout(25, rest.p, Vec3());
  on.guide = &guide;
  CHECK(approx(tracking_cost(on, w), 0.0));
  Rollout off = make_rollout(25, rest.p + Vec3(1, 0, 0), Vec3());
  off.guide = &guide;
  CHECK(approx(tracking_cost(off, w), 375.0, 1e-12));
  Rollout off2 = make_rollout(25, rest.p + Vec3(2, 0, 0), Vec3());
  off2.guide = &guide;
  CHECK(approx(tracking_cost(off2, w), 2.0 * tracking_cost(off, w)));
}

KAT("velocity norm cost", "test_costs.cpp:63") {
  CostWeights w;
  CHECK(approx(vnorm_cost(make_rollout(25, Vec3(), Vec3()), w), 0.0));
  CHECK(approx(vnorm_cost(make_rollout(25, Vec3(), Vec3(2, 0, 0)), w), 15.0, 1e-9));
  CHECK(approx(vnorm_cost(make_rollout(25, Vec3(), Vec3(6, 0, 0)), w), 135.0, 1e-9));
}

KAT("control cost index ranges", "test_costs.cpp:73") {
  CostWeights w;
  ControlInput prev{0.0, Vec3()};
  CHECK(approx(control_cost(make_rollout(5, Vec3(), Vec3()), w, prev), 0.0));
  Rollout constant = make_rollout(25, Vec3(), Vec3());
  for (auto& u : constant.controls) u = ControlInput{2.0, Vec3(1, 0, 0)};
  CHECK(approx(control_cost(constant, w, prev), 24.0 * 0.5 * 5.0, 1e-12));
  Rollout three = make_rollout(3, Vec3(), Vec3());
  three.controls[0] = ControlInput{1.0, Vec3()};
  three.controls[1] = ControlInput{3.0, Vec3()};
  three.controls[2] = ControlInput{100.0, Vec3()};
  CHECK(approx(control_cost(three, w, prev), 7.0, 1e-12));
  CHECK(approx(control_cost(three, w, ControlInput{50.0, Vec3(1, 1, 1)}), 7.0, 1e-12));
}

KAT("goal cost at the goal and under yaw error", "test_costs.cpp:97") {
  CostWeights w;
  GoalSpec goal;
  goal.p_goal = Vec3(3, 0, 2);
  CHECK(approx(goal_cost(make_rollout(25, goal.p_goal, Vec3()), goal, w), 0.0, 1e-12));
  GoalSpec yawed = goal;
  yawed.q_goal = yaw(0.7);
  Rollout aligned = make_rollout(25, goal.p_goal, Vec3());
  for (auto& s : aligned.states) s.q = yawed.q_goal;
  CHECK(approx(goal_cost(aligned, yawed, w), 0.0, 1e-12));
  Rollout flipped = make_rollout(1, goal.p_goal, Vec3());
  flipped.states[0].q = yaw(M_PI);
  CHECK(approx(goal_cost(flipped, goal, w), std::sqrt(8.0), 1e-9));
}

KAT("attitude term is invariant to a global rotation", "test_costs.cpp:118") {
  CostWeights w;
  w.q_p = 0.0;
  w.q_v = 0.0;
  RandomStream rs(5);
  for (int trial = 0; trial < 100; ++trial) {
    GoalSpec goal;
    {
      const double a = rs.normal(), b = rs.normal(), c = rs.normal(), d = rs.normal();
      const double n = Vec4(a, b, c, d).norm();
      goal.q_goal = Quat(a / n, b / n, c / n, d / n);
    }
    Rollout r = random_rollout(rs, 5);
    const double before = goal_cost(r, goal, w);
    const double a = rs.normal(), b = rs.normal(), c = rs.normal(), d = rs.normal();
    const double n = Vec4(a, b, c, d).norm();
    const Quat rot(a / n, b / n, c / n, d / n);
    GoalSpec goal2 = goal;
    goal2.q_goal = rot * goal.q_goal;
    Rollout r2 = r;
    for (auto& s : r2.states) s.q = rot * s.q;
    CHECK(approx(goal_cost(r2, goal2, w), before, 1e-9));
  }
}

KAT("collision term branch table", "test_costs.cpp:141") {
  CostWeights w;
  CHECK(approx(collision_term(0.2, w), 1.0e6));
  CHECK(approx(collision_term(0.4, w), 1.0e6));
  CHECK(approx(collision_term(0.6, w), 1.0e6 * std::exp(-1.0), 1e-12));
  CHECK(approx(collision_term(0.6, w), 367879.44117144233, 1e-9));
  CHECK(collision_term(1.0, w) == 0.0);
  CHECK(approx(collision_term(std::nextafter(1.0, 0.0), w), 1.0e6 * std::exp(-3.0), 1e-6));
  double prev = kInf;
  for (double d = 0.0; d <= 2.0; d += 0.01) {
    const double c = collision_term(d, w);
    CHECK(c <= prev + 1e-9);
    prev = c;
  }
}

KAT("collision cost over rollouts", "test_costs.cpp:162") {
  CostWeights w;
  FilteredCloud empty;
  Rollout r = make_rollout(25, Vec3(), Vec3());
  CHECK(collision_cost(r, empty, w) == 0.0);
  FilteredCloud one;
  one.points = {Vec3(0.2, 0, 0)};
  CHECK(approx(collision_cost(r, one, w), 2.5e7));
  Rollout far = make_rollout(25, Vec3(-1, 0, 0), Vec3());
  CHECK(collision_cost(far, one, w) <= collision_cost(r, one, w));
}

KAT("stage decomposition identity", "test_costs.cpp:177") {
  CostWeights w;
  RandomStream rs(77);
  BoundaryCondition s, e;
  e.p = Vec3(5, 1, 0);
  GuidingTrajectory guide = solve_quintic(s, e, 1.25);
  GoalSpec goal;
  goal.p_goal = Vec3(10, 0, 2);
  ControlInput prev{9.81, Vec3()};
  std::vector<Vec3> cloud;
  for (int k = 0; k < 500; ++k) {
    const double x = rs.uniform(-8, 8), y = rs.uniform(-8, 8), z = rs.uniform(-8, 8);
    cloud.emplace_back(x, y, z);
  }
  FilteredCloud fc = filtered_cloud(build_partition(cloud, 10.0));
  ClearanceIndex index(fc);
  for (int trial = 0; trial < 50; ++trial) {
    Rollout r = random_rollout(rs, 25);
    r.guide = &guide;
    const double s1 = stage1_cost(r, goal, index, w, prev);
    const double s2 = stage2_cost(r, goal, index, w);
    const double parts = tracking_cost(r, w) + vnorm_cost(r, w) + control_cost(r, w, prev);
    CHECK(approx(s1 - s2, parts, 1e-9));
    const double recomposed = tracking_cost(r, w) + vnorm_cost(r, w) + control_cost(r, w, prev) +
                              goal_cost(r, goal, w) + collision_cost(r, index, w);
    CHECK(approx(s1, recomposed, 1e-9));
    CHECK(approx(stage2_cost(r, goal, fc, w), s2, 1e-12));
    CHECK(s1 >= 0.0);
    CHECK(s2 >= 0.0);
  }
}

KAT("cost breakdown mirrors the individual terms", "test_costs.cpp:214") {
  CostWeights w;
  RandomStream rs(88);
  Rollout r = random_rollout(rs, 10);
  GoalSpec goal;
  goal.p_goal = Vec3(4, 4, 2);
  FilteredCloud fc;
  fc.points = {Vec3(1, 1, 1)};
  ClearanceIndex index(fc);
  ControlInput prev{9.81, Vec3()};
  CostBreakdown b = cost_breakdown(r, goal, index, w, prev);
  CHECK(approx(b.track, tracking_cost(r, w)));
  CHECK(approx(b.vnorm, vnorm_cost(r, w)));
  CHECK(approx(b.ctrl, control_cost(r, w, prev)));
  CHECK(approx(b.goal, goal_cost(r, goal, w)));
  CHECK(approx(b.collision, collision_cost(r, index, w)));
  CHECK(approx(b.stage1(), stage1_cost(r, goal, index, w, prev)));
  CHECK(approx(b.stage2(), stage2_cost(r, goal, index, w)));
}

// ===========================================================================
// test_mppi.cpp
// ===========================================================================
KAT("zero sigma gives zero perturbations", "test_mppi.cpp:11") {
  MppiConfig cfg;
  cfg.sigma = Vec4(0, 0, 0, 0);
  for (const auto& d : sample_perturbations(cfg, StreamKey{1, 0, 0})) CHECK(d.norm() == 0.0);
}

KAT("perturbation sample means satisfy the CLT bound", "test_mppi.cpp:18") {
  MppiConfig cfg;
  cfg.rollouts = 4000;
  cfg.horizon = 25;
  auto all = sample_perturbations(cfg, StreamKey{7, 0, 0});
  Vec4 mean;
  for (const auto& d : all) mean = mean + d;
  const double n = static_cast<double>(all.size());
  for (int c = 0; c < 4; ++c) CHECK(std::abs(mean[c] / n) < 4.0 * cfg.sigma[c] / std::sqrt(n));
}

KAT("same stream key reproduces the same tensor", "test_mppi.cpp:31") {
  MppiConfig cfg;
  auto a = sample_perturbations(cfg, StreamKey{3, 2, 11});
  auto b = sample_perturbations(cfg, StreamKey{3, 2, 11});
  for (std::size_t i = 0; i < a.size(); ++i) CHECK((a[i] - b[i]).norm() == 0.0);
  auto c = sample_perturbations(cfg, StreamKey{3, 2, 12});
  bool any_diff = false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if ((a[i] - c[i]).norm() != 0.0) any_diff = true;
  CHECK(any_diff);
}

KAT("hover nominal with zero noise stays put", "test_mppi.cpp:44") {
  DynamicsParams prm;
  MppiConfig cfg;
  NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
  std::vector<Vec4> delta(cfg.horizon);
  State x0;
  x0.p = Vec3(1, 1, 2);
  Rollout r = rollout(x0, nominal, delta, prm);
  CHECK(r.valid);
  for (const auto& s : r.states) CHECK((s.p - x0.p).norm() < 1e-9);
}

KAT("rollout equals sequential re-propagation", "test_mppi.cpp:56") {
  DynamicsParams prm;
  MppiConfig cfg;
  NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
  auto delta = sample_perturbations(cfg, StreamKey{5, 0, 0});
  const std::vector<Vec4> sampled(delta.begin(), delta.begin() + cfg.horizon);
  std::span<Vec4> d0(delta.data(), cfg.horizon);
  State x0;
  x0.p = Vec3(0, 0, 2);
  Rollout r = rollout(x0, nominal, d0, prm);
  State x = x0;
  for (int j = 0; j < cfg.horizon; ++j) {
    const ControlInput u = clamp_control(ControlInput::from_vec(nominal.controls[j].vec() + sampled[j]), prm);
    CHECK((r.controls[j].vec() - u.vec()).norm() == 0.0);
    x = rk4_step(x, u, prm);
    CHECK((r.states[j + 1].p - x.p).norm() == 0.0);
    CHECK((r.states[j + 1].v - x.v).norm() == 0.0);
    CHECK((quat_vec(r.states[j + 1].q) - quat_vec(x.q)).norm() == 0.0);
  }
  for (int j = 0; j < cfg.horizon; ++j) {
    CHECK((r.controls[j].vec() - (nominal.controls[j].vec() + d0[j])).norm() < 1e-12);
    CHECK(r.controls[j].thrust <= prm.thrust_max);
    CHECK(r.controls[j].thrust >= prm.thrust_min);
  }
}

KAT("equal costs give uniform weights", "test_mppi.cpp:86") {
  auto w = compute_weights({5.0, 5.0, 5.0, 5.0}, 0.1);
  double sum = 0;
  for (double x : w) {
    CHECK(approx(x, 0.25, 1e-12));
    sum += x;
  }
  CHECK(std::abs(sum - 1.0) < 1e-12);
}

KAT("two-cost weights match the closed form", "test_mppi.cpp:94") {
  const double lambda = 0.1;
  auto w = compute_weights({0.0, lambda}, lambda);
  CHECK(approx(w[0], 1.0 / (1.0 + std::exp(-1.0)), 1e-12));
  CHECK(approx(w[1], std::exp(-1.0) / (1.0 + std::exp(-1.0)), 1e-12));
  CHECK(approx(w[0], 0.73106, 1e-4));
  CHECK(approx(w[1], 0.26894, 1e-4));
}

KAT("softmin limit selects the argmin", "test_mppi.cpp:104") {
  auto w = compute_weights({1.0, 0.0, 2.0}, 1e-6);
  CHECK(approx(w[1], 1.0, 1e-9));
  CHECK(approx(w[0], 0.0));
  CHECK(approx(w[2], 0.0));
}

KAT("weights are exactly invariant to cost translation", "test_mppi.cpp:111") {
  std::vector<double> costs{1.0, 2.0, 4.0, 8.0};
  auto base = compute_weights(costs, 0.1);
  for (double shift : {16.0, 256.0, -32.0}) {
    std::vector<double> moved;
    for (double c : costs) moved.push_back(c + shift);
    auto w = compute_weights(moved, 0.1);
    for (std::size_t i = 0; i < w.size(); ++i) CHECK(w[i] == base[i]);
  }
}

KAT("invalid rollouts get zero weight, all invalid throws", "test_mppi.cpp:123") {
  auto w = compute_weights({1.0, kInf, 1.0}, 0.1);
  CHECK(w[1] == 0.0);
  CHECK(approx(w[0], 0.5, 1e-12));
  CHECK_THROWS(compute_weights({kInf, kInf}, 0.1), std::runtime_error);
}

KAT("nominal update against a dense double-loop oracle", "test_mppi.cpp:132") {
  DynamicsParams prm;
  const int n = 10, k_count = 16;
  MppiConfig cfg;
  cfg.horizon = n;
  cfg.rollouts = k_count;
  NominalSequence nominal = NominalSequence::constant({9.0, Vec3(0.1, 0, 0)}, n);
  auto deltas = sample_perturbations(cfg, StreamKey{21, 0, 0});
  for (auto& d : deltas) d = 0.05 * d;
  std::vector<double> costs;
  RandomStream rs(3);
  for (int k = 0; k < k_count; ++k) costs.push_back(rs.uniform(0, 1));
  auto weights = compute_weights(costs, 0.5);
  NominalSequence updated = nominal;
  update_nominal(updated, deltas, weights, prm);
  for (int j = 0; j < n; ++j) {
    Vec4 expect = nominal.controls[j].vec();
    for (int k = 0; k < k_count; ++k) expect = expect + weights[k] * deltas[k * n + j];
    CHECK((updated.controls[j].vec() - expect).norm() < 1e-12);
  }
}

KAT("all-zero perturbations leave the nominal unchanged", "test_mppi.cpp:157") {
  DynamicsParams prm;
  NominalSequence nominal = NominalSequence::constant({5.0, Vec3(1, -1, 0.5)}, 8);
  std::vector<Vec4> deltas(8 * 4);
  auto weights = compute_weights(std::vector<double>(4, 1.0), 0.1);
  NominalSequence updated = nominal;
  update_nominal(updated, deltas, weights, prm);
  for (int j = 0; j < 8; ++j) CHECK((updated.controls[j].vec() - nominal.controls[j].vec()).norm() == 0.0);
}

KAT("single-rollout update reproduces the applied controls", "test_mppi.cpp:168") {
  DynamicsParams prm;
  MppiConfig cfg;
  cfg.rollouts = 1;
  cfg.horizon = 12;
  NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
  auto delta = sample_perturbations(cfg, StreamKey{9, 1, 4});
  Rollout r = rollout(State{}, nominal, std::span<Vec4>(delta.data(), cfg.horizon), prm);
  NominalSequence updated = nominal;
  update_nominal(updated, delta, {1.0}, prm);
  for (int j = 0; j < cfg.horizon; ++j) CHECK((updated.controls[j].vec() - r.controls[j].vec()).norm() < 1e-12);
}

KAT("shift_nominal drops the head and repeats the tail", "test_mppi.cpp:182") {
  NominalSequence n;
  n.controls = {{1.0, Vec3()}, {2.0, Vec3()}, {3.0, Vec3()}};
  auto s = shift_nominal(n);
  CHECK(s.controls.size() == 3);
  CHECK(s.controls[0].thrust == 2.0 && s.controls[1].thrust == 3.0 && s.controls[2].thrust == 3.0);
  auto sc = shift_nominal(NominalSequence::constant({4.0, Vec3(1, 1, 1)}, 5));
  for (const auto& u : sc.controls) CHECK(u.thrust == 4.0);
  CHECK(sc.controls.size() == 5);
}

KAT_SLOW("mppi improves a goal-cost-only problem for most seeds", "test_mppi.cpp:211") {
  DynamicsParams prm;
  MppiConfig cfg;
  cfg.rollouts = 64;
  CostWeights w;
  GoalSpec goal;
  goal.p_goal = Vec3(6, 0, 2);
  State x0;
  x0.p = Vec3(0, 0, 2);
  auto nominal_cost = [&](const NominalSequence& nominal) {
    std::vector<Vec4> zeros(nominal.controls.size());
    Rollout r = rollout(x0, nominal, zeros, prm);
    return goal_cost(r, goal, w);
  };
  int improved = 0;
  RolloutBatch batch;
  for (int seed = 1; seed <= 100; ++seed) {
    NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
    const double before = nominal_cost(nominal);
    for (int iter = 0; iter < 10; ++iter)
      mppi_step(nominal, x0, cfg, prm, StreamKey{static_cast<std::uint64_t>(seed), 0, static_cast<std::uint64_t>(iter)},
                [&](const Rollout& r) { return goal_cost(r, goal, w); }, batch);
    if (nominal_cost(nominal) <= before) ++improved;
  }
  CHECK(improved >= 95);
}

KAT("mppi_step is bit-identical across worker counts", "test_mppi.cpp:240") {
  DynamicsParams prm;
  MppiConfig cfg;
  CostWeights w;
  GoalSpec goal;
  goal.p_goal = Vec3(5, 2, 3);
  State x0;
  x0.p = Vec3(0, 0, 2);
  auto run = [&](unsigned workers) {
    set_worker_count(workers);
    NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
    RolloutBatch batch;
    mppi_step(nominal, x0, cfg, prm, StreamKey{17, 3, 9}, [&](const Rollout& r) { return goal_cost(r, goal, w); },
              batch);
    return nominal;
  };
  auto a = run(1), b = run(2), c = run(7);
  set_worker_count(0);
  for (int j = 0; j < cfg.horizon; ++j) {
    CHECK((a.controls[j].vec() - b.controls[j].vec()).norm() == 0.0);
    CHECK((a.controls[j].vec() - c.controls[j].vec()).norm() == 0.0);
  }
}

KAT("invalid rollouts never contaminate the update", "test_mppi.cpp:268") {
  DynamicsParams prm;
  MppiConfig cfg;
  cfg.rollouts = 8;
  cfg.horizon = 5;
  NominalSequence nominal = NominalSequence::constant(prm.hover(), cfg.horizon);
  RolloutBatch batch;
  std::atomic<int> calls{0};
  set_worker_count(1);
  auto diag = mppi_step(nominal, State{}, cfg, prm, StreamKey{2, 0, 0},
                        [&](const Rollout&) { return (++calls % 3 == 0) ? kInf : 1.0; }, batch);
  set_worker_count(0);
  CHECK(std::isfinite(diag.min_cost));
  for (const auto& u : nominal.controls) {
    CHECK(u.finite());
    CHECK(u.thrust <= prm.thrust_max);
  }
}

// ===========================================================================
// test_ensemble.cpp
// ===========================================================================
namespace {
std::vector<Vec3> wall_cloud() {  // test_ensemble.cpp:15-21
  std::vector<Vec3> pts;
  for (double y = -3.0; y <= 0.5; y += 0.08)
    for (double z = 0.5; z <= 3.5; z += 0.12) pts.emplace_back(4.0, y, z);
  return pts;
}
}  // namespace

KAT("single-instance ensemble equals one plain MPPI step", "test_ensemble.cpp:32") {
  EnsembleConfig cfg;
  cfg.grid.m_h = cfg.grid.m_v = 1;
  cfg.mppi.rollouts = 32;
  State x;
  x.p = Vec3(0, 0, 2);
  GoalSpec goal = GoalSpec::facing(x.p, Vec3(20, 0, 2));
  PerceptionSnapshot snap = build_snapshot_points({}, x);
  const ControlInput hover = cfg.dynamics.hover();
  auto plan = plan_step(x, goal, snap, cfg, NominalSequence{}, hover, 5, 77);
  AnchorGrid grid = cfg.grid;
  auto anchors = refine_endpoints(sample_initial_endpoints(x.p, goal.p_goal, grid), snap.coarse, snap.pose,
                                  grid.lookahead, cfg.weights.collision.d_max, grid.min_anchor_distance);
  auto guides = build_guides(anchors, x, hover, cfg.dynamics, grid.terminal_speed, cfg.mppi.horizon * cfg.mppi.dt);
  NominalSequence nominal = NominalSequence::constant(hover, cfg.mppi.horizon);
  RolloutBatch batch;
  mppi_step(nominal, x, cfg.mppi, cfg.dynamics, StreamKey{77, 0, 5},
            [&](const Rollout& r) {
              Rollout with_guide = r;
              with_guide.guide = &guides[0];
              return stage1_cost(with_guide, goal, snap.clearance_index, cfg.weights, hover);
            },
            batch);
  CHECK(plan.winner == 0);
  CHECK(plan.per_instance.size() == 1);
  for (int j = 0; j < cfg.mppi.horizon; ++j)
    CHECK((plan.per_instance[0].nominal.controls[j].vec() - nominal.controls[j].vec()).norm() == 0.0);
  CHECK((plan.control.vec() - clamp_control(nominal.controls.front(), cfg.dynamics).vec()).norm() == 0.0);
}

KAT("winner avoids the instance whose corridor is blocked", "test_ensemble.cpp:78") {
  EnsembleConfig cfg;
  cfg.grid.m_h = 2;
  cfg.grid.m_v = 1;
  cfg.mppi.rollouts = 64;
  State x;
  x.p = Vec3(0, 0, 2);
  x.v = Vec3(2.0, 0, 0);
  GoalSpec goal = GoalSpec::facing(x.p, Vec3(20, 0, 2));
  PerceptionSnapshot snap = build_snapshot_points(wall_cloud(), x);
  auto plan = plan_step(x, goal, snap, cfg, NominalSequence{}, cfg.dynamics.hover(), 0, 3);
  CHECK(plan.per_instance.size() == 2);
  CHECK(plan.winner == 1);
  CHECK(plan.per_instance[0].stage2 > plan.per_instance[1].stage2);
}

KAT("plan_step is deterministic and worker-count independent", "test_ensemble.cpp:100") {
  EnsembleConfig cfg;
  cfg.mppi.rollouts = 32;
  State x;
  x.p = Vec3(0, 0, 2);
  GoalSpec goal = GoalSpec::facing(x.p, Vec3(30, 5, 2));
  PerceptionSnapshot snap = build_snapshot_points(wall_cloud(), x);
  auto run = [&](unsigned workers) {
    set_worker_count(workers);
    auto plan = plan_step(x, goal, snap, cfg, NominalSequence{}, cfg.dynamics.hover(), 2, 9);
    set_worker_count(0);
    return plan;
  };
  auto a = run(1), b = run(2), c = run(5);
  CHECK(a.winner == b.winner && a.winner == c.winner);
  CHECK((a.control.vec() - b.control.vec()).norm() == 0.0);
  CHECK((a.control.vec() - c.control.vec()).norm() == 0.0);
  for (std::size_t m = 0; m < a.per_instance.size(); ++m) CHECK(a.per_instance[m].stage2 == b.per_instance[m].stage2);
}

KAT("stage-II optimality, bijection, and control feasibility", "test_ensemble.cpp:127") {
  EnsembleConfig cfg;
  cfg.mppi.rollouts = 32;
  State x;
  x.p = Vec3(0, 0, 2);
  GoalSpec goal = GoalSpec::facing(x.p, Vec3(25, -3, 2));
  PerceptionSnapshot snap = build_snapshot_points(wall_cloud(), x);
  NominalSequence previous;
  for (std::uint64_t cycle = 0; cycle < 5; ++cycle) {
    auto plan = plan_step(x, goal, snap, cfg, previous, cfg.dynamics.hover(), cycle, 31);
    CHECK(plan.winner >= 0);
    CHECK(plan.per_instance.size() == static_cast<std::size_t>(cfg.grid.count()));
    CHECK(plan.anchors.size() == plan.per_instance.size());
    CHECK(plan.guides.size() == plan.per_instance.size());
    for (const auto& rec : plan.per_instance)
      if (rec.valid) CHECK(plan.per_instance[plan.winner].stage2 <= rec.stage2);
    CHECK(plan.control.thrust >= cfg.dynamics.thrust_min && plan.control.thrust <= cfg.dynamics.thrust_max);
    CHECK(std::abs(plan.control.omega.x) <= cfg.dynamics.omega_xy_max);
    CHECK(std::abs(plan.control.omega.z) <= cfg.dynamics.omega_z_max);
    previous = plan.per_instance[plan.winner].nominal;
  }
}

KAT_SLOW("hover regulation stays bounded near the goal over 5 s", "test_ensemble.cpp:155") {
  EnsembleConfig cfg;
  World world;
  world.scene.kind = "empty";
  world.scene.start = Vec3(0, 0, 2);
  world.scene.goal = Vec3(0, 0, 2);
  world.lidar.r_max = cfg.r_max;
  EpisodeParams params;
  params.goal_radius = 0.0;
  params.timeout = 5.0;
  EpisodeState es = make_episode_state(world, cfg);
  GoalSpec goal;
  goal.p_goal = world.scene.goal;
  PlanScratch scratch;
  std::vector<Vec3> track;
  while (es.status == EpisodeStatus::running) {
    execute_cycle(es, world, goal, cfg, params, 13, scratch);
    track.push_back(es.x.p);
  }
  CHECK(es.status == EpisodeStatus::timeout);
  CHECK(track.size() == es.cycle);
  for (const auto& p : track) CHECK((p - world.scene.start).norm() <= 0.5);
}

KAT_SLOW("open-field goal is reached well before the timeout", "test_ensemble.cpp:217") {
  EnsembleConfig cfg;
  World world;
  world.scene.kind = "empty";
  world.lidar.r_max = cfg.r_max;
  EpisodeParams params;
  EpisodeState es = make_episode_state(world, cfg);
  GoalSpec goal = GoalSpec::facing(world.scene.start, world.scene.goal);
  PlanScratch scratch;
  while (es.status == EpisodeStatus::running && es.t < params.timeout + 1.0)
    execute_cycle(es, world, goal, cfg, params, 1, scratch);
  CHECK(es.status == EpisodeStatus::success);
  CHECK(es.t < 60.0);
  CHECK((es.x.p - world.scene.goal).norm() <= params.goal_radius);
}

// ===========================================================================
// acceptance.cpp hot-path criteria
// ===========================================================================
KAT("acceptance 1: quintic correctness (seed 1234)", "acceptance.cpp:57") {
  RandomStream rs(1234);
  for (int trial = 0; trial < 1000; ++trial) {
    BoundaryCondition s, e;
    for (int axis = 0; axis < 3; ++axis) {
      s.p[axis] = rs.uniform(-10, 10);
      s.v[axis] = rs.uniform(-5, 5);
      s.a[axis] = rs.uniform(-10, 10);
      e.p[axis] = rs.uniform(-10, 10);
      e.v[axis] = rs.uniform(-5, 5);
      e.a[axis] = rs.uniform(-10, 10);
    }
    const double T = rs.uniform(0.3, 3.0);
    const GuidingTrajectory g = solve_quintic(s, e, T);
    CHECK((eval_guide(g, 0.0) - s.p).norm() < 1e-9);
    CHECK((eval_guide_velocity(g, 0.0) - s.v).norm() < 1e-9);
    CHECK((eval_guide_acceleration(g, 0.0) - s.a).norm() < 1e-9);
    CHECK((eval_guide(g, T) - e.p).norm() < 1e-9);
    CHECK((eval_guide_velocity(g, T) - e.v).norm() < 1e-9);
    CHECK((eval_guide_acceleration(g, T) - e.a).norm() < 1e-9);
  }
}

KAT("acceptance 3: mppi weight law", "acceptance.cpp:114") {
  for (double w : compute_weights({3.0, 3.0, 3.0, 3.0, 3.0}, 0.1)) CHECK(std::abs(w - 0.2) <= 1e-12);
  const std::vector<double> costs{1.0, 2.0, 4.0, 8.0};
  auto base = compute_weights(costs, 0.1);
  for (double shift : {16.0, 1024.0, -64.0}) {
    std::vector<double> moved;
    for (double s : costs) moved.push_back(s + shift);
    auto w = compute_weights(moved, 0.1);
    for (std::size_t i = 0; i < w.size(); ++i) CHECK(w[i] == base[i]);
  }
  auto two = compute_weights({0.0, 0.1}, 0.1);
  CHECK(std::abs(two[0] - 0.73106) <= 1e-5);
  CHECK(std::abs(two[1] - 0.26894) <= 1e-5);
}

KAT("acceptance 4: collision-cost branch table", "acceptance.cpp:139") {
  CostWeights w;
  CHECK(collision_term(0.2, w) == 1.0e6);
  CHECK(collision_term(0.4, w) == 1.0e6);
  const double expected = 1.0e6 * std::exp(-1.0);
  CHECK(std::abs(collision_term(0.6, w) - expected) / expected <= 1e-6);
  CHECK(collision_term(1.0, w) == 0.0);
}

KAT("acceptance 5: partition oracle equivalence (seed 777)", "acceptance.cpp:152") {
  RandomStream rs(777);
  for (int trial = 0; trial < 100; ++trial) {
    std::vector<Vec3> cloud;
    cloud.reserve(10000);
    for (int k = 0; k < 10000; ++k) {
      const double x = rs.uniform(-12, 12), y = rs.uniform(-12, 12), z = rs.uniform(-12, 12);
      cloud.emplace_back(x, y, z);
    }
    const SphericalPartition part = build_partition(cloud, 10.0);
    BinOracle oracle(cloud, 10.0);
    bool ranges_ok = true;
    for (int f = 0; f < kCells; ++f) ranges_ok = ranges_ok && part.ranges[f] == oracle.ranges[f];
    CHECK(ranges_ok);
    const CoarsePartition coarse = pool_coarse(part);
    bool pool_ok = true;
    for (int I = 0; I < kCoarseAzimuthCells; ++I)
      for (int J = 0; J < kCoarseElevationCells; ++J) {
        double best = -1.0;
        int bi = 0, bj = 0;
        for (int i = I * kPoolFactor; i < (I + 1) * kPoolFactor; ++i)
          for (int j = J * kPoolFactor; j < (J + 1) * kPoolFactor; ++j)
            if (part.range(i, j) > best) {
              best = part.range(i, j);
              bi = i;
              bj = j;
            }
        const int f = CoarsePartition::flat(I, J);
        pool_ok = pool_ok && coarse.safe_range[f] == best && (coarse.safe_dir[f] - cell_direction(bi, bj)).norm() == 0.0;
      }
    CHECK(pool_ok);
    const FilteredCloud fc = filtered_cloud(part);
    const ClearanceIndex index(fc);
    bool clr_ok = true;
    for (int q = 0; q < 100; ++q) {
      const double x = rs.uniform(-14, 14), y = rs.uniform(-14, 14), z = rs.uniform(-14, 14);
      const Vec3 p(x, y, z);
      clr_ok = clr_ok && index.nearest(p) == clearance(fc, p);
    }
    CHECK(clr_ok);
  }
}

KAT_SLOW("acceptance 10: planning throughput (forest seed 1, median < 100 ms)", "acceptance.cpp:339") {
  const EnsembleConfig cfg;
  World world{generate_scenario(ScenarioKind::forest, 1), LidarModel{}};
  EpisodeState es = make_episode_state(world, cfg);
  const GoalSpec goal = GoalSpec::facing(world.scene.start, world.scene.goal);
  EpisodeParams params;
  PlanScratch scratch;
  for (int i = 0; i < 100 && es.status == EpisodeStatus::running; ++i)
    execute_cycle(es, world, goal, cfg, params, 1, scratch);
  std::vector<double> samples;
  for (int i = 0; i < 50 && es.status == EpisodeStatus::running; ++i) {
    es.buffer.push(lidar_scan(world.scene, es.x, world.lidar, mix64(1) + es.cycle));
    const auto t0 = std::chrono::steady_clock::now();
    PerceptionSnapshot snap = build_snapshot(es.buffer, es.x, cfg.r_max);
    auto plan = plan_step(es.x, goal, snap, cfg, es.nominal, es.last_applied, es.cycle, 1, scratch);
    es.nominal = plan.per_instance[plan.winner].nominal;
    const auto t1 = std::chrono::steady_clock::now();
    samples.push_back(1000.0 * std::chrono::duration<double>(t1 - t0).count());
    DynamicsParams step_prm = cfg.dynamics;
    step_prm.dt = 1.0 / cfg.replan_hz;
    es.x = rk4_step(es.x, es.nominal.controls.front(), step_prm);
    ++es.cycle;
  }
  std::sort(samples.begin(), samples.end());
  const double median = samples[samples.size() / 2];
  std::printf("    median build_snapshot+plan_step %.2f ms over %zu cycles, %u workers\n", median, samples.size(),
              worker_count());
  CHECK(median < 100.0);
}

// ===========================================================================
int main(int argc, char** argv) {
  bool slow = false;
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::strcmp(argv[i], "--slow") == 0)
      slow = true;
    else
      filter = argv[i];
  }
  int cases = 0, failed_cases = 0;
  for (const auto& c : registry()) {
    if (c.slow && !slow) continue;
    if (filter && std::strstr(c.name, filter) == nullptr) continue;
    g_current = c.name;
    const int before = g_failures;
    const auto t0 = std::chrono::steady_clock::now();
    c.fn();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ++cases;
    const bool ok = g_failures == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s (%s) %.2fs\n", ok ? "PASS" : "FAIL", c.name, c.origin, dt);
  }
  std::printf("%d cases, %d checks, %d failed checks, %d failed cases\n", cases, g_checks, g_failures,
              failed_cases);
  return failed_cases == 0 ? 0 : 1;
}
