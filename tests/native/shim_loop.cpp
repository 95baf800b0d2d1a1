// TEST PROGRAM (links the CPU oracle's C API for the synthetic world only).
//
// The reference's closed-loop cycle, execute_cycle (ensemble.cpp:245-305),
// written against the C++ shim include/amppi_b200.hpp exactly as a reference
// caller writes it: lidar_scan -> PointCloudBuffer::push -> build_snapshot ->
// plan_step(..., scratch) with hover fallback on "planning failed" ->
// rk4_step at 1/replan_hz.  Episodes run back to back with per-job configs
// from apply_velocity_cap (the run_batch pattern, metrics.cpp:141-147), on one
// thread, so the shim must re-apply each job's weights.  The world (scenario,
// LiDAR) comes from the oracle's restatement of sim_world.cpp via its C API.
//
// Phase 1 also checks value semantics of PerceptionSnapshot: a snapshot built
// before another one still plans to the same result.
//
// usage: shim_loop <kind> <scene_seed> <seed> <cycles> <cap> [<cap> ...]
// prints one JSON line per cycle.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/amppi_b200.hpp"
#include "../../oracle/oracle_capi.h"

using namespace amppi_b200;

namespace {

std::uint64_t mix64(std::uint64_t z) {  // rng.hpp
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

std::vector<Vec3> lidar_scan(void* scene, const State& x, double r_max, std::uint64_t frame_seed) {
  const double x10[10] = {x.p[0], x.p[1], x.p[2], x.q[0], x.q[1], x.q[2], x.q[3], x.v[0], x.v[1], x.v[2]};
  std::vector<double> buf(3 * 4096);
  const std::int64_t n = oracle_lidar_scan(scene, x10, frame_seed, r_max, buf.data(), 4096);
  std::vector<Vec3> out(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) out[i] = {buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]};
  return out;
}

EnsembleConfig base_config() {  // BASELINE C1/C2 sizes
  EnsembleConfig cfg;
  cfg.grid.m_h = 4;
  cfg.grid.m_v = 2;
  cfg.mppi.rollouts = 256;
  cfg.mppi.horizon = 30;
  return cfg;
}

void print_plan(const char* tag, double cap, std::uint64_t cycle, int winner, const ControlInput& u, double stage2,
                const State& x) {
  std::printf(
      "{\"tag\": \"%s\", \"cap\": %.17g, \"cycle\": %llu, \"winner\": %d, \"control\": [%.17g, %.17g, %.17g, %.17g], "
      "\"stage2\": %.17g, \"x\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g]}\n",
      tag, cap, static_cast<unsigned long long>(cycle), winner, u.thrust, u.omega[0], u.omega[1], u.omega[2], stage2,
      x.p[0], x.p[1], x.p[2], x.q[0], x.q[1], x.q[2], x.q[3], x.v[0], x.v[1], x.v[2]);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s kind scene_seed seed cycles cap [cap ...]\n", argv[0]);
    return 2;
  }
  const int kind = std::atoi(argv[1]);
  const std::uint64_t scene_seed = std::strtoull(argv[2], nullptr, 10);
  const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  const int cycles = std::atoi(argv[4]);
  void* scene = oracle_scene_new(kind, scene_seed);
  const Vec3 start{0.0, 0.0, 2.0}, target{45.0, 0.0, 2.0};  // Scenario::start / goal

  // phase 1: snapshot value semantics
  {
    const EnsembleConfig cfg = base_config();
    State x;
    x.p = start;
    const GoalSpec goal = GoalSpec::facing(start, target);
    PointCloudBuffer ba(10), bb(10);
    ba.push(lidar_scan(scene, x, cfg.r_max, 11));
    State y = x;
    y.p = {6.0, -1.0, 2.0};
    bb.push(lidar_scan(scene, y, cfg.r_max, 12));
    const PerceptionSnapshot a = build_snapshot(ba, x, cfg.r_max);
    const PlanResult first = plan_step(x, goal, a, cfg, NominalSequence{}, cfg.dynamics.hover(), 3, seed);
    const PerceptionSnapshot b = build_snapshot(bb, y, cfg.r_max);
    const PlanResult other = plan_step(y, goal, b, cfg, NominalSequence{}, cfg.dynamics.hover(), 3, seed);
    const PlanResult again = plan_step(x, goal, a, cfg, NominalSequence{}, cfg.dynamics.hover(), 3, seed);
    print_plan("snap_first", 0.0, 3, first.winner, first.control, first.per_instance[first.winner].stage2, x);
    print_plan("snap_other", 0.0, 3, other.winner, other.control, other.per_instance[other.winner].stage2, y);
    print_plan("snap_again", 0.0, 3, again.winner, again.control, again.per_instance[again.winner].stage2, x);
  }

  // phase 2: back-to-back episodes with per-job velocity caps
  for (int a = 5; a < argc; ++a) {
    const double cap = std::atof(argv[a]);
    const EnsembleConfig cfg = apply_velocity_cap(base_config(), cap);
    // make_episode_state (ensemble.cpp:238-243)
    State x;
    x.p = start;
    ControlInput last_applied = cfg.dynamics.hover();
    PointCloudBuffer buffer(10);
    NominalSequence nominal;
    PlanScratch scratch;
    const GoalSpec goal = GoalSpec::facing(start, target);
    for (std::uint64_t cycle = 0; cycle < static_cast<std::uint64_t>(cycles); ++cycle) {
      // execute_cycle (ensemble.cpp:245-305)
      buffer.push(lidar_scan(scene, x, cfg.r_max, mix64(seed) + cycle));
      const PerceptionSnapshot snap = build_snapshot(buffer, x, cfg.r_max);
      ControlInput u = cfg.dynamics.hover();
      int winner = -1;
      double stage2 = HUGE_VAL;
      try {
        PlanResult plan = plan_step(x, goal, snap, cfg, nominal, last_applied, cycle, seed, scratch);
        u = plan.control;
        winner = plan.winner;
        stage2 = plan.per_instance[plan.winner].stage2;
        nominal = std::move(plan.per_instance[plan.winner].nominal);
      } catch (const std::runtime_error&) {
      }
      print_plan("loop", cap, cycle, winner, u, stage2, x);
      DynamicsParams step_prm = cfg.dynamics;
      step_prm.dt = 1.0 / cfg.replan_hz;
      x = rk4_step(x, u, step_prm);
      last_applied = u;
    }
  }
  oracle_scene_free(scene);
  return 0;
}
