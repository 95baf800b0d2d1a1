// Reference-style use of the C++ shim (include/amppi_b200.hpp): the
// test_ensemble.cpp:127-153 scenario (wall of points 4 m ahead, goal
// (25,-3,2), 5 cycles feeding the winner nominal back).  Prints one JSON line
// per cycle: winner, control, winner stage-2 cost.
#include <cstdio>
#include <vector>

#include "../include/amppi_b200.hpp"

using namespace amppi_b200;

int main() {
  EnsembleConfig cfg;
  cfg.mppi.rollouts = 32;
  std::vector<Vec3> wall;
  for (double y = -3.0; y <= 0.5; y += 0.08)
    for (double z = 0.5; z <= 3.5; z += 0.12) wall.push_back({4.0, y, z});
  PointCloudBuffer buffer;
  buffer.push(wall);
  State x;
  x.p = {0, 0, 2};
  const GoalSpec goal = GoalSpec::facing(x.p, {25, -3, 2});
  NominalSequence previous;
  PlanScratch scratch;  // reused across cycles, as execute_cycle does
  for (std::uint64_t cycle = 0; cycle < 5; ++cycle) {
    const PerceptionSnapshot snap = build_snapshot(buffer, x, cfg.r_max);
    try {
      const PlanResult plan = plan_step(x, goal, snap, cfg, previous, cfg.dynamics.hover(), cycle, 31, scratch);
      std::printf("{\"cycle\": %llu, \"winner\": %d, \"control\": [%.17g, %.17g, %.17g, %.17g], \"stage2\": %.17g}\n",
                  static_cast<unsigned long long>(cycle), plan.winner, plan.control.thrust, plan.control.omega[0],
                  plan.control.omega[1], plan.control.omega[2], plan.per_instance[plan.winner].stage2);
      previous = plan.per_instance[plan.winner].nominal;
    } catch (const std::runtime_error& e) {
      std::printf("{\"cycle\": %llu, \"error\": \"%s\"}\n", static_cast<unsigned long long>(cycle), e.what());
    }
  }
  return 0;
}
