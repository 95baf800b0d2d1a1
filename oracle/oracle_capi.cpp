// CPU ORACLE C API — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
#include "oracle_capi.h"

#include <cmath>
#include <memory>
#include <stdexcept>

#include "oracle.hpp"

using namespace oracle;

namespace {

EnsembleConfig to_cfg(const oracle_config* c) {
  EnsembleConfig e;
  e.grid.m_h = c->m_h;
  e.grid.m_v = c->m_v;
  e.grid.lookahead = c->lookahead;
  e.grid.spacing_deg = c->spacing_deg;
  e.grid.terminal_speed = c->terminal_speed;
  e.grid.min_anchor_distance = c->min_anchor_distance;
  e.mppi.rollouts = c->rollouts;
  e.mppi.horizon = c->horizon;
  e.mppi.lambda = c->lambda;
  e.mppi.sigma = Vec4(c->sigma[0], c->sigma[1], c->sigma[2], c->sigma[3]);
  e.mppi.dt = c->mppi_dt;
  e.mppi.iterations = c->iterations;
  e.weights.q_track = c->q_track;
  e.weights.q_vnorm = c->q_vnorm;
  e.weights.q_c = c->q_c;
  e.weights.q_c_delta = c->q_c_delta;
  e.weights.q_p = c->q_p;
  e.weights.q_v = c->q_v;
  e.weights.q_q = c->q_q;
  e.weights.collision.scale = c->col_scale;
  e.weights.collision.slope = c->col_slope;
  e.weights.collision.d_min = c->col_d_min;
  e.weights.collision.d_max = c->col_d_max;
  e.dynamics.mass = c->mass;
  e.dynamics.gravity = Vec3(c->gravity[0], c->gravity[1], c->gravity[2]);
  e.dynamics.dt = c->dyn_dt;
  e.dynamics.thrust_min = c->thrust_min;
  e.dynamics.thrust_max = c->thrust_max;
  e.dynamics.omega_xy_max = c->omega_xy_max;
  e.dynamics.omega_z_max = c->omega_z_max;
  e.replan_hz = c->replan_hz;
  e.r_max = c->r_max;
  return e;
}

State to_state(const double* s) {
  State x;
  x.p = Vec3(s[0], s[1], s[2]);
  x.q = Quat(s[3], s[4], s[5], s[6]);
  x.v = Vec3(s[7], s[8], s[9]);
  return x;
}

void from_state(const State& x, double* s) {
  s[0] = x.p.x; s[1] = x.p.y; s[2] = x.p.z;
  s[3] = x.q.w; s[4] = x.q.x; s[5] = x.q.y; s[6] = x.q.z;
  s[7] = x.v.x; s[8] = x.v.y; s[9] = x.v.z;
}

void put3(const Vec3& v, double* o) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
}

void put4(const ControlInput& u, double* o) {
  o[0] = u.thrust;
  o[1] = u.omega.x;
  o[2] = u.omega.y;
  o[3] = u.omega.z;
}

struct Loop {
  World world;
  EnsembleConfig cfg;
  EpisodeParams params;
  EpisodeState es;
  GoalSpec goal;
  PlanScratch scratch;
  std::uint64_t seed{0};
  std::vector<CycleRecord> records;
};

}  // namespace

extern "C" {

void oracle_config_default(oracle_config* c) {
  const EnsembleConfig e;
  c->m_h = e.grid.m_h;
  c->m_v = e.grid.m_v;
  c->lookahead = e.grid.lookahead;
  c->spacing_deg = e.grid.spacing_deg;
  c->terminal_speed = e.grid.terminal_speed;
  c->min_anchor_distance = e.grid.min_anchor_distance;
  c->rollouts = e.mppi.rollouts;
  c->horizon = e.mppi.horizon;
  c->lambda = e.mppi.lambda;
  for (int i = 0; i < 4; ++i) c->sigma[i] = e.mppi.sigma[i];
  c->mppi_dt = e.mppi.dt;
  c->iterations = e.mppi.iterations;
  c->q_track = e.weights.q_track;
  c->q_vnorm = e.weights.q_vnorm;
  c->q_c = e.weights.q_c;
  c->q_c_delta = e.weights.q_c_delta;
  c->q_p = e.weights.q_p;
  c->q_v = e.weights.q_v;
  c->q_q = e.weights.q_q;
  c->col_scale = e.weights.collision.scale;
  c->col_slope = e.weights.collision.slope;
  c->col_d_min = e.weights.collision.d_min;
  c->col_d_max = e.weights.collision.d_max;
  c->mass = e.dynamics.mass;
  c->gravity[0] = e.dynamics.gravity.x;
  c->gravity[1] = e.dynamics.gravity.y;
  c->gravity[2] = e.dynamics.gravity.z;
  c->dyn_dt = e.dynamics.dt;
  c->thrust_min = e.dynamics.thrust_min;
  c->thrust_max = e.dynamics.thrust_max;
  c->omega_xy_max = e.dynamics.omega_xy_max;
  c->omega_z_max = e.dynamics.omega_z_max;
  c->replan_hz = e.replan_hz;
  c->r_max = e.r_max;
}

void oracle_set_workers(unsigned n) { set_worker_count(n); }
unsigned oracle_workers(void) { return worker_count(); }

void* oracle_snapshot_new(const double* pts, int64_t n, const double* pose10, double r_max) {
  std::vector<Vec3> cloud(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) cloud[i] = Vec3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  return new PerceptionSnapshot(build_snapshot_points(cloud, to_state(pose10), r_max));
}

void oracle_snapshot_free(void* s) { delete static_cast<PerceptionSnapshot*>(s); }

int64_t oracle_snapshot_filtered_count(void* s) {
  return static_cast<int64_t>(static_cast<PerceptionSnapshot*>(s)->filtered.points.size());
}

void oracle_snapshot_get(void* sp, double* ranges, uint8_t* has_point, double* nearest,
                         double* safe_range, double* safe_dir, double* safe_point, double* filtered) {
  const auto& s = *static_cast<PerceptionSnapshot*>(sp);
  for (int f = 0; f < kCells; ++f) {
    if (ranges) ranges[f] = s.partition.ranges[f];
    if (has_point) has_point[f] = s.partition.has_point[f];
    if (nearest) put3(s.partition.nearest[f], nearest + 3 * f);
  }
  for (int f = 0; f < kCoarseCells; ++f) {
    if (safe_range) safe_range[f] = s.coarse.safe_range[f];
    if (safe_dir) put3(s.coarse.safe_dir[f], safe_dir + 3 * f);
    if (safe_point) put3(s.coarse.safe_point[f], safe_point + 3 * f);
  }
  if (filtered)
    for (std::size_t i = 0; i < s.filtered.points.size(); ++i) put3(s.filtered.points[i], filtered + 3 * i);
}

double oracle_snapshot_nearest(void* sp, const double* p) {
  return static_cast<PerceptionSnapshot*>(sp)->clearance_index.nearest(Vec3(p[0], p[1], p[2]));
}

int oracle_plan(void* sp, const oracle_config* c, const double* x10, const double* goal_p,
                const double* goal_v, const double* goal_q, const double* prev, int32_t prev_len,
                const double* last_applied, uint64_t cycle, uint64_t seed, const double* injected,
                oracle_plan_out* out) {
  const auto& snap = *static_cast<PerceptionSnapshot*>(sp);
  const EnsembleConfig cfg = to_cfg(c);
  const State x = to_state(x10);
  GoalSpec goal;
  goal.p_goal = Vec3(goal_p[0], goal_p[1], goal_p[2]);
  goal.v_goal = Vec3(goal_v[0], goal_v[1], goal_v[2]);
  goal.q_goal = Quat(goal_q[0], goal_q[1], goal_q[2], goal_q[3]);
  NominalSequence previous;
  for (int j = 0; j < prev_len; ++j)
    previous.controls.push_back(ControlInput::from_vec(Vec4(prev[4 * j], prev[4 * j + 1], prev[4 * j + 2], prev[4 * j + 3])));
  const ControlInput la = ControlInput::from_vec(Vec4(last_applied[0], last_applied[1], last_applied[2], last_applied[3]));

  const int M = cfg.grid.count(), K = cfg.mppi.rollouts, N = cfg.mppi.horizon;
  std::vector<Vec4> inj;
  PlanDebug dbg;
  if (injected) {
    const std::size_t total = static_cast<std::size_t>(cfg.mppi.iterations) * M * K * N;
    inj.resize(total);
    for (std::size_t i = 0; i < total; ++i)
      inj[i] = Vec4(injected[4 * i], injected[4 * i + 1], injected[4 * i + 2], injected[4 * i + 3]);
    dbg.injected_delta = &inj;
  }
  PlanScratch scratch;
  PlanResult r;
  int rc = 0;
  try {
    r = plan_step(x, goal, snap, cfg, previous, la, cycle, seed, scratch, &dbg);
  } catch (const std::runtime_error&) {
    rc = 1;
  }
  if (!out) return rc;
  if (out->sample_costs)
    for (std::size_t i = 0; i < dbg.stage1_costs.size(); ++i) out->sample_costs[i] = dbg.stage1_costs[i];
  if (out->sample_margin)
    for (std::size_t i = 0; i < dbg.collision_margin.size(); ++i) out->sample_margin[i] = dbg.collision_margin[i];
  if (rc != 0) return rc;
  if (out->winner) *out->winner = r.winner;
  if (out->control) put4(r.control, out->control);
  for (int m = 0; m < M; ++m) {
    const InstanceRecord& rec = r.per_instance[m];
    if (out->stage1) out->stage1[m] = rec.stage1;
    if (out->stage2) out->stage2[m] = rec.stage2;
    if (out->ess) out->ess[m] = rec.ess;
    if (out->valid) out->valid[m] = rec.valid ? 1 : 0;
    if (out->nominal)
      for (int j = 0; j < N; ++j) {
        double* o = out->nominal + (static_cast<std::size_t>(m) * N + j) * 4;
        if (rec.valid)
          put4(rec.nominal.controls[j], o);
        else
          o[0] = o[1] = o[2] = o[3] = std::nan("");
      }
    const Anchor& a = r.anchors[m];
    if (out->anchor_initial) put3(a.initial_endpoint, out->anchor_initial + 3 * m);
    if (out->anchor_refined) put3(a.refined_endpoint, out->anchor_refined + 3 * m);
    if (out->anchor_safe_dir) put3(a.safe_dir, out->anchor_safe_dir + 3 * m);
    if (out->anchor_safe_range) out->anchor_safe_range[m] = a.safe_range;
    if (out->anchor_ij) {
      out->anchor_ij[2 * m] = a.coarse_i;
      out->anchor_ij[2 * m + 1] = a.coarse_j;
    }
    if (out->guide_coeffs)
      for (int axis = 0; axis < 3; ++axis)
        for (int k = 0; k < 6; ++k) out->guide_coeffs[(m * 3 + axis) * 6 + k] = r.guides[m].coeffs[k][axis];
  }
  if (out->breakdown) {
    out->breakdown[0] = r.breakdown.track;
    out->breakdown[1] = r.breakdown.vnorm;
    out->breakdown[2] = r.breakdown.ctrl;
    out->breakdown[3] = r.breakdown.goal;
    out->breakdown[4] = r.breakdown.collision;
  }
  if (out->winner_states)
    for (int t = 0; t <= N; ++t) from_state(r.winner_rollout.states[t], out->winner_states + 10 * t);
  return 0;
}

void oracle_perturbations(const oracle_config* c, uint64_t seed, uint64_t instance, uint64_t cycle,
                          int32_t k, double* out) {
  const EnsembleConfig cfg = to_cfg(c);
  std::vector<Vec4> d(cfg.mppi.horizon);
  sample_rollout_perturbations(cfg.mppi, StreamKey{seed, instance, cycle}, k, d);
  for (int j = 0; j < cfg.mppi.horizon; ++j)
    for (int cc = 0; cc < 4; ++cc) out[4 * j + cc] = d[j][cc];
}

void oracle_goal_facing(const double* from, const double* target, double* q) {
  const GoalSpec g = GoalSpec::facing(Vec3(from[0], from[1], from[2]), Vec3(target[0], target[1], target[2]));
  q[0] = g.q_goal.w;
  q[1] = g.q_goal.x;
  q[2] = g.q_goal.y;
  q[3] = g.q_goal.z;
}

void* oracle_scene_new(int32_t kind, uint64_t seed) {
  return new Scenario(generate_scenario(static_cast<ScenarioKind>(kind), seed));
}
void oracle_scene_free(void* s) { delete static_cast<Scenario*>(s); }
int64_t oracle_scene_obstacle_count(void* s) {
  return static_cast<int64_t>(static_cast<Scenario*>(s)->obstacles.size());
}

int64_t oracle_lidar_scan(void* s, const double* pose10, uint64_t frame_seed, double r_max,
                          double* out, int64_t cap) {
  LidarModel model;
  model.r_max = r_max;
  const auto pts = lidar_scan(*static_cast<Scenario*>(s), to_state(pose10), model, frame_seed);
  const int64_t n = static_cast<int64_t>(pts.size());
  for (int64_t i = 0; i < n && i < cap; ++i) put3(pts[i], out + 3 * i);
  return n;
}

double oracle_true_clearance(void* s, const double* p) {
  return true_clearance(*static_cast<Scenario*>(s), Vec3(p[0], p[1], p[2]));
}

void* oracle_loop_new(int32_t kind, uint64_t scene_seed, const oracle_config* c, uint64_t seed,
                      int32_t buffer_capacity) {
  auto* L = new Loop();
  L->world.scene = generate_scenario(static_cast<ScenarioKind>(kind), scene_seed);
  L->cfg = to_cfg(c);
  L->world.lidar.r_max = L->cfg.r_max;
  L->es = make_episode_state(L->world, L->cfg);
  L->es.buffer = PointCloudBuffer(static_cast<std::size_t>(buffer_capacity));
  L->es.recorder = &L->records;
  L->goal = GoalSpec::facing(L->world.scene.start, L->world.scene.goal);
  L->seed = seed;
  return L;
}

int64_t oracle_loop_run(void* lp, int64_t cycles) {
  auto* L = static_cast<Loop*>(lp);
  int64_t n = 0;
  for (; n < cycles && L->es.status == EpisodeStatus::running; ++n)
    execute_cycle(L->es, L->world, L->goal, L->cfg, L->params, L->seed, L->scratch);
  return n;
}

int32_t oracle_loop_status(void* lp) { return static_cast<int32_t>(static_cast<Loop*>(lp)->es.status); }
int64_t oracle_loop_records(void* lp) { return static_cast<int64_t>(static_cast<Loop*>(lp)->records.size()); }
int64_t oracle_loop_cloud_size(void* lp, int64_t idx) {
  return static_cast<int64_t>(static_cast<Loop*>(lp)->records.at(idx).cloud.size());
}

void oracle_loop_get(void* lp, int64_t idx, double* cloud, double* x10, double* prev, int32_t* prev_len,
                     double* last_applied, uint64_t* cycle, int32_t* planned, int32_t* winner,
                     double* control, double* stage2, double* winner_nominal) {
  const CycleRecord& r = static_cast<Loop*>(lp)->records.at(idx);
  if (cloud)
    for (std::size_t i = 0; i < r.cloud.size(); ++i) put3(r.cloud[i], cloud + 3 * i);
  if (x10) from_state(r.x, x10);
  if (prev_len) *prev_len = static_cast<int32_t>(r.previous.controls.size());
  if (prev)
    for (std::size_t j = 0; j < r.previous.controls.size(); ++j) put4(r.previous.controls[j], prev + 4 * j);
  if (last_applied) put4(r.last_applied, last_applied);
  if (cycle) *cycle = r.cycle;
  if (planned) *planned = r.planned ? 1 : 0;
  if (winner) *winner = r.winner;
  if (control) put4(r.control, control);
  if (stage2) *stage2 = r.stage2;
  if (winner_nominal)
    for (std::size_t j = 0; j < r.winner_nominal.controls.size(); ++j)
      put4(r.winner_nominal.controls[j], winner_nominal + 4 * j);
}

void oracle_loop_goal(void* lp, double* gp, double* gv, double* gq) {
  const GoalSpec& g = static_cast<Loop*>(lp)->goal;
  put3(g.p_goal, gp);
  put3(g.v_goal, gv);
  gq[0] = g.q_goal.w;
  gq[1] = g.q_goal.x;
  gq[2] = g.q_goal.y;
  gq[3] = g.q_goal.z;
}

void oracle_loop_state(void* lp, double* x10) { from_state(static_cast<Loop*>(lp)->es.x, x10); }

void oracle_loop_free(void* lp) { delete static_cast<Loop*>(lp); }

}  // extern "C"
