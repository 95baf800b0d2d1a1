/* CPU ORACLE C API — TEST INFRASTRUCTURE ONLY.
 *
 * ctypes entry points into the oracle restatement (oracle.hpp) for tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg.  Layouts:
 *   state  = double[10]  p(3), q(w,x,y,z), v(3)
 *   control= double[4]   thrust, omega(3)
 *   oracle_config mirrors amppi_config in include/amppi_b200.h field for field.
 */
#ifndef AMPPI_ORACLE_CAPI_H
#define AMPPI_ORACLE_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t m_h, m_v;
  double lookahead, spacing_deg, terminal_speed, min_anchor_distance;
  int32_t rollouts, horizon;
  double lambda;
  double sigma[4];
  double mppi_dt;
  int32_t iterations;
  double q_track, q_vnorm, q_c, q_c_delta, q_p, q_v, q_q;
  double col_scale, col_slope, col_d_min, col_d_max;
  double mass;
  double gravity[3];
  double dyn_dt;
  double thrust_min, thrust_max, omega_xy_max, omega_z_max;
  double replan_hz, r_max;
} oracle_config;

typedef struct {
  int32_t* winner;
  double* control;
  double* stage1;
  double* stage2;
  double* ess;
  uint8_t* valid;
  double* nominal;          /* M*N*4, NaN for invalid instances */
  double* anchor_initial;   /* M*3 */
  double* anchor_refined;   /* M*3 */
  double* anchor_safe_dir;  /* M*3 */
  double* anchor_safe_range;/* M */
  int32_t* anchor_ij;       /* M*2 */
  double* guide_coeffs;     /* M*3*6 [m][axis][k] */
  double* breakdown;        /* 5: track, vnorm, ctrl, goal, collision */
  double* winner_states;    /* (N+1)*10 */
  double* sample_costs;     /* M*K, last iteration */
  double* sample_margin;    /* M*K */
} oracle_plan_out;

void oracle_config_default(oracle_config* cfg);
void oracle_set_workers(unsigned n);
unsigned oracle_workers(void);

void* oracle_snapshot_new(const double* world_pts, int64_t n, const double* pose10, double r_max);
void oracle_snapshot_free(void* snap);
int64_t oracle_snapshot_filtered_count(void* snap);
void oracle_snapshot_get(void* snap, double* ranges, uint8_t* has_point, double* nearest,
                         double* safe_range, double* safe_dir, double* safe_point, double* filtered);
double oracle_snapshot_nearest(void* snap, const double* p3);

int oracle_plan(void* snap, const oracle_config* cfg, const double* x10, const double* goal_p,
                const double* goal_v, const double* goal_q, const double* prev, int32_t prev_len,
                const double* last_applied, uint64_t cycle, uint64_t seed, const double* injected,
                oracle_plan_out* out);

/* Per-rollout perturbations exactly as sample_rollout_perturbations draws them. */
void oracle_perturbations(const oracle_config* cfg, uint64_t seed, uint64_t instance, uint64_t cycle,
                          int32_t k, double* out /* N*4 */);
void oracle_goal_facing(const double* from3, const double* target3, double* q_out4);

void* oracle_scene_new(int32_t kind, uint64_t seed);
void oracle_scene_free(void* scene);
int64_t oracle_scene_obstacle_count(void* scene);
int64_t oracle_lidar_scan(void* scene, const double* pose10, uint64_t frame_seed, double r_max,
                          double* out, int64_t cap);
double oracle_true_clearance(void* scene, const double* p3);

void* oracle_loop_new(int32_t kind, uint64_t scene_seed, const oracle_config* cfg, uint64_t seed,
                      int32_t buffer_capacity);
int64_t oracle_loop_run(void* loop, int64_t cycles);
int32_t oracle_loop_status(void* loop);
int64_t oracle_loop_records(void* loop);
int64_t oracle_loop_cloud_size(void* loop, int64_t idx);
void oracle_loop_get(void* loop, int64_t idx, double* cloud, double* x10, double* prev,
                     int32_t* prev_len, double* last_applied, uint64_t* cycle, int32_t* planned,
                     int32_t* winner, double* control, double* stage2, double* winner_nominal);
void oracle_loop_goal(void* loop, double* goal_p, double* goal_v, double* goal_q);
void oracle_loop_state(void* loop, double* x10);
void oracle_loop_free(void* loop);

#ifdef __cplusplus
}
#endif
#endif
