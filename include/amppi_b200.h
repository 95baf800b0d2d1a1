/* amppi_b200 — B200-native AERO-MPPI plan-cycle hot path, C ABI.
 *
 * Drop-in boundary for the reference planner's two hot-path entry points:
 *
 *   PerceptionSnapshot build_snapshot(const PointCloudBuffer&, const State& pose,
 *                                     double r_max = 10.0);
 *       proj/include/amppi/perception.hpp:142-143, proj/src/perception.cpp:237-246
 *       -> amppi_snapshot() / amppi_snapshot_f64()
 *
 *   PlanResult plan_step(const State& x, const GoalSpec& goal,
 *                        const PerceptionSnapshot& snap, const EnsembleConfig& cfg,
 *                        const NominalSequence& previous,
 *                        const ControlInput& last_applied, std::uint64_t cycle,
 *                        std::uint64_t seed, PlanScratch& scratch);
 *       proj/include/amppi/ensemble.hpp:59-69, proj/src/ensemble.cpp:29-179
 *       -> amppi_plan()
 *
 * plus a batched-scene form of the same cycle (amppi_cycle_batch*, SURVEY.md
 * §8 config C5).  Plain C types only: pointers, sizes, POD structs.  No
 * exceptions cross the ABI; every call returns an amppi_status and the
 * message of the last failure is available from amppi_last_error().  The C++
 * shim include/amppi_b200.hpp re-creates the reference signatures and
 * exceptions on top of this header.
 *
 * Threading: one context per host thread; calls on one context are
 * serialised by the caller.  Host-pointer calls are synchronous (outputs are
 * in caller memory on return); *_device calls are asynchronous on the
 * context's stream.
 */
#ifndef AMPPI_B200_H
#define AMPPI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMPPI_ABI_VERSION 2

typedef enum {
  AMPPI_OK = 0,
  AMPPI_PLANNING_FAILED = 1,   /* every instance invalid: std::runtime_error("planning failed"), ensemble.cpp:158 */
  AMPPI_INVALID_ARGUMENT = 2,  /* std::invalid_argument */
  AMPPI_CUDA_ERROR = 3,
  AMPPI_NCCL_ERROR = 4,
  AMPPI_NO_SNAPSHOT = 5        /* amppi_plan before any amppi_snapshot */
} amppi_status;

/* Plain mirror of EnsembleConfig (ensemble.hpp:16-23) and its nested
 * AnchorGrid (guidance.hpp:10-19), MppiConfig (mppi.hpp:14-21), CostWeights /
 * CollisionParams (costs.hpp:13-29) and DynamicsParams (types.hpp:40-53).
 * mppi_dt is MppiConfig::dt (guide horizon N*dt); dyn_dt is DynamicsParams::dt
 * (RK4 step, tracking-cost time base) — they are distinct in the reference. */
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
} amppi_config;

/* State x = [p, q, v]; q scalar-first (w, x, y, z) as in types.hpp:13-26. */
typedef struct {
  double p[3];
  double q[4];
  double v[3];
} amppi_state;

/* ControlInput (types.hpp:29-38): collective thrust [N], body rates [rad/s]. */
typedef struct {
  double thrust;
  double omega[3];
} amppi_control;

/* GoalSpec (costs.hpp:42-56). */
typedef struct {
  double p_goal[3];
  double v_goal[3];
  double q_goal[4];
} amppi_goal;

/* Schedule knobs: they change how a call is split over streams and chunks,
 * never its results (tests drive every path with them).  0 = automatic. */
typedef struct {
  int32_t pipeline_chunks;   /* amppi_cycle_batch: host-upload pipeline chunks (auto: up to 6) */
  double pipeline_ratio;     /* growth ratio of successive pipeline chunks (auto: 1.2; >= 1) */
  int32_t pipeline_streams;  /* compute streams chunks rotate over, 2..4 (auto: 3) */
  int32_t device_chunks;     /* amppi_cycle_batch_device: concurrent chunks (auto: up to 2) */
  int32_t chunk_gather;      /* host pipeline: gather each chunk's results as it finishes (auto/1) or once (-1) */
  int32_t loop_graph;        /* closed loop: replay one captured cycle as a CUDA graph (auto/1) or launch (-1) */
  int32_t plan_graph;        /* amppi_plan: replay the plan kernels as a cached CUDA graph (auto/1) or launch (-1) */
  int32_t trace;             /* 1: print the host pipeline's upload / compute timeline to stderr */
} amppi_schedule;

typedef struct {
  int32_t device;          /* CUDA ordinal */
  int32_t precision;       /* 32: FP32 stage-I screening + FP64 softmin support (default)
                              64: FP64 stage I */
  int32_t max_scenes;      /* batch capacity (>= 1) */
  int64_t max_points;      /* total point capacity over a batch */
  int32_t profile;         /* 1: time every kernel with CUDA events */
  void* stream;            /* optional cudaStream_t to launch on; NULL: own stream */
  int64_t refine_split_cap;/* FP64 refine: support pairs taken by the split (trajectory | collision)
                              kernels before the fused overflow kernel; -1 = automatic (4 per instance) */
  amppi_schedule schedule;
} amppi_options;

/* PlanResult (ensemble.hpp:33-41) as caller-owned buffers; any pointer may be
 * NULL.  Sizes: M = m_h*m_v, N = horizon, K = rollouts. */
typedef struct {
  int32_t winner;              /* out */
  amppi_control control;       /* out: clamp(nominal_winner[0]) */
  double breakdown[5];         /* out: track, vnorm, ctrl, goal, collision (costs.hpp:165-187) */
  double* stage1;              /* [M] InstanceRecord::stage1 */
  double* stage2;              /* [M] InstanceRecord::stage2 (+inf when invalid) */
  double* ess;                 /* [M] */
  uint8_t* valid;              /* [M] */
  double* nominal;             /* [M*N*4] updated nominal per instance (NaN when invalid) */
  double* winner_states;       /* [(N+1)*10] winner_rollout states p,q(wxyz),v */
  double* winner_controls;     /* [N*4] winner_rollout controls */
  double* anchor_initial;      /* [M*3] Anchor::initial_endpoint */
  double* anchor_refined;      /* [M*3] */
  double* anchor_safe_dir;     /* [M*3] */
  double* anchor_safe_range;   /* [M] */
  int32_t* anchor_ij;          /* [M*2] coarse (I, J) */
  double* guide_coeffs;        /* [M*3*6] GuidingTrajectory::coeffs, [m][axis][power] */
  double* sample_costs;        /* [M*K] stage-I screening cost of every sample, last iteration (verification);
                                  a sample with a clearance within the d_max band reports a lower bound */
} amppi_plan_result;

/* Snapshot contents for verification (SphericalPartition / CoarsePartition /
 * FilteredCloud, perception.hpp:60-94).  Cell arrays use flat(i,j)=i*60+j. */
typedef struct {
  double* ranges;              /* [7200] */
  uint8_t* has_point;          /* [7200] */
  double* nearest;             /* [7200*3] body frame (0 where empty) */
  double* safe_range;          /* [200] flat(I,J)=I*10+J */
  double* safe_dir;            /* [200*3] body frame */
  double* safe_point;          /* [200*3] */
  double* filtered;            /* [<=7200*3] world frame, flat-cell order */
  int64_t n_filtered;          /* out */
} amppi_snapshot_view;

/* Batched scenes: scene s owns points [point_offsets[s], point_offsets[s+1]).
 * Host-pointer form (amppi_cycle_batch) copies inputs in and results out;
 * device form (amppi_cycle_batch_device) takes device pointers for every
 * array and enqueues on the context stream. */
typedef struct {
  int32_t n_scenes;
  const int64_t* point_offsets;     /* [n_scenes+1] */
  const float* xyz;                 /* [total*3] world frame, float32 */
  const amppi_state* poses;         /* [n_scenes] snapshot pose */
  const amppi_state* states;        /* [n_scenes] plan state x */
  const amppi_goal* goals;          /* [n_scenes] */
  const double* previous;           /* [n_scenes*N*4] or NULL */
  const int32_t* previous_len;      /* [n_scenes] (0 or N) or NULL */
  const amppi_control* last_applied;/* [n_scenes] */
  const uint64_t* cycles;           /* [n_scenes] */
  const uint64_t* seeds;            /* [n_scenes] */
  double r_max;
} amppi_batch_input;

typedef struct {
  int32_t* status;                  /* [n_scenes] 0 ok, 1 planning failed */
  int32_t* winner;                  /* [n_scenes] */
  double* control;                  /* [n_scenes*4] */
  double* winner_nominal;           /* [n_scenes*N*4] */
  double* stage2;                   /* [n_scenes*M] */
  double* breakdown;                /* [n_scenes*5] */
} amppi_batch_output;

typedef struct amppi_ctx amppi_ctx;

/* Limits of this implementation (the reference has none): horizon N <= 64
 * (the screening kernels stage the nominal and guide tables in shared
 * memory), anchors M = m_h*m_v <= 1024, at most 2^32-1 points per scene.
 * amppi_create returns AMPPI_INVALID_ARGUMENT past them.
 *
 * Capacity contract: a context holds max_scenes scenes and max_points points
 * per call.  The host-pointer entry points grow the point buffers as needed;
 * amppi_cycle_batch_device cannot see its per-scene counts, so
 * point_offsets[n_scenes] must not exceed max_points -- a batch past it is
 * reported as AMPPI_INVALID_ARGUMENT at the next synchronising call. */

void amppi_config_default(amppi_config* cfg);
void amppi_options_default(amppi_options* opt);
int amppi_abi_version(void);

/* Context: device arenas sized from cfg/opt, one stream, cached CUDA graphs. */
int amppi_create(const amppi_config* cfg, const amppi_options* opt, amppi_ctx** out);
int amppi_destroy(amppi_ctx* ctx);
const char* amppi_last_error(const amppi_ctx* ctx);
int amppi_synchronize(amppi_ctx* ctx);

/* Replace the context's configuration (plan_step takes cfg per call,
 * ensemble.hpp:59-63): every weight, dynamics, anchor-grid spacing and
 * sampling parameter may change; the sizes (m_h, m_v, rollouts, horizon,
 * iterations) may not (AMPPI_INVALID_ARGUMENT: create a context for them).
 * Takes effect for the next call; the current snapshot stays valid unless
 * col_d_max changes (its collision grid is sized from d_max), in which case
 * the snapshot must be rebuilt (amppi_plan returns AMPPI_NO_SNAPSHOT). */
int amppi_set_config(amppi_ctx* ctx, const amppi_config* cfg);
int amppi_get_config(const amppi_ctx* ctx, amppi_config* cfg);
int amppi_set_schedule(amppi_ctx* ctx, const amppi_schedule* schedule);

/* == build_snapshot(buffer, pose, r_max): the buffer's frames concatenated
 * oldest-first (PointCloudBuffer::body_points order, perception.cpp:55-62). */
int amppi_snapshot(amppi_ctx* ctx, const float* world_xyz, int64_t n_points,
                   const amppi_state* pose, double r_max);
int amppi_snapshot_f64(amppi_ctx* ctx, const double* world_xyz, int64_t n_points,
                       const amppi_state* pose, double r_max);
/* The same from a device-resident float32 cloud (read in place, enqueued on
 * the context stream; the buffer must stay valid until the snapshot kernels
 * ran, i.e. until the next synchronising call). */
int amppi_snapshot_device(amppi_ctx* ctx, const float* d_world_xyz, int64_t n_points, const amppi_state* pose,
                          double r_max);
int amppi_snapshot_download(amppi_ctx* ctx, amppi_snapshot_view* view);

/* == plan_step(x, goal, snapshot, cfg, previous, last_applied, cycle, seed).
 * previous: previous_len controls (N*4) or NULL/0 (hover warm start,
 * ensemble.cpp:68-77).  injected_delta: NULL for the reference RNG stream, or
 * [iterations*M*K*N*4] perturbations replacing the draws (verification).
 * Returns AMPPI_PLANNING_FAILED when every instance is invalid. */
int amppi_plan(amppi_ctx* ctx, const amppi_state* x, const amppi_goal* goal,
               const double* previous, int32_t previous_len, const amppi_control* last_applied,
               uint64_t cycle, uint64_t seed, const double* injected_delta,
               amppi_plan_result* out);

/* Snapshot + plan for a batch of independent scenes (one plan cycle each). */
int amppi_cycle_batch(amppi_ctx* ctx, const amppi_batch_input* in, amppi_batch_output* out);
int amppi_cycle_batch_device(amppi_ctx* ctx, const amppi_batch_input* in_device,
                             amppi_batch_output* out_device);

/* Streaming form of amppi_cycle_batch: submit queues one batch (uploads on the
 * copy engine, planning on the compute streams) and returns a ticket; wait
 * returns that batch's results.  Up to three batches may be in flight, so the
 * next batch's upload overlaps the current batch's planning and is queued
 * before the previous batch is collected.  The caller's xyz
 * buffer (pinned memory for an asynchronous copy) must stay valid until the
 * batch is waited for; the per-scene arrays are copied at submit.  Tickets
 * are waited for in submit order. */
int amppi_cycle_batch_submit(amppi_ctx* ctx, const amppi_batch_input* in, int64_t* ticket);
int amppi_cycle_batch_wait(amppi_ctx* ctx, int64_t ticket, amppi_batch_output* out);

/* Sample-sharded plan_step (config C4): one context per GPU,
 * each owning samples [k_begin, k_end) of every instance (the global sample
 * index keys the perturbation stream, so the draws equal the unsharded plan).
 * Per iteration: screen -> all-reduce MIN of local_min[M] over the shards ->
 * partials -> all-gather of the [M * stride] partials (stride =
 * amppi_shard_partials_stride) in shard order -> update.  Then finish, which
 * fills *out like amppi_plan (identical on every shard).  All pointers except
 * out are DEVICE pointers; work is enqueued on the context stream and the
 * caller runs the collectives (e.g. NCCL) on that stream.  Replaces the inner
 * loop of plan_step (ensemble.cpp:79-129) with the merge of DESIGN.md §6. */
int amppi_shard_begin(amppi_ctx* ctx, const amppi_state* x, const amppi_goal* goal, const double* previous,
                      int32_t previous_len, const amppi_control* last_applied, uint64_t cycle, uint64_t seed,
                      int32_t k_begin, int32_t k_end);
int amppi_shard_screen(amppi_ctx* ctx, int32_t iter, float* local_min);
int amppi_shard_partials(amppi_ctx* ctx, int32_t iter, const float* global_min, double* partials);
int amppi_shard_update(amppi_ctx* ctx, int32_t iter, const double* all_partials, int32_t n_shards);
int amppi_shard_finish(amppi_ctx* ctx, amppi_plan_result* out);
int32_t amppi_shard_partials_stride(const amppi_ctx* ctx);

/* Native NCCL form of the same protocol (the caller owns the communicator,
 * one rank per GPU, every rank calls with the same inputs and gets the same
 * result): shard range = balanced split of [0, rollouts) by rank, the
 * all-reduce MIN and all-gather run on the context's stream.  NCCL is loaded
 * at run time (dlopen libnccl.so.2); without it these return AMPPI_NCCL_ERROR.
 * The comm helpers let a host program without NCCL headers create a
 * communicator: rank 0 calls amppi_nccl_unique_id, ships the 128 bytes to
 * every rank, and each rank calls amppi_nccl_comm_init. */
int amppi_nccl_version(int32_t* version);
int amppi_nccl_unique_id(void* id_out /* 128 bytes */);
int amppi_nccl_comm_init(void** comm_out, int32_t nranks, const void* id /* 128 bytes */, int32_t rank,
                         int32_t device);
int amppi_nccl_comm_destroy(void* comm);
int amppi_plan_sharded(amppi_ctx* ctx, void* nccl_comm, int32_t rank, int32_t nranks, const amppi_state* x,
                       const amppi_goal* goal, const double* previous, int32_t previous_len,
                       const amppi_control* last_applied, uint64_t cycle, uint64_t seed, amppi_plan_result* out);

/* GPU-resident closed loop (execute_cycle, ensemble.cpp:245-305; SURVEY.md
 * §8f row 1): the reference's scenario family `scene_kind` (0 empty,
 * 1 forest, 2 verticals, 3 inclines, 4 two_gap; generate_scenario seed
 * `scene_seed`), its LiDAR and PointCloudBuffer ring (`buffer_capacity`
 * frames) and the vehicle at 1/replan_hz all stay on the device; every cycle
 * is scan -> build_snapshot -> plan_step -> vehicle step with no host
 * traffic.  Episode parameters are the reference's defaults (goal radius 1 m,
 * timeout 60 s, drone radius 0.2 m, 50 consecutive planner failures).  The
 * loop drives the context's planner (configuration and stream). */
typedef struct amppi_loop amppi_loop;
typedef struct {
  uint64_t cycle;
  int32_t planned;             /* 0: "planning failed" (hover applied) */
  int32_t winner;              /* -1 when not planned */
  double x[10];                /* state the plan saw: p, q (w x y z), v */
  double control[4];           /* applied control */
  double stage2;               /* winner's stage-II cost */
  int32_t status;              /* after the cycle: 0 running, 1 success, 2 collision, 3 timeout, 4 planner failure */
  int32_t n_points;            /* points in the buffer the plan saw */
  /* TrajectoryLog LogRecord (ensemble.hpp:84-94): after the vehicle step */
  double t;                    /* episode time */
  double x_after[10];          /* p, q (w x y z), v */
  double clearance;            /* true clearance of the new position */
  double breakdown[5];         /* winner's cost breakdown (zeros when not planned) */
} amppi_loop_record;

/* EpisodeMetrics (metrics.hpp:11-18) from the device log (compute_metrics,
 * metrics.cpp:12-49); needs >= 4 cycles. */
typedef struct {
  double avg_vel, max_vel, smoothness, path_length, avg_clearance, min_clearance;
} amppi_episode_metrics;

int amppi_loop_create(amppi_ctx* ctx, int32_t scene_kind, uint64_t scene_seed, uint64_t seed,
                      int32_t buffer_capacity, int64_t max_cycles, amppi_loop** out);
/* Runs up to `cycles` cycles (fewer once the episode ends); *ran = cycles executed. */
int amppi_loop_run(amppi_loop* loop, int64_t cycles, int64_t* ran);
int amppi_loop_records(amppi_loop* loop, amppi_loop_record* out, int64_t cap, int64_t* count);
int amppi_loop_state(amppi_loop* loop, double* x10, int32_t* status, double* t);
int amppi_loop_metrics(amppi_loop* loop, amppi_episode_metrics* out);
int amppi_loop_destroy(amppi_loop* loop);

/* Formats around the path (host only, no context).
 * Cloud frames: the reference's text "# amppi-cloud v1" (io.cpp:24-66,
 * %.17g: exact round trip) or "# amppi-cloud-bin v1" (u64 frame id, u64
 * count, n x 3 float64).  amppi_cloud_read detects the format, writes up to
 * `cap` points and always reports the frame's point count in *n_points.
 * amppi_partition_csv / amppi_anchors_csv write the reference's debug dumps
 * (io.cpp:68-99) from a snapshot's ranges [7200] (flat i*60+j) and a plan's
 * refined anchors [M*3] + guide coefficients [M*18]. */
int amppi_cloud_read(const char* path, double* xyz, int64_t cap, int64_t* n_points, uint64_t* frame_id);
int amppi_cloud_write(const char* path, const double* xyz, int64_t n_points, uint64_t frame_id, int32_t binary);
int amppi_partition_csv(const char* path, const double* ranges);
int amppi_anchors_csv(const char* path, int32_t step, int32_t n_anchors, const double* refined,
                      const double* guide_coeffs, double horizon, int32_t samples);

/* Profiling: per-kernel device time accumulated since the last reset
 * (requires opt.profile = 1).  names/ms/launches are caller arrays of cap. */
int amppi_kernel_times(amppi_ctx* ctx, const char** names, double* ms, int64_t* launches,
                       int32_t cap, int32_t* count);
int amppi_kernel_times_reset(amppi_ctx* ctx);

/* Screening-drift diagnostic (verification only; DESIGN.md §2 "The d_max
 * jump"): after amppi_cycle_batch_device over in_device, integrates every
 * sample_stride-th sample of every instance twice -- as the FP32 screening
 * does (no abort bound) and as the FP64 refine does -- with the current
 * nominal and the perturbation stream of `iteration`, and compares them step
 * by step.  stats[8]: rollouts compared, max |p32 - p64| (m), max |d32 - d64|
 * where the clearance is below the grid cell size (1.001 d_max; both queries
 * exact there) minus 1e-4 (m), steps compared there, steps
 * on opposite sides of d_max outside the screening band (must be 0), steps the
 * screening flags, max relative stage-I cost difference of unflagged
 * rollouts, rollouts valid in one precision only. */
int amppi_screen_drift(amppi_ctx* ctx, const amppi_batch_input* in_device, int32_t iteration,
                       int32_t sample_stride, double* stats);
int amppi_set_stream(amppi_ctx* ctx, void* stream);
void* amppi_get_stream(const amppi_ctx* ctx);  /* the cudaStream_t the context launches on */

/* Synthetic input generator (not on the plan path):
 * scenario families of sim_world.cpp:174-246 (kind 0 empty, 1 forest,
 * 2 verticals, 3 inclines, 4 two_gap) and the per-cell jittered LiDAR of
 * sim_world.cpp:248-328 ray-cast on the GPU in FP32.  Frame f of scene s uses
 * poses[s*frames+f] / frame_seeds[s*frames+f]; hits are packed per scene in
 * frame-then-ray order, at most cap_per_scene points per scene;
 * xyz_out holds n_scenes*cap_per_scene*3 floats. */
int amppi_sim_scan(int32_t n_scenes, const int32_t* kinds, const uint64_t* scene_seeds, int32_t frames,
                   const amppi_state* poses, const uint64_t* frame_seeds, double r_max, int64_t cap_per_scene,
                   float* xyz_out, int64_t* offsets_out, int32_t device);

/* The same scans computed on the host (no GPU needed): the kernel's FP32
 * arithmetic is shared source (sim_ray.h) built without FMA contraction on
 * both sides, so the output bytes are identical to amppi_sim_scan's. */
int amppi_sim_scan_host(int32_t n_scenes, const int32_t* kinds, const uint64_t* scene_seeds, int32_t frames,
                        const amppi_state* poses, const uint64_t* frame_seeds, double r_max, int64_t cap_per_scene,
                        float* xyz_out, int64_t* offsets_out);

/* Measured FP32 FMA-pipe throughput of the device (TFLOP/s, FMA = 2 flops):
 * the roofline denominator for the CUDA-core rollout kernel. */
int amppi_probe_fp32_peak(int32_t device, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* AMPPI_B200_H */
