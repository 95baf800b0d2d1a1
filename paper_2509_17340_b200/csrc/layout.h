// Device-side data layout shared by the host runtime and the kernels.
// Everything here is POD; see DESIGN.md "Data layout in HBM".
#pragma once

#include <cstdint>

namespace amppi_dev {

// Partition geometry (perception.hpp:12-22).
constexpr int kAz = 120;
constexpr int kEl = 60;
constexpr int kPool = 6;
constexpr int kCAz = kAz / kPool;
constexpr int kCEl = kEl / kPool;
constexpr int kCells = kAz * kEl;       // 7200, flat(i,j) = i*60 + j
constexpr int kCoarse = kCAz * kCEl;    // 200, flat(I,J) = I*10 + J
constexpr double kMinPointRange = 0.05;
constexpr double kHorizonReach = 25.0;

// Collision grid: at most kGridAxis cells per axis, cell size >= d_max.
// Every cell owns a 32-byte record (two uint4: {start | count << 16, first
// leaf, lo.x, hi.x}, {lo.y, hi.y, lo.z, hi.z}; the float box holds the cell's
// points, rounded outward from FP64; per-axis (lo, hi) pairs feed the packed
// FP32x2 box test).  A cell's points (sorted by Morton code of the 1/8-cell
// sub-position) form leaves of kLeafSize consecutive points; a leaf box is
// {lo.x, hi.x, lo.y, hi.y}, {lo.z, hi.z, -, -} in float (outward-rounded).  The padded lattice (dims+2)^3 holds, per cell, the
// 27-bit mask of its non-empty neighbours (bit i*9+j*3+k <-> offset
// (i-1, j-1, k-1)); mask 0 = no point within one cell.
#ifndef AMPPI_WINDOW_LAMBDAS
#define AMPPI_WINDOW_LAMBDAS 64.0
#endif
// Softmin support window of the FP32 screening, in units of lambda (plus the
// FP32 error terms): samples beyond it carry weight < e^-kWindowLambdas.
constexpr double kWindowLambdas = AMPPI_WINDOW_LAMBDAS;
constexpr int kGridAxis = 24;
#ifndef AMPPI_LEAF_SIZE
#define AMPPI_LEAF_SIZE 16
#endif
constexpr uint32_t kLeafSize = AMPPI_LEAF_SIZE;
constexpr uint32_t kPointBlock = 4;  // FP32 query points per struct-of-arrays block
constexpr uint32_t kNoHint = 0xFFFFFFFFu;
constexpr int kGridCells = kGridAxis * kGridAxis * kGridAxis;
constexpr int kPadAxis = kGridAxis + 2;
constexpr int kPadCells = kPadAxis * kPadAxis * kPadAxis;
constexpr uint32_t kNbrCenter = 1u << 13;
constexpr uint32_t kNbrFaces = (1u << 4) | (1u << 10) | (1u << 12) | (1u << 14) | (1u << 16) | (1u << 22);

constexpr uint64_t kEmptyCell = 0xFFFFFFFFFFFFFFFFull;  // > bits of any finite positive double

// Scenes of at most this many points take the fused per-scene snapshot
// (k_snapshot_scene); larger ones the many-CTA keying, whose candidate log
// and counter are shared by every scene of a launch (so a batch containing
// such a scene runs as one chunk).
constexpr int64_t kFusedMaxPoints = 1 << 16;

// Bits of the device error word (Perception::flags, host-mapped).
constexpr uint32_t kFlagCandOverflow = 1u;  // a candidate log ran past its capacity: results invalid

// Flat copy of amppi_config plus derived sizes.
struct DevConfig {
  int m_h, m_v, M, K, N, iterations;
  int k_lo, k_hi;  // samples [k_lo, k_hi) of every instance are screened here (sample sharding); 0, K otherwise
  double lookahead, spacing_deg, terminal_speed, min_anchor_distance;
  double lambda, sigma[4], mppi_dt;
  double q_track, q_vnorm, q_c, q_c_delta, q_p, q_v, q_q;
  double col_scale, col_slope, col_d_min, col_d_max;
  double mass, gravity[3], dyn_dt, thrust_min, thrust_max, omega_xy_max, omega_z_max;
  double r_max;
};

struct GridMeta {
  double org[3];  // the FP32 local frame: FP32 grid data and screening positions are float(x - org) (the snapshot pose)
  double origin[3];
  double h, inv_h;
  float origin_f[3];
  float inv_h_f, h_f;
  int dims[3];
  int n_points;
};

// Per-batch input arrays (device pointers).  States/goals are 10 doubles:
// p(3) q(w,x,y,z) v(3) and p_goal(3) v_goal(3) q_goal(4).
struct BatchIn {
  const float* xyz;
  const double* xyz64;        // alternative FP64 input (single-scene API), or null
  const int64_t* offsets;     // [S+1]
  const double* poses;        // [S*10]
  const double* states;       // [S*10]
  const double* goals;        // [S*10]
  const double* prev;         // [S*N*4] or null
  const int32_t* prev_len;    // [S] or null
  const double* last_applied; // [S*4]
  const uint64_t* cycles;     // [S]
  const uint64_t* seeds;      // [S]
  const double* injected;     // [S*iters*M*K*N*4] or null
  int S;
  double r_max;
};

struct Candidate {
  uint32_t cell;   // scene*kCells + f
  uint32_t idx;    // point index within the scene
  uint64_t bits;   // range as IEEE bits
};

struct Perception {
  uint64_t* cell_r;            // [S*7200] min range bits (kEmptyCell when empty)
  uint32_t* cell_idx;          // [S*7200] argmin point index
  Candidate* cand;             // [cap]
  unsigned long long* cand_count;
  int64_t cand_cap;            // Candidate slots (the fused kernel logs one Candidate per logged point)
  uint32_t* flags;             // device error word (kFlag*), mapped host memory
  const double* cell_dir;      // [7200*3] cell-centre directions (host libm)
  // outputs
  double* ranges;              // [S*7200] or null (verification)
  uint8_t* has_point;          // [S*7200] or null
  double* nearest;             // [S*7200*3] or null
  double* filtered;            // [S*7200*3] or null (flat-cell order)
  double* safe_range;          // [S*200]
  double* safe_dir;            // [S*600]
  double* safe_point;          // [S*600]
  int32_t* n_filtered;         // [S]
  GridMeta* grid;              // [S]
  uint4* grid_rec;             // [S*kGridCells*2] cell records (written for non-empty cells only)
  uint32_t* grid_nbr;          // [S*kPadCells] neighbour masks over the padded lattice
  uint4* grid_leaf;            // [S*7200*2] leaf boxes
  double* grid_pts64;          // [S*7200*3] sorted by grid cell
  float4* grid_pts32;          // [S*7200]: per scene 1800 blocks of kPointBlock points {x4, y4, z4} (+inf padding)
};

// Non-collision cost sums of a deferred-collision FP64 rollout (latency path).
struct TrajSums {
  double trk, vn, mag, rate, goal;
  int valid;
};

// Rollouts up to this count per call run the latency path: one warp per
// rollout (k_stage1_warp32).
constexpr int kLatencyRollouts = 148 * 128;

constexpr int kColCountStride = 160;  // unsigned ints per chunk in Plan::col_count

struct Plan {
  // anchors / guides (FP64)
  double* anchor_init;         // [S*M*3]
  double* anchor_ref;          // [S*M*3]
  double* anchor_dir;          // [S*M*3]
  double* anchor_range;        // [S*M]
  int32_t* anchor_ij;          // [S*M*2]
  double* guide_coef;          // [S*M*18] [axis][power]
  double* guide64;             // [S*M*N*3]
  float4* guide32;             // [S*M*N]
  double* nominal;             // [S*M*N*4] current nominal (FP64 always)
  float4* unom32;              // [S*M*N] the nominal in float for the screening kernels (bulk-copied to smem)
  // stage I
  float* cost32;               // [S*M*K]
  double* cost64;              // [S*M*K]
  uint8_t* alive;              // [S*M]
  // per instance
  double* stage1;              // [S*M]
  double* stage2;              // [S*M]
  double* ess;                 // [S*M]
  uint8_t* valid;              // [S*M]
  double* breakdown;           // [S*M*5]
  uint32_t* n_support;         // [S*M] softmin support size (diagnostics)
  // deferred-collision scratch (latency path and stage II)
  double* pos64;               // [pos_cap*N*4]
  TrajSums* tsum;              // [pos_cap]
  int64_t pos_cap;             // support pairs the split refine handles (pos64/tsum hold max(4*S*M, kLatencyRollouts))
  double* col_terms;           // [pos_cap*N] per-step collision terms of the deferred trajectories
  uint32_t* col_work;          // [pos_cap*N] (trajectory*N + step) queries with a point within d_max
  unsigned int* col_count;     // work-list counters ([kColCountStride] per concurrent chunk: length, bucket counts)
  // per scene
  int32_t* done;               // [S] arrival counter (self-resetting)
  int32_t* winner;             // [S]
  int32_t* status;             // [S]
  double* control;             // [S*4]
  double* winner_states;       // [S*(N+1)*10] or null
  double* winner_controls;     // [S*N*4] or null
};

}  // namespace amppi_dev
