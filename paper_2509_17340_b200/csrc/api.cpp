// Host runtime behind include/amppi_b200.h: context, device arenas, pinned
// staging, kernel sequencing and the C-ABI entry points.  No CPU compute path:
// every planning result comes from the CUDA kernels in k_*.cu; a context
// cannot be created without a CUDA device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <new>
#include <numbers>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only; the ranges cost nothing unless a profiler injects a tool

#include "../../include/amppi_b200.h"
#include "kernels.h"
#include "layout.h"
#include "loop.h"

using namespace amppi_dev;

namespace {

constexpr double kPi = std::numbers::pi;
constexpr int kMaxChunks = 8;  // chunks of a pipelined batch (one work-list counter block each)
constexpr int kExtraStreams = 2;  // compute streams beyond stream / stream2

struct Arena {
  std::vector<void*> blocks;
  cudaError_t alloc(void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) blocks.push_back(*p);
    return e;
  }
  void release() {
    for (void* p : blocks) cudaFree(p);
    blocks.clear();
  }
};

// Contiguous per-scene input block for one-copy uploads.
struct InputBlock {
  double* poses;
  double* states;
  double* goals;
  double* last;
  double* prev;
  int64_t* offsets;
  uint64_t* cycles;
  uint64_t* seeds;
  int32_t* prev_len;
  size_t bytes;
};

template <typename T>
T* carve(unsigned char*& cur, size_t count) {
  const size_t align = 16;
  uintptr_t p = reinterpret_cast<uintptr_t>(cur);
  p = (p + align - 1) & ~(align - 1);
  T* out = reinterpret_cast<T*>(p);
  cur = reinterpret_cast<unsigned char*>(p + count * sizeof(T));
  return out;
}

InputBlock layout_inputs(unsigned char* base, int S, int N) {
  InputBlock b{};
  unsigned char* cur = base;
  b.poses = carve<double>(cur, static_cast<size_t>(S) * 10);
  b.states = carve<double>(cur, static_cast<size_t>(S) * 10);
  b.goals = carve<double>(cur, static_cast<size_t>(S) * 10);
  b.last = carve<double>(cur, static_cast<size_t>(S) * 4);
  b.prev = carve<double>(cur, static_cast<size_t>(S) * N * 4);
  b.offsets = carve<int64_t>(cur, static_cast<size_t>(S) + 1);
  b.cycles = carve<uint64_t>(cur, S);
  b.seeds = carve<uint64_t>(cur, S);
  b.prev_len = carve<int32_t>(cur, S);
  b.bytes = static_cast<size_t>(cur - base) + 16;
  return b;
}

// Contiguous single-scene result block for one-copy downloads.
struct ResultBlock {
  int32_t* winner;
  int32_t* status;
  uint8_t* valid;
  uint8_t* alive;
  double* control;
  double* stage1;
  double* stage2;
  double* ess;
  double* breakdown;
  double* nominal;
  double* anchor_init;
  double* anchor_ref;
  double* anchor_dir;
  double* anchor_range;
  int32_t* anchor_ij;
  double* guide_coef;
  uint32_t* n_support;
  size_t bytes;
};

ResultBlock layout_results(unsigned char* base, int S, int M, int N) {
  ResultBlock r{};
  unsigned char* cur = base;
  const size_t SM = static_cast<size_t>(S) * M;
  r.winner = carve<int32_t>(cur, S);
  r.status = carve<int32_t>(cur, S);
  r.valid = carve<uint8_t>(cur, SM);
  r.alive = carve<uint8_t>(cur, SM);
  r.control = carve<double>(cur, static_cast<size_t>(S) * 4);
  r.stage1 = carve<double>(cur, SM);
  r.stage2 = carve<double>(cur, SM);
  r.ess = carve<double>(cur, SM);
  r.breakdown = carve<double>(cur, SM * 5);
  r.nominal = carve<double>(cur, SM * N * 4);
  r.anchor_init = carve<double>(cur, SM * 3);
  r.anchor_ref = carve<double>(cur, SM * 3);
  r.anchor_dir = carve<double>(cur, SM * 3);
  r.anchor_range = carve<double>(cur, SM);
  r.anchor_ij = carve<int32_t>(cur, SM * 2);
  r.guide_coef = carve<double>(cur, SM * 18);
  r.n_support = carve<uint32_t>(cur, SM);
  r.bytes = static_cast<size_t>(cur - base) + 16;
  return r;
}

}  // namespace

struct amppi_ctx {
  amppi_config cfg{};
  amppi_options opt{};
  DevConfig dc{};
  cudaStream_t stream{nullptr};
  bool own_stream{false};
  cudaStream_t copy_stream{nullptr};  // host->device point copies overlapped with planning
  cudaStream_t stream2{nullptr};      // second compute stream: alternate chunks of a batch run concurrently
  cudaStream_t xstream[kExtraStreams]{};  // further compute streams for pipelined chunks
  cudaEvent_t inputs_read{nullptr};   // single-scene snapshot inputs copied (staging reusable)
  std::vector<cudaEvent_t> join;
  std::vector<cudaEvent_t> chunk_ready;
  std::string err;
  int S_cap{1};
  int64_t P_cap{0};
  Arena arena;
  // inputs
  unsigned char* d_in{nullptr};
  unsigned char* h_in{nullptr};  // pinned mirror
  InputBlock din{}, hin{};
  float* d_xyz{nullptr};
  double* d_xyz64{nullptr};
  float* h_xyz{nullptr};  // pinned staging
  size_t h_xyz_bytes{0};
  double* d_injected{nullptr};
  size_t injected_bytes{0};
  // results
  unsigned char* d_res{nullptr};
  unsigned char* h_res{nullptr};
  ResultBlock dres{}, hres{};
  // device state
  Perception P{};
  Plan pl{};
  uint32_t* cand_k{nullptr};
  double* cand_s{nullptr};
  double* cand_w{nullptr};
  uint2* pairs{nullptr};
  unsigned long long* pair_count{nullptr};
  unsigned char* d_gather{nullptr};
  unsigned char* h_gather{nullptr};  // pinned mirror of d_gather (per-chunk result copies)
  std::vector<cudaEvent_t> chunk_done;
  // streaming batches (amppi_cycle_batch_submit / _wait): three input slots,
  // so batch t+1's upload overlaps batch t's planning and can be queued
  // before batch t-1 is collected (no host round trip between them)
  struct StreamSlot {
    float* d_xyz{nullptr};
    int64_t xyz_cap{0};
    unsigned char* d_in{nullptr};
    unsigned char* h_in{nullptr};
    InputBlock din{}, hin{};
    unsigned char* h_gather{nullptr};
    cudaEvent_t uploaded{nullptr}, done{nullptr};
    bool busy{false};
    int S{0};
    int64_t ticket{-1};
  };
  static constexpr int kStreamSlots = 3;
  StreamSlot slots[kStreamSlots];
  int64_t next_ticket{0};
  uint32_t* h_flags{nullptr};  // mapped device error word (Perception::flags)
  // single-scene plan captured as a CUDA graph (the plan kernels of one
  // amppi_plan call), replayed while its key matches
  struct PlanGraphKey {
    bool want_states{false};
    bool injected{false};
    double r_max{0.0};
    uint64_t points_gen{0};
    amppi_config cfg{};
  };
  cudaGraphExec_t plan_graph{nullptr};
  PlanGraphKey plan_graph_key{};
  uint64_t points_gen{0};      // bumped when the point buffers are reallocated (captured graphs refer to them)
  // single-scene snapshot bookkeeping
  bool have_snapshot{false};
  double snap_d_max{0.0};      // col_d_max the snapshot's collision grid was sized with
  double snap_r_max{10.0};
  double snap_pose[10]{};
  int64_t snap_points{0};
  KernelTimer timer;
  // sample-sharded plan in progress (amppi_shard_*)
  bool shard_active{false};
  DevConfig shard_dc{};
  BatchIn shard_in{};

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* where) {
    err = std::string(where) + ": " + cudaGetErrorString(e);
    return AMPPI_CUDA_ERROR;
  }
};

#define CK(expr)                                              \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ctx->cuda_fail(_e, #expr);  \
  } while (0)

// NVTX range over a host entry point (nsys / ncu --nvtx see the API phases).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {

DevConfig to_dev(const amppi_config& c) {
  DevConfig d{};
  d.m_h = c.m_h;
  d.m_v = c.m_v;
  d.M = c.m_h * c.m_v;
  d.K = c.rollouts;
  d.k_lo = 0;
  d.k_hi = c.rollouts;
  d.N = c.horizon;
  d.iterations = c.iterations;
  d.lookahead = c.lookahead;
  d.spacing_deg = c.spacing_deg;
  d.terminal_speed = c.terminal_speed;
  d.min_anchor_distance = c.min_anchor_distance;
  d.lambda = c.lambda;
  for (int i = 0; i < 4; ++i) d.sigma[i] = c.sigma[i];
  d.mppi_dt = c.mppi_dt;
  d.q_track = c.q_track;
  d.q_vnorm = c.q_vnorm;
  d.q_c = c.q_c;
  d.q_c_delta = c.q_c_delta;
  d.q_p = c.q_p;
  d.q_v = c.q_v;
  d.q_q = c.q_q;
  d.col_scale = c.col_scale;
  d.col_slope = c.col_slope;
  d.col_d_min = c.col_d_min;
  d.col_d_max = c.col_d_max;
  d.mass = c.mass;
  for (int i = 0; i < 3; ++i) d.gravity[i] = c.gravity[i];
  d.dyn_dt = c.dyn_dt;
  d.thrust_min = c.thrust_min;
  d.thrust_max = c.thrust_max;
  d.omega_xy_max = c.omega_xy_max;
  d.omega_z_max = c.omega_z_max;
  d.r_max = c.r_max;
  return d;
}

std::string validate(const amppi_config& c) {
  if (c.m_h < 1 || c.m_v < 1) return "anchor grid must be at least 1x1";
  if (c.m_h * c.m_v > 1024) return "at most 1024 anchors";
  if (c.rollouts < 1) return "rollouts must be positive";
  if (c.horizon < 1 || c.horizon > 64) return "horizon must be in [1, 64]";
  if (c.iterations < 1) return "iterations must be positive";
  if (!(c.lambda > 0.0)) return "lambda must be positive";
  if (!(c.mass > 0.0)) return "mass must be positive";
  if (!(c.dyn_dt > 0.0) || !(c.mppi_dt > 0.0)) return "dt must be positive";
  if (!(c.col_d_max > 0.0)) return "d_obs_max must be positive";
  if (!(c.r_max > 0.0)) return "r_max must be positive";
  return "";
}

// cell_direction(i, j) for every fine cell (perception.cpp:36-42), host libm.
std::vector<double> cell_direction_table() {
  std::vector<double> t(static_cast<size_t>(kCells) * 3);
  const double az_step = 2.0 * kPi / kAz, el_step = kPi / kEl;
  for (int i = 0; i < kAz; ++i)
    for (int j = 0; j < kEl; ++j) {
      const double az = -kPi + (i + 0.5) * az_step;
      const double el = -0.5 * kPi + (j + 0.5) * el_step;
      const double ce = std::cos(el);
      double* o = t.data() + 3 * (i * kEl + j);
      o[0] = ce * std::cos(az);
      o[1] = ce * std::sin(az);
      o[2] = std::sin(el);
    }
  return t;
}

int alloc_points(amppi_ctx* ctx, int64_t P) {
  if (P <= ctx->P_cap && ctx->d_xyz) return AMPPI_OK;
  const int64_t cap = std::max<int64_t>(P, 1024);
  if (ctx->d_xyz) cudaFree(ctx->d_xyz);
  if (ctx->d_xyz64) cudaFree(ctx->d_xyz64);
  if (ctx->P.cand) cudaFree(ctx->P.cand);
  if (ctx->h_xyz) cudaFreeHost(ctx->h_xyz);
  ctx->d_xyz = nullptr;
  ctx->d_xyz64 = nullptr;
  ctx->P.cand = nullptr;
  ctx->h_xyz = nullptr;
  CK(cudaMalloc(&ctx->d_xyz, static_cast<size_t>(cap) * 3 * sizeof(float)));
  CK(cudaMalloc(&ctx->d_xyz64, static_cast<size_t>(cap) * 3 * sizeof(double)));
  CK(cudaMalloc(&ctx->P.cand, static_cast<size_t>(cap) * sizeof(Candidate)));
  ctx->h_xyz_bytes = static_cast<size_t>(cap) * 3 * sizeof(double);
  CK(cudaMallocHost(&ctx->h_xyz, ctx->h_xyz_bytes));
  ctx->P.cand_cap = cap;
  ctx->P_cap = cap;
  ++ctx->points_gen;
  return AMPPI_OK;
}

int create_impl(amppi_ctx* ctx) {
  const int S = ctx->S_cap;
  const DevConfig& dc = ctx->dc;
  const int M = dc.M, K = dc.K, N = dc.N;
  const size_t SM = static_cast<size_t>(S) * M;
  CK(cudaSetDevice(ctx->opt.device));
  if (ctx->opt.stream) {
    ctx->stream = static_cast<cudaStream_t>(ctx->opt.stream);
  } else {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
  for (cudaStream_t& x : ctx->xstream) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->inputs_read, cudaEventDisableTiming));
  for (int i = 0; i < 2 + kExtraStreams; ++i) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->join.push_back(ev);
  }
  CK(init_kernel_attributes());
  Arena& A = ctx->arena;
  // inputs (device + pinned mirror with identical layout)
  {
    const InputBlock probe = layout_inputs(nullptr, S, N);
    void* p = nullptr;
    CK(A.alloc(&p, probe.bytes));
    ctx->d_in = static_cast<unsigned char*>(p);
    CK(cudaMallocHost(&p, probe.bytes));
    ctx->h_in = static_cast<unsigned char*>(p);
    ctx->din = layout_inputs(ctx->d_in, S, N);
    ctx->hin = layout_inputs(ctx->h_in, S, N);
  }
  {
    const ResultBlock probe = layout_results(nullptr, S, M, N);
    void* p = nullptr;
    CK(A.alloc(&p, probe.bytes));
    ctx->d_res = static_cast<unsigned char*>(p);
    CK(cudaMemset(ctx->d_res, 0, probe.bytes));
    CK(cudaMallocHost(&p, probe.bytes));
    ctx->h_res = static_cast<unsigned char*>(p);
    ctx->dres = layout_results(ctx->d_res, S, M, N);
    ctx->hres = layout_results(ctx->h_res, S, M, N);
  }
  if (int rc = alloc_points(ctx, std::max<int64_t>(ctx->opt.max_points, 1024)); rc != AMPPI_OK) return rc;

  Perception& P = ctx->P;
  void* p = nullptr;
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * sizeof(uint64_t)));
  P.cell_r = static_cast<uint64_t*>(p);
  CK(cudaMemset(P.cell_r, 0xFF, static_cast<size_t>(S) * kCells * sizeof(uint64_t)));
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * sizeof(uint32_t)));
  P.cell_idx = static_cast<uint32_t*>(p);
  CK(cudaMemset(P.cell_idx, 0xFF, static_cast<size_t>(S) * kCells * sizeof(uint32_t)));
  CK(A.alloc(&p, sizeof(unsigned long long)));
  P.cand_count = static_cast<unsigned long long*>(p);
  {
    void* hf = nullptr;
    CK(cudaHostAlloc(&hf, sizeof(uint32_t), cudaHostAllocMapped));
    ctx->h_flags = static_cast<uint32_t*>(hf);
    *ctx->h_flags = 0u;
    void* df = nullptr;
    CK(cudaHostGetDevicePointer(&df, hf, 0));
    P.flags = static_cast<uint32_t*>(df);
  }
  {
    const std::vector<double> dirs = cell_direction_table();
    CK(A.alloc(&p, dirs.size() * sizeof(double)));
    CK(cudaMemcpy(p, dirs.data(), dirs.size() * sizeof(double), cudaMemcpyHostToDevice));
    P.cell_dir = static_cast<const double*>(p);
  }
  if (S <= 64) {  // verification views (single-scene API)
    CK(A.alloc(&p, static_cast<size_t>(S) * kCells * sizeof(double)));
    P.ranges = static_cast<double*>(p);
    CK(A.alloc(&p, static_cast<size_t>(S) * kCells));
    P.has_point = static_cast<uint8_t*>(p);
    CK(A.alloc(&p, static_cast<size_t>(S) * kCells * 3 * sizeof(double)));
    P.nearest = static_cast<double*>(p);
  }
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * 3 * sizeof(double)));
  P.filtered = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCoarse * sizeof(double)));
  P.safe_range = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCoarse * 3 * sizeof(double)));
  P.safe_dir = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCoarse * 3 * sizeof(double)));
  P.safe_point = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * sizeof(int32_t)));
  P.n_filtered = static_cast<int32_t*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * sizeof(GridMeta)));
  P.grid = static_cast<GridMeta*>(p);
  CK(cudaMemset(P.grid, 0, static_cast<size_t>(S) * sizeof(GridMeta)));
  CK(A.alloc(&p, static_cast<size_t>(S) * kGridCells * 2 * sizeof(uint4)));
  P.grid_rec = static_cast<uint4*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kPadCells * sizeof(uint32_t)));
  P.grid_nbr = static_cast<uint32_t*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * 2 * sizeof(uint4)));
  P.grid_leaf = static_cast<uint4*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * 3 * sizeof(double)));
  P.grid_pts64 = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * kCells * sizeof(float4)));
  P.grid_pts32 = static_cast<float4*>(p);

  Plan& pl = ctx->pl;
  const ResultBlock& r = ctx->dres;
  pl.anchor_init = r.anchor_init;
  pl.anchor_ref = r.anchor_ref;
  pl.anchor_dir = r.anchor_dir;
  pl.anchor_range = r.anchor_range;
  pl.anchor_ij = r.anchor_ij;
  pl.guide_coef = r.guide_coef;
  pl.nominal = r.nominal;
  pl.alive = r.alive;
  pl.stage1 = r.stage1;
  pl.stage2 = r.stage2;
  pl.ess = r.ess;
  pl.valid = r.valid;
  pl.breakdown = r.breakdown;
  pl.n_support = r.n_support;
  pl.winner = r.winner;
  pl.status = r.status;
  pl.control = r.control;
  CK(A.alloc(&p, SM * N * 3 * sizeof(double)));
  pl.guide64 = static_cast<double*>(p);
  CK(A.alloc(&p, SM * N * sizeof(float4)));
  pl.guide32 = static_cast<float4*>(p);
  CK(A.alloc(&p, SM * N * sizeof(float4)));
  pl.unom32 = static_cast<float4*>(p);
  CK(A.alloc(&p, SM * K * sizeof(float)));
  pl.cost32 = static_cast<float*>(p);
  CK(A.alloc(&p, SM * K * sizeof(double)));
  pl.cost64 = static_cast<double*>(p);
  {
    // deferred-collision rollouts: stage II (S*M) and the split FP64 refine
    // (~4 support samples per instance; more spill to the fused k_refine)
    const size_t jobs = std::max<size_t>(4 * SM, static_cast<size_t>(kLatencyRollouts));
    pl.pos_cap = static_cast<int64_t>(jobs);
    if (ctx->opt.refine_split_cap >= 0)  // tests: force the fused-refine overflow path
      pl.pos_cap = std::min<int64_t>(pl.pos_cap, ctx->opt.refine_split_cap);
    CK(A.alloc(&p, jobs * N * 4 * sizeof(double)));
    pl.pos64 = static_cast<double*>(p);
    CK(A.alloc(&p, jobs * sizeof(TrajSums)));
    pl.tsum = static_cast<TrajSums*>(p);
    CK(A.alloc(&p, jobs * N * sizeof(double)));
    pl.col_terms = static_cast<double*>(p);
    CK(A.alloc(&p, jobs * N * sizeof(uint32_t)));
    pl.col_work = static_cast<uint32_t*>(p);
    CK(A.alloc(&p, kMaxChunks * kColCountStride * sizeof(unsigned int)));
    pl.col_count = static_cast<unsigned int*>(p);
  }
  CK(A.alloc(&p, static_cast<size_t>(S) * sizeof(int32_t)));
  pl.done = static_cast<int32_t*>(p);
  CK(cudaMemset(pl.done, 0, static_cast<size_t>(S) * sizeof(int32_t)));
  CK(A.alloc(&p, static_cast<size_t>(S) * (N + 1) * 10 * sizeof(double)));
  pl.winner_states = static_cast<double*>(p);
  CK(A.alloc(&p, static_cast<size_t>(S) * N * 4 * sizeof(double)));
  pl.winner_controls = static_cast<double*>(p);
  CK(A.alloc(&p, SM * K * sizeof(uint32_t)));
  ctx->cand_k = static_cast<uint32_t*>(p);
  CK(A.alloc(&p, SM * K * sizeof(double)));
  ctx->cand_s = static_cast<double*>(p);
  CK(A.alloc(&p, SM * K * sizeof(double)));
  ctx->cand_w = static_cast<double*>(p);
  CK(A.alloc(&p, SM * K * sizeof(uint2)));
  ctx->pairs = static_cast<uint2*>(p);
  CK(A.alloc(&p, kMaxChunks * sizeof(unsigned long long)));  // one work-list counter per concurrent chunk
  ctx->pair_count = static_cast<unsigned long long*>(p);
  ctx->timer.enabled = ctx->opt.profile != 0;
  return AMPPI_OK;
}

BatchIn batch_from_block(amppi_ctx* ctx, int S, double r_max, bool f64_points) {
  BatchIn in{};
  in.xyz = ctx->d_xyz;
  in.xyz64 = f64_points ? ctx->d_xyz64 : nullptr;
  in.offsets = ctx->din.offsets;
  in.poses = ctx->din.poses;
  in.states = ctx->din.states;
  in.goals = ctx->din.goals;
  in.prev = ctx->din.prev;
  in.prev_len = ctx->din.prev_len;
  in.last_applied = ctx->din.last;
  in.cycles = ctx->din.cycles;
  in.seeds = ctx->din.seeds;
  in.injected = nullptr;
  in.S = S;
  in.r_max = r_max;
  return in;
}

// The plan arrays of scenes [s0, ...): a chunk of a batch planned on its own
// writes its per-scene results at their batch position (perception and
// per-iteration scratch are consumed within the chunk and are reused).
Plan shift_plan(const Plan& p, int64_t s0, const DevConfig& c) {
  const int64_t sm = s0 * c.M;
  Plan q = p;
  q.anchor_init += sm * 3;
  q.anchor_ref += sm * 3;
  q.anchor_dir += sm * 3;
  q.anchor_range += sm;
  q.anchor_ij += sm * 2;
  q.guide_coef += sm * 18;
  q.guide64 += sm * c.N * 3;
  q.guide32 += sm * c.N;
  q.unom32 += sm * c.N;
  q.nominal += sm * c.N * 4;
  q.cost32 += sm * c.K;
  q.cost64 += sm * c.K;
  q.alive += sm;
  q.stage1 += sm;
  q.stage2 += sm;
  q.ess += sm;
  q.valid += sm;
  q.breakdown += sm * 5;
  q.n_support += sm;
  q.done += s0;
  q.winner += s0;
  q.status += s0;
  q.control += s0 * 4;
  if (q.winner_states) q.winner_states += s0 * (c.N + 1) * 10;
  if (q.winner_controls) q.winner_controls += s0 * c.N * 4;
  return q;
}

// Compute streams that pipelined chunks rotate over (schedule.pipeline_streams,
// 2..4, default 3: best measured with tools/pipe_sweep.py).
int pipeline_streams(const amppi_ctx* ctx) {
  const int n = ctx->opt.schedule.pipeline_streams;
  return n > 0 ? std::max(2, std::min(2 + kExtraStreams, n)) : 3;
}

cudaStream_t compute_stream(amppi_ctx* ctx, int c) {
  const int i = c % pipeline_streams(ctx);
  return i == 0 ? ctx->stream : (i == 1 ? ctx->stream2 : ctx->xstream[i - 2]);
}

// Fork the compute streams off ctx->stream / join them back into it.
int fork_streams(amppi_ctx* ctx) {
  CK(cudaEventRecord(ctx->join[0], ctx->stream));
  for (int i = 1; i < pipeline_streams(ctx); ++i) CK(cudaStreamWaitEvent(compute_stream(ctx, i), ctx->join[0], 0));
  return AMPPI_OK;
}

int join_streams(amppi_ctx* ctx) {
  for (int i = 1; i < pipeline_streams(ctx); ++i) {
    CK(cudaEventRecord(ctx->join[i], compute_stream(ctx, i)));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->join[i], 0));
  }
  return AMPPI_OK;
}

Perception shift_perception(const Perception& p, int64_t s0) {
  Perception q = p;
  q.cell_r += s0 * kCells;
  q.cell_idx += s0 * kCells;
  if (q.ranges) q.ranges += s0 * kCells;
  if (q.has_point) q.has_point += s0 * kCells;
  if (q.nearest) q.nearest += s0 * kCells * 3;
  q.filtered += s0 * kCells * 3;
  q.safe_range += s0 * kCoarse;
  q.safe_dir += s0 * kCoarse * 3;
  q.safe_point += s0 * kCoarse * 3;
  q.n_filtered += s0;
  q.grid += s0;
  q.grid_rec += s0 * kGridCells * 2;
  q.grid_nbr += s0 * kPadCells;
  q.grid_leaf += s0 * kCells * 2;
  q.grid_pts64 += s0 * kCells * 3;
  q.grid_pts32 += s0 * kCells;
  return q;
}

// Snapshot + plan of the batch's scenes [s0, s0 + in.S) with every array
// (perception, plan, support scratch, refine scratch, work-list counter) at
// the chunk's own offset, so chunks can run concurrently on different
// streams.  Needs the fused snapshot (>= 148 scenes per chunk).
int run_chunk(amppi_ctx* ctx, const BatchIn& in, int64_t max_pts_scene, int64_t s0, int chunk, cudaStream_t st) {
  NvtxRange nvtx_range("amppi chunk (snapshot + plan)");
  const DevConfig& dc = ctx->dc;
  const Perception P = shift_perception(ctx->P, s0);
  Plan pl = shift_plan(ctx->pl, s0, dc);
  const int64_t sm0 = s0 * dc.M, smc = static_cast<int64_t>(in.S) * dc.M;
  pl.pos64 += 4 * sm0 * dc.N * 4;
  pl.tsum += 4 * sm0;
  pl.col_terms += 4 * sm0 * dc.N;
  pl.col_work += 4 * sm0 * dc.N;
  pl.col_count += chunk * kColCountStride;
  pl.pos_cap = std::min<int64_t>(4 * smc, ctx->pl.pos_cap);
  cudaError_t e = launch_snapshot(in, P, dc, max_pts_scene, st, &ctx->timer);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_snapshot");
  const int64_t ks = sm0 * dc.K;
  e = launch_plan_impl(in, P, pl, dc, ctx->opt.precision, false, ctx->cand_k + ks, ctx->cand_s + ks, ctx->cand_w + ks,
                       ctx->pairs + ks, ctx->pair_count + chunk, st, &ctx->timer);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_plan");
}

int run_cycle(amppi_ctx* ctx, const BatchIn& in, int64_t max_pts_scene, bool do_snapshot, bool do_plan,
              bool winner_rollout, int64_t s0 = 0) {
  if (do_snapshot) {
    cudaError_t e = launch_snapshot(in, ctx->P, ctx->dc, max_pts_scene, ctx->stream, &ctx->timer);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_snapshot");
  }
  if (do_plan) {
    const Plan pl = s0 ? shift_plan(ctx->pl, s0, ctx->dc) : ctx->pl;
    cudaError_t e = launch_plan_impl(in, ctx->P, pl, ctx->dc, ctx->opt.precision, winner_rollout, ctx->cand_k,
                                     ctx->cand_s, ctx->cand_w, ctx->pairs, ctx->pair_count, ctx->stream, &ctx->timer);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_plan");
  }
  return AMPPI_OK;
}

int sync_and_collect(amppi_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->timer.enabled) ctx->timer.collect();
  if (ctx->h_flags && *ctx->h_flags) {
    *ctx->h_flags = 0u;
    return ctx->fail(AMPPI_INVALID_ARGUMENT,
                     "a batch exceeded the context's point capacity (max_points); its results are invalid");
  }
  return AMPPI_OK;
}

void put_pose(double* o, const amppi_state* s) {
  std::memcpy(o, s, 10 * sizeof(double));
}

}  // namespace

extern "C" {

int amppi_abi_version(void) { return AMPPI_ABI_VERSION; }

void amppi_config_default(amppi_config* c) {
  // Table I defaults, i.e. the reference's EnsembleConfig{} (ensemble.hpp:16-23)
  c->m_h = 5;
  c->m_v = 3;
  c->lookahead = 5.0;
  c->spacing_deg = 18.0;
  c->terminal_speed = 3.0;
  c->min_anchor_distance = 0.5;
  c->rollouts = 128;
  c->horizon = 25;
  c->lambda = 0.1;
  c->sigma[0] = 1.0;
  c->sigma[1] = 1.0;
  c->sigma[2] = 1.0;
  c->sigma[3] = 0.5;
  c->mppi_dt = 0.05;
  c->iterations = 1;
  c->q_track = 15.0;
  c->q_vnorm = 0.15;
  c->q_c = 0.5;
  c->q_c_delta = 0.5;
  c->q_p = 3.0;
  c->q_v = 0.25;
  c->q_q = 1.0;
  c->col_scale = 1.0e6;
  c->col_slope = 5.0;
  c->col_d_min = 0.4;
  c->col_d_max = 1.0;
  c->mass = 1.0;
  c->gravity[0] = 0.0;
  c->gravity[1] = 0.0;
  c->gravity[2] = -9.81;
  c->dyn_dt = 0.05;
  c->thrust_min = 0.3;
  c->thrust_max = 16.35;
  c->omega_xy_max = 3.0;
  c->omega_z_max = 2.0;
  c->replan_hz = 50.0;
  c->r_max = 10.0;
}

void amppi_options_default(amppi_options* o) {
  o->device = 0;
  o->precision = 32;
  o->max_scenes = 1;
  o->max_points = 1 << 20;
  o->profile = 0;
  o->stream = nullptr;
  o->refine_split_cap = -1;
  o->schedule = amppi_schedule{};
}

int amppi_create(const amppi_config* cfg, const amppi_options* opt, amppi_ctx** out) {
  if (!cfg || !out) return AMPPI_INVALID_ARGUMENT;
  *out = nullptr;
  const std::string bad = validate(*cfg);
  if (!bad.empty()) return AMPPI_INVALID_ARGUMENT;
  auto* ctx = new (std::nothrow) amppi_ctx();
  if (!ctx) return AMPPI_CUDA_ERROR;
  ctx->cfg = *cfg;
  if (opt)
    ctx->opt = *opt;
  else
    amppi_options_default(&ctx->opt);
  if (ctx->opt.precision != 32 && ctx->opt.precision != 64) ctx->opt.precision = 32;
  ctx->S_cap = std::max(1, ctx->opt.max_scenes);
  ctx->dc = to_dev(*cfg);
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    delete ctx;
    return AMPPI_CUDA_ERROR;
  }
  const int rc = create_impl(ctx);
  if (rc != AMPPI_OK) {
    std::fprintf(stderr, "amppi_create: %s\n", ctx->err.c_str());
    amppi_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return AMPPI_OK;
}

int amppi_destroy(amppi_ctx* ctx) {
  if (!ctx) return AMPPI_OK;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->arena.release();
  if (ctx->d_xyz) cudaFree(ctx->d_xyz);
  if (ctx->d_xyz64) cudaFree(ctx->d_xyz64);
  if (ctx->P.cand) cudaFree(ctx->P.cand);
  if (ctx->d_injected) cudaFree(ctx->d_injected);
  if (ctx->h_xyz) cudaFreeHost(ctx->h_xyz);
  if (ctx->h_in) cudaFreeHost(ctx->h_in);
  if (ctx->h_res) cudaFreeHost(ctx->h_res);
  if (ctx->h_gather) cudaFreeHost(ctx->h_gather);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  if (ctx->plan_graph) cudaGraphExecDestroy(ctx->plan_graph);
  for (auto& sl : ctx->slots) {
    if (sl.d_xyz) cudaFree(sl.d_xyz);
    if (sl.d_in) cudaFree(sl.d_in);
    if (sl.h_in) cudaFreeHost(sl.h_in);
    if (sl.h_gather) cudaFreeHost(sl.h_gather);
    if (sl.uploaded) cudaEventDestroy(sl.uploaded);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  for (cudaStream_t x : ctx->xstream)
    if (x) cudaStreamDestroy(x);
  if (ctx->inputs_read) cudaEventDestroy(ctx->inputs_read);
  for (cudaEvent_t e : ctx->join) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->chunk_ready) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->chunk_done) cudaEventDestroy(e);
  delete ctx;
  return AMPPI_OK;
}

const char* amppi_last_error(const amppi_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int amppi_synchronize(amppi_ctx* ctx) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  return sync_and_collect(ctx);
}

int amppi_set_config(amppi_ctx* ctx, const amppi_config* cfg) {
  if (!ctx || !cfg) return ctx ? ctx->fail(AMPPI_INVALID_ARGUMENT, "null config") : AMPPI_INVALID_ARGUMENT;
  const std::string bad = validate(*cfg);
  if (!bad.empty()) return ctx->fail(AMPPI_INVALID_ARGUMENT, bad);
  const amppi_config& c = ctx->cfg;
  if (cfg->m_h != c.m_h || cfg->m_v != c.m_v || cfg->rollouts != c.rollouts || cfg->horizon != c.horizon ||
      cfg->iterations != c.iterations)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "amppi_set_config cannot change m_h, m_v, rollouts, horizon or "
                                             "iterations (the device arenas are sized from them)");
  if (ctx->shard_active) return ctx->fail(AMPPI_INVALID_ARGUMENT, "a sharded plan is in progress");
  // kernels take the configuration by value at launch: work already queued
  // keeps the old one, the next call uses the new one
  ctx->cfg = *cfg;
  ctx->dc = to_dev(*cfg);
  return AMPPI_OK;
}

int amppi_get_config(const amppi_ctx* ctx, amppi_config* cfg) {
  if (!ctx || !cfg) return AMPPI_INVALID_ARGUMENT;
  *cfg = ctx->cfg;
  return AMPPI_OK;
}

int amppi_set_schedule(amppi_ctx* ctx, const amppi_schedule* schedule) {
  if (!ctx || !schedule) return AMPPI_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->opt.schedule = *schedule;
  return AMPPI_OK;
}

void* amppi_get_stream(const amppi_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int amppi_set_stream(amppi_ctx* ctx, void* stream) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->own_stream = false;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return AMPPI_OK;
}

static int snapshot_common(amppi_ctx* ctx, const void* pts, bool f64, int64_t n, const amppi_state* pose,
                           double r_max, bool on_device = false) {
  NvtxRange nvtx_range("amppi_snapshot");
  if (!ctx || (!pts && n > 0) || !pose || n < 0) return ctx ? ctx->fail(AMPPI_INVALID_ARGUMENT, "bad arguments")
                                                            : AMPPI_INVALID_ARGUMENT;
  if (!(r_max > 0.0)) return ctx->fail(AMPPI_INVALID_ARGUMENT, "r_max must be positive");
  if (n > 0xFFFFFFFFll) return ctx->fail(AMPPI_INVALID_ARGUMENT, "at most 2^32-1 points per scene");
  if (int rc = alloc_points(ctx, n); rc != AMPPI_OK) return rc;
  const size_t bytes = static_cast<size_t>(n) * 3 * (f64 ? sizeof(double) : sizeof(float));
  if (n > 0 && !on_device) {
    // page-locked caller memory is read by the DMA engine directly; anything
    // else goes through the context's pinned staging buffer
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, pts) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    if (!pinned) cudaGetLastError();  // clear a possible "invalid value" from unregistered memory
    const void* src = pts;
    if (!pinned) {
      std::memcpy(ctx->h_xyz, pts, bytes);
      src = ctx->h_xyz;
    }
    CK(cudaMemcpyAsync(f64 ? static_cast<void*>(ctx->d_xyz64) : static_cast<void*>(ctx->d_xyz), src, bytes,
                       cudaMemcpyHostToDevice, ctx->stream));
  }
  put_pose(ctx->hin.poses, pose);
  ctx->hin.offsets[0] = 0;
  ctx->hin.offsets[1] = n;
  // upload pose + offsets (the start of the input block)
  CK(cudaMemcpyAsync(ctx->din.poses, ctx->hin.poses, 10 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->din.offsets, ctx->hin.offsets, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->inputs_read, ctx->stream));
  BatchIn in = batch_from_block(ctx, 1, r_max, f64);
  if (on_device) in.xyz = static_cast<const float*>(pts);  // read straight from the caller's device buffer
  if (int rc = run_cycle(ctx, in, n, true, false, false); rc != AMPPI_OK) return rc;
  ctx->have_snapshot = true;
  ctx->snap_d_max = ctx->dc.col_d_max;
  ctx->snap_r_max = r_max;
  ctx->snap_points = n;
  std::memcpy(ctx->snap_pose, pose, sizeof(ctx->snap_pose));
  // Return once the inputs have been copied (the caller's buffer and the
  // staging block may be reused); the snapshot kernels keep running and the
  // plan that follows queues behind them on the stream -- no host round trip
  // between build_snapshot and plan_step.  Kernel errors surface at the next
  // synchronising call.
  CK(cudaEventSynchronize(ctx->inputs_read));
  return AMPPI_OK;
}

int amppi_snapshot(amppi_ctx* ctx, const float* xyz, int64_t n, const amppi_state* pose, double r_max) {
  return snapshot_common(ctx, xyz, false, n, pose, r_max);
}

int amppi_snapshot_f64(amppi_ctx* ctx, const double* xyz, int64_t n, const amppi_state* pose, double r_max) {
  return snapshot_common(ctx, xyz, true, n, pose, r_max);
}

int amppi_snapshot_device(amppi_ctx* ctx, const float* d_xyz, int64_t n, const amppi_state* pose, double r_max) {
  return snapshot_common(ctx, d_xyz, false, n, pose, r_max, true);
}

int amppi_snapshot_download(amppi_ctx* ctx, amppi_snapshot_view* v) {
  if (!ctx || !v) return AMPPI_INVALID_ARGUMENT;
  if (!ctx->have_snapshot) return ctx->fail(AMPPI_NO_SNAPSHOT, "no snapshot");
  if (int rc = sync_and_collect(ctx); rc != AMPPI_OK) return rc;  // the snapshot kernels may still run
  const Perception& P = ctx->P;
  if ((v->ranges || v->has_point || v->nearest) && !P.ranges)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "verification views need max_scenes <= 64");
  if (v->ranges) CK(cudaMemcpy(v->ranges, P.ranges, kCells * sizeof(double), cudaMemcpyDeviceToHost));
  if (v->has_point) CK(cudaMemcpy(v->has_point, P.has_point, kCells, cudaMemcpyDeviceToHost));
  if (v->nearest) CK(cudaMemcpy(v->nearest, P.nearest, kCells * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  if (v->safe_range) CK(cudaMemcpy(v->safe_range, P.safe_range, kCoarse * sizeof(double), cudaMemcpyDeviceToHost));
  if (v->safe_dir) CK(cudaMemcpy(v->safe_dir, P.safe_dir, kCoarse * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  if (v->safe_point) CK(cudaMemcpy(v->safe_point, P.safe_point, kCoarse * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  int32_t nf = 0;
  CK(cudaMemcpy(&nf, P.n_filtered, sizeof(int32_t), cudaMemcpyDeviceToHost));
  v->n_filtered = nf;
  if (v->filtered && nf > 0)
    CK(cudaMemcpy(v->filtered, P.filtered, static_cast<size_t>(nf) * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  return AMPPI_OK;
}

}  // extern "C"

namespace {

// plan_step inputs of the single-scene API -> device input block (+ optional
// injected perturbations); *in receives the batch view.
int stage_plan_inputs(amppi_ctx* ctx, const amppi_state* x, const amppi_goal* goal, const double* previous,
                      int32_t previous_len, const amppi_control* last_applied, uint64_t cycle, uint64_t seed,
                      const double* injected, BatchIn* in_out) {
  if (!x || !goal || !last_applied) return ctx->fail(AMPPI_INVALID_ARGUMENT, "null argument");
  if (!ctx->have_snapshot) return ctx->fail(AMPPI_NO_SNAPSHOT, "amppi_plan before amppi_snapshot");
  if (ctx->snap_d_max != ctx->dc.col_d_max)
    return ctx->fail(AMPPI_NO_SNAPSHOT, "the snapshot's collision grid was built for another col_d_max");
  const DevConfig& dc = ctx->dc;
  const int M = dc.M, K = dc.K, N = dc.N;
  InputBlock& h = ctx->hin;
  put_pose(h.states, x);
  std::memcpy(h.goals, goal, 10 * sizeof(double));
  std::memcpy(h.last, last_applied, 4 * sizeof(double));
  const bool has_prev = previous && previous_len == N;
  if (has_prev) std::memcpy(h.prev, previous, static_cast<size_t>(N) * 4 * sizeof(double));
  h.prev_len[0] = has_prev ? N : 0;
  h.cycles[0] = cycle;
  h.seeds[0] = seed;
  // one upload of the whole single-scene input block (poses..prev_len)
  const size_t span = static_cast<size_t>(reinterpret_cast<unsigned char*>(h.prev_len + 1) -
                                          reinterpret_cast<unsigned char*>(h.poses));
  CK(cudaMemcpyAsync(ctx->din.poses, h.poses, span, cudaMemcpyHostToDevice, ctx->stream));
  BatchIn in = batch_from_block(ctx, 1, ctx->snap_r_max, false);
  if (injected) {
    const size_t bytes = static_cast<size_t>(dc.iterations) * M * K * N * 4 * sizeof(double);
    if (bytes > ctx->injected_bytes) {
      if (ctx->d_injected) cudaFree(ctx->d_injected);
      ctx->d_injected = nullptr;
      CK(cudaMalloc(&ctx->d_injected, bytes));
      ctx->injected_bytes = bytes;
    }
    CK(cudaMemcpyAsync(ctx->d_injected, injected, bytes, cudaMemcpyHostToDevice, ctx->stream));
    in.injected = ctx->d_injected;
  }
  *in_out = in;
  return AMPPI_OK;
}

// Results of a single-scene plan (k_gather'd block + optional arrays) ->
// caller buffers; syncs the stream.
int collect_plan_result(amppi_ctx* ctx, amppi_plan_result* out, bool want_states) {
  const DevConfig& dc = ctx->dc;
  const int M = dc.M, K = dc.K, N = dc.N;
  CK(cudaMemcpyAsync(ctx->h_res, ctx->d_res, ctx->dres.bytes, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<float> c32;
  std::vector<double> c64;
  if (out && out->sample_costs) {
    if (ctx->opt.precision == 32) {
      c32.resize(static_cast<size_t>(M) * K);
      CK(cudaMemcpyAsync(c32.data(), ctx->pl.cost32, c32.size() * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      CK(cudaMemcpyAsync(out->sample_costs, ctx->pl.cost64, static_cast<size_t>(M) * K * sizeof(double),
                         cudaMemcpyDeviceToHost, ctx->stream));
    }
  }
  if (want_states && out->winner_states)
    CK(cudaMemcpyAsync(out->winner_states, ctx->pl.winner_states, static_cast<size_t>(N + 1) * 10 * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (want_states && out->winner_controls)
    CK(cudaMemcpyAsync(out->winner_controls, ctx->pl.winner_controls, static_cast<size_t>(N) * 4 * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (int rc = sync_and_collect(ctx); rc != AMPPI_OK) return rc;
  const ResultBlock& r = ctx->hres;
  const int status = r.status[0];
  if (out) {
    if (!c32.empty())
      for (size_t i = 0; i < c32.size(); ++i) out->sample_costs[i] = std::fabs(c32[i]);  // flagged: a lower bound
    out->winner = r.winner[0];
    if (status == 0) {
      out->control.thrust = r.control[0];
      for (int i = 0; i < 3; ++i) out->control.omega[i] = r.control[1 + i];
      for (int i = 0; i < 5; ++i) out->breakdown[i] = r.breakdown[static_cast<size_t>(r.winner[0]) * 5 + i];
    }
    for (int m = 0; m < M; ++m) {
      if (out->stage1) out->stage1[m] = r.stage1[m];
      if (out->stage2) out->stage2[m] = r.stage2[m];
      if (out->ess) out->ess[m] = r.ess[m];
      if (out->valid) out->valid[m] = r.valid[m];
      if (out->nominal)
        for (int i = 0; i < N * 4; ++i)
          out->nominal[static_cast<size_t>(m) * N * 4 + i] =
              r.valid[m] ? r.nominal[static_cast<size_t>(m) * N * 4 + i] : std::numeric_limits<double>::quiet_NaN();
      for (int a = 0; a < 3; ++a) {
        if (out->anchor_initial) out->anchor_initial[3 * m + a] = r.anchor_init[3 * m + a];
        if (out->anchor_refined) out->anchor_refined[3 * m + a] = r.anchor_ref[3 * m + a];
        if (out->anchor_safe_dir) out->anchor_safe_dir[3 * m + a] = r.anchor_dir[3 * m + a];
      }
      if (out->anchor_safe_range) out->anchor_safe_range[m] = r.anchor_range[m];
      if (out->anchor_ij) {
        out->anchor_ij[2 * m] = r.anchor_ij[2 * m];
        out->anchor_ij[2 * m + 1] = r.anchor_ij[2 * m + 1];
      }
      if (out->guide_coeffs)
        for (int i = 0; i < 18; ++i) out->guide_coeffs[18 * m + i] = r.guide_coef[18 * m + i];
    }
  }
  if (status != 0) return ctx->fail(AMPPI_PLANNING_FAILED, "planning failed");
  return AMPPI_OK;
}

}  // namespace


extern "C" {

int amppi_plan(amppi_ctx* ctx, const amppi_state* x, const amppi_goal* goal, const double* previous,
               int32_t previous_len, const amppi_control* last_applied, uint64_t cycle, uint64_t seed,
               const double* injected, amppi_plan_result* out) {
  NvtxRange nvtx_range("amppi_plan");
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  BatchIn in{};
  if (int rc = stage_plan_inputs(ctx, x, goal, previous, previous_len, last_applied, cycle, seed, injected, &in);
      rc != AMPPI_OK)
    return rc;
  const bool want_states = out && (out->winner_states || out->winner_controls);
  // The plan kernels of a single-scene call depend only on the sizes, the
  // configuration, r_max and the context's (fixed) arrays: they are captured
  // once as a CUDA graph and replayed (one launch instead of ~12).
  const bool graph = !ctx->timer.enabled && ctx->opt.schedule.plan_graph >= 0;
  if (graph) {
    amppi_ctx::PlanGraphKey key;
    key.want_states = want_states;
    key.injected = in.injected != nullptr;
    key.r_max = in.r_max;
    key.points_gen = ctx->points_gen;
    key.cfg = ctx->cfg;
    const amppi_ctx::PlanGraphKey& k0 = ctx->plan_graph_key;
    const bool hit = ctx->plan_graph && k0.want_states == key.want_states && k0.injected == key.injected &&
                     k0.r_max == key.r_max && k0.points_gen == key.points_gen &&
                     std::memcmp(&k0.cfg, &key.cfg, sizeof(key.cfg)) == 0;
    if (!hit) {
      if (ctx->plan_graph) cudaGraphExecDestroy(ctx->plan_graph);
      ctx->plan_graph = nullptr;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      const int rc = run_cycle(ctx, in, ctx->snap_points, false, true, want_states);
      const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
      if (rc != AMPPI_OK) return rc;
      if (ce != cudaSuccess) return ctx->cuda_fail(ce, "plan graph capture");
      const cudaError_t ie = cudaGraphInstantiate(&ctx->plan_graph, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) return ctx->cuda_fail(ie, "plan graph instantiate");
      ctx->plan_graph_key = key;
    }
    CK(cudaGraphLaunch(ctx->plan_graph, ctx->stream));
  } else if (int rc = run_cycle(ctx, in, ctx->snap_points, false, true, want_states); rc != AMPPI_OK) {
    return rc;
  }
  return collect_plan_result(ctx, out, want_states);
}

// ---- sample-sharded plan (config C4) ----
int amppi_shard_begin(amppi_ctx* ctx, const amppi_state* x, const amppi_goal* goal, const double* previous,
                      int32_t previous_len, const amppi_control* last_applied, uint64_t cycle, uint64_t seed,
                      int32_t k_begin, int32_t k_end) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (ctx->opt.precision != 32) return ctx->fail(AMPPI_INVALID_ARGUMENT, "sample sharding needs precision 32");
  if (k_begin < 0 || k_end > ctx->dc.K || k_begin >= k_end)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "sample range out of [0, rollouts)");
  BatchIn in{};
  if (int rc = stage_plan_inputs(ctx, x, goal, previous, previous_len, last_applied, cycle, seed, nullptr, &in);
      rc != AMPPI_OK)
    return rc;
  ctx->shard_dc = ctx->dc;
  ctx->shard_dc.k_lo = k_begin;
  ctx->shard_dc.k_hi = k_end;
  ctx->shard_in = in;
  ctx->shard_active = true;
  cudaError_t e = launch_plan_begin(in, ctx->P, ctx->pl, ctx->shard_dc, ctx->stream, &ctx->timer);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_plan_begin");
}

int amppi_shard_screen(amppi_ctx* ctx, int32_t iter, float* local_min) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (!ctx->shard_active || !local_min || iter < 0 || iter >= ctx->dc.iterations)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "amppi_shard_screen: no shard plan / bad iteration");
  cudaError_t e = launch_shard_screen(ctx->shard_in, ctx->P, ctx->pl, ctx->shard_dc, iter, local_min, ctx->stream,
                                      &ctx->timer);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_shard_screen");
}

int amppi_shard_partials(amppi_ctx* ctx, int32_t iter, const float* global_min, double* partials) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (!ctx->shard_active || !global_min || !partials || iter < 0 || iter >= ctx->dc.iterations)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "amppi_shard_partials: no shard plan / bad argument");
  cudaError_t e = launch_shard_partials(ctx->shard_in, ctx->P, ctx->pl, ctx->shard_dc, ctx->cand_k, ctx->cand_s,
                                        ctx->cand_w, ctx->pairs, ctx->pair_count, iter, global_min, partials,
                                        ctx->stream, &ctx->timer);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_shard_partials");
}

int amppi_shard_update(amppi_ctx* ctx, int32_t iter, const double* all_partials, int32_t n_shards) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (!ctx->shard_active || !all_partials || iter < 0 || iter >= ctx->dc.iterations || n_shards < 1 ||
      n_shards > 64)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "amppi_shard_update: no shard plan / bad argument");
  cudaError_t e = launch_shard_merge(ctx->shard_in, ctx->pl, ctx->shard_dc, all_partials, n_shards, ctx->stream,
                                     &ctx->timer);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_shard_merge");
}

int amppi_shard_finish(amppi_ctx* ctx, amppi_plan_result* out) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (!ctx->shard_active) return ctx->fail(AMPPI_INVALID_ARGUMENT, "amppi_shard_finish: no shard plan");
  ctx->shard_active = false;
  const bool want_states = out && (out->winner_states || out->winner_controls);
  cudaError_t e = launch_plan_finish(ctx->shard_in, ctx->P, ctx->pl, ctx->dc, want_states, ctx->stream, &ctx->timer);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_plan_finish");
  return collect_plan_result(ctx, out, want_states);
}

int32_t amppi_shard_partials_stride(const amppi_ctx* ctx) { return ctx ? 3 + 4 * ctx->dc.N : 0; }

static int batch_outputs_gather(amppi_ctx* ctx, int S, amppi_batch_output* out, bool device_out);
static int plan_device_batch(amppi_ctx* ctx, const BatchIn& bin, int64_t max_scene);
static int ensure_gather(amppi_ctx* ctx, bool pinned);
static int gather_chunk(amppi_ctx* ctx, int s0, int s1, const amppi_batch_output* out, cudaStream_t st);
static void collect_chunk(amppi_ctx* ctx, int s0, int s1, amppi_batch_output* out);

int amppi_cycle_batch(amppi_ctx* ctx, const amppi_batch_input* in, amppi_batch_output* out) {
  NvtxRange nvtx_range("amppi_cycle_batch");
  if (!ctx || !in) return AMPPI_INVALID_ARGUMENT;
  const int S = in->n_scenes;
  if (S < 1 || S > ctx->S_cap) return ctx->fail(AMPPI_INVALID_ARGUMENT, "n_scenes out of range");
  const int N = ctx->dc.N;
  if (!in->point_offsets || !in->xyz || !in->poses || !in->states || !in->goals || !in->last_applied ||
      !in->cycles || !in->seeds)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "null batch input array");
  if (in->point_offsets[0] != 0) return ctx->fail(AMPPI_INVALID_ARGUMENT, "point_offsets[0] must be 0");
  int64_t max_scene = 0;
  for (int s = 0; s < S; ++s) {
    const int64_t n = in->point_offsets[s + 1] - in->point_offsets[s];
    if (n < 0) return ctx->fail(AMPPI_INVALID_ARGUMENT, "point_offsets must be non-decreasing");
    if (n > 0xFFFFFFFFll) return ctx->fail(AMPPI_INVALID_ARGUMENT, "at most 2^32-1 points per scene");
    max_scene = std::max(max_scene, n);
  }
  const int64_t total = in->point_offsets[S];
  if (int rc = alloc_points(ctx, total); rc != AMPPI_OK) return rc;
  ctx->have_snapshot = false;  // the batch overwrites the single-scene perception slot
  // inputs: points straight from the caller's buffer, per-scene arrays via the
  // pinned block
  InputBlock& h = ctx->hin;
  std::memcpy(h.poses, in->poses, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.states, in->states, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.goals, in->goals, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.last, in->last_applied, static_cast<size_t>(S) * 4 * sizeof(double));
  if (in->previous) std::memcpy(h.prev, in->previous, static_cast<size_t>(S) * N * 4 * sizeof(double));
  std::memcpy(h.offsets, in->point_offsets, static_cast<size_t>(S + 1) * sizeof(int64_t));
  std::memcpy(h.cycles, in->cycles, static_cast<size_t>(S) * sizeof(uint64_t));
  std::memcpy(h.seeds, in->seeds, static_cast<size_t>(S) * sizeof(uint64_t));
  for (int s = 0; s < S; ++s) h.prev_len[s] = in->previous ? (in->previous_len ? in->previous_len[s] : N) : 0;
  const size_t span = static_cast<size_t>(reinterpret_cast<unsigned char*>(h.prev_len + ctx->S_cap) -
                                          reinterpret_cast<unsigned char*>(h.poses));
  // Pipeline: the points of chunk c+1 cross PCIe on the copy stream while
  // chunk c is planned.  Chunks are whole scenes (>= 2 fused-snapshot waves);
  // results land at each scene's batch position.
  // Up to 6 chunks of >= ~8M points and >= 296 scenes (the smallest one must
  // keep the fused snapshot: >= 148 scenes).
  int chunks = static_cast<int>(std::min<int64_t>(6, std::max<int64_t>(1, total / (8 << 20))));
  chunks = std::max(1, std::min(chunks, S / 296));
  double ratio = 1.2;  // C5 on a B200 over PCIe 5: best of 4-8 chunks x ratio 1.0-1.6 (tools/pipe_sweep.py)
  const amppi_schedule& sched = ctx->opt.schedule;
  if (sched.pipeline_chunks > 0) chunks = std::max(1, std::min(S, sched.pipeline_chunks));  // tests
  if (sched.pipeline_ratio > 0.0) ratio = std::max(1.0, sched.pipeline_ratio);
  chunks = std::min(chunks, kMaxChunks);
  // the many-CTA snapshot of a scene past kFusedMaxPoints shares one candidate
  // log and counter per launch: such a batch is not split into concurrent chunks
  if (max_scene > kFusedMaxPoints) chunks = 1;
  auto first_chunk = [&](int n) { return ratio > 1.0 ? S * (ratio - 1.0) / (std::pow(ratio, n) - 1.0) : 1.0 * S / n; };
  while (chunks > 1 && first_chunk(chunks) < 148) --chunks;  // smallest chunk >= 148
  while (static_cast<int>(ctx->chunk_ready.size()) < chunks) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->chunk_ready.push_back(ev);
  }
  // the copy stream must not overwrite inputs a previous call is still using;
  // the per-scene block goes first on the copy stream (H2D copies share the
  // copy engine in issue order, so it must not queue behind the points)
  CK(cudaEventRecord(ctx->chunk_ready[0], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ready[0], 0));
  CK(cudaMemcpyAsync(ctx->din.poses, h.poses, span, cudaMemcpyHostToDevice, ctx->copy_stream));
  const bool trace = sched.trace != 0;  // diagnostics
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  tmark(ctx->copy_stream);
  // chunks rotate over the compute streams (each chunk's arrays live at its
  // own offset), so one chunk's latency-bound tail overlaps the next chunks'
  // work; every stream joins ctx->stream before the gather
  const bool concurrent = chunks > 1;
  if (concurrent)
    if (int rc = fork_streams(ctx); rc != AMPPI_OK) return rc;
  // each chunk's results are gathered and copied to the pinned mirror on its
  // own stream as soon as it is planned; the host copies chunk c out while
  // later chunks still run (C5: hides all but the last chunk's result tail)
  const bool chunk_gather = sched.chunk_gather >= 0;
  const bool chunk_out = concurrent && out && chunk_gather;
  if (chunk_out) {
    if (int rc = ensure_gather(ctx, true); rc != AMPPI_OK) return rc;
    while (static_cast<int>(ctx->chunk_done.size()) < chunks) {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ctx->chunk_done.push_back(ev);
    }
  }
  // Chunk sizes grow geometrically: the first chunk's upload is the only one
  // not hidden behind planning, so it is the smallest; later chunks grow so
  // their uploads stay ahead of the planning.
  std::vector<int> bound(chunks + 1, 0);
  {
    double w = 1.0, sum = 0.0;
    std::vector<double> cum(chunks + 1, 0.0);
    for (int c = 0; c < chunks; ++c, w *= ratio) cum[c + 1] = (sum += w);
    for (int c = 1; c <= chunks; ++c) bound[c] = static_cast<int>(std::llround(S * cum[c] / sum));
    bound[chunks] = S;
  }
  for (int c = 0; c < chunks; ++c) {
    const int s0 = bound[c];
    const int s1 = bound[c + 1];
    const int64_t p0 = in->point_offsets[s0], p1 = in->point_offsets[s1];
    if (p1 > p0)
      CK(cudaMemcpyAsync(ctx->d_xyz + 3 * p0, in->xyz + 3 * p0, static_cast<size_t>(p1 - p0) * 3 * sizeof(float),
                         cudaMemcpyHostToDevice, ctx->copy_stream));
    CK(cudaEventRecord(ctx->chunk_ready[c], ctx->copy_stream));
    tmark(ctx->copy_stream);
    const cudaStream_t cst = concurrent ? compute_stream(ctx, c) : ctx->stream;
    CK(cudaStreamWaitEvent(cst, ctx->chunk_ready[c], 0));
    int64_t max_chunk_scene = 0;
    for (int s = s0; s < s1; ++s)
      max_chunk_scene = std::max(max_chunk_scene, in->point_offsets[s + 1] - in->point_offsets[s]);
    BatchIn bin = batch_from_block(ctx, s1 - s0, in->r_max, false);
    bin.offsets += s0;
    bin.poses += 10 * s0;
    bin.states += 10 * s0;
    bin.goals += 10 * s0;
    bin.prev += static_cast<int64_t>(s0) * N * 4;
    bin.prev_len += s0;
    bin.last_applied += 4 * s0;
    bin.cycles += s0;
    bin.seeds += s0;
    if (concurrent) {
      if (int rc = run_chunk(ctx, bin, max_chunk_scene, s0, c, cst); rc != AMPPI_OK) return rc;
      if (chunk_out) {
        if (int rc = gather_chunk(ctx, s0, s1, out, cst); rc != AMPPI_OK) return rc;
        CK(cudaEventRecord(ctx->chunk_done[c], cst));
      }
    } else if (int rc = run_cycle(ctx, bin, max_chunk_scene, true, true, false, s0); rc != AMPPI_OK) {
      return rc;
    }
    tmark(cst);
  }
  if (concurrent)
    if (int rc = join_streams(ctx); rc != AMPPI_OK) return rc;
  if (trace) {
    cudaDeviceSynchronize();
    std::fprintf(stderr, "pipeline %d chunks:", chunks);
    for (size_t i = 1; i < tev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      std::fprintf(stderr, " %.2f", ms);
    }
    std::fprintf(stderr, "\n");
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  (void)max_scene;
  if (chunk_out) {
    for (int c = 0; c < chunks; ++c) {
      CK(cudaEventSynchronize(ctx->chunk_done[c]));
      collect_chunk(ctx, bound[c], bound[c + 1], out);
    }
    return sync_and_collect(ctx);
  }
  return batch_outputs_gather(ctx, S, out, false);
}

int amppi_cycle_batch_device(amppi_ctx* ctx, const amppi_batch_input* in, amppi_batch_output* out) {
  NvtxRange nvtx_range("amppi_cycle_batch_device");
  if (!ctx || !in) return AMPPI_INVALID_ARGUMENT;
  const int S = in->n_scenes;
  if (S < 1 || S > ctx->S_cap) return ctx->fail(AMPPI_INVALID_ARGUMENT, "n_scenes out of range");
  if (!in->point_offsets || !in->xyz || !in->poses || !in->states || !in->goals || !in->last_applied ||
      !in->cycles || !in->seeds)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "null batch input array");
  ctx->have_snapshot = false;  // the batch overwrites the single-scene perception slot
  BatchIn bin{};
  bin.xyz = in->xyz;
  bin.xyz64 = nullptr;
  bin.offsets = in->point_offsets;
  bin.poses = reinterpret_cast<const double*>(in->poses);
  bin.states = reinterpret_cast<const double*>(in->states);
  bin.goals = reinterpret_cast<const double*>(in->goals);
  bin.prev = in->previous;
  bin.prev_len = in->previous_len;
  bin.last_applied = reinterpret_cast<const double*>(in->last_applied);
  bin.cycles = in->cycles;
  bin.seeds = in->seeds;
  bin.injected = nullptr;
  bin.S = S;
  bin.r_max = in->r_max;
  // per-scene point counts are device-resident: size the keying grid from the
  // context's capacity (blocks beyond a scene's end exit immediately)
  const int64_t max_scene = std::max<int64_t>(1, ctx->P_cap / S);
  if (ctx->P.cand_cap < ctx->P_cap) return ctx->fail(AMPPI_INVALID_ARGUMENT, "point capacity");
  if (int rc = plan_device_batch(ctx, bin, max_scene); rc != AMPPI_OK) return rc;
  return batch_outputs_gather(ctx, S, out, true);
}

// Snapshot + plan of a batch whose inputs are on the device (bin), on the
// context's compute streams; results stay in the plan arrays.
static int plan_device_batch(amppi_ctx* ctx, const BatchIn& bin, int64_t max_scene) {
  const int S = bin.S;
  // Device-resident inputs need no upload pipeline, but two chunks on the
  // compute streams still overlap one chunk's latency-bound tail kernels with
  // the other's work (C5, r02 kernels: 1 chunk 17.03 ms, 2 chunks 16.54,
  // 3 chunks 16.71, 4 chunks 19.37, 6 chunks 19.0; gpurun_out/r44_*.log).
  int chunks = std::min(pipeline_streams(ctx), S / (2 * 148));
  chunks = std::max(1, std::min(chunks, 2));
  if (ctx->opt.schedule.device_chunks > 0) chunks = std::max(1, std::min(kMaxChunks, ctx->opt.schedule.device_chunks));
  if (chunks > 1 && S / chunks < 148) chunks = 1;
  // scenes past kFusedMaxPoints take the many-CTA snapshot (shared candidate
  // log): no concurrent chunks
  if (max_scene > kFusedMaxPoints) chunks = 1;
  if (chunks == 1) return run_cycle(ctx, bin, max_scene, true, true, false);
  if (int rc = fork_streams(ctx); rc != AMPPI_OK) return rc;
  for (int c = 0; c < chunks; ++c) {
    const int s0 = static_cast<int>(static_cast<int64_t>(S) * c / chunks);
    const int s1 = static_cast<int>(static_cast<int64_t>(S) * (c + 1) / chunks);
    BatchIn cb = bin;
    cb.S = s1 - s0;
    cb.offsets += s0;
    cb.poses += 10 * s0;
    cb.states += 10 * s0;
    cb.goals += 10 * s0;
    if (cb.prev) cb.prev += static_cast<int64_t>(s0) * ctx->dc.N * 4;
    if (cb.prev_len) cb.prev_len += s0;
    cb.last_applied += 4 * s0;
    cb.cycles += s0;
    cb.seeds += s0;
    if (int rc = run_chunk(ctx, cb, max_scene, s0, c, compute_stream(ctx, c)); rc != AMPPI_OK) return rc;
  }
  return join_streams(ctx);
}

int amppi_kernel_times(amppi_ctx* ctx, const char** names, double* ms, int64_t* launches, int32_t cap,
                       int32_t* count) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  int i = 0;
  for (const auto& kv : ctx->timer.totals) {
    if (i < cap) {
      if (names) names[i] = kv.first.c_str();
      if (ms) ms[i] = kv.second.first;
      if (launches) launches[i] = kv.second.second;
    }
    ++i;
  }
  if (count) *count = i;
  return AMPPI_OK;
}

int amppi_kernel_times_reset(amppi_ctx* ctx) {
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (int rc = sync_and_collect(ctx); rc != AMPPI_OK) return rc;  // drop in-flight events too
  ctx->timer.totals.clear();
  return AMPPI_OK;
}

int amppi_screen_drift(amppi_ctx* ctx, const amppi_batch_input* in, int32_t iteration, int32_t sample_stride,
                       double* stats) {
  NvtxRange nvtx_range("amppi_screen_drift");
  if (!ctx || !in || !stats) return AMPPI_INVALID_ARGUMENT;
  const DevConfig& dc = ctx->dc;
  const int S = in->n_scenes;
  if (S < 1 || S > ctx->S_cap) return ctx->fail(AMPPI_INVALID_ARGUMENT, "n_scenes out of range");
  if (sample_stride < 1 || iteration < 0 || iteration >= dc.iterations)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "sample_stride < 1 or iteration out of range");
  if (dc.N > 64) return ctx->fail(AMPPI_INVALID_ARGUMENT, "horizon > 64");
  if (!in->states || !in->goals || !in->cycles || !in->seeds)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "null batch input array");
  BatchIn bin{};
  bin.states = reinterpret_cast<const double*>(in->states);
  bin.goals = reinterpret_cast<const double*>(in->goals);
  bin.cycles = in->cycles;
  bin.seeds = in->seeds;
  bin.S = S;
  const int kn = (dc.k_hi - dc.k_lo + sample_stride - 1) / sample_stride;
  const int64_t per_scene = static_cast<int64_t>(dc.M) * kn;
  // scenes per launch pair: at most 512 MB of per-step records
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(S, (int64_t{1} << 29) / (per_scene * dc.N * 16)));
  float4* steps = nullptr;
  float* cost = nullptr;
  unsigned long long* acc = nullptr;
  auto release = [&] {
    cudaFree(steps);
    cudaFree(cost);
    cudaFree(acc);
  };
  cudaError_t e = cudaMalloc(&steps, static_cast<size_t>(chunk * per_scene * dc.N) * sizeof(float4));
  if (e == cudaSuccess) e = cudaMalloc(&cost, static_cast<size_t>(chunk * per_scene) * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&acc, (kDriftSlots + 1) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(acc, 0, (kDriftSlots + 1) * sizeof(unsigned long long), ctx->stream);
  for (int64_t s0 = 0; e == cudaSuccess && s0 < S; s0 += chunk) {
    const int n = static_cast<int>(std::min<int64_t>(chunk, S - s0));
    e = launch_drift32(bin, ctx->P, ctx->pl, dc, iteration, static_cast<int>(s0), n, sample_stride, steps, cost,
                       ctx->stream);
    if (e == cudaSuccess)
      e = launch_drift64(bin, ctx->P, ctx->pl, dc, iteration, static_cast<int>(s0), n, sample_stride, steps, cost, acc,
                         ctx->stream);
  }
  unsigned long long h[kDriftSlots] = {};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  release();
  if (e != cudaSuccess) return ctx->cuda_fail(e, "amppi_screen_drift");
  for (int i = 0; i < kDriftSlots; ++i) {
    const bool is_max = i == 1 || i == 2 || i == 6;
    double v;
    std::memcpy(&v, &h[i], sizeof(v));
    stats[i] = is_max ? v : static_cast<double>(h[i]);
  }
  return AMPPI_OK;
}

}  // extern "C"

// Gathered results: one field-major block of S_cap scenes (device, and a
// pinned host mirror for the per-chunk copies of the host pipeline).
static int ensure_gather(amppi_ctx* ctx, bool pinned) {
  const size_t Sc = static_cast<size_t>(ctx->S_cap);
  const size_t bytes = Sc * (2 * sizeof(int32_t) + (4 + 5 + static_cast<size_t>(ctx->dc.N) * 4 + ctx->dc.M) * sizeof(double)) + 256;
  void* p = nullptr;
  if (!ctx->d_gather) {
    CK(ctx->arena.alloc(&p, bytes));
    ctx->d_gather = static_cast<unsigned char*>(p);
  }
  if (pinned && !ctx->h_gather) {
    CK(cudaMallocHost(&p, bytes));
    ctx->h_gather = static_cast<unsigned char*>(p);
  }
  return AMPPI_OK;
}

// The gather block's fields, shifted to scene s0.
static GatherOut gather_view(const amppi_ctx* ctx, unsigned char* base, int64_t s0) {
  const size_t Sc = static_cast<size_t>(ctx->S_cap);
  const int64_t M = ctx->dc.M, N = ctx->dc.N;
  unsigned char* cur = base;
  GatherOut g{};
  g.status = carve<int32_t>(cur, Sc) + s0;
  g.winner = carve<int32_t>(cur, Sc) + s0;
  g.control = carve<double>(cur, Sc * 4) + 4 * s0;
  g.breakdown = carve<double>(cur, Sc * 5) + 5 * s0;
  g.winner_nominal = carve<double>(cur, Sc * N * 4) + N * 4 * s0;
  g.stage2 = carve<double>(cur, Sc * M) + M * s0;
  return g;
}

// Scenes [s0, s1) of the host pipeline: gather on the chunk's stream and copy
// the requested fields into the pinned mirror, so they cross PCIe while later
// chunks are planned.  chunk_done[c] marks the copies.
static int gather_chunk(amppi_ctx* ctx, int s0, int s1, const amppi_batch_output* out, cudaStream_t st) {
  const int64_t M = ctx->dc.M, N = ctx->dc.N, n = s1 - s0;
  GatherOut d = gather_view(ctx, ctx->d_gather, s0);
  const GatherOut h = gather_view(ctx, ctx->h_gather, s0);
  if (!out->status) d.status = nullptr;
  if (!out->winner) d.winner = nullptr;
  if (!out->control) d.control = nullptr;
  if (!out->breakdown) d.breakdown = nullptr;
  if (!out->winner_nominal) d.winner_nominal = nullptr;
  if (!out->stage2) d.stage2 = nullptr;
  cudaError_t e = launch_gather(shift_plan(ctx->pl, s0, ctx->dc), ctx->dc, static_cast<int>(n), d, st);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_gather");
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    return src ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
  };
  CK(d2h(h.status, d.status, n * sizeof(int32_t)));
  CK(d2h(h.winner, d.winner, n * sizeof(int32_t)));
  CK(d2h(h.control, d.control, n * 4 * sizeof(double)));
  CK(d2h(h.breakdown, d.breakdown, n * 5 * sizeof(double)));
  CK(d2h(h.winner_nominal, d.winner_nominal, n * N * 4 * sizeof(double)));
  CK(d2h(h.stage2, d.stage2, n * M * sizeof(double)));
  return AMPPI_OK;
}

// Copy scenes [s0, s1) from the pinned mirror into the caller's buffers (after
// the chunk's copies completed).
static void collect_chunk(amppi_ctx* ctx, int s0, int s1, amppi_batch_output* out) {
  const int64_t M = ctx->dc.M, N = ctx->dc.N, n = s1 - s0;
  const GatherOut h = gather_view(ctx, ctx->h_gather, s0);
  auto put = [](void* dst, const void* src, size_t bytes) {
    if (dst) std::memcpy(dst, src, bytes);
  };
  put(out->status ? out->status + s0 : nullptr, h.status, n * sizeof(int32_t));
  put(out->winner ? out->winner + s0 : nullptr, h.winner, n * sizeof(int32_t));
  put(out->control ? out->control + 4 * s0 : nullptr, h.control, n * 4 * sizeof(double));
  put(out->breakdown ? out->breakdown + 5 * s0 : nullptr, h.breakdown, n * 5 * sizeof(double));
  put(out->winner_nominal ? out->winner_nominal + N * 4 * s0 : nullptr, h.winner_nominal, n * N * 4 * sizeof(double));
  put(out->stage2 ? out->stage2 + M * s0 : nullptr, h.stage2, n * M * sizeof(double));
}

// Gather the per-scene winner outputs on the device; copy them out for the
// host-pointer API.
static int batch_outputs_gather(amppi_ctx* ctx, int S, amppi_batch_output* out, bool device_out) {
  if (!out) return device_out ? AMPPI_OK : sync_and_collect(ctx);
  const int M = ctx->dc.M, N = ctx->dc.N;
  if (device_out) {
    GatherOut g{out->status, out->winner, out->control, out->winner_nominal, out->stage2, out->breakdown};
    cudaError_t e = launch_gather(ctx->pl, ctx->dc, S, g, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_gather");
    return AMPPI_OK;
  }
  if (int rc = ensure_gather(ctx, false); rc != AMPPI_OK) return rc;
  const GatherOut g = gather_view(ctx, ctx->d_gather, 0);
  cudaError_t e = launch_gather(ctx->pl, ctx->dc, S, g, ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_gather");
  const cudaStream_t st = ctx->stream;
  if (out->status) CK(cudaMemcpyAsync(out->status, g.status, S * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (out->winner) CK(cudaMemcpyAsync(out->winner, g.winner, S * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (out->control) CK(cudaMemcpyAsync(out->control, g.control, S * 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out->breakdown)
    CK(cudaMemcpyAsync(out->breakdown, g.breakdown, S * 5 * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out->winner_nominal)
    CK(cudaMemcpyAsync(out->winner_nominal, g.winner_nominal, static_cast<size_t>(S) * N * 4 * sizeof(double),
                       cudaMemcpyDeviceToHost, st));
  if (out->stage2)
    CK(cudaMemcpyAsync(out->stage2, g.stage2, static_cast<size_t>(S) * M * sizeof(double), cudaMemcpyDeviceToHost, st));
  return sync_and_collect(ctx);
}

// ---------------------------------------------------------------------------
// Streaming batches: submit returns once the batch is queued; wait returns its
// results.  Inputs go through one of three device slots: with two batches in
// flight the next batch's point upload (copy engine) runs under the current
// batch's planning (SMs) -- the steady state is max(upload, planning) instead
// of their sum; a third lets the caller queue batch t+1 before collecting
// batch t-1, so the upload starts the moment the copy engine is free rather
// than after a host round trip.  Planning arrays are shared: batches plan one
// after another on the context's streams.
// ---------------------------------------------------------------------------
static size_t gather_bytes(const amppi_ctx* ctx) {
  const size_t Sc = static_cast<size_t>(ctx->S_cap);
  return Sc * (2 * sizeof(int32_t) + (4 + 5 + static_cast<size_t>(ctx->dc.N) * 4 + ctx->dc.M) * sizeof(double)) + 256;
}

extern "C" int amppi_cycle_batch_submit(amppi_ctx* ctx, const amppi_batch_input* in, int64_t* ticket) {
  NvtxRange nvtx_range("amppi_cycle_batch_submit");
  if (!ctx || !in || !ticket) return AMPPI_INVALID_ARGUMENT;
  const int S = in->n_scenes;
  if (S < 1 || S > ctx->S_cap) return ctx->fail(AMPPI_INVALID_ARGUMENT, "n_scenes out of range");
  const int N = ctx->dc.N;
  if (!in->point_offsets || !in->xyz || !in->poses || !in->states || !in->goals || !in->last_applied ||
      !in->cycles || !in->seeds)
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "null batch input array");
  if (in->point_offsets[0] != 0) return ctx->fail(AMPPI_INVALID_ARGUMENT, "point_offsets[0] must be 0");
  int64_t max_scene = 0;
  for (int s = 0; s < S; ++s) {
    const int64_t n = in->point_offsets[s + 1] - in->point_offsets[s];
    if (n < 0) return ctx->fail(AMPPI_INVALID_ARGUMENT, "point_offsets must be non-decreasing");
    if (n > 0xFFFFFFFFll) return ctx->fail(AMPPI_INVALID_ARGUMENT, "at most 2^32-1 points per scene");
    max_scene = std::max(max_scene, n);
  }
  const int64_t total = in->point_offsets[S];
  amppi_ctx::StreamSlot& sl = ctx->slots[ctx->next_ticket % amppi_ctx::kStreamSlots];
  if (sl.busy) return ctx->fail(AMPPI_INVALID_ARGUMENT, "three batches already in flight: wait for one first");
  if (total > ctx->P_cap) {  // the candidate log and point tables are sized by P_cap
    CK(cudaDeviceSynchronize());
    if (int rc = alloc_points(ctx, total); rc != AMPPI_OK) return rc;
  }
  if (int rc = ensure_gather(ctx, false); rc != AMPPI_OK) return rc;
  void* p = nullptr;
  if (!sl.uploaded) {
    CK(cudaEventCreateWithFlags(&sl.uploaded, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    const InputBlock probe = layout_inputs(nullptr, ctx->S_cap, N);
    CK(cudaMalloc(&p, probe.bytes));
    sl.d_in = static_cast<unsigned char*>(p);
    CK(cudaMallocHost(&p, probe.bytes));
    sl.h_in = static_cast<unsigned char*>(p);
    sl.din = layout_inputs(sl.d_in, ctx->S_cap, N);
    sl.hin = layout_inputs(sl.h_in, ctx->S_cap, N);
    CK(cudaMallocHost(&p, gather_bytes(ctx)));
    sl.h_gather = static_cast<unsigned char*>(p);
  }
  if (sl.xyz_cap < total) {
    CK(cudaStreamSynchronize(ctx->copy_stream));
    if (sl.d_xyz) cudaFree(sl.d_xyz);
    sl.d_xyz = nullptr;
    sl.xyz_cap = std::max<int64_t>(total, 1024);
    CK(cudaMalloc(&p, static_cast<size_t>(sl.xyz_cap) * 3 * sizeof(float)));
    sl.d_xyz = static_cast<float*>(p);
  }
  // per-scene arrays -> the slot's pinned block (its previous upload is over:
  // that batch was waited for)
  InputBlock& h = sl.hin;
  std::memcpy(h.poses, in->poses, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.states, in->states, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.goals, in->goals, static_cast<size_t>(S) * 10 * sizeof(double));
  std::memcpy(h.last, in->last_applied, static_cast<size_t>(S) * 4 * sizeof(double));
  if (in->previous) std::memcpy(h.prev, in->previous, static_cast<size_t>(S) * N * 4 * sizeof(double));
  std::memcpy(h.offsets, in->point_offsets, static_cast<size_t>(S + 1) * sizeof(int64_t));
  std::memcpy(h.cycles, in->cycles, static_cast<size_t>(S) * sizeof(uint64_t));
  std::memcpy(h.seeds, in->seeds, static_cast<size_t>(S) * sizeof(uint64_t));
  for (int s = 0; s < S; ++s) h.prev_len[s] = in->previous ? (in->previous_len ? in->previous_len[s] : N) : 0;
  const size_t span = static_cast<size_t>(reinterpret_cast<unsigned char*>(h.prev_len + ctx->S_cap) -
                                          reinterpret_cast<unsigned char*>(h.poses));
  // upload on the copy stream (the slot's device buffers were last read by
  // that earlier batch's planning, which it waited for)
  CK(cudaStreamWaitEvent(ctx->copy_stream, sl.done, 0));
  CK(cudaMemcpyAsync(sl.din.poses, h.poses, span, cudaMemcpyHostToDevice, ctx->copy_stream));
  if (total > 0)
    CK(cudaMemcpyAsync(sl.d_xyz, in->xyz, static_cast<size_t>(total) * 3 * sizeof(float), cudaMemcpyHostToDevice,
                       ctx->copy_stream));
  CK(cudaEventRecord(sl.uploaded, ctx->copy_stream));
  // plan on the compute streams once uploaded, then gather into the slot's pinned mirror
  CK(cudaStreamWaitEvent(ctx->stream, sl.uploaded, 0));
  BatchIn bin{};
  bin.xyz = sl.d_xyz;
  bin.offsets = sl.din.offsets;
  bin.poses = sl.din.poses;
  bin.states = sl.din.states;
  bin.goals = sl.din.goals;
  bin.prev = sl.din.prev;
  bin.prev_len = sl.din.prev_len;
  bin.last_applied = sl.din.last;
  bin.cycles = sl.din.cycles;
  bin.seeds = sl.din.seeds;
  bin.S = S;
  bin.r_max = in->r_max;
  ctx->have_snapshot = false;  // the batch overwrites the single-scene perception slot
  if (int rc = plan_device_batch(ctx, bin, max_scene); rc != AMPPI_OK) return rc;
  const GatherOut g = gather_view(ctx, ctx->d_gather, 0);
  cudaError_t e = launch_gather(ctx->pl, ctx->dc, S, g, ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_gather");
  CK(cudaMemcpyAsync(sl.h_gather, ctx->d_gather, gather_bytes(ctx), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(sl.done, ctx->stream));
  sl.busy = true;
  sl.S = S;
  sl.ticket = ctx->next_ticket;
  *ticket = ctx->next_ticket++;
  return AMPPI_OK;
}

extern "C" int amppi_cycle_batch_wait(amppi_ctx* ctx, int64_t ticket, amppi_batch_output* out) {
  NvtxRange nvtx_range("amppi_cycle_batch_wait");
  if (!ctx) return AMPPI_INVALID_ARGUMENT;
  if (ticket < 0) return ctx->fail(AMPPI_INVALID_ARGUMENT, "unknown ticket");
  amppi_ctx::StreamSlot& sl = ctx->slots[ticket % amppi_ctx::kStreamSlots];
  if (!sl.busy || sl.ticket != ticket) return ctx->fail(AMPPI_INVALID_ARGUMENT, "unknown or already collected ticket");
  CK(cudaEventSynchronize(sl.done));
  sl.busy = false;
  if (ctx->timer.enabled) ctx->timer.collect();
  if (ctx->h_flags && *ctx->h_flags) {
    *ctx->h_flags = 0u;
    return ctx->fail(AMPPI_INVALID_ARGUMENT, "a batch exceeded the context's point capacity; its results are invalid");
  }
  if (out) {
    unsigned char* saved = ctx->h_gather;
    ctx->h_gather = sl.h_gather;  // collect_chunk reads the pinned mirror
    collect_chunk(ctx, 0, sl.S, out);
    ctx->h_gather = saved;
  }
  return AMPPI_OK;
}

// ---------------------------------------------------------------------------
// GPU-resident closed loop
// ---------------------------------------------------------------------------
struct amppi_loop {
  amppi_ctx* ctx{nullptr};
  amppi_dev::LoopDev L{};
  amppi_dev::LoopParams prm{};
  void* mem{nullptr};
  int64_t max_cycles{0};
  cudaGraphExec_t cycle_graph{nullptr};  // one captured cycle, replayed (all state lives on the device)
  uint64_t graph_points_gen{0};          // ctx->points_gen at capture
};

static_assert(sizeof(amppi_loop_record) == sizeof(amppi_dev::LoopRecord), "record layout");
static_assert(sizeof(amppi_episode_metrics) == sizeof(amppi_dev::LoopMetrics), "metrics layout");

extern "C" {

int amppi_loop_create(amppi_ctx* ctx, int32_t scene_kind, uint64_t scene_seed, uint64_t seed,
                      int32_t buffer_capacity, int64_t max_cycles, amppi_loop** out) {
  using namespace amppi_dev;
  if (!ctx || !out) return AMPPI_INVALID_ARGUMENT;
  if (buffer_capacity < 1 || max_cycles < 1) return ctx->fail(AMPPI_INVALID_ARGUMENT, "bad loop size");
  std::vector<LoopPrim> prims;
  try {
    prims = loop_scenario(scene_kind, scene_seed);
  } catch (const std::exception& e) {
    return ctx->fail(AMPPI_INVALID_ARGUMENT, e.what());
  }
  if (prims.size() > 1024) return ctx->fail(AMPPI_INVALID_ARGUMENT, "more than 1024 obstacles");
  const int64_t cloud_cap = static_cast<int64_t>(buffer_capacity) * kLidarRays;
  if (int rc = alloc_points(ctx, cloud_cap); rc != AMPPI_OK) return rc;
  const int N = ctx->dc.N;
  auto* lp = new (std::nothrow) amppi_loop();
  if (!lp) return ctx->fail(AMPPI_CUDA_ERROR, "out of host memory");
  lp->ctx = ctx;
  lp->max_cycles = max_cycles;
  // one device block: prims | state | frames | frame_n | cloud | offsets | goal | nominal | hover | cycles | seeds | records
  auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
  const size_t sizes[] = {std::max<size_t>(prims.size(), 1) * sizeof(LoopPrim), sizeof(LoopState),
                          static_cast<size_t>(cloud_cap) * 3 * sizeof(double), buffer_capacity * sizeof(int32_t),
                          static_cast<size_t>(cloud_cap) * 3 * sizeof(double), 2 * sizeof(int64_t),
                          10 * sizeof(double), static_cast<size_t>(N) * 4 * sizeof(double), 4 * sizeof(double),
                          sizeof(uint64_t), sizeof(uint64_t), static_cast<size_t>(max_cycles) * sizeof(LoopRecord)};
  size_t total = 0;
  for (size_t s : sizes) total += align(s);
  if (cudaMalloc(&lp->mem, total) != cudaSuccess) {
    delete lp;
    return ctx->fail(AMPPI_CUDA_ERROR, "loop allocation");
  }
  unsigned char* cur = static_cast<unsigned char*>(lp->mem);
  auto take = [&](size_t s) {
    void* p = cur;
    cur += align(s);
    return p;
  };
  LoopDev& L = lp->L;
  L.prims = static_cast<const LoopPrim*>(take(sizes[0]));
  L.st = static_cast<LoopState*>(take(sizes[1]));
  L.frames = static_cast<double*>(take(sizes[2]));
  L.frame_n = static_cast<int32_t*>(take(sizes[3]));
  L.cloud = static_cast<double*>(take(sizes[4]));
  L.offsets = static_cast<int64_t*>(take(sizes[5]));
  L.goal = static_cast<double*>(take(sizes[6]));
  L.nominal = static_cast<double*>(take(sizes[7]));
  L.hover = static_cast<double*>(take(sizes[8]));
  L.cycles = static_cast<uint64_t*>(take(sizes[9]));
  L.seeds = static_cast<uint64_t*>(take(sizes[10]));
  L.records = static_cast<LoopRecord*>(take(sizes[11]));
  L.max_records = max_cycles;
  // initial episode (make_episode_state, ensemble.cpp:238-243): start (0, 0, 2) at rest,
  // last applied = hover, goal = GoalSpec::facing(start, goal (45, 0, 2))
  const amppi_config& c = ctx->cfg;
  const double g = std::sqrt((c.gravity[0] * c.gravity[0] + c.gravity[1] * c.gravity[1]) + c.gravity[2] * c.gravity[2]);
  const double hover[4] = {c.mass * g, 0.0, 0.0, 0.0};
  LoopState st{};
  st.x[0] = 0.0; st.x[1] = 0.0; st.x[2] = 2.0;
  st.x[3] = 1.0;
  for (int k = 0; k < 4; ++k) st.last[k] = hover[k];
  st.ring_head = buffer_capacity - 1;
  const double sx = 0.0, sy = 0.0, gxp = 45.0, gyp = 0.0;
  const double yaw = std::atan2(gyp - sy, gxp - sx), hy = 0.5 * yaw;
  const double goal[10] = {45.0, 0.0, 2.0, 0.0, 0.0, 0.0, std::cos(hy), 0.0, 0.0, std::sin(hy)};
  CK(cudaMemcpy(const_cast<LoopPrim*>(L.prims), prims.data(), prims.size() * sizeof(LoopPrim), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(L.st, &st, sizeof(st), cudaMemcpyHostToDevice));
  CK(cudaMemset(L.frame_n, 0, sizes[3]));
  CK(cudaMemcpy(L.goal, goal, sizeof(goal), cudaMemcpyHostToDevice));
  CK(cudaMemset(L.nominal, 0, sizes[7]));
  CK(cudaMemcpy(L.hover, hover, sizeof(hover), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(L.seeds, &seed, sizeof(seed), cudaMemcpyHostToDevice));
  LoopParams& prm = lp->prm;
  prm.n_prims = static_cast<int>(prims.size());
  prm.capacity = buffer_capacity;
  prm.seed = seed;
  prm.r_max = c.r_max;
  prm.el_min = -45.0 * std::numbers::pi / 180.0;
  prm.el_max = 45.0 * std::numbers::pi / 180.0;
  prm.range_sigma = 0.01;
  prm.goal_radius = 1.0;
  prm.timeout = 60.0;
  prm.drone_radius = 0.2;
  prm.max_failures = 50;
  prm.step_dt = 1.0 / c.replan_hz;
  *out = lp;
  return AMPPI_OK;
}

int amppi_loop_run(amppi_loop* lp, int64_t cycles, int64_t* ran) {
  NvtxRange nvtx_range("amppi_loop_run");
  using namespace amppi_dev;
  if (!lp) return AMPPI_INVALID_ARGUMENT;
  amppi_ctx* ctx = lp->ctx;
  const LoopDev& L = lp->L;
  uint64_t c0 = 0;
  CK(cudaMemcpyAsync(&c0, &L.st->cycle, sizeof(c0), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int64_t room = lp->max_cycles - static_cast<int64_t>(c0);
  if (cycles > room) cycles = std::max<int64_t>(room, 0);
  BatchIn in{};
  in.xyz = nullptr;
  in.xyz64 = L.cloud;
  in.offsets = L.offsets;
  in.poses = L.st->x;
  in.states = L.st->x;
  in.goals = L.goal;
  in.prev = L.nominal;
  in.prev_len = &L.st->prev_len;
  in.last_applied = L.st->last;
  in.cycles = L.cycles;
  in.seeds = L.seeds;
  in.injected = nullptr;
  in.S = 1;
  in.r_max = ctx->cfg.r_max;
  const int64_t max_pts = static_cast<int64_t>(lp->prm.capacity) * kLidarRays;
  auto one_cycle = [&]() -> int {
    cudaError_t e = launch_loop_scan(L, lp->prm, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "launch_loop_scan");
    if (int rc = run_cycle(ctx, in, max_pts, true, true, false); rc != AMPPI_OK) return rc;
    e = launch_loop_step(L, lp->prm, ctx->pl, ctx->dc, ctx->stream);
    return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "launch_loop_step");
  };
  // Every cycle launches the same kernels on device-resident state, so one
  // captured cycle is replayed as a CUDA graph (no per-kernel launch cost);
  // with per-kernel profiling on, the cycles are launched individually.
  const bool graph = !ctx->timer.enabled && ctx->opt.schedule.loop_graph >= 0;
  ctx->have_snapshot = false;  // the loop overwrites the single-scene perception slot
  // the captured cycle refers to the context's point buffers: capture again
  // after they were reallocated (a larger snapshot or batch in between)
  if (lp->cycle_graph && lp->graph_points_gen != ctx->points_gen) {
    cudaGraphExecDestroy(lp->cycle_graph);
    lp->cycle_graph = nullptr;
  }
  if (graph && !lp->cycle_graph && cycles > 0) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = one_cycle();
    const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
    if (rc != AMPPI_OK) return rc;
    if (ce != cudaSuccess) return ctx->cuda_fail(ce, "graph capture");
    const cudaError_t ie = cudaGraphInstantiate(&lp->cycle_graph, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return ctx->cuda_fail(ie, "graph instantiate");
    lp->graph_points_gen = ctx->points_gen;
  }
  for (int64_t i = 0; i < cycles; ++i) {
    if (graph) {
      CK(cudaGraphLaunch(lp->cycle_graph, ctx->stream));
    } else if (int rc = one_cycle(); rc != AMPPI_OK) {
      return rc;
    }
  }
  uint64_t c1 = 0;
  CK(cudaMemcpyAsync(&c1, &L.st->cycle, sizeof(c1), cudaMemcpyDeviceToHost, ctx->stream));
  if (int rc = sync_and_collect(ctx); rc != AMPPI_OK) return rc;
  if (ran) *ran = static_cast<int64_t>(c1 - c0);
  return AMPPI_OK;
}

int amppi_loop_records(amppi_loop* lp, amppi_loop_record* out, int64_t cap, int64_t* count) {
  if (!lp) return AMPPI_INVALID_ARGUMENT;
  amppi_ctx* ctx = lp->ctx;
  uint64_t c = 0;
  CK(cudaMemcpy(&c, &lp->L.st->cycle, sizeof(c), cudaMemcpyDeviceToHost));
  const int64_t n = std::min<int64_t>(static_cast<int64_t>(c), lp->max_cycles);
  if (count) *count = n;
  if (out && cap > 0)
    CK(cudaMemcpy(out, lp->L.records, static_cast<size_t>(std::min(n, cap)) * sizeof(amppi_loop_record),
                  cudaMemcpyDeviceToHost));
  return AMPPI_OK;
}

int amppi_loop_state(amppi_loop* lp, double* x10, int32_t* status, double* t) {
  if (!lp) return AMPPI_INVALID_ARGUMENT;
  amppi_ctx* ctx = lp->ctx;
  amppi_dev::LoopState st{};
  CK(cudaMemcpy(&st, lp->L.st, sizeof(st), cudaMemcpyDeviceToHost));
  if (x10) std::memcpy(x10, st.x, sizeof(st.x));
  if (status) *status = st.status;
  if (t) *t = st.t;
  return AMPPI_OK;
}

int amppi_loop_metrics(amppi_loop* lp, amppi_episode_metrics* out) {
  if (!lp || !out) return AMPPI_INVALID_ARGUMENT;
  amppi_ctx* ctx = lp->ctx;
  uint64_t c = 0;
  CK(cudaMemcpy(&c, &lp->L.st->cycle, sizeof(c), cudaMemcpyDeviceToHost));
  const int64_t n = std::min<int64_t>(static_cast<int64_t>(c), lp->max_cycles);
  if (n < 4) return ctx->fail(AMPPI_INVALID_ARGUMENT, "log too short for jerk estimation");
  void* d = nullptr;
  CK(cudaMalloc(&d, sizeof(amppi_dev::LoopMetrics)));
  cudaError_t e = amppi_dev::launch_loop_metrics(lp->L, n, static_cast<amppi_dev::LoopMetrics*>(d), ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(*out), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  return e == cudaSuccess ? AMPPI_OK : ctx->cuda_fail(e, "loop metrics");
}

int amppi_loop_destroy(amppi_loop* lp) {
  if (!lp) return AMPPI_OK;
  cudaStreamSynchronize(lp->ctx->stream);
  if (lp->cycle_graph) cudaGraphExecDestroy(lp->cycle_graph);
  cudaFree(lp->mem);
  delete lp;
  return AMPPI_OK;
}

}  // extern "C"
