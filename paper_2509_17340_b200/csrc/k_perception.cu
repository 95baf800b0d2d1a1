// Snapshot kernels: LiDAR ingest + 3°/18° multi-resolution partition +
// filtered cloud + collision grid.  Replaces build_snapshot
// (proj/src/perception.cpp:237-246) and everything under it.
//
// Built with -fmad=false: every FP64 value that feeds an integer decision
// (cell keys, per-cell argmin, pooled argmax) is computed with the oracle's
// operation order and IEEE rounding, so keys and ranges are bit-exact.
//
// Cell keys: FP32 atan2 decides unless its quotient lies within 1e-3 cells of
// a boundary (FP32 error < 3e-5 cells); then FP64 atan2 decides unless within
// 1e-9 cells (CUDA's FP64 error < 1e-13 cells); then the correctly rounded
// atan2 (cr_math.cuh) decides, matching glibc's floor() result.
//
// Two schedules:
//   scenes of <= kFusedMaxPoints points: k_snapshot_scene, one CTA per scene,
//     per-cell (range, index) minimum with shared-memory atomics (pass A:
//     64-bit atomicMin of the range bits, pass B: points at the minimum take
//     atomicMin of their index = "strict <, first point wins",
//     perception.cpp:80-86), then the finalize body below;
//   larger scenes: k_key_points (global 64-bit atomicMin + candidate log over
//     many CTAs), k_resolve_ties, k_finalize_scene.
// Finalize body (per scene): ranges / has_point, 6x6 argmax pooling, flat-order
// compaction + world transform, collision grid (bitonic sort by (cell, Morton
// code), 16-point leaves with float boxes, cell records, padded neighbour
// masks, FP32 point blocks for the packed query).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "cr_math.cuh"
#include "device_math.cuh"
#include "kernels.h"

namespace amppi_dev {

namespace {

#ifdef AMPPI_STATS
// Per-phase cycle counts of the per-scene snapshot CTA (stats builds only):
// thread 0 adds the clock delta since the previous mark to slot 16 + i.
#define SNAP_PHASE(i)                                                                            \
  do {                                                                                           \
    if (threadIdx.x == 0) {                                                                      \
      const long long now = clock64();                                                           \
      atomicAdd(&g_query_stats[16 + (i)], static_cast<unsigned long long>(now - phase_t));       \
      phase_t = now;                                                                             \
    }                                                                                            \
  } while (0)
#define SNAP_PHASE_INIT long long phase_t = clock64()
#else
#define SNAP_PHASE(i) ((void)0)
#define SNAP_PHASE_INIT ((void)0)
#endif

constexpr double kPiD = 0x1.921fb54442d18p+1;      // std::numbers::pi
constexpr double kHalfPi = 0x1.921fb54442d18p+0;   // 0.5 * pi
constexpr double kAzStep = 0x1.acee9f37bebd5p-5;   // 2*pi/120 == pi/60
constexpr double kElStep = 0x1.acee9f37bebd5p-5;
constexpr double kGuard = 1e-9;   // cells, FP64 stage
constexpr float kGuardF = 1e-3f;  // cells, FP32 stage

// Correctly-rounded recomputation, kept out of line: taken only for keys
// within 1e-9 of a cell boundary.
__device__ __noinline__ double atan2_slow(double y, double x) { return crm::atan2_cr(y, x); }

__device__ __forceinline__ bool near_integer(double v) {
  const double fl = floor(v);
  return (v - fl) < kGuard || ((fl + 1.0) - v) < kGuard;
}

// FP32 atan2 for the keying fast path: odd degree-11 polynomial for atan on
// [0, 1] (max error 1.8e-6 rad, measured over 2e7 float arguments), one
// approximate division (2 ulp) and the octant fold.  Total error < 3e-6 rad
// = 6e-5 cells, well inside the 1e-3-cell guard band that sends a point to
// the FP64 / correctly rounded stages.  (0, 0) returns NaN, which fast_cell
// also sends there.
__device__ __forceinline__ float fast_atan2f(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float a = __fdividef(fminf(ax, ay), fmaxf(ax, ay));
  const float s = a * a;
  float r = -0.01172120f;
  r = r * s + 0.05265332f;
  r = r * s - 0.11643287f;
  r = r * s + 0.19354346f;
  r = r * s - 0.33262347f;
  r = r * s + 0.99997726f;
  r = r * a;
  if (ay > ax) r = 1.57079632679f - r;
  if (x < 0.f) r = 3.14159265359f - r;
  return y < 0.f ? -r : r;
}

// FP32 quotient -> cell index, or -1 when within the guard band.
__device__ __forceinline__ int fast_cell(float num, float den, float offset, float inv_step) {
  const float v = (fast_atan2f(num, den) + offset) * inv_step;
  const float fl = floorf(v);
  if (!(v - fl >= kGuardF) || !((fl + 1.f) - v >= kGuardF)) return -1;  // (NaN too)
  return static_cast<int>(fl);
}

// azimuth_cell(atan2(y, x)) (perception.cpp:17-21), FP64 stages.
__device__ __noinline__ int az_cell_slow(double y, double x) {
  double az = atan2(y, x);
  double v = (az + kPiD) / kAzStep;
  if (near_integer(v)) {
    az = atan2_slow(y, x);
    v = (az + kPiD) / kAzStep;
  }
  return static_cast<int>(floor(v));
}

// elevation_cell(atan2(z, rho)) (perception.cpp:23-26), FP64 stages.
__device__ __noinline__ int el_cell_slow(double z, double rho) {
  double el = atan2(z, rho);
  double v = (el + kHalfPi) / kElStep;
  if (near_integer(v)) {
    el = atan2_slow(z, rho);
    v = (el + kHalfPi) / kElStep;
  }
  return static_cast<int>(floor(v));
}

// Flat cell f = i*60 + j of a body-frame point.
// The FP32 stage takes rho in FP32 (relative error ~3e-7: < 1e-5 cells, inside
// the same guard band); the exact FP64 rho is formed only for the FP64 stages.
__device__ __forceinline__ int cell_key(V3<double> p) {
  constexpr float kInvStepF = static_cast<float>(1.0 / 0x1.acee9f37bebd5p-5);
  const float xf = static_cast<float>(p.x), yf = static_cast<float>(p.y);
  int i = fast_cell(yf, xf, 3.14159265358979f, kInvStepF);
  if (i < 0) i = az_cell_slow(p.y, p.x);
  if (i >= kAz) i -= kAz;  // +pi wraps onto -pi
  i = i < 0 ? 0 : (i > kAz - 1 ? kAz - 1 : i);
  int j = fast_cell(static_cast<float>(p.z), sqrtf(xf * xf + yf * yf), 1.57079632679490f, kInvStepF);
  if (j < 0) j = el_cell_slow(p.z, sqrt(p.x * p.x + p.y * p.y));
  j = j < 0 ? 0 : (j > kEl - 1 ? kEl - 1 : j);  // pole belongs to the top cell
  return i * kEl + j;
}

struct PoseFrame {
  V3<double> p;
  M3 r;  // body -> world
};

__device__ __forceinline__ PoseFrame load_pose(const double* s10) {
  PoseFrame f;
  f.p = {s10[0], s10[1], s10[2]};
  f.r = rotmat(Q4<double>{s10[3], s10[4], s10[5], s10[6]});
  return f;
}

__device__ __forceinline__ V3<double> load_point(const BatchIn& in, int64_t g) {
  if (in.xyz64) return {in.xyz64[3 * g], in.xyz64[3 * g + 1], in.xyz64[3 * g + 2]};
  return {static_cast<double>(in.xyz[3 * g]), static_cast<double>(in.xyz[3 * g + 1]),
          static_cast<double>(in.xyz[3 * g + 2])};
}

// PointCloudBuffer::body_points: R^T (p - pose.p) (perception.cpp:58-61).
__device__ __forceinline__ V3<double> to_body(const PoseFrame& f, V3<double> w) {
  return mat_t_vec(f.r, w - f.p);
}

// build_partition's per-point work (perception.cpp:72-79): false when the
// point is outside (kMinPointRange, r_max].
__device__ __forceinline__ bool key_point(const PoseFrame& pose, V3<double> w, double r_max, int& f, uint64_t& bits) {
  const V3<double> p = to_body(pose, w);
  const double r = sqrt(sqnorm(p));
  if (!(r > kMinPointRange) || r > r_max) return false;
  f = cell_key(p);
  bits = static_cast<uint64_t>(__double_as_longlong(r));
  return true;
}

// key_point without the FP64 / correctly rounded fallbacks: 0 = out of range,
// 1 = keyed, 2 = inside a guard band (the caller defers it to key_point, so
// a warp does not idle behind the one lane on the slow path)
__device__ __forceinline__ int key_point_fast(const PoseFrame& pose, V3<double> w, double r_max, int& f,
                                              uint64_t& bits) {
  const V3<double> p = to_body(pose, w);
  const double r = sqrt(sqnorm(p));
  if (!(r > kMinPointRange) || r > r_max) return 0;
  constexpr float kInvStepF = static_cast<float>(1.0 / 0x1.acee9f37bebd5p-5);
  const float xf = static_cast<float>(p.x), yf = static_cast<float>(p.y);
  int i = fast_cell(yf, xf, 3.14159265358979f, kInvStepF);
  const int j = fast_cell(static_cast<float>(p.z), sqrtf(xf * xf + yf * yf), 1.57079632679490f, kInvStepF);
  if (i < 0 || j < 0) return 2;
  if (i >= kAz) i -= kAz;  // as cell_key
  i = i > kAz - 1 ? kAz - 1 : i;
  f = i * kEl + (j > kEl - 1 ? kEl - 1 : j);
  bits = static_cast<uint64_t>(__double_as_longlong(r));
  return 1;
}

// ---------------------------------------------------------------------------
// global schedule (large scenes)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_key_points(BatchIn in, Perception P) {
  const int s = blockIdx.y;
  __shared__ PoseFrame pose;
  if (threadIdx.x == 0) pose = load_pose(in.poses + 10 * s);
  __syncthreads();
  const int64_t b = in.offsets[s], e = in.offsets[s + 1];
  uint64_t* __restrict__ cell_r = P.cell_r + static_cast<int64_t>(s) * kCells;
  for (int64_t g = b + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < e;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int f;
    uint64_t bits;
    if (!key_point(pose, load_point(in, g), in.r_max, f, bits)) continue;
    const uint64_t old = atomicMin(reinterpret_cast<unsigned long long*>(cell_r + f), bits);
    if (old >= bits) {  // may be the cell minimum: log for the index tie-break
      const unsigned long long slot = atomicAdd(P.cand_count, 1ull);
      if (slot < static_cast<unsigned long long>(P.cand_cap))
        P.cand[slot] = Candidate{static_cast<uint32_t>(s * kCells + f), static_cast<uint32_t>(g - b), bits};
      else
        atomicOr(P.flags, kFlagCandOverflow);  // a lost candidate could drop a cell's point
    }
  }
}

// The same keying with the per-cell minimum first reduced inside a thread-block
// cluster: every CTA keeps the scene's whole 7200-cell table in shared memory
// (shared-memory 64-bit atomicMin per point, on chip), and after a cluster
// barrier CTA r of the cluster reduces cells [900 r, 900 r + 900) over the 8
// tables through distributed shared memory (remote loads) and merges the
// non-empty ones into the global table.  A scene of P points then costs P
// on-chip atomics and 7200 global ones per cluster instead of P contended
// global atomics.  (A 64-bit atomicMin on a remote CTA's shared memory is not
// a native operation on sm_100a: the compiler's fallback applies it to the
// issuing CTA's own table -- measured, lost updates -- hence local tables and
// remote loads.)  Candidates for the index tie-break are logged as in
// k_key_points: a point that was not <= its CTA's running minimum cannot be
// the global minimum.
__device__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total);

#ifndef AMPPI_KEY_PPT
#define AMPPI_KEY_PPT 8  // cluster keying: target points per thread (sets the clusters per scene)
#endif
constexpr int kKeyCluster = 8;
constexpr int kKeyCellsPerRank = kCells / kKeyCluster;  // 900
constexpr int kKeyThreads = 512;
static_assert(kCells % kKeyCluster == 0, "cells split evenly over the cluster");

__global__ void __cluster_dims__(kKeyCluster, 1, 1) __launch_bounds__(kKeyThreads)
    k_key_points_cluster(BatchIn in, Perception P, int clusters_per_scene) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char key_smem[];
  unsigned long long* tab = reinterpret_cast<unsigned long long*>(key_smem);  // [kCells]
  __shared__ PoseFrame pose;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int s = blockIdx.y;
  for (int c = threadIdx.x; c < kCells; c += blockDim.x) tab[c] = kEmptyCell;
  if (threadIdx.x == 0) pose = load_pose(in.poses + 10 * s);
  __syncthreads();
  const int64_t b = in.offsets[s], e = in.offsets[s + 1];
  const int64_t stride = static_cast<int64_t>(clusters_per_scene) * kKeyCluster * blockDim.x;
  // block-uniform loop: each iteration's candidates get their log slots from
  // one atomicAdd per CTA (a block scan), not one per warp
  __shared__ uint32_t warp_sums[kKeyThreads / 32];
  __shared__ uint32_t n_iter;
  __shared__ unsigned long long log_base;
  for (int64_t g0 = b + static_cast<int64_t>(blockIdx.x) * blockDim.x; g0 < e; g0 += stride) {
    const int64_t g = g0 + threadIdx.x;
    int f = 0;
    uint64_t bits = 0;
    bool cand = false;
    if (g < e && key_point(pose, load_point(in, g), in.r_max, f, bits))
      cand = atomicMin(tab + f, bits) >= bits;  // may be the cell minimum: log for the index tie-break
    const uint32_t pos = block_exclusive_scan(cand ? 1u : 0u, warp_sums, &n_iter);
    if (threadIdx.x == 0) log_base = n_iter ? atomicAdd(P.cand_count, static_cast<unsigned long long>(n_iter)) : 0ull;
    __syncthreads();
    if (cand) {
      const unsigned long long slot = log_base + pos;
      if (slot < static_cast<unsigned long long>(P.cand_cap))
        P.cand[slot] = Candidate{static_cast<uint32_t>(s * kCells + f), static_cast<uint32_t>(g - b), bits};
      else
        atomicOr(P.flags, kFlagCandOverflow);  // a lost candidate could drop a cell's point
    }
    __syncthreads();  // log_base / n_iter are rewritten next iteration
  }
  cl.sync();  // every table of the cluster is final
  uint64_t* __restrict__ cell_r = P.cell_r + static_cast<int64_t>(s) * kCells;
  for (int c = rank * kKeyCellsPerRank + threadIdx.x; c < static_cast<int>(rank + 1) * kKeyCellsPerRank;
       c += blockDim.x) {
    unsigned long long m = tab[c];
#pragma unroll
    for (int q = 1; q < kKeyCluster; ++q) {
      const unsigned long long v = cl.map_shared_rank(tab, (rank + q) % kKeyCluster)[c];
      m = v < m ? v : m;
    }
    if (m != kEmptyCell) atomicMin(reinterpret_cast<unsigned long long*>(cell_r + c), m);
  }
  cl.sync();  // no CTA leaves while the others read its table
}

__global__ void __launch_bounds__(256) k_resolve_ties(Perception P) {
  const unsigned long long n = min(*P.cand_count, static_cast<unsigned long long>(P.cand_cap));
  for (unsigned long long c = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
       c += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const Candidate cd = P.cand[c];
    if (P.cell_r[cd.cell] == cd.bits) atomicMin(P.cell_idx + cd.cell, cd.idx);
  }
}

// ---------------------------------------------------------------------------
// finalize body
// ---------------------------------------------------------------------------
#ifndef AMPPI_SNAP_THREADS
#define AMPPI_SNAP_THREADS 512
#endif
constexpr int kFinalizeThreads = AMPPI_SNAP_THREADS;  // fused per-scene CTAs (two per SM)
constexpr int kFinalizeThreadsFew = 1024;  // k_finalize_scene for a handful of scenes (latency)
constexpr int kMaxWarps = kFinalizeThreadsFew / 32;
constexpr uint32_t kCellsPow2 = 8192;  // sort capacity >= kCells
#ifndef AMPPI_SORT_REGS
#define AMPPI_SORT_REGS 1  // grid-build sort: in-window stages in registers (0: every stage in shared memory)
#endif
#ifndef AMPPI_POOL_STRIDED
#define AMPPI_POOL_STRIDED 1  // filtered compaction: one thread per filtered slot (0: per-thread cell chunks)
#endif
#ifndef AMPPI_KEY_DEFER
#define AMPPI_KEY_DEFER 512  // fused pass A: guard-band points deferred per scene (then keyed by full warps)
#endif
#ifndef AMPPI_LOG_BITS
#define AMPPI_LOG_BITS 1  // fused pass A logs (cell, index, range bits); 0: (cell, index), pass B re-keys
#endif
#ifndef AMPPI_LEAF_SCAN
#define AMPPI_LEAF_SCAN 0  // 1: each cell's first thread walks the cell to flag its leaf starts (r01)
#endif
#ifndef AMPPI_LOCAL_FRAME
#define AMPPI_LOCAL_FRAME 1  // FP32 grid data and screening relative to the snapshot pose (0: world frame)
#endif

// The rng..idx region (86 KB) is reused phase by phase: keying's u64 range
// bits (rng) and argmin indices (idx); pooling's ranges; the compaction map
// (comp_k / comp_f in rng); the grid build's byte layout from rng:
// keys u32[8192] @0, vals u16[8192] @32K (then the cells' first leaves),
// leaf flags u8[8192] @48K, cell-start bitmap u32[256] @56K, and the leaf
// start table u32[] in idx.
constexpr uint32_t kKeyDeferCap = AMPPI_KEY_DEFER;  // (0 keeps the slow path inline)

struct FinalizeSmem {
  double rng[kCells];
  uint32_t idx[kCells + 1];
  uint32_t rows[kGridAxis * kGridAxis];  // non-empty grid cells: bit z of row (x, y)
  uint32_t warp_sums[kMaxWarps];
  double bbox_lo[kMaxWarps][3];
  double bbox_hi[kMaxWarps][3];
  GridMeta meta;
  PoseFrame pose;
  uint32_t total;
  uint32_t n_cand;
  uint32_t n_defer;
  uint32_t defer[kKeyDeferCap];  // fused pass A: points whose fast key hit a guard band
};

// Block-wide exclusive scan of one value per thread; returns the prefix and
// writes the total to *total (all threads see it after the call).
__device__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t w = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive
    if (lane == nw - 1) *total = w;
  }
  __syncthreads();
  const uint32_t base = warp > 0 ? warp_sums[warp - 1] : 0u;
  const uint32_t out = base + x - v;
  __syncthreads();
  return out;
}

// Everything after the per-cell (range, index) minimum.  Expects sm.rng /
// sm.idx (empty cells: r_max / 0xFFFFFFFF) and sm.pose filled and a
// preceding __syncthreads().
__device__ void finalize_body(FinalizeSmem& sm, const BatchIn& in, const Perception& P, const DevConfig& cfg,
                              int s) {
  SNAP_PHASE_INIT;
  const int tid = threadIdx.x;
  const int64_t cell_base = static_cast<int64_t>(s) * kCells;
  const int64_t pt_base = in.offsets[s];
  for (int w = tid; w < kGridAxis * kGridAxis; w += blockDim.x) sm.rows[w] = 0u;
  if (P.ranges)
    for (int f = tid; f < kCells; f += blockDim.x) {
      P.ranges[cell_base + f] = sm.rng[f];
      P.has_point[cell_base + f] = sm.idx[f] != 0xFFFFFFFFu ? 1 : 0;
    }

  // pool_coarse: 6x6 argmax, i outer / j inner, strict > (perception.cpp:99-121)
  if (tid < kCoarse) {
    const int I = tid / kCEl, J = tid % kCEl;
    int bi = I * kPool, bj = J * kPool;
    double best = -1.0;
    for (int i = I * kPool; i < (I + 1) * kPool; ++i)
      for (int j = J * kPool; j < (J + 1) * kPool; ++j) {
        const double r = sm.rng[i * kEl + j];
        if (r > best) {
          best = r;
          bi = i;
          bj = j;
        }
      }
    const int c = bi * kEl + bj;
    const double dx = P.cell_dir[3 * c], dy = P.cell_dir[3 * c + 1], dz = P.cell_dir[3 * c + 2];
    const int64_t o = static_cast<int64_t>(s) * kCoarse + tid;
    P.safe_range[o] = best;
    P.safe_dir[3 * o] = dx;
    P.safe_dir[3 * o + 1] = dy;
    P.safe_dir[3 * o + 2] = dz;
    P.safe_point[3 * o] = best * dx;
    P.safe_point[3 * o + 1] = best * dy;
    P.safe_point[3 * o + 2] = best * dz;
  }

  // filtered_cloud + to_world_frame in flat order (perception.cpp:124-144)
  const int chunk = (kCells + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
  const int f0 = tid * chunk;
  const int f1 = min(f0 + chunk, kCells);
  uint32_t mine = 0;
  for (int f = f0; f < f1; ++f) mine += sm.idx[f] != 0xFFFFFFFFu;
  const uint32_t pos0 = block_exclusive_scan(mine, sm.warp_sums, &sm.total);
  const uint32_t n_pts = sm.total;
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  double* __restrict__ filt = P.filtered + cell_base * 3;
#if AMPPI_POOL_STRIDED
  // Compaction map first (filtered slot -> point index and cell, in the dead
  // range table once pool_coarse has read it), then one thread per filtered
  // slot: the point gathers are independent across a warp and the filtered
  // records are written coalesced.
  {
    uint32_t* comp_k = reinterpret_cast<uint32_t*>(sm.rng);           // [<= 7200]
    uint16_t* comp_f = reinterpret_cast<uint16_t*>(comp_k + kCells);  // [<= 7200]
    __syncthreads();  // pool_coarse has read sm.rng
    uint32_t pos = pos0;
    for (int f = f0; f < f1; ++f) {
      const uint32_t k = sm.idx[f];
      if (k == 0xFFFFFFFFu) continue;
      comp_k[pos] = k;
      comp_f[pos] = static_cast<uint16_t>(f);
      ++pos;
    }
    __syncthreads();
    if (P.nearest)
      for (int f = tid; f < kCells; f += blockDim.x)
        if (sm.idx[f] == 0xFFFFFFFFu) {
          P.nearest[(cell_base + f) * 3] = 0.0;
          P.nearest[(cell_base + f) * 3 + 1] = 0.0;
          P.nearest[(cell_base + f) * 3 + 2] = 0.0;
        }
#pragma unroll 4
    for (uint32_t q = tid; q < n_pts; q += blockDim.x) {
      const uint32_t k = comp_k[q];
      const V3<double> pb = to_body(sm.pose, load_point(in, pt_base + k));
      const V3<double> pw = sm.pose.p + mat_vec(sm.pose.r, pb);
      if (P.nearest) {
        const int f = comp_f[q];
        P.nearest[(cell_base + f) * 3] = pb.x;
        P.nearest[(cell_base + f) * 3 + 1] = pb.y;
        P.nearest[(cell_base + f) * 3 + 2] = pb.z;
      }
      filt[3 * q] = pw.x;
      filt[3 * q + 1] = pw.y;
      filt[3 * q + 2] = pw.z;
      lo[0] = fmin(lo[0], pw.x); lo[1] = fmin(lo[1], pw.y); lo[2] = fmin(lo[2], pw.z);
      hi[0] = fmax(hi[0], pw.x); hi[1] = fmax(hi[1], pw.y); hi[2] = fmax(hi[2], pw.z);
    }
  }
#else
  uint32_t pos = pos0;
#pragma unroll 5
  for (int f = f0; f < f1; ++f) {
    const uint32_t k = sm.idx[f];
    if (k == 0xFFFFFFFFu) {
      if (P.nearest) {
        P.nearest[(cell_base + f) * 3] = 0.0;
        P.nearest[(cell_base + f) * 3 + 1] = 0.0;
        P.nearest[(cell_base + f) * 3 + 2] = 0.0;
      }
      continue;
    }
    const V3<double> pb = to_body(sm.pose, load_point(in, pt_base + k));
    const V3<double> pw = sm.pose.p + mat_vec(sm.pose.r, pb);
    if (P.nearest) {
      P.nearest[(cell_base + f) * 3] = pb.x;
      P.nearest[(cell_base + f) * 3 + 1] = pb.y;
      P.nearest[(cell_base + f) * 3 + 2] = pb.z;
    }
    filt[3 * pos] = pw.x;
    filt[3 * pos + 1] = pw.y;
    filt[3 * pos + 2] = pw.z;
    lo[0] = fmin(lo[0], pw.x); lo[1] = fmin(lo[1], pw.y); lo[2] = fmin(lo[2], pw.z);
    hi[0] = fmax(hi[0], pw.x); hi[1] = fmax(hi[1], pw.y); hi[2] = fmax(hi[2], pw.z);
    ++pos;
  }
#endif
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) {
      sm.bbox_lo[warp][a] = lo[a];
      sm.bbox_hi[warp][a] = hi[a];
    }
  }
  __syncthreads();
  SNAP_PHASE(3);  // pooling + filtered compaction + bbox
  if (tid == 0) {
    GridMeta m{};
    m.n_points = static_cast<int>(n_pts);
#if AMPPI_LOCAL_FRAME
    m.org[0] = sm.pose.p.x;  // the FP32 local frame (to_local_f)
    m.org[1] = sm.pose.p.y;
    m.org[2] = sm.pose.p.z;
#endif
    if (n_pts > 0) {
      double L[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, H[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
        for (int a = 0; a < 3; ++a) {
          L[a] = fmin(L[a], sm.bbox_lo[w][a]);
          H[a] = fmax(H[a], sm.bbox_hi[w][a]);
        }
      const double ext = fmax(fmax(H[0] - L[0], H[1] - L[1]), H[2] - L[2]);
      // cell >= d_max (with margin) so the 27-cell neighbourhood contains every
      // point closer than d_max; at most kGridAxis cells per axis
      double h = cfg.col_d_max * (1.0 + 1e-3) + 1e-6;
      const double h_cap = ext / (kGridAxis - 1) * (1.0 + 1e-9);
      if (h_cap > h) h = h_cap;
      m.h = h;
      m.inv_h = 1.0 / h;
      for (int a = 0; a < 3; ++a) {
        m.origin[a] = L[a];
        m.origin_f[a] = static_cast<float>(L[a] - m.org[a]);
        int d = static_cast<int>(floor((H[a] - L[a]) * m.inv_h)) + 1;
        m.dims[a] = d < 1 ? 1 : (d > kGridAxis ? kGridAxis : d);
      }
      m.inv_h_f = static_cast<float>(m.inv_h);
      m.h_f = static_cast<float>(m.h);
    }
    sm.meta = m;
    P.grid[s] = m;
    P.n_filtered[s] = static_cast<int32_t>(n_pts);
  }
  __syncthreads();
  const GridMeta meta = sm.meta;
  if (n_pts == 0) return;  // dims = 0: every query returns +inf
  SNAP_PHASE(4);  // grid meta

  // collision grid: sort the filtered points by (cell, Morton code of the
  // 1/8-cell sub-position) in shared memory (the per-cell tables are dead by
  // now): each cell's points become contiguous and spatially ordered.
  uint32_t* keys = reinterpret_cast<uint32_t*>(sm.rng);             // [<= 8192]
  uint16_t* vals = reinterpret_cast<uint16_t*>(keys + kCellsPow2);  // [<= 8192]
  auto cell_of = [&](const V3<double>& p, int* c3, int* sub3) {
    const double rel[3] = {p.x - meta.origin[0], p.y - meta.origin[1], p.z - meta.origin[2]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double u = rel[a] * meta.inv_h;
      int c = static_cast<int>(floor(u));
      c = c < 0 ? 0 : (c > meta.dims[a] - 1 ? meta.dims[a] - 1 : c);
      int sc = static_cast<int>(floor((u - c) * 8.0));
      c3[a] = c;
      sub3[a] = sc < 0 ? 0 : (sc > 7 ? 7 : sc);
    }
    return (c3[0] * meta.dims[1] + c3[1]) * meta.dims[2] + c3[2];
  };
  auto key_of = [&](uint32_t k) {
    const V3<double> pw{filt[3 * k], filt[3 * k + 1], filt[3 * k + 2]};
    int c3[3], s3[3];
    const int c = cell_of(pw, c3, s3);
    uint32_t mort = 0;
#pragma unroll
    for (int bit = 2; bit >= 0; --bit)
      mort = (mort << 3) | (((s3[0] >> bit) & 1) << 2) | (((s3[1] >> bit) & 1) << 1) | ((s3[2] >> bit) & 1);
    return (static_cast<uint32_t>(c) << 9) | mort;
  };
  uint32_t n2 = 1;
  while (n2 < n_pts) n2 <<= 1;
  // Bitonic network in its all-ascending form (each merge starts with a
  // flip stage, i against the mirror of i in its block, then half-cleaners;
  // every compare-exchange puts the smaller key at the lower index).  The
  // +inf padding past n_pts is larger than every key, so it only ever moves
  // up and never leaves [n_pts, n2): every pair reaching past n_pts is a
  // no-op and is skipped -- the work follows n_pts, not the padded n2
  // (C5 scenes hold 700-2800 filtered points, padded to 1024-4096).
  for (uint32_t k = tid; k < n_pts; k += blockDim.x) {
    keys[k] = key_of(k);
    vals[k] = static_cast<uint16_t>(k);
  }
  __syncthreads();
  auto cx = [&](uint32_t i, uint32_t j) {
    if (j < n_pts) {
      const uint32_t ki = keys[i], kj = keys[j];
      if (ki > kj) {
        keys[i] = kj;
        keys[j] = ki;
        const uint16_t v = vals[i];
        vals[i] = vals[j];
        vals[j] = v;
      }
    }
  };
#if AMPPI_SORT_REGS
  // Stages that stay inside a 64-key window (every stage of sizes <= 64, and
  // the strides 32..1 that end every larger merge) run in registers: each
  // warp loads a window as two 64-bit (key << 16 | value) words per lane
  // (positions l and l + 32), exchanges them with shuffles and stores once.
  // The comparisons are on the key alone with the shared-memory stages' tie
  // rule (swap only when the lower position holds the larger key).
  {
    const int lane = tid & 31, nw = static_cast<int>(blockDim.x >> 5);
    const uint32_t nwin = (n_pts + 63) / 64;
    auto kof = [](uint64_t x) { return static_cast<uint32_t>(x >> 16); };
    auto ce_lane = [&](uint64_t& x, int partner, bool lower) {
      const uint64_t y = __shfl_sync(0xffffffffu, x, partner);
      if (lower ? kof(x) > kof(y) : kof(y) > kof(x)) x = y;
    };
    auto ce_slot = [&](uint64_t& a, uint64_t& b) {  // positions l (a) and l + 32 (b)
      if (kof(a) > kof(b)) {
        const uint64_t t = a;
        a = b;
        b = t;
      }
    };
    auto halves = [&](uint64_t& a, uint64_t& b, int from) {  // half-cleaners, strides from..1 (<= 16)
      for (int st = from; st > 0; st >>= 1) {
        ce_lane(a, lane ^ st, !(lane & st));
        ce_lane(b, lane ^ st, !(lane & st));
      }
    };
    auto window = [&](bool first) {
      for (uint32_t w = tid >> 5; w < nwin; w += nw) {
        const uint32_t i0 = 64 * w + lane, i1 = i0 + 32;
        uint64_t a = i0 < n_pts ? (static_cast<uint64_t>(keys[i0]) << 16) | vals[i0] : ~0ull;
        uint64_t b = i1 < n_pts ? (static_cast<uint64_t>(keys[i1]) << 16) | vals[i1] : ~0ull;
        if (first) {  // sizes 2..32 in each half, then size 64 across the halves
          for (int size = 2; size <= 32; size <<= 1) {
            ce_lane(a, lane ^ (size - 1), !(lane & (size >> 1)));  // flip
            ce_lane(b, lane ^ (size - 1), !(lane & (size >> 1)));
            halves(a, b, size >> 2);
          }
          const uint64_t am = __shfl_sync(0xffffffffu, a, lane ^ 31), bm = __shfl_sync(0xffffffffu, b, lane ^ 31);
          if (kof(a) > kof(bm)) a = bm;  // flip of 64: l (lower) <-> 63 - l
          if (kof(am) > kof(b)) b = am;
          halves(a, b, 16);
        } else {  // the end of a larger merge: strides 32..1
          ce_slot(a, b);
          halves(a, b, 16);
        }
        if (i0 < n_pts) {
          keys[i0] = kof(a);
          vals[i0] = static_cast<uint16_t>(a & 0xFFFFu);
        }
        if (i1 < n_pts) {
          keys[i1] = kof(b);
          vals[i1] = static_cast<uint16_t>(b & 0xFFFFu);
        }
      }
    };
    window(true);
    __syncthreads();
    for (uint32_t size = 128; size <= n2; size <<= 1) {
      const uint32_t half = size >> 1;
      const uint32_t tf = min(n2 >> 1, (n_pts + size) >> 1);
      for (uint32_t t = tid; t < tf; t += blockDim.x) {  // flip: i <-> mirror in its block
        const uint32_t o = t & (half - 1);
        const uint32_t i = 2 * t - o;
        cx(i, i + size - 1 - 2 * o);
      }
      __syncthreads();
      for (uint32_t stride = half >> 1; stride >= 64; stride >>= 1) {
        const uint32_t th = min(n2 >> 1, (n_pts + stride) >> 1);
        for (uint32_t t = tid; t < th; t += blockDim.x) {
          const uint32_t i = 2 * t - (t & (stride - 1));
          cx(i, i + stride);
        }
        __syncthreads();
      }
      window(false);
      __syncthreads();
    }
  }
#else
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    const uint32_t half = size >> 1;
    const uint32_t tf = min(n2 >> 1, (n_pts + size) >> 1);
    for (uint32_t t = tid; t < tf; t += blockDim.x) {  // flip: i <-> mirror in its block
      const uint32_t o = t & (half - 1);
      const uint32_t i = 2 * t - o;
      cx(i, i + size - 1 - 2 * o);
    }
    if (size > 64) __syncthreads(); else __syncwarp();
    for (uint32_t stride = half >> 1; stride > 0; stride >>= 1) {
      const uint32_t th = min(n2 >> 1, (n_pts + stride) >> 1);
      for (uint32_t t = tid; t < th; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1));
        cx(i, i + stride);
      }
      const uint32_t next = stride > 1 ? stride >> 1 : size;  // the next stage's reach (stride, or flip of 2*size)
      if (stride > 32 || next > 32) __syncthreads(); else __syncwarp();
    }
  }
  __syncthreads();
#endif
  SNAP_PHASE(5);  // sort keys + bitonic sort
  // scatter into sorted order and flag leaf starts: every cell's points form
  // leaves of kLeafSize consecutive (Morton-ordered) points
  double* __restrict__ gp64 = P.grid_pts64 + cell_base * 3;
  float4* __restrict__ gp32 = P.grid_pts32 + cell_base;
  uint4* __restrict__ grec = P.grid_rec + static_cast<int64_t>(s) * kGridCells * 2;
  uint4* __restrict__ gleaf = P.grid_leaf + cell_base * 2;
  uint8_t* lflag = reinterpret_cast<uint8_t*>(vals + kCellsPow2);  // [8192] (inside rng, past keys/vals)
  for (uint32_t i = tid; i < kCellsPow2; i += blockDim.x) lflag[i] = 0;
#if !AMPPI_LEAF_SCAN
  uint32_t* cstart = reinterpret_cast<uint32_t*>(lflag + kCellsPow2);  // [256] bitmap of cell starts (inside rng)
  for (uint32_t i = tid; i < kCellsPow2 / 32; i += blockDim.x) cstart[i] = 0u;
#endif
  // +inf padding of the last FP32 point block
  if (n_pts + tid < (n_pts + kPointBlock - 1) / kPointBlock * kPointBlock) {
    const uint32_t i = n_pts + tid;
    float* blk = reinterpret_cast<float*>(gp32 + 3 * (i / kPointBlock)) + i % kPointBlock;
    blk[0] = blk[kPointBlock] = blk[2 * kPointBlock] = __int_as_float(0x7f800000);
  }
  __syncthreads();
  for (uint32_t i = tid; i < n_pts; i += blockDim.x) {
    const uint32_t k = vals[i];
    const double x = filt[3 * k], y = filt[3 * k + 1], z = filt[3 * k + 2];
    gp64[3 * i] = x;
    gp64[3 * i + 1] = y;
    gp64[3 * i + 2] = z;
    float* blk = reinterpret_cast<float*>(gp32 + 3 * (i / kPointBlock)) + i % kPointBlock;
    blk[0] = static_cast<float>(x - meta.org[0]);
    blk[kPointBlock] = static_cast<float>(y - meta.org[1]);
    blk[2 * kPointBlock] = static_cast<float>(z - meta.org[2]);
    const uint32_t c = keys[i] >> 9;
    if (i == 0 || (keys[i - 1] >> 9) != c) {  // first point of cell c
#if AMPPI_LEAF_SCAN
      uint32_t e = i + 1;
      while (e < n_pts && (keys[e] >> 9) == c) ++e;
      for (uint32_t t = i; t < e; t += kLeafSize) lflag[t] = 1;
#else
      atomicOr(&cstart[i >> 5], 1u << (i & 31));
#endif
      atomicOr(&sm.rows[c / meta.dims[2]], 1u << (c % meta.dims[2]));  // row x*dims[1]+y, bit z
    }
  }
  __syncthreads();
#if !AMPPI_LEAF_SCAN
  // leaf starts: every point finds its cell's first point (the highest cell
  // start at or below it, a few bitmap words back) and starts a leaf at
  // offsets 0, kLeafSize, ... -- all threads in parallel, where a serial walk
  // by each cell's first thread held its warp for the length of a dense cell
  for (uint32_t i = tid; i < n_pts; i += blockDim.x) {
    int w = static_cast<int>(i >> 5);
    uint32_t bits = cstart[w] & (0xFFFFFFFFu >> (31u - (i & 31u)));
    while (bits == 0u) bits = cstart[--w];
    const uint32_t first = (static_cast<uint32_t>(w) << 5) + 31u - __clz(bits);
    lflag[i] = ((i - first) % kLeafSize) == 0u;
  }
  __syncthreads();
#endif
  SNAP_PHASE(6);  // scatter + leaf flags
  // leaf ids = prefix count of leaf starts (contiguous 16-point chunks per thread)
  const uint32_t kPerThread = kCellsPow2 / blockDim.x;  // blockDim.x divides 8192
  const uint32_t i0 = tid * kPerThread;
  // (and the cells' first leaves: leaf starts in the low 16 bits of the
  // scanned count, cell starts in the high 16; both <= 8192)
  auto cell_start = [&](uint32_t i) { return i == 0 || (keys[i - 1] >> 9) != (keys[i] >> 9); };
  uint32_t counts = 0;
  for (uint32_t i = i0; i < i0 + kPerThread; ++i)
    if (lflag[i]) counts += 1u + (i < n_pts && cell_start(i) ? 0x10000u : 0u);
  const uint32_t first = block_exclusive_scan(counts, sm.warp_sums, &sm.total);
  const uint32_t n_leaves = sm.total & 0xFFFFu, n_cells = sm.total >> 16;
  // leaf start table (sm.idx is dead by now): point index, bit 31 = starts a
  // cell; and the cells' first leaves in cell order (u16, in the dead vals)
  uint32_t* lstart = sm.idx;
  uint16_t* cleaf = vals;  // [n_cells + 1]
  {
    uint32_t leaf = first & 0xFFFFu, cell = first >> 16;
    for (uint32_t i = i0; i < i0 + kPerThread && i < n_pts; ++i) {
      if (!lflag[i]) continue;
      const bool cs = cell_start(i);
      if (cs) cleaf[cell++] = static_cast<uint16_t>(leaf);
      lstart[leaf++] = i | (cs ? 0x80000000u : 0u);
    }
    if (tid == 0) {
      lstart[n_leaves] = n_pts | 0x80000000u;  // sentinel
      cleaf[n_cells] = static_cast<uint16_t>(n_leaves);
    }
  }
  __syncthreads();
  // leaf boxes: 16 lanes per leaf (2 leaves per warp, warp-uniform loop),
  // coalesced point loads and a 16-lane min/max reduction
  const int sub = lane & 15;
  const uint32_t wstride = 2 * (blockDim.x >> 5);
  for (uint32_t l0 = 2 * warp; l0 < n_leaves; l0 += wstride) {
    const uint32_t l = l0 + (lane >> 4);
    // each point's local coordinate rounded down / up to float, then a float
    // min / max: rounding is monotone, so this is the outward-rounded box of
    // the FP64 minimum and maximum, in half the shuffles
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    static_assert(kLeafSize <= 16, "one lane per leaf point");
    if (l < n_leaves) {
      const uint32_t t = (lstart[l] & 0x7FFFFFFFu) + sub;
      if (t < (lstart[l + 1] & 0x7FFFFFFFu))
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double v = gp64[3 * t + a] - meta.org[a];  // local frame, as gp32
          lo[a] = __double2float_rd(v);
          hi[a] = __double2float_ru(v);
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
        hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
      }
    if (sub == 0 && l < n_leaves) {
      gleaf[2 * l] = make_uint4(__float_as_uint(lo[0]), __float_as_uint(hi[0]), __float_as_uint(lo[1]),
                                __float_as_uint(hi[1]));
      gleaf[2 * l + 1] = make_uint4(__float_as_uint(lo[2]), __float_as_uint(hi[2]), 0u, 0u);
    }
  }
  __syncthreads();
  SNAP_PHASE(7);  // leaf boxes
  // cell records: 16 lanes per non-empty cell (its leaves run from its first
  // leaf to the next cell's, cleaf); box = union of the leaf boxes
  for (uint32_t c0 = 2 * warp; c0 < n_cells; c0 += wstride) {  // one non-empty cell per 16 lanes
    const uint32_t ci = c0 + (lane >> 4);
    const bool act = ci < n_cells;
    const uint32_t l = act ? cleaf[ci] : 0u, nl = act ? cleaf[ci + 1] - l : 0u;
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (uint32_t k = sub; k < nl; k += 16) {
      const uint4 la = gleaf[2 * (l + k)], lb = gleaf[2 * (l + k) + 1];
      lo[0] = fminf(lo[0], __uint_as_float(la.x)); lo[1] = fminf(lo[1], __uint_as_float(la.z));
      lo[2] = fminf(lo[2], __uint_as_float(lb.x));
      hi[0] = fmaxf(hi[0], __uint_as_float(la.y)); hi[1] = fmaxf(hi[1], __uint_as_float(la.w));
      hi[2] = fmaxf(hi[2], __uint_as_float(lb.y));
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
        hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
      }
    if (sub == 0 && act) {
      const uint32_t i = lstart[l] & 0x7FFFFFFFu, e = lstart[l + nl] & 0x7FFFFFFFu;
      const uint32_t c = keys[i] >> 9;
      grec[2 * c] = make_uint4(i | ((e - i) << 16), l, __float_as_uint(lo[0]), __float_as_uint(hi[0]));
      grec[2 * c + 1] = make_uint4(__float_as_uint(lo[1]), __float_as_uint(hi[1]), __float_as_uint(lo[2]),
                                   __float_as_uint(hi[2]));
    }
  }
  __syncthreads();
  SNAP_PHASE(8);  // cell records
  // neighbour masks over the padded lattice: bit i*9+j*3+k of padded cell
  // (x, y, z) <-> grid cell (x-2+i, y-2+j, z-2+k) is non-empty
  uint32_t* __restrict__ gnbr = P.grid_nbr + static_cast<int64_t>(s) * kPadCells;
  const int p1 = meta.dims[1] + 2, p2 = meta.dims[2] + 2;
  const int npad = (meta.dims[0] + 2) * p1 * p2;
  for (int c = tid; c < npad; c += blockDim.x) {
    const int z = c % p2, y = (c / p2) % p1, x = c / (p2 * p1);
    uint32_t m = 0u;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int ux = x - 2 + i;
      if (ux < 0 || ux >= meta.dims[0]) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int uy = y - 2 + j;
        if (uy < 0 || uy >= meta.dims[1]) continue;
        const uint32_t r = sm.rows[ux * meta.dims[1] + uy] << 2;
        m |= ((r >> z) & 7u) << (i * 9 + j * 3);
      }
    }
    gnbr[c] = m;
  }
#ifdef AMPPI_STATS
  __syncthreads();
  SNAP_PHASE(9);  // neighbour masks
#endif
}

// Global schedule, last step: tables from K1/K1b (reset for the next cycle).
__global__ void __launch_bounds__(kFinalizeThreadsFew, 1) k_finalize_scene(BatchIn in, Perception P, DevConfig cfg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FinalizeSmem& sm = *reinterpret_cast<FinalizeSmem*>(smem_raw);
  const int s = blockIdx.x;
  const int64_t cell_base = static_cast<int64_t>(s) * kCells;
  if (threadIdx.x == 0) sm.pose = load_pose(in.poses + 10 * s);
  for (int f = threadIdx.x; f < kCells; f += blockDim.x) {
    const uint64_t bits = P.cell_r[cell_base + f];
    const bool has = bits != kEmptyCell;
    sm.rng[f] = has ? __longlong_as_double(static_cast<long long>(bits)) : in.r_max;
    sm.idx[f] = has ? P.cell_idx[cell_base + f] : 0xFFFFFFFFu;
    P.cell_r[cell_base + f] = kEmptyCell;
    P.cell_idx[cell_base + f] = 0xFFFFFFFFu;
  }
  __syncthreads();
  finalize_body(sm, in, P, cfg, s);
}

// Fused schedule: one CTA per scene, per-cell minimum in shared memory.
#ifndef AMPPI_SNAP_MINB
#define AMPPI_SNAP_MINB 2
#endif
__global__ void __launch_bounds__(kFinalizeThreads, AMPPI_SNAP_MINB) k_snapshot_scene(BatchIn in, Perception P, DevConfig cfg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FinalizeSmem& sm = *reinterpret_cast<FinalizeSmem*>(smem_raw);
  unsigned long long* cell_bits = reinterpret_cast<unsigned long long*>(sm.rng);
  const int s = blockIdx.x;
  const int tid = threadIdx.x;
  SNAP_PHASE_INIT;
  if (tid == 0) sm.pose = load_pose(in.poses + 10 * s);
  for (int f = tid; f < kCells; f += blockDim.x) {
    cell_bits[f] = kEmptyCell;
    sm.idx[f] = 0xFFFFFFFFu;
  }
  __syncthreads();
  SNAP_PHASE(0);  // table init
  const PoseFrame pose = sm.pose;
  const int64_t b = in.offsets[s], e = in.offsets[s + 1];
  const double r_max = in.r_max;
  // pass A: minimum range bits per cell; a point that was <= the running
  // minimum when it arrived may be the final minimum and is logged (cell,
  // index) for the tie-break -- typically a third of the points
#if AMPPI_LOG_BITS
  // log entries carry the candidate's range bits, so pass B compares instead
  // of re-keying (no second point load, FP64 transform and sqrt)
  Candidate* __restrict__ log = P.cand + b;  // [points of this scene]
  const bool rekey = e - b > 0x10000 || e > P.cand_cap;
#else
  uint32_t* __restrict__ log = reinterpret_cast<uint32_t*>(P.cand) + b;  // [points of this scene]
  const bool rekey = e - b > 0x10000 || e > 4 * P.cand_cap;
#endif
  if (tid == 0) {
    sm.n_cand = 0u;
    sm.n_defer = 0u;
  }
  __syncthreads();
  // the log holds the scene's candidates at [b, e) of the context's candidate
  // buffer; a scene past 2^16 points or past that buffer re-keys in pass B
  const int lane = tid & 31;
  // a warp's new candidates appended to the log (one shared atomic per warp)
  auto log_cand = [&](bool cand, int f, int64_t g, uint64_t bits) {
    const unsigned want = __ballot_sync(0xffffffffu, cand);
    if (want) {
      uint32_t base = 0;
      if (lane == __ffs(want) - 1) base = atomicAdd(&sm.n_cand, static_cast<uint32_t>(__popc(want)));
      base = __shfl_sync(0xffffffffu, base, __ffs(want) - 1);
      if (cand && !rekey) {
#if AMPPI_LOG_BITS
        log[base + __popc(want & ((1u << lane) - 1u))] =
            Candidate{static_cast<uint32_t>(f), static_cast<uint32_t>(g - b), bits};
#else
        log[base + __popc(want & ((1u << lane) - 1u))] = (static_cast<uint32_t>(f) << 16) | static_cast<uint32_t>(g - b);
#endif
      }
    }
  };
  constexpr int kUnroll = 4;  // points per thread per iteration
  // software pipeline: the next iteration's points are loaded before this
  // iteration's keys are computed, so the HBM latency overlaps the keying
  V3<float> nxt[kUnroll];
  auto fetch = [&](int64_t g0n) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t g = g0n + u * blockDim.x + tid;
      nxt[u] = g < e ? V3<float>{in.xyz[3 * g], in.xyz[3 * g + 1], in.xyz[3 * g + 2]} : V3<float>{0.f, 0.f, 0.f};
    }
  };
  if (!in.xyz64) fetch(b);
  for (int64_t g0 = b; g0 < e; g0 += kUnroll * blockDim.x) {
    V3<double> w[kUnroll];
    if (in.xyz64) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t g = g0 + u * blockDim.x + tid;
        w[u] = g < e ? load_point(in, g) : V3<double>{0.0, 0.0, 0.0};
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) w[u] = {nxt[u].x, nxt[u].y, nxt[u].z};
      fetch(g0 + kUnroll * blockDim.x);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t g = g0 + u * blockDim.x + tid;
      int f = 0;
      uint64_t bits = 0;
      bool cand = false;
      bool skip = g >= e;
      if (!skip) {
        int kr;
        if constexpr (kKeyDeferCap > 0) {
          kr = key_point_fast(pose, w[u], r_max, f, bits);
          if (kr == 2) {
            const uint32_t slot = atomicAdd(&sm.n_defer, 1u);
            if (slot < kKeyDeferCap) {
              sm.defer[slot] = static_cast<uint32_t>(g - b);
              kr = 0;
            } else {
              kr = key_point(pose, w[u], r_max, f, bits) ? 1 : 0;  // (queue full: inline)
            }
          }
        } else {
          kr = key_point(pose, w[u], r_max, f, bits) ? 1 : 0;
        }
        if (kr == 1) cand = atomicMin(cell_bits + f, bits) >= bits;
      }
      log_cand(cand, f, g, bits);
    }
  }
  __syncthreads();
  if constexpr (kKeyDeferCap > 0) {
    // the deferred guard-band points, keyed with the FP64 / correctly rounded
    // fallbacks by full warps (any arrival order gives the same minima, and a
    // point tied with its cell's final minimum is logged whenever it arrives)
    const uint32_t n_def = min(sm.n_defer, kKeyDeferCap);
    for (uint32_t q0 = 0; q0 < n_def; q0 += blockDim.x) {
      const uint32_t q = q0 + tid;
      int f = 0;
      uint64_t bits = 0;
      bool cand = false;
      const int64_t g = b + (q < n_def ? sm.defer[q] : 0u);
      if (q < n_def && key_point(pose, load_point(in, g), r_max, f, bits)) cand = atomicMin(cell_bits + f, bits) >= bits;
      log_cand(cand, f, g, bits);
    }
    __syncthreads();
  }
  SNAP_PHASE(1);  // pass A keying
  // pass B: lowest point index among the logged points at the minimum
  // ("strict <, first point wins", perception.cpp:80-86).  The log packs the
  // index in 16 bits; a scene past that (possible on the device entry point,
  // whose per-scene counts the host cannot see), or one whose points lie past
  // the log's capacity, re-keys all its points.
  if (rekey) {
    for (int64_t g = b + tid; g < e; g += blockDim.x) {
      int f;
      uint64_t bits;
      if (key_point(pose, load_point(in, g), r_max, f, bits) && cell_bits[f] == bits)
        atomicMin(sm.idx + f, static_cast<uint32_t>(g - b));
    }
  }
  const uint32_t n_cand = rekey ? 0u : sm.n_cand;
  for (uint32_t c = tid; c < n_cand; c += blockDim.x) {
#if AMPPI_LOG_BITS
    const Candidate cd = log[c];
    if (cell_bits[cd.cell] == cd.bits) atomicMin(sm.idx + cd.cell, cd.idx);
#else
    const uint32_t en = log[c];
    const int f = static_cast<int>(en >> 16);
    const uint32_t idx = en & 0xFFFFu;
    const V3<double> p = to_body(pose, load_point(in, b + idx));
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(sqrt(sqnorm(p))));
    if (cell_bits[f] == bits) atomicMin(sm.idx + f, idx);
#endif
  }
  __syncthreads();
  for (int f = tid; f < kCells; f += blockDim.x) {
    const uint64_t bits = cell_bits[f];
    sm.rng[f] = bits != kEmptyCell ? __longlong_as_double(static_cast<long long>(bits)) : r_max;
  }
  __syncthreads();
  SNAP_PHASE(2);  // pass B ties
  finalize_body(sm, in, P, cfg, s);
}

}  // namespace

size_t finalize_smem_bytes() { return sizeof(FinalizeSmem); }

#ifdef AMPPI_STATS
extern "C" int amppi_snapshot_phase_cycles(unsigned long long* out10, int reset) {
  cudaMemcpyFromSymbol(out10, g_query_stats, sizeof(unsigned long long) * 10, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[10] = {};
    cudaMemcpyToSymbol(g_query_stats, z, sizeof(z), sizeof(unsigned long long) * 16);
  }
  return 0;
}
#endif

cudaError_t init_kernel_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_finalize_scene, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(FinalizeSmem)));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_key_points_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kCells * sizeof(unsigned long long)));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_snapshot_scene, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(sizeof(FinalizeSmem)));
}

cudaError_t launch_snapshot(const BatchIn& in, const Perception& P, const DevConfig& cfg, int64_t max_points_per_scene,
                            cudaStream_t st, KernelTimer* timer) {
  // fused per-scene CTAs once there is at least a GPU's worth of scenes; the
  // many-CTA keying has lower latency for a handful of scenes
  if (max_points_per_scene <= kFusedMaxPoints && in.S >= 148) {
    TimedRegion t(timer, "k_snapshot_scene", st);
    k_snapshot_scene<<<in.S, kFinalizeThreads, sizeof(FinalizeSmem), st>>>(in, P, cfg);
    return cudaGetLastError();
  }
  cudaError_t err = cudaMemsetAsync(P.cand_count, 0, sizeof(unsigned long long), st);
  if (err != cudaSuccess) return err;
  {
    // clusters per scene: ~8 points per thread, at most ~2 waves of clusters
    constexpr int64_t kPer = AMPPI_KEY_PPT;  // target points per thread
    int64_t cps = (max_points_per_scene + kPer * kKeyCluster * kKeyThreads - 1) / (kPer * kKeyCluster * kKeyThreads);
    cps = cps < 1 ? 1 : (cps > 64 ? 64 : cps);
    TimedRegion t(timer, "k_key_points", st);
    k_key_points_cluster<<<dim3(static_cast<unsigned>(cps * kKeyCluster), in.S), kKeyThreads,
                           kCells * sizeof(unsigned long long), st>>>(in, P, static_cast<int>(cps));
  }
  {
    TimedRegion t(timer, "k_resolve_ties", st);
    k_resolve_ties<<<148 * 4, 256, 0, st>>>(P);
  }
  {
    TimedRegion t(timer, "k_finalize_scene", st);
    k_finalize_scene<<<in.S, kFinalizeThreadsFew, sizeof(FinalizeSmem), st>>>(in, P, cfg);
  }
  return cudaGetLastError();
}

}  // namespace amppi_dev
