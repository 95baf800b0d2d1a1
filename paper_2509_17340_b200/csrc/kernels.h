// Host-side launch interface of the plan-cycle kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "layout.h"

namespace amppi_dev {

// Optional per-kernel CUDA-event timing (amppi_options.profile).
struct KernelTimer {
  bool enabled{false};
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<double, int64_t>> totals;  // ms, launches

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // Accumulate finished events (call after a stream sync).
  void collect() {
    for (auto& p : pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, p.a, p.b);
      auto& t = totals[p.name];
      t.first += ms;
      t.second += 1;
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
  ~KernelTimer() {
    for (auto& p : pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct TimedRegion {
  KernelTimer* t;
  const char* name;
  cudaStream_t st;
  cudaEvent_t a{nullptr};
  TimedRegion(KernelTimer* timer, const char* n, cudaStream_t s) : t(timer), name(n), st(s) {
    if (t && t->enabled) {
      a = t->get();
      cudaEventRecord(a, st);
    }
  }
  ~TimedRegion() {
    if (t && t->enabled) {
      cudaEvent_t b = t->get();
      cudaEventRecord(b, st);
      t->pending.push_back({name, a, b});
    }
  }
};

size_t finalize_smem_bytes();
cudaError_t init_kernel_attributes();

// Snapshot (K1, K1b, K2).
cudaError_t launch_snapshot(const BatchIn& in, const Perception& P, const DevConfig& cfg,
                            int64_t max_points_per_scene, cudaStream_t st, KernelTimer* timer);

// Plan: anchors + guides + warm start (K4), stage-I iterations (K3 + K4b),
// stage II + selection (inside K4b's last iteration).  cand_* are [S*M*K]
// scratch arrays for the softmin support.
cudaError_t launch_plan_impl(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                             int precision, bool want_winner_rollout, uint32_t* cand_k, double* cand_s,
                             double* cand_w, uint2* pairs, unsigned long long* pair_count, cudaStream_t st,
                             KernelTimer* timer);

// Phases of launch_plan_impl, used directly by the sample-sharded plan
// (config C4): begin (anchors, guides, warm start) ... finish (stage II,
// selection).  Screening / partials / merge work on samples [cfg.k_lo,
// cfg.k_hi); partials are [S*M*(3+4N)] doubles, all_partials n_shards of them.
cudaError_t launch_plan_begin(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                              cudaStream_t st, KernelTimer* timer);
cudaError_t launch_plan_finish(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                               bool want_winner_rollout, cudaStream_t st, KernelTimer* timer);
cudaError_t launch_shard_screen(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                                float* local_min, cudaStream_t st, KernelTimer* timer);
cudaError_t launch_shard_partials(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg,
                                  uint32_t* cand_k, double* cand_s, double* cand_w, uint2* pairs,
                                  unsigned long long* pair_count, int iter, const float* global_min, double* partials,
                                  cudaStream_t st, KernelTimer* timer);
cudaError_t launch_shard_merge(const BatchIn& in, const Plan& pl, const DevConfig& cfg, const double* all_partials,
                               int n_shards, cudaStream_t st, KernelTimer* timer);

// Per-scene winner outputs gathered into dense arrays (any pointer may be null).
struct GatherOut {
  int32_t* status;
  int32_t* winner;
  double* control;
  double* winner_nominal;
  double* stage2;
  double* breakdown;
};
cudaError_t launch_gather(const Plan& pl, const DevConfig& cfg, int S, const GatherOut& g, cudaStream_t st);

// FP32 stage-I screening rollouts (k_plan32.cu).
int device_sms();  // SM count of the current device (cached)
cudaError_t launch_stage1_f32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                              cudaStream_t st, KernelTimer* timer);

// Screening-drift diagnostic (amppi_screen_drift): sampled rollouts of scenes
// [s0, s0 + S) in FP32 as the screening runs them (k_plan32.cu), then in FP64
// as the refine runs them, compared per step (k_plan64.cu).  steps: [rows*N],
// cost: [rows], rows = S * M * ceil((k_hi - k_lo) / kstride); acc: [8].
constexpr int kDriftSlots = 8;
cudaError_t launch_drift32(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                           int s0, int S, int kstride, float4* steps, float* cost, cudaStream_t st);
cudaError_t launch_drift64(const BatchIn& in, const Perception& P, const Plan& pl, const DevConfig& cfg, int iter,
                           int s0, int S, int kstride, const float4* steps, const float* cost,
                           unsigned long long* acc, cudaStream_t st);

}  // namespace amppi_dev
