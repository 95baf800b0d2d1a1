// Native sample-sharded plan_step over NCCL (config C4): one
// context per GPU, the whole exchange protocol of DESIGN.md §6 run from C++
// so a host caller of the C ABI can shard without a Python runtime.
//
// Per MPPI iteration, on the context's stream:
//   k_stage1_f32* screen the rank's samples -> ncclAllReduce(MIN) of the M
//   per-instance FP32 minima -> FP64 refine of the rank's support + softmin
//   partials -> ncclAllGather of the M x (3 + 4N) partials -> fixed-order
//   merge + nominal update (identical on every rank).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): a process that has
// already loaded NCCL (e.g. through torch) gets that same library, so a
// communicator created by the caller's NCCL is usable here; a process that
// never shards does not need NCCL at all.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/amppi_b200.h"

namespace {

struct NcclApi {
  void* handle{nullptr};
  ncclResult_t (*get_unique_id)(ncclUniqueId*){nullptr};
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int){nullptr};
  ncclResult_t (*comm_destroy)(ncclComm_t){nullptr};
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t){nullptr};
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t){nullptr};
  const char* (*error_string)(ncclResult_t){nullptr};
  ncclResult_t (*get_version)(int*){nullptr};
  std::string err;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(api.handle, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_reduce || !api.all_gather ||
        !api.error_string || !api.get_version) {
      api.err = "libnccl.so.2 lacks a required symbol";
      api.handle = nullptr;
    }
  });
  return api;
}

// Device scratch of one sharded plan, kept per context (grown on demand).
struct ShardBuffers {
  float* local_min{nullptr};
  double* partials{nullptr};
  double* gathered{nullptr};
  size_t min_n{0}, part_n{0}, gath_n{0};
};

}  // namespace

extern "C" {

int amppi_nccl_version(int32_t* version) {
  NcclApi& a = nccl();
  if (!a.handle) return AMPPI_NCCL_ERROR;
  int v = 0;
  if (a.get_version(&v) != ncclSuccess) return AMPPI_NCCL_ERROR;
  if (version) *version = v;
  return AMPPI_OK;
}

int amppi_nccl_unique_id(void* id_out) {
  NcclApi& a = nccl();
  if (!id_out) return AMPPI_INVALID_ARGUMENT;
  if (!a.handle) return AMPPI_NCCL_ERROR;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return AMPPI_NCCL_ERROR;
  std::memcpy(id_out, &id, sizeof(id));
  return AMPPI_OK;
}

int amppi_nccl_comm_init(void** comm_out, int32_t nranks, const void* id, int32_t rank, int32_t device) {
  NcclApi& a = nccl();
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return AMPPI_INVALID_ARGUMENT;
  if (!a.handle) return AMPPI_NCCL_ERROR;
  if (cudaSetDevice(device) != cudaSuccess) return AMPPI_CUDA_ERROR;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (a.comm_init_rank(&c, nranks, uid, rank) != ncclSuccess) return AMPPI_NCCL_ERROR;
  *comm_out = c;
  return AMPPI_OK;
}

int amppi_nccl_comm_destroy(void* comm) {
  NcclApi& a = nccl();
  if (!comm) return AMPPI_OK;
  if (!a.handle) return AMPPI_NCCL_ERROR;
  return a.comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? AMPPI_OK : AMPPI_NCCL_ERROR;
}

int amppi_plan_sharded(amppi_ctx* ctx, void* comm, int32_t rank, int32_t nranks, const amppi_state* x,
                       const amppi_goal* goal, const double* previous, int32_t previous_len,
                       const amppi_control* last_applied, uint64_t cycle, uint64_t seed, amppi_plan_result* out) {
  if (!ctx || !comm || nranks < 1 || rank < 0 || rank >= nranks) return AMPPI_INVALID_ARGUMENT;
  NcclApi& a = nccl();
  if (!a.handle) return AMPPI_NCCL_ERROR;
  amppi_config cfg{};
  amppi_get_config(ctx, &cfg);
  const int M = cfg.m_h * cfg.m_v, K = cfg.rollouts;
  if (nranks > K) return AMPPI_INVALID_ARGUMENT;
  // balanced contiguous sample range of this rank (sharding.shard_ranges)
  const int base = K / nranks, extra = K % nranks;
  const int k0 = rank * base + std::min(rank, extra);
  const int k1 = k0 + base + (rank < extra ? 1 : 0);
  const size_t stride = static_cast<size_t>(amppi_shard_partials_stride(ctx));
  thread_local ShardBuffers buf;  // per host thread (one context per thread, see amppi_b200.h)
  auto grow = [](auto*& p, size_t& have, size_t need) {
    if (have >= need) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    have = 0;
    cudaError_t e = cudaMalloc(&p, need * sizeof(*p));
    if (e == cudaSuccess) have = need;
    return e;
  };
  if (grow(buf.local_min, buf.min_n, M) != cudaSuccess || grow(buf.partials, buf.part_n, M * stride) != cudaSuccess ||
      grow(buf.gathered, buf.gath_n, static_cast<size_t>(nranks) * M * stride) != cudaSuccess)
    return AMPPI_CUDA_ERROR;
  int rc = amppi_shard_begin(ctx, x, goal, previous, previous_len, last_applied, cycle, seed, k0, k1);
  if (rc != AMPPI_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(amppi_get_stream(ctx));
  for (int it = 0; it < cfg.iterations; ++it) {
    if ((rc = amppi_shard_screen(ctx, it, buf.local_min)) != AMPPI_OK) return rc;
    if (a.all_reduce(buf.local_min, buf.local_min, static_cast<size_t>(M), ncclFloat32, ncclMin,
                     static_cast<ncclComm_t>(comm), st) != ncclSuccess)
      return AMPPI_NCCL_ERROR;
    if ((rc = amppi_shard_partials(ctx, it, buf.local_min, buf.partials)) != AMPPI_OK) return rc;
    if (a.all_gather(buf.partials, buf.gathered, M * stride, ncclFloat64, static_cast<ncclComm_t>(comm), st) !=
        ncclSuccess)
      return AMPPI_NCCL_ERROR;
    if ((rc = amppi_shard_update(ctx, it, buf.gathered, nranks)) != AMPPI_OK) return rc;
  }
  return amppi_shard_finish(ctx, out);
}

}  // extern "C"
