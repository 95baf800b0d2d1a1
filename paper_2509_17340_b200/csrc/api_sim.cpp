// C-ABI of the synthetic input generator (amppi_sim_scan): scenario families
// placed on the host (threads over scenes), LiDAR cast on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/amppi_b200.h"
#include "sim.h"

using namespace amppi_sim;

namespace {

struct DevBuf {
  void* p{nullptr};
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
};

#define SCK(expr)                                                                   \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      std::fprintf(stderr, "amppi_sim_scan: %s: %s\n", #expr, cudaGetErrorString(_e)); \
      return AMPPI_CUDA_ERROR;                                                      \
    }                                                                               \
  } while (0)

}  // namespace

extern "C" int amppi_sim_scan(int32_t n_scenes, const int32_t* kinds, const uint64_t* scene_seeds,
                              int32_t frames, const amppi_state* poses, const uint64_t* frame_seeds, double r_max,
                              int64_t cap_per_scene, float* xyz_out, int64_t* offsets_out, int32_t device) {
  if (n_scenes < 1 || frames < 1 || !kinds || !scene_seeds || !poses || !frame_seeds || !xyz_out || !offsets_out ||
      cap_per_scene < 0)
    return AMPPI_INVALID_ARGUMENT;
  SCK(cudaSetDevice(device));
  // 1. scenarios (host threads)
  std::vector<std::vector<Prim>> scenes(n_scenes);
  {
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (int s = static_cast<int>(t); s < n_scenes; s += static_cast<int>(nt))
          scenes[s] = generate_scenario(kinds[s], scene_seeds[s]);
      });
    for (auto& th : pool) th.join();
  }
  std::vector<DevPrim> prims;
  std::vector<int> prim_off(n_scenes + 1, 0);
  for (int s = 0; s < n_scenes; ++s) {
    for (const auto& p : scenes[s]) prims.push_back(to_device(p));
    prim_off[s + 1] = static_cast<int>(prims.size());
  }
  cudaStream_t st;
  SCK(cudaStreamCreate(&st));
  DevBuf d_prims, d_off;
  SCK(d_prims.alloc(prims.size() * sizeof(DevPrim)));
  SCK(d_off.alloc(prim_off.size() * sizeof(int)));
  SCK(cudaMemcpy(d_prims.p, prims.data(), prims.size() * sizeof(DevPrim), cudaMemcpyHostToDevice));
  SCK(cudaMemcpy(d_off.p, prim_off.data(), prim_off.size() * sizeof(int), cudaMemcpyHostToDevice));

  const float el_min = static_cast<float>(-45.0 * 3.141592653589793 / 180.0);
  const float el_max = static_cast<float>(45.0 * 3.141592653589793 / 180.0);
  const int n_rays = lidar_rays(el_min, el_max);
  const int scenes_per_chunk = std::max(1, 8192 / frames);
  const int max_frames = scenes_per_chunk * frames;
  DevBuf d_frames, d_slots, d_hits, d_off_f, d_take, d_xyz;
  SCK(d_frames.alloc(static_cast<size_t>(max_frames) * sizeof(Frame)));
  SCK(d_slots.alloc(static_cast<size_t>(max_frames) * n_rays * sizeof(float4)));
  SCK(d_hits.alloc(static_cast<size_t>(max_frames) * sizeof(int)));
  SCK(d_off_f.alloc(static_cast<size_t>(max_frames) * sizeof(int)));
  SCK(d_take.alloc(static_cast<size_t>(max_frames) * sizeof(int)));
  const size_t chunk_pts = static_cast<size_t>(scenes_per_chunk) * static_cast<size_t>(std::min<int64_t>(
                               cap_per_scene, static_cast<int64_t>(frames) * n_rays));
  SCK(d_xyz.alloc(chunk_pts * 3 * sizeof(float)));
  std::vector<Frame> hf(max_frames);
  std::vector<int> hits(max_frames), off_f(max_frames), take(max_frames);
  offsets_out[0] = 0;
  for (int s0 = 0; s0 < n_scenes; s0 += scenes_per_chunk) {
    const int ns = std::min(scenes_per_chunk, n_scenes - s0);
    const int nf = ns * frames;
    for (int f = 0; f < nf; ++f) {
      const int s = s0 + f / frames;
      const amppi_state& ps = poses[static_cast<int64_t>(s) * frames + f % frames];
      Frame fr{};
      fr.scene = s;
      for (int i = 0; i < 3; ++i) fr.p[i] = static_cast<float>(ps.p[i]);
      for (int i = 0; i < 4; ++i) fr.q[i] = static_cast<float>(ps.q[i]);
      fr.seed = frame_seeds[static_cast<int64_t>(s) * frames + f % frames];
      hf[f] = fr;
    }
    SCK(cudaMemcpyAsync(d_frames.p, hf.data(), nf * sizeof(Frame), cudaMemcpyHostToDevice, st));
    SCK(launch_lidar(static_cast<DevPrim*>(d_prims.p), static_cast<int*>(d_off.p), static_cast<Frame*>(d_frames.p),
                     nf, static_cast<float>(r_max), el_min, el_max, 0.01f, static_cast<float4*>(d_slots.p),
                     static_cast<int*>(d_hits.p), st));
    SCK(cudaMemcpyAsync(hits.data(), d_hits.p, nf * sizeof(int), cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    int64_t chunk_base = 0;
    for (int k = 0; k < ns; ++k) {
      const int s = s0 + k;
      int64_t run = 0;
      for (int f = k * frames; f < (k + 1) * frames; ++f) {
        const int64_t t = std::max<int64_t>(0, std::min<int64_t>(hits[f], cap_per_scene - run));
        take[f] = static_cast<int>(t);
        off_f[f] = static_cast<int>(chunk_base + run);
        run += t;
      }
      offsets_out[s + 1] = offsets_out[s] + run;
      chunk_base += run;
    }
    SCK(cudaMemcpyAsync(d_off_f.p, off_f.data(), nf * sizeof(int), cudaMemcpyHostToDevice, st));
    SCK(cudaMemcpyAsync(d_take.p, take.data(), nf * sizeof(int), cudaMemcpyHostToDevice, st));
    SCK(launch_compact(static_cast<float4*>(d_slots.p), n_rays, static_cast<int*>(d_off_f.p),
                       static_cast<int*>(d_take.p), nf, static_cast<float*>(d_xyz.p), st));
    SCK(cudaMemcpyAsync(xyz_out + 3 * offsets_out[s0], d_xyz.p, static_cast<size_t>(chunk_base) * 3 * sizeof(float),
                        cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
  }
  cudaStreamDestroy(st);
  return AMPPI_OK;
}

// Host form of amppi_sim_scan (same arithmetic as the kernel, sim_ray.h):
// identical output bytes without a GPU -- the CPU baseline plans exactly the
// scenes the device planned.  Threads over scenes.
extern "C" int amppi_sim_scan_host(int32_t n_scenes, const int32_t* kinds, const uint64_t* scene_seeds,
                                   int32_t frames, const amppi_state* poses, const uint64_t* frame_seeds,
                                   double r_max, int64_t cap_per_scene, float* xyz_out, int64_t* offsets_out) {
  if (n_scenes < 1 || frames < 1 || !kinds || !scene_seeds || !poses || !frame_seeds || !xyz_out || !offsets_out ||
      cap_per_scene < 0)
    return AMPPI_INVALID_ARGUMENT;
  const float el_min = static_cast<float>(-45.0 * 3.141592653589793 / 180.0);
  const float el_max = static_cast<float>(45.0 * 3.141592653589793 / 180.0);
  std::vector<std::vector<float>> pts(n_scenes);
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (int s = static_cast<int>(t); s < n_scenes; s += static_cast<int>(nt)) {
        const std::vector<Prim> sc = generate_scenario(kinds[s], scene_seeds[s]);
        std::vector<DevPrim> dp;
        for (const auto& p : sc) dp.push_back(to_device(p));
        std::vector<Frame> fr(frames);
        for (int f = 0; f < frames; ++f) {
          const amppi_state& ps = poses[static_cast<int64_t>(s) * frames + f];
          fr[f].scene = s;
          for (int i = 0; i < 3; ++i) fr[f].p[i] = static_cast<float>(ps.p[i]);
          for (int i = 0; i < 4; ++i) fr[f].q[i] = static_cast<float>(ps.q[i]);
          fr[f].seed = frame_seeds[static_cast<int64_t>(s) * frames + f];
        }
        std::vector<float> out(static_cast<size_t>(cap_per_scene) * 3);
        const int64_t n = scan_host(dp.data(), static_cast<int>(dp.size()), fr.data(), frames,
                                    static_cast<float>(r_max), el_min, el_max, 0.01f, cap_per_scene, out.data());
        out.resize(static_cast<size_t>(n) * 3);
        pts[s] = std::move(out);
      }
    });
  for (auto& th : pool) th.join();
  offsets_out[0] = 0;
  for (int s = 0; s < n_scenes; ++s) {
    const int64_t n = static_cast<int64_t>(pts[s].size() / 3);
    std::memcpy(xyz_out + 3 * offsets_out[s], pts[s].data(), pts[s].size() * sizeof(float));
    offsets_out[s + 1] = offsets_out[s] + n;
  }
  return AMPPI_OK;
}
