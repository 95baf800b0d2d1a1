// FP32 FMA-pipe throughput probe: the measured denominator of the rollout
// kernel's roofline (MEASURED_PEAKS.json carries HBM and bf16 tensor peaks
// only).  8 independent FFMA chains per thread, grid = 8 CTAs x 256 threads
// per SM.
#include <cuda_runtime.h>

#include "../../include/amppi_b200.h"

namespace {

__global__ void __launch_bounds__(256) k_ffma_peak(float* out, int iters, float m, float c) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = static_cast<float>(threadIdx.x + k) * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chains live
}

}  // namespace

extern "C" int amppi_probe_fp32_peak(int32_t device, double* tflops, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return AMPPI_CUDA_ERROR;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 1024 * sizeof(float)) != cudaSuccess) return AMPPI_CUDA_ERROR;
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_ffma_peak<<<blocks, threads>>>(out, iters / 8, 0.9999f, 1e-4f);
  double best = 0.0, best_ms = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    k_ffma_peak<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 8.0 * static_cast<double>(iters) * blocks * threads;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) {
      best = tf;
      best_ms = ms;
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return AMPPI_CUDA_ERROR;
  if (tflops) *tflops = best;
  if (ms_out) *ms_out = best_ms;
  return AMPPI_OK;
}
