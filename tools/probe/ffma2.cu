// Throughput of scalar FFMA vs packed FFMA2 (sm_100): 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) k1(float* out, int iters, float m, float c) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) k2(float* out, int iters, float m, float c) {
  float2 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
  const float2 mm = make_float2(m, m), cc = make_float2(c, c);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __ffma2_rn(a[k], mm, cc);
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k].x + a[k].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 1 << 14, blocks = sms * 8;
  for (int w = 0; w < 2; ++w) { k1<<<blocks, 256>>>(o, iters, 0.9999f, 1e-4f); k2<<<blocks, 256>>>(o, iters, 0.9999f, 1e-4f); }
  for (int v = 0; v < 2; ++v) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      if (v == 0) k1<<<blocks, 256>>>(o, iters, 0.9999f, 1e-4f); else k2<<<blocks, 256>>>(o, iters, 0.9999f, 1e-4f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * iters * (double)blocks * 256 * (v ? 2 : 1);
    printf("%s: %.3f ms, %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA", best, flops / (best * 1e-3) / 1e12);
  }
  return 0;
}
