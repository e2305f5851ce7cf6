// Diagnostics: FP32 FFMA throughput probe (roofline denominator for the
// ZNCC sweep; MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
#include <cuda_runtime.h>

#include "../../include/mshbm.h"

namespace {

__global__ void ffma_probe(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

__global__ void dfma_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" int mshbm_probe_fp64_peak(int device, int iters, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return MSHBM_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return MSHBM_ERR_CUDA;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_probe<<<blocks, threads>>>(out, 16, 0.999, 1e-4);
  cudaEventRecord(e0);
  dfma_probe<<<blocks, threads>>>(out, iters, 0.999, 1e-4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return MSHBM_ERR_CUDA;
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
  if (ms) *ms = t;
  return MSHBM_OK;
}

extern "C" int mshbm_probe_fp32_peak(int device, int iters, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return MSHBM_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return MSHBM_ERR_CUDA;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_probe<<<blocks, threads>>>(out, 64, 0.999f, 1e-4f);   // warm-up
  cudaEventRecord(e0);
  ffma_probe<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return MSHBM_ERR_CUDA;
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
  if (ms) *ms = t;
  return MSHBM_OK;
}
