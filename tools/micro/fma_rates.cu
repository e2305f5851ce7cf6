// Microbenchmark: issue rate of FFMA (register/uniform operands) vs FFMA2
// (packed f32x2) on this GPU.  Informs the sweep's inner loop design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rates fma_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r)
               : "l"(*reinterpret_cast<unsigned long long*>(&a)),
                 "l"(*reinterpret_cast<unsigned long long*>(&b)),
                 "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

// 3 distinct vector registers per FFMA: acc[k] = w[k] * v[k&3] + acc[k]
__global__ void k_ffma3(float* out, int iters) {
  float acc[16], w[16], v[4];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x + k, w[k] = 1.0001f + k * 1e-4f;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = 0.999f - k * 1e-4f + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = fmaf(w[k], v[(k + u) & 3], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = acc[k] * 1e-9f + v[k];
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  if (s == 1.2345f) out[0] = s;
}

// FFMA2, scalar broadcast weight: acc2[k] = (w,w) * v2[.] + acc2[k]
__global__ void k_ffma2s(float* out, int iters) {
  float2 acc[8], v[4];
  float w[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x + k, k), w[k] = 1.0001f + k * 1e-4f;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = make_float2(0.999f - k * 1e-4f, 0.998f + threadIdx.x * 1e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = ffma2(make_float2(w[k], w[k]), v[(k + u) & 3], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k].x = acc[k].x * 1e-9f + v[k].x;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  if (s == 1.2345f) out[0] = s;
}

// FFMA2 all-pair operands
__global__ void k_ffma2p(float* out, int iters) {
  float2 acc[8], v[4], w[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x + k, k), w[k] = make_float2(1.0001f + k * 1e-4f, 1.f);
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = make_float2(0.999f - k * 1e-4f, 0.998f + threadIdx.x * 1e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = ffma2(w[k], v[(k + u) & 3], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k].x = acc[k].x * 1e-9f + v[k].x;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  if (s == 1.2345f) out[0] = s;
}

// FFMA2 interleaved with an equal number of ALU ops (FMNMX) -- dual issue?
__global__ void k_ffma2_alu(float* out, int iters) {
  float2 acc[8], v[4];
  float w[8], m[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x + k, k), w[k] = 1.0001f + k * 1e-4f, m[k] = -k;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = make_float2(0.999f - k * 1e-4f, 0.998f + threadIdx.x * 1e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc[k] = ffma2(make_float2(w[k], w[k]), v[(k + u) & 3], acc[k]);
        m[k] = fmaxf(m[k], v[(k + u + 1) & 3].y);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k].x = acc[k].x * 1e-9f + v[k].x + m[k] * 1e-12f;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y + m[k];
  if (s == 1.2345f) out[0] = s;
}

// FFMA (3-reg) interleaved with FMNMX
__global__ void k_ffma3_alu(float* out, int iters) {
  float acc[16], w[16], v[4], m[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = threadIdx.x + k, w[k] = 1.0001f + k * 1e-4f, m[k] = -k;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = 0.999f - k * 1e-4f + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        acc[k] = fmaf(w[k], v[(k + u) & 3], acc[k]);
        m[k] = fmaxf(m[k], v[(k + u + 1) & 3]);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = acc[k] * 1e-9f + v[k] + m[k] * 1e-12f;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k] + m[k];
  if (s == 1.2345f) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, double fma_per_iter, double instr_per_iter) {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  kern<<<blocks, threads>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double thr = (double)blocks * threads * iters;
  printf("%-12s %8.3f ms  %7.1f TFLOP/s  %7.2f Twarp-instr/s (loop instr)\n", name, ms,
         thr * fma_per_iter * 2 / ms / 1e9, thr * instr_per_iter / 32 / ms / 1e9);
  cudaFree(out);
}

int main() {
  run("ffma3", k_ffma3, 128 + 4, 128 + 8);
  run("ffma2s", k_ffma2s, 128 + 4, 64 + 8);
  run("ffma2p", k_ffma2p, 128 + 4, 64 + 8);
  run("ffma2+alu", k_ffma2_alu, 128 + 4, 128 + 12);
  run("ffma3+alu", k_ffma3_alu, 128 + 4, 256 + 12);
  return 0;
}
