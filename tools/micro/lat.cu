// Microbenchmark: dependent-chain latency (cycles) of FFMA / DFMA / DADD.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
  double x = threadIdx.x;
  float f = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { f = fmaf(f, (float)a, (float)b); f = fmaf(f, (float)a, (float)b); f = fmaf(f, (float)a, (float)b); f = fmaf(f, (float)a, (float)b); }
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { x = x + b; x = x + a; x = x + b; x = x + a; }
  long long t3 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; long long h[3];
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 24);
  const int n = 4096;
  k<<<1, 32>>>(o, c, n, 0.999, 1e-3);
  k<<<1, 32>>>(o, c, n, 0.999, 1e-3);
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("DFMA %.2f  FFMA %.2f  DADD %.2f cycles per dependent op\n", h[0] / (4.0 * n), h[1] / (4.0 * n), h[2] / (4.0 * n));
  return 0;
}
