// Microbenchmark: shared-memory wavefronts of LDS.64 access patterns
// (run under ncu, metric l1tex__data_pipe_lsu_wavefronts_mem_shared).
#include <cstdio>
#include <cuda_runtime.h>

template <int P>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31;
  int w;
  if (P == 0) w = 2 * l;                                   // contiguous 8-byte
  else if (P == 1) w = (l & 1) ? 1232 + l - 1 : l;         // pair copies 16 banks apart
  else if (P == 2) w = (l & 1) ? 1024 + l - 1 : l;         // 32 banks apart (same banks)
  else if (P == 3) w = (l & 1) ? 1040 + l - 1 : l;         // 16 banks apart, 1040
  else if (P == 4) w = (l < 16) ? 2 * l : 1024 + 2 * (l - 16);  // halves in different copies
  else if (P == 5) w = (l & 1) ? 1232 + l + 15 : l;       // odd lanes shifted by 16 more
  else w = ((l & 1) ? 1232 + l - 1 : l) + 2 * (P - 6);     // P >= 6: pattern 1 + base offset
  const float2* p = reinterpret_cast<const float2*>(s + w);
  float2 acc = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
    const float2 v = p[(it & 7) * 64];
    acc.x += v.x;
    acc.y += v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  k<0><<<1, 32>>>(out, 64);
  k<1><<<1, 32>>>(out, 64);
  k<2><<<1, 32>>>(out, 64);
  k<3><<<1, 32>>>(out, 64);
  k<4><<<1, 32>>>(out, 64);
  k<5><<<1, 32>>>(out, 64);
  k<6><<<1, 32>>>(out, 64);
  k<7><<<1, 32>>>(out, 64);
  k<8><<<1, 32>>>(out, 64);
  k<9><<<1, 32>>>(out, 64);
  k<10><<<1, 32>>>(out, 64);
  k<13><<<1, 32>>>(out, 64);
  k<14><<<1, 32>>>(out, 64);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
