// Shared device helpers for libmshbm (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <utility>

#define MSHBM_DEV __device__ __forceinline__

namespace mshbm {

// Per-device dynamic shared-memory opt-in for one kernel.  The limit is a
// per-device function attribute, and one process may drive several devices
// (one context per device); calls may come from several host threads.
struct SmemAttr {
  std::mutex m;
  size_t bytes[64] = {};
  template <typename F>
  cudaError_t ensure(F* kernel, size_t need) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(m);
    if (bytes[dev & 63] >= need) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
    if (e == cudaSuccess) bytes[dev & 63] = need;
    return e;
  }
};


constexpr int kWcNone = -2147483647 - 1;   // "untrusted" window centre
// sweep4 levels: the trusted-window selection (sweep4.cu prior_select_kernel)
// runs before the dense sweep and marks its trusted pixels as done (final
// outputs written) or low (the sweep computes their 3x3 refinement).  Real
// window centres are >= -radius, so these never collide, and c -+ radius
// cannot overflow.
constexpr int kWcLow = -(1 << 30);
constexpr int kWcDone = -(1 << 30) - 1;

MSHBM_DEV int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its stream predecessor is still finishing; it must call
// pdl_wait() before touching any memory the predecessor reads or writes
// (every pipeline kernel does so first thing; a no-op without PDL).
MSHBM_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Warp-wide sum of a 64-bit counter.
MSHBM_DEV unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

MSHBM_DEV long long warp_max_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Block-aggregated atomic add: one atomic per warp (lane 0).
MSHBM_DEV void warp_atomic_add(unsigned long long* dst, unsigned long long v) {
  v = warp_sum_u64(v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

MSHBM_DEV void warp_atomic_max(long long* dst, long long v) {
  v = warp_max_i64(v);
  if ((threadIdx.x & 31) == 0 && v > 0) atomicMax((long long*)dst, v);
}

// Per-level device counters (int64), see mshbm_level_trace; each level owns
// kCntCopies copies of kCntSlots counters.
enum CounterSlot {
  kCntTrusted = 0,
  kCntTrustedEvals = 1,
  kCntWindowMax = 2,
  kCntRefined = 3,
  kCntNeeded = 4,
  kCntMedianReplaced = 5,
  kCntSlots = 8
};
constexpr int kCntCopies = 64;
MSHBM_DEV int kCntCopyStride(unsigned b) { return (int)(b % kCntCopies); }

// Block-level counter accumulation: warp shuffles, one shared-memory atomic
// per warp, one global atomic per block (same-address global atomics from
// every warp serialise in L2).  Every thread of the block must call it.
template <int NSLOT>
MSHBM_DEV void block_accumulate(unsigned long long* __restrict__ gdst, const int (&slot)[NSLOT],
                                const unsigned long long (&val)[NSLOT], const bool (&is_max)[NSLOT]) {
  // per-thread values are small (< 2^32 per block): 32-bit warp reductions
  // (REDUX, one instruction), 32-bit shared atomics, one 64-bit global
  // atomic per block and slot
  __shared__ unsigned acc[NSLOT];
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  if (tid < NSLOT) acc[tid] = 0u;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NSLOT; ++k) {
    const unsigned x = (unsigned)val[k];
    const unsigned r = is_max[k] ? __reduce_max_sync(0xffffffffu, x) : __reduce_add_sync(0xffffffffu, x);
    if ((tid & 31) == 0 && r) {
      if (is_max[k]) atomicMax(&acc[k], r);
      else atomicAdd(&acc[k], r);
    }
  }
  __syncthreads();
  // counters are spread over kCntCopies cache-line-separated copies (block
  // index modulo): same-address atomics from every block would serialise in
  // L2; the host sums (or maxes) the copies when it reads the trace
  if (tid < NSLOT && acc[tid]) {
    unsigned long long* dst = gdst + (size_t)kCntSlots * kCntCopyStride(blockIdx.x + gridDim.x * blockIdx.y) + slot[tid];
    if (is_max[tid]) atomicMax(dst, (unsigned long long)acc[tid]);
    else atomicAdd(dst, (unsigned long long)acc[tid]);
  }
}

}  // namespace mshbm
