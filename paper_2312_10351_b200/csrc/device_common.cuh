// Device helpers shared by every kernel family.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace opara {

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Kernel timeline probes (opara_exec_trace): block-level earliest start and
// warp-level latest end, one u64 pair per op.  A null pointer costs a branch.
__device__ __forceinline__ void trace_begin(unsigned long long* t) {
  if (t && threadIdx.x == 0 && threadIdx.y == 0) atomicMin(t, global_ns());
}
__device__ __forceinline__ void trace_end(unsigned long long* t) {
  if (t && (threadIdx.x & 31) == 0) atomicMax(t + 1, global_ns());
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace opara
