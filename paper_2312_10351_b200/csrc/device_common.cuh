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

// Split-K arrival: every thread has stored its partials (st.global.cg); the
// CTA fences, one thread bumps the tile's arrival counter, and the CTA that
// arrives last (returns true) owns the reduction.  The last arrival resets the
// counter so the next graph replay starts from zero.  Reductions then read the
// partials with ld.global.cg in split order, so results are deterministic.
__device__ __forceinline__ bool splitk_arrive_last(unsigned* cnt, int splits) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const unsigned prev = atomicAdd(cnt, 1u);
    s_last = prev == static_cast<unsigned>(splits - 1);
    if (s_last) atomicExch(cnt, 0u);
  }
  __syncthreads();
  const bool last = s_last != 0;
  if (last) __threadfence();
  return last;
}

// Programmatic dependent launch: let the next kernel of the stream start its
// prologue now, and wait (before touching predecessor outputs) until every
// predecessor grid has completed and flushed its memory.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Fused epilogue activation (opara_op CONV2D i[24]): 0 none, 1 ReLU, 2 GELU (erf), 3 tanh, 4 sigmoid.
__device__ __forceinline__ float apply_act(float v, int act) {
  switch (act) {
    case 1: return fmaxf(v, 0.f);
    case 2: return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
    case 3: return tanhf(v);
    case 4: return 1.f / (1.f + expf(-v));
    default: return v;
  }
}

// Activation code of a CONV2D record: i[24] when set, else ReLU from i[17].
inline int conv_act_code(long long act, long long relu) { return act ? static_cast<int>(act) : (relu ? 1 : 0); }

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
