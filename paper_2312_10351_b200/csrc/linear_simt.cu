// Skinny fp32 linear layer y = act(x W^T + b) for the small-row GEMMs of batch-1
// inference (classifier heads, DeepFM MLP rows 1-32).  One warp per output
// feature and row group: the weight row streams once with 128-bit loads while
// up to kRows activation rows (L1/L2 resident) are reused from registers.

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct LinArgs {
  const float* __restrict__ x;
  const float* __restrict__ w;
  const float* __restrict__ b;
  float* __restrict__ y;
  int M, K, N, act, xs, ys;
};

__device__ __forceinline__ float activate(float v, int act) {
  switch (act) {
    case 1: return fmaxf(v, 0.f);
    case 2: return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
    case 3: return tanhf(v);
    case 4: return 1.f / (1.f + expf(-v));
    default: return v;
  }
}

template <int kRows, bool kVec>
__global__ void __launch_bounds__(256) linear_rows_f32(LinArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int lane = threadIdx.x & 31;
  const int warps_per_block = blockDim.x / 32;
  const int row_groups = (a.M + kRows - 1) / kRows;
  const int64_t total = static_cast<int64_t>(a.N) * row_groups;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(warps_per_block) + threadIdx.x / 32; t < total;
       t += static_cast<int64_t>(gridDim.x) * warps_per_block) {
    const int n = static_cast<int>(t % a.N);
    const int m0 = static_cast<int>(t / a.N) * kRows;
    const float* wrow = a.w + static_cast<int64_t>(n) * a.K;
    float acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = 0.f;
    if constexpr (kVec) {
      const int K4 = a.K / 4;
      for (int k = lane; k < K4; k += 32) {
        const float4 wv = __ldg(reinterpret_cast<const float4*>(wrow) + k);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (m0 + r < a.M) {
            const float4 xv =
                __ldg(reinterpret_cast<const float4*>(a.x + static_cast<int64_t>(m0 + r) * a.xs) + k);
            acc[r] = fmaf(wv.x, xv.x, acc[r]);
            acc[r] = fmaf(wv.y, xv.y, acc[r]);
            acc[r] = fmaf(wv.z, xv.z, acc[r]);
            acc[r] = fmaf(wv.w, xv.w, acc[r]);
          }
        }
      }
    } else {
      for (int k = lane; k < a.K; k += 32) {
        const float wv = __ldg(wrow + k);
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (m0 + r < a.M) acc[r] = fmaf(wv, __ldg(a.x + static_cast<int64_t>(m0 + r) * a.xs + k), acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const float v = warp_sum(acc[r]);
      if (lane == 0 && m0 + r < a.M)
        a.y[static_cast<int64_t>(m0 + r) * a.ys + n] = activate(v + (a.b ? __ldg(a.b + n) : 0.f), a.act);
    }
  }
  trace_end(trace);
}

}  // namespace

opara_status launch_linear(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                           LaunchCfg* cfg, bool dry) {
  LinArgs a;
  a.x = static_cast<const float*>(op.p[0]);
  a.w = static_cast<const float*>(op.p[1]);
  a.b = static_cast<const float*>(op.p[2]);
  a.y = static_cast<float*>(op.p[3]);
  a.M = (int)op.i[0]; a.K = (int)op.i[1]; a.N = (int)op.i[2]; a.act = (int)op.i[3];
  a.xs = op.i[4] ? (int)op.i[4] : a.K;
  a.ys = op.i[5] ? (int)op.i[5] : a.N;
  if (op.i[18] != 0) return fail(OPARA_ERR_VALUE, "linear simt engine: fp32 only");
  const bool vec = (a.K % 4 == 0) && (a.xs % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(a.w) % 16 == 0);
  LaunchCfg c;
  const int rows = a.M >= 4 ? 4 : (a.M >= 2 ? 2 : 1);
  if (vec) {
    c.func = rows == 4 ? reinterpret_cast<const void*>(&linear_rows_f32<4, true>)
           : rows == 2 ? reinterpret_cast<const void*>(&linear_rows_f32<2, true>)
                       : reinterpret_cast<const void*>(&linear_rows_f32<1, true>);
  } else {
    c.func = rows == 4 ? reinterpret_cast<const void*>(&linear_rows_f32<4, false>)
           : rows == 2 ? reinterpret_cast<const void*>(&linear_rows_f32<2, false>)
                       : reinterpret_cast<const void*>(&linear_rows_f32<1, false>);
  }
  const int64_t warps = static_cast<int64_t>(a.N) * ((a.M + rows - 1) / rows);
  c.block = dim3(256);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(warps, 8), 148u * 2u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
