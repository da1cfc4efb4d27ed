// Depthwise 2-D convolution over NHWC channel views (NASNet separable convs):
//
//   y[b, oh, ow, c] = act( sum_{r,s} f(x[b, oh*sh - ph + r, ow*sw - pw + s, c]) * w[r, s, c] + bias[c] )
//
// with f = ReLU when the op's input ReLU is fused (relu_in; NASNet applies
// ReLU in front of every separable conv) and act = none / ReLU.
// Per-channel work is only k*k MACs, so the kernel is bound by moving the
// activations: one thread owns one output pixel x one 16-byte channel vector
// (4 fp32 / 8 bf16 channels), reads every input vector of its window with a
// 128-bit load (the k*k-fold window overlap between neighbouring threads is
// served by L1), the tap weights as fp32 float4 from the read-only path, and
// accumulates in fp32.  Consecutive threads walk channels first, so a warp's
// loads and stores are contiguous along C.  The grid is bounded to a few CTAs
// per SM (grid-stride) so concurrent branches co-reside.
//
// Record (include/opara.h OPARA_OP_DWCONV2D):
//   i: 0 N, 1 H, 2 W, 3 C, 4 in_cs, 5 in_coff, 6 OH, 7 OW, 8 out_cs, 9 out_coff,
//      10 kh, 11 kw, 12 sh, 13 sw, 14 ph, 15 pw, 16 relu_in, 17 act (0 none, 1 ReLU),
//      18 dtype (0 f32, 1 bf16)
//   p: 0 in, 1 weight [kh*kw][C] fp32, 2 bias [C] fp32 (nullable), 3 out

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct DwArgs {
  const void* in;
  const float* __restrict__ w;
  const float* __restrict__ bias;
  void* out;
  int N, H, W, C, in_cs, in_coff, OH, OW, out_cs, out_coff;
  int kh, kw, sh, sw, ph, pw, relu_in, act;
};

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* src, float* f) {
  if constexpr (sizeof(T) == 4 && V == 4) {
    const float4 r = __ldg(reinterpret_cast<const float4*>(src));
    f[0] = r.x; f[1] = r.y; f[2] = r.z; f[3] = r.w;
  } else if constexpr (sizeof(T) == 4 && V == 8) {
    const float4 r0 = __ldg(reinterpret_cast<const float4*>(src));
    const float4 r1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
    f[0] = r0.x; f[1] = r0.y; f[2] = r0.z; f[3] = r0.w;
    f[4] = r1.x; f[5] = r1.y; f[6] = r1.z; f[7] = r1.w;
  } else if constexpr (sizeof(T) == 2 && V == 8) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(src));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 t = __bfloat1622float2(h[k]);
      f[2 * k] = t.x;
      f[2 * k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if constexpr (sizeof(T) == 2) f[e] = __bfloat162float(src[e]); else f[e] = src[e];
    }
  }
}

template <typename T, int V>
__device__ __forceinline__ void store_vec(T* dst, const float* f) {
  if constexpr (sizeof(T) == 4 && V == 4) {
    *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
  } else if constexpr (sizeof(T) == 2 && V == 8) {
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
    *reinterpret_cast<uint4*>(dst) = r;
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if constexpr (sizeof(T) == 2) dst[e] = __float2bfloat16_rn(f[e]); else dst[e] = f[e];
    }
  }
}

template <typename T, int V>
__global__ void __launch_bounds__(256) dwconv2d_nhwc(DwArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int cv = a.C / V;
  const int64_t total = static_cast<int64_t>(a.N) * a.OH * a.OW * cv;
  const T* in = static_cast<const T*>(a.in);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % cv) * V;
    int64_t q = t / cv;
    const int ow = static_cast<int>(q % a.OW);
    q /= a.OW;
    const int oh = static_cast<int>(q % a.OH);
    const int b = static_cast<int>(q / a.OH);
    const int ih0 = oh * a.sh - a.ph, iw0 = ow * a.sw - a.pw;
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
    for (int r = 0; r < a.kh; ++r) {
      const int ih = ih0 + r;
      if (ih < 0 || ih >= a.H) continue;
      const T* row = in + (static_cast<int64_t>(b) * a.H + ih) * a.W * a.in_cs + a.in_coff + c;
      const float* wrow = a.w + static_cast<int64_t>(r) * a.kw * a.C + c;
      for (int s = 0; s < a.kw; ++s) {
        const int iw = iw0 + s;
        if (iw < 0 || iw >= a.W) continue;
        float x[V], w[V];
        load_vec<T, V>(row + static_cast<int64_t>(iw) * a.in_cs, x);
        load_vec<float, V>(wrow + static_cast<int64_t>(s) * a.C, w);
        if (a.relu_in) {
#pragma unroll
          for (int e = 0; e < V; ++e) x[e] = fmaxf(x[e], 0.f);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = fmaf(x[e], w[e], acc[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < V; ++e) {
      float v = acc[e] + (a.bias ? __ldg(a.bias + c + e) : 0.f);
      acc[e] = a.act == 1 ? fmaxf(v, 0.f) : v;
    }
    store_vec<T, V>(static_cast<T*>(a.out) + ((static_cast<int64_t>(b) * a.OH + oh) * a.OW + ow) * a.out_cs +
                        a.out_coff + c,
                    acc);
  }
  trace_end(trace);
}

}  // namespace

opara_status launch_dwconv2d(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                             LaunchCfg* cfg, bool dry) {
  DwArgs a;
  a.in = op.p[0];
  a.w = static_cast<const float*>(op.p[1]);
  a.bias = static_cast<const float*>(op.p[2]);
  a.out = op.p[3];
  a.N = (int)op.i[0]; a.H = (int)op.i[1]; a.W = (int)op.i[2]; a.C = (int)op.i[3];
  a.in_cs = (int)op.i[4]; a.in_coff = (int)op.i[5];
  a.OH = (int)op.i[6]; a.OW = (int)op.i[7]; a.out_cs = (int)op.i[8]; a.out_coff = (int)op.i[9];
  a.kh = (int)op.i[10]; a.kw = (int)op.i[11]; a.sh = (int)op.i[12]; a.sw = (int)op.i[13];
  a.ph = (int)op.i[14]; a.pw = (int)op.i[15]; a.relu_in = (int)op.i[16]; a.act = (int)op.i[17];
  if (a.N <= 0 || a.OH <= 0 || a.OW <= 0 || a.C <= 0 || a.kh <= 0 || a.kw <= 0)
    return fail(OPARA_ERR_VALUE, "dwconv2d: empty shape");
  const bool bf = op.i[18] == 1;
  const int V = bf ? 8 : 4;
  const bool vec = a.C % V == 0 && a.in_cs % V == 0 && a.in_coff % V == 0 && a.out_cs % V == 0 &&
                   a.out_coff % V == 0 && reinterpret_cast<uintptr_t>(a.in) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(a.out) % 16 == 0 && reinterpret_cast<uintptr_t>(a.w) % 16 == 0;
  LaunchCfg c;
  c.func = bf ? (vec ? reinterpret_cast<const void*>(&dwconv2d_nhwc<__nv_bfloat16, 8>)
                     : reinterpret_cast<const void*>(&dwconv2d_nhwc<__nv_bfloat16, 1>))
              : (vec ? reinterpret_cast<const void*>(&dwconv2d_nhwc<float, 4>)
                     : reinterpret_cast<const void*>(&dwconv2d_nhwc<float, 1>));
  const int64_t work = static_cast<int64_t>(a.N) * a.OH * a.OW * (a.C / (vec ? V : 1));
  c.block = dim3(256);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(work, 256), 148u * 4u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
