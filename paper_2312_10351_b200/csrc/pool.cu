// NHWC pooling kernels (memory-bound).  One thread per (output pixel, 4
// channels): 128-bit loads/stores when the channel view is 16-byte aligned,
// scalar otherwise.  Grid-stride loops with a bounded grid.

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct PoolArgs {
  const void* in;
  void* out;
  int N, H, W, C, in_cs, in_coff;
  int OH, OW, out_cs, out_coff;
  int kh, kw, sh, sw, ph, pw;
  int include_pad;
};

// Window semantics follow torch's pooling (max: padding never wins; avg:
// divisor counts padded cells when count_include_pad, clipped at H+pad).
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// V-wide vector of T: 16 B for fp32 x4 and bf16 x8, 8 B for bf16 x4
template <typename T, int V> struct Vec;
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<__nv_bfloat16, 4> { using type = uint2; };
template <> struct Vec<__nv_bfloat16, 8> { using type = uint4; };

template <typename T, int V>
__device__ __forceinline__ void load_v(const T* src, float* x) {
  if constexpr (V == 1) {
    x[0] = to_f(*src);
  } else {
    const typename Vec<T, V>::type t = __ldg(reinterpret_cast<const typename Vec<T, V>::type*>(src));
    const T* e = reinterpret_cast<const T*>(&t);
#pragma unroll
    for (int v = 0; v < V; ++v) x[v] = to_f(e[v]);
  }
}

template <typename T, int V>
__device__ __forceinline__ void store_v(T* dst, const float* acc) {
  if constexpr (V == 1) {
    *dst = from_f<T>(acc[0]);
  } else {
    typename Vec<T, V>::type t;
    T* e = reinterpret_cast<T*>(&t);
#pragma unroll
    for (int v = 0; v < V; ++v) e[v] = from_f<T>(acc[v]);
    *reinterpret_cast<typename Vec<T, V>::type*>(dst) = t;
  }
}

template <bool kMax>
__device__ __forceinline__ float pool_acc(float acc, float x) {
  // max: NaN propagates like torch (x > acc || isnan(x))
  if constexpr (kMax) return (x > acc || isnan(x)) ? x : acc;
  return acc + x;
}

// KS > 0: the window is KS x KS and every tap's load is issued before the
// first reduction (all KS*KS loads in flight: the kernel is a single
// memory round trip instead of KS*KS dependent ones); KS == 0: any window.
template <bool kMax, int V, typename T, int KS>
__global__ void __launch_bounds__(256) pool2d_nhwc(PoolArgs a, unsigned long long* trace) {
  const T* in = static_cast<const T*>(a.in);
  T* outp = static_cast<T*>(a.out);
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int cv = a.C / V;
  const int64_t total = static_cast<int64_t>(a.N) * a.OH * a.OW * cv;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(idx % cv) * V;
    const int64_t q = idx / cv;
    const int ow = static_cast<int>(q % a.OW);
    const int oh = static_cast<int>((q / a.OW) % a.OH);
    const int b = static_cast<int>(q / (static_cast<int64_t>(a.OW) * a.OH));
    int hs = oh * a.sh - a.ph, ws = ow * a.sw - a.pw;
    int he = min(hs + a.kh, a.H + a.ph), we = min(ws + a.kw, a.W + a.pw);
    const int pool_size = (he - hs) * (we - ws);
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = kMax ? -INFINITY : 0.f;
    const T* base = in + static_cast<int64_t>(b) * a.H * a.W * a.in_cs + a.in_coff + c;
    int cnt;
    if constexpr (KS > 0) {
      float x[KS * KS][V];
      bool ok[KS * KS];
#pragma unroll
      for (int t = 0; t < KS * KS; ++t) {
        const int ih = hs + t / KS, iw = ws + t % KS;
        ok[t] = ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
        if (ok[t]) load_v<T, V>(base + (static_cast<int64_t>(ih) * a.W + iw) * a.in_cs, x[t]);
      }
      cnt = 0;
#pragma unroll
      for (int t = 0; t < KS * KS; ++t) {
        if (!ok[t]) continue;
        ++cnt;
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = pool_acc<kMax>(acc[v], x[t][v]);
      }
    } else {
      hs = max(hs, 0);
      ws = max(ws, 0);
      he = min(he, a.H);
      we = min(we, a.W);
      cnt = (he - hs) * (we - ws);
      for (int ih = hs; ih < he; ++ih) {
        for (int iw = ws; iw < we; ++iw) {
          float x[V];
          load_v<T, V>(base + (static_cast<int64_t>(ih) * a.W + iw) * a.in_cs, x);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = pool_acc<kMax>(acc[v], x[v]);
        }
      }
    }
    if constexpr (!kMax) {
      const int div = a.include_pad ? pool_size : cnt;
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = acc[v] / static_cast<float>(div);
    }
    store_v<T, V>(outp + q * a.out_cs + a.out_coff + c, acc);
  }
  trace_end(trace);
}

// Global average pool: one warp per (batch, 4-channel group) when C is large;
// the warp strides over the H*W pixels and shuffles the partial sums.
template <typename T>
__global__ void __launch_bounds__(256) global_avgpool_nhwc(const T* __restrict__ in,
                                                           float* __restrict__ out, int N, int HW,
                                                           int C, int in_cs, int in_coff, int relu_in,
                                                           int out_cs, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  const int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32; w < total;
       w += warps) {
    const int c = static_cast<int>(w % C);
    const int b = static_cast<int>(w / C);
    float s = 0.f;
    for (int p = lane; p < HW; p += 32) {
      const float v = to_f(in[(static_cast<int64_t>(b) * HW + p) * in_cs + in_coff + c]);
      s += relu_in ? fmaxf(v, 0.f) : v;
    }
    s = warp_sum(s);
    if (lane == 0) out[static_cast<int64_t>(b) * out_cs + c] = s / static_cast<float>(HW);
  }
  trace_end(trace);
}

// Small-HW variant: one thread per channel, sequential over pixels; coalesced
// across channels (the common 7x7 / 8x8 tail of CNNs).
template <typename T>
__global__ void __launch_bounds__(128) global_avgpool_nhwc_cols(const T* __restrict__ in,
                                                                float* __restrict__ out, int N,
                                                                int HW, int C, int in_cs,
                                                                int in_coff, int relu_in, int out_cs,
                                                                unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % C);
    const int b = static_cast<int>(t / C);
    const T* src = in + static_cast<int64_t>(b) * HW * in_cs + in_coff + c;
    float s = 0.f;
    for (int p = 0; p < HW; ++p) {
      const float v = to_f(src[static_cast<int64_t>(p) * in_cs]);
      s += relu_in ? fmaxf(v, 0.f) : v;
    }
    out[static_cast<int64_t>(b) * out_cs + c] = s / static_cast<float>(HW);
  }
  trace_end(trace);
}

}  // namespace

opara_status launch_pool2d(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                           LaunchCfg* cfg, bool dry) {
  PoolArgs a;
  a.in = op.p[0];
  a.out = op.p[3];
  a.N = (int)op.i[0]; a.H = (int)op.i[1]; a.W = (int)op.i[2]; a.C = (int)op.i[3];
  a.in_cs = (int)op.i[4]; a.in_coff = (int)op.i[5];
  a.OH = (int)op.i[6]; a.OW = (int)op.i[7]; a.out_cs = (int)op.i[8]; a.out_coff = (int)op.i[9];
  a.kh = (int)op.i[10]; a.kw = (int)op.i[11]; a.sh = (int)op.i[12]; a.sw = (int)op.i[13];
  a.ph = (int)op.i[14]; a.pw = (int)op.i[15]; a.include_pad = (int)op.i[16];
  const bool bf = op.i[18] == 1;
  const bool is_max = op.kind == OPARA_OP_MAXPOOL2D;
  auto aligned = [&](int v, int bytes) {
    return a.C % v == 0 && a.in_cs % v == 0 && a.in_coff % v == 0 && a.out_cs % v == 0 && a.out_coff % v == 0 &&
           reinterpret_cast<uintptr_t>(a.in) % bytes == 0 && reinterpret_cast<uintptr_t>(a.out) % bytes == 0;
  };
  // vector width: 16 B per load where the channel views allow it
  const int V = bf && aligned(8, 16) ? 8 : aligned(4, bf ? 8 : 16) ? 4 : 1;
  const bool k3 = a.kh == 3 && a.kw == 3;
  const int64_t work = static_cast<int64_t>(a.N) * a.OH * a.OW * (a.C / V);
  LaunchCfg c;
#define OPARA_POOL_PICK(T, VV)                                                                          \
  (is_max ? (k3 ? reinterpret_cast<const void*>(&pool2d_nhwc<true, VV, T, 3>)                          \
                : reinterpret_cast<const void*>(&pool2d_nhwc<true, VV, T, 0>))                         \
          : (k3 ? reinterpret_cast<const void*>(&pool2d_nhwc<false, VV, T, 3>)                         \
                : reinterpret_cast<const void*>(&pool2d_nhwc<false, VV, T, 0>)))
  if (bf)
    c.func = V == 8 ? OPARA_POOL_PICK(__nv_bfloat16, 8) : V == 4 ? OPARA_POOL_PICK(__nv_bfloat16, 4)
                                                                 : OPARA_POOL_PICK(__nv_bfloat16, 1);
  else
    c.func = V == 4 ? OPARA_POOL_PICK(float, 4) : OPARA_POOL_PICK(float, 1);
#undef OPARA_POOL_PICK
  c.block = dim3(256);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(work, 256), 148u * 4u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

opara_status launch_global_avgpool(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                                   LaunchCfg* cfg, bool dry) {
  const void* in = op.p[0];
  float* out = static_cast<float*>(op.p[3]);  // always fp32 (feeds the classifier)
  int N = (int)op.i[0], H = (int)op.i[1], W = (int)op.i[2], C = (int)op.i[3];
  int in_cs = (int)op.i[4], in_coff = (int)op.i[5], relu_in = (int)op.i[17];
  int out_cs = op.i[8] > 0 ? (int)op.i[8] : C;   // p[3] points at the output view's first channel
  const bool bf = op.i[18] == 1;
  int HW = H * W;
  LaunchCfg c;
  const int64_t total = static_cast<int64_t>(N) * C;
  if (HW <= 128) {
    c.func = bf ? reinterpret_cast<const void*>(&global_avgpool_nhwc_cols<__nv_bfloat16>)
                : reinterpret_cast<const void*>(&global_avgpool_nhwc_cols<float>);
    c.block = dim3(128);
    c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(total, 128), 148u * 4u)));
  } else {
    c.func = bf ? reinterpret_cast<const void*>(&global_avgpool_nhwc<__nv_bfloat16>)
                : reinterpret_cast<const void*>(&global_avgpool_nhwc<float>);
    c.block = dim3(256);
    c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(total, 8), 148u * 4u)));
  }
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&in, &out, &N, &HW, &C, &in_cs, &in_coff, &relu_in, &out_cs, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
