// Memory-bound n-ary elementwise operator over NHWC channel views:
//
//   ADD   y = act(x0 + x1 (+ x2 (+ x3)))       (NASNet cell combinations, DeepFM head)
//   COPY  y = act(x0)                           (a graph input copied into a concat slice)
//   RELU  y = relu(x0)                          (unfused fallback)
//
// Every operand is a channel view (buffer, cstride, coff) of P pixels x C
// channels, so inputs and the output may live inside concatenated buffers.
// One thread owns a 16-byte vector (4 fp32 / 8 bf16 channels) of one pixel when
// every view is vector aligned, otherwise one element; loads are 128-bit and
// coalesced along channels, sums are fp32, the grid is bounded to a few CTAs
// per SM (grid-stride) so concurrent branches can co-reside.
//
// Record (include/opara.h OPARA_OP_ADD / COPY / RELU):
//   i: 0 P (pixels), 1 C, 2 n_in (1..4), 3 act (0 none, 1 ReLU, 4 sigmoid),
//      4 out_cs, 5 out_coff, 6..9 in_cs[j], 10..13 in_coff[j], 18 dtype (0 f32, 1 bf16)
//   p: 0, 1, 2, 4 inputs x0..x3; 3 out

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct EwArgs {
  const void* in[4];
  void* out;
  int64_t P;
  int C, n_in, act, out_cs, out_coff;
  int in_cs[4], in_coff[4];
};

__device__ __forceinline__ float ew_act(float v, int act) {
  if (act == 1) return fmaxf(v, 0.f);
  if (act == 4) return 1.f / (1.f + expf(-v));
  return v;
}

template <typename T, int V>
struct Vec;
template <>
struct Vec<float, 4> {
  using raw = float4;
  __device__ static void unpack(const raw& r, float* f) { f[0] = r.x; f[1] = r.y; f[2] = r.z; f[3] = r.w; }
  __device__ static raw pack(const float* f) { return make_float4(f[0], f[1], f[2], f[3]); }
};
template <>
struct Vec<__nv_bfloat16, 8> {
  using raw = uint4;
  __device__ static void unpack(const raw& r, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 t = __bfloat1622float2(h[k]);
      f[2 * k] = t.x;
      f[2 * k + 1] = t.y;
    }
  }
  __device__ static raw pack(const float* f) {
    raw r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
    return r;
  }
};

template <typename T, int V>
__global__ void __launch_bounds__(256) ew_vec(EwArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  using VT = Vec<T, V>;
  const int cv = a.C / V;
  const int64_t total = a.P * cv;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = t / cv;
    const int c = static_cast<int>(t - p * cv) * V;
    float acc[V], x[V];
    VT::unpack(*reinterpret_cast<const typename VT::raw*>(static_cast<const T*>(a.in[0]) + p * a.in_cs[0] +
                                                           a.in_coff[0] + c),
               acc);
    for (int j = 1; j < a.n_in; ++j) {
      VT::unpack(*reinterpret_cast<const typename VT::raw*>(static_cast<const T*>(a.in[j]) + p * a.in_cs[j] +
                                                             a.in_coff[j] + c),
                 x);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] += x[e];
    }
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = ew_act(acc[e], a.act);
    *reinterpret_cast<typename VT::raw*>(static_cast<T*>(a.out) + p * a.out_cs + a.out_coff + c) = VT::pack(acc);
  }
  trace_end(trace);
}

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*p); else return *p;
}

template <typename T>
__global__ void __launch_bounds__(256) ew_scalar(EwArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int64_t total = a.P * a.C;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = t / a.C;
    const int c = static_cast<int>(t - p * a.C);
    float acc = 0.f;
    for (int j = 0; j < a.n_in; ++j)
      acc += ld_f(static_cast<const T*>(a.in[j]) + p * a.in_cs[j] + a.in_coff[j] + c);
    acc = ew_act(acc, a.act);
    T* dst = static_cast<T*>(a.out) + p * a.out_cs + a.out_coff + c;
    if constexpr (sizeof(T) == 2) *dst = __float2bfloat16_rn(acc); else *dst = acc;
  }
  trace_end(trace);
}

// PACK_INPUT: the fp32 NCHW graph image -> NHWC (bf16 or fp32) with the
// channels zero-padded to Cp (a multiple of the 16-byte vector width), so the
// stem conv gathers one 16-byte vector per (pixel, tap) instead of Cin scalar
// strided loads.  Thread = (pixel, channel group): reads coalesced along
// pixels, one 16-byte store.
template <typename T, int V>
__global__ void __launch_bounds__(256) pack_input_nchw(const float* __restrict__ in, T* out, int N, int HW, int C,
                                                       int Cp, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int groups = Cp / V;
  const int64_t npix = static_cast<int64_t>(N) * HW;
  const int64_t total = npix * groups;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = t / npix;
    const int64_t q = t - g * npix;  // pixel index over the batch
    const int64_t b = q / HW, pix = q - b * HW;
    float f[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int c = static_cast<int>(g) * V + e;
      f[e] = c < C ? __ldg(in + (b * C + c) * HW + pix) : 0.f;
    }
    *reinterpret_cast<typename Vec<T, V>::raw*>(out + q * Cp + g * V) = Vec<T, V>::pack(f);
  }
  trace_end(trace);
}

}  // namespace

opara_status launch_pack_input(const opara_op& op, cudaStream_t s, unsigned long long* trace, LaunchCfg* cfg,
                               bool dry) {
  const float* in = static_cast<const float*>(op.p[0]);
  void* out = op.p[3];
  int N = (int)op.i[0], HW = (int)(op.i[1] * op.i[2]), C = (int)op.i[3], Cp = (int)op.i[4];
  const bool bf16 = op.i[18] == 1;
  const int V = bf16 ? 8 : 4;
  if (Cp % V || Cp < C || N <= 0 || HW <= 0) return fail(OPARA_ERR_VALUE, "pack_input: bad shape");
  LaunchCfg c;
  c.func = bf16 ? reinterpret_cast<const void*>(&pack_input_nchw<__nv_bfloat16, 8>)
                : reinterpret_cast<const void*>(&pack_input_nchw<float, 4>);
  c.block = dim3(256);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(static_cast<int64_t>(N) * HW * (Cp / V), 256), 148u * 4u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&in, &out, &N, &HW, &C, &Cp, &trace};
  return launch_kernel(c, args, s);
}

opara_status launch_elementwise(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                                LaunchCfg* cfg, bool dry) {
  EwArgs a;
  a.P = op.i[0];
  a.C = (int)op.i[1];
  a.n_in = op.kind == OPARA_OP_ADD ? (int)op.i[2] : 1;
  a.act = op.kind == OPARA_OP_RELU ? 1 : (int)op.i[3];
  a.out_cs = (int)op.i[4];
  a.out_coff = (int)op.i[5];
  const void* ptr_slot[4] = {op.p[0], op.p[1], op.p[2], op.p[4]};
  if (a.n_in < 1 || a.n_in > 4) return fail(OPARA_ERR_VALUE, "elementwise: 1..4 inputs");
  if (a.P <= 0 || a.C <= 0) return fail(OPARA_ERR_VALUE, "elementwise: empty shape");
  const bool bf = op.i[18] == 1;
  const int V = bf ? 8 : 4;
  bool vec = a.C % V == 0 && a.out_cs % V == 0 && a.out_coff % V == 0 &&
             reinterpret_cast<uintptr_t>(op.p[3]) % 16 == 0;
  for (int j = 0; j < 4; ++j) {
    a.in[j] = j < a.n_in ? ptr_slot[j] : nullptr;
    a.in_cs[j] = (int)op.i[6 + j];
    a.in_coff[j] = (int)op.i[10 + j];
    if (j < a.n_in) {
      if (!dry && !a.in[j]) return fail(OPARA_ERR_VALUE, "elementwise: null input");
      vec = vec && a.in_cs[j] % V == 0 && a.in_coff[j] % V == 0 && reinterpret_cast<uintptr_t>(a.in[j]) % 16 == 0;
    }
  }
  a.out = op.p[3];
  LaunchCfg c;
  c.func = vec ? (bf ? reinterpret_cast<const void*>(&ew_vec<__nv_bfloat16, 8>)
                     : reinterpret_cast<const void*>(&ew_vec<float, 4>))
               : (bf ? reinterpret_cast<const void*>(&ew_scalar<__nv_bfloat16>)
                     : reinterpret_cast<const void*>(&ew_scalar<float>));
  const int64_t work = a.P * (vec ? a.C / V : a.C);
  c.block = dim3(256);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(work, 256), 148u * 4u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
