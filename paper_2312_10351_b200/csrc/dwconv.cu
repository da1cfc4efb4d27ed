// Depthwise 2-D convolution over NHWC channel views (NASNet separable convs):
//
//   y[b, oh, ow, c] = act( sum_{r,s} f(x[b, oh*sh - ph + r, ow*sw - pw + s, c]) * w[r, s, c] + bias[c] )
//
// with f = ReLU when the op's input ReLU is fused (relu_in; NASNet applies
// ReLU in front of every separable conv) and act = none / ReLU.
// Per-channel work is only k*k MACs, so the kernel is bound by moving the
// activations: one thread owns kPx adjacent output pixels x one 16-byte
// channel vector (4 fp32 / 8 bf16 channels; 8 / 4-byte vectors for channel
// counts that are not multiples of 8), reads every input vector of its window
// with a vector load (the window overlap between neighbours is served by L1),
// each tap's fp32 weights once for its kPx pixels, and accumulates in fp32.  Consecutive threads walk channels first, so a warp's
// loads and stores are contiguous along C.  The grid is bounded to a few CTAs
// per SM (grid-stride) so concurrent branches co-reside.
//
// Record (include/opara.h OPARA_OP_DWCONV2D):
//   i: 0 N, 1 H, 2 W, 3 C, 4 in_cs, 5 in_coff, 6 OH, 7 OW, 8 out_cs, 9 out_coff,
//      10 kh, 11 kw, 12 sh, 13 sw, 14 ph, 15 pw, 16 relu_in, 17 act (0 none, 1 ReLU),
//      18 dtype (0 f32, 1 bf16)
//   p: 0 in, 1 weight [kh*kw][C] fp32, 2 bias [C] fp32 (nullable), 3 out

#include <cuda_bf16.h>

#include <cstdlib>

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
  } else if constexpr (sizeof(T) == 2 && V == 4) {
    const uint2 r = __ldg(reinterpret_cast<const uint2*>(src));
    const float2 t0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    const float2 t1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
    f[0] = t0.x; f[1] = t0.y; f[2] = t1.x; f[3] = t1.y;
  } else if constexpr (sizeof(T) == 2 && V == 2) {
    const float2 t = __bfloat1622float2(__ldg(reinterpret_cast<const __nv_bfloat162*>(src)));
    f[0] = t.x; f[1] = t.y;
  } else if constexpr (sizeof(T) == 4 && V == 2) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(src));
    f[0] = t.x; f[1] = t.y;
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

// Plain (generic / shared-memory) vector load: 16-byte bf16x8 or fp32x4, 8-byte bf16x4.
template <typename T, int V>
__device__ __forceinline__ void load_vec_plain(const T* src, float* f) {
  if constexpr (sizeof(T) == 2 && V == 8) {
    const uint4 r = *reinterpret_cast<const uint4*>(src);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 t = __bfloat1622float2(h[k]);
      f[2 * k] = t.x;
      f[2 * k + 1] = t.y;
    }
  } else if constexpr (sizeof(T) == 4 && V == 4) {
    const float4 r = *reinterpret_cast<const float4*>(src);
    f[0] = r.x; f[1] = r.y; f[2] = r.z; f[3] = r.w;
  } else if constexpr (sizeof(T) == 2 && V == 4) {
    const uint2 r = *reinterpret_cast<const uint2*>(src);
    const float2 t0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    const float2 t1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
    f[0] = t0.x; f[1] = t0.y; f[2] = t1.x; f[3] = t1.y;
  } else if constexpr (sizeof(T) == 4 && V == 2) {
    const float2 r = *reinterpret_cast<const float2*>(src);
    f[0] = r.x; f[1] = r.y;
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
  } else if constexpr (sizeof(T) == 2 && V == 4) {
    uint2 r;
    *reinterpret_cast<__nv_bfloat162*>(&r.x) = __floats2bfloat162_rn(f[0], f[1]);
    *reinterpret_cast<__nv_bfloat162*>(&r.y) = __floats2bfloat162_rn(f[2], f[3]);
    *reinterpret_cast<uint2*>(dst) = r;
  } else if constexpr (sizeof(T) == 2 && V == 2) {
    *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(f[0], f[1]);
  } else if constexpr (sizeof(T) == 4 && V == 2) {
    *reinterpret_cast<float2*>(dst) = make_float2(f[0], f[1]);
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

// A thread owns one 16-byte channel vector of kPx horizontally adjacent
// output pixels: each tap's weights are loaded once and reused for the kPx
// pixels (L1 serves the overlapping input columns).  Square k x k windows
// known at compile time (KS = 3, 5, 7) unroll both tap loops so a thread's
// window loads are all in flight together; KS = 0 is the generic fallback.
constexpr int kPx = 1;   // 4 was measured slower: too few threads on small maps

template <typename T, int V, int KS>
__global__ void __launch_bounds__(256) dwconv2d_nhwc(DwArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int cv = a.C / V;
  const int owb = (a.OW + kPx - 1) / kPx;
  const int64_t total = static_cast<int64_t>(a.N) * a.OH * owb * cv;
  const T* in = static_cast<const T*>(a.in);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % cv) * V;
    int64_t q = t / cv;
    const int ow0 = static_cast<int>(q % owb) * kPx;
    q /= owb;
    const int oh = static_cast<int>(q % a.OH);
    const int b = static_cast<int>(q / a.OH);
    const int ih0 = oh * a.sh - a.ph;
    float acc[kPx][V];
#pragma unroll
    for (int p = 0; p < kPx; ++p)
#pragma unroll
      for (int e = 0; e < V; ++e) acc[p][e] = 0.f;
    const T* base = in + static_cast<int64_t>(b) * a.H * a.W * a.in_cs + a.in_coff + c;
    auto tap = [&](int r, int s) {
      const int ih = ih0 + r;
      if (ih < 0 || ih >= a.H) return;
      float w[V];
      load_vec<float, V>(a.w + static_cast<int64_t>(r * a.kw + s) * a.C + c, w);
      const T* row = base + static_cast<int64_t>(ih) * a.W * a.in_cs;
#pragma unroll
      for (int p = 0; p < kPx; ++p) {
        const int iw = (ow0 + p) * a.sw - a.pw + s;
        if (ow0 + p >= a.OW || iw < 0 || iw >= a.W) continue;
        float x[V];
        load_vec<T, V>(row + static_cast<int64_t>(iw) * a.in_cs, x);
        if (a.relu_in) {
#pragma unroll
          for (int e = 0; e < V; ++e) x[e] = fmaxf(x[e], 0.f);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[p][e] = fmaf(x[e], w[e], acc[p][e]);
      }
    };
    if constexpr (KS > 0) {
#pragma unroll
      for (int r = 0; r < KS; ++r)
#pragma unroll
        for (int s = 0; s < KS; ++s) tap(r, s);
    } else {
      for (int r = 0; r < a.kh; ++r)
        for (int s = 0; s < a.kw; ++s) tap(r, s);
    }
    float bias[V];
#pragma unroll
    for (int e = 0; e < V; ++e) bias[e] = a.bias ? __ldg(a.bias + c + e) : 0.f;
#pragma unroll
    for (int p = 0; p < kPx; ++p) {
      if (ow0 + p >= a.OW) break;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float v = acc[p][e] + bias[e];
        acc[p][e] = a.act == 1 ? fmaxf(v, 0.f) : v;
      }
      store_vec<T, V>(static_cast<T*>(a.out) + ((static_cast<int64_t>(b) * a.OH + oh) * a.OW + ow0 + p) * a.out_cs +
                          a.out_coff + c,
                      acc[p]);
    }
  }
  trace_end(trace);
}

// Shared-memory tiled variant (16-byte channel vectors, square 3/5/7 windows):
// a CTA owns an 8 x 8 output tile x kCV channel vectors.  Its weights are
// staged before griddepcontrol.wait (parameters), its input halo tile right
// after with one coalesced 16-byte load per chunk (a single memory round trip
// for the whole window), then every thread computes one output pixel-vector
// from shared memory.
constexpr int kTile = 8, kCV = 4;

template <typename T, int V, int KS, int SS>
__global__ void __launch_bounds__(kTile * kTile * kCV) dwconv2d_tiled(DwArgs a, unsigned long long* trace) {
  constexpr int IH = (kTile - 1) * SS + KS, IW = IH;
  constexpr int CW = kCV * V;   // channels per CTA
  extern __shared__ __align__(16) uint8_t dsm[];
  float* ws = reinterpret_cast<float*>(dsm);                       // [KS*KS][CW]
  T* xs = reinterpret_cast<T*>(dsm + KS * KS * CW * sizeof(float));  // [IH][IW][CW]
  pdl_trigger();
  const int tid = threadIdx.x;
  const int tiles_w = (a.OW + kTile - 1) / kTile, tiles_h = (a.OH + kTile - 1) / kTile;
  int bid = blockIdx.x;
  const int tw = bid % tiles_w;
  bid /= tiles_w;
  const int th = bid % tiles_h;
  bid /= tiles_h;
  const int cgroups = (a.C + CW - 1) / CW;
  const int cg = bid % cgroups;
  const int b = bid / cgroups;
  const int c0 = cg * CW;
  // weights: KS*KS*kCV chunks of V fp32
  for (int u = tid; u < KS * KS * kCV; u += blockDim.x) {
    const int tap = u / kCV, cv = u % kCV, c = c0 + cv * V;
    float w[V];
    if (c < a.C) load_vec<float, V>(a.w + static_cast<int64_t>(tap) * a.C + c, w);
    else {
#pragma unroll
      for (int e = 0; e < V; ++e) w[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < V; ++e) ws[tap * CW + cv * V + e] = w[e];
  }
  pdl_wait();
  trace_begin(trace);
  const int ih0 = th * kTile * SS - a.ph, iw0 = tw * kTile * SS - a.pw;
  const T* in = static_cast<const T*>(a.in) + static_cast<int64_t>(b) * a.H * a.W * a.in_cs + a.in_coff;
  for (int u = tid; u < IH * IW * kCV; u += blockDim.x) {
    const int cv = u % kCV, px = u / kCV, iy = px / IW, ix = px % IW;
    const int ih = ih0 + iy, iw = iw0 + ix, c = c0 + cv * V;
    float x[V];
    if (ih >= 0 && ih < a.H && iw >= 0 && iw < a.W && c < a.C) {
      load_vec<T, V>(in + (static_cast<int64_t>(ih) * a.W + iw) * a.in_cs + c, x);
      if (a.relu_in) {
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = fmaxf(x[e], 0.f);
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) x[e] = 0.f;
    }
    store_vec<T, V>(xs + px * CW + cv * V, x);
  }
  __syncthreads();
  const int cv = tid % kCV, p = tid / kCV, oy = p / kTile, ox = p % kTile;
  const int oh = th * kTile + oy, ow = tw * kTile + ox, c = c0 + cv * V;
  if (oh < a.OH && ow < a.OW && c < a.C) {
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
#pragma unroll
    for (int r = 0; r < KS; ++r)
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        float x[V];
        load_vec_plain<T, V>(xs + ((oy * SS + r) * IW + ox * SS + q) * CW + cv * V, x);
        const float* w = ws + (r * KS + q) * CW + cv * V;
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = fmaf(x[e], w[e], acc[e]);
      }
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const float v = acc[e] + (a.bias ? __ldg(a.bias + c + e) : 0.f);
      acc[e] = a.act == 1 ? fmaxf(v, 0.f) : v;
    }
    store_vec<T, V>(static_cast<T*>(a.out) + ((static_cast<int64_t>(b) * a.OH + oh) * a.OW + ow) * a.out_cs +
                        a.out_coff + c,
                    acc);
  }
  trace_end(trace);
}

template <int KS, int SS>
constexpr size_t tiled_smem(int v, int esz) {
  return static_cast<size_t>(KS * KS * kCV * v) * 4 +
         static_cast<size_t>(((kTile - 1) * SS + KS) * ((kTile - 1) * SS + KS) * kCV * v) * esz;
}

bool tiled_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("OPARA_DW_TILED");
    return v && v[0] == '0';
  }();
  return off;
}

template <typename T, int V>
const void* pick_tiled(int ks, int ss, size_t* smem) {
  constexpr int esz = sizeof(T);
#define OPARA_DW_T(K, S)                                               \
  if (ks == K && ss == S) {                                            \
    *smem = tiled_smem<K, S>(V, esz);                                  \
    return reinterpret_cast<const void*>(&dwconv2d_tiled<T, V, K, S>); \
  }
  OPARA_DW_T(3, 1) OPARA_DW_T(5, 1) OPARA_DW_T(7, 1) OPARA_DW_T(3, 2) OPARA_DW_T(5, 2) OPARA_DW_T(7, 2)
#undef OPARA_DW_T
  return nullptr;
}

template <typename T, int V>
const void* pick_ks(int ks) {
  switch (ks) {
    case 3: return reinterpret_cast<const void*>(&dwconv2d_nhwc<T, V, 3>);
    case 5: return reinterpret_cast<const void*>(&dwconv2d_nhwc<T, V, 5>);
    case 7: return reinterpret_cast<const void*>(&dwconv2d_nhwc<T, V, 7>);
    default: return reinterpret_cast<const void*>(&dwconv2d_nhwc<T, V, 0>);
  }
}

template <typename T>
const void* pick_dw(int vw, int ks) {
  if (vw == 8 && sizeof(T) == 2) return pick_ks<T, 8>(ks);
  if (vw == 4) return pick_ks<T, 4>(ks);
  if (vw == 2) return pick_ks<T, 2>(ks);
  return pick_ks<T, 1>(ks);
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
  // vector width: 16 bytes when every view allows it, else 8 / 4 bytes, else scalar
  auto fits = [&](int v) {
    return a.C % v == 0 && a.in_cs % v == 0 && a.in_coff % v == 0 && a.out_cs % v == 0 && a.out_coff % v == 0;
  };
  int vw = 1;
  if (vec) vw = V;
  else if (bf && fits(4) && reinterpret_cast<uintptr_t>(a.in) % 8 == 0 && reinterpret_cast<uintptr_t>(a.out) % 8 == 0)
    vw = 4;
  else if (fits(2) && reinterpret_cast<uintptr_t>(a.in) % (bf ? 4 : 8) == 0 &&
           reinterpret_cast<uintptr_t>(a.out) % (bf ? 4 : 8) == 0)
    vw = 2;
  const int ks = (a.kh == a.kw && (a.kh == 3 || a.kh == 5 || a.kh == 7)) ? a.kh : 0;
  LaunchCfg c;
  // tiled shared-memory kernel for 16-byte vectors (8-byte ones when the
  // 16-byte tiling would leave fewer than two CTAs per SM), square windows,
  // equal strides 1/2
  const bool tiled_ok = vw >= V / 2;
  if (tiled_ok && ks && a.sh == a.sw && (a.sh == 1 || a.sh == 2) && !tiled_disabled()) {
    size_t smem = 0;
    const int64_t tiles = static_cast<int64_t>((a.OW + kTile - 1) / kTile) * ((a.OH + kTile - 1) / kTile) * a.N;
    const int tv = (vw == V && tiles * ((a.C + kCV * V - 1) / (kCV * V)) >= 2 * 148) ? V : V / 2;
    if (bf)
      c.func = tv == 8 ? pick_tiled<__nv_bfloat16, 8>(ks, a.sh, &smem) : pick_tiled<__nv_bfloat16, 4>(ks, a.sh, &smem);
    else
      c.func = tv == 4 ? pick_tiled<float, 4>(ks, a.sh, &smem) : pick_tiled<float, 2>(ks, a.sh, &smem);
    if (c.func) {
      const int cgroups = (a.C + kCV * tv - 1) / (kCV * tv);
      c.block = dim3(kTile * kTile * kCV);
      c.grid = dim3(static_cast<unsigned>(((a.OW + kTile - 1) / kTile) * ((a.OH + kTile - 1) / kTile) * cgroups * a.N));
      c.smem = smem;
      if (cfg) *cfg = c;
      if (dry) return OPARA_OK;
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(c.func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return cuda_fail(e, "dwconv2d_tiled smem attribute");
      }
      void* args[] = {&a, &trace};
      return launch_kernel(c, args, s);
    }
  }
  c.func = bf ? pick_dw<__nv_bfloat16>(vw, ks) : pick_dw<float>(vw, ks);
  const int64_t work = static_cast<int64_t>(a.N) * a.OH * ((a.OW + kPx - 1) / kPx) * (a.C / vw);
  c.block = dim3(256);   // (smaller CTAs on small maps measured slower)
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(work, 256), 148u * 4u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
