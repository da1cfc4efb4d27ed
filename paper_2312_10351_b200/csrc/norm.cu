// Row kernels of the transformer path (memory-bound, one warp per row):
//   EMBEDDING  y[t] = LN(word[ids[t]] + pos[t + pos_off] + type[tt[t]])   (HF BertEmbeddings)
//   LAYERNORM  y[t] = LN(a[t] (+ b[t]))                                   (residual add fused)
// fp32 statistics (two-pass over registers: mean, then centred variance,
// like torch's layer_norm), bf16 in/out, fp32 gamma/beta.  Rows are held in
// registers (C <= 32 * kMaxPerLane), loads/stores are 8- or 16-byte vectors.

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

constexpr int kMaxPerLane = 32;  // C <= 1024

struct RowArgs {
  const void* a;
  const __nv_bfloat16* b;      // residual (LAYERNORM) or null
  const int64_t* ids;          // token ids (EMBEDDING)
  const int64_t* type_ids;     // token-type ids or null (type 0)
  const float* word;           // [vocab][C]
  const float* pos;            // [max_pos][C]
  const float* type;           // [types][C]
  const float* gamma;
  const float* beta;
  __nv_bfloat16* out;
  int rows, C, a_stride, b_stride, out_stride, pos_off;
  float eps;
};

template <int kPer>
__device__ __forceinline__ void ln_store(float (&x)[kPer], const RowArgs& a, int row, int lane) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kPer; ++i) s += x[i];
  const float mean = warp_sum(s) / a.C;
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const float d = x[i] - mean;
    v += d * d;
  }
  const float rstd = rsqrtf(warp_sum(v) / a.C + a.eps);
  __nv_bfloat16* out = a.out + static_cast<int64_t>(row) * a.out_stride;
#pragma unroll
  for (int i = 0; i < kPer; i += 2) {
    const int c = (i / 2) * 64 + lane * 2;  // lane owns column pairs c, c+1 of each 64-wide slab
    const float y0 = (x[i] - mean) * rstd * __ldg(a.gamma + c) + __ldg(a.beta + c);
    const float y1 = (x[i + 1] - mean) * rstd * __ldg(a.gamma + c + 1) + __ldg(a.beta + c + 1);
    *reinterpret_cast<__nv_bfloat162*>(out + c) = __floats2bfloat162_rn(y0, y1);
  }
}

template <int kPer>
__global__ void __launch_bounds__(256) layernorm_rows(RowArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row < a.rows) {
    const __nv_bfloat16* pa = static_cast<const __nv_bfloat16*>(a.a) + static_cast<int64_t>(row) * a.a_stride;
    const __nv_bfloat16* pb = a.b ? a.b + static_cast<int64_t>(row) * a.b_stride : nullptr;
    float x[kPer];
#pragma unroll
    for (int i = 0; i < kPer; i += 2) {
      const int c = (i / 2) * 64 + lane * 2;
      float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(pa + c));
      if (pb) {
        const float2 r = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(pb + c));
        v.x += r.x;
        v.y += r.y;
      }
      x[i] = v.x;
      x[i + 1] = v.y;
    }
    ln_store<kPer>(x, a, row, lane);
  }
  trace_end(trace);
}

template <int kPer>
__global__ void __launch_bounds__(256) embedding_ln_rows(RowArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row < a.rows) {
    const int64_t id = __ldg(a.ids + row);
    const int64_t tt = a.type_ids ? __ldg(a.type_ids + row) : 0;
    const float* w = a.word + id * a.C;
    const float* p = a.pos + static_cast<int64_t>(row + a.pos_off) * a.C;
    const float* t = a.type + tt * a.C;
    float x[kPer];
#pragma unroll
    for (int i = 0; i < kPer; i += 2) {
      const int c = (i / 2) * 64 + lane * 2;
      const float2 wv = __ldg(reinterpret_cast<const float2*>(w + c));
      const float2 pv = __ldg(reinterpret_cast<const float2*>(p + c));
      const float2 tv = __ldg(reinterpret_cast<const float2*>(t + c));
      x[i] = wv.x + tv.x + pv.x;  // HF order: (inputs_embeds + token_type) + position
      x[i + 1] = wv.y + tv.y + pv.y;
    }
    ln_store<kPer>(x, a, row, lane);
  }
  trace_end(trace);
}

// ---- 16-byte-vector variants (C % 256 == 0; BERT's 768): lane owns kCh
// chunks of 8 columns at 8 * (lane + 32 * j).  gamma / beta (and the position
// / type rows) are parameters, so they are loaded before griddepcontrol.wait,
// i.e. while the predecessor kernel still runs; after the wait only the
// activations are read (all of a row's 16-byte loads in flight at once).

__device__ __forceinline__ void bf8_to_f(const uint4& r, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

template <int kCh>
struct Affine {
  float g[kCh][8], b[kCh][8];
  __device__ __forceinline__ void load(const float* gamma, const float* beta, int lane) {
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      const int c = 8 * (lane + 32 * j);
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + c));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + c + 4));
      g[j][0] = g0.x; g[j][1] = g0.y; g[j][2] = g0.z; g[j][3] = g0.w;
      g[j][4] = g1.x; g[j][5] = g1.y; g[j][6] = g1.z; g[j][7] = g1.w;
      b[j][0] = b0.x; b[j][1] = b0.y; b[j][2] = b0.z; b[j][3] = b0.w;
      b[j][4] = b1.x; b[j][5] = b1.y; b[j][6] = b1.z; b[j][7] = b1.w;
    }
  }
};

template <int kCh>
__device__ __forceinline__ void ln_store_v(float (&x)[kCh][8], const Affine<kCh>& af, const RowArgs& a, int row,
                                           int lane) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kCh; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) s += x[j][e];
  const float mean = warp_sum(s) / a.C;
  float v = 0.f;
#pragma unroll
  for (int j = 0; j < kCh; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = x[j][e] - mean;
      v += d * d;
    }
  const float rstd = rsqrtf(warp_sum(v) / a.C + a.eps);
  __nv_bfloat16* out = a.out + static_cast<int64_t>(row) * a.out_stride;
#pragma unroll
  for (int j = 0; j < kCh; ++j) {
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      h[k] = __floats2bfloat162_rn((x[j][2 * k] - mean) * rstd * af.g[j][2 * k] + af.b[j][2 * k],
                                   (x[j][2 * k + 1] - mean) * rstd * af.g[j][2 * k + 1] + af.b[j][2 * k + 1]);
    *reinterpret_cast<uint4*>(out + 8 * (lane + 32 * j)) = r;
  }
}

template <int kCh>
__global__ void __launch_bounds__(128) layernorm_rows_v(RowArgs a, unsigned long long* trace) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  Affine<kCh> af;
  af.load(a.gamma, a.beta, lane);
  pdl_wait();
  trace_begin(trace);
  if (row < a.rows) {
    const __nv_bfloat16* pa = static_cast<const __nv_bfloat16*>(a.a) + static_cast<int64_t>(row) * a.a_stride;
    const __nv_bfloat16* pb = a.b ? a.b + static_cast<int64_t>(row) * a.b_stride : nullptr;
    uint4 ra[kCh], rb[kCh];
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      ra[j] = *reinterpret_cast<const uint4*>(pa + 8 * (lane + 32 * j));
      if (pb) rb[j] = *reinterpret_cast<const uint4*>(pb + 8 * (lane + 32 * j));
    }
    float x[kCh][8];
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      bf8_to_f(ra[j], x[j]);
      if (pb) {
        float y[8];
        bf8_to_f(rb[j], y);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[j][e] += y[e];
      }
    }
    ln_store_v<kCh>(x, af, a, row, lane);
  }
  trace_end(trace);
}

template <int kCh>
__global__ void __launch_bounds__(128) embedding_ln_rows_v(RowArgs a, unsigned long long* trace) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  Affine<kCh> af;
  af.load(a.gamma, a.beta, lane);
  pdl_wait();
  trace_begin(trace);
  if (row < a.rows) {
    const int64_t id = __ldg(a.ids + row);
    const int64_t tt = a.type_ids ? __ldg(a.type_ids + row) : 0;
    const float* w = a.word + id * a.C;
    const float* p = a.pos + static_cast<int64_t>(row + a.pos_off) * a.C;
    const float* t = a.type + tt * a.C;
    float4 wv[kCh][2], pv[kCh][2], tv[kCh][2];
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      const int c = 8 * (lane + 32 * j);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        wv[j][h] = __ldg(reinterpret_cast<const float4*>(w + c) + h);
        pv[j][h] = __ldg(reinterpret_cast<const float4*>(p + c) + h);
        tv[j][h] = __ldg(reinterpret_cast<const float4*>(t + c) + h);
      }
    }
    float x[kCh][8];
#pragma unroll
    for (int j = 0; j < kCh; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // HF order: (inputs_embeds + token_type) + position
        x[j][4 * h + 0] = wv[j][h].x + tv[j][h].x + pv[j][h].x;
        x[j][4 * h + 1] = wv[j][h].y + tv[j][h].y + pv[j][h].y;
        x[j][4 * h + 2] = wv[j][h].z + tv[j][h].z + pv[j][h].z;
        x[j][4 * h + 3] = wv[j][h].w + tv[j][h].w + pv[j][h].w;
      }
    ln_store_v<kCh>(x, af, a, row, lane);
  }
  trace_end(trace);
}

template <int kPer>
const void* pick(bool emb) {
  return emb ? reinterpret_cast<const void*>(&embedding_ln_rows<kPer>)
             : reinterpret_cast<const void*>(&layernorm_rows<kPer>);
}

}  // namespace

// LAYERNORM  i: 0 rows, 1 C, 2 a_stride, 3 b_stride, 4 out_stride; f[0] eps
//            p: 0 a, 1 residual b (nullable), 2 gamma, 3 beta, 4 out
// EMBEDDING  i: 0 rows, 1 C, 4 out_stride, 5 pos_offset; f[0] eps
//            p: 0 ids (int64), 1 type ids (nullable), 2 gamma, 3 beta, 4 out,
//               5 word table, 6 position table, 7 type table (fp32)
opara_status launch_rows(const opara_op& op, cudaStream_t s, unsigned long long* trace, LaunchCfg* cfg,
                         bool dry) {
  const bool emb = op.kind == OPARA_OP_EMBEDDING;
  RowArgs a = {};
  a.rows = (int)op.i[0];
  a.C = (int)op.i[1];
  a.a_stride = op.i[2] ? (int)op.i[2] : a.C;
  a.b_stride = op.i[3] ? (int)op.i[3] : a.C;
  a.out_stride = op.i[4] ? (int)op.i[4] : a.C;
  a.pos_off = (int)op.i[5];
  a.eps = static_cast<float>(op.f[0]);
  a.gamma = static_cast<const float*>(op.p[2]);
  a.beta = static_cast<const float*>(op.p[3]);
  a.out = static_cast<__nv_bfloat16*>(op.p[4]);
  if (emb) {
    a.ids = static_cast<const int64_t*>(op.p[0]);
    a.type_ids = static_cast<const int64_t*>(op.p[1]);
    a.word = static_cast<const float*>(op.p[5]);
    a.pos = static_cast<const float*>(op.p[6]);
    a.type = static_cast<const float*>(op.p[7]);
  } else {
    a.a = op.p[0];
    a.b = static_cast<const __nv_bfloat16*>(op.p[1]);
  }
  if (a.C % 64 != 0 || a.C > 32 * kMaxPerLane)
    return fail(OPARA_ERR_VALUE, "layernorm/embedding: C must be a multiple of 64 and <= 1024");
  const int per = a.C / 32;
  LaunchCfg c;
  const bool aligned = a.C % 256 == 0 && a.out_stride % 8 == 0 && reinterpret_cast<uintptr_t>(a.out) % 16 == 0 &&
                       (emb || (a.a_stride % 8 == 0 && reinterpret_cast<uintptr_t>(a.a) % 16 == 0 &&
                                (!a.b || (a.b_stride % 8 == 0 && reinterpret_cast<uintptr_t>(a.b) % 16 == 0))));
  if (aligned && (a.C == 256 || a.C == 512 || a.C == 768 || a.C == 1024)) {
    switch (a.C / 256) {
      case 1: c.func = emb ? (const void*)&embedding_ln_rows_v<1> : (const void*)&layernorm_rows_v<1>; break;
      case 2: c.func = emb ? (const void*)&embedding_ln_rows_v<2> : (const void*)&layernorm_rows_v<2>; break;
      case 3: c.func = emb ? (const void*)&embedding_ln_rows_v<3> : (const void*)&layernorm_rows_v<3>; break;
      default: c.func = emb ? (const void*)&embedding_ln_rows_v<4> : (const void*)&layernorm_rows_v<4>; break;
    }
    c.block = dim3(128);
    c.grid = dim3(ceil_div(a.rows, 4));
    if (cfg) *cfg = c;
    if (dry) return OPARA_OK;
    void* args[] = {&a, &trace};
    return launch_kernel(c, args, s);
  }
  switch (per) {
    case 2: c.func = pick<2>(emb); break;
    case 4: c.func = pick<4>(emb); break;
    case 8: c.func = pick<8>(emb); break;
    case 12: c.func = pick<12>(emb); break;
    case 16: c.func = pick<16>(emb); break;
    case 24: c.func = pick<24>(emb); break;
    case 32: c.func = pick<32>(emb); break;
    default: return fail(OPARA_ERR_VALUE, "layernorm/embedding: unsupported C");
  }
  c.block = dim3(256);
  c.grid = dim3(ceil_div(a.rows, 8));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
