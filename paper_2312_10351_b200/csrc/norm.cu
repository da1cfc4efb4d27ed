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
