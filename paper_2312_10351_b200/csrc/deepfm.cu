// DeepFM operators (recommendation DAG: per-field embedding gathers feeding an
// FM interaction and an MLP in parallel).  All fp32, memory/latency bound.
//
//   FIELD_EMBEDDING  out[b, :] = table[ids[b, field], :]          one op per sparse field
//                    (rows land straight in their slice of the MLP input: concat eliminated)
//   FIRST_ORDER      out[b] = sum_f w1[f][ids[b, f]] + dense[b, :] . wd + bias
//   FM               out[b] = 0.5 * sum_d ((sum_f v[b,f,d])^2 - sum_f v[b,f,d]^2)
//
// Ids outside [0, vocab) read row 0 of nothing: they produce zeros (the CPU
// model would raise; the device cannot, so the host validates its inputs).
//
// Records (include/opara.h):
//   FIELD_EMBEDDING i: 0 B, 1 dim, 2 field, 3 ids_stride, 4 out_cs, 5 out_coff, 6 vocab
//                   p: 0 ids int64 [B][ids_stride], 1 table [vocab][dim], 3 out
//   FIRST_ORDER     i: 0 B, 1 fields, 2 ids_stride, 3 n_dense, 4 dense_stride, 5 vocab, 6 out_cs
//                   p: 0 ids, 1 w1 [fields][vocab], 2 wd [n_dense], 4 dense [B][dense_stride], 3 out
//                   f: 0 bias
//   FM              i: 0 B, 1 fields, 2 dim, 3 in_cs, 4 in_coff, 5 out_cs
//                   p: 0 embeddings (field-major [fields][dim] inside each row), 3 out

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct FieldArgs {
  const int64_t* ids;
  const float* __restrict__ table;
  float* out;
  int B, dim, field, ids_stride, out_cs, out_coff;
  int64_t vocab;
};

// One thread per (row, 4-float chunk) when dim % 4 == 0, else per element.
template <int V>
__global__ void __launch_bounds__(128) field_embedding(FieldArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int per_row = a.dim / V;
  const int64_t total = static_cast<int64_t>(a.B) * per_row;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(t / per_row);
    const int c = static_cast<int>(t - static_cast<int64_t>(b) * per_row) * V;
    const int64_t id = a.ids[static_cast<int64_t>(b) * a.ids_stride + a.field];
    const bool ok = id >= 0 && id < a.vocab;
    float* dst = a.out + static_cast<int64_t>(b) * a.out_cs + a.out_coff + c;
    if constexpr (V == 4) {
      const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(a.table + id * a.dim + c))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(dst) = v;
    } else {
      *dst = ok ? __ldg(a.table + id * a.dim + c) : 0.f;
    }
  }
  trace_end(trace);
}

struct FirstArgs {
  const int64_t* ids;
  const float* __restrict__ w1;
  const float* __restrict__ wd;
  const float* dense;
  float* out;
  int B, fields, ids_stride, n_dense, dense_stride, out_cs;
  int64_t vocab;
  float bias;
};

// One warp per row: lanes stride over the fields and the dense features.
__global__ void __launch_bounds__(128) first_order(FirstArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; b < a.B; b += warps) {
    float s = 0.f;
    for (int f = lane; f < a.fields; f += 32) {
      const int64_t id = a.ids[static_cast<int64_t>(b) * a.ids_stride + f];
      if (id >= 0 && id < a.vocab) s += __ldg(a.w1 + static_cast<int64_t>(f) * a.vocab + id);
    }
    for (int d = lane; d < a.n_dense; d += 32)
      s = fmaf(a.dense[static_cast<int64_t>(b) * a.dense_stride + d], __ldg(a.wd + d), s);
    s = warp_sum(s);
    if (lane == 0) a.out[static_cast<int64_t>(b) * a.out_cs] = s + a.bias;
  }
  trace_end(trace);
}

struct FmArgs {
  const float* in;
  float* out;
  int B, fields, dim, in_cs, in_coff, out_cs;
};

// One warp per row; lane d < dim accumulates the field sum and the sum of
// squares of embedding dimension d (dim <= 32 per pass, looped above).
__global__ void __launch_bounds__(128) fm_interaction(FmArgs a, unsigned long long* trace) {
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; b < a.B; b += warps) {
    const float* row = a.in + static_cast<int64_t>(b) * a.in_cs + a.in_coff;
    float t = 0.f;
    for (int d = lane; d < a.dim; d += 32) {
      float s = 0.f, q = 0.f;
      for (int f = 0; f < a.fields; ++f) {
        const float v = row[f * a.dim + d];
        s += v;
        q = fmaf(v, v, q);
      }
      t += s * s - q;
    }
    t = warp_sum(t);
    if (lane == 0) a.out[static_cast<int64_t>(b) * a.out_cs] = 0.5f * t;
  }
  trace_end(trace);
}

}  // namespace

opara_status launch_deepfm(const opara_op& op, cudaStream_t s, unsigned long long* trace, LaunchCfg* cfg,
                           bool dry) {
  LaunchCfg c;
  c.block = dim3(128);
  if (op.kind == OPARA_OP_FIELD_EMBEDDING) {
    FieldArgs l;
    l.ids = static_cast<const int64_t*>(op.p[0]);
    l.table = static_cast<const float*>(op.p[1]);
    l.out = static_cast<float*>(op.p[3]);
    l.B = (int)op.i[0]; l.dim = (int)op.i[1]; l.field = (int)op.i[2]; l.ids_stride = (int)op.i[3];
    l.out_cs = (int)op.i[4]; l.out_coff = (int)op.i[5]; l.vocab = op.i[6];
    if (l.B <= 0 || l.dim <= 0 || l.vocab <= 0) return fail(OPARA_ERR_VALUE, "field_embedding: empty shape");
    const bool vec = l.dim % 4 == 0 && l.out_cs % 4 == 0 && l.out_coff % 4 == 0 &&
                     reinterpret_cast<uintptr_t>(l.out) % 16 == 0 && reinterpret_cast<uintptr_t>(l.table) % 16 == 0;
    c.func = vec ? reinterpret_cast<const void*>(&field_embedding<4>) : reinterpret_cast<const void*>(&field_embedding<1>);
    c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(static_cast<int64_t>(l.B) * (l.dim / (vec ? 4 : 1)), 128), 148u)));
    if (cfg) *cfg = c;
    if (dry) return OPARA_OK;
    void* args[] = {&l, &trace};
    return launch_kernel(c, args, s);
  }
  if (op.kind == OPARA_OP_FIRST_ORDER) {
    FirstArgs l;
    l.ids = static_cast<const int64_t*>(op.p[0]);
    l.w1 = static_cast<const float*>(op.p[1]);
    l.wd = static_cast<const float*>(op.p[2]);
    l.dense = static_cast<const float*>(op.p[4]);
    l.out = static_cast<float*>(op.p[3]);
    l.B = (int)op.i[0]; l.fields = (int)op.i[1]; l.ids_stride = (int)op.i[2]; l.n_dense = (int)op.i[3];
    l.dense_stride = (int)op.i[4]; l.vocab = op.i[5]; l.out_cs = (int)op.i[6];
    l.bias = static_cast<float>(op.f[0]);
    if (l.B <= 0) return fail(OPARA_ERR_VALUE, "first_order: empty batch");
    c.func = reinterpret_cast<const void*>(&first_order);
    c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(l.B, 4), 148u)));
    if (cfg) *cfg = c;
    if (dry) return OPARA_OK;
    void* args[] = {&l, &trace};
    return launch_kernel(c, args, s);
  }
  FmArgs l;
  l.in = static_cast<const float*>(op.p[0]);
  l.out = static_cast<float*>(op.p[3]);
  l.B = (int)op.i[0]; l.fields = (int)op.i[1]; l.dim = (int)op.i[2]; l.in_cs = (int)op.i[3];
  l.in_coff = (int)op.i[4]; l.out_cs = (int)op.i[5];
  if (l.B <= 0 || l.fields <= 0 || l.dim <= 0) return fail(OPARA_ERR_VALUE, "fm: empty shape");
  c.func = reinterpret_cast<const void*>(&fm_interaction);
  c.grid = dim3(std::max(1u, std::min<unsigned>(ceil_div(l.B, 4), 148u)));
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&l, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
