// Multi-head self-attention for one sequence, one CTA (16 warps) per head, on tcgen05:
//   S = Q K^T          (tcgen05.mma kind::f16, M = 128 queries, N = 128 keys, K = 64)
//   P = exp((S - max) * scale)   rows in registers straight from TMEM (tcgen05.ld)
//   O = P V / rowsum   (tcgen05.mma, M = 128 queries, N = 64, K = 128 keys)
// Q, K, V and O are channel views of [tokens][C] bf16 buffers (head h reads
// columns off + h*64 ..); S and O accumulate in TMEM (fp32).  Every operand
// lands by TMA (2-D tiled maps, 32-column x 128-row boxes, 64-byte swizzle)
// straight from its natural row layout: Q, K as K-major atoms, V as an
// MN-major operand (8-key x 32-d atoms; descriptor LBO = MN atom stride, SBO =
// 8-key group stride, probed in scripts/micro/umma_mn.cu), so no transpose
// pass; P is written by the softmax warps.  Softmax: the four warps w, w+4, w+8, w+12 share TMEM lane
// quarter w % 4 (query rows 32(w%4)..) and split the 128 keys in quarters;
// row max and row sum are combined through shared memory.  Shapes: tokens =
// 128, head_dim = 64 (BERT-base, seq 128).

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"
#include "tc_common.cuh"
#include "tma_host.h"

namespace opara {
namespace {

constexpr int kT = 128, kD = 64, kThreads = 512, kWarps = kThreads / 32;
constexpr uint32_t kQBytes = kT * kD * 2, kKBytes = kT * kD * 2, kPBytes = kT * kT * 2, kVBytes = kD * kT * 2;

struct AttnArgs {
  CUtensorMap tq, tk, tv;   // 2-D tiled maps of the Q, K, V buffers: 32-column x 128-row boxes, SW64
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* out;
  int q_stride, k_stride, v_stride, out_stride;
  int q_off, k_off, v_off, out_off;
  float scale;
};

// Byte offset of 16-byte chunk `c16` (8 bf16 along K) of `row` in a SW64
// K-major operand with `rows` rows: K is split into 32-element blocks of
// rows * 64 B, each an array of 8-row x 64 B swizzle atoms.
__device__ __forceinline__ uint32_t sw64(int rows, int row, int c16) {
  const int kb = c16 >> 2, cw = c16 & 3, r8 = row & 7;
  return static_cast<uint32_t>(kb * rows * 64 + (row >> 3) * 512 + r8 * 64 + ((cw ^ ((r8 >> 1) & 3)) << 4));
}

// MN-major SW64 V operand as two TMA boxes of 32 head dims x 128 keys: key
// row = 64 B, 8-key atoms 512 B apart along K, the second 32 dims 8 KB on.
constexpr uint32_t kVLbo = kT * 64, kVSbo = 512;   // MN atom stride, 8-key group stride

__device__ __forceinline__ uint64_t desc_mn_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;   // SWIZZLE_64B
  return d;
}

__global__ void __launch_bounds__(kThreads, 1) attention_tc(const __grid_constant__ AttnArgs a,
                                                             unsigned long long* trace) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* qs = smem;
  uint8_t* ks = qs + kQBytes;
  uint8_t* ps = ks + kKBytes;
  uint8_t* vs = ps + kPBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(vs + kVBytes);  // [0] S ready, [1] O ready, [2] Q+K, [3] V landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  __shared__ float red_max[4][kT], red_sum[4][kT];

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x;
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) tc::mbar_init(&bar[b], 1);
    tc::fence_barrier_init();
    tc::prefetch_tmap(&a.tq);
    tc::prefetch_tmap(&a.tk);
    tc::prefetch_tmap(&a.tv);
  }
  if (warp == 0) tc::tmem_alloc(tslot, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;

  pdl_wait();
  trace_begin(trace);
  // ---- Q, K (K-major: two 32-column boxes each) and V (MN-major: two 32-dim
  // boxes) land by TMA; S = Q K^T is issued once Q and K have landed, while V
  // is still on the way
  constexpr uint32_t kIdS = tc::instr_desc(1, 128, 128);
  constexpr uint32_t kIdO = tc::instr_desc(1, 128, 64) | (1u << 16);   // B (V) MN-major
  if (tid == 0) {
    const int qc = a.q_off + h * kD, kc = a.k_off + h * kD, vc = a.v_off + h * kD;
    tc::mbar_arrive_expect_tx(&bar[2], kQBytes + kKBytes);
    tc::tma_tile_2d(qs, &a.tq, qc, 0, &bar[2]);
    tc::tma_tile_2d(qs + kT * 64, &a.tq, qc + 32, 0, &bar[2]);
    tc::tma_tile_2d(ks, &a.tk, kc, 0, &bar[2]);
    tc::tma_tile_2d(ks + kT * 64, &a.tk, kc + 32, 0, &bar[2]);
    tc::mbar_arrive_expect_tx(&bar[3], kVBytes);
    tc::tma_tile_2d(vs, &a.tv, vc, 0, &bar[3]);
    tc::tma_tile_2d(vs + kVLbo, &a.tv, vc + 32, 0, &bar[3]);
    tc::mbar_wait(&bar[2], 0);
    tc::tc_fence_after();
#pragma unroll
    for (int s = 0; s < kD / 16; ++s) {
      const uint32_t off = (s >> 1) * kT * 64 + (s & 1) * 32;
      tc::mma_f16(tS, tc::smem_desc_sw64(tc::smem_u32(qs) + off, 512),
                  tc::smem_desc_sw64(tc::smem_u32(ks) + off, 512), kIdS, s != 0);
    }
    tc::mma_commit(&bar[0]);
  }
  tc::mbar_wait(&bar[0], 0);
  tc::tc_fence_after();

  // ---- softmax: thread = (query row, quarter of the key columns), 32 scores in registers
  const int quarter = warp & 3, kq = warp >> 2;
  const int q = quarter * 32 + lane;
  const uint32_t trow = static_cast<uint32_t>(quarter * 32) << 16;
  constexpr int kQuart = kT / 4;
  float sc[kQuart];
  {
    float v0[16], v1[16];
    tc::tmem_ld16x2(tS + trow + kq * kQuart, tS + trow + kq * kQuart + 16, v0, v1);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      sc[e] = v0[e];
      sc[16 + e] = v1[e];
    }
  }
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < kQuart; ++j) mx = fmaxf(mx, sc[j]);
  red_max[kq][q] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red_max[0][q], red_max[1][q]), fmaxf(red_max[2][q], red_max[3][q]));
  float sum = 0.f;
#pragma unroll
  for (int c16 = 0; c16 < kQuart / 8; ++c16) {
    __nv_bfloat16 pv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float p = __expf((sc[c16 * 8 + e] - mx) * a.scale);
      const __nv_bfloat16 pb = __float2bfloat16_rn(p);
      sum += __bfloat162float(pb);  // normalise by exactly what the PV MMA consumes
      pv[e] = pb;
    }
    *reinterpret_cast<uint4*>(ps + sw64(kT, q, kq * (kQuart / 8) + c16)) = *reinterpret_cast<const uint4*>(pv);
  }
  red_sum[kq][q] = sum;
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  sum = (red_sum[0][q] + red_sum[1][q]) + (red_sum[2][q] + red_sum[3][q]);

  // ---- O = P V
  if (tid == 0) {
    tc::mbar_wait(&bar[3], 0);   // V landed
    tc::tc_fence_after();
#pragma unroll
    for (int s = 0; s < kT / 16; ++s) {
      tc::mma_f16(tO, tc::smem_desc_sw64(tc::smem_u32(ps) + (s >> 1) * kT * 64 + (s & 1) * 32, 512),
                  desc_mn_sw64(tc::smem_u32(vs) + s * 2 * kVSbo, kVLbo, kVSbo), kIdO, s != 0);
    }
    tc::mma_commit(&bar[1]);
  }
  tc::mbar_wait(&bar[1], 0);
  tc::tc_fence_after();
  // thread = (query row, 16 of the 64 head dims)
  const float inv = 1.f / sum;
  float o[16];
  tc::tmem_ld16x1(tO + trow + kq * 16, o);
  __nv_bfloat16 ob[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) ob[e] = __float2bfloat16_rn(o[e] * inv);
  __nv_bfloat16* og = a.out + static_cast<int64_t>(q) * a.out_stride + a.out_off + h * kD + kq * 16;
  reinterpret_cast<uint4*>(og)[0] = reinterpret_cast<const uint4*>(ob)[0];
  reinterpret_cast<uint4*>(og)[1] = reinterpret_cast<const uint4*>(ob)[1];
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 256);
  }
  trace_end(trace);
}

}  // namespace

// ATTENTION  i: 0 tokens (128), 1 heads, 2 head_dim (64), 3 q_stride, 4 k_stride, 5 v_stride,
//               6 out_stride, 7 q_off, 8 k_off, 9 v_off, 10 out_off;  f[0] scale
//            p: 0 q, 1 k, 2 v, 3 out (bf16 [tokens][stride] buffers)
opara_status launch_attention(const opara_op& op, cudaStream_t s, unsigned long long* trace, LaunchCfg* cfg,
                              bool dry) {
  if (op.i[0] != kT || op.i[2] != kD)
    return fail(OPARA_ERR_VALUE, "attention_tc: tokens must be 128 and head_dim 64");
  AttnArgs a;
  a.q = static_cast<const __nv_bfloat16*>(op.p[0]);
  a.k = static_cast<const __nv_bfloat16*>(op.p[1]);
  a.v = static_cast<const __nv_bfloat16*>(op.p[2]);
  a.out = static_cast<__nv_bfloat16*>(op.p[3]);
  a.q_stride = (int)op.i[3]; a.k_stride = (int)op.i[4]; a.v_stride = (int)op.i[5]; a.out_stride = (int)op.i[6];
  a.q_off = (int)op.i[7]; a.k_off = (int)op.i[8]; a.v_off = (int)op.i[9]; a.out_off = (int)op.i[10];
  a.scale = static_cast<float>(op.f[0]);
  for (int x : {a.q_stride, a.k_stride, a.v_stride, a.out_stride, a.q_off, a.k_off, a.v_off, a.out_off})
    if (x % 8) return fail(OPARA_ERR_VALUE, "attention_tc: strides/offsets must be multiples of 8");
  LaunchCfg c;
  c.func = reinterpret_cast<const void*>(&attention_tc);
  c.grid = dim3(static_cast<unsigned>(op.i[1]));
  c.block = dim3(kThreads);
  c.smem = kQBytes + kKBytes + kPBytes + kVBytes + 64 + 1024;
  c.tmem_cols = 256;
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(c.func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(c.smem));
    if (e != cudaSuccess) return cuda_fail(e, "attention_tc smem attribute");
    attr = true;
  }
  if (!make_tiled_bf16_map(&a.tq, a.q, a.q_stride, kT, 32, kT) ||
      !make_tiled_bf16_map(&a.tk, a.k, a.k_stride, kT, 32, kT) ||
      !make_tiled_bf16_map(&a.tv, a.v, a.v_stride, kT, 32, kT))
    return fail(OPARA_ERR_CUDA, "attention_tc: cuTensorMapEncodeTiled failed");
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
