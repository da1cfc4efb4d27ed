// NHWC implicit-GEMM convolution, fp32 SIMT engine (exact fp32 FFMA).
//
//   D[m, n] = sum_k A[m, k] * B[k, n];  m = output pixel, n = output channel,
//   k = (r*S + s)*Cin + c, A gathered from the input on the fly (padding -> 0),
//   B = folded weights [K][Cout].  Epilogue: + folded-BN bias, ReLU, store into
//   the output channel view (concat slice).
//
// Batch-1 layers are small in M (49..12544 pixels), so the launcher spreads
// one conv over a bounded number of CTAs with split-K: every split writes its
// partial tile to a private workspace, and the last split to arrive (per-tile
// arrival counter) reduces the partials in split order — deterministic — and
// runs the epilogue.  The tensor-core engines live in conv_tc.cu.

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct ConvArgs {
  const float* __restrict__ in;
  const float* __restrict__ w;
  const float* __restrict__ bias;
  float* __restrict__ out;      // fp32 output, or bf16 when out_bf16 (bf16 models' fp32-input stems)
  float* __restrict__ ws;       // [splits][M][Cout] partials (split-K only)
  unsigned* __restrict__ cnt;   // per output tile arrival counters (split-K only)
  int N, H, W, Cin, in_cs, in_coff;
  int OH, OW, Cout, out_cs, out_coff;
  int R, S, sh, sw, ph, pw;
  int relu, relu_in, out_bf16;
  int M, K;
  int splits, kt_per_split;
  // input element (b, ih, iw, c) lives at in[b*sN + ih*sH + iw*sW + c*sC + in_coff]
  int64_t sN, sH, sW, sC;
};

constexpr int BK = 16;

template <int BM, int BN, int TM, int TN, bool kVec>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    conv2d_f32_simt(ConvArgs a, unsigned long long* trace) {
  constexpr int T = (BM / TM) * (BN / TN);
  static_assert(T % BK == 0, "thread count must be a multiple of BK");
  // scalar gather: one k lane per thread; vector gather: one 4-channel chunk
  constexpr int A_LANES = kVec ? BK / 4 : BK;
  constexpr int A_ROWS = T / A_LANES;
  constexpr int A_PER = (BM + A_ROWS - 1) / A_ROWS;  // rows past BM idle (small tiles)
  static_assert(BM % A_ROWS == 0 || A_ROWS % BM == 0, "bad A split");
  constexpr int B_PER = BK * BN / T;
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  pdl_trigger();
  pdl_wait();
  trace_begin(trace);  // timeline starts once the inputs are ready (after the PDL wait)

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);

  const int a_lane = tid % A_LANES;
  const int a_row = tid / A_LANES;
  int a_base[A_PER], a_ih0[A_PER], a_iw0[A_PER];
  const int ohw = a.OH * a.OW;
#pragma unroll
  for (int j = 0; j < A_PER; ++j) {
    const int m = m0 + a_row + j * A_ROWS;
    if (m < a.M && a_row + j * A_ROWS < BM) {
      const int b = m / ohw, rem = m - b * ohw;
      const int oh = rem / a.OW, ow = rem - oh * a.OW;
      a_base[j] = b;
      a_ih0[j] = oh * a.sh - a.ph;
      a_iw0[j] = ow * a.sw - a.pw;
    } else {
      a_base[j] = -1;
      a_ih0[j] = 0;
      a_iw0[j] = 0;
    }
  }
  const int b_n = tid % BN;
  const int b_k0 = tid / BN;
  constexpr int B_KSTEP = T / BN;

  constexpr int AV = kVec ? 4 : 1;
  float ra[A_PER][AV], rb[B_PER];
  auto load_tile = [&](int k0) {
    const int k = k0 + a_lane * AV;
    int c = 0, r = 0, s = 0;
    const bool kin = k < a.K;
    if (kin) {
      c = k % a.Cin;
      const int rs = k / a.Cin;
      r = rs / a.S;
      s = rs - r * a.S;
    }
#pragma unroll
    for (int j = 0; j < A_PER; ++j) {
      const int ih = a_ih0[j] + r, iw = a_iw0[j] + s;
      const bool ok = kin && a_base[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
      const float* src = a.in + a_base[j] * a.sN + ih * a.sH + iw * a.sW + c * a.sC + a.in_coff;
      if constexpr (kVec) {
        float4 v = ok ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
        ra[j][0] = v.x; ra[j][1] = v.y; ra[j][2] = v.z; ra[j][3] = v.w;
      } else {
        ra[j][0] = ok ? __ldg(src) : 0.f;
      }
      if (a.relu_in) {  // fused input ReLU
#pragma unroll
        for (int e = 0; e < AV; ++e) ra[j][e] = fmaxf(ra[j][e], 0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < B_PER; ++j) {
      const int kk = k0 + b_k0 + j * B_KSTEP;
      const int n = n0 + b_n;
      rb[j] = (kk < a.K && n < a.Cout) ? __ldg(a.w + static_cast<int64_t>(kk) * a.Cout + n) : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < A_PER; ++j)
      if (a_row + j * A_ROWS < BM)
#pragma unroll
        for (int e = 0; e < AV; ++e) As[buf][a_lane * AV + e][a_row + j * A_ROWS] = ra[j][e];
#pragma unroll
    for (int j = 0; j < B_PER; ++j) Bs[buf][b_k0 + j * B_KSTEP][b_n] = rb[j];
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int ktiles = (a.K + BK - 1) / BK;
  const int kt_begin = blockIdx.z * a.kt_per_split;
  const int kt_end = min(ktiles, kt_begin + a.kt_per_split);
  if (kt_begin < kt_end) {
    load_tile(kt_begin * BK);
    store_tile(0);
    __syncthreads();
    for (int kt = kt_begin; kt < kt_end; ++kt) {
      const int buf = (kt - kt_begin) & 1;
      if (kt + 1 < kt_end) load_tile((kt + 1) * BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (kt + 1 < kt_end) store_tile(buf ^ 1);
      __syncthreads();
    }
  }

  if (a.splits > 1) {
    // publish this split's partial tile, then let the last arrival reduce
    const int64_t plane = static_cast<int64_t>(a.M) * a.Cout;
    float* mine = a.ws + blockIdx.z * plane;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = m0 + ty * TM + i;
      if (m >= a.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = n0 + tx * TN + j;
        if (n < a.Cout) __stcg(mine + static_cast<int64_t>(m) * a.Cout + n, acc[i][j]);
      }
    }
    if (!splitk_arrive_last(a.cnt + blockIdx.x + blockIdx.y * gridDim.x, a.splits)) {
      trace_end(trace);
      return;
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = m0 + ty * TM + i;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = n0 + tx * TN + j;
        float s = 0.f;
        if (m < a.M && n < a.Cout)
          for (int z = 0; z < a.splits; ++z) s += __ldcg(a.ws + z * plane + static_cast<int64_t>(m) * a.Cout + n);
        acc[i][j] = s;
      }
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= a.M) continue;
    float* orow = a.out + static_cast<int64_t>(m) * a.out_cs + a.out_coff;
    __nv_bfloat16* orow_bf = reinterpret_cast<__nv_bfloat16*>(a.out) + static_cast<int64_t>(m) * a.out_cs + a.out_coff;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < a.Cout) {
        float v = acc[i][j] + (a.bias ? __ldg(a.bias + n) : 0.f);
        if (a.relu) v = apply_act(v, a.relu);
        if (a.out_bf16) orow_bf[n] = __float2bfloat16_rn(v);
        else orow[n] = v;
      }
    }
  }
  trace_end(trace);
}

struct Variant {
  int bm, bn;
  const void* func[2];  // [scalar gather, 4-channel vector gather]
  int threads;
};

template <int BM, int BN, int TM, int TN>
Variant make_variant() {
  return {BM, BN,
          {reinterpret_cast<const void*>(&conv2d_f32_simt<BM, BN, TM, TN, false>),
           reinterpret_cast<const void*>(&conv2d_f32_simt<BM, BN, TM, TN, true>)},
          (BM / TM) * (BN / TN)};
}

const Variant* variants(int* count) {
  static const Variant v[] = {
      make_variant<64, 64, 4, 4>(),   // 0
      make_variant<32, 64, 2, 4>(),   // 1
      make_variant<64, 32, 4, 2>(),   // 2
      make_variant<32, 32, 2, 2>(),   // 3
      make_variant<128, 64, 8, 4>(),  // 4
      make_variant<16, 64, 1, 4>(),   // 5
  };
  *count = static_cast<int>(sizeof(v) / sizeof(v[0]));
  return v;
}

struct Choice {
  int id, splits, kt_per_split;
};

// Latency-first tiling for one branch: largest tile whose grid, after
// split-K, reaches `target` CTAs while every split keeps >= 4 k-tiles.
Choice auto_choice(int64_t M, int64_t N, int64_t K, int64_t target) {
  int count = 0;
  const Variant* v = variants(&count);
  const int64_t ktiles = (K + BK - 1) / BK;
  const int prefs[] = {4, 0, 1, 2, 3, 5};
  Choice best{3, 1, static_cast<int>(ktiles)};
  double best_cost = 1e30;
  for (int id : prefs) {
    const int64_t base = ((M + v[id].bm - 1) / v[id].bm) * ((N + v[id].bn - 1) / v[id].bn);
    int64_t splits = std::max<int64_t>(1, (target + base - 1) / base);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, ktiles / 4));
    splits = std::min<int64_t>(splits, 32);
    const int64_t kps = (ktiles + splits - 1) / splits;
    splits = (ktiles + kps - 1) / kps;
    const int64_t ctas = base * splits;
    // cost model: waves of one CTA's k-loop over a 148-SM, 2-CTA/SM machine,
    // plus a reduction term when split
    const double waves = std::ceil(static_cast<double>(ctas) / (148.0 * 2.0));
    const double per_cta = static_cast<double>(kps) * v[id].bm * v[id].bn;
    const double cost = waves * per_cta * 1.0 + (splits > 1 ? 0.15 * splits * v[id].bm * v[id].bn : 0.0) +
                        2000.0 * splits;  // fixed overhead per split pass
    if (cost < best_cost) {
      best_cost = cost;
      best = {id, static_cast<int>(splits), static_cast<int>(kps)};
    }
  }
  return best;
}

}  // namespace

opara_status launch_conv2d(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                           LaunchCfg* cfg, bool dry) {
  ConvArgs a;
  a.in = static_cast<const float*>(op.p[0]);
  a.w = static_cast<const float*>(op.p[1]);
  a.bias = static_cast<const float*>(op.p[2]);
  a.out = static_cast<float*>(op.p[3]);
  a.N = (int)op.i[0]; a.H = (int)op.i[1]; a.W = (int)op.i[2]; a.Cin = (int)op.i[3];
  a.in_cs = (int)op.i[4]; a.in_coff = (int)op.i[5];
  a.OH = (int)op.i[6]; a.OW = (int)op.i[7]; a.Cout = (int)op.i[8];
  a.out_cs = (int)op.i[9]; a.out_coff = (int)op.i[10];
  a.R = (int)op.i[11]; a.S = (int)op.i[12]; a.sh = (int)op.i[13]; a.sw = (int)op.i[14];
  a.ph = (int)op.i[15]; a.pw = (int)op.i[16];
  a.relu = conv_act_code(op.i[24], op.i[17]);   // `relu` carries the activation code
  a.relu_in = (int)op.i[25];
  a.out_bf16 = op.i[23] == 1 ? 1 : 0;   // record i[23]: output dtype (0 fp32, 1 bf16)
  if (op.i[18] != 0) return fail(OPARA_ERR_VALUE, "conv2d simt engine: fp32 input only");
  a.M = a.N * a.OH * a.OW;
  a.K = a.R * a.S * a.Cin;
  const bool nchw = op.i[20] != 0;
  if (nchw) {  // dense NCHW input
    a.sC = static_cast<int64_t>(a.H) * a.W;
    a.sW = 1;
    a.sH = a.W;
    a.sN = a.sC * a.Cin;
    a.in_coff = 0;
  } else {
    a.sC = 1;
    a.sW = a.in_cs;
    a.sH = static_cast<int64_t>(a.W) * a.in_cs;
    a.sN = a.sH * a.H;
  }
  if (a.M <= 0 || a.Cout <= 0 || a.K <= 0) return fail(OPARA_ERR_VALUE, "conv2d: empty shape");
  int count = 0;
  const Variant* v = variants(&count);
  const int64_t target = op.i[21] > 0 ? op.i[21] : 296;
  Choice ch = auto_choice(a.M, a.Cout, a.K, target);
  if (op.variant >= 0 && op.variant < count) {
    ch.id = op.variant;
    ch.splits = op.i[19] > 1 ? static_cast<int>(op.i[19]) : 1;
    const int ktiles = (a.K + BK - 1) / BK;
    ch.kt_per_split = (ktiles + ch.splits - 1) / ch.splits;
    ch.splits = (ktiles + ch.kt_per_split - 1) / ch.kt_per_split;
  }
  a.splits = ch.splits;
  a.kt_per_split = ch.kt_per_split;
  const bool vec = !nchw && a.Cin % 4 == 0 && a.in_cs % 4 == 0 && a.in_coff % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(a.in) % 16 == 0;
  LaunchCfg c;
  c.func = v[ch.id].func[vec ? 1 : 0];
  c.grid = dim3(ceil_div(a.M, v[ch.id].bm), ceil_div(a.Cout, v[ch.id].bn), ch.splits);
  c.block = dim3(v[ch.id].threads, 1, 1);
  c.smem = 0;
  const int64_t tiles = static_cast<int64_t>(c.grid.x) * c.grid.y;
  c.workspace = ch.splits > 1 ? splitk_workspace_bytes(static_cast<int64_t>(a.M) * a.Cout * ch.splits, tiles) : 0;
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  if (ch.splits > 1) {
    if (!op.p[7]) return fail(OPARA_ERR_INTERNAL, "conv2d: split-K workspace missing");
    a.ws = static_cast<float*>(op.p[7]);
    a.cnt = splitk_counters(op.p[7], static_cast<int64_t>(a.M) * a.Cout * ch.splits);
  } else {
    a.ws = nullptr;
    a.cnt = nullptr;
  }
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s);
}

}  // namespace opara
