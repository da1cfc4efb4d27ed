// NHWC implicit-GEMM convolution, fp32 SIMT engine (exact fp32 FFMA).
//
//   D[m, n] = sum_k A[m, k] * B[k, n];  m = output pixel, n = output channel,
//   k = (r*S + s)*Cin + c, A gathered from the input on the fly (padding -> 0),
//   B = folded weights [K][Cout].  Epilogue: + folded-BN bias, ReLU, store into
//   the output channel view (concat slice).
//
// This is the exact-fp32 engine used for the fp32 parity configs; the tensor-
// core (tcgen05) engines live in conv_tc.cu.  Grids are bounded by the tile
// choice so independent branches can co-reside.

#include "device_common.cuh"
#include "ops.h"
#include "status.h"

namespace opara {
namespace {

struct ConvArgs {
  const float* __restrict__ in;
  const float* __restrict__ w;
  const float* __restrict__ bias;
  float* __restrict__ out;
  int N, H, W, Cin, in_cs, in_coff;
  int OH, OW, Cout, out_cs, out_coff;
  int R, S, sh, sw, ph, pw;
  int relu;
  int M, K;
  // input element (b, ih, iw, c) lives at in[b*sN + ih*sH + iw*sW + c*sC + in_coff]
  int64_t sN, sH, sW, sC;
};

constexpr int BK = 16;

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    conv2d_f32_simt(ConvArgs a, unsigned long long* trace) {
  constexpr int T = (BM / TM) * (BN / TN);
  static_assert(T % BK == 0, "thread count must be a multiple of BK");
  constexpr int A_PER = BM * BK / T;
  constexpr int B_PER = BK * BN / T;
  constexpr int A_ROWS = T / BK;  // m rows covered per pass
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  trace_begin(trace);

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);

  // Per-thread A gather coordinates: fixed k lane, A_PER output pixels.
  const int a_k = tid % BK;
  int a_base[A_PER], a_ih0[A_PER], a_iw0[A_PER];
  const int ohw = a.OH * a.OW;
#pragma unroll
  for (int j = 0; j < A_PER; ++j) {
    const int m = m0 + tid / BK + j * A_ROWS;
    if (m < a.M) {
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

  float ra[A_PER], rb[B_PER];
  auto load_tile = [&](int k0) {
    const int k = k0 + a_k;
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
      float v = 0.f;
      if (kin && a_base[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W)
        v = __ldg(a.in + a_base[j] * a.sN + ih * a.sH + iw * a.sW + c * a.sC + a.in_coff);
      ra[j] = v;
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
    for (int j = 0; j < A_PER; ++j) As[buf][a_k][tid / BK + j * A_ROWS] = ra[j];
#pragma unroll
    for (int j = 0; j < B_PER; ++j) Bs[buf][b_k0 + j * B_KSTEP][b_n] = rb[j];
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int ktiles = (a.K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
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
    if (kt + 1 < ktiles) store_tile(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= a.M) continue;
    float* orow = a.out + static_cast<int64_t>(m) * a.out_cs + a.out_coff;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < a.Cout) {
        float v = acc[i][j] + (a.bias ? __ldg(a.bias + n) : 0.f);
        if (a.relu) v = fmaxf(v, 0.f);
        orow[n] = v;
      }
    }
  }
  trace_end(trace);
}

struct Variant {
  int bm, bn;
  const void* func;
  int threads;
};

template <int BM, int BN, int TM, int TN>
Variant make_variant() {
  return {BM, BN, reinterpret_cast<const void*>(&conv2d_f32_simt<BM, BN, TM, TN>),
          (BM / TM) * (BN / TN)};
}

const Variant* variants(int* count) {
  static const Variant v[] = {
      make_variant<64, 64, 4, 4>(),  // 0
      make_variant<32, 64, 2, 4>(),  // 1
      make_variant<64, 32, 4, 2>(),  // 2
      make_variant<32, 32, 2, 2>(),  // 3  (256 threads, 2x2 micro tiles)
      make_variant<128, 64, 8, 4>(), // 4
      make_variant<16, 64, 1, 4>(),  // 5
  };
  *count = static_cast<int>(sizeof(v) / sizeof(v[0]));
  return v;
}

// Pick the largest tile that still yields enough CTAs to spread one branch
// over a bounded share of the 148 SMs.
int auto_variant(int64_t M, int64_t N) {
  int count = 0;
  const Variant* v = variants(&count);
  const int prefs[] = {4, 0, 1, 2, 3, 5};
  for (int id : prefs) {
    const int64_t ctas = ((M + v[id].bm - 1) / v[id].bm) * ((N + v[id].bn - 1) / v[id].bn);
    if (ctas >= 96) return id;
  }
  return M <= 16 ? 5 : 3;
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
  a.ph = (int)op.i[15]; a.pw = (int)op.i[16]; a.relu = (int)op.i[17];
  if (op.i[18] != 0) return fail(OPARA_ERR_VALUE, "conv2d simt engine: fp32 only");
  a.M = a.N * a.OH * a.OW;
  a.K = a.R * a.S * a.Cin;
  if (op.i[20]) {  // dense NCHW input
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
  int id = op.variant;
  if (id < 0 || id >= count) id = auto_variant(a.M, a.Cout);
  LaunchCfg c;
  c.func = v[id].func;
  c.grid = dim3(ceil_div(a.M, v[id].bm), ceil_div(a.Cout, v[id].bn), 1);
  c.block = dim3(v[id].threads, 1, 1);
  c.smem = 0;
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  void* args[] = {&a, &trace};
  return cuda_fail(cudaLaunchKernel(c.func, c.grid, c.block, args, c.smem, s), "conv2d launch");
}

}  // namespace opara
