// bf16 NHWC implicit-GEMM convolution / linear layer on tcgen05 (kind::f16,
// bf16 operands, fp32 accumulation in TMEM).  Same GEMM view as the 3xTF32
// engine (conv_tc.cu): weights on M (128 output channels per tile), output
// pixels (or tokens, for a linear layer = 1x1 conv over a [tokens][K] map) on
// N = BN, k = (r*S + s)*Cin + c.
//
// One pass, one operand plane each, so the ring is deeper and lighter:
//   warps 0-3  gather: im2col with cp.async (16 B = 8 bf16 channels, zero-fill
//              for padding) into 64-byte-swizzled K-major atoms; completion is
//              signalled straight onto the stage's `full` mbarrier
//              (cp.async.mbarrier.arrive.noinc).  Inputs that are not 8-channel
//              aligned (stems, the fp32 NCHW graph input) take a register path
//              that converts to bf16 and arrives after fence.proxy.async;
//   warp 4     weight loader: one cp.async.bulk of the host-packed 8 KB W block;
//   warp 5     MMA issuer: 2 x tcgen05.mma (K = 16) per 32-wide k step.
// Epilogue as in conv_tc.cu: TMEM -> smem tile -> (cluster split-K DSMEM
// reduction in rank order) -> + bias, activation (none/ReLU/GELU-erf), store
// bf16 or fp32 into the output channel view.

#include <cuda_bf16.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "device_common.cuh"
#include "ops.h"
#include "status.h"
#include "tc_common.cuh"
#include "tma_host.h"

namespace opara {
namespace {

// Diagnostic build only (-DOPARA_PHASE_PROBE): CTA (0,0,0) of every launch
// records %globaltimer at entry, after griddepcontrol.wait, first / last MMA
// issue, accumulator ready and exit, read back by opara_debug_phase_read.
#ifdef OPARA_PHASE_PROBE
__device__ unsigned long long g_phase[4096][12];
__device__ unsigned g_phase_n;
#define PHASE(k)                                                              \
  do {                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ph[k] = global_ns(); \
  } while (0)
#define PHASE_FLUSH()                                                                               \
  do {                                                                                              \
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {                        \
      ph[7] = global_ns();                                                                          \
      const unsigned slot = atomicAdd(&g_phase_n, 1u) & 4095u;                                      \
      for (int q = 0; q < 8; ++q) g_phase[slot][q] = ph[q];                                         \
      g_phase[slot][10] = ph[8];                                                                    \
      g_phase[slot][11] = ph[9];                                                                    \
      g_phase[slot][8] = (static_cast<unsigned long long>(a.M) << 40) | (static_cast<unsigned long long>(a.Cout) << 20) | a.K; \
      g_phase[slot][9] = (static_cast<unsigned long long>(gridDim.x * gridDim.y * gridDim.z) << 32) | (static_cast<unsigned long long>(BN) << 24) | (nkb << 8) | (a.push ? 0x80 : 0) | (a.l2red ? 0x40 : 0) | (a.ln_in ? 0x20 : 0) | (a.res_stats ? 0x10 : 0) | a.splits; \
    }                                                                                               \
  } while (0)
#else
#define PHASE(k) \
  do {           \
  } while (0)
#define PHASE_FLUSH() \
  do {                \
  } while (0)
#endif

constexpr int kBK = 32;                     // bf16 k elements per stage (64 B rows)
constexpr int kGatherWarps = 4;
constexpr int kLoadWarp = 4, kMmaWarp = 5;
constexpr int kXWarp = 6;          // folded-LayerNorm consumers: issues the o + r TMA tiles
constexpr int kMaxLnTiles = 8;     // folded LayerNorm: channels <= 1024
constexpr int kThreads = 224;      // (a 7th warp measured neutral on the CNNs, BERT 0.440 -> 0.430 ms vs sharing a gather warp)
constexpr int kMaxSplits = 8;
constexpr int kPushMaxKB = 48;   // split-K push receive buffer limit (KB of smem beyond the ring)
constexpr uint32_t kWBytes = 128 * kBK * 2;  // 8 KB

// Ring depth per tile width.  The 16-wide tile keeps a 24-deep ring (216 KB):
// one CTA per SM can hold a whole K = 768 weight slice, all of it fetched
// before griddepcontrol.wait (weights do not depend on the predecessor), so
// after the wait only the small activation tile is on the critical path.
__host__ __device__ constexpr int bf_stages(int bn) { return bn == 16 ? 24 : bn <= 64 ? 8 : 6; }
// full[], empty[], accum, tmem slot, push barrier, landed[], LayerNorm stats: rounded up to 128 bytes
__host__ __device__ constexpr int bf_bar_bytes(int stages) { return ((3 * stages + 4) * 8 + 127) / 128 * 128; }

// kVecBf16: 16-byte cp.async of 8 channels (Cin % 8 == 0); kSub4 / kSub2: each
// 16-byte smem chunk assembled from 8- / 4-byte cp.asyncs of 4 / 2 channels
// (Cin % 4 / % 2 == 0, e.g. NASNet's 84 / 42 channels), every sub-chunk with
// its own incrementally tracked (r, s, c); scalar register paths otherwise.
// kTma: one thread loads each stage's X tile with a TMA im2col load (bf16
// input, Cin % 32 == 0, 16-byte aligned view, no fused input ReLU).
enum GatherMode { kVecBf16 = 0, kScalarBf16 = 1, kScalarF32 = 2, kSub4 = 3, kSub2 = 4, kTma = 5 };
constexpr int kModes = 6;

__device__ __forceinline__ void cp_async_sub(uint32_t dst, const void* src, int bytes, bool ok) {
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}

struct BfArgs {
  CUtensorMap tmap;                         // im2col map of the input view (kTma only)
  CUtensorMap tmap_r;                       // map of the LayerNorm residual view (ln_in only)
  const void* in;
  const __nv_bfloat16* __restrict__ wpack;  // [m_tiles][kblocks][atom][row][chunk][8]
  const float* __restrict__ bias;
  void* out;
  int N, H, W, Cin, in_coff;
  int OH, OW, Cout, out_cs, out_coff;
  int R, S, sh, sw, ph, pw;
  int act, vec_out, relu_in;
  int M, K, kblocks;
  int splits, kb_per_split;
  int push, rows_per;   // split-K reduction: 1 = partials pushed to the owner CTA (st.async)
  int l2red;            // split-K reduction through L2 (partial tiles in `ws`, one cluster barrier)
  float* ws;
  const int4* ktab;     // scalar gathers: per k (dr, dq, input offset) from the host (no divisions)
  int64_t sN, sH, sW, sC;
  // Folded LayerNorm y = LN(o + r) (frontend.PendingLN).  Producer GEMM
  // (res_stats): stores o = bf16(acc + bias) as usual and, per token, the sum
  // and sum of squares of o + r (fp32, r = the bf16 residual view) over this
  // CTA's 128 channels into stats_out[token][m-tile][2].  Consumer GEMM
  // (ln_in): the X warp lands the o and r tiles of every stage; the gather
  // warps form (o + r - mean) * rstd * gamma + beta in place (the same
  // roundings as the unfolded LayerNorm kernel) before the MMA reads it; lnout
  // (first consumer, m-tile 0 CTAs) receives the normalised rows.
  int res_stats, res_cs;
  const __nv_bfloat16* res;
  float* stats_out;
  int ln_in, ln_tiles, lnout_cs;
  const float* stats_in;
  const float* gb;          // [2][Cin]: gamma, beta
  __nv_bfloat16* lnout;
  float eps;
  uint32_t r_off;           // smem byte offset of the residual tiles (kStages x BN x 64 B), then mean / rstd [BN]
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ float act_fn(float v, int act) {
  if (act == 1) return fmaxf(v, 0.f);
  if (act == 2) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
  if (act == 3) return tanhf(v);
  return v;
}

template <int BN, int kMode, typename TO>
__global__ void __launch_bounds__(kThreads, 1) conv2d_tc_bf16(const __grid_constant__ BfArgs a, unsigned long long* trace) {
  constexpr int kStages = bf_stages(BN);
  constexpr uint32_t kXBytes = BN * kBK * 2;
  constexpr uint32_t kStage = kWBytes + kXBytes;
  constexpr uint32_t kSbo = 512;
  constexpr int kRowGroups = BN / 8;
  constexpr int kRowsPerThread = (kRowGroups + 3) / 4;
  constexpr uint32_t kIdesc = tc::instr_desc(1, 128, BN);
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  static_assert(BN * 128 * 4 <= kStages * kStage, "epilogue tile must fit in the pipeline smem");
  static_assert(kPushMaxKB * 1024 <= kStages * kStage, "push staging blocks must fit in the pipeline smem");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint64_t* empty = full + kStages;
  uint64_t* accum = empty + kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accum + 1);

  pdl_trigger();
#ifdef OPARA_PHASE_PROBE
  __shared__ unsigned long long ph[10];
  if (threadIdx.x < 10) ph[threadIdx.x] = 0;
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) PHASE(0);
  const int n0 = blockIdx.x * BN;
  const int mt = blockIdx.y;
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int nkb = min(a.kblocks, kb0 + a.kb_per_split) - kb0;
  // the pull epilogue's bias (lane = 4 channels) is a parameter: fetch it now,
  // before griddepcontrol.wait, so its latency hides under the predecessor
  const int ch = mt * 128 + lane * 4;
  float bias[4] = {0.f, 0.f, 0.f, 0.f};
  if (a.bias && !a.push) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (ch + e < a.Cout) bias[e] = __ldg(a.bias + ch + e);
  }
  // the push epilogue's owner reduction: thread = output channel
  const float push_bias = ((a.push || a.splits > 1) && a.bias && tid < 128 && mt * 128 + tid < a.Cout) ? __ldg(a.bias + mt * 128 + tid) : 0.f;

  // push-mode split-K: receive buffer [src rank][128 channels][rows_per columns]
  // fp32 behind the ring (other CTAs may push while this CTA's ring is busy)
  uint64_t* rbar = accum + 2;
  uint64_t* landed = rbar + 1;   // TMA tile landed (folded-LayerNorm consumers: normalised before full[])
  uint64_t* statbar = landed + kStages;   // folded-LayerNorm consumers: per-token mean / rstd in smem
  float* recv = reinterpret_cast<float*>(smem + kStages * kStage + bf_bar_bytes(kStages));
  const bool push = a.push != 0;
  const bool ln_in = kMode == kTma && a.ln_in;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      // gather threads (or the TMA thread's expect_tx arrive, or the normalising
      // threads after it) + the weight loader
      tc::mbar_init(&full[s], kMode == kTma ? (ln_in ? 32 + 1 : 2) : 32 * kGatherWarps + 1);
      tc::mbar_init(&empty[s], 1);
      if (ln_in) tc::mbar_init(&landed[s], 1);
    }
    if (ln_in) tc::mbar_init(statbar, 32 * kGatherWarps);
    tc::mbar_init(accum, 1);
    if (push) tc::mbar_init(rbar, 1);
    tc::fence_barrier_init();
  }
  constexpr int kTmemWarp = kMmaWarp;   // the MMA warp is idle in every epilogue: it frees TMEM off the critical path
  if (warp == kTmemWarp) tc::tmem_alloc(tslot, kTmemCols);   // (and frees them: an epilogue-idle warp)
  tc::tc_fence_before();
  if (push) {
    // every CTA's receive barrier is initialised before anyone pushes (this
    // runs before griddepcontrol.wait, overlapping the predecessor kernel)
    tc::cluster_sync();
    if (tid == 0) {
      // every rank bulk-copies one whole [128][rows_per] block to each owner
      const int r0 = static_cast<int>(tc::cluster_ctarank()) * a.rows_per;
      // every other rank's block; the owner's own partial stays in its ring
      if (r0 < BN) tc::mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((a.splits - 1) * a.rows_per * 128 * 4));
    }
  } else {
    __syncthreads();
  }
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp < kGatherWarps) {
    // ------------------------------------------------------------ gather
    const int rw = warp, r8 = lane & 7, cl = lane >> 3;
    auto x_off = [&](int j) -> uint32_t {
      return static_cast<uint32_t>(rw + 4 * j) * kSbo + r8 * 64u +
             static_cast<uint32_t>((cl ^ ((r8 >> 1) & 3)) * 16);
    };
    int pb[kRowsPerThread], pih[kRowsPerThread], piw[kRowsPerThread];
    const int ohw = a.OH * a.OW;
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j) {
      const int p = n0 + (rw + 4 * j) * 8 + r8;
      if (rw + 4 * j < kRowGroups && p < a.M) {
        const int b = p / ohw, rem = p - b * ohw, oh = rem / a.OW, ow = rem - oh * a.OW;
        pb[j] = b;
        pih[j] = oh * a.sh - a.ph;
        piw[j] = ow * a.sw - a.pw;
      } else {
        pb[j] = -1;
        pih[j] = 0;
        piw[j] = 0;
      }
    }
    // folded-LayerNorm consumers: gamma / beta of this warp's first stage are
    // parameters — fetched before griddepcontrol.wait, beside the predecessor
    float4 ln_g0 = make_float4(0.f, 0.f, 0.f, 0.f), ln_g1 = ln_g0, ln_b0 = ln_g0, ln_b1 = ln_g0;
    if (ln_in && rw < nkb) {
      const int c0 = (kb0 + rw) * kBK + (lane & 3) * 8;
      const float4* g4 = reinterpret_cast<const float4*>(a.gb + c0);
      const float4* b4 = reinterpret_cast<const float4*>(a.gb + a.Cin + c0);
      ln_g0 = __ldg(g4);
      ln_g1 = __ldg(g4 + 1);
      ln_b0 = __ldg(b4);
      ln_b1 = __ldg(b4 + 1);
    }
    if (kMode == kTma && tid == 0 && !ln_in) tc::prefetch_tmap(&a.tmap);
    pdl_wait();
    trace_begin(trace);
    if (tid == 0) PHASE(1);
    // Fused input ReLU (relu_in): the copies of stage i are committed as one
    // cp.async group; once stage i-1's group has landed this thread clamps
    // its own chunks of it in place (bf16 max with 0), fences them into the
    // async proxy and arrives, so the transform trails the gather by a stage.
    auto relu_stage = [&](int st) {
      uint8_t* xs_g = smem + st * kStage + kWBytes;
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j) {
        if (rw + 4 * j >= kRowGroups) break;
        uint4* q = reinterpret_cast<uint4*>(xs_g + x_off(j));
        uint4 v = *q;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
        const __nv_bfloat162 z = __float2bfloat162_rn(0.f);
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __hmax2(h[e], z);
        *q = v;
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&full[st]);
    };
    if constexpr (kMode == kTma) {
      // k = (r*S + s)*Cin + c with Cin % 32 == 0: every stage is one tap's
      // 32-channel slice of BN output pixels; padding and the tile tail are zeros
      if (ln_in) {
        // Folded LayerNorm on load (1x1 row GEMMs: k = channel).  The X warp
        // lands each stage's o and r tiles on landed[]; gather warp w
        // normalises whole stages i = w (mod 4) in place — four stages in
        // flight, one warp each — and releases full[].  Lane l owns chunk
        // l % 4 (8 channels) of rows l / 4, l / 4 + 8, ...  Per-token mean and
        // rstd (from the producer's partial sums, summed in m-tile order) are
        // computed once into smem (behind the residual tiles).
        float* ln_mean = reinterpret_cast<float*>(smem + a.r_off + kStages * kXBytes);
        float* ln_rstd = ln_mean + BN;
        for (int row = tid; row < BN; row += 32 * kGatherWarps) {
          const int p = n0 + row;
          float s1 = 0.f, s2 = 0.f;
          if (p < a.M) {
            const float2* st = reinterpret_cast<const float2*>(a.stats_in) + static_cast<int64_t>(p) * a.ln_tiles;
            float2 v[kMaxLnTiles];   // every partial's load in flight
#pragma unroll
            for (int t = 0; t < kMaxLnTiles; ++t)
              if (t < a.ln_tiles) v[t] = __ldcg(st + t);
#pragma unroll
            for (int t = 0; t < kMaxLnTiles; ++t)
              if (t < a.ln_tiles) {
                s1 += v[t].x;
                s2 += v[t].y;
              }
          }
          const float mu = s1 / a.Cin;
          ln_mean[row] = mu;
          ln_rstd[row] = rsqrtf(fmaxf(s2 / a.Cin - mu * mu, 0.f) + a.eps);
        }
        // every gather thread has published its rows' statistics (an mbarrier
        // among the gather warps only; the other warps never wait on it)
        tc::mbar_arrive(statbar);
        tc::mbar_wait(statbar, 0);
        const int c4 = lane & 3, rl = lane >> 2;
        const bool write = a.lnout && mt == 0;
        for (int i = rw; i < nkb; i += kGatherWarps) {
          const int s = i % kStages;
          const int c0 = (kb0 + i) * kBK + c4 * 8;   // this lane's 8 channels
          const float4* g4 = reinterpret_cast<const float4*>(a.gb + c0);
          const float4* b4 = reinterpret_cast<const float4*>(a.gb + a.Cin + c0);
          const bool first = i == rw;   // prefetched before the PDL wait
          const float4 ga = first ? ln_g0 : __ldg(g4), gb2 = first ? ln_g1 : __ldg(g4 + 1);
          const float4 ba = first ? ln_b0 : __ldg(b4), bb = first ? ln_b1 : __ldg(b4 + 1);
          const float g[8] = {ga.x, ga.y, ga.z, ga.w, gb2.x, gb2.y, gb2.z, gb2.w};
          const float b[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
          tc::mbar_wait(&landed[s], (i / kStages) & 1);
          uint8_t* xs = smem + s * kStage + kWBytes;
          const uint8_t* rs = smem + a.r_off + s * kXBytes;
#pragma unroll 4
          for (int row = rl; row < BN; row += 8) {
            const int r8 = row & 7;
            const uint32_t off = static_cast<uint32_t>(row >> 3) * kSbo + r8 * 64u +
                                 static_cast<uint32_t>((c4 ^ ((r8 >> 1) & 3)) * 16);
            uint4 v = *reinterpret_cast<const uint4*>(xs + off);
            const uint4 rv = *reinterpret_cast<const uint4*>(rs + off);
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&v);
            const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
            const float mu = ln_mean[row], rsd = ln_rstd[row];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h2[e]), fr = __bfloat1622float2(r2[e]);
              h2[e] = __floats2bfloat162_rn((f.x + fr.x - mu) * rsd * g[2 * e] + b[2 * e],
                                            (f.y + fr.y - mu) * rsd * g[2 * e + 1] + b[2 * e + 1]);
            }
            *reinterpret_cast<uint4*>(xs + off) = v;
            if (write && n0 + row < a.M)
              *reinterpret_cast<uint4*>(a.lnout + static_cast<int64_t>(n0 + row) * a.lnout_cs + c0) = v;
          }
          tc::fence_proxy_async_smem();
          tc::mbar_arrive(&full[s]);
        }
      } else if (tid == 0) {
        const int ohw = a.OH * a.OW;
        const int b = n0 / ohw, rem = n0 - b * ohw, oh = rem / a.OW, ow = rem - oh * a.OW;
        const int w0 = ow * a.sw - a.pw, h0 = oh * a.sh - a.ph;
        const int kc = kb0 * kBK, rs = kc / a.Cin;
        int dc = kc - rs * a.Cin, dr = rs / a.S, dq = rs - dr * a.S;
        for (int i = 0; i < nkb; ++i) {
          const int s = i % kStages;
          if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
          tc::mbar_arrive_expect_tx(&full[s], kXBytes);
          tc::tma_im2col_4d(smem + s * kStage + kWBytes, &a.tmap, dc, w0, h0, b, dq, dr, &full[s]);
          dc += kBK;
          if (dc == a.Cin) {
            dc = 0;
            if (++dq == a.S) {
              dq = 0;
              ++dr;
            }
          }
        }
      }
    } else if constexpr (kMode == kVecBf16) {
      const __nv_bfloat16* in = static_cast<const __nv_bfloat16*>(a.in);
      const __nv_bfloat16* rowbase[kRowsPerThread];
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j)
        rowbase[j] = in + (pb[j] >= 0 ? pb[j] * a.sN + pih[j] * a.sH + piw[j] * a.sW + a.in_coff : 0);
      int kc = kb0 * kBK + cl * 8, dc = 0, dr = 0, dq = 0;
      if (kc < a.K) {
        dc = kc % a.Cin;
        const int rs = kc / a.Cin;
        dr = rs / a.S;
        dq = rs - dr * a.S;
      }
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        const uint32_t xs = tc::smem_u32(smem + s * kStage + kWBytes);
        const bool kin = kc < a.K;
        const int64_t koff = dr * a.sH + dq * a.sW + dc;
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
          const int ih = pih[j] + dr, iw = piw[j] + dq;
          const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
          if (rw + 4 * j < kRowGroups) cp_async16(xs + x_off(j), ok ? rowbase[j] + koff : in, ok);
        }
        if (a.relu_in) {
          cp_async_commit();
          if (i > 0) {
            cp_async_wait<1>();
            relu_stage((i - 1) % kStages);
          }
        } else {
          tc::cp_async_arrive_noinc(&full[s]);
        }
        kc += kBK;
        dc += kBK;
        while (dc >= a.Cin) {
          dc -= a.Cin;
          if (++dq == a.S) {
            dq = 0;
            ++dr;
          }
        }
      }
      if (a.relu_in && nkb > 0) {
        cp_async_wait<0>();
        relu_stage((nkb - 1) % kStages);
      }
    } else if constexpr (kMode == kSub4 || kMode == kSub2) {
      constexpr int G = kMode == kSub4 ? 4 : 2;   // channels per cp.async
      constexpr int NS = 8 / G;                   // sub-chunks per 16-byte chunk
      const __nv_bfloat16* in = static_cast<const __nv_bfloat16*>(a.in);
      const __nv_bfloat16* rowbase[kRowsPerThread];
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j)
        rowbase[j] = in + (pb[j] >= 0 ? pb[j] * a.sN + pih[j] * a.sH + piw[j] * a.sW + a.in_coff : 0);
      int kc[NS], dc[NS], dr[NS], dq[NS];
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        kc[u] = kb0 * kBK + cl * 8 + u * G;
        dc[u] = dr[u] = dq[u] = 0;
        if (kc[u] < a.K) {
          dc[u] = kc[u] % a.Cin;
          const int rs = kc[u] / a.Cin;
          dr[u] = rs / a.S;
          dq[u] = rs - dr[u] * a.S;
        }
      }
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        const uint32_t xs = tc::smem_u32(smem + s * kStage + kWBytes);
#pragma unroll
        for (int u = 0; u < NS; ++u) {
          const bool kin = kc[u] < a.K;
          const int64_t koff = dr[u] * a.sH + dq[u] * a.sW + dc[u];
#pragma unroll
          for (int j = 0; j < kRowsPerThread; ++j) {
            const int ih = pih[j] + dr[u], iw = piw[j] + dq[u];
            const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
            if (rw + 4 * j < kRowGroups) cp_async_sub(xs + x_off(j) + u * G * 2, ok ? rowbase[j] + koff : in, G * 2, ok);
          }
          kc[u] += kBK;
          dc[u] += kBK;
          while (dc[u] >= a.Cin) {
            dc[u] -= a.Cin;
            if (++dq[u] == a.S) {
              dq[u] = 0;
              ++dr[u];
            }
          }
        }
        if (a.relu_in) {
          cp_async_commit();
          if (i > 0) {
            cp_async_wait<1>();
            relu_stage((i - 1) % kStages);
          }
        } else {
          tc::cp_async_arrive_noinc(&full[s]);
        }
      }
      if (a.relu_in && nkb > 0) {
        cp_async_wait<0>();
        relu_stage((nkb - 1) % kStages);
      }
    } else {
      using TIn = typename std::conditional<kMode == kScalarF32, float, __nv_bfloat16>::type;
      const TIn* in = static_cast<const TIn*>(a.in);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        uint8_t* xs = smem + s * kStage + kWBytes;
        const int kbase = (kb0 + i) * kBK + cl * 8;
        __nv_bfloat16 v[kRowsPerThread][8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int k = kbase + e;
          const bool kin = k < a.K;
          int r = 0, q = 0;
          int64_t koff = 0;
          if (kin) {
            if (a.ktab) {   // host-built (dr, dq, offset) per k: no integer divisions per element
              const int4 t = __ldg(a.ktab + k);
              r = t.x;
              q = t.y;
              koff = t.z;
            } else {
              const int c = k % a.Cin;
              const int rs = k / a.Cin;
              r = rs / a.S;
              q = rs - r * a.S;
              koff = r * a.sH + q * a.sW + c * a.sC;
            }
          }
#pragma unroll
          for (int j = 0; j < kRowsPerThread; ++j) {
            const int ih = pih[j] + r, iw = piw[j] + q;
            const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
            float x = 0.f;
            if (ok) {
              const TIn t = in[pb[j] * a.sN + pih[j] * a.sH + piw[j] * a.sW + koff + a.in_coff];
              if constexpr (kMode == kScalarF32) x = t; else x = __bfloat162float(t);
              if (a.relu_in) x = fmaxf(x, 0.f);
            }
            v[j][e] = __float2bfloat16_rn(x);
          }
        }
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j)
          if (rw + 4 * j < kRowGroups) *reinterpret_cast<uint4*>(xs + x_off(j)) = *reinterpret_cast<const uint4*>(v[j]);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[s]);
      }
    }
  } else if (warp == kXWarp) {
    if (ln_in && lane == 0) {
      // folded-LayerNorm consumers: each stage's o and r tiles land on
      // landed[]; the gather warps normalise them before releasing full[]
      tc::prefetch_tmap(&a.tmap);
      tc::prefetch_tmap(&a.tmap_r);
      pdl_wait();
      const int kc = kb0 * kBK;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&landed[s], 2 * kXBytes);
        tc::tma_im2col_4d(smem + s * kStage + kWBytes, &a.tmap, kc + i * kBK, n0, 0, 0, 0, 0, &landed[s]);
        tc::tma_im2col_4d(smem + a.r_off + s * kXBytes, &a.tmap_r, kc + i * kBK, n0, 0, 0, 0, 0, &landed[s]);
      }
    }
  } else if (warp == kLoadWarp) {
    if (lane == 0) {
      // ring refills beyond the first kStages come from L2: request the rest of
      // the CTA's contiguous weight slice now, before the predecessor finishes
      const __nv_bfloat16* wslice = a.wpack + (static_cast<int64_t>(mt) * a.kblocks + kb0) * (kWBytes / 2);
      if (nkb > kStages)
        tc::bulk_prefetch_l2(wslice + static_cast<int64_t>(kStages) * (kWBytes / 2),
                             static_cast<uint64_t>(nkb - kStages) * kWBytes);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&full[s], kWBytes);
        const __nv_bfloat16* src = wslice + static_cast<int64_t>(i) * (kWBytes / 2);
        tc::bulk_g2s(smem + s * kStage, src, kWBytes, &full[s]);
      }
    }
  } else if (warp == kMmaWarp && lane == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      tc::mbar_wait(&full[s], (i / kStages) & 1);
      tc::tc_fence_after();
      if (i == 0) PHASE(2);
      const uint32_t base = tc::smem_u32(smem + s * kStage);
#pragma unroll
      for (int ks = 0; ks < kBK / 16; ++ks) {
        const uint64_t ad = tc::smem_desc_sw64(base + 32 * ks, kSbo);
        const uint64_t bd = tc::smem_desc_sw64(base + kWBytes + 32 * ks, kSbo);
        tc::mma_f16(tmem, ad, bd, kIdesc, (i | ks) != 0);
      }
      tc::mma_commit(&empty[s]);
    }
    PHASE(3);
    tc::mma_commit(accum);
  }
  __syncwarp();

  // ------------------------------------------------------------ epilogue
  if (push) {
    // TMEM -> registers -> this CTA's smem (the drained ring), laid out as one
    // contiguous [128 channels][rows_per] block per owning rank; then one
    // thread bulk-copies each block into its owner's receive slot (TMA engine,
    // complete_tx on the owner's mbarrier).  No cluster barrier, no remote loads.
    const uint32_t me = tc::cluster_ctarank();
    const int rp = a.rows_per;
    float* stage = reinterpret_cast<float*>(smem);
    if (warp < 4) {
      tc::mbar_wait(accum, 0);
      tc::tc_fence_after();
      if (tid == 0) PHASE(4);
      const int chl = warp * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 2
      for (int c8 = 0; c8 < BN / 8; ++c8) {
        float v[8];
        tc::tmem_ld8(trow + c8 * 8, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {   // block = [owner][rows_per cols][128 ch]: lanes write consecutive words
          const int col = c8 * 8 + e;
          const int owner = col / rp;
          stage[(owner * rp + (col - owner * rp)) * 128 + chl] = v[e];
        }
      }
      tc::fence_proxy_async_smem();   // generic-proxy writes -> the bulk copy engine
      if (tid == 0) PHASE(8);
    }
    tc::tc_fence_before();
    // the owners' receive buffers sit behind their rings (always free)
    float* rbuf = recv;
    __syncthreads();
    if (tid == 0) {
      PHASE(9);
      const uint32_t block = static_cast<uint32_t>(128 * rp * 4);
      const uint32_t rbar_s = tc::smem_u32(rbar), recv_s = tc::smem_u32(rbuf), stage_s = tc::smem_u32(stage);
      for (int o = 0; o < a.splits && o * rp < BN; ++o)
        if (o != static_cast<int>(me))
          tc::bulk_s2cluster(tc::map_cluster(recv_s + me * block, o), stage_s + o * block, block,
                           tc::map_cluster(rbar_s, o));
      tc::bulk_commit();
    }
    if (warp == kTmemWarp) {
      tc::tc_fence_after();
      tc::tmem_dealloc(tmem, kTmemCols);
    }
    // owner: wait for every rank's block, reduce in rank order (thread = channel)
    const int r0 = static_cast<int>(me) * rp;
    const int mine = max(0, min(BN, r0 + rp) - r0);
    if (mine > 0 && tid < 128) {
      tc::mbar_wait_cluster(rbar, 0);
      if (tid == 0) PHASE(5);
      TO* out = static_cast<TO*>(a.out);
      const int chl = tid, ch = mt * 128 + chl;
      if (ch < a.Cout) {
        for (int c0 = 0; c0 < mine; c0 += 4) {   // recv = [src rank][rows_per cols][128 ch]
          float part[kMaxSplits][4];               // every load of 4 columns issued before the adds
#pragma unroll
          for (int z = 0; z < kMaxSplits; ++z)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (z < a.splits) part[z][e] = z == static_cast<int>(me) ? stage[(r0 + c0 + e) * 128 + chl]
                                                                      : rbuf[(z * rp + c0 + e) * 128 + chl];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float acc = part[0][e];
#pragma unroll
            for (int z = 1; z < kMaxSplits; ++z)
              if (z < a.splits) acc += part[z][e];
            const int p = n0 + r0 + c0 + e;
            if (p < a.M) {
              TO* dst = out + static_cast<int64_t>(p) * a.out_cs + a.out_coff + ch;
              const float y = act_fn(acc + push_bias, a.act);
              if constexpr (std::is_same<TO, float>::value) *dst = y;
              else *dst = __float2bfloat16_rn(y);
            }
          }
        }
      }
    }
    if (tid == 0) PHASE(6);   // owner reduction done; exit waits for this CTA's outgoing copies
    if (tid == 0) tc::bulk_wait_read();   // the source blocks stay valid until the engine has read them
    PHASE_FLUSH();
    trace_end(trace);
    return;
  }
  float* tile = reinterpret_cast<float*>(smem);
  if (warp < 4) {
    tc::mbar_wait(accum, 0);
    tc::tc_fence_after();
    if (tid == 0) PHASE(4);
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    // L2 reduction: the partial goes to this rank's workspace slice instead
    // of smem (the DSMEM pull moves each tile twice through the smem ports)
    float* mine = a.l2red ? a.ws + (static_cast<int64_t>(blockIdx.z) * gridDim.x * gridDim.y + blockIdx.x +
                                    blockIdx.y * gridDim.x) * BN * 128 + warp * 32 + lane
                          : nullptr;
#pragma unroll 4
    for (int c8 = 0; c8 < BN / 8; ++c8) {
      float v[8];
      tc::tmem_ld8(trow + c8 * 8, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (a.l2red) __stcg(mine + (c8 * 8 + e) * 128, v[e]);
        else tile[(c8 * 8 + e) * 128 + warp * 32 + lane] = v[e];
      }
    }
    if (tid == 0) PHASE(8);
  }
  tc::tc_fence_before();
  const int splits = a.splits;
  if (splits > 1)
    tc::cluster_sync();
  else
    __syncthreads();
  if (tid == 0) PHASE(9);
  // every TMEM read is done (the tile is in smem): free the columns now so a
  // PDL-launched successor CTA on this SM can allocate while we reduce
  if (warp == kTmemWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
  if (tid == 0) PHASE(5);
  const int rank = splits > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;
  const int rows_per = (BN + splits - 1) / splits;
  const int r0 = rank * rows_per, r1 = min(BN, r0 + rows_per);
  const uint32_t tile_s = tc::smem_u32(tile);
  const int64_t zstride = static_cast<int64_t>(gridDim.x) * gridDim.y * BN * 128;
  const float* l2base = a.l2red ? a.ws + (static_cast<int64_t>(blockIdx.x + blockIdx.y * gridDim.x)) * BN * 128 + lane * 4
                                : nullptr;
  TO* out = static_cast<TO*>(a.out);
  // a row per warp iteration, every split's DSMEM load issued before the first add
  constexpr int kRB = 1, kWarps = kThreads / 32;   // (2 rows in flight measured slower: Inception 0.390 -> 0.402 ms)
  for (int row0 = r0 + warp; row0 < r1; row0 += kRB * kWarps) {
    float4 part[kRB][kMaxSplits];
    bool ok[kRB];
#pragma unroll
    for (int rb = 0; rb < kRB; ++rb) {
      const int row = row0 + rb * kWarps;
      ok[rb] = row < r1 && n0 + row < a.M;
      const uint32_t off = static_cast<uint32_t>((row * 128 + lane * 4) * 4);
      if (!ok[rb]) continue;
      if (splits > 1) {
#pragma unroll
        for (int z = 0; z < kMaxSplits; ++z)
          if (z < splits)
            part[rb][z] = a.l2red ? __ldcg(reinterpret_cast<const float4*>(l2base + z * zstride + row * 128))
                                  : tc::ld_dsmem_f4(tc::map_cluster(tile_s + off, z));
      } else {
        part[rb][0] = *reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(tile) + off);
      }
    }
#pragma unroll
    for (int rb = 0; rb < kRB; ++rb) {
      if (!ok[rb]) continue;
      const int p = n0 + row0 + rb * kWarps;
      float4 acc = part[rb][0];
#pragma unroll
      for (int z = 1; z < kMaxSplits; ++z)
        if (z < splits) {
          acc.x += part[rb][z].x; acc.y += part[rb][z].y; acc.z += part[rb][z].z; acc.w += part[rb][z].w;
        }
      float y[4] = {act_fn(acc.x + bias[0], a.act), act_fn(acc.y + bias[1], a.act),
                    act_fn(acc.z + bias[2], a.act), act_fn(acc.w + bias[3], a.act)};
      if (a.res_stats) {
        // folded LayerNorm producer: the warp holds this token's 128 channels of
        // the m-tile; the sum and sum of squares of o + r (fixed xor-tree order)
        // go to stats_out[token][m-tile]
        const uint2 rr = *reinterpret_cast<const uint2*>(a.res + static_cast<int64_t>(p) * a.res_cs + ch);
        const float2 r01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rr.x));
        const float2 r23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rr.y));
        const float r[4] = {r01.x, r01.y, r23.x, r23.y};
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {   // the consumer normalises bf16(o) + r: the same values
          const float u = __bfloat162float(__float2bfloat16_rn(y[e])) + r[e];
          s1 += u;
          s2 += u * u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane == 0)
          reinterpret_cast<float2*>(a.stats_out)[static_cast<int64_t>(p) * gridDim.y + mt] = make_float2(s1, s2);
      }
      TO* dst = out + static_cast<int64_t>(p) * a.out_cs + a.out_coff + ch;
      if constexpr (std::is_same<TO, float>::value) {
        if (a.vec_out && ch + 3 < a.Cout) {
          *reinterpret_cast<float4*>(dst) = make_float4(y[0], y[1], y[2], y[3]);
          continue;
        }
      } else {
        if (a.vec_out && ch + 3 < a.Cout) {
          __nv_bfloat162 lo2 = __floats2bfloat162_rn(y[0], y[1]);
          __nv_bfloat162 hi2 = __floats2bfloat162_rn(y[2], y[3]);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo2);
          pk.y = *reinterpret_cast<uint32_t*>(&hi2);
          *reinterpret_cast<uint2*>(dst) = pk;
          continue;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (ch + e < a.Cout) {
          if constexpr (std::is_same<TO, float>::value) dst[e] = y[e];
          else dst[e] = __float2bfloat16_rn(y[e]);
        }
      }
    }
  }
  if (tid == 0) PHASE(6);
  if (splits > 1 && !a.l2red) tc::cluster_sync();  // peers may still be reading this CTA's tile
  PHASE_FLUSH();
    trace_end(trace);
}

template <int BN>
constexpr size_t bf_smem_bytes() {
  return bf_stages(BN) * (kWBytes + static_cast<size_t>(BN) * kBK * 2) + bf_bar_bytes(bf_stages(BN)) + 1024;
}

struct BfVariant {
  int bn;
  const void* func[kModes][2];  // [gather mode][out bf16, out f32]
  size_t smem;
};

template <int BN>
BfVariant make_bf() {
  BfVariant v;
  v.bn = BN;
  v.func[kVecBf16][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kVecBf16, __nv_bfloat16>);
  v.func[kVecBf16][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kVecBf16, float>);
  v.func[kScalarBf16][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kScalarBf16, __nv_bfloat16>);
  v.func[kScalarBf16][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kScalarBf16, float>);
  v.func[kScalarF32][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kScalarF32, __nv_bfloat16>);
  v.func[kScalarF32][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kScalarF32, float>);
  v.func[kSub4][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kSub4, __nv_bfloat16>);
  v.func[kSub4][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kSub4, float>);
  v.func[kSub2][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kSub2, __nv_bfloat16>);
  v.func[kSub2][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kSub2, float>);
  v.func[kTma][0] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kTma, __nv_bfloat16>);
  v.func[kTma][1] = reinterpret_cast<const void*>(&conv2d_tc_bf16<BN, kTma, float>);
  v.smem = bf_smem_bytes<BN>();
  return v;
}

const BfVariant* bf_variants() {
  static const BfVariant v[] = {make_bf<32>(), make_bf<64>(), make_bf<128>(), make_bf<256>(), make_bf<16>()};
  return v;
}

constexpr size_t kPushMaxBytes = kPushMaxKB * 1024;
constexpr size_t kSmemLimit = 232448 - 1024;   // 227 KB opt-in smem per CTA, minus static smem headroom
inline size_t attr_smem(size_t ring) { return std::min(ring + kPushMaxBytes, kSmemLimit); }

opara_status set_attr_once(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<const void*, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  if (done[func]) return OPARA_OK;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "conv2d_tc_bf16 smem attribute");
  done[func] = true;
  return OPARA_OK;
}

int64_t max_clusters(const void* func, int size, size_t smem, size_t smem_attr) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int64_t> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(func, size, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int64_t result = 2 * 148 / size;
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0 &&
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_attr)) == cudaSuccess) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(1, 1, size);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = size;
    lc.attrs = attr;
    lc.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, func, &lc) == cudaSuccess && n > 0) result = n;
  }
  cudaGetLastError();
  cache[key] = result;
  return result;
}

}  // namespace

// CONV2D with i[22] == 2 (engine "tc_bf16"): i[18] = input dtype (0 f32, 1 bf16),
// i[23] = output dtype, i[24] = activation (0 none, 1 ReLU, 2 GELU, 3 tanh;
// i[17] relu=1 also selects ReLU), i[25] = relu_in; p[1] = bf16 weights packed by
// engine.pack_conv_weights_bf16.
opara_status launch_conv2d_tc_bf16(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                                   LaunchCfg* cfg, bool dry) {
  BfArgs a;
  a.in = op.p[0];
  a.wpack = static_cast<const __nv_bfloat16*>(op.p[1]);
  a.bias = static_cast<const float*>(op.p[2]);
  a.out = op.p[3];
  a.N = (int)op.i[0]; a.H = (int)op.i[1]; a.W = (int)op.i[2]; a.Cin = (int)op.i[3];
  const int in_cs = (int)op.i[4];
  a.in_coff = (int)op.i[5];
  a.OH = (int)op.i[6]; a.OW = (int)op.i[7]; a.Cout = (int)op.i[8];
  a.out_cs = (int)op.i[9]; a.out_coff = (int)op.i[10];
  a.R = (int)op.i[11]; a.S = (int)op.i[12]; a.sh = (int)op.i[13]; a.sw = (int)op.i[14];
  a.ph = (int)op.i[15]; a.pw = (int)op.i[16];
  a.act = op.i[24] ? (int)op.i[24] : (op.i[17] ? 1 : 0);
  a.relu_in = (int)op.i[25];
  const bool in_f32 = op.i[18] == 0;
  const bool out_f32 = op.i[23] == 0;
  a.M = a.N * a.OH * a.OW;
  a.K = a.R * a.S * a.Cin;
  a.kblocks = (a.K + kBK - 1) / kBK;
  const bool nchw = op.i[20] != 0;
  if (nchw) {
    a.sC = static_cast<int64_t>(a.H) * a.W;
    a.sW = 1;
    a.sH = a.W;
    a.sN = a.sC * a.Cin;
    a.in_coff = 0;
  } else {
    a.sC = 1;
    a.sW = in_cs;
    a.sH = static_cast<int64_t>(a.W) * in_cs;
    a.sN = a.sH * a.H;
  }
  if (a.M <= 0 || a.Cout <= 0 || a.K <= 0) return fail(OPARA_ERR_VALUE, "conv2d: empty shape");
  auto vec_ok = [&](int g) {
    return !nchw && a.Cin % g == 0 && in_cs % g == 0 && a.in_coff % g == 0 &&
           reinterpret_cast<uintptr_t>(a.in) % (2 * g) == 0;
  };
  const bool tma = !in_f32 && !nchw && !a.relu_in &&
                   im2col_eligible(a.in, 2, a.Cin, in_cs, a.in_coff, a.H, a.W, a.OH, a.OW, a.sh, a.sw, a.ph, a.pw, kBK);
  const int mode = in_f32 ? kScalarF32 : tma ? kTma : vec_ok(8) ? kVecBf16 : vec_ok(4) ? kSub4 : vec_ok(2) ? kSub2 : kScalarBf16;
  auto encode = [&](int bn) {
    return !tma || make_im2col_map(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, op.p[0], a.N, a.H, a.W, a.Cin, in_cs,
                                   a.in_coff, a.OH, a.OW, a.sh, a.sw, a.ph, a.pw, kBK, bn);
  };
  const int align = out_f32 ? 16 : 8;
  a.vec_out = (a.out_cs % 4 == 0 && a.out_coff % 4 == 0 && reinterpret_cast<uintptr_t>(a.out) % align == 0) ? 1 : 0;
  const BfVariant* v = bf_variants();
  const int mtiles = (a.Cout + 127) / 128;
  a.ktab = static_cast<const int4*>(op.p[5]);
  a.res_stats = static_cast<int>(op.i[27]);
  a.res_cs = static_cast<int>(op.i[28]);
  a.res = a.res_stats ? static_cast<const __nv_bfloat16*>(op.p[4]) : nullptr;
  a.stats_out = a.res_stats ? static_cast<float*>(op.p[6]) : nullptr;
  a.ln_in = static_cast<int>(op.i[29]);
  a.lnout_cs = static_cast<int>(op.i[30]);
  a.ln_tiles = static_cast<int>(op.i[31]);
  a.stats_in = a.ln_in ? static_cast<const float*>(op.p[4]) : nullptr;
  a.gb = a.ln_in ? static_cast<const float*>(op.p[5]) : nullptr;
  a.lnout = a.ln_in ? static_cast<__nv_bfloat16*>(op.p[6]) : nullptr;
  a.eps = static_cast<float>(op.f[0]);
  if (a.res_stats && a.ln_in) return fail(OPARA_ERR_VALUE, "conv2d_tc_bf16: one folded LayerNorm role per GEMM");
  if (a.res_stats && (a.Cout % 128 || a.act != 0 || out_f32 || a.res_cs % 4))
    return fail(OPARA_ERR_VALUE, "conv2d_tc_bf16: residual + stats epilogue needs whole 128-channel tiles, "
                                 "no activation, bf16 output");
  if (a.ln_in && (mode != kTma || a.R != 1 || a.S != 1 || a.Cin % 128 || (a.lnout && a.lnout_cs % 8)))
    return fail(OPARA_ERR_VALUE, "conv2d_tc_bf16: LayerNorm on load needs a TMA-eligible 1x1 row GEMM");
  int id = op.variant;
  if (id < 0 || id > 4) {   // 0..3: tile width 32 << id, 4: width 16 (deep weight ring)
    id = 0;
    const int bns[4] = {32, 64, 128, 256};
    for (int k = 3; k >= 0; --k) {
      const int64_t tiles = static_cast<int64_t>((a.M + bns[k] - 1) / bns[k]) * mtiles;
      if (tiles >= 32 || k == 0) {
        id = k;
        break;
      }
    }
  }
  const int bn = v[id].bn;
  const int64_t base = static_cast<int64_t>((a.M + bn - 1) / bn) * mtiles;
  const int64_t target = op.i[21] > 0 ? op.i[21] : 148;
  // i[19]: > 1 forces that split-K, -1 forces none (autotuner), else automatic
  int64_t splits = op.i[19] > 1 ? op.i[19] : op.i[19] == -1 ? 1 : std::max<int64_t>(1, target / base);
  splits = std::min<int64_t>(splits, kMaxSplits);
  splits = std::min<int64_t>(splits, std::max(1, a.kblocks / 2));
  splits = std::max<int64_t>(1, splits);
  const void* func = v[id].func[mode][out_f32 ? 1 : 0];
  if (splits > 1 && op.i[19] <= 1)
    while (splits > 1) {
      const int rp = ((bn + static_cast<int>(splits) - 1) / static_cast<int>(splits) + 3) / 4 * 4;
      const size_t rb = static_cast<size_t>(splits) * 128 * rp * 4;
      const bool pu = rb <= kPushMaxBytes && v[id].smem + rb <= kSmemLimit && op.i[26] == 0 && !a.res_stats &&
                      !a.ln_in;
      const size_t sm = v[id].smem + (pu ? rb : 0);
      if (base <= max_clusters(func, static_cast<int>(splits), sm, attr_smem(v[id].smem))) break;
      --splits;
    }
  a.kb_per_split = static_cast<int>((a.kblocks + splits - 1) / splits);
  a.splits = (a.kblocks + a.kb_per_split - 1) / a.kb_per_split;
  // Split-K reduction mode: push (each rank st.async's its partial columns to
  // the owning rank, which waits on byte counts) when the receive buffer is
  // small; otherwise pull over DSMEM after a cluster barrier.
  a.rows_per = ((bn + a.splits - 1) / a.splits + 3) / 4 * 4;
  const size_t recv_bytes = static_cast<size_t>(a.splits) * 128 * a.rows_per * 4;
  // (the residual + stats epilogue lives in the pull / L2 reduction loop, and
  // LayerNorm-on-load consumers keep their residual tiles where push receives)
  const bool folded = a.res_stats || a.ln_in;
  a.push = (a.splits > 1 && recv_bytes <= kPushMaxBytes && v[id].smem + recv_bytes <= kSmemLimit &&
            op.i[26] == 0 && !folded) ? 1 : 0;
  a.l2red = (a.splits > 1 && (op.i[26] == 2 || (op.i[26] == 0 && folded))) ? 1 : 0;
  // LayerNorm-on-load: the residual tiles (kStages x BN x 64 B) behind the ring and barriers
  const size_t ring = static_cast<size_t>(bf_stages(bn)) * (kWBytes + static_cast<size_t>(bn) * kBK * 2);
  a.r_off = static_cast<uint32_t>((ring + bf_bar_bytes(bf_stages(bn)) + 1023) / 1024 * 1024);
  const size_t r_bytes = a.ln_in ? static_cast<size_t>(bf_stages(bn)) * bn * kBK * 2 + 2 * bn * 4 + 1024 : 0;
  if (a.ln_in && v[id].smem + r_bytes > std::min(attr_smem(v[id].smem), kSmemLimit))
    return fail(OPARA_ERR_VALUE, "conv2d_tc_bf16: LayerNorm on load: residual tiles do not fit this tile width");
  a.ws = nullptr;
  LaunchCfg c;
  c.func = func;
  c.grid = dim3(ceil_div(a.M, bn), mtiles, a.splits);
  c.block = dim3(kThreads);
  c.smem = v[id].smem + (a.push ? recv_bytes : 0) + r_bytes;
  c.tmem_cols = bn < 32 ? 32 : bn;
  c.cluster = a.splits;
  c.workspace = a.l2red ? static_cast<size_t>(c.grid.x) * c.grid.y * c.grid.z * bn * 128 * 4 : 0;
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  if (a.l2red) {
    if (!op.p[7]) return fail(OPARA_ERR_INTERNAL, "conv2d_tc_bf16: split-K workspace missing");
    a.ws = static_cast<float*>(op.p[7]);
  }
  opara_status st = set_attr_once(func, attr_smem(v[id].smem));
  if (st != OPARA_OK) return st;
  if (!encode(bn)) return fail(OPARA_ERR_CUDA, "conv2d_tc_bf16: cuTensorMapEncodeIm2col failed");
  if (a.ln_in) {   // the residual view r of LN(o + r): i[32] address, i[33] cstride (same [T][C] shape)
    const void* rbase = reinterpret_cast<const void*>(static_cast<uintptr_t>(op.i[32]));
    if (!rbase || !make_im2col_map(&a.tmap_r, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rbase, a.N, a.H, a.W, a.Cin,
                                   op.i[33], 0, a.OH, a.OW, a.sh, a.sw, a.ph, a.pw, kBK, bn))
      return fail(OPARA_ERR_CUDA, "conv2d_tc_bf16: LayerNorm residual tensor map");
  }
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s, a.splits > 1 ? static_cast<unsigned>(a.splits) : 1u);
}

}  // namespace opara

#ifdef OPARA_PHASE_PROBE
extern "C" int opara_debug_phase_read(unsigned long long* host, int max_records, int reset) {
  unsigned n = 0;
  cudaMemcpyFromSymbol(&n, opara::g_phase_n, sizeof(n));
  const int k = static_cast<int>(std::min<unsigned>(n, std::min(max_records, 4096)));
  if (k > 0) cudaMemcpyFromSymbol(host, opara::g_phase, sizeof(unsigned long long) * 12 * k);
  if (reset) {
    const unsigned z = 0;
    cudaMemcpyToSymbol(opara::g_phase_n, &z, sizeof(z));
  }
  return k;
}
#endif
