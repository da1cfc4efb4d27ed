// NHWC implicit-GEMM convolution on the 5th-generation tensor cores (tcgen05),
// fp32 in / fp32 out with 3xTF32 split precision (|error| ~ 2^-21 relative,
// inside the 1e-4 fp32 parity budget that a single TF32 pass would miss).
//
// GEMM view, swap-AB ("weights on M"):
//   D[co, p] = sum_k W[co, k] * X[p, k]        co = output channel (UMMA M = 128)
//                                              p  = output pixel   (UMMA N = BN)
//                                              k  = (r*S + s)*Cin + c
// The accumulator tile lives in TMEM as 128 lanes (channels) x BN columns
// (pixels).
//
// Per CTA (160 threads):
//   warps 0-3  producers: im2col gather of X with cp.async (16-byte chunks of
//              4 channels, zero-fill for padding) straight into the UMMA
//              no-swizzle K-major core-matrix layout, S-2 stages in flight;
//              then an in-place split x -> (tf32 hi, tf32 lo).  Thread 0 also
//              pulls the host-packed W hi/lo block of each stage with one bulk
//              async copy (cp.async.bulk, completion on the stage mbarrier);
//   warp 4     MMA issuer (one lane): 3 tcgen05.mma per 8-wide k step
//              (hi*hi + hi*lo + lo*hi); tcgen05.commit releases the stage;
//   epilogue   TMEM -> registers (tcgen05.ld) -> a [BN][128] fp32 tile in the
//              now idle pipeline smem.
// Split-K (batch-1 layers are short in M and deep in K) runs as a thread-block
// cluster along z: every split CTA stages its partial tile in its own smem,
// one cluster barrier, then CTA rank r reduces rows [r*BN/S, (r+1)*BN/S) by
// reading that row from every rank over DSMEM in rank order (deterministic),
// adds the folded-BN bias, applies ReLU and stores 16-byte vectors of 4
// channels into the output channel view (the concat slice).  No workspace, no
// atomics, no second kernel.

#include "device_common.cuh"
#include "ops.h"
#include "status.h"
#include "tc_common.cuh"
#include "tma_host.h"

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

namespace opara {
namespace {

constexpr int kBKF = 16;            // k elements (fp32) per stage
constexpr int kProducerWarps = 8;  // gather + convert; one warp per scheduler is not enough
constexpr int kMmaWarp = kProducerWarps;      // one elected lane issues tcgen05.mma
constexpr int kLoadWarp = kProducerWarps + 1;  // one lane streams the packed weights
constexpr int kThreads = 32 * (kProducerWarps + 2);
constexpr int kMaxSplits = 8;       // portable cluster size
constexpr uint32_t kWBytes = 128 * kBKF * 4;  // one precision plane of the W stage

// Ring depth per pixel tile: the small tiles keep the CTA under ~113 KB so two
// CTAs (two concurrent branches) can share an SM.
// (deeper rings measured neutral: the k loop is paced by the tensor pipe)
__host__ __device__ constexpr int tc_stages(int bn) { return bn == 32 ? 5 : bn == 64 ? 4 : bn == 128 ? 6 : 4; }

struct TcArgs {
  CUtensorMap tmap;                 // im2col map of the input view (kLoad == kLoadTma only)
  const float* __restrict__ in;
  const float* __restrict__ wpack;  // [m_tiles][kblocks][hi|lo][chunk][rg][8][4]
  const float* __restrict__ bias;
  float* __restrict__ out;
  unsigned long long* dbg;          // optional phase timestamps (CTA 0): [warp][8]
  int N, H, W, Cin, in_coff;
  int OH, OW, Cout, out_cs, out_coff;
  int R, S, sh, sw, ph, pw;
  int relu, vec_out, relu_in;
  int M, K, kblocks;
  int splits, kb_per_split;
  int push, rows_per;   // split-K reduction: 1 = partials pushed to the owner CTA (st.async)
  int l2red;            // split-K reduction through L2: partial tiles in `ws`, one cluster barrier
  float* ws;
  int64_t sN, sH, sW, sC;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Sum the 3xTF32 accumulators of this warp's lane quarter (hh, hl[, lh] at
// columns c, BN + c, 2 BN + c) over its half of the BN pixel columns, 16
// columns per step with every TMEM load in flight before one wait, and hand
// each (column, sum) to `put`.  Summation order hh + (hl + lh) throughout.
template <int BN, int kAcc, typename Put>
__device__ __forceinline__ void drain_accumulators(uint32_t trow, int half, Put put) {
  constexpr int kCols = BN / 2;   // two warps per lane quarter
#pragma unroll 1
  for (int c = half * kCols; c < (half + 1) * kCols; c += 16) {
    float v[16], c1[16], c2[16];
    if constexpr (kAcc == 3)
      tc::tmem_ld16x3(trow + c, trow + BN + c, trow + 2 * BN + c, v, c1, c2);
    else
      tc::tmem_ld16x2(trow + c, trow + BN + c, v, c1);
#pragma unroll
    for (int e = 0; e < 16; ++e) put(c + e, v[e] + (kAcc == 3 ? (c1[e] + c2[e]) : c1[e]));
  }
}

// Activation load path: scalar 4-byte cp.async gathers, 16-byte cp.async
// gathers (4 channels), or TMA im2col loads of the whole stage (one thread).
enum { kLoadScalar = 0, kLoadVec = 1, kLoadTma = 2 };

template <int BN, int kLoad>
__global__ void __launch_bounds__(kThreads, 1) conv2d_tc_tf32x3(const __grid_constant__ TcArgs a, unsigned long long* trace) {
  constexpr bool kVec = kLoad == kLoadVec;
  constexpr int kStages = tc_stages(BN);
  constexpr uint32_t kXBytes = BN * kBKF * 4;
  constexpr uint32_t kStage = 2 * kWBytes + 2 * kXBytes;
  // Operand planes use the 64-byte-swizzled K-major layout: a row holds the
  // stage's 16 fp32 k values (64 B = 4 chunks of 16 B), 8-row atoms of 512 B
  // are stacked along M/N (SBO = 512), and chunk c of row r sits at chunk
  // position c ^ ((r >> 1) & 3) — bank-conflict-free operand reads for the
  // tensor core.  An 8-wide k step advances the descriptor start by 32 B.
  constexpr uint32_t kSbo = 512;
  constexpr int kRowGroups = BN / 8;
  constexpr int kRowsPerThread = (kRowGroups + 3) / 4;  // atoms per gather/convert thread
  constexpr uint32_t kIdesc = tc::instr_desc(2, 128, BN);
  constexpr uint32_t kIdesc2 = tc::instr_desc(2, 128, BN <= 128 ? 2 * BN : BN);   // hi*[hi; lo]
  // Separate TMEM accumulators for hi*hi, hi*lo and lo*hi: consecutive MMAs
  // then target different tiles and overlap in the tensor pipe instead of
  // serialising on one accumulator (BN = 256 shares one for both corrections).
  constexpr int kAcc = BN >= 256 ? 2 : 3;
  constexpr uint32_t kTmemCols = BN >= 256 ? 512 : (BN * 4 <= 32 ? 32 : BN * 4);
  static_assert(BN * 128 * 4 <= kStages * kStage, "epilogue tile must fit in the pipeline smem");
  static_assert(48 * 1024 <= kStages * kStage, "push staging blocks must fit in the pipeline smem");

  // No-swizzle UMMA operands need 16-byte alignment only; indexing the extern
  // array directly keeps every access in the shared state space (LDS/STS).
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzle atoms must sit on 512-byte boundaries: align the carve-out base
  // (offsetting the extern array keeps accesses in the shared state space)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint64_t* empty = full + kStages;
  uint64_t* landed = empty + kStages;  // gather copies of the stage complete
  uint64_t* accum = landed + kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accum + 1);

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool dbg = a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lane == 0;
#define DBG(slot) \
  if (dbg) a.dbg[warp * 8 + (slot)] = global_ns();
  // split-K rank skew: every rank of cluster (0, 0) stamps accumulator ready /
  // partial drained / after the cluster barrier at dbg[2048 + 4 z + k]
#define RSTAMP(k) \
  if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) a.dbg[2048 + 4 * blockIdx.z + (k)] = global_ns();
  DBG(0);
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (a.dbg && tid == 0 && cta_lin < 96) a.dbg[64 + 2 * cta_lin] = global_ns();
  const int n0 = blockIdx.x * BN;   // first pixel
  const int mt = blockIdx.y;        // 128-channel tile
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int nkb = min(a.kblocks, kb0 + a.kb_per_split) - kb0;
  // pull-epilogue bias (lane = 4 channels): a parameter, fetched before griddepcontrol.wait
  const int ch = mt * 128 + lane * 4;
  float4 bias4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (a.bias && !a.push) {
    if (ch + 0 < a.Cout) bias4.x = __ldg(a.bias + ch + 0);
    if (ch + 1 < a.Cout) bias4.y = __ldg(a.bias + ch + 1);
    if (ch + 2 < a.Cout) bias4.z = __ldg(a.bias + ch + 2);
    if (ch + 3 < a.Cout) bias4.w = __ldg(a.bias + ch + 3);
  }
  // push-epilogue owner reduction: thread = output channel
  const float push_bias = ((a.push || a.splits > 1) && a.bias && tid < 128 && mt * 128 + tid < a.Cout) ? __ldg(a.bias + mt * 128 + tid) : 0.f;

  // push-mode split-K receive buffer [src rank][128 channels][rows_per] fp32, behind the ring
  uint64_t* rbar = accum + 2;
  float* recv = reinterpret_cast<float*>(smem + kStages * kStage + 512);
  const bool push = a.push != 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 32 * (kProducerWarps / 2) + 1);  // converters + the weight loader
      // one noinc arrive per gather thread, or the TMA thread's expect_tx arrive
      tc::mbar_init(&landed[s], kLoad == kLoadTma ? 1 : 32 * (kProducerWarps / 2));
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(accum, 1);
    if (push) tc::mbar_init(rbar, 1);
    tc::fence_barrier_init();
  }
  // TMEM is allocated and freed by the MMA warp: idle in every epilogue
  if (warp == kMmaWarp) tc::tmem_alloc(tslot, kTmemCols);
  tc::tc_fence_before();
  if (push) {   // receive barriers initialised cluster-wide before anyone pushes
    tc::cluster_sync();
    if (tid == 0) {   // every rank bulk-copies one whole [rows_per][128] block to each owner
      const int r0 = static_cast<int>(tc::cluster_ctarank()) * a.rows_per;
      // every other rank's block; the owner's own partial stays in its ring
      if (r0 < BN) tc::mbar_arrive_expect_tx(rbar, static_cast<uint32_t>((a.splits - 1) * a.rows_per * 128 * 4));
    }
  } else {
    __syncthreads();
  }
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  DBG(1);

  if (warp < kProducerWarps) {
    // -------------------------------------------- gather (warps 0-3) / convert (4-7)
    // Warp w and warp w+4 own the same X units: rows of 8-row atoms rw, rw+4, ...
    // The gather warp streams them into the hi plane with cp.async and the
    // landed[s] mbarrier fires when its copies complete; the convert warp then
    // writes lo = x - trunc_tf32(x) and arrives on full[s].  Splitting the
    // roles lets the gathers run a full ring ahead of the MMA.
    const bool gather = warp < kProducerWarps / 2;
    const int rw = warp & 3;
    const int r8 = lane & 7, cl = lane >> 3;  // row within atom, 16-byte chunk
    auto x_off = [&](int j) -> uint32_t {     // byte offset of my unit j inside an X plane
      return static_cast<uint32_t>(rw + 4 * j) * kSbo + r8 * 64u +
             static_cast<uint32_t>((cl ^ ((r8 >> 1) & 3)) * 16);
    };
    if (kLoad == kLoadTma && gather) {
      // One lane streams each stage's X tile (BN pixels x 16 channels of one
      // tap, K = (r*S + s)*Cin + c with Cin % 16 == 0) into the hi plane with
      // a TMA im2col load; padding and the tile tail arrive as zeros.
      if (warp == 0 && lane == 0) {
        const int ohw = a.OH * a.OW;
        const int b = n0 / ohw, rem = n0 - b * ohw, oh = rem / a.OW, ow = rem - oh * a.OW;
        const int w0 = ow * a.sw - a.pw, h0 = oh * a.sh - a.ph;
        const int kc = kb0 * kBKF, rs = kc / a.Cin;
        int dc = kc - rs * a.Cin, dr = rs / a.S, dq = rs - dr * a.S;
        tc::prefetch_tmap(&a.tmap);
        pdl_wait();
        trace_begin(trace);
        for (int i = 0; i < nkb; ++i) {
          const int s = i % kStages;
          if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
          if (dbg && i < 64) a.dbg[768 + i] = global_ns();
          tc::mbar_arrive_expect_tx(&landed[s], kXBytes);
          tc::tma_im2col_4d(smem + s * kStage + 2 * kWBytes, &a.tmap, dc, w0, h0, b, dq, dr, &landed[s]);
          dc += kBKF;
          if (dc == a.Cin) {
            dc = 0;
            if (++dq == a.S) {
              dq = 0;
              ++dr;
            }
          }
        }
      }
    } else if (gather) {
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
      // vector gather: my 4-channel chunk's k = (r*S + q)*Cin + c, advanced
      // incrementally by kBKF per stage (no divisions in the loop)
      const float* rowbase[kRowsPerThread];
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j)
        rowbase[j] = a.in + (pb[j] >= 0 ? pb[j] * a.sN + pih[j] * a.sH + piw[j] * a.sW + a.in_coff : 0);
      int kc = kb0 * kBKF + cl * 4, dc = 0, dr = 0, dq = 0;
      if (kVec && kc < a.K) {
        dc = kc % a.Cin;
        const int rs = kc / a.Cin;
        dr = rs / a.S;
        dq = rs - dr * a.S;
      }
      pdl_wait();  // the input activations come from the predecessor grid
      trace_begin(trace);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        if (dbg && tid == 0 && i < 64) a.dbg[768 + i] = global_ns();
        const uint32_t xh = tc::smem_u32(smem + s * kStage + 2 * kWBytes);
        if constexpr (kVec) {
          const bool kin = kc < a.K;
          const int64_t koff = dr * a.sH + dq * a.sW + dc;
#pragma unroll
          for (int j = 0; j < kRowsPerThread; ++j) {
            const int ih = pih[j] + dr, iw = piw[j] + dq;
            const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
            if (rw + 4 * j < kRowGroups) cp_async16(xh + x_off(j), ok ? rowbase[j] + koff : a.in, ok);
          }
          kc += kBKF;
          dc += kBKF;
          while (dc >= a.Cin) {
            dc -= a.Cin;
            if (++dq == a.S) {
              dq = 0;
              ++dr;
            }
          }
        } else {
          const int kbase = (kb0 + i) * kBKF + cl * 4;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = kbase + e;
            const bool kin = k < a.K;
            int c = 0, r = 0, q = 0;
            if (kin) {
              c = k % a.Cin;
              const int rs = k / a.Cin;
              r = rs / a.S;
              q = rs - r * a.S;
            }
#pragma unroll
            for (int j = 0; j < kRowsPerThread; ++j) {
              const int ih = pih[j] + r, iw = piw[j] + q;
              const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
              const float* src = ok ? a.in + pb[j] * a.sN + ih * a.sH + iw * a.sW + c * a.sC + a.in_coff : a.in;
              if (rw + 4 * j < kRowGroups) cp_async4(xh + x_off(j) + 4 * e, src, ok);
            }
          }
        }
        tc::cp_async_arrive_noinc(&landed[s]);
      }
    } else {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        tc::mbar_wait(&landed[s], (i / kStages) & 1);
        if (dbg && warp == 4 && lane == 0 && i < 64) a.dbg[256 + i] = global_ns();
        uint8_t* xh = smem + s * kStage + 2 * kWBytes;
        uint8_t* xl = xh + kXBytes;
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
          if (rw + 4 * j >= kRowGroups) break;
          // The tensor core reads an fp32 operand as tf32 by dropping the low
          // 13 mantissa bits, so the raw x already serves as the hi plane;
          // only lo = x - trunc_tf32(x) (exact in fp32) is materialised.
          float4 v = *reinterpret_cast<const float4*>(xh + x_off(j));
          if (a.relu_in) {  // fused input ReLU: clamp the hi plane in place
            v.x = fmaxf(v.x, 0.f);
            v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f);
            v.w = fmaxf(v.w, 0.f);
            *reinterpret_cast<float4*>(xh + x_off(j)) = v;
          }
          float4 lo;
          lo.x = v.x - tc::trunc_tf32(v.x);
          lo.y = v.y - tc::trunc_tf32(v.y);
          lo.z = v.z - tc::trunc_tf32(v.z);
          lo.w = v.w - tc::trunc_tf32(v.w);
          *reinterpret_cast<float4*>(xl + x_off(j)) = lo;
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[s]);
      }
    }
  } else if (warp == kLoadWarp) {
    // ------------------------------------------------------------ weight loader
    if (lane == 0) {
      // The CTA's whole weight slice is one contiguous run of packed stages.
      // The ring holds kStages of them; the rest is requested into L2 now
      // (before the predecessor has finished), so every later refill is an
      // L2 hit instead of an HBM round trip (the k-loop was weight-latency bound).
      const float* wslice = a.wpack + (static_cast<int64_t>(mt) * a.kblocks + kb0) * (2 * kWBytes / 4);
      if (nkb > kStages)
        tc::bulk_prefetch_l2(wslice + static_cast<int64_t>(kStages) * (2 * kWBytes / 4),
                             static_cast<uint64_t>(nkb - kStages) * 2 * kWBytes);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % kStages;
        if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&full[s], 2 * kWBytes);
        const float* src = wslice + static_cast<int64_t>(i) * (2 * kWBytes / 4);
        tc::bulk_g2s(smem + s * kStage, src, 2 * kWBytes, &full[s]);
      }
    }
  } else if (lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      tc::mbar_wait(&full[s], (i / kStages) & 1);
      tc::tc_fence_after();
      if (dbg && i < 64) a.dbg[512 + i] = global_ns();
      const uint32_t base = tc::smem_u32(smem + s * kStage);
      const uint32_t w_hi = base, w_lo = base + kWBytes;
      const uint32_t x_hi = base + 2 * kWBytes, x_lo = x_hi + kXBytes;
#pragma unroll
      for (int ks = 0; ks < kBKF / 8; ++ks) {
        const uint64_t ah = tc::smem_desc_sw64(w_hi + 32 * ks, kSbo);
        const uint64_t al = tc::smem_desc_sw64(w_lo + 32 * ks, kSbo);
        const uint64_t bh = tc::smem_desc_sw64(x_hi + 32 * ks, kSbo);
        const uint32_t first = (i | ks) != 0;
        if constexpr (kAcc == 3) {
          // The lo plane's atoms follow the hi plane's (x_lo = x_hi + BN/8
          // atoms at the same SBO), so one N = 2 BN MMA computes hi*hi
          // (columns [0, BN)) and hi*lo ([BN, 2 BN)) reading the W hi tile
          // once: the tf32 MMAs are shared-memory-bandwidth bound.
          tc::mma_tf32(tmem, ah, bh, kIdesc2, first);
          tc::mma_tf32(tmem + 2 * BN, al, bh, kIdesc, first);
        } else {
          const uint64_t bl = tc::smem_desc_sw64(x_lo + 32 * ks, kSbo);
          tc::mma_tf32(tmem, ah, bh, kIdesc, first);
          tc::mma_tf32(tmem + BN, ah, bl, kIdesc, first);
          tc::mma_tf32(tmem + BN, al, bh, kIdesc, 1u);
        }
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(accum);
    DBG(2);
  }
  __syncwarp();

  // ------------------------------------------------------------ epilogue
  // TMEM -> [BN][128] fp32 tile in the idle pipeline smem (all MMAs, hence all
  // smem reads by the tensor core, are complete once `accum` fires).
  DBG(3);
  if (push) {
    // TMEM -> registers (sum of the 3xTF32 accumulators) -> this CTA's idle ring
    // smem as one contiguous [rows_per cols][128 ch] block per owning rank;
    // one thread bulk-copies each block into its owner's receive slot (TMA
    // engine, complete_tx on the owner's mbarrier); owners reduce in rank order.
    const uint32_t me = tc::cluster_ctarank();
    const int rp = a.rows_per;
    float* stage = reinterpret_cast<float*>(smem);
    if (warp < kProducerWarps) {
      tc::mbar_wait(accum, 0);
      tc::tc_fence_after();
      const int quarter = warp & 3, half = warp >> 2;
      const int chl = quarter * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      // the owner blocks are [rows_per cols][128 ch] back to back: column col
      // lands at stage[col * 128 + channel] whatever its owner
      drain_accumulators<BN, kAcc>(trow, half, [&](int col, float val) { stage[col * 128 + chl] = val; });
      tc::fence_proxy_async_smem();   // generic-proxy writes -> the bulk copy engine
      DBG(4);
    }
    tc::tc_fence_before();
    // the owners' receive buffers sit behind their rings (always free)
    float* rbuf = recv;
    __syncthreads();
    if (tid == 0) {
      const uint32_t block = static_cast<uint32_t>(128 * rp * 4);
      const uint32_t rbar_s = tc::smem_u32(rbar), recv_s = tc::smem_u32(rbuf), stage_s = tc::smem_u32(stage);
      for (int o = 0; o < a.splits && o * rp < BN; ++o)
        if (o != static_cast<int>(me))
          tc::bulk_s2cluster(tc::map_cluster(recv_s + me * block, o), stage_s + o * block, block,
                             tc::map_cluster(rbar_s, o));
      tc::bulk_commit();
    }
    if (warp == kMmaWarp) {
      tc::tc_fence_after();
      tc::tmem_dealloc(tmem, kTmemCols);
    }
    const int r0 = static_cast<int>(me) * rp;
    const int mine = max(0, min(BN, r0 + rp) - r0);
    const int ch = mt * 128 + tid;
    if (mine > 0 && tid < 128 && ch < a.Cout) {
      tc::mbar_wait_cluster(rbar, 0);
      DBG(5);
      for (int c0 = 0; c0 < mine; c0 += 4) {   // recv = [src rank][rows_per cols][128 ch]
        float part[kMaxSplits][4];               // every load of 4 columns issued before the adds
#pragma unroll
        for (int z = 0; z < kMaxSplits; ++z)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (z < a.splits) part[z][e] = z == static_cast<int>(me) ? stage[(r0 + c0 + e) * 128 + tid]
                                                                      : rbuf[(z * rp + c0 + e) * 128 + tid];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float acc = part[0][e];
#pragma unroll
          for (int z = 1; z < kMaxSplits; ++z)
            if (z < a.splits) acc += part[z][e];
          const int p = n0 + r0 + c0 + e;
          if (p < a.M) a.out[static_cast<int64_t>(p) * a.out_cs + a.out_coff + ch] = apply_act(acc + push_bias, a.relu);
        }
      }
    }
    DBG(6);
    if (tid == 0) tc::bulk_wait_read();   // the source blocks stay valid until the engine has read them
    DBG(7);
    trace_end(trace);
    return;
  }
  if (a.l2red) {
    // Split-K through L2: each rank stores its partial [BN][128] tile to its
    // workspace slice (coalesced along channels), one cluster barrier
    // (release / acquire at cluster scope orders the global stores), then
    // rank r reduces rows [r*BN/S, (r+1)*BN/S) from every slice in rank order
    // (deterministic).  The smem ports carry nothing: the DSMEM pull moved
    // each tile twice through them (~17-21 B/clk per SM) and measured ~2.4 us.
    const int tiles = gridDim.x * gridDim.y, tile_id = blockIdx.x + blockIdx.y * gridDim.x;
    const int64_t plane = static_cast<int64_t>(BN) * 128;
    if (warp < kProducerWarps) {
      tc::mbar_wait(accum, 0);
      tc::tc_fence_after();
      DBG(4);
      const int quarter = warp & 3, half = warp >> 2;
      const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      RSTAMP(0);
      float* mine = a.ws + (static_cast<int64_t>(blockIdx.z) * tiles + tile_id) * plane + quarter * 32 + lane;
      drain_accumulators<BN, kAcc>(trow, half, [&](int col, float val) { __stcg(mine + col * 128, val); });
      RSTAMP(1);
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    RSTAMP(2);
    if (warp == kMmaWarp) {
      tc::tc_fence_after();
      tc::tmem_dealloc(tmem, kTmemCols);
    }
    DBG(5);
    const int splits = a.splits;
    const int rows_per = (BN + splits - 1) / splits;
    const int r0 = static_cast<int>(blockIdx.z) * rows_per, r1 = min(min(BN, r0 + rows_per), a.M - n0);
    const float* base = a.ws + static_cast<int64_t>(tile_id) * plane + lane * 4;
    const int64_t zstride = static_cast<int64_t>(tiles) * plane;
    for (int row = r0 + warp; row < r1; row += kThreads / 32) {
      float4 part[kMaxSplits];   // every rank's load in flight before the first add
#pragma unroll
      for (int z = 0; z < kMaxSplits; ++z)
        if (z < splits) part[z] = __ldcg(reinterpret_cast<const float4*>(base + z * zstride + row * 128));
      float4 acc = part[0];
#pragma unroll
      for (int z = 1; z < kMaxSplits; ++z)
        if (z < splits) {
          acc.x += part[z].x; acc.y += part[z].y; acc.z += part[z].z; acc.w += part[z].w;
        }
      acc.x += bias4.x; acc.y += bias4.y; acc.z += bias4.z; acc.w += bias4.w;
      if (a.relu) {
        acc.x = apply_act(acc.x, a.relu); acc.y = apply_act(acc.y, a.relu);
        acc.z = apply_act(acc.z, a.relu); acc.w = apply_act(acc.w, a.relu);
      }
      float* dst = a.out + static_cast<int64_t>(n0 + row) * a.out_cs + a.out_coff + ch;
      if (a.vec_out && ch + 3 < a.Cout) {
        *reinterpret_cast<float4*>(dst) = acc;
      } else {
        if (ch + 0 < a.Cout) dst[0] = acc.x;
        if (ch + 1 < a.Cout) dst[1] = acc.y;
        if (ch + 2 < a.Cout) dst[2] = acc.z;
        if (ch + 3 < a.Cout) dst[3] = acc.w;
      }
    }
    DBG(6);
    DBG(7);
    if (a.dbg && tid == 0 && cta_lin < 96) a.dbg[64 + 2 * cta_lin + 1] = global_ns();
    trace_end(trace);
    return;
  }
  float* tile = reinterpret_cast<float*>(smem);
  if (warp < kProducerWarps) {
    // warp w may only touch TMEM lanes [32*(w%4), +32): lane quarter w%4,
    // column half w/4
    tc::mbar_wait(accum, 0);
    tc::tc_fence_after();
    DBG(4);
    const int quarter = warp & 3, half = warp >> 2;
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    RSTAMP(0);
    drain_accumulators<BN, kAcc>(trow, half,
                                 [&](int col, float val) { tile[col * 128 + quarter * 32 + lane] = val; });
    RSTAMP(1);
  }
  tc::tc_fence_before();
  const int splits = a.splits;
  if (splits > 1)
    tc::cluster_sync();
  else
    __syncthreads();
  RSTAMP(2);
  // every TMEM read is done (the tile is in smem): free the columns now so a
  // PDL-launched successor CTA on this SM can allocate while we reduce
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
  DBG(5);
  // rows [r0, r1) of the tile are reduced (over the cluster) and stored by this CTA
  const int rank = splits > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;
  const int rows_per = (BN + splits - 1) / splits;
  const int r0 = rank * rows_per, r1 = min(BN, r0 + rows_per);
  const uint32_t tile_s = tc::smem_u32(tile);
  for (int row = r0 + warp; row < r1; row += kThreads / 32) {
    const int p = n0 + row;
    if (p >= a.M) break;
    const uint32_t off = static_cast<uint32_t>((row * 128 + lane * 4) * 4);
    float4 acc;
    if (splits > 1) {
      float4 part[kMaxSplits];
#pragma unroll
      for (int z = 0; z < kMaxSplits; ++z)
        if (z < splits) part[z] = tc::ld_dsmem_f4(tc::map_cluster(tile_s + off, z));
      acc = part[0];
#pragma unroll
      for (int z = 1; z < kMaxSplits; ++z)
        if (z < splits) {
          acc.x += part[z].x; acc.y += part[z].y; acc.z += part[z].z; acc.w += part[z].w;
        }
    } else {
      acc = *reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(tile) + off);
    }
    acc.x += bias4.x; acc.y += bias4.y; acc.z += bias4.z; acc.w += bias4.w;
    if (a.relu) {
      acc.x = apply_act(acc.x, a.relu); acc.y = apply_act(acc.y, a.relu);
      acc.z = apply_act(acc.z, a.relu); acc.w = apply_act(acc.w, a.relu);
    }
    float* dst = a.out + static_cast<int64_t>(p) * a.out_cs + a.out_coff + ch;
    if (a.vec_out && ch + 3 < a.Cout) {
      *reinterpret_cast<float4*>(dst) = acc;
    } else {
      if (ch + 0 < a.Cout) dst[0] = acc.x;
      if (ch + 1 < a.Cout) dst[1] = acc.y;
      if (ch + 2 < a.Cout) dst[2] = acc.z;
      if (ch + 3 < a.Cout) dst[3] = acc.w;
    }
  }
  DBG(6);
  if (splits > 1) tc::cluster_sync();  // peers may still be reading this CTA's tile
  DBG(7);
  if (a.dbg && tid == 0 && cta_lin < 96) a.dbg[64 + 2 * cta_lin + 1] = global_ns();
#undef DBG
#undef RSTAMP
  trace_end(trace);
}

// ---------------------------------------------------------------------------
// Pixel-major variant for narrow convolutions (Cout <= NW = 32 / 64): the
// output pixels sit on UMMA M (128 per CTA) and the channels on N = NW, so a
// 32-channel stem conv does not pad its weights to 128 MMA rows (4x wasted
// tensor work in the channel-major kernel above).  Same producer structure
// (cp.async im2col into the 64-byte-swizzled X planes, convert warps for the
// tf32 lo plane, bulk-copied host-packed W hi/lo planes of NW rows, one MMA
// lane issuing 3 tcgen05.mma per 8-wide k step); no split-K (narrow layers
// are pixel-rich).  Epilogue: thread = pixel row (TMEM lane), its NW channel
// columns summed over the three accumulators, bias + activation, stored as
// 16-byte vectors of the pixel's output row.
constexpr int kPxStages = 4;

template <int NW, bool kVec>
__global__ void __launch_bounds__(kThreads, 1) conv2d_tc_tf32x3_px(TcArgs a, unsigned long long* trace) {
  constexpr int BM = 128;                           // pixels per CTA (UMMA M)
  constexpr uint32_t kWB = NW * kBKF * 4;           // one W plane per stage
  constexpr uint32_t kXB = BM * kBKF * 4;           // one X plane per stage
  constexpr uint32_t kStage = 2 * kWB + 2 * kXB;
  constexpr uint32_t kSbo = 512;
  constexpr int kRowGroups = BM / 8;
  constexpr int kRowsPerThread = kRowGroups / 4;
  constexpr uint32_t kIdesc = tc::instr_desc(2, 128, NW);
  constexpr uint32_t kTmemCols = 3 * NW <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPxStages * kStage);
  uint64_t* empty = full + kPxStages;
  uint64_t* landed = empty + kPxStages;
  uint64_t* accum = landed + kPxStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accum + 1);
  float* bias_s = reinterpret_cast<float*>(accum + 2);   // NW fp32

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * BM;
  const int nkb = a.kblocks;
  if (tid < NW) bias_s[tid] = (a.bias && tid < a.Cout) ? __ldg(a.bias + tid) : 0.f;   // parameter: pre-wait
  if (tid == 0) {
    for (int st = 0; st < kPxStages; ++st) {
      tc::mbar_init(&full[st], 32 * (kProducerWarps / 2) + 1);
      tc::mbar_init(&landed[st], 32 * (kProducerWarps / 2));
      tc::mbar_init(&empty[st], 1);
    }
    tc::mbar_init(accum, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, kTmemCols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp < kProducerWarps) {
    const bool gather = warp < kProducerWarps / 2;
    const int rw = warp & 3;
    const int r8 = lane & 7, cl = lane >> 3;
    auto x_off = [&](int j) -> uint32_t {
      return static_cast<uint32_t>(rw + 4 * j) * kSbo + r8 * 64u + static_cast<uint32_t>((cl ^ ((r8 >> 1) & 3)) * 16);
    };
    if (gather) {
      int pb[kRowsPerThread], pih[kRowsPerThread], piw[kRowsPerThread];
      const int ohw = a.OH * a.OW;
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j) {
        const int p = n0 + (rw + 4 * j) * 8 + r8;
        if (p < a.M) {
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
      const float* rowbase[kRowsPerThread];
#pragma unroll
      for (int j = 0; j < kRowsPerThread; ++j)
        rowbase[j] = a.in + (pb[j] >= 0 ? pb[j] * a.sN + pih[j] * a.sH + piw[j] * a.sW + a.in_coff : 0);
      int kc = cl * 4, dc = 0, dr = 0, dq = 0;
      if (kVec && kc < a.K) {
        dc = kc % a.Cin;
        const int rs = kc / a.Cin;
        dr = rs / a.S;
        dq = rs - dr * a.S;
      }
      pdl_wait();
      trace_begin(trace);
      for (int i = 0; i < nkb; ++i) {
        const int st = i % kPxStages;
        if (i >= kPxStages) tc::mbar_wait(&empty[st], ((i / kPxStages) - 1) & 1);
        const uint32_t xh = tc::smem_u32(smem + st * kStage + 2 * kWB);
        if constexpr (kVec) {
          const bool kin = kc < a.K;
          const int64_t koff = dr * a.sH + dq * a.sW + dc;
#pragma unroll
          for (int j = 0; j < kRowsPerThread; ++j) {
            const int ih = pih[j] + dr, iw = piw[j] + dq;
            const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
            cp_async16(xh + x_off(j), ok ? rowbase[j] + koff : a.in, ok);
          }
          kc += kBKF;
          dc += kBKF;
          while (dc >= a.Cin) {
            dc -= a.Cin;
            if (++dq == a.S) {
              dq = 0;
              ++dr;
            }
          }
        } else {
          const int kbase = i * kBKF + cl * 4;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = kbase + e;
            const bool kin = k < a.K;
            int c = 0, r = 0, q = 0;
            if (kin) {
              c = k % a.Cin;
              const int rs = k / a.Cin;
              r = rs / a.S;
              q = rs - r * a.S;
            }
#pragma unroll
            for (int j = 0; j < kRowsPerThread; ++j) {
              const int ih = pih[j] + r, iw = piw[j] + q;
              const bool ok = kin && pb[j] >= 0 && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W;
              const float* src = ok ? a.in + pb[j] * a.sN + ih * a.sH + iw * a.sW + c * a.sC + a.in_coff : a.in;
              cp_async4(xh + x_off(j) + 4 * e, src, ok);
            }
          }
        }
        tc::cp_async_arrive_noinc(&landed[st]);
      }
    } else {
      for (int i = 0; i < nkb; ++i) {
        const int st = i % kPxStages;
        tc::mbar_wait(&landed[st], (i / kPxStages) & 1);
        uint8_t* xh = smem + st * kStage + 2 * kWB;
        uint8_t* xl = xh + kXB;
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
          float4 v = *reinterpret_cast<const float4*>(xh + x_off(j));
          if (a.relu_in) {
            v.x = fmaxf(v.x, 0.f);
            v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f);
            v.w = fmaxf(v.w, 0.f);
            *reinterpret_cast<float4*>(xh + x_off(j)) = v;
          }
          float4 lo;
          lo.x = v.x - tc::trunc_tf32(v.x);
          lo.y = v.y - tc::trunc_tf32(v.y);
          lo.z = v.z - tc::trunc_tf32(v.z);
          lo.w = v.w - tc::trunc_tf32(v.w);
          *reinterpret_cast<float4*>(xl + x_off(j)) = lo;
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[st]);
      }
    }
  } else if (warp == kLoadWarp) {
    if (lane == 0) {
      if (nkb > kPxStages)   // the rest of the weight stream into L2 (see the channel-major kernel)
        tc::bulk_prefetch_l2(a.wpack + static_cast<int64_t>(kPxStages) * (2 * kWB / 4),
                             static_cast<uint64_t>(nkb - kPxStages) * 2 * kWB);
      for (int i = 0; i < nkb; ++i) {
        const int st = i % kPxStages;
        if (i >= kPxStages) tc::mbar_wait(&empty[st], ((i / kPxStages) - 1) & 1);
        tc::mbar_arrive_expect_tx(&full[st], 2 * kWB);
        tc::bulk_g2s(smem + st * kStage, a.wpack + static_cast<int64_t>(i) * (2 * kWB / 4), 2 * kWB, &full[st]);
      }
    }
  } else if (lane == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int st = i % kPxStages;
      tc::mbar_wait(&full[st], (i / kPxStages) & 1);
      tc::tc_fence_after();
      const uint32_t base = tc::smem_u32(smem + st * kStage);
      const uint32_t w_hi = base, w_lo = base + kWB, x_hi = base + 2 * kWB, x_lo = x_hi + kXB;
#pragma unroll
      for (int ks = 0; ks < kBKF / 8; ++ks) {
        const uint64_t ah = tc::smem_desc_sw64(x_hi + 32 * ks, kSbo);   // A = X (pixels on M)
        const uint64_t al = tc::smem_desc_sw64(x_lo + 32 * ks, kSbo);
        const uint64_t bh = tc::smem_desc_sw64(w_hi + 32 * ks, kSbo);   // B = W (channels on N)
        const uint64_t bl = tc::smem_desc_sw64(w_lo + 32 * ks, kSbo);
        const uint32_t acc = (i | ks) != 0;
        tc::mma_tf32(tmem, ah, bh, kIdesc, acc);
        tc::mma_tf32(tmem + NW, ah, bl, kIdesc, acc);
        tc::mma_tf32(tmem + 2 * NW, al, bh, kIdesc, acc);
      }
      tc::mma_commit(&empty[st]);
    }
    tc::mma_commit(accum);
  }
  __syncwarp();

  if (warp < 4) {
    tc::mbar_wait(accum, 0);
    tc::tc_fence_after();
    const int p = n0 + warp * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float* orow = a.out + static_cast<int64_t>(p) * a.out_cs + a.out_coff;
#pragma unroll
    for (int c8 = 0; c8 < NW / 8; ++c8) {
      float v[8], v1[8], v2[8];
      tc::tmem_ld8(trow + c8 * 8, v);
      tc::tmem_ld8(trow + NW + c8 * 8, v1);
      tc::tmem_ld8(trow + 2 * NW + c8 * 8, v2);
      if (p < a.M) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = apply_act(v[e] + (v1[e] + v2[e]) + bias_s[c8 * 8 + e], a.relu);
        const int c0 = c8 * 8;
        if (a.vec_out && c0 + 7 < a.Cout) {
          *reinterpret_cast<float4*>(orow + c0) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(orow + c0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c0 + e < a.Cout) orow[c0 + e] = v[e];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, kTmemCols);
  }
  trace_end(trace);
}

template <int NW>
constexpr size_t tc_px_smem_bytes() {
  return kPxStages * (2 * static_cast<size_t>(NW) * kBKF * 4 + 2 * 128 * kBKF * 4) + 512 + 1024;
}

template <int BN>
constexpr size_t tc_smem_bytes() {
  return tc_stages(BN) * (2 * kWBytes + 2 * static_cast<size_t>(BN) * kBKF * 4) + 512 + 1024;
}

struct TcVariant {
  int bn;
  const void* func[3];   // [kLoad]
  size_t smem;
};

template <int BN>
TcVariant make_tc() {
  return {BN,
          {reinterpret_cast<const void*>(&conv2d_tc_tf32x3<BN, kLoadScalar>),
           reinterpret_cast<const void*>(&conv2d_tc_tf32x3<BN, kLoadVec>),
           reinterpret_cast<const void*>(&conv2d_tc_tf32x3<BN, kLoadTma>)},
          tc_smem_bytes<BN>()};
}

const TcVariant* tc_variants(int* count) {
  static const TcVariant v[] = {make_tc<32>(), make_tc<64>(), make_tc<128>(), make_tc<256>()};
  *count = 4;
  return v;
}

constexpr size_t kPushMaxBytes = 48 * 1024;
constexpr size_t kSmemLimit = 232448 - 1024;   // 227 KB opt-in smem per CTA, minus static smem headroom
inline size_t attr_smem(size_t ring) { return std::min(ring + kPushMaxBytes, kSmemLimit); }

opara_status set_smem_attr(const TcVariant& v) {
  static bool done[4][3] = {};
  int idx = v.bn == 32 ? 0 : v.bn == 64 ? 1 : v.bn == 128 ? 2 : 3;
  for (int k = 0; k < 3; ++k) {
    if (done[idx][k]) continue;
    cudaError_t e = cudaFuncSetAttribute(v.func[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(attr_smem(v.smem)));
    if (e != cudaSuccess) return cuda_fail(e, "conv2d_tc smem attribute");
    done[idx][k] = true;
  }
  return OPARA_OK;
}

// How many clusters of `size` CTAs fit on the device at once (cached per
// kernel/size; without a device assume the 148-SM / one-CTA-per-SM bound).
int64_t max_active_clusters(const void* func, int size, size_t smem, size_t smem_attr) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int64_t> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(func, size, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int64_t result = 148 / size;
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0 &&
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_attr)) ==
          cudaSuccess) {
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

// Tile/split choice: pixel tile BN and split count so one conv spreads over
// about `target` CTAs (clusters of <= 8 splits), keeping >= 2 k-blocks each.
void choose_tiling(const TcArgs& a, int64_t target, int forced_bn, int forced_splits, int* bn_id,
                   int* splits) {
  const int mtiles = (a.Cout + 127) / 128;
  int id = forced_bn;
  if (id < 0) {
    // largest tile that still gives >= 32 output tiles, else the smallest
    id = 0;
    const int bns[4] = {32, 64, 128, 256};
    for (int k = 3; k >= 0; --k) {
      const int64_t tiles = static_cast<int64_t>((a.M + bns[k] - 1) / bns[k]) * mtiles;
      if (tiles >= 32 || k == 0) {
        id = k;
        break;
      }
    }
    // pixel counts just above a tile multiple waste a whole tile: step down
    if (id > 0 && a.M < 64 * 2) id = a.M > 32 ? 1 : 0;
  }
  const int bn = 32 << id;
  const int64_t base = static_cast<int64_t>((a.M + bn - 1) / bn) * mtiles;
  // one CTA per SM (the pipeline uses most of the 228 KB): stay within one
  // wave of 148 CTAs, a second wave would double the latency
  int64_t s = forced_splits > 0 ? forced_splits : std::max<int64_t>(1, target / base);
  s = std::min<int64_t>(s, kMaxSplits);
  s = std::min<int64_t>(s, std::max(1, a.kblocks / 2));
  s = std::max<int64_t>(1, s);
  *bn_id = id;
  *splits = static_cast<int>(s);
}

}  // namespace

// CONV2D with i[22] == 1 (engine "tc"): weights in p[1] are pre-packed by the
// host (engine.pack_conv_weights_tf32x3); everything else as in launch_conv2d.
opara_status launch_conv2d_tc(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                              LaunchCfg* cfg, bool dry) {
  TcArgs a;
  a.in = static_cast<const float*>(op.p[0]);
  a.wpack = static_cast<const float*>(op.p[1]);
  a.bias = static_cast<const float*>(op.p[2]);
  a.out = static_cast<float*>(op.p[3]);
  a.dbg = static_cast<unsigned long long*>(op.p[6]);
  a.N = (int)op.i[0]; a.H = (int)op.i[1]; a.W = (int)op.i[2]; a.Cin = (int)op.i[3];
  const int in_cs = (int)op.i[4];
  a.in_coff = (int)op.i[5];
  a.OH = (int)op.i[6]; a.OW = (int)op.i[7]; a.Cout = (int)op.i[8];
  a.out_cs = (int)op.i[9]; a.out_coff = (int)op.i[10];
  a.R = (int)op.i[11]; a.S = (int)op.i[12]; a.sh = (int)op.i[13]; a.sw = (int)op.i[14];
  a.ph = (int)op.i[15]; a.pw = (int)op.i[16];
  a.relu = conv_act_code(op.i[24], op.i[17]);   // `relu` carries the activation code
  a.relu_in = (int)op.i[25];
  if (op.i[18] != 0) return fail(OPARA_ERR_VALUE, "conv2d tc engine: fp32 (3xTF32) only");
  a.M = a.N * a.OH * a.OW;
  a.K = a.R * a.S * a.Cin;
  a.kblocks = (a.K + kBKF - 1) / kBKF;
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
  const bool vec = !nchw && a.Cin % 4 == 0 && in_cs % 4 == 0 && a.in_coff % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(a.in) % 16 == 0;
  a.vec_out = (a.out_cs % 4 == 0 && a.out_coff % 4 == 0 && reinterpret_cast<uintptr_t>(a.out) % 16 == 0) ? 1 : 0;
  if (op.variant == 4 || op.variant == 5) {
    // pixel-major tile for narrow convs: p[1] holds W packed with NW rows
    // (engine.pack_conv_weights_tf32x3(w, rows=NW)); no split-K
    const int nw = op.variant == 4 ? 32 : 64;
    if (a.Cout > nw) return fail(OPARA_ERR_VALUE, "conv2d_tc pixel-major tile: Cout exceeds the tile width");
    a.splits = 1;
    a.kb_per_split = a.kblocks;
    a.push = 0;
    LaunchCfg c;
    c.func = nw == 32 ? (vec ? reinterpret_cast<const void*>(&conv2d_tc_tf32x3_px<32, true>)
                             : reinterpret_cast<const void*>(&conv2d_tc_tf32x3_px<32, false>))
                      : (vec ? reinterpret_cast<const void*>(&conv2d_tc_tf32x3_px<64, true>)
                             : reinterpret_cast<const void*>(&conv2d_tc_tf32x3_px<64, false>));
    c.grid = dim3(ceil_div(a.M, 128), 1, 1);
    c.block = dim3(kThreads);
    c.smem = nw == 32 ? tc_px_smem_bytes<32>() : tc_px_smem_bytes<64>();
    c.tmem_cols = 3 * nw <= 128 ? 128 : 256;
    if (cfg) *cfg = c;
    if (dry) return OPARA_OK;
    static std::mutex mu;
    static std::map<const void*, bool> done;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!done[c.func]) {
        cudaError_t e = cudaFuncSetAttribute(c.func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(c.smem));
        if (e != cudaSuccess) return cuda_fail(e, "conv2d_tc_px smem attribute");
        done[c.func] = true;
      }
    }
    void* args[] = {&a, &trace};
    return launch_kernel(c, args, s);
  }
  int count = 0;
  const TcVariant* v = tc_variants(&count);
  int id = 0, splits = 1;
  const int64_t target = op.i[21] > 0 ? op.i[21] : 148;
  choose_tiling(a, target, (op.variant >= 0 && op.variant < count) ? op.variant : -1,
                op.i[19] > 1 ? static_cast<int>(op.i[19]) : op.i[19] == -1 ? 1 : 0, &id, &splits);
  // TMA im2col loads whenever the view allows them (16-channel taps, 16-byte
  // aligned view); the pixel tile of this variant is the map's pixel count
  const bool tma = !nchw && im2col_eligible(a.in, 4, a.Cin, in_cs, a.in_coff, a.H, a.W, a.OH, a.OW, a.sh, a.sw, a.ph, a.pw, kBKF);
  const void* func = v[id].func[tma ? kLoadTma : vec ? kLoadVec : kLoadScalar];
  if (splits > 1 && op.i[19] <= 1) {
    // clusters must be co-resident inside a GPC: keep every cluster in the
    // first wave (a second wave doubles the latency of the whole conv)
    const int64_t clusters = static_cast<int64_t>((a.M + v[id].bn - 1) / v[id].bn) * ((a.Cout + 127) / 128);
    while (splits > 1) {
      const int rp = ((v[id].bn + splits - 1) / splits + 3) / 4 * 4;
      const size_t rb = static_cast<size_t>(splits) * 128 * rp * 4;
      const bool pu = rb <= kPushMaxBytes && v[id].smem + rb <= kSmemLimit && op.i[26] == 0;
      const size_t sm = v[id].smem + (pu ? rb : 0);
      if (clusters <= max_active_clusters(func, splits, sm, attr_smem(v[id].smem))) break;
      --splits;
    }
  }
  a.kb_per_split = (a.kblocks + splits - 1) / splits;
  a.splits = (a.kblocks + a.kb_per_split - 1) / a.kb_per_split;
  // split-K reduction: push (st.async to the owning rank) when its buffer is small, else DSMEM pull
  a.rows_per = ((v[id].bn + a.splits - 1) / a.splits + 3) / 4 * 4;
  const size_t recv_bytes = static_cast<size_t>(a.splits) * 128 * a.rows_per * 4;
  a.push = (a.splits > 1 && recv_bytes <= kPushMaxBytes && v[id].smem + recv_bytes <= kSmemLimit &&
            op.i[26] == 0) ? 1 : 0;
  a.l2red = (a.splits > 1 && op.i[26] == 2) ? 1 : 0;
  a.ws = nullptr;
  LaunchCfg c;
  c.func = func;
  c.grid = dim3(ceil_div(a.M, v[id].bn), (a.Cout + 127) / 128, a.splits);
  c.block = dim3(kThreads);
  c.smem = v[id].smem + (a.push ? recv_bytes : 0);
  c.tmem_cols = v[id].bn >= 256 ? 512 : std::max(32, v[id].bn * 4);
  c.cluster = a.splits;
  c.workspace = a.l2red ? static_cast<size_t>(c.grid.x) * c.grid.y * c.grid.z * v[id].bn * 128 * 4 : 0;
  if (cfg) *cfg = c;
  if (dry) return OPARA_OK;
  if (a.l2red) {
    if (!op.p[7]) return fail(OPARA_ERR_INTERNAL, "conv2d_tc: split-K workspace missing");
    a.ws = static_cast<float*>(op.p[7]);
  }
  opara_status st = set_smem_attr(v[id]);
  if (st != OPARA_OK) return st;
  if (tma && !make_im2col_map(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, op.p[0], a.N, a.H, a.W, a.Cin, in_cs,
                              a.in_coff, a.OH, a.OW, a.sh, a.sw, a.ph, a.pw, kBKF, v[id].bn))
    return fail(OPARA_ERR_CUDA, "conv2d_tc: cuTensorMapEncodeIm2col failed");
  void* args[] = {&a, &trace};
  return launch_kernel(c, args, s, a.splits > 1 ? static_cast<unsigned>(a.splits) : 1u);
}

}  // namespace opara
