// tcgen05.mma issue rate vs commit cadence: the fp32 conv's k loop issues
// (N = 2 BN, N = BN) kind::tf32 MMA pairs per 8-wide k step and commits to the
// stage's mbarrier every 4 MMAs (one 16-deep stage).  Here one thread issues
// 96 MMAs per iteration with a tcgen05.commit every `per` MMAs, to separate
// the tensor pipe's per-MMA cost from the cost of committing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_10351_b200/csrc mma_commit.cu -o mma_commit
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace opara;

__device__ __forceinline__ uint64_t desc64(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (ignored for swizzled K-major)
  d |= static_cast<uint64_t>(512 >> 4) << 32;          // SBO 512 B (8 rows x 64 B)
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;                 // SW64
  return d;
}

template <int BN>
__global__ void bench(int iters, int per, int wait_each, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[64];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f800000u;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 64; ++k) tc::mbar_init(&bar[k], 1);
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (mode >= 3 && warp == 0) {
    // warp-uniform issue: every lane runs the loop, descriptors precomputed and
    // advanced with 64-bit adds, the MMA itself under elect.sync
    constexpr uint32_t id2 = tc::instr_desc(2, 128, 2 * BN), id1 = tc::instr_desc(2, 128, BN);
    const uint32_t a = tc::smem_u32(smem), b = a + 32768;
    const uint64_t da = desc64(a), dl = desc64(a + 16384), db = desc64(b), db2 = desc64(b + 8192);
    long long t0 = clock64();
    int c = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int m = 0; m < 96; m += 2) {
        const uint64_t off = (m & 2) ? 2 : 0;
        if (tc::elect_one()) {
          if (mode == 3) {
            tc::mma_tf32(tmem, da + off, db + off, id2, 1);
            tc::mma_tf32(tmem + 2 * BN, dl + off, db + off, id1, 1);
          } else {
            tc::mma_tf32(tmem, da + off, db + off, id1, 1);
            tc::mma_tf32(tmem + BN, da + off, db2 + off, id1, 1);
            tc::mma_tf32(tmem + 2 * BN, dl + off, db + off, id1, 1);
          }
        }
        __syncwarp();
        if ((m + 2) % per == 0) {
          if (tc::elect_one()) tc::mma_commit(&bar[c % 64]);
          __syncwarp();
          ++c;
        }
      }
    }
    if (tc::elect_one()) tc::mma_commit(&bar[c % 64]);
    __syncwarp();
    tc::mbar_wait(&bar[c % 64], (c / 64) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  } else if (mode == 5 && threadIdx.x == 0) {
    // single issuing thread, descriptors = loop-invariant bases + compile-time
    // offsets (the stage loop unrolled by the ring depth, as in the conv)
    constexpr uint32_t id2 = tc::instr_desc(2, 128, 2 * BN), id1 = tc::instr_desc(2, 128, BN);
    const uint32_t a = tc::smem_u32(smem);
    const uint64_t d0 = desc64(a);
    long long t0 = clock64();
    int c = 0;
    for (int it = 0; it < iters; ++it) {
      for (int m0 = 0; m0 < 96; m0 += 8) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {          // 4 "stages" of one 8-wide k step pair each
          const uint64_t st = d0 + s * (6144 >> 4);
#pragma unroll
          for (int ks = 0; ks < 1; ++ks) {
            tc::mma_tf32(tmem, st + 2 * ks, st + (32768 >> 4) + 2 * ks, id2, 1);
            tc::mma_tf32(tmem + 2 * BN, st + (16384 >> 4) + 2 * ks, st + (32768 >> 4) + 2 * ks, id1, 1);
          }
          if (per <= 4) { tc::mma_commit(&bar[c % 64]); ++c; }
        }
      }
    }
    tc::mma_commit(&bar[c % 64]);
    tc::mbar_wait(&bar[c % 64], (c / 64) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  } else if (mode < 3 && threadIdx.x == 0) {
    constexpr uint32_t id2 = tc::instr_desc(2, 128, 2 * BN), id1 = tc::instr_desc(2, 128, BN);
    const uint32_t a = tc::smem_u32(smem), b = a + 32768;
    long long t0 = clock64();
    int c = 0;
    for (int it = 0; it < iters; ++it) {
      for (int m = 0; m < 96; m += 2) {
        const uint64_t off = (m & 2) ? 2 : 0;     // next 32-byte k slice of the atom
        if (mode == 0) {          // the conv: hi x [hi; lo] (N = 2 BN), lo x hi (N = BN)
          tc::mma_tf32(tmem, desc64(a) + off, desc64(b) + off, id2, 1);
          tc::mma_tf32(tmem + 2 * BN, desc64(a + 16384) + off, desc64(b) + off, id1, 1);
        } else if (mode == 1) {   // same shape twice: lo x [hi; hi'] (N = 2 BN, half wasted)
          tc::mma_tf32(tmem, desc64(a) + off, desc64(b) + off, id2, 1);
          tc::mma_tf32(tmem + 2 * BN, desc64(a + 16384) + off, desc64(b) + off, id2, 1);
        } else {                  // three N = BN MMAs (hh, hl, lh), one shape
          tc::mma_tf32(tmem, desc64(a) + off, desc64(b) + off, id1, 1);
          tc::mma_tf32(tmem + BN, desc64(a) + off, desc64(b + 8192) + off, id1, 1);
          tc::mma_tf32(tmem + 2 * BN, desc64(a + 16384) + off, desc64(b) + off, id1, 1);
        }
        if ((m + 2) % per == 0) {
          tc::mma_commit(&bar[c % 64]);
          if (wait_each) tc::mbar_wait(&bar[c % 64], (c / 64) & 1);
          ++c;
        }
      }
    }
    tc::mma_commit(&bar[c % 64]);
    tc::mbar_wait(&bar[c % 64], (c / 64) & 1);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

template <int BN>
void run(long long* d, int per, int wait_each, int mode, int smem_kb = 100) {
  auto f = bench<BN>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  const int iters = 20;
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    f<<<148, 128, smem_kb * 1024>>>(iters, per, wait_each, mode, d);
    cudaDeviceSynchronize();
  }
  cudaError_t e = cudaGetLastError();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("smem %3d KB mode %d (%s) BN=%3d commit every %2d pairs, %s: %6.1f cyc per 8-wide k step  %s\n", smem_kb, mode,
         mode == 0 ? "N=2BN + N=BN   " : mode == 1 ? "N=2BN + N=2BN  " : mode == 2 ? "3 x N=BN       " :
         mode == 3 ? "warp N=2BN+N=BN" : mode == 4 ? "warp 3 x N=BN  " : "unrolled consts", BN, per / 2,
         wait_each ? "wait each" : "no wait  ", h / (iters * 48.0), cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int kb : {140})
    for (int mode : {0, 5})
      for (int per : {4, 96}) { run<32>(d, per, 0, mode, kb); run<64>(d, per, 0, mode, kb); }
  return 0;
}
