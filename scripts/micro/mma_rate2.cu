// tcgen05.mma rate vs operand swizzle mode, N and M (one CTA per SM, operands
// resident in shared memory, 12 MMAs per commit).  Layout types (sm_100
// descriptor bits 61-63): 0 none (interleaved 8x16B core matrices), 6 SW32,
// 4 SW64, 2 SW128.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_10351_b200/csrc mma_rate2.cu -o mma_rate2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace opara;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

template <int KIND, int M, int N, int LAYOUT>
__global__ void bench(int iters, int vary, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f800000u;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::instr_desc(KIND == 3 ? 2 : KIND, M, N);
    const uint32_t a = tc::smem_u32(smem), b = a + 65536;
    // row pitch of one 8-row group: none -> 256 B (2 core matrices of 8x16 along K), swizzles: 8 x swizzle bytes
    constexpr uint32_t sw = LAYOUT == 2 ? 128 : LAYOUT == 4 ? 64 : LAYOUT == 6 ? 32 : 0;
    constexpr uint32_t sbo = sw ? 8 * sw : 256;
    constexpr uint32_t lbo = sw ? 16 : 128;
    const uint64_t da = desc(a, lbo, sbo, LAYOUT), db = desc(b, lbo, sbo, LAYOUT);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int m = 0; m < 12; ++m) {
        // vary 0: same operands; 1: next 32-byte k slice (m % 2) of the atom;
        // 2: a different 16 KB buffer per MMA (m % 4); 3: both
        const uint64_t off = ((vary & 1) ? (uint64_t)((m % 2) * 32 >> 4) : 0) +
                             ((vary & 2) ? (uint64_t)(((m % 4) * 16384) >> 4) : 0);
        if (KIND == 3) {   // the conv's pair: N then N/2 alternating (tf32)
          constexpr uint32_t idesc_h = tc::instr_desc(2, M, N / 2);
          if (m % 2 == 0) tc::mma_tf32(tmem, da + off, db + off, tc::instr_desc(2, M, N), 1);
          else tc::mma_tf32(tmem + N, da + off, db + off, idesc_h, 1);
        } else if (KIND == 2) tc::mma_tf32(tmem + (m % 2) * N, da + off, db + off, idesc, 1);
        else tc::mma_f16(tmem + (m % 2) * N, da + off, db + off, idesc, 1);
      }
      tc::mma_commit(&bar);
    }
    long long t1 = clock64();
    tc::mbar_wait(&bar, (iters - 1) & 1);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

template <int KIND, int M, int N, int LAYOUT>
void run(long long* d, int vary = 0) {
  auto f = bench<KIND, M, N, LAYOUT>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const int iters = 40;
  long long h[2] = {0, 0};
  for (int rep = 0; rep < 3; ++rep) {
    f<<<148, 128, 140 * 1024>>>(iters, vary, d);
    cudaDeviceSynchronize();
  }
  cudaError_t e = cudaGetLastError();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = iters * 12.0;
  const double macs = double(M) * (KIND == 3 ? 0.75 * N : N) * (KIND >= 2 ? 8 : 16);
  printf("vary=%d %s M=%3d N=%3d layout=%d: %6.1f cyc/MMA (issue %6.1f)  %7.1f MAC/cyc  %s\n", vary, KIND == 3 ? "pair" : KIND == 2 ? "tf32" : "bf16", M, N,
         LAYOUT, h[1] / n, h[0] / n, macs / (h[1] / n), cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int v = 0; v < 4; v += 3) {
    run<2, 128, 64, 4>(d, v); run<2, 128, 128, 4>(d, v);
    run<3, 128, 64, 4>(d, v); run<3, 128, 128, 4>(d, v); run<3, 128, 256, 4>(d, v);
  }
  return 0;
}
