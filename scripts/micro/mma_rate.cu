// tcgen05.mma issue-to-completion rate for the conv engines' tile shapes, one
// CTA per SM, operands already in shared memory (no loads): is a 3xTF32
// k-stage (2 k-steps x 3 MMAs, M=128, N=BN) bound by the tensor pipe?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_10351_b200/csrc mma_rate.cu -o mma_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

using namespace opara;

template <int KIND, int N>   // KIND 2 = tf32 (K=8 / MMA), 1 = bf16 (K=16 / MMA)
__global__ void bench(int stages, int nacc, int ksteps, int per_stage, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[64];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) tc::mbar_init(&bars[i], 1);
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::instr_desc(KIND, 128, N);
    const uint32_t base = tc::smem_u32(smem);
    long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      const uint32_t w = base + (s & 3) * 40960, x = w + 32768;
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t a = tc::smem_desc_sw64(w + 32 * ks, 512);
        const uint64_t b = tc::smem_desc_sw64(x + 32 * ks, 512);
        for (int m = 0; m < per_stage; ++m) {
          const uint32_t d = tmem + (m % nacc) * N;
          if (KIND == 2) tc::mma_tf32(d, a, b, idesc, 1);
          else tc::mma_f16(d, a, b, idesc, 1);
        }
      }
      tc::mma_commit(&bars[s & 63]);
    }
    long long t1 = clock64();
    tc::mbar_wait(&bars[(stages - 1) & 63], ((stages - 1) / 64) & 1);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 512); }
}

template <int KIND, int N>
void run(const char* name, int nacc, int ksteps, int per_stage, long long* d) {
  auto f = bench<KIND, N>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int stages = 60;
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) {
    f<<<148, 128, 170 * 1024>>>(stages, nacc, ksteps, per_stage, d);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const int mmas = stages * ksteps * per_stage;
  printf("%-28s N=%3d acc=%d: %6.1f cyc/MMA issue, %6.1f cyc/MMA complete, %7.1f cyc/stage (%d MMAs/stage) %s\n",
         name, N, nacc, double(h[0]) / mmas, double(h[1]) / mmas, double(h[1]) / stages, ksteps * per_stage,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<2, 32>("tf32 3xTF32 stage", 3, 2, 3, d);
  run<2, 64>("tf32 3xTF32 stage", 3, 2, 3, d);
  run<2, 128>("tf32 3xTF32 stage", 3, 2, 3, d);
  run<2, 64>("tf32 1 acc", 1, 2, 3, d);
  run<2, 64>("tf32 4 ksteps x 3", 3, 4, 3, d);
  run<2, 256>("tf32 N256", 2, 2, 3, d);
  run<1, 64>("bf16 3-term stage", 3, 1, 3, d);
  run<1, 64>("bf16 1 MMA/stage x2ks", 1, 2, 1, d);
  run<1, 128>("bf16 3-term stage", 3, 1, 3, d);
  run<1, 256>("bf16 N256 x4ks", 1, 4, 1, d);
  return 0;
}
