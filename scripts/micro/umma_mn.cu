// Probe of the MN-major B operand (tcgen05 kind::f16, SWIZZLE_64B): O = P V
// with V stored in its natural [key][d] row layout (no transpose).  Layout:
// 8-key x 64-byte (32 d) atoms, MN atoms 512 B apart, key groups 1024 B apart;
// the descriptor is tried as (LBO, SBO) = (512, 1024) and (1024, 512).
// nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2312_10351_b200/csrc -o umma_mn umma_mn.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc_common.cuh"
using namespace opara;

__device__ __forceinline__ uint64_t desc_mn_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}
__device__ __forceinline__ uint32_t sw64(int rows, int row, int c16) {
  const int kb = c16 >> 2, cw = c16 & 3, r8 = row & 7;
  return static_cast<uint32_t>(kb * rows * 64 + (row >> 3) * 512 + r8 * 64 + ((cw ^ ((r8 >> 1) & 3)) << 4));
}
__device__ __forceinline__ uint32_t mn_off(int key, int c16) {   // V[key][8*c16 .. +7]
  const int r = key & 7;
  return static_cast<uint32_t>((c16 >> 2) * 512 + (key >> 3) * 1024 + r * 64 + (((c16 & 3) ^ ((r >> 1) & 3)) << 4));
}

__global__ void k(const __nv_bfloat16* P, const __nv_bfloat16* V, float* O, int lbo, int sbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ps = smem;              // 32 KB
  uint8_t* vs = smem + 32768;      // 16 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int u = tid; u < 128 * 16; u += 128) {
    const int row = u >> 4, c16 = u & 15;
    *reinterpret_cast<uint4*>(ps + sw64(128, row, c16)) = *reinterpret_cast<const uint4*>(P + row * 128 + c16 * 8);
  }
  for (int u = tid; u < 128 * 8; u += 128) {
    const int key = u >> 3, c16 = u & 7;
    *reinterpret_cast<uint4*>(vs + mn_off(key, c16)) = *reinterpret_cast<const uint4*>(V + key * 64 + c16 * 8);
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 64);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  constexpr uint32_t id = tc::instr_desc(1, 128, 64) | (1u << 16);   // B MN-major
  if (tid == 0) {
    for (int s = 0; s < 8; ++s)
      tc::mma_f16(tmem, tc::smem_desc_sw64(tc::smem_u32(ps) + (s >> 1) * 128 * 64 + (s & 1) * 32, 512),
                  desc_mn_sw64(tc::smem_u32(vs) + s * 2 * 1024, lbo, sbo), id, s != 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int c8 = 0; c8 < 8; ++c8) {
    float v[8];
    tc::tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c8 * 8, v);
    for (int e = 0; e < 8; ++e) O[(warp * 32 + lane) * 64 + c8 * 8 + e] = v[e];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 64); }
}

int main() {
  std::vector<__nv_bfloat16> hp(128 * 128), hv(128 * 64);
  std::vector<float> fp(128 * 128), fv(128 * 64);
  srand(1);
  for (int i = 0; i < 128 * 128; ++i) { hp[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fp[i] = __bfloat162float(hp[i]); }
  for (int i = 0; i < 128 * 64; ++i) { hv[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fv[i] = __bfloat162float(hv[i]); }
  __nv_bfloat16 *dp, *dv; float* dout;
  cudaMalloc(&dp, hp.size() * 2); cudaMalloc(&dv, hv.size() * 2); cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(dp, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int variants[2][2] = {{512, 1024}, {1024, 512}};
  for (auto& vr : variants) {
    cudaMemset(dout, 0, 128 * 64 * 4);
    k<<<1, 128, 64 * 1024>>>(dp, dv, dout, vr[0], vr[1]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("lbo %d sbo %d: error %s\n", vr[0], vr[1], cudaGetErrorString(e)); return 1; }
    std::vector<float> o(128 * 64);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int q = 0; q < 128; ++q) for (int d = 0; d < 64; ++d) {
      double ref = 0;
      for (int kk = 0; kk < 128; ++kk) ref += (double)fp[q * 128 + kk] * fv[kk * 64 + d];
      maxerr = fmax(maxerr, fabs(ref - o[q * 64 + d]));
    }
    printf("lbo %d sbo %d: max abs err %.3e (O[0][0..3] = %g %g %g %g)\n", vr[0], vr[1], maxerr, o[0], o[1], o[2], o[3]);
  }
  return 0;
}
