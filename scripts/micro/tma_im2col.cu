// Probe of TMA im2col-mode semantics (cp.async.bulk.tensor.4d ... .im2col):
// the input encodes (n, h, w, c) in every int32 element; each case loads one
// box (channelsPerPixel x pixelsPerColumn) and prints which input pixel / channel
// landed in every smem row (0 = out-of-bounds fill).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_im2col tma_im2col.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__global__ void k_load(const __grid_constant__ CUtensorMap map, int* out, int c, int w, int h, int n, int offw, int offh, int bytes) {
  extern __shared__ __align__(1024) int sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t bb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes));
    const uint16_t ow = static_cast<uint16_t>(offw), oh = static_cast<uint16_t>(offh);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};"
        ::"r"(sb), "l"(&map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bb), "h"(ow), "h"(oh) : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(bb) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  struct Case { const char* name; int N, H, W, C, lw, lh, uw, uh, cpp, ppc, sw, sh, c, w, h, n, offw, offh; };
  // lower/upper corners given as {W, H} (array index 0 = W) -- the probe checks this
  Case cases[] = {
    {"3x3 p1 s1 H=W=5, start (w=-1,h=-1) off(0,0)", 1, 5, 5, 32, -1, -1, -1, -1, 16, 32, 1, 1, 0, -1, -1, 0, 0, 0},
    {"3x3 p1 s1 H=W=5, start (w=-1,h=-1) off(2,1) c=16", 1, 5, 5, 32, -1, -1, -1, -1, 16, 32, 1, 1, 16, -1, -1, 0, 2, 1},
    {"3x3 p1 s1 H=W=5, start pixel 7 = (oh1,ow2)->(w=1,h=0)", 1, 5, 5, 32, -1, -1, -1, -1, 16, 16, 1, 1, 0, 1, 0, 0, 0, 0},
    {"1x7 pw3 ph0 H=W=5 (lw=-3,lh=0,uw=-3,uh=0), start(w=-3,h=0) off(3,0)", 1, 5, 5, 32, -3, 0, -3, 0, 16, 32, 1, 1, 0, -3, 0, 0, 3, 0},
    {"3x3 p0 s2 H=W=7 (OH=3), start(0,0) off(0,0)", 2, 7, 7, 32, 0, 0, -2, -2, 16, 24, 2, 2, 0, 0, 0, 0, 0, 0},
    {"3x3 p0 s2 H=W=7, start(0,0) off(2,2) n wrap", 2, 7, 7, 32, 0, 0, -2, -2, 16, 24, 2, 2, 0, 0, 0, 0, 2, 2},
    // subsample(x, 1) -> 1x1 stride 2: pad -1, box [1, W] (past the edge), OW = (W+1)/2
    {"1x1 s2 pad -1 H=W=7 (lower 1, upper 1), start(1,1)", 1, 7, 7, 32, 1, 1, 1, 1, 16, 16, 2, 2, 0, 1, 1, 0, 0, 0},
    {"1x1 s2 pad -1 H=W=7 (lower 1, upper -1), start(1,1)", 1, 7, 7, 32, 1, 1, -1, -1, 16, 16, 2, 2, 0, 1, 1, 0, 0, 0},
    {"1x1 s2 pad 0 H=W=7 (lower 0, upper 0), start(0,0)", 1, 7, 7, 32, 0, 0, 0, 0, 16, 16, 2, 2, 0, 0, 0, 0, 0, 0},
  };
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int idx = -1;
  for (auto& cs : cases) {
    if (only >= 0 && ++idx != only) continue;
    const size_t ne = (size_t)cs.N * cs.H * cs.W * cs.C;
    std::vector<int> hin(ne);
    for (int n = 0; n < cs.N; ++n) for (int h = 0; h < cs.H; ++h) for (int w = 0; w < cs.W; ++w) for (int c = 0; c < cs.C; ++c)
      hin[(((size_t)n * cs.H + h) * cs.W + w) * cs.C + c] = 0x40000000 | (n << 24) | (h << 16) | (w << 8) | c;
    int* din; int* dout;
    cudaMalloc(&din, ne * 4); cudaMalloc(&dout, 1 << 20);
    cudaMemcpy(din, hin.data(), ne * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[4] = {(cuuint64_t)cs.C, (cuuint64_t)cs.W, (cuuint64_t)cs.H, (cuuint64_t)cs.N};
    cuuint64_t strides[3] = {(cuuint64_t)cs.C * 4, (cuuint64_t)cs.C * 4 * cs.W, (cuuint64_t)cs.C * 4 * cs.W * cs.H};
    int lower[2] = {cs.lw, cs.lh}, upper[2] = {cs.uw, cs.uh};
    cuuint32_t es[4] = {1, (cuuint32_t)cs.sw, (cuuint32_t)cs.sh, 1};
    CUresult r = cuTensorMapEncodeIm2col(&map, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, din, dims, strides, lower, upper,
                                         cs.cpp, cs.ppc, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("== %s: encode %d\n", cs.name, (int)r);
    if (r) continue;
    const int bytes = cs.cpp * cs.ppc * 4;
    k_load<<<1, 128, bytes + 1024>>>(map, dout, cs.c, cs.w, cs.h, cs.n, cs.offw, cs.offh, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("   launch error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<int> ho(bytes / 4);
    cudaMemcpy(ho.data(), dout, bytes, cudaMemcpyDeviceToHost);
    printf("   ");
    for (int p = 0; p < cs.ppc; ++p) {
      const int v = ho[p * cs.cpp], v1 = ho[p * cs.cpp + cs.cpp - 1];
      if (!v) printf("[oob] ");
      else printf("[n%d h%d w%d c%d-%d] ", (v >> 24) & 63, (v >> 16) & 255, (v >> 8) & 255, v & 255, v1 & 255);
    }
    printf("\n");
    cudaFree(din); cudaFree(dout);
  }
  return 0;
}
