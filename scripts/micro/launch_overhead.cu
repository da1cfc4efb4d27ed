// Fixed per-launch costs on B200 inside a CUDA graph: empty kernel vs large
// dynamic smem vs TMEM alloc/dealloc vs cluster launch.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) { if (p && threadIdx.x == 1000) p[0] = 1; }

__global__ void k_smem(int* p) {
  extern __shared__ uint8_t sm[];
  if (threadIdx.x == 0) sm[0] = 1;
  __syncthreads();
  if (p && sm[1] == 42) p[0] = 1;
}

__global__ void k_tmem(int* p) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = slot;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t));
  if (p && sm[1] == 42) p[0] = 1;
}

template <typename F>
float time_graph(F launch, int reps) {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) launch(s);
  cudaError_t ce = cudaStreamEndCapture(s, &g);
  if (ce != cudaSuccess) { printf("capture failed: %s\n", cudaGetErrorString(ce)); fflush(stdout); cudaGetLastError(); return -1.f; }
  ce = cudaGraphInstantiate(&ge, g, 0);
  if (ce != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(ce)); fflush(stdout); cudaGetLastError(); return -1.f; }
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return best * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int reps = 50;
  const char* mode = argc > 1 ? argv[1] : "empty";
  const int ctas = argc > 2 ? atoi(argv[2]) : 25;
  const int kb = argc > 3 ? atoi(argv[3]) : 0;
  const int cz = argc > 4 ? atoi(argv[4]) : 1;
  cudaFree(0);
  cudaError_t e1 = cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaError_t e2 = cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  if (e1 || e2) printf("attr errors %d %d\n", (int)e1, (int)e2);
  float us = -1;
  if (!strcmp(mode, "empty")) us = time_graph([&](cudaStream_t s) { k_empty<<<ctas, 160, 0, s>>>(nullptr); }, reps);
  else if (!strcmp(mode, "smem")) us = time_graph([&](cudaStream_t s) { k_smem<<<ctas, 160, kb * 1024, s>>>(nullptr); }, reps);
  else if (!strcmp(mode, "tmem")) us = time_graph([&](cudaStream_t s) {
        if (cz == 1) { k_tmem<<<ctas, 160, kb * 1024, s>>>(nullptr); return; }
        cudaLaunchConfig_t lc = {}; lc.gridDim = dim3(1, 1, ctas); lc.blockDim = dim3(160); lc.dynamicSmemBytes = kb * 1024; lc.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = cz;
        lc.attrs = at; lc.numAttrs = 1; int* np = nullptr; void* args[] = {&np};
        cudaLaunchKernelExC(&lc, (const void*)k_tmem, args); }, reps);
  printf("%-6s ctas=%4d smem=%3dKB cluster=%d : %.2f us/launch\n", mode, ctas, kb, cz, us);
  return 0;
}
