// Dependent-chain latency per kernel inside a CUDA graph with PDL, on B200:
// what a short kernel on the critical path costs before doing any work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_chain.cu -o pdl_chain
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

struct P { float* buf; int mode; };

__global__ void k(P p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (p.mode & 4) {  // TMEM alloc
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  if (p.mode & 8) {  // mbarrier init
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float v = 0.f;
  if (p.mode & 1) {  // dependent global read + write (L2)
    v = p.buf[blockIdx.x * blockDim.x + threadIdx.x];
    p.buf[blockIdx.x * blockDim.x + threadIdx.x] = v + 1.f;
  }
  if (p.mode & 2) {  // cluster barrier
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (p.mode & 4) {
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
  }
  if (v == 12345.f) sm[0] = 1;
}

int main(int argc, char** argv) {
  float* buf;
  cudaMalloc(&buf, 1 << 24);
  cudaMemset(buf, 0, 1 << 24);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int reps = 200;
  struct Case { const char* name; int ctas, threads, smem_kb, cluster, mode, pdl; };
  Case cases[] = {
      {"empty nopdl", 148, 128, 0, 1, 0, 0},     {"empty pdl", 148, 128, 0, 1, 0, 1},
      {"rw pdl", 148, 128, 0, 1, 1, 1},          {"rw 16cta", 16, 256, 0, 1, 1, 1},
      {"rw smem80", 148, 192, 80, 1, 1, 1},      {"rw cluster4", 148, 192, 80, 4, 3, 1},
      {"rw cl4 tmem", 148, 192, 80, 4, 7, 1},    {"rw cl4 tmem mbar", 148, 192, 80, 4, 15, 1},
      {"rw cl8 tmem mbar", 144, 192, 80, 8, 15, 1}, {"rw tmem", 148, 192, 80, 1, 5, 1},
      {"rw 296cta", 296, 192, 80, 1, 1, 1},
  };
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto& c : cases) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(c.ctas);
      lc.blockDim = dim3(c.threads);
      lc.dynamicSmemBytes = c.smem_kb * 1024;
      lc.stream = s;
      cudaLaunchAttribute at[2];
      int n = 0;
      if (c.pdl) { at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[n].val.programmaticStreamSerializationAllowed = 1; ++n; }
      if (c.cluster > 1) { at[n].id = cudaLaunchAttributeClusterDimension; at[n].val.clusterDim.x = c.cluster; at[n].val.clusterDim.y = 1; at[n].val.clusterDim.z = 1; ++n; }
      lc.attrs = at;
      lc.numAttrs = n;
      P p{buf, c.mode};
      cudaLaunchKernelEx(&lc, k, p);
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("%-20s error %s\n", c.name, cudaGetErrorString(e)); cudaGetLastError(); continue; }
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int t = 0; t < 5; ++t) {
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-20s ctas=%3d thr=%3d smem=%3dKB cluster=%d : %.2f us/kernel\n", c.name, c.ctas, c.threads, c.smem_kb,
           c.cluster, 1000.f * best / reps);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
