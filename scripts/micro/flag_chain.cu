// Hand-off latency of a dependent kernel chain inside a CUDA graph (PDL on):
// griddepcontrol.wait (grid completion + flush) vs a release/acquire counter
// per kernel (each CTA adds 1 after its stores; the next kernel's CTAs spin
// until the counter reaches this replay's target, generation from an entry counter).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 flag_chain.cu -o flag_chain
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct P { float* buf; unsigned* entered; unsigned* done; const unsigned* prev_done; unsigned prev_grid; int mode; };

__global__ void k(P p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ unsigned gen;
  if (threadIdx.x == 0) gen = atomicAdd(p.entered, 1u) / gridDim.x;
  __syncthreads();
  if (p.mode == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else if (p.prev_done) {
    if (threadIdx.x == 0) {
      const unsigned target = (gen + 1) * p.prev_grid;
      unsigned v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.prev_done) : "memory");
        if (v >= target) break;
        if (p.mode == 2) __nanosleep(32);
      }
    }
    __syncthreads();
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  p.buf[i] = p.buf[i] + 1.f;
  __syncthreads();
  if (threadIdx.x == 0 && p.mode != 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done) : "memory");
  }
}

int main() {
  float* buf;
  unsigned* ctr;
  const int reps = 200;
  cudaMalloc(&buf, 1 << 24);
  cudaMemset(buf, 0, 1 << 24);
  cudaMalloc(&ctr, 2 * reps * sizeof(unsigned));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Case { const char* name; int ctas, threads, smem_kb, mode; };
  Case cases[] = {{"griddepcontrol.wait", 148, 128, 0, 0}, {"flag spin", 148, 128, 0, 1},
                  {"flag nanosleep", 148, 128, 0, 2},     {"wait smem100", 148, 128, 100, 0},
                  {"flag smem100", 148, 128, 100, 1},     {"wait 40cta", 40, 256, 100, 0},
                  {"flag 40cta", 40, 256, 100, 1},        {"wait smem200", 148, 128, 200, 0},
                  {"flag smem200", 148, 128, 200, 1}};
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (auto& c : cases) {
    cudaMemset(ctr, 0, 2 * reps * sizeof(unsigned));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(c.ctas);
      lc.blockDim = dim3(c.threads);
      lc.dynamicSmemBytes = c.smem_kb * 1024;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      P p{buf, ctr + 2 * i, ctr + 2 * i + 1, i ? ctr + 2 * (i - 1) + 1 : nullptr, (unsigned)c.ctas, c.mode};
      cudaLaunchKernelEx(&lc, k, p);
    }
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("%-20s error %s\n", c.name, cudaGetErrorString(e)); return 1; }
    cudaGraphLaunch(ge, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { printf("%-20s run error %s\n", c.name, cudaGetErrorString(e)); return 1; }
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
    printf("%-22s ctas=%3d thr=%3d smem=%3dKB : %.3f us/kernel\n", c.name, c.ctas, c.threads, c.smem_kb, 1000.f * best / reps);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
