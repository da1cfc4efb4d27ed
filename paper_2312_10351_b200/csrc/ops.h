// Operator registry shared by the executor and the kernel families.
//
// Parameter layout of opara_op per kind (all shapes NHWC, batch-major; a
// "channel view" is (buffer, cstride, coff): element (pixel q, channel c)
// lives at buffer[q * cstride + coff + c], which is how concat is eliminated —
// producers store straight into their slice of the concatenated buffer).
//
// CONV2D       i: 0 N, 1 H, 2 W, 3 Cin, 4 in_cstride, 5 in_coff,
//                 6 OH, 7 OW, 8 Cout, 9 out_cstride, 10 out_coff,
//                 11 R, 12 S, 13 stride_h, 14 stride_w, 15 pad_h, 16 pad_w,
//                 17 relu, 18 dtype (0 f32), 19 split_k (> 1 forced, -1 forced none, else auto),
//                 20 in_nchw (1: input is a dense NCHW tensor, e.g. the graph input),
//                 21 target CTAs for split-K (0 = default), 22 engine (0 SIMT fp32,
//                 1 tcgen05 3xTF32, 2 tcgen05 bf16), 23 output dtype, 24 activation
//                 (0 none, 1 ReLU, 2 GELU, 3 tanh), 25 relu_in (ReLU fused on the input),
//                 26 split-K reduction (0 push partials to the owner CTA when its buffer
//                 fits, 1 pull over DSMEM after a cluster barrier, 2 partial tiles through
//                 an L2 workspace in p[7] after a cluster barrier),
//                 folded LayerNorm y = LN(o + r) (bf16 engine, conv_tc_bf16.cu BfArgs):
//                 27 producer epilogue (p[4] residual r view, i[28] its cstride, p[6] stats
//                 [T][Cout/128][2] of o + r), 29 LayerNorm on load (p[4] stats, i[31] stats
//                 tiles, p[5] gamma|beta fp32 [2][Cin], f[0] eps, i[32] r view address,
//                 i[33] its cstride, p[6] + i[30] normalised-rows view written, or null)
//              p: 0 in, 1 weight: engine 0 [R*S*Cin][Cout] (k = (r*S + s)*Cin + c);
//                 engine 1 packed tf32 hi/lo UMMA images (conv_tc.cu), 2 bias [Cout], 3 out,
//                 7 split-K workspace (executor-owned)
//              variant: tile id (tile width 32 << id), -1 = auto
// MAXPOOL2D /  i: 0 N, 1 H, 2 W, 3 C, 4 in_cstride, 5 in_coff, 6 OH, 7 OW, 8 out_cstride,
// AVGPOOL2D       9 out_coff, 10 kh, 11 kw, 12 sh, 13 sw, 14 ph, 15 pw,
//                 16 count_include_pad (avg), 18 dtype
//              p: 0 in, 3 out
// GLOBAL_AVGPOOL i: 0 N, 1 H, 2 W, 3 C, 4 in_cstride, 5 in_coff, 8 out_cstride (0 = C),
//                 17 relu_in, 18 dtype;  p: 0 in, 3 out fp32 (first channel of the output view)
// PACK_INPUT   i: 0 N, 1 H, 2 W, 3 C, 4 Cp (padded channels: multiple of 8 bf16 / 4 fp32),
//              18 out dtype;  p: 0 in (fp32 NCHW), 3 out (NHWC [N][H][W][Cp])
// ADD / COPY / RELU, DWCONV2D, FIELD_EMBEDDING / FIRST_ORDER / FM: see the header comment of
//              elementwise.cu, dwconv.cu and deepfm.cu
// LINEAR       i: 0 M (rows), 1 K, 2 N (out features), 3 act (0 none, 1 relu, 2 gelu, 3 tanh),
//                 4 x_stride, 5 y_stride, 18 dtype
//              p: 0 x [M][K], 1 W [N][K], 2 bias [N] (nullable), 3 y [M][N]
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "opara.h"

namespace opara {

struct LaunchCfg {
  const void* func = nullptr;
  dim3 grid{1, 1, 1};
  dim3 block{1, 1, 1};
  size_t smem = 0;
  size_t workspace = 0;  // private device scratch the executor allocates into op.p[7]
  int tmem_cols = 0;     // TMEM columns one block allocates (co-residency: 512 per SM)
  int cluster = 1;       // thread-block cluster size of the launch
};

// Split-K workspace: `floats` partial values, then one u32 arrival counter per
// output tile (zeroed once at allocation; the last arrival re-zeroes it).
inline size_t splitk_workspace_bytes(int64_t floats, int64_t tiles) {
  return static_cast<size_t>(((floats * 4 + 255) / 256) * 256 + tiles * 4);
}
inline unsigned* splitk_counters(void* ws, int64_t floats) {
  return reinterpret_cast<unsigned*>(static_cast<char*>(ws) + ((floats * 4 + 255) / 256) * 256);
}

// trace: nullable device pointer to two u64 slots (min start, max end ns).
// dry: only fill `cfg` (no device access), used for profiles on CPU hosts.
using Launcher = opara_status (*)(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                                  LaunchCfg* cfg, bool dry);

opara_status launch_conv2d(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_conv2d_tc(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_conv2d_tc_bf16(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_pool2d(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_global_avgpool(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*,
                                   bool);
opara_status launch_linear(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_rows(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_attention(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_elementwise(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_pack_input(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_dwconv2d(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);
opara_status launch_deepfm(const opara_op&, cudaStream_t, unsigned long long*, LaunchCfg*, bool);

// Dispatch on op.kind.
opara_status launch_op(const opara_op& op, cudaStream_t s, unsigned long long* trace,
                       LaunchCfg* cfg, bool dry);

opara_status cuda_fail(cudaError_t e, const char* what);

// Launch `cfg` on `s` with programmatic dependent launch (PDL) enabled, and as
// a (1, 1, cluster_z) thread-block cluster when cluster_z > 1.  Every kernel
// of the executor starts with griddepcontrol.launch_dependents and executes
// griddepcontrol.wait before its first read of a predecessor's output, so a
// same-stream successor's prologue (barrier init, TMEM alloc, weight
// prefetch) overlaps this kernel's tail inside the captured graph.
opara_status launch_kernel(const LaunchCfg& cfg, void** args, cudaStream_t s, unsigned cluster_z = 1);
opara_status launch_kernel_cluster(const LaunchCfg& cfg, void** args, cudaStream_t s, dim3 cluster);
bool pdl_enabled();

inline unsigned ceil_div(int64_t a, int64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace opara
