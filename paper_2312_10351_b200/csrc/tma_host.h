// Host side of the TMA activation loads: an im2col-mode tensor map over an
// NHWC channel view, built at launch (capture) time and passed to the conv
// kernels as a __grid_constant__ parameter.
//
// Semantics (measured, scripts/micro/tma_im2col.cu): for a 4-D map {C, W, H, N}
// with pixel-box corners lower = {-pw, -ph}, upper = {pw - (S-1), ph - (R-1)}
// (im2col_corners: exactly OW x OH window origins) and traversal strides {1, sw, sh, 1}, one load at coordinates
// {c, ow*sw - pw, oh*sh - ph, n} with offsets {s, r} returns, for
// pixelsPerColumn consecutive output pixels (row-major over (n, oh, ow),
// wrapping rows and images), the channelsPerPixel channels [c, c + cpp) of
// input pixel (oh*sh - ph + r, ow*sw - pw + s); every out-of-range pixel or
// channel (padding, the tile tail past the last image) reads as zero.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace opara {

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The driver's encoder through the runtime's entry-point query (no -lcuda).
inline EncodeIm2colFn encode_im2col_fn() {
  static const EncodeIm2colFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeIm2col", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeIm2colFn>(nullptr);
    }
    return reinterpret_cast<EncodeIm2colFn>(p);
  }();
  return fn;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static const EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D tiled map over a bf16 [rows][cstride] row-major buffer: boxes of
// box_cols x box_rows elements with the 64-byte swizzle (box_cols * 2 <= 64).
inline bool make_tiled_bf16_map(CUtensorMap* map, const void* base, int64_t cstride, int64_t rows, int box_cols,
                                int box_rows) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cstride), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cstride) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// OPARA_TMA=0 keeps every conv on the cp.async gathers (A/B switch; read at
// every launch-record time, i.e. per capture, so a test can compare both paths).
inline bool tma_enabled() {
  const char* e = std::getenv("OPARA_TMA");
  return !(e && e[0] == '0');
}

// Pixel-box corners of the im2col traversal: lower = the first window origin
// (-pad), upper (an offset from the far edge) so that the box holds exactly
// O window origins at the traversal stride; a negative pad (the frontend's
// stride-2 subsample at offset 1) moves the box past the edge, where loads
// read zeros like the zero-extended map they stand for.
inline void im2col_corners(int dim, int out, int stride, int pad, int* lower, int* upper) {
  *lower = -pad;
  *upper = -pad + (out - 1) * stride - (dim - 1);
}

// Shape conditions for an im2col map over a channel view (elem = bytes per
// element, cpp = channels per load): 16-byte aligned view start and pixel
// stride, whole loads per tap (Cin % cpp == 0), corner offsets and traversal
// strides inside the hardware's ranges.
inline bool im2col_eligible(const void* base, int elem, int Cin, int64_t cstride, int coff, int H, int W, int OH, int OW,
                            int sh, int sw, int ph, int pw, int cpp) {
  const uintptr_t start = reinterpret_cast<uintptr_t>(base) + static_cast<uintptr_t>(coff) * elem;
  auto in8 = [](int v) { return v >= -128 && v <= 127; };
  int lw, uw, lh, uh;
  im2col_corners(W, OW, sw, pw, &lw, &uw);
  im2col_corners(H, OH, sh, ph, &lh, &uh);
  return tma_enabled() && Cin % cpp == 0 && start % 16 == 0 && (cstride * elem) % 16 == 0 && sh >= 1 && sh <= 8 &&
         sw >= 1 && sw <= 8 && in8(lw) && in8(uw) && in8(lh) && in8(uh);
}

// Encode the map; false if the driver refuses (callers then fail loudly).
inline bool make_im2col_map(CUtensorMap* map, CUtensorMapDataType dt, int elem, const void* base, int N, int H, int W,
                            int Cin, int64_t cstride, int coff, int OH, int OW, int sh, int sw, int ph, int pw, int cpp,
                            int ppc) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn) return false;
  void* start = const_cast<char*>(static_cast<const char*>(base)) + static_cast<int64_t>(coff) * elem;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(N)};
  const cuuint64_t px = static_cast<cuuint64_t>(cstride) * elem;
  const cuuint64_t strides[3] = {px, px * W, px * W * H};
  int lower[2], upper[2];
  im2col_corners(W, OW, sw, pw, &lower[0], &upper[0]);
  im2col_corners(H, OH, sh, ph, &lower[1], &upper[1]);
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(sw), static_cast<cuuint32_t>(sh), 1};
  return fn(map, dt, 4, start, dims, strides, lower, upper, static_cast<cuuint32_t>(cpp), static_cast<cuuint32_t>(ppc),
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace opara
