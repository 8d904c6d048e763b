// tsb_internal.cuh — records, workspace layout and helpers shared by the
// libtsb.so translation units (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/tsb.h"
#include "tsb_math.h"

namespace tsb {

// Per-splat geometry record staged in shared memory by the rasterizer:
// the linear intersection forms (tsb_make_lin: D, Nu, Nv coefficients,
// det(M), opacity, reject bound), the pixel test box = reference rect
// intersected with the alpha-cut ellipse box (tsb_test_box), packed as
// 16-bit pairs (x0 | x1 << 16, y0 | y1 << 16), and the splat id. 64 B.
struct __align__(16) GeomRec {
  float lin[TSB_LIN_WORDS];
  uint32_t bx, by;
  int32_t id;
  float r2lo;  // tsb_lin_r2lo(lin): "surely live" bound of the pre-decision
};
static_assert(sizeof(GeomRec) == 64, "GeomRec is 64 B");

// Per-splat material record, read from global (L1/L2) only when a fragment
// composites: frame columns, clamped SH radiance, chart origin. 64 B.
struct __align__(16) MatRec {
  float frame[9];   // t_u, t_v, t_u x t_v
  float l_ind[3];
  float tex_x, tex_y;  // chart origin in texels (cx*T, cy*T)
  int32_t page;
  int32_t lin_off;     // page*page_h*page_w + cy*T*page_w + cx*T (texels)
};
static_assert(sizeof(MatRec) == 64, "MatRec is 64 B");

// fp64 M + opacity for the alpha guard-band recheck and the backward pass.
constexpr int kM64Stride = 10;

struct AtlasTex {
  cudaArray_t arr_a = nullptr, arr_b = nullptr;
  cudaTextureObject_t tex_a = 0, tex_b = 0;
  int32_t page_w = 0, page_h = 0, pages = 0, format = 0;
};

// Workspace carve-up; every offset is 256-B aligned.
struct WsLayout {
  size_t geom, rects, mat, m64, dkeys_in, dkeys_out, dk32_in, dk32_out, ids_in, ids_out, tile_count,
      counts_sorted, offsets, rank, ekeys_in, ekeys_out, evals_in, evals_out,
      ranges, tcost_in, tcost_out, torder_in, torder_out, counters, cub_tmp;
  size_t cub_bytes;
  size_t total;
  int32_t tiles_x, tiles_y, num_tiles, tile_bits;
};

bool ws_layout(int32_t P, int32_t W, int32_t H, int32_t tile, int64_t cap, WsLayout* L);

void set_error(const std::string& msg);
int cuda_fail(const char* what, cudaError_t err);

inline tsb_cam_params to_cam(const tsb_camera* c) {
  static_assert(sizeof(tsb_cam_params) == sizeof(tsb_camera), "camera layouts match");
  tsb_cam_params p;
  std::memcpy(&p, c, sizeof(p));
  return p;
}

template <typename T>
inline T* ws_ptr(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}
template <typename T>
inline const T* ws_ptr(const void* ws, size_t off) {
  return reinterpret_cast<const T*>(static_cast<const char*>(ws) + off);
}

}  // namespace tsb

#define TSB_CHECK_LAUNCH(what)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::tsb::cuda_fail(what, _e);    \
  } while (0)

#define TSB_CUDA(call)                                           \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::tsb::cuda_fail(#call, _e);   \
  } while (0)
