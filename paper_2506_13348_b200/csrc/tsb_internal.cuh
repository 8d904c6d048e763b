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

constexpr int kM64Stride = 10;

// What the rasterizer's decide loop reads of one staged splat: 48 bytes,
// three broadcast 128-bit loads (a 48-byte lane stride also makes the
// staging stores conflict-free).
struct __align__(16) DecRec {
  float lin[10];      // L0..L9: D, Nu, Nv forms and det
  float r2hi;         // L11
  uint32_t pixmask;   // pixels of the current 8x4 block inside the test box
};

// Pixels of the 8x4 block at (bx0, by0) (clipped to [bx0,bx1) x [by0,by1))
// inside a packed test box: bit (row * 8 + col).
__device__ __forceinline__ uint32_t tsb_block_pixmask(uint32_t gbx, uint32_t gby, int bx0,
                                                      int by0, int bx1, int by1) {
  const int cx0 = min(max((int)(gbx & 0xFFFF) - bx0, 0), 8);
  const int cx1 = min(max((int)(gbx >> 16) - bx0, 0), bx1 - bx0);
  const int cy0 = min(max((int)(gby & 0xFFFF) - by0, 0), 4);
  const int cy1 = min(max((int)(gby >> 16) - by0, 0), by1 - by0);
  if (cx1 <= cx0 || cy1 <= cy0) return 0u;
  const uint32_t row = ((1u << cx1) - 1u) & ~((1u << cx0) - 1u);
  const uint32_t rows = (uint32_t)(((1ull << (8 * cy1)) - 1ull) & ~((1ull << (8 * cy0)) - 1ull));
  return (row * 0x01010101u) & rows;
}

#ifndef TSB_DECIDE_ILP
#define TSB_DECIDE_ILP 2
#endif

// Live bits of one pixel (this lane) over the candidate mask `m` of a
// staged step: the division-free pre-decision, two candidates per
// iteration (independent chains), then the exact fp32 path and the fp64
// guard band for the rare undecided pairs. `lin` is the step's [11][32]
// structure-of-arrays copy of L0..L10, `sid` its splat ids. The result is
// exactly tsb_eval_lin + tsb_live_f64 of every candidate (tsb_math.h).
__device__ __forceinline__ uint32_t tsb_decide_step(const DecRec* dec, const float (*lin)[32],
                                                    const int32_t* sid, uint32_t m, int lane,
                                                    float x, float y, float near_f,
                                                    const tsb_cam_params& cam, const double* m64,
                                                    int px, int py) {
  uint32_t live = 0, undecided = 0;
  while (m) {
    int kk[TSB_DECIDE_ILP];
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      kk[j] = m ? __ffs(m) - 1 : kk[0];
      m &= m - 1;
    }
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      const DecRec& g = dec[kk[j]];
      const bool in = (g.pixmask >> lane) & 1u;
      const int r = tsb_predecide_lin_nb(g.lin, g.r2hi, x, y, near_f);
      live |= (in && r == 1 ? 1u : 0u) << kk[j];
      undecided |= (in && r == 2 ? 1u : 0u) << kk[j];
    }
  }
  for (uint32_t u = undecided; u; u &= u - 1) {
    const int k = __ffs(u) - 1;
    float L[12];
#pragma unroll
    for (int c = 0; c < 11; ++c) L[c] = lin[c][k];
    L[11] = dec[k].r2hi;
    float uu, vv, z, a;
    int r = tsb_eval_lin(L, x, y, near_f, &uu, &vv, &z, &a);
    if (r == 2) {
      const double* mm = m64 + (size_t)kM64Stride * sid[k];
      r = tsb_live_f64(mm, mm[9], tsb_pixel_x(&cam, px), tsb_pixel_y(&cam, py), cam.near_z);
    }
    if (r) live |= 1u << k;
  }
  return live;
}

// Stage splat `id` of a step into lane slot `lane`: the decide record (AoS)
// and the structure-of-arrays intersection forms. Returns the pixel mask.
__device__ __forceinline__ uint32_t tsb_stage_geom(const GeomRec* __restrict__ geom, int id,
                                                   int lane, int bx0, int by0, int bx1, int by1,
                                                   DecRec* dec, float (*lin)[32]) {
  const float4* gq = reinterpret_cast<const float4*>(geom + id);
  const float4 gv[4] = {__ldg(gq), __ldg(gq + 1), __ldg(gq + 2), __ldg(gq + 3)};
  const uint32_t pm = tsb_block_pixmask(__float_as_uint(gv[3].x), __float_as_uint(gv[3].y), bx0,
                                        by0, bx1, by1);
  float4* d = reinterpret_cast<float4*>(dec + lane);
  d[0] = gv[0];
  d[1] = gv[1];
  d[2] = make_float4(gv[2].x, gv[2].y, gv[2].w, __uint_as_float(pm));
  const float gl[11] = {gv[0].x, gv[0].y, gv[0].z, gv[0].w, gv[1].x, gv[1].y,
                        gv[1].z, gv[1].w, gv[2].x, gv[2].y, gv[2].z};
#pragma unroll
  for (int c = 0; c < 11; ++c) lin[c][lane] = gl[c];
  return pm;
}

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
