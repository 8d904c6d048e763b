// tsb_internal.cuh — records, workspace layout and helpers shared by the
// libtsb.so translation units (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <mutex>
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
// guard band for the rare undecided pairs (live0 / und0: pairs already
// pre-decided elsewhere, e.g. by tsb_decide_candidate). `load_lin(k, L)` fills L[0..11]
// (tsb_make_lin's words) of staged entry k, `sid` holds the splat ids. The
// result is exactly tsb_eval_lin + tsb_live_f64 of every candidate (tsb_math.h).
// What the decide loop reads of staged entry k: the linear forms L0..L9
// (+ opacity, r2hi), the α-cut reject bound r2hi and the block pixel mask.
struct DecRef {
  const float* lin;
  float r2hi;
  uint32_t pixmask;
};

template <class DecAt, class LoadLin>
__device__ __forceinline__ uint32_t tsb_decide_step(DecAt dec_at, LoadLin load_lin,
                                                    const int32_t* sid, uint32_t m, uint32_t zs,
                                                    int lane, float x, float y, float near_f,
                                                    const tsb_cam_params& cam, const double* m64,
                                                    int px, int py, uint32_t live0 = 0,
                                                    uint32_t und0 = 0) {
  uint32_t live = 0, undecided = 0;
  // z-safe candidates (kBlockZSafe): tsb_predecide_lin_nb reduces to the two
  // q tests (|D| > eps and the depth test hold on the whole block)
  live = live0;
  undecided = und0;
  for (uint32_t mz = m & zs; mz;) {
    int kk[TSB_DECIDE_ILP];
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      kk[j] = mz ? __ffs(mz) - 1 : kk[0];
      mz &= mz - 1;
    }
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      const DecRef g = dec_at(kk[j]);
      const bool in = (g.pixmask >> lane) & 1u;
      const float D = fmaf(g.lin[0], x, fmaf(g.lin[1], y, g.lin[2]));
      const float Nu = fmaf(g.lin[3], x, fmaf(g.lin[4], y, g.lin[5]));
      const float Nv = fmaf(g.lin[6], x, fmaf(g.lin[7], y, g.lin[8]));
      const float q = fmaf(Nu, Nu, Nv * Nv);
      const float D2 = D * D;
      const bool sure = q <= tsb_lin_r2lo(g.r2hi) * D2;
      const bool maybe = q <= g.r2hi * D2;
      live |= (in && sure ? 1u : 0u) << kk[j];
      undecided |= (in && maybe && !sure ? 1u : 0u) << kk[j];
    }
  }
  m &= ~zs;
  while (m) {
    int kk[TSB_DECIDE_ILP];
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      kk[j] = m ? __ffs(m) - 1 : kk[0];
      m &= m - 1;
    }
#pragma unroll
    for (int j = 0; j < TSB_DECIDE_ILP; ++j) {
      const DecRef g = dec_at(kk[j]);
      const bool in = (g.pixmask >> lane) & 1u;
      const int r = tsb_predecide_lin_nb(g.lin, g.r2hi, x, y, near_f);
      live |= (in && r == 1 ? 1u : 0u) << kk[j];
      undecided |= (in && r == 2 ? 1u : 0u) << kk[j];
    }
  }
  for (uint32_t u = undecided; u; u &= u - 1) {
    const int k = __ffs(u) - 1;
    float L[12];
    load_lin(k, L);
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

// 32x32 bit-matrix transpose across a warp: lane r holds row r (bit c =
// element (r, c)); returns column `lane` (bit r = element (r, lane)). Five
// butterfly stages of one shuffle each.
__device__ __forceinline__ uint32_t tsb_warp_transpose32(uint32_t x, int lane) {
  constexpr uint32_t kMask[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int s = 16 >> i;
    const uint32_t m = kMask[i];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

// Candidate-per-lane form of the z-safe part of tsb_decide_step: lane k
// tests ITS staged splat (forms L0..L8 in g0..g2, r2hi = g2.w) at all 32
// pixels of the 8x4 block with exactly the arithmetic of the per-pixel loop
// (D = fmaf(L0, x, fmaf(L1, y, L2)), ...), so every q/D^2 test gives the same
// bits; xs[c] are the block's fp32 column coordinates, row r's y comes from
// lane 8r's `ylane` (every lane must call this). Returns the
// pixels where the pair is surely live (bit row*8+col) and sets `und` to the
// pixels in the annulus between the bounds (exact path). A warp instruction
// here serves 32 candidates at once instead of one (no shared-memory loads).
__device__ __forceinline__ uint32_t tsb_decide_candidate(const float4& g0, const float4& g1,
                                                         const float4& g2, const float* xs,
                                                         float ylane, uint32_t& und) {
  const float r2hi = g2.w;
  const float r2lo = tsb_lin_r2lo(r2hi);
  uint32_t live = 0;
  und = 0;
#pragma unroll 1
  for (int r = 0; r < 4; ++r) {
    const float y = __shfl_sync(0xffffffffu, ylane, 8 * r);  // all lanes call this
    const float Dr = fmaf(g0.y, y, g0.z);
    const float Ur = fmaf(g1.x, y, g1.y);
    const float Vr = fmaf(g1.w, y, g2.x);
    uint32_t lrow = 0, urow = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float x = xs[c];
      const float D = fmaf(g0.x, x, Dr);
      const float Nu = fmaf(g0.w, x, Ur);
      const float Nv = fmaf(g1.z, x, Vr);
      const float q = fmaf(Nu, Nu, Nv * Nv);
      const float D2 = D * D;
      const bool sure = q <= r2lo * D2;
      const bool maybe = q <= r2hi * D2;
      const uint32_t bit = 1u << c;
      if (sure) lrow |= bit;
      if (maybe && !sure) urow |= bit;
    }
    live |= lrow << (8 * r);
    und |= urow << (8 * r);
  }
  return live;
}

// Camera-plane extent of a warp's 8x4 pixel block (clipped to the image):
// the fp32 pixel coordinates x(bx0), x(bx1-1), y(by0), y(by1-1) — exactly the
// values the block's lanes evaluate at its corners — and the block's pixel mask.
struct BlockBox {
  float x0, y0, dx, dy;  // corner (x0, y0) and the extents to the opposite corner
  float X, Y;            // max |x|, |y| over the block
  uint32_t valid;
};

__device__ __forceinline__ BlockBox tsb_block_box(const tsb_cam_params& cam, int bx0, int by0,
                                                  int bx1, int by1) {
  BlockBox b;
  const float xa = (float)tsb_pixel_x(&cam, bx0), xb = (float)tsb_pixel_x(&cam, bx1 - 1);
  const float ya = (float)tsb_pixel_y(&cam, by0), yb = (float)tsb_pixel_y(&cam, by1 - 1);
  b.x0 = xa; b.dx = xb - xa;
  b.y0 = ya; b.dy = yb - ya;
  b.X = fmaxf(fabsf(xa), fabsf(xb));
  b.Y = fmaxf(fabsf(ya), fabsf(yb));
  b.valid = tsb_block_pixmask((uint32_t)bx0 | ((uint32_t)bx1 << 16),
                              (uint32_t)by0 | ((uint32_t)by1 << 16), bx0, by0, bx1, by1);
  return b;
}

// Block-level facts about a splat, each true only if it holds at EVERY fp32
// pixel point (x, y) of the block rectangle (performance shortcuts that never
// change a decision):
//   kBlockZSafe: |D~| > eps and the depth test of tsb_predecide_lin_nb passes
//                (z surely > near), so the pixel's answer depends on q alone;
//   kBlockLive:  additionally q <= r2lo D^2, i.e. the answer is 1 (live) — the
//                warp sets the splat's live bit for all its pixels untested.
// With S_F = |a|X+|b|Y+|c| for a form F = a x + b y + c (X, Y = max |x|, |y|):
//  * e_F = 2^-21 S_F bounds the error of F's fp32 value at a pixel (two
//    roundings: 2^-23 S_F) and at the corners, which are stepped from
//    (x0, y0) by one or two more fmaf's with the rounded extents dx, dy.
//  * D is affine: with every corner |D~| > eD of one sign, the exact D keeps
//    that sign on the block and |D| >= dlo = min |D~_c| - eD there.
//  * z: zs > zt holds with a 3e-5 relative margin at the largest pixel |D~|.
//  * (x,y) -> (u,v) = (Nu/D, Nv/D) is projective without a pole on the block,
//    so the block maps onto the convex quad of its corner images: the exact
//    |(u,v)| on the block is at most its largest corner value rho.
//  * corner test q~_c <= 0.8999 r2lo (|D~_c| - eD)^2 and eN <= 0.01 sqrt(r2lo) dlo
//    (eN = e_Nu + e_Nv) give rho <= 0.9587 sqrt(r2lo); with eD <= 0.03 dlo the
//    per-pixel fp32 N~ <= rho|D| + eN stays below 0.99999 sqrt(r2lo)(|D| - eD),
//    so the pixel's own q <= r2lo D^2 (three roundings) holds; q <= r2hi D^2 too.
// The GPU-vs-oracle bit-exact tests (tests/test_gpu_forward.py) check both.
constexpr uint32_t kBlockZSafe = 1u, kBlockLive = 2u;

__device__ __forceinline__ uint32_t tsb_block_flags(const float4& g0, const float4& g1,
                                                    const float4& g2, float r2lo,
                                                    const BlockBox& b, float near_z) {
  // L0..L8 = D, Nu, Nv coefficients, L9 = det (tsb_make_lin)
  const float k21 = 4.76837158203125e-7f;  // 2^-21
  const float eD = k21 * fmaf(fabsf(g0.x), b.X, fmaf(fabsf(g0.y), b.Y, fabsf(g0.z)));
  const float eN = k21 * (fmaf(fabsf(g0.w), b.X, fmaf(fabsf(g1.x), b.Y, fabsf(g1.y))) +
                          fmaf(fabsf(g1.z), b.X, fmaf(fabsf(g1.w), b.Y, fabsf(g2.x))));
  float D[4], U[4], V[4];
  D[0] = fmaf(g0.x, b.x0, fmaf(g0.y, b.y0, g0.z));
  U[0] = fmaf(g0.w, b.x0, fmaf(g1.x, b.y0, g1.y));
  V[0] = fmaf(g1.z, b.x0, fmaf(g1.w, b.y0, g2.x));
  D[1] = fmaf(g0.x, b.dx, D[0]); U[1] = fmaf(g0.w, b.dx, U[0]); V[1] = fmaf(g1.z, b.dx, V[0]);
  D[2] = fmaf(g0.y, b.dy, D[0]); U[2] = fmaf(g1.x, b.dy, U[0]); V[2] = fmaf(g1.w, b.dy, V[0]);
  D[3] = fmaf(g0.y, b.dy, D[1]); U[3] = fmaf(g1.x, b.dy, U[1]); V[3] = fmaf(g1.w, b.dy, V[1]);
  const float c = 0.8999f * r2lo;
  bool pos = true, neg = true, in = true;
  float dmin = 3.0e38f, dmax = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    pos = pos && D[i] > eD;
    neg = neg && D[i] < -eD;
    const float aD = fabsf(D[i]);
    dmin = fminf(dmin, aD);
    dmax = fmaxf(dmax, aD);
    const float t = aD - eD;
    in = in && fmaf(U[i], U[i], V[i] * V[i]) <= (t * t) * c;
  }
  const float dlo = dmin - eD;
  const float dhi = dmax + 2.f * eD;
  const float zl = pos ? g2.y : -g2.y;
  const bool zsafe = (pos || neg) && dlo > 2e-9f && eD <= 0.03f * dlo &&
                     zl - near_z * dhi >= 3e-5f * (fabsf(g2.y) + near_z * dhi);
  const bool live = zsafe && in && eN * eN <= 0.99e-4f * r2lo * (dlo * dlo);
  return (zsafe ? kBlockZSafe : 0u) | (live ? kBlockLive : 0u);
}

// Stage splat `id` of a step into lane slot `lane`: the decide record (AoS);
// gv receives the GeomRec words (lin[0..11] in gv[0..2]). Returns the pixel
// mask; `flags` = tsb_block_flags (kBlockLive only if the test box also covers
// the whole block), so the decide loop can skip or simplify the splat.
__device__ __forceinline__ uint32_t tsb_stage_geom(const GeomRec* __restrict__ geom, int id,
                                                   int lane, int bx0, int by0, int bx1, int by1,
                                                   DecRec* dec, const BlockBox& bb, float near_z,
                                                   uint32_t& flags, float4* gv) {
  const float4* gq = reinterpret_cast<const float4*>(geom + id);
  gv[0] = __ldg(gq); gv[1] = __ldg(gq + 1); gv[2] = __ldg(gq + 2); gv[3] = __ldg(gq + 3);
  const uint32_t pm = tsb_block_pixmask(__float_as_uint(gv[3].x), __float_as_uint(gv[3].y), bx0,
                                        by0, bx1, by1);
  flags = pm ? tsb_block_flags(gv[0], gv[1], gv[2], gv[3].w, bb, near_z) : 0u;
  if (pm != bb.valid) flags &= ~kBlockLive;
  if (dec) {  // (the forward reads the forms from its own record instead)
    float4* d = reinterpret_cast<float4*>(dec + lane);
    d[0] = gv[0];
    d[1] = gv[1];
    d[2] = make_float4(gv[2].x, gv[2].y, gv[2].w, __uint_as_float(pm));
  }
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
      rank, ekeys_in, ekeys_out, evals_in, evals_out, ranges, torder_out, max_needed, counters,
      bin, status, long_runs;
  size_t status_words;                       // one-sweep look-back words (zeroed per frame)
  int32_t nb_depth, nb_dup, nb_tiley;        // one-sweep CTAs per pass
  size_t total;
  int32_t tiles_x, tiles_y, num_tiles, tile_bits;
};

bool ws_layout(int32_t P, int32_t W, int32_t H, int32_t tile, int64_t cap, WsLayout* L);

// One-time per-device setup (function attributes, __constant__ uploads,
// persistent grid sizes): one value per device ordinal, computed on first
// use on that device, thread-safe. `init` returns > 0 on success, or a
// negative cudaError_t.
constexpr int kMaxDevices = 64;
struct PerDevice {
  std::mutex m;
  int val[kMaxDevices] = {};
  template <class F>
  cudaError_t get(F&& init, int* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(m);
    if (val[dev] <= 0) {
      const int v = init(dev);
      if (v <= 0) return v < 0 ? (cudaError_t)(-v) : cudaErrorUnknown;
      val[dev] = v;
    }
    *out = val[dev];
    return cudaSuccess;
  }
};

// Per-camera constants of the shading kernels' view directions (K6, K7):
// the unnormalised direction of pixel (px, py) is px * vx + py * vy + v0
// (splats.py:128-140 folded with the pixel centres (px + 0.5 - cx) / fx;
// fp32, tolerance-checked), and the pixel row is an exact multiply-shift.
struct ViewCoeffs {
  float vx[3], vy[3], v0[3];
  uint64_t row_magic;  // py = (pix * row_magic) >> 40, exact for pix < 2^24, W < 2^16
};

inline ViewCoeffs view_coeffs(const tsb_camera* camera) {
  ViewCoeffs v;
  const double* Wv = camera->world_to_view;
  for (int j = 0; j < 3; ++j) {
    v.vx[j] = (float)(Wv[j] / camera->fx);
    v.vy[j] = (float)(Wv[4 + j] / camera->fy);
    v.v0[j] = (float)(Wv[8 + j] + Wv[j] * (0.5 - camera->cx) / camera->fx +
                      Wv[4 + j] * (0.5 - camera->cy) / camera->fy);
  }
  v.row_magic = (((uint64_t)1 << 40) + (uint64_t)camera->width - 1) / (uint64_t)camera->width;
  return v;
}

// -omega_o (the unit direction toward the camera) of pixel index pix.
__device__ __forceinline__ void view_dir_pix(const ViewCoeffs& v, int pix, int W, float* wo) {
  const int py = (int)(((uint64_t)pix * v.row_magic) >> 40), px = pix - py * W;
  const float fx = (float)px, fy = (float)py;
  float d[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) d[j] = fmaf(fy, v.vy[j], fmaf(fx, v.vx[j], v.v0[j]));
  const float r = -rsqrtf((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) wo[j] = d[j] * r;
}

// Programmatic dependent launch (sm_90+): a frame's kernels are launched
// with programmatic stream serialisation, so each one's CTAs are scheduled
// while its predecessor drains and wait in pdl_wait() (griddepcontrol.wait:
// the predecessor has completed and its writes are visible) instead of
// paying a full launch gap per kernel. Every such kernel calls pdl_wait()
// before touching its predecessor's output (a no-op without the attribute).
#ifndef TSB_PDL
#define TSB_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if TSB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
#if TSB_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
#else
  kernel<<<grid, block, smem, st>>>(args...);
  return cudaGetLastError();
#endif
}

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
