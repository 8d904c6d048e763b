// tsb_forward.cu — forward render path for sm_100a.
//
//   K1 k_preprocess     per splat, fp64: rect/cull, centre depth key, M, frame,
//                       SH radiance -> GeomRec / MatRec / fp64 M
//   S1 depth sort       stable LSD radix sort of fp64 depth bits (ids in id
//                       order => ties broken by id, == np.lexsort((ids, z)))
//   K2 k_rank_counts    per rank: tile count, rank of id
//   S2 exclusive scan   entry offsets in draw order
//   K3 k_duplicate      (tile, id) entries in draw order
//   S3 tile sort        stable radix sort on tile bits only => per-tile lists
//                       keep draw order (== keys (tile << 32) | rank)
//   K4 k_ranges         [start, end) per tile
//   K5 k_raster_fwd     CTA per tile: staged geometry in smem, fp32
//                       intersection with fp64 guard band, TEX/verify/flat
//                       texel fetch, 13-channel front-to-back composite
//   K6 k_shade          per pixel split-sum PBR (shading.py:126-183)
//
// Reference: /root/reference/pkg/src/texsplat/rasterize.py:127-438,
// shading.py:51-183 (see tsb_math.h for line-level citations).

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "tsb_internal.cuh"

namespace tsb {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(const char* what, cudaError_t err) {
  g_err = std::string(what) + ": " + cudaGetErrorString(err);
  return TSB_ERR_CUDA;
}

static inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

bool ws_layout(int32_t P, int32_t W, int32_t H, int32_t tile, int64_t cap, WsLayout* L) {
  if (P < 0 || W <= 0 || H <= 0 || cap < 0) return false;
  if (tile != 8 && tile != 16 && tile != 32) return false;
  L->tiles_x = (W + tile - 1) / tile;
  L->tiles_y = (H + tile - 1) / tile;
  L->num_tiles = L->tiles_x * L->tiles_y;
  int bits = 1;
  while ((1ll << bits) <= (int64_t)L->num_tiles) ++bits;
  L->tile_bits = bits;
  const size_t Pn = (size_t)std::max(P, 1);
  const size_t C = (size_t)std::max<int64_t>(cap, 1);

  // CUB temp storage (size queries only; nothing is launched).
  size_t b_depth = 0, b_scan = 0, b_tile = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b_depth, (const uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)Pn, 0, 64);
  cub::DeviceScan::ExclusiveSum(nullptr, b_scan, (const int32_t*)nullptr,
                                (int32_t*)nullptr, (int)Pn);
  cub::DeviceRadixSort::SortPairs(nullptr, b_tile, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)C, 0, bits);
  L->cub_bytes = std::max(b_depth, std::max(b_scan, b_tile));

  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  L->geom = take(Pn * sizeof(GeomRec));
  L->mat = take(Pn * sizeof(MatRec));
  L->m64 = take(Pn * kM64Stride * sizeof(double));
  L->dkeys_in = take(Pn * 8);
  L->dkeys_out = take(Pn * 8);
  L->ids_in = take(Pn * 4);
  L->ids_out = take(Pn * 4);
  L->tile_count = take(Pn * 4);
  L->counts_sorted = take(Pn * 4);
  L->offsets = take(Pn * 4);
  L->rank = take(Pn * 4);
  L->ekeys_in = take(C * 4);
  L->ekeys_out = take(C * 4);
  L->evals_in = take(C * 4);
  L->evals_out = take(C * 4);
  L->ranges = take((size_t)L->num_tiles * 8);
  L->counters = take(64);
  L->cub_tmp = take(L->cub_bytes);
  L->total = o;
  return true;
}

// ---------------------------------------------------------------------------
// K1 preprocess
// ---------------------------------------------------------------------------
struct PrepParams {
  tsb_cam_params cam;
  int32_t P, sh_degree, tile, tiles_x;
  const double* pos;
  const double* tu;
  const double* tv;
  const double* sc;
  const double* op;
  const double* sh;
  const int32_t* entries;   // may be null (flat mode)
  int32_t T, page_w, page_h;
  GeomRec* geom;
  MatRec* mat;
  double* m64;
  uint64_t* dkeys;
  int32_t* ids;
  int32_t* tile_count;
};

__global__ void __launch_bounds__(256) k_preprocess(PrepParams p) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= p.P) return;
  const int K = (p.sh_degree + 1) * (p.sh_degree + 1);
  double pos[3], tu[3], tv[3], s[2], sh[48];
  for (int j = 0; j < 3; ++j) {
    pos[j] = p.pos[3 * id + j];
    tu[j] = p.tu[3 * id + j];
    tv[j] = p.tv[3 * id + j];
  }
  s[0] = p.sc[2 * id];
  s[1] = p.sc[2 * id + 1];
  for (int k = 0; k < 3 * K; ++k) sh[k] = p.sh[(size_t)3 * K * id + k];
  tsb_prep r;
  tsb_preprocess_splat(&p.cam, pos, tu, tv, s, sh, p.sh_degree, &r);
  const double op = p.op[id];

  GeomRec g;
  for (int k = 0; k < 9; ++k) g.m[k] = (float)r.m[k];
  g.opacity = (float)op;
  g.x0 = r.x0; g.x1 = r.x1; g.y0 = r.y0; g.y1 = r.y1;
  g.id = id;
  g.pad = 0;
  p.geom[id] = g;

  MatRec m;
  for (int k = 0; k < 9; ++k) m.frame[k] = (float)r.frame[k];
  for (int k = 0; k < 3; ++k) m.l_ind[k] = (float)r.l_ind[k];
  if (p.entries) {
    const int cx = p.entries[3 * id], cy = p.entries[3 * id + 1], pg = p.entries[3 * id + 2];
    m.tex_x = (float)(cx * p.T);
    m.tex_y = (float)(cy * p.T);
    m.page = pg;
    m.lin_off = (int32_t)((int64_t)pg * p.page_h * p.page_w + (int64_t)cy * p.T * p.page_w +
                          (int64_t)cx * p.T);
  } else {
    m.tex_x = m.tex_y = 0.f; m.page = 0; m.lin_off = 0;
  }
  p.mat[id] = m;

  double* m64 = p.m64 + (size_t)kM64Stride * id;
  for (int k = 0; k < 9; ++k) m64[k] = r.m[k];
  m64[9] = op;

  p.dkeys[id] = r.keep ? tsb_f64_bits(r.view_z) : ~0ull;
  p.ids[id] = id;
  p.tile_count[id] = r.keep ? tsb_rect_tile_count(r.x0, r.x1, r.y0, r.y1, p.tile) : 0;
}

// K2: per draw-order rank: tile count and rank of each id.
__global__ void k_rank_counts(int32_t P, const int32_t* __restrict__ sorted_ids,
                              const int32_t* __restrict__ tile_count,
                              int32_t* __restrict__ counts_sorted, int32_t* __restrict__ rank) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P) return;
  const int id = sorted_ids[r];
  counts_sorted[r] = tile_count[id];
  rank[id] = r;
}

// K3: duplicate each splat into every tile its rect touches, in draw order.
__global__ void k_duplicate(int32_t P, int32_t tile, int32_t tiles_x, int64_t cap,
                            const int32_t* __restrict__ sorted_ids,
                            const int32_t* __restrict__ counts_sorted,
                            const int32_t* __restrict__ offsets,
                            const GeomRec* __restrict__ geom, uint32_t* __restrict__ ekeys,
                            int32_t* __restrict__ evals, int64_t* __restrict__ counters) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P) return;
  const int cnt = counts_sorted[r];
  const int64_t off = offsets[r];
  if (r == P - 1) counters[0] = off + cnt;
  if (cnt == 0 || off + cnt > cap) return;
  const int id = sorted_ids[r];
  const GeomRec g = geom[id];
  int64_t o = off;
  for (int ty = g.y0 / tile; ty <= (g.y1 - 1) / tile; ++ty)
    for (int tx = g.x0 / tile; tx <= (g.x1 - 1) / tile; ++tx) {
      ekeys[o] = (uint32_t)(ty * tiles_x + tx);
      evals[o] = id;
      ++o;
    }
}

// K4: tile ranges from the tile-sorted entry keys.
__global__ void k_ranges(int64_t cap, const uint32_t* __restrict__ keys,
                         const int64_t* __restrict__ counters, int32_t* __restrict__ ranges) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = counters[0];
  if (total > cap) total = 0;  // overflowed frame: leave every tile empty
  if (i >= total) return;
  const uint32_t t = keys[i];
  if (i == 0 || keys[i - 1] != t) ranges[2 * t] = (int32_t)i;
  if (i == total - 1 || keys[i + 1] != t) ranges[2 * t + 1] = (int32_t)(i + 1);
}

// ---------------------------------------------------------------------------
// K5 rasterize forward
// ---------------------------------------------------------------------------
struct RasterParams {
  tsb_cam_params cam;
  int32_t W, H, tiles_x;
  float near_f;
  const int32_t* ranges;
  const int32_t* evals;
  const GeomRec* geom;
  const MatRec* mat;
  const double* m64;
  // texture sources
  int32_t T, page_w;
  const float4* fam_a;
  const float4* fam_b;
  const float* flat;
  cudaTextureObject_t tex_a, tex_b;
  // outputs
  float* gbuf;
  int32_t* n_contrib;
  int32_t* last_entry;
  float* final_T;
  float* T_last;
};

template <int MODE>
__device__ __forceinline__ void fetch_attrs(const RasterParams& p, int id, float u, float v,
                                            float z, float* xa) {
  const float4* mr = reinterpret_cast<const float4*>(p.mat + id);
  const float4 q0 = __ldg(mr), q1 = __ldg(mr + 1), q2 = __ldg(mr + 2);
  const float frame[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
  if (MODE == TSB_MODE_FLAT) {
    const float* f = p.flat + 5 * id;
    xa[0] = __ldg(f); xa[1] = __ldg(f + 1); xa[2] = __ldg(f + 2);
    xa[3] = __ldg(f + 3); xa[4] = __ldg(f + 4);
    xa[5] = frame[6]; xa[6] = frame[7]; xa[7] = frame[8];
  } else {
    const float4 q3 = __ldg(mr + 3);
    tsb_texc tc;
    tsb_texel_coords(u, v, p.T, &tc);
    float4 A, B;
    if (MODE == TSB_MODE_HW) {
      const float sx = q3.x + tc.xs + 0.5f;
      const float sy = q3.y + tc.yt + 0.5f;
      const int layer = __float_as_int(q3.z);
      A = tex2DLayered<float4>(p.tex_a, sx, sy, layer);
      B = tex2DLayered<float4>(p.tex_b, sx, sy, layer);
    } else {
      const int base = __float_as_int(q3.w);
      const int r0 = base + tc.j0 * p.page_w, r1 = base + tc.j1 * p.page_w;
      const float4 a00 = __ldg(p.fam_a + r0 + tc.i0), a01 = __ldg(p.fam_a + r0 + tc.i1);
      const float4 a10 = __ldg(p.fam_a + r1 + tc.i0), a11 = __ldg(p.fam_a + r1 + tc.i1);
      const float4 b00 = __ldg(p.fam_b + r0 + tc.i0), b01 = __ldg(p.fam_b + r0 + tc.i1);
      const float4 b10 = __ldg(p.fam_b + r1 + tc.i0), b11 = __ldg(p.fam_b + r1 + tc.i1);
      A.x = tsb_lerp4(a00.x, a01.x, a10.x, a11.x, tc.fs, tc.ft);
      A.y = tsb_lerp4(a00.y, a01.y, a10.y, a11.y, tc.fs, tc.ft);
      A.z = tsb_lerp4(a00.z, a01.z, a10.z, a11.z, tc.fs, tc.ft);
      A.w = tsb_lerp4(a00.w, a01.w, a10.w, a11.w, tc.fs, tc.ft);
      B.x = tsb_lerp4(b00.x, b01.x, b10.x, b11.x, tc.fs, tc.ft);
      B.y = tsb_lerp4(b00.y, b01.y, b10.y, b11.y, tc.fs, tc.ft);
      B.z = tsb_lerp4(b00.z, b01.z, b10.z, b11.z, tc.fs, tc.ft);
      B.w = 0.f;
    }
    xa[0] = A.x; xa[1] = A.y; xa[2] = A.z;
    xa[3] = B.z;  // metallic
    xa[4] = A.w;  // roughness
    tsb_decode_normal(B.x, B.y, frame, xa + 5);
  }
  xa[8] = q2.y; xa[9] = q2.z; xa[10] = q2.w;
  xa[11] = z;
}

template <int TILE, int MODE>
__global__ void __launch_bounds__(TILE * TILE) k_raster_fwd(RasterParams p) {
  constexpr int BLOCK = TILE * TILE;
  constexpr int BATCH = BLOCK < 256 ? BLOCK : 256;
  __shared__ GeomRec s_geom[BATCH];

  const int tile = blockIdx.x;
  const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
  const int lx = threadIdx.x % TILE, ly = threadIdx.x / TILE;
  const int px = tx * TILE + lx, py = ty * TILE + ly;
  const bool inside = px < p.W && py < p.H;
  const double xd = tsb_pixel_x(&p.cam, px), yd = tsb_pixel_y(&p.cam, py);
  const float x = (float)xd, y = (float)yd;
  const int start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];

  float acc[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) acc[c] = 0.f;
  float T = 1.f, T_last = 1.f;
  int n = 0, last = -1;
  bool done = !inside;
  const float teps = (float)TSB_TRANSMIT_EPS;

  for (int base = start; base < end; base += BATCH) {
    if (__syncthreads_count(done) == BLOCK) break;
    const int i = base + (int)threadIdx.x;
    if (threadIdx.x < BATCH && i < end) s_geom[threadIdx.x] = p.geom[p.evals[i]];
    __syncthreads();
    const int cnt = min(BATCH, end - base);
    if (!done) {
      for (int j = 0; j < cnt; ++j) {
        const GeomRec& g = s_geom[j];
        if (px < g.x0 || px >= g.x1 || py < g.y0 || py >= g.y1) continue;
        float u, v, z, a;
        const int r = tsb_intersect_f32(g.m, g.opacity, x, y, p.near_f, &u, &v, &z, &a);
        if (r == 0) continue;
        if (r == 2) {
          const double* m64 = p.m64 + (size_t)kM64Stride * g.id;
          if (!tsb_live_f64(m64, m64[9], xd, yd, p.cam.near_z)) continue;
        }
        float xa[12];
        fetch_attrs<MODE>(p, g.id, u, v, z, xa);
        T_last = T;
        T = tsb_composite(acc, xa, a, T);
        ++n;
        last = base + j;
        if (!(T > teps)) { done = true; break; }
      }
    }
  }
  if (!inside) return;
  const int HW = p.W * p.H;
  const int pix = py * p.W + px;
#pragma unroll
  for (int c = 0; c < 13; ++c) p.gbuf[(size_t)c * HW + pix] = acc[c];
  p.n_contrib[pix] = n;
  p.last_entry[pix] = last;
  p.final_T[pix] = T;
  p.T_last[pix] = T_last;
}

// ---------------------------------------------------------------------------
// K6 shade
// ---------------------------------------------------------------------------
struct ShadeParams {
  tsb_cam_params cam;
  tsb_env_params env;
  float bg[3];
  const float* gbuf;
  float* color;
  float* diffuse;
  float* specular;
};

__global__ void __launch_bounds__(256) k_shade(ShadeParams p) {
  const int W = p.cam.width, H = p.cam.height;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= W * H) return;
  const int px = pix % W, py = pix / W;
  float g[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) g[c] = __ldg(p.gbuf + (size_t)c * W * H + pix);
  float wo[3];
  tsb_view_dir(&p.cam, tsb_pixel_x(&p.cam, px), tsb_pixel_y(&p.cam, py), wo);
  float col[3], dif[3], spe[3];
  tsb_shade_pixel(g, wo, &p.env, p.bg, col, dif, spe);
#pragma unroll
  for (int c = 0; c < 3; ++c) p.color[3 * pix + c] = col[c];
  if (p.diffuse)
    for (int c = 0; c < 3; ++c) p.diffuse[3 * pix + c] = dif[c];
  if (p.specular)
    for (int c = 0; c < 3; ++c) p.specular[3 * pix + c] = spe[c];
}

// ---------------------------------------------------------------------------
// Export + atlas textures + TEX probe
// ---------------------------------------------------------------------------
__global__ void k_export_keys(int64_t cap, const uint32_t* __restrict__ ekeys,
                              const int32_t* __restrict__ evals, const int32_t* __restrict__ rank,
                              const int64_t* __restrict__ counters, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  int64_t total = counters[0];
  if (total > cap) total = 0;
  keys[i] = i < total ? (((int64_t)ekeys[i] << 32) | (int64_t)(uint32_t)rank[evals[i]]) : -1;
}

__global__ void k_export_rects(int32_t P, const GeomRec* __restrict__ geom, int32_t* __restrict__ rects) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P) return;
  const GeomRec g = geom[id];
  rects[4 * id] = g.x0; rects[4 * id + 1] = g.x1; rects[4 * id + 2] = g.y0; rects[4 * id + 3] = g.y1;
}

__global__ void k_f32_to_f16x4(const float4* __restrict__ src, ushort4* __restrict__ dst, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    const float4 v = src[i];
    ushort4 h;
    h.x = __half_as_ushort(__float2half_rn(v.x));
    h.y = __half_as_ushort(__float2half_rn(v.y));
    h.z = __half_as_ushort(__float2half_rn(v.z));
    h.w = __half_as_ushort(__float2half_rn(v.w));
    dst[i] = h;
  }
}

__global__ void k_tex_probe(cudaTextureObject_t tex, int32_t window, int32_t iters, float* sink) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  float fx = 0.37f + (float)(t % window);
  float fy = 0.61f + (float)((t / window) % window);
  for (int k = 0; k < iters; ++k) {
    const float4 v = tex2DLayered<float4>(tex, fx, fy, 0);
    acc += v.x + v.y + v.z + v.w;
    fx += 1.13f; if (fx > (float)window) fx -= (float)window;
    fy += 0.71f; if (fy > (float)window) fy -= (float)window;
  }
  sink[t] = acc;
}

template <int TILE>
inline void launch_raster(int mode, int blocks, cudaStream_t st, const RasterParams& rp) {
  if (mode == TSB_MODE_HW)
    k_raster_fwd<TILE, TSB_MODE_HW><<<blocks, TILE * TILE, 0, st>>>(rp);
  else if (mode == TSB_MODE_VERIFY)
    k_raster_fwd<TILE, TSB_MODE_VERIFY><<<blocks, TILE * TILE, 0, st>>>(rp);
  else
    k_raster_fwd<TILE, TSB_MODE_FLAT><<<blocks, TILE * TILE, 0, st>>>(rp);
}

}  // namespace tsb

using namespace tsb;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* tsb_last_error(void) { return g_err.c_str(); }

const char* tsb_version(void) { return "tsb 0.1.0 sm_100a"; }

int tsb_frame_workspace_size(int32_t P, int32_t W, int32_t H, int32_t tile, int64_t cap,
                             uint64_t* bytes) {
  WsLayout L;
  if (!bytes || !ws_layout(P, W, H, tile, cap, &L)) {
    set_error("tsb_frame_workspace_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *bytes = L.total;
  return TSB_OK;
}

static int validate_frame(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                          int32_t mode, int32_t tile, void* ws, uint64_t ws_bytes, int64_t cap,
                          WsLayout* L) {
  if (!scene || !camera || !atlas || !ws) {
    set_error("null argument");
    return TSB_ERR_VALUE;
  }
  if (mode < TSB_MODE_HW || mode > TSB_MODE_FLAT) {
    set_error("unknown texture mode");
    return TSB_ERR_VALUE;
  }
  if (scene->sh_degree < 0 || scene->sh_degree > 3) {
    set_error("SH degree must be in [0, 3]");
    return TSB_ERR_VALUE;
  }
  if (mode == TSB_MODE_HW && !atlas->tex) {
    set_error("HW texture mode needs an atlas texture (tsb_atlas_tex_create)");
    return TSB_ERR_VALUE;
  }
  if (mode == TSB_MODE_VERIFY && (!atlas->family_a || !atlas->family_b)) {
    set_error("verify mode needs linear atlas pages");
    return TSB_ERR_VALUE;
  }
  if (mode == TSB_MODE_FLAT && !atlas->flat_attrs) {
    set_error("flat mode needs flat_attrs");
    return TSB_ERR_VALUE;
  }
  if (mode != TSB_MODE_FLAT && !atlas->entries) {
    set_error("textured modes need atlas indirection entries");
    return TSB_ERR_VALUE;
  }
  if (!ws_layout(scene->num_splats, camera->width, camera->height, tile, cap, L)) {
    set_error("invalid size/tile arguments");
    return TSB_ERR_VALUE;
  }
  if (ws_bytes < L->total) {
    set_error("workspace too small");
    return TSB_ERR_CAPACITY;
  }
  return TSB_OK;
}

int tsb_render_binning(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                       int32_t mode, int32_t tile, void* ws, uint64_t ws_bytes, int64_t cap,
                       int64_t* entries_needed, void* stream) {
  WsLayout L;
  int rc = validate_frame(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, &L);
  if (rc != TSB_OK) return rc;
  const int32_t P = scene->num_splats;
  cudaStream_t st = (cudaStream_t)stream;
  const tsb_cam_params cam = to_cam(camera);
  GeomRec* geom = ws_ptr<GeomRec>(ws, L.geom);
  MatRec* mat = ws_ptr<MatRec>(ws, L.mat);
  double* m64 = ws_ptr<double>(ws, L.m64);
  uint64_t* dk_in = ws_ptr<uint64_t>(ws, L.dkeys_in);
  uint64_t* dk_out = ws_ptr<uint64_t>(ws, L.dkeys_out);
  int32_t* ids_in = ws_ptr<int32_t>(ws, L.ids_in);
  int32_t* ids_out = ws_ptr<int32_t>(ws, L.ids_out);
  int32_t* tcount = ws_ptr<int32_t>(ws, L.tile_count);
  int32_t* csorted = ws_ptr<int32_t>(ws, L.counts_sorted);
  int32_t* offsets = ws_ptr<int32_t>(ws, L.offsets);
  int32_t* rank = ws_ptr<int32_t>(ws, L.rank);
  uint32_t* ek_in = ws_ptr<uint32_t>(ws, L.ekeys_in);
  uint32_t* ek_out = ws_ptr<uint32_t>(ws, L.ekeys_out);
  int32_t* ev_in = ws_ptr<int32_t>(ws, L.evals_in);
  int32_t* ev_out = ws_ptr<int32_t>(ws, L.evals_out);
  int32_t* ranges = ws_ptr<int32_t>(ws, L.ranges);
  int64_t* counters = ws_ptr<int64_t>(ws, L.counters);
  void* cub_tmp = ws_ptr<char>(ws, L.cub_tmp);
  size_t cub_bytes = L.cub_bytes;

  TSB_CUDA(cudaMemsetAsync(counters, 0, 64, st));
  TSB_CUDA(cudaMemsetAsync(ranges, 0, (size_t)L.num_tiles * 8, st));
  if (P > 0) {
    PrepParams pp;
    pp.cam = cam;
    pp.P = P; pp.sh_degree = scene->sh_degree; pp.tile = tile; pp.tiles_x = L.tiles_x;
    pp.pos = scene->positions; pp.tu = scene->tangent_u; pp.tv = scene->tangent_v;
    pp.sc = scene->scales; pp.op = scene->opacities; pp.sh = scene->sh;
    pp.entries = mode == TSB_MODE_FLAT ? nullptr : atlas->entries;
    pp.T = atlas->resolution; pp.page_w = atlas->page_w; pp.page_h = atlas->page_h;
    pp.geom = geom; pp.mat = mat; pp.m64 = m64; pp.dkeys = dk_in; pp.ids = ids_in;
    pp.tile_count = tcount;
    k_preprocess<<<(P + 255) / 256, 256, 0, st>>>(pp);
    TSB_CHECK_LAUNCH("k_preprocess");

    TSB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, dk_in, dk_out, ids_in, ids_out,
                                             P, 0, 64, st));
    k_rank_counts<<<(P + 255) / 256, 256, 0, st>>>(P, ids_out, tcount, csorted, rank);
    TSB_CHECK_LAUNCH("k_rank_counts");
    cub_bytes = L.cub_bytes;
    TSB_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, csorted, offsets, P, st));
    const int64_t C = std::max<int64_t>(cap, 1);
    TSB_CUDA(cudaMemsetAsync(ek_in, 0xFF, (size_t)C * 4, st));
    k_duplicate<<<(P + 255) / 256, 256, 0, st>>>(P, tile, L.tiles_x, cap, ids_out, csorted,
                                                 offsets, geom, ek_in, ev_in, counters);
    TSB_CHECK_LAUNCH("k_duplicate");
    cub_bytes = L.cub_bytes;
    TSB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, ek_in, ek_out, ev_in, ev_out,
                                             (int)C, 0, L.tile_bits, st));
    k_ranges<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(cap, ek_out, counters, ranges);
    TSB_CHECK_LAUNCH("k_ranges");
  }
  if (entries_needed)
    TSB_CUDA(cudaMemcpyAsync(entries_needed, counters, 8, cudaMemcpyDeviceToDevice, st));
  return TSB_OK;
}

int tsb_render_composite(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                         int32_t mode, int32_t tile, void* ws, uint64_t ws_bytes, int64_t cap,
                         float* gbuf, const tsb_pixel_state* px, void* stream) {
  WsLayout L;
  int rc = validate_frame(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, &L);
  if (rc != TSB_OK) return rc;
  if (!gbuf || !px) {
    set_error("tsb_render_composite: null output");
    return TSB_ERR_VALUE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  RasterParams rp;
  rp.cam = to_cam(camera);
  rp.W = camera->width; rp.H = camera->height; rp.tiles_x = L.tiles_x;
  rp.near_f = (float)camera->near_z;
  rp.ranges = ws_ptr<int32_t>(ws, L.ranges);
  rp.evals = ws_ptr<int32_t>(ws, L.evals_out);
  rp.geom = ws_ptr<GeomRec>(ws, L.geom);
  rp.mat = ws_ptr<MatRec>(ws, L.mat);
  rp.m64 = ws_ptr<double>(ws, L.m64);
  rp.T = atlas->resolution; rp.page_w = atlas->page_w;
  rp.fam_a = reinterpret_cast<const float4*>(atlas->family_a);
  rp.fam_b = reinterpret_cast<const float4*>(atlas->family_b);
  rp.flat = atlas->flat_attrs;
  rp.tex_a = atlas->tex ? reinterpret_cast<AtlasTex*>(atlas->tex)->tex_a : 0;
  rp.tex_b = atlas->tex ? reinterpret_cast<AtlasTex*>(atlas->tex)->tex_b : 0;
  rp.gbuf = gbuf; rp.n_contrib = px->n_contrib; rp.last_entry = px->last_entry;
  rp.final_T = px->final_T; rp.T_last = px->T_last;
  if (tile == 8) launch_raster<8>(mode, L.num_tiles, st, rp);
  else if (tile == 16) launch_raster<16>(mode, L.num_tiles, st, rp);
  else launch_raster<32>(mode, L.num_tiles, st, rp);
  TSB_CHECK_LAUNCH("k_raster_fwd");
  return TSB_OK;
}

int tsb_render_forward(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                       int32_t mode, int32_t tile, void* ws, uint64_t ws_bytes, int64_t cap,
                       float* gbuf, const tsb_pixel_state* px, int64_t* entries_needed,
                       void* stream) {
  if (!gbuf || !px) {
    set_error("tsb_render_forward: null output");
    return TSB_ERR_VALUE;
  }
  int rc = tsb_render_binning(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, entries_needed,
                              stream);
  if (rc != TSB_OK) return rc;
  return tsb_render_composite(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, gbuf, px,
                              stream);
}

int tsb_frame_export(int32_t P, int32_t W, int32_t H, int32_t tile, int64_t cap,
                     const void* ws, int32_t* sorted_ids, int64_t* keys, int32_t* ranges,
                     int32_t* rects, void* stream) {
  WsLayout L;
  if (!ws || !ws_layout(P, W, H, tile, cap, &L)) {
    set_error("tsb_frame_export: invalid arguments");
    return TSB_ERR_VALUE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (sorted_ids && P > 0)
    TSB_CUDA(cudaMemcpyAsync(sorted_ids, ws_ptr<int32_t>(ws, L.ids_out), (size_t)P * 4,
                             cudaMemcpyDeviceToDevice, st));
  if (ranges)
    TSB_CUDA(cudaMemcpyAsync(ranges, ws_ptr<int32_t>(ws, L.ranges), (size_t)L.num_tiles * 8,
                             cudaMemcpyDeviceToDevice, st));
  if (keys && cap > 0) {
    k_export_keys<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(
        cap, ws_ptr<uint32_t>(ws, L.ekeys_out), ws_ptr<int32_t>(ws, L.evals_out),
        ws_ptr<int32_t>(ws, L.rank), ws_ptr<int64_t>(ws, L.counters), keys);
    TSB_CHECK_LAUNCH("k_export_keys");
  }
  if (rects && P > 0) {
    k_export_rects<<<(P + 255) / 256, 256, 0, st>>>(P, ws_ptr<GeomRec>(ws, L.geom), rects);
    TSB_CHECK_LAUNCH("k_export_rects");
  }
  return TSB_OK;
}

int tsb_shade_forward(const float* gbuf, const tsb_camera* camera, const tsb_environment* env,
                      const float* background, float* color, float* diffuse, float* specular,
                      void* stream) {
  if (!gbuf || !camera || !env || !color) {
    set_error("tsb_shade_forward: null argument");
    return TSB_ERR_VALUE;
  }
  if (env->levels < 1 || env->levels > TSB_ENV_MAX_LEVELS || !env->lut || !env->diffuse) {
    set_error("tsb_shade_forward: bad environment");
    return TSB_ERR_VALUE;
  }
  ShadeParams sp;
  sp.cam = to_cam(camera);
  sp.env.levels = env->levels;
  for (int l = 0; l < TSB_MAX_LEVELS; ++l) {
    if (l < env->levels) {
      sp.env.mips[l].data = env->spec_mips[l];
      sp.env.mips[l].h = env->mip_h[l];
      sp.env.mips[l].w = env->mip_w[l];
    } else {
      sp.env.mips[l].data = nullptr; sp.env.mips[l].h = sp.env.mips[l].w = 0;
    }
  }
  sp.env.diffuse.data = env->diffuse;
  sp.env.diffuse.h = env->diff_h;
  sp.env.diffuse.w = env->diff_w;
  sp.env.lut = env->lut;
  sp.env.lut_res = env->lut_res;
  for (int c = 0; c < 3; ++c) sp.bg[c] = background ? background[c] : 0.f;
  sp.gbuf = gbuf; sp.color = color; sp.diffuse = diffuse; sp.specular = specular;
  const int n = camera->width * camera->height;
  k_shade<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(sp);
  TSB_CHECK_LAUNCH("k_shade");
  return TSB_OK;
}

static int make_layered(const float* src, int32_t pw, int32_t ph, int32_t pages, int32_t fmt,
                        cudaArray_t* arr, cudaTextureObject_t* tex, void* tmp16, cudaStream_t st) {
  cudaChannelFormatDesc cd = fmt == TSB_TEXEL_RGBA16F ? cudaCreateChannelDescHalf4()
                                                      : cudaCreateChannelDesc<float4>();
  TSB_CUDA(cudaMalloc3DArray(arr, &cd, make_cudaExtent(pw, ph, pages), cudaArrayLayered));
  cudaMemcpy3DParms cp = {};
  const size_t esz = fmt == TSB_TEXEL_RGBA16F ? 8 : 16;
  const void* from = src;
  if (fmt == TSB_TEXEL_RGBA16F) {
    const size_t n = (size_t)pw * ph * pages;
    k_f32_to_f16x4<<<1184, 256, 0, st>>>(reinterpret_cast<const float4*>(src),
                                        reinterpret_cast<ushort4*>(tmp16), n);
    TSB_CHECK_LAUNCH("k_f32_to_f16x4");
    from = tmp16;
  }
  cp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(from), (size_t)pw * esz, pw, ph);
  cp.dstArray = *arr;
  cp.extent = make_cudaExtent(pw, ph, pages);
  cp.kind = cudaMemcpyDeviceToDevice;
  TSB_CUDA(cudaMemcpy3DAsync(&cp, st));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = *arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModeLinear;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  TSB_CUDA(cudaCreateTextureObject(tex, &rd, &td, nullptr));
  return TSB_OK;
}

int tsb_atlas_tex_create(const float* fam_a, const float* fam_b, int32_t pw, int32_t ph,
                         int32_t pages, int32_t fmt, tsb_atlas_tex_t* out, void* stream) {
  if (!fam_a || !fam_b || !out || pw <= 0 || ph <= 0 || pages <= 0 ||
      (fmt != TSB_TEXEL_RGBA32F && fmt != TSB_TEXEL_RGBA16F)) {
    set_error("tsb_atlas_tex_create: invalid arguments");
    return TSB_ERR_VALUE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  AtlasTex* t = new AtlasTex();
  t->page_w = pw; t->page_h = ph; t->pages = pages; t->format = fmt;
  void* tmp16 = nullptr;
  if (fmt == TSB_TEXEL_RGBA16F) {
    cudaError_t e = cudaMallocAsync(&tmp16, (size_t)pw * ph * pages * 8, st);
    if (e != cudaSuccess) { delete t; return cuda_fail("cudaMallocAsync", e); }
  }
  int rc = make_layered(fam_a, pw, ph, pages, fmt, &t->arr_a, &t->tex_a, tmp16, st);
  if (rc == TSB_OK) rc = make_layered(fam_b, pw, ph, pages, fmt, &t->arr_b, &t->tex_b, tmp16, st);
  if (tmp16) {
    cudaStreamSynchronize(st);
    cudaFreeAsync(tmp16, st);
  }
  if (rc != TSB_OK) {
    tsb_atlas_tex_destroy(reinterpret_cast<tsb_atlas_tex_t>(t));
    return rc;
  }
  *out = reinterpret_cast<tsb_atlas_tex_t>(t);
  return TSB_OK;
}

int tsb_atlas_tex_destroy(tsb_atlas_tex_t h) {
  if (!h) return TSB_OK;
  AtlasTex* t = reinterpret_cast<AtlasTex*>(h);
  if (t->tex_a) cudaDestroyTextureObject(t->tex_a);
  if (t->tex_b) cudaDestroyTextureObject(t->tex_b);
  if (t->arr_a) cudaFreeArray(t->arr_a);
  if (t->arr_b) cudaFreeArray(t->arr_b);
  delete t;
  return TSB_OK;
}

int tsb_tex_probe(tsb_atlas_tex_t h, int32_t window, int32_t iters, float* sink, int32_t blocks,
                  int32_t threads, void* stream) {
  if (!h || !sink || window <= 0 || iters <= 0 || blocks <= 0 || threads <= 0) {
    set_error("tsb_tex_probe: invalid arguments");
    return TSB_ERR_VALUE;
  }
  AtlasTex* t = reinterpret_cast<AtlasTex*>(h);
  k_tex_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(t->tex_a, window, iters, sink);
  TSB_CHECK_LAUNCH("k_tex_probe");
  return TSB_OK;
}

}  // extern "C"
