// tsb_forward.cu — forward render path for sm_100a.
//
//   K1 k_preprocess     per splat, fp64: rect/cull, centre depth key, M, frame,
//                       SH radiance -> GeomRec / MatRec / fp64 M; per-CTA
//                       digit histograms of the depth key and of the entries'
//                       tile columns / rows (difference arrays)
//   S1 depth order      4 one-sweep passes + k_fix_runs (+ k_sort_long_runs):
//                       exact (fp64 z, id) order == np.lexsort((ids, z))
//   S2 tile lists       k_dup_tx (duplication fused with the tile-x pass) +
//                       one-sweep tile-y pass => per-tile lists in draw order
//   K4 k_ranges         [start, end) per tile          (S1, S2, K4: tsb_binning.cu)
//   K5 k_raster_fwd     persistent warps over (tile, 8x4 block) units: staged
//                       geometry in smem, fp32 intersection with fp64 guard
//                       band, TEX/verify/flat texel fetch, 13-channel
//                       front-to-back composite
//   K6 k_shade          per pixel split-sum PBR (shading.py:126-183)
//
// Reference: /root/reference/pkg/src/texsplat/rasterize.py:127-438,
// shading.py:51-183 (see tsb_math.h for line-level citations).

#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <vector>

#include "tsb_binning.cuh"
#include "tsb_internal.cuh"

// Rasterizer CTA shape: persistent warps, so any tile size runs with the
// same CTA (TSB_RASTER_WARPS warps, TSB_RASTER_MINB resident CTAs per SM).
#ifndef TSB_RASTER_WARPS
#define TSB_RASTER_WARPS 8
#endif
#ifndef TSB_RASTER_MINB
#define TSB_RASTER_MINB 3
#endif

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
  // entry keys (tile_y << 8 | tile_x): at most 256 tiles per axis
  if (L->tiles_x > kMaxTileAxis || L->tiles_y > kMaxTileAxis) return false;
  if (cap >= (int64_t)1 << 30) return false;  // look-back words hold 30-bit counts
  L->num_tiles = L->tiles_x * L->tiles_y;
  int bits = 1;
  while ((1ll << bits) <= (int64_t)L->num_tiles) ++bits;
  L->tile_bits = bits;
  const size_t Pn = (size_t)std::max(P, 1);
  const size_t C = (size_t)std::max<int64_t>(cap, 1);
  L->nb_depth = (int32_t)((Pn + kOsTileDepth - 1) / kOsTileDepth);
  L->nb_dup = (int32_t)((Pn + kOsThreads - 1) / kOsThreads);
  L->nb_tiley = (int32_t)((C + kOsTile - 1) / kOsTile);
  L->status_words = kDepthPasses * pass_status_words(L->nb_depth) +
                    pass_status_words(L->nb_dup) + pass_status_words(L->nb_tiley);

  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  L->geom = take(Pn * sizeof(GeomRec));
  L->rects = take(Pn * 8);
  L->mat = take(Pn * sizeof(MatRec));
  L->m64 = take(Pn * kM64Stride * sizeof(double));
  L->dkeys_in = take(Pn * 8);   // full fp64 depth bits by id
  L->dkeys_out = take(Pn * 8);  // scratch of k_sort_long_runs
  L->dk32_in = take(Pn * 4);
  L->dk32_out = take(Pn * 4);
  L->ids_in = take(Pn * 4);
  L->ids_out = take(Pn * 4);    // the draw order
  L->tile_count = take(Pn * 8);  // BinRec (uint2) by id: record slot, tile box
  L->rank = take(Pn * 4);
  L->long_runs = take((Pn / (kShortRun + 2) + 1) * 8);
  L->ekeys_in = take(C * 4);
  L->ekeys_out = take(C * 4);
  L->evals_in = take(C * 4);
  L->evals_out = take(C * 4);
  L->ranges = take((size_t)L->num_tiles * 8);
  L->torder_out = take((size_t)L->num_tiles * 4);
  L->max_needed = take(8);  // running max over frames (never reset by a frame)
  // zeroed per frame as one block: counters, binning state, look-back words
  L->counters = take(64);
  L->bin = take(sizeof(BinCounters));
  L->status = take(L->status_words * 4);
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
  uint2* rects;
  MatRec* mat;
  double* m64;
  uint64_t* dkeys;
  uint32_t* dkey32;
  uint32_t near_hi;      // high word of bits(near)
  int32_t* ids;
  uint2* bin_rec;         // by id: (record slot, tile box) for k_dup_tx
  const int32_t* slot;  // record storage permutation (tsb_scene.record_slot) or null
  BinCounters* bin;     // digit histograms, kept count
  int64_t* total;       // entries of the frame (counters[0])
};

#ifndef TSB_PREP_MINB
#define TSB_PREP_MINB 3  // 80 registers: 3 CTAs/SM hide the fp64 and store latency
#endif
__global__ void __launch_bounds__(256, TSB_PREP_MINB) k_preprocess(PrepParams p) {
  // per-CTA binning histograms (merged into p.bin with one atomic per non-zero bin)
  __shared__ int32_t s_hd[kDepthPasses][kRadixBins];
  __shared__ int32_t s_hx[kRadixBins + 1], s_hy[kRadixBins + 1];
  __shared__ int32_t s_kept;
  __shared__ unsigned long long s_total;
  for (int i = threadIdx.x; i < kDepthPasses * (int)kRadixBins; i += blockDim.x)
    (&s_hd[0][0])[i] = 0;
  for (int i = threadIdx.x; i <= (int)kRadixBins; i += blockDim.x) s_hx[i] = s_hy[i] = 0;
  if (threadIdx.x == 0) { s_kept = 0; s_total = 0ull; }
  __syncthreads();
  // grid-stride over the splats (the grid is capped at a few CTAs per SM, so
  // the shared-memory histograms are cleared and merged once per CTA, not
  // once per 256 splats)
  for (int id0 = blockIdx.x * blockDim.x; id0 < p.P; id0 += gridDim.x * blockDim.x) {
  const int id = id0 + threadIdx.x;
  uint32_t kkey = kDepthCulled32, kkept = 0, ktiles = 0;  // this splat's binning facts
  if (id < p.P) {
  const int K = (p.sh_degree + 1) * (p.sh_degree + 1);
  double pos[3], tu[3], tv[3], s[2];
  for (int j = 0; j < 3; ++j) {
    pos[j] = p.pos[3 * id + j];
    tu[j] = p.tu[3 * id + j];
    tv[j] = p.tv[3 * id + j];
  }
  s[0] = p.sc[2 * id];
  s[1] = p.sc[2 * id + 1];
  // SH coefficients read in place (a local copy would live in local memory)
  const double* sh = p.sh + (size_t)3 * K * id;
  tsb_prep r;
  tsb_prep_cull(&p.cam, pos, tu, tv, s, &r);  // centre depth, rect, keep
  p.rects[id] = make_uint2((uint32_t)r.x0 | ((uint32_t)r.x1 << 16),
                           (uint32_t)r.y0 | ((uint32_t)r.y1 << 16));
  p.ids[id] = id;
  if (!r.keep) {  // culled: no M / frame / SH work, no entries, sorts last
    p.bin_rec[id] = make_uint2(0u, kBinNoTiles);
    p.dkeys[id] = ~0ull;
    p.dkey32[id] = kDepthCulled32;
  } else {
  tsb_prep_kept(&p.cam, pos, tu, tv, s, sh, p.sh_degree, &r);
  const double op = p.op[id];

  GeomRec g;
  tsb_make_lin(r.m, op, g.lin);
  g.r2lo = tsb_lin_r2lo(g.lin[11]);
  int32_t tb[4];
  tsb_test_box(&p.cam, r.m, g.lin[11], r.x0, r.x1, r.y0, r.y1, tb);
  g.bx = (uint32_t)tb[0] | ((uint32_t)tb[1] << 16);
  g.by = (uint32_t)tb[2] | ((uint32_t)tb[3] << 16);
  g.id = id;
  // Tile binning by the test box (reference rect ∩ alpha-cut ellipse box):
  // a strictly tighter, conservative version of _tile_lists' rect binning
  // (rasterize.py:246-258) — tiles outside it cannot hold a live pixel.
  const bool binned = tb[1] > tb[0] && tb[3] > tb[2];
  int32_t ntiles = 0;
  uint32_t tbox = kBinNoTiles;
  if (binned) {
    const int tx0 = tb[0] / p.tile, tx1 = (tb[1] - 1) / p.tile;
    const int ty0 = tb[2] / p.tile, ty1 = (tb[3] - 1) / p.tile;
    const int nx = tx1 - tx0 + 1, ny = ty1 - ty0 + 1;
    ntiles = nx * ny;
    tbox = (uint32_t)tx0 | ((uint32_t)ty0 << 8) | ((uint32_t)(nx - 1) << 16) |
           ((uint32_t)(ny - 1) << 24);
    // entries per tile column / row as difference arrays (k_dup_tx, tile-y pass)
    atomicAdd(&s_hx[tx0], ny);
    atomicAdd(&s_hx[tx1 + 1], -ny);
    atomicAdd(&s_hy[ty0], nx);
    atomicAdd(&s_hy[ty1 + 1], -nx);
  }
  p.bin_rec[id] = make_uint2(binned ? (uint32_t)(p.slot ? p.slot[id] : id) : 0u, tbox);
  // 32-bit depth key: the high word of bits(z) minus that of bits(near) is
  // monotone in z for z > near (positive doubles order like their bit
  // patterns; 2^-20 relative resolution, no clamping); k_fix_runs re-orders
  // equal keys by the full 64-bit pattern => the exact (z, id) order.
  const uint64_t full = tsb_f64_bits(r.view_z);
  p.dkeys[id] = full;
  const uint32_t k32 = (uint32_t)(full >> 32) - p.near_hi;
  p.dkey32[id] = k32;
  kkey = k32;  // (the depth histograms count kept splats only)
  kkept = 1;
  ktiles = (uint32_t)ntiles;
  // the rasterizer and the backward read records only through tile-list
  // entries: splats without entries (culled, or no pixel in the box) skip them
  if (binned) {
  const int sl = p.slot ? p.slot[id] : id;  // records live at the splat's slot
  p.geom[sl] = g;

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
  p.mat[sl] = m;

  double* m64 = p.m64 + (size_t)kM64Stride * id;  // the rare fp64 recheck: by id
  for (int k = 0; k < 9; ++k) m64[k] = r.m[k];
  m64[9] = op;
  }
  }  // kept
  }
  // warp-aggregated histogram updates (equal digits of a warp: one atomic)
  {
    const int lane = threadIdx.x & 31;
    const bool valid = id < p.P && kkept;
#pragma unroll
    for (int q = 0; q < kDepthPasses; ++q) {
      const uint32_t d = valid ? (kkey >> (8 * q)) & 255u : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (valid && lane == __ffs(peers) - 1) atomicAdd(&s_hd[q][d], __popc(peers));
    }
    const uint32_t nk = __reduce_add_sync(0xffffffffu, kkept);
    const uint32_t nt = __reduce_add_sync(0xffffffffu, ktiles);
    if (lane == 0 && nk) atomicAdd(&s_kept, (int)nk);
    if (lane == 0 && nt) atomicAdd(&s_total, (unsigned long long)nt);
  }
  }  // grid-stride
  __syncthreads();
  for (int i = threadIdx.x; i < kDepthPasses * (int)kRadixBins; i += blockDim.x) {
    const int v = (&s_hd[0][0])[i];
    if (v) atomicAdd(&(&p.bin->hist_depth[0][0])[i], v);
  }
  for (int i = threadIdx.x; i <= (int)kRadixBins; i += blockDim.x) {
    if (s_hx[i]) atomicAdd(&p.bin->hist_tx[i], s_hx[i]);
    if (s_hy[i]) atomicAdd(&p.bin->hist_ty[i], s_hy[i]);
  }
  if (threadIdx.x == 0) {
    if (s_kept) atomicAdd(&p.bin->kept, s_kept);
    if (s_total) atomicAdd(reinterpret_cast<unsigned long long*>(p.total), s_total);
  }
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
  int32_t T, page_w, tstride;
  float t6, t2, tmh;  // T/6, T/2, T-1/2 (HW-mode texel coordinates)
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
  uint8_t* touched;
  int32_t num_tiles;
  int32_t* work_counter;      // zeroed per frame
  const int32_t* tile_order;  // tiles by descending list length (may be null)
};

// tsb_decode_normal with the SFU's approximate square roots (HW-texture mode
// only, whose texels are already filtered with 8-bit weights; verify mode
// keeps the correctly rounded path that matches the oracle bit for bit).
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void tsb_decode_normal_approx(float ea, float eb, const float* frame,
                                                         float* nw) {
  float nx = fmaf(2.0f, ea, -1.0f);
  float ny = fmaf(2.0f, eb, -1.0f);
  const float d2 = fmaf(nx, nx, ny * ny);
  float nz = 0.0f;  // projected onto the unit disk: |n_xy| = 1, n_z = 0
  if (d2 > 1.0f) {
    const float sc = rsqrt_approx(d2);
    nx *= sc;
    ny *= sc;
  } else {
    nz = sqrt_approx(1.0f - d2);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
    nw[i] = fmaf(nz, frame[6 + i], fmaf(ny, frame[3 + i], nx * frame[i]));
}

#ifndef TSB_PAIR_ILP_VERIFY
#define TSB_PAIR_ILP_VERIFY 1
#endif
#ifndef TSB_PAIR_ILP_FLAT
#define TSB_PAIR_ILP_FLAT 2
#endif
#ifndef TSB_PAIR_ILP
#define TSB_PAIR_ILP 2
#endif
#ifndef TSB_RASTER_CARVEOUT
#define TSB_RASTER_CARVEOUT 44  // percent of 228 KB: 100 KB for 3 x 31 KB CTAs
#endif

#ifdef TSB_STATS
// Work counters of k_raster_fwd (instrumented builds only: make EXTRA=-DTSB_STATS):
// 0 units, 1 steps, 2 candidates, 3 block-full candidates, 5 pair iterations,
// 6 composited pairs, 8 undone lanes at decide, 9 live pairs, 10 undone lanes x candidates.
__device__ unsigned long long g_tsb_stats[16];
#endif

// Warp-private shared memory of the rasterizer.
struct DecCopy {
  DecRec dec[32];             // 48-B decide records (verify mode, see below)
};
struct NoDecCopy {};

template <bool SEP_DEC>
struct WarpSmemT : std::conditional_t<SEP_DEC, DecCopy, NoDecCopy> {
  int32_t sid[32];            // splat ids
  uint32_t pm[32];            // the entry's pixel mask of the current block
  // one 112-byte record per entry, read with 128-bit loads (7 x 16 B: the
  // stride is odd in 16-byte units, so lanes reading different entries of one
  // quarter-warp rarely share banks); texturing reads all of it and, in HW
  // and flat mode, the decide loop reads [0..2] with every lane on the same
  // entry (broadcast). One copy per warp keeps the CTA at 31 KB of shared
  // memory, so 3 CTAs/SM fit the 100 KB carveout and L1 keeps ~156 KB for
  // the atlas. Verify mode keeps a separate 48-B decide copy (measured: its
  // global-load texel path runs 2.5-5% faster with it, HW mode 1% slower):
  //   [0] L0..L3  [1] L4..L7  [2] L8, det, opacity, r2hi   (intersection forms)
  //   [3] chart origin x, y (texels), page, linear offset
  //   [4] frame 0..3  [5] frame 4..7  [6] frame 8, clamped SH radiance rgb
  float4 rec[32][7];
  BlockBox bb;                // the current unit's block (read by the stage step)
};
template <int MODE>
using WarpSmem = WarpSmemT<MODE == TSB_MODE_VERIFY>;
template <int MODE>
constexpr size_t kRasterWarpSmem = (sizeof(WarpSmem<MODE>) + 15) & ~size_t(15);

// A pair whose texel fetch is in flight.
struct PairFetch {
  float4 A, B;
  float z, a;
  int k;
};

// Stage 1 of texturing a (pixel, splat) pair: intersection values and the
// texel fetch issue (tex2DLayered in HW mode, 8 corner loads in verify
// mode); no use of the fetched data yet, so several pairs overlap.
template <int MODE>
__device__ __forceinline__ void pair_issue(const RasterParams& p, const WarpSmem<MODE>& ws, int q,
                                           float2 xy, PairFetch& f) {
  const int k = q & 31;
  const float4 r0 = ws.rec[k][0], r1 = ws.rec[k][1], r2 = ws.rec[k][2], r3 = ws.rec[k][3];
  const float L[11] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y, r2.z};
  float u, v;
  tsb_uvza_lin(L, xy.x, xy.y, &u, &v, &f.z, &f.a);
  f.k = k;
  if (MODE == TSB_MODE_FLAT) {
    const float* fl = p.flat + 5 * ws.sid[k];
    f.A = make_float4(__ldg(fl), __ldg(fl + 1), __ldg(fl + 2), __ldg(fl + 4));
    f.B = make_float4(0.f, 0.f, __ldg(fl + 3), 0.f);
    return;
  }
  if (MODE == TSB_MODE_HW) {
    // texture-unit coordinates of the reference footprint (textures.py:152-200):
    // xs = clamp(clamp((u+3)/6, h, 1-h) T - 0.5, 0, T-1), sampled at xs + 0.5,
    // i.e. chart origin + clamp(u T/6 + T/2, 1/2, T - 1/2) (the filter's own
    // 8-bit weights dominate the rounding difference; tolerance-checked mode)
    const float sx = r3.x + fminf(fmaxf(fmaf(u, p.t6, p.t2), 0.5f), p.tmh);
    const float sy = r3.y + fminf(fmaxf(fmaf(v, p.t6, p.t2), 0.5f), p.tmh);
    const int page = __float_as_int(r3.z);
#ifdef TSB_PROBE_NOTEX
    f.A = make_float4(sx * 1e-9f, 0.5f, 0.5f, 0.5f);
    f.B = make_float4(0.5f, sy * 1e-9f + 0.5f, 0.2f, 0.f);
#else
    f.A = tex2DLayered<float4>(p.tex_a, sx, sy, page);
    f.B = tex2DLayered<float4>(p.tex_b, sx, sy, page);
#endif
  } else {
    tsb_texc tc;
    tsb_texel_coords(u, v, p.T, &tc);
    const int S = p.tstride;
    const int loff = __float_as_int(r3.w);
    const int r0 = loff + tc.j0 * p.page_w, r1 = loff + tc.j1 * p.page_w;
    const float4 a00 = __ldg(p.fam_a + S * (r0 + tc.i0)), a01 = __ldg(p.fam_a + S * (r0 + tc.i1));
    const float4 a10 = __ldg(p.fam_a + S * (r1 + tc.i0)), a11 = __ldg(p.fam_a + S * (r1 + tc.i1));
    const float4 b00 = __ldg(p.fam_b + S * (r0 + tc.i0)), b01 = __ldg(p.fam_b + S * (r0 + tc.i1));
    const float4 b10 = __ldg(p.fam_b + S * (r1 + tc.i0)), b11 = __ldg(p.fam_b + S * (r1 + tc.i1));
    f.A.x = tsb_lerp4(a00.x, a01.x, a10.x, a11.x, tc.fs, tc.ft);
    f.A.y = tsb_lerp4(a00.y, a01.y, a10.y, a11.y, tc.fs, tc.ft);
    f.A.z = tsb_lerp4(a00.z, a01.z, a10.z, a11.z, tc.fs, tc.ft);
    f.A.w = tsb_lerp4(a00.w, a01.w, a10.w, a11.w, tc.fs, tc.ft);
    f.B.x = tsb_lerp4(b00.x, b01.x, b10.x, b11.x, tc.fs, tc.ft);
    f.B.y = tsb_lerp4(b00.y, b01.y, b10.y, b11.y, tc.fs, tc.ft);
    f.B.z = tsb_lerp4(b00.z, b01.z, b10.z, b11.z, tc.fs, tc.ft);
    f.B.w = 0.f;
  }
}

// Stage 2: normal decode (rasterize.py:313-314) and the pair's attribute
// row into result slot t.
template <int MODE>
__device__ __forceinline__ void pair_result(const WarpSmem<MODE>& ws, const PairFetch& f, float* rv) {
  const float4 r4 = ws.rec[f.k][4], r5 = ws.rec[f.k][5], r6 = ws.rec[f.k][6];
  const float fr[9] = {r4.x, r4.y, r4.z, r4.w, r5.x, r5.y, r5.z, r5.w, r6.x};
  float nw[3];
  if (MODE == TSB_MODE_FLAT) {
    nw[0] = fr[6]; nw[1] = fr[7]; nw[2] = fr[8];
  } else if (MODE == TSB_MODE_HW) {
    tsb_decode_normal_approx(f.B.x, f.B.y, fr, nw);
  } else {
    tsb_decode_normal(f.B.x, f.B.y, fr, nw);
  }
  rv[0] = f.A.x;
  rv[1] = f.A.y;
  rv[2] = f.A.z;
  rv[3] = f.B.z;  // metallic
  rv[4] = f.A.w;  // roughness
  rv[5] = nw[0];
  rv[6] = nw[1];
  rv[7] = nw[2];
  rv[8] = f.z;
  rv[9] = f.a;
  rv[10] = r6.y;  // clamped SH radiance
  rv[11] = r6.z;
  rv[12] = r6.w;
}


// K5. One CTA per TILE x TILE tile; each warp owns 8 x 4 pixel blocks of the
// tile and walks the tile's draw-ordered list on its own (no CTA barriers; a
// warp retires as soon as its pixels saturate). Per step of 32 list entries:
//   stage    the 32 splat records into warp-private shared memory (SoA) and
//            ballot the ones whose test box (rect ∩ alpha-cut ellipse box)
//            touches the block;
//   decide   per pixel, which candidates composite (test box, 6-FMA linear
//            forms, division-free reject, alpha cut + fp64 guard band) —
//            a live bitmask; nothing here depends on transmittance;
//   texture  each lane walks its pixel's live bits in draw order, two pairs
//   + blend  per iteration (both texel fetches in flight before the first
//            blend), and composites them with the reference's T gate
//            (rasterize.py:366-381); a saturated pixel stops fetching.
// (An earlier variant compacted the live pairs of all 32 pixels into a
// round-robin list so texturing ran with full lanes; the compaction's shared-
// memory round trips cost more than the idle lanes it saved: 0.49 -> 0.35 ms
// on cfg2.)
// The per-pixel decision and blend sequence is exactly the reference's
// (tsb_math.h); the work split never changes a bit of the result.
template <int TILE, int MODE>
__global__ void __launch_bounds__(32 * TSB_RASTER_WARPS, TSB_RASTER_MINB)
k_raster_fwd(RasterParams p) {
  pdl_wait();
  constexpr int NBLK = TILE * TILE / 32;  // 8 x 4 pixel blocks per tile
  constexpr int WX = TILE / 8;            // blocks per tile row
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr bool SEP = MODE == TSB_MODE_VERIFY;
  WarpSmem<MODE>& ws =
      *reinterpret_cast<WarpSmem<MODE>*>(s_raw + (size_t)warp * kRasterWarpSmem<MODE>);
  const float teps = (float)TSB_TRANSMIT_EPS;

  // Persistent warps: each warp pulls (tile, 8x4 block) work units from a
  // global counter, in descending order of the tile's list length (heavy
  // silhouette tiles first), so the frame has no long tail.
  const int num_units = p.num_tiles * NBLK;
  while (true) {
    int unit = 0;
    if (lane == 0) unit = atomicAdd(p.work_counter, 1);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= num_units) break;
#ifdef TSB_STATS
    if (lane == 0) atomicAdd(&g_tsb_stats[0], 1ull);
#endif
    const int tile = p.tile_order ? p.tile_order[unit / NBLK] : unit / NBLK;
    const int blk = unit % NBLK;
    const int start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
    {
    const int bx0 = (tile % p.tiles_x) * TILE + (blk % WX) * 8;
    const int by0 = (tile / p.tiles_x) * TILE + (blk / WX) * 4;
    if (bx0 >= p.W || by0 >= p.H) continue;
    const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
    const bool inside = px < p.W && py < p.H;
    const float x = (float)tsb_pixel_x(&p.cam, px), y = (float)tsb_pixel_y(&p.cam, py);
    const int bx1 = min(bx0 + 8, p.W), by1 = min(by0 + 4, p.H);
    __syncwarp();
    if (lane == 0) ws.bb = tsb_block_box(p.cam, bx0, by0, bx1, by1);
    __syncwarp();
    const BlockBox& bb = ws.bb;

    float acc[13];
#pragma unroll
    for (int c = 0; c < 13; ++c) acc[c] = 0.f;
    float T = 1.f, T_last = 1.f;
    int n = 0, last = -1;
    bool done = !inside;

    for (int base = start; base < end; base += 32) {
      if (__all_sync(0xffffffffu, done)) break;
      // ---- stage
      const int e = base + lane;
      bool hit = false;
      uint32_t bflags = 0;
      __syncwarp();
      if (e < end) {
        const int rs = __ldg(p.evals + e);  // the entry's record slot
        float4 gv[4];
        DecRec* dcopy = nullptr;
        if constexpr (SEP) dcopy = ws.dec;
        const uint32_t pm = tsb_stage_geom(p.geom, rs, lane, bx0, by0, bx1, by1, dcopy, bb,
                                           p.near_f, bflags, gv);
        hit = pm != 0;
        ws.sid[lane] = __float_as_int(gv[3].z);  // splat id (GeomRec.id)
        ws.pm[lane] = pm;
        if (hit) {  // the material record only for splats touching the block
          const float4* mq = reinterpret_cast<const float4*>(p.mat + rs);
          float4* rec = ws.rec[lane];
          rec[0] = gv[0]; rec[1] = gv[1]; rec[2] = gv[2];
          rec[4] = __ldg(mq); rec[5] = __ldg(mq + 1); rec[6] = __ldg(mq + 2); rec[3] = __ldg(mq + 3);
        }
      }
      const uint32_t cand = __ballot_sync(0xffffffffu, hit);
      const uint32_t fullm = __ballot_sync(0xffffffffu, (bflags & kBlockLive) != 0);
      const uint32_t zsm = __ballot_sync(0xffffffffu, (bflags & kBlockZSafe) != 0);
      __syncwarp();
      if (!cand) continue;
      // ---- decide (splats surely live on the whole block need no per-pixel test)
      // z-safe candidates: each lane tests its own splat at all 32 pixels
      // (tsb_decide_candidate), then a bit transpose gives each pixel lane its
      // live / undecided candidates; the rest go through the per-pixel loop.
      uint32_t lc = 0, uc = 0;
      const bool zc = hit && (bflags & (kBlockZSafe | kBlockLive)) == kBlockZSafe;
      if (__any_sync(0xffffffffu, zc)) {
        float xs[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) xs[c] = __shfl_sync(0xffffffffu, x, c);
        // (the staged forms of this lane's own entry; written for every hit)
        lc = tsb_decide_candidate(ws.rec[lane][0], ws.rec[lane][1], ws.rec[lane][2], xs, y, uc);
        const uint32_t keep = zc ? ws.pm[lane] : 0u;
        lc &= keep;
        uc &= keep;
        lc = tsb_warp_transpose32(lc, lane);
        uc = tsb_warp_transpose32(uc, lane);
      }
      uint32_t live = 0;
      if (!done)
        live = fullm | tsb_decide_step(
                           [&](int k) {
                             if constexpr (SEP) {
                               const DecRec& d = ws.dec[k];
                               return DecRef{d.lin, d.r2hi, d.pixmask};
                             } else {
                               const float* l = reinterpret_cast<const float*>(ws.rec[k]);
                               return DecRef{l, l[11], ws.pm[k]};
                             }
                           },
                           [&](int k, float* L) {
                             const float4 a = ws.rec[k][0], b = ws.rec[k][1], c = ws.rec[k][2];
                             L[0] = a.x; L[1] = a.y; L[2] = a.z; L[3] = a.w;
                             L[4] = b.x; L[5] = b.y; L[6] = b.z; L[7] = b.w;
                             L[8] = c.x; L[9] = c.y; L[10] = c.z; L[11] = c.w;
                           },
                           ws.sid, cand & ~fullm & ~zsm, 0u, lane, x, y, p.near_f, p.cam, p.m64,
                           px, py, lc, uc);
#ifdef TSB_STATS
      {
        const uint32_t nd = __ballot_sync(0xffffffffu, !done);
        const int lv = __reduce_add_sync(0xffffffffu, (unsigned)__popc(live));
        if (lane == 0) {
          atomicAdd(&g_tsb_stats[1], 1ull);
          atomicAdd(&g_tsb_stats[2], (unsigned long long)__popc(cand));
          atomicAdd(&g_tsb_stats[3], (unsigned long long)__popc(fullm));
          atomicAdd(&g_tsb_stats[8], (unsigned long long)__popc(nd));
          atomicAdd(&g_tsb_stats[9], (unsigned long long)lv);
          atomicAdd(&g_tsb_stats[10], (unsigned long long)__popc(nd) * __popc(cand));
        }
      }
#endif
      // ---- texture + blend, in order, ILP live pairs per lane per iteration
      // (verify mode consumes its 8 corner loads inside pair_issue, so a
      // second pair in flight only costs registers there)
      constexpr int ILP = MODE == TSB_MODE_VERIFY ? TSB_PAIR_ILP_VERIFY
                          : MODE == TSB_MODE_FLAT ? TSB_PAIR_ILP_FLAT : TSB_PAIR_ILP;
      while (__any_sync(0xffffffffu, live != 0)) {
#ifdef TSB_STATS
        if (lane == 0) atomicAdd(&g_tsb_stats[5], 1ull);
#endif
        if (live) {
          int kk[ILP];
          bool hv[ILP];
          PairFetch f[ILP];
#pragma unroll
          for (int j = 0; j < ILP; ++j) {
            hv[j] = live != 0;
            kk[j] = hv[j] ? __ffs(live) - 1 : 0;
            live &= live - 1;
            if (hv[j]) pair_issue<MODE>(p, ws, kk[j], make_float2(x, y), f[j]);
          }
#pragma unroll
          for (int j = 0; j < ILP; ++j) {
            if (hv[j] && !done) {
              const int k = kk[j];
              float rv[13];
              pair_result<MODE>(ws, f[j], rv);
              float xa[12];
#pragma unroll
              for (int c = 0; c < 8; ++c) xa[c] = rv[c];
              xa[8] = rv[10]; xa[9] = rv[11]; xa[10] = rv[12];
              xa[11] = rv[8];
              T_last = T;
              T = tsb_composite(acc, xa, rv[9], T);
              ++n;
              last = base + k;
#ifdef TSB_STATS
              atomicAdd(&g_tsb_stats[6], 1ull);
#endif
              if (p.touched) p.touched[ws.sid[k]] = 1;
              if (!(T > teps)) { done = true; live = 0; }
            }
          }
        }
      }
      __syncwarp();
    }
    if (inside) {
      const int HW = p.W * p.H;
      const int pix = py * p.W + px;
#pragma unroll
      for (int c = 0; c < 13; ++c) p.gbuf[(size_t)c * HW + pix] = acc[c];
      p.n_contrib[pix] = n;
      p.last_entry[pix] = last;
      p.final_T[pix] = T;
      p.T_last[pix] = T_last;
    }
    }
  }
}

// The persistent rasterizer's schedule: tiles by descending list length
// (longest-processing-time first). One CTA counting-sorts the tiles on
// length/2 (clamped at 2047); the order inside a bucket is free — the
// schedule never changes a result.
constexpr int kSchedThreads = 1024;
__global__ void __launch_bounds__(kSchedThreads) k_tile_schedule(int32_t nt,
                                                                 const int32_t* __restrict__ ranges,
                                                                 int32_t* __restrict__ order,
                                                                 int32_t* __restrict__ work_counter) {
  pdl_wait();
  if (threadIdx.x == 0) *work_counter = 0;  // K5's unit counter (K5 waits for this kernel)
  __shared__ int cursor[kSchedThreads];
  __shared__ int wsum[kSchedThreads / 32];
  const int tid = threadIdx.x;
  cursor[tid] = 0;
  __syncthreads();
  auto bucket = [&](int t) {
    const int c = ranges[2 * t + 1] - ranges[2 * t];
    return kSchedThreads - 1 - (min(c, 2 * kSchedThreads - 1) >> 1);
  };
  for (int t = tid; t < nt; t += kSchedThreads) atomicAdd(&cursor[bucket(t)], 1);
  __syncthreads();
  const int h = cursor[tid];
  int x = h;  // block exclusive scan: warp scans, then a scan of the warp totals
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  cursor[tid] = (w ? wsum[w - 1] : 0) + x - h;
  __syncthreads();
  for (int t = tid; t < nt; t += kSchedThreads) order[atomicAdd(&cursor[bucket(t)], 1)] = t;
}

struct ShadeParams {
  tsb_cam_params cam;
  tsb_env_params env;
  float bg[3];
  ViewCoeffs view;  // K6 view directions
  const float* gbuf;
  float* color;
  float* diffuse;
  float* specular;
};

__global__ void __launch_bounds__(256) k_shade(ShadeParams p) {
  pdl_wait();
  const int W = p.cam.width, H = p.cam.height;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= W * H) return;
  float g[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) g[c] = __ldg(p.gbuf + (size_t)c * W * H + pix);
  float wo[3];
  view_dir_pix(p.view, pix, W, wo);
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
                              const int32_t* __restrict__ evals, const GeomRec* __restrict__ geom,
                              const int32_t* __restrict__ rank,
                              const int64_t* __restrict__ counters, int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  int64_t total = counters[0];
  if (total > cap) total = 0;
  keys[i] = i < total ? (((int64_t)ekeys[i] << 32) | (int64_t)(uint32_t)rank[geom[evals[i]].id])
                      : -1;  // entries name record slots; the record carries the id
}

__global__ void k_export_rects(int32_t P, const uint2* __restrict__ rc, int32_t* __restrict__ rects) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= P) return;
  const uint32_t rx = rc[id].x, ry = rc[id].y;
  rects[4 * id] = rx & 0xFFFF; rects[4 * id + 1] = rx >> 16;
  rects[4 * id + 2] = ry & 0xFFFF; rects[4 * id + 3] = ry >> 16;
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

// Scattered float atomic adds into an L2-resident buffer (the backward's
// gradient scatter pattern, no contention): the RED throughput peak for the
// K8 roofline. Each thread issues `iters` independent adds.
__global__ void k_red_probe(float* __restrict__ buf, uint32_t mask, int32_t iters) {
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int k = 0; k < iters; ++k) {
    h = h * 1664525u + 1013904223u;
    atomicAdd(buf + ((h >> 7) & mask), 1.0f);
  }
}

template <int TILE, int MODE>
inline cudaError_t launch_raster_mode(int blocks, cudaStream_t st, const RasterParams& rp) {
  constexpr int threads = 32 * TSB_RASTER_WARPS;
  const size_t smem = (size_t)(threads / 32) * kRasterWarpSmem<MODE>;
  static PerDevice s_resident;  // per instantiation and device: persistent grid size
  int resident = 0;
  cudaError_t e = s_resident.get(
      [smem](int dev) {
        cudaError_t r = cudaFuncSetAttribute(k_raster_fwd<TILE, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // the smallest shared-memory carveout that holds the resident CTAs: the
        // rest of the 256 KB stays L1, which caches the atlas texels
        if (r == cudaSuccess)
          r = cudaFuncSetAttribute(k_raster_fwd<TILE, MODE>,
                                   cudaFuncAttributePreferredSharedMemoryCarveout,
                                   MODE == TSB_MODE_VERIFY ? -1 : TSB_RASTER_CARVEOUT);
        int sms = 0, per_sm = 0;
        if (r == cudaSuccess) r = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess)
          r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster_fwd<TILE, MODE>,
                                                            threads, smem);
        return r == cudaSuccess ? std::max(1, sms * per_sm) : -(int)r;
      },
      &resident);
  if (e != cudaSuccess) return e;
  // one warp per (tile, 8x4 block) unit at most
  const int units = blocks * (TILE * TILE / 32);
  const int grid = std::min((units + TSB_RASTER_WARPS - 1) / TSB_RASTER_WARPS, resident);
  return launch_pdl(k_raster_fwd<TILE, MODE>, grid, threads, smem, st, rp);
}

template <int TILE>
inline cudaError_t launch_raster(int mode, int blocks, cudaStream_t st, const RasterParams& rp) {
  if (mode == TSB_MODE_HW) return launch_raster_mode<TILE, TSB_MODE_HW>(blocks, st, rp);
  if (mode == TSB_MODE_VERIFY) return launch_raster_mode<TILE, TSB_MODE_VERIFY>(blocks, st, rp);
  return launch_raster_mode<TILE, TSB_MODE_FLAT>(blocks, st, rp);
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
    set_error("tsb_frame_workspace_size: invalid arguments (tile 8/16/32, at most 256 tiles "
              "per image axis, max_entries < 2^30)");
    return TSB_ERR_VALUE;
  }
  *bytes = L.total;
  return TSB_OK;
}

int tsb_frame_workspace_max_needed_offset(int32_t P, int32_t W, int32_t H, int32_t tile,
                                          int64_t cap, uint64_t* offset) {
  WsLayout L;
  if (!offset || !ws_layout(P, W, H, tile, cap, &L)) {
    set_error("tsb_frame_workspace_max_needed_offset: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *offset = L.max_needed;
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
  if (scene->num_splats > 0 && mode == TSB_MODE_HW && !atlas->tex) {
    set_error("HW texture mode needs an atlas texture (tsb_atlas_tex_create)");
    return TSB_ERR_VALUE;
  }
  if (scene->num_splats > 0 && mode == TSB_MODE_VERIFY && (!atlas->family_a || !atlas->family_b)) {
    set_error("verify mode needs linear atlas pages");
    return TSB_ERR_VALUE;
  }
  if (scene->num_splats > 0 && mode == TSB_MODE_FLAT && !atlas->flat_attrs) {
    set_error("flat mode needs flat_attrs");
    return TSB_ERR_VALUE;
  }
  if (scene->num_splats > 0 && mode != TSB_MODE_FLAT && !atlas->entries) {
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

// K1's grid: enough CTAs to fill every SM PREP_WAVES times at TSB_PREP_MINB
// CTAs per SM; larger scenes loop (grid-stride).
#ifndef TSB_PREP_WAVES
#define TSB_PREP_WAVES 2
#endif
static int prep_grid_cap() {
  static PerDevice s_cap;
  int cap = 0;
  if (s_cap.get(
          [](int dev) {
            int sms = 0;
            cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            return e == cudaSuccess ? sms * TSB_PREP_MINB * TSB_PREP_WAVES : -(int)e;
          },
          &cap) != cudaSuccess)
    return 148 * TSB_PREP_MINB * TSB_PREP_WAVES;
  return cap;
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
  uint64_t* dk64 = ws_ptr<uint64_t>(ws, L.dkeys_in);
  uint32_t* k32a = ws_ptr<uint32_t>(ws, L.dk32_out);  // K1 writes here; the sorted keys end here
  uint32_t* k32b = ws_ptr<uint32_t>(ws, L.dk32_in);
  uint32_t* idsa = ws_ptr<uint32_t>(ws, L.ids_out);   // the draw order ends here
  uint32_t* idsb = ws_ptr<uint32_t>(ws, L.ids_in);
  uint2* binrec = ws_ptr<uint2>(ws, L.tile_count);
  int32_t* rank = ws_ptr<int32_t>(ws, L.rank);
  int32_t* ranges = ws_ptr<int32_t>(ws, L.ranges);
  int64_t* counters = ws_ptr<int64_t>(ws, L.counters);
  BinCounters* bin = ws_ptr<BinCounters>(ws, L.bin);
  uint32_t* status = ws_ptr<uint32_t>(ws, L.status);

  // counters, binning state and look-back words are one contiguous block
  TSB_CUDA(cudaMemsetAsync(counters, 0, L.status + L.status_words * 4 - L.counters, st));
  TSB_CUDA(cudaMemsetAsync(ranges, 0, (size_t)L.num_tiles * 8, st));
  if (P > 0) {
    PrepParams pp;
    pp.cam = cam;
    pp.P = P; pp.sh_degree = scene->sh_degree; pp.tile = tile; pp.tiles_x = L.tiles_x;
    pp.pos = scene->positions; pp.tu = scene->tangent_u; pp.tv = scene->tangent_v;
    pp.sc = scene->scales; pp.op = scene->opacities; pp.sh = scene->sh;
    pp.entries = mode == TSB_MODE_FLAT ? nullptr : atlas->entries;
    pp.T = atlas->resolution; pp.page_w = atlas->page_w; pp.page_h = atlas->page_h;
    pp.geom = geom; pp.rects = ws_ptr<uint2>(ws, L.rects); pp.mat = ws_ptr<MatRec>(ws, L.mat);
    pp.m64 = ws_ptr<double>(ws, L.m64); pp.dkeys = dk64;
    pp.ids = reinterpret_cast<int32_t*>(idsa);
    pp.dkey32 = k32a;
    pp.near_hi = (uint32_t)(tsb_f64_bits(camera->near_z) >> 32);
    pp.bin_rec = binrec;
    pp.slot = scene->record_slot;
    pp.bin = bin;
    pp.total = counters;
    k_preprocess<<<std::min((P + 255) / 256, prep_grid_cap()), 256, 0, st>>>(pp);
    TSB_CHECK_LAUNCH("k_preprocess");

    // S1: depth order (4 one-sweep passes a -> b -> a -> b -> a)
    uint32_t* st_words = status;
    for (int q = 0; q < kDepthPasses; ++q) {
      OnesweepArgs oa;
      const bool fwd = (q & 1) == 0;
      oa.kin = fwd ? k32a : k32b; oa.vin = fwd ? idsa : idsb;
      oa.kout = fwd ? k32b : k32a; oa.vout = fwd ? idsb : idsa;
      oa.n = P; oa.n_dev = nullptr; oa.cap = 0;
      oa.shift = 8 * q;
      oa.hist = bin->hist_depth[q];
      oa.hist_is_diff = 0;
      oa.tiles_x = 0;
      oa.status = st_words;
      oa.nb = L.nb_depth;
      oa.mode = q == 0 ? kOsFirst : kOsLater;
      oa.kept = &bin->kept;
      oa.ticket = &bin->tickets[q];
      TSB_CUDA(launch_pdl(k_onesweep<kOsItemsDepth>, L.nb_depth, kOsThreads, 0, st, oa));
      TSB_CHECK_LAUNCH("k_onesweep(depth)");
      st_words += pass_status_words(L.nb_depth);
    }
    FixRunsArgs fa;
    fa.P = P; fa.k32 = k32a; fa.k64 = dk64; fa.ids = reinterpret_cast<int32_t*>(idsa);
    fa.rank = rank; fa.n_long = &bin->n_long; fa.long_runs = ws_ptr<int32_t>(ws, L.long_runs);
    TSB_CUDA(launch_pdl(k_fix_runs, (P + 255) / 256, 256, 0, st, fa));
    TSB_CHECK_LAUNCH("k_fix_runs");
    LongRunArgs la;
    la.n_long = &bin->n_long; la.long_runs = fa.long_runs; la.k64 = dk64;
    la.ids = fa.ids; la.scratch = ws_ptr<int32_t>(ws, L.dkeys_out); la.rank = rank;
    TSB_CUDA(launch_pdl(k_sort_long_runs, 16, 128, 0, st, la));
    TSB_CHECK_LAUNCH("k_sort_long_runs");

    // S2: tile lists (duplication fused with the tile-x pass, then tile-y)
    DupArgs da;
    da.sorted_ids = fa.ids; da.bin_rec = binrec;
    da.kept = &bin->kept; da.total = counters; da.cap = cap;
    da.hist_tx = bin->hist_tx;
    da.kout = ws_ptr<uint32_t>(ws, L.ekeys_in); da.vout = ws_ptr<uint32_t>(ws, L.evals_in);
    da.status = st_words;
    da.nb = L.nb_dup;
    da.ticket = &bin->tickets[4];
    TSB_CUDA(launch_pdl(k_dup_tx, L.nb_dup, kOsThreads, 0, st, da));
    TSB_CHECK_LAUNCH("k_dup_tx");
    st_words += pass_status_words(L.nb_dup);
    OnesweepArgs ya;
    ya.kin = da.kout; ya.vin = da.vout;
    ya.kout = ws_ptr<uint32_t>(ws, L.ekeys_out); ya.vout = ws_ptr<uint32_t>(ws, L.evals_out);
    ya.n = 0; ya.n_dev = counters; ya.cap = cap;
    ya.shift = 8;
    ya.hist = bin->hist_ty;
    ya.hist_is_diff = 1;
    ya.tiles_x = L.tiles_x;
    ya.status = st_words;
    ya.nb = L.nb_tiley;
    ya.mode = kOsPlain;
    ya.kept = nullptr;
    ya.ticket = &bin->tickets[5];
    TSB_CUDA(launch_pdl(k_onesweep<kOsItems>, L.nb_tiley, kOsThreads, 0, st, ya));
    TSB_CHECK_LAUNCH("k_onesweep(tile_y)");
    const int64_t C = std::max<int64_t>(cap, 1);
    TSB_CUDA(launch_pdl(k_ranges, (unsigned)std::min<int64_t>((C + 255) / 256, 148 * 16), 256,
                        0, st, (int64_t)cap, (const uint32_t*)ya.kout, (const int64_t*)counters,
                        ranges, ws_ptr<int64_t>(ws, L.max_needed)));
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
  rp.tstride = atlas->texel_stride > 0 ? atlas->texel_stride : 1;
  rp.t6 = (float)atlas->resolution / 6.0f;
  rp.t2 = 0.5f * (float)atlas->resolution;
  rp.tmh = (float)atlas->resolution - 0.5f;
  rp.fam_a = reinterpret_cast<const float4*>(atlas->family_a);
  rp.fam_b = reinterpret_cast<const float4*>(atlas->family_b);
  rp.flat = atlas->flat_attrs;
  rp.tex_a = atlas->tex ? reinterpret_cast<AtlasTex*>(atlas->tex)->tex_a : 0;
  rp.tex_b = atlas->tex ? reinterpret_cast<AtlasTex*>(atlas->tex)->tex_b : 0;
  rp.gbuf = gbuf; rp.n_contrib = px->n_contrib; rp.last_entry = px->last_entry;
  rp.final_T = px->final_T; rp.T_last = px->T_last;
  rp.touched = px->splat_touched;
  rp.num_tiles = L.num_tiles;
  rp.work_counter = reinterpret_cast<int32_t*>(ws_ptr<int64_t>(ws, L.counters) + 1);
  rp.tile_order = nullptr;
  TSB_CUDA(launch_pdl(k_tile_schedule, 1, kSchedThreads, 0, st, (int32_t)L.num_tiles,
                      (const int32_t*)rp.ranges, ws_ptr<int32_t>(ws, L.torder_out),
                      rp.work_counter));
  TSB_CHECK_LAUNCH("k_tile_schedule");
  rp.tile_order = ws_ptr<int32_t>(ws, L.torder_out);
  cudaError_t e;
  if (tile == 8) e = launch_raster<8>(mode, L.num_tiles, st, rp);
  else if (tile == 16) e = launch_raster<16>(mode, L.num_tiles, st, rp);
  else e = launch_raster<32>(mode, L.num_tiles, st, rp);
  if (e != cudaSuccess) return cuda_fail("k_raster_fwd", e);
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
        ws_ptr<GeomRec>(ws, L.geom), ws_ptr<int32_t>(ws, L.rank), ws_ptr<int64_t>(ws, L.counters),
        keys);
    TSB_CHECK_LAUNCH("k_export_keys");
  }
  if (rects && P > 0) {
    k_export_rects<<<(P + 255) / 256, 256, 0, st>>>(P, ws_ptr<uint2>(ws, L.rects), rects);
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
  sp.view = view_coeffs(camera);
  sp.gbuf = gbuf; sp.color = color; sp.diffuse = diffuse; sp.specular = specular;
  const int n = camera->width * camera->height;
  TSB_CUDA(launch_pdl(k_shade, (n + 255) / 256, 256, 0, (cudaStream_t)stream, sp));
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

#ifdef TSB_STATS
int tsb_debug_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, tsb::g_tsb_stats, sizeof(unsigned long long) * 16);
  if (reset) {
    static const unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(tsb::g_tsb_stats, z, sizeof(z));
  }
  return 0;
}
#endif

int tsb_red_probe(float* buf, int32_t log2_floats, int32_t iters, int32_t blocks, int32_t threads,
                  void* stream) {
  if (!buf || log2_floats < 1 || log2_floats > 30 || iters <= 0 || blocks <= 0 || threads <= 0) {
    set_error("tsb_red_probe: invalid arguments");
    return TSB_ERR_VALUE;
  }
  k_red_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(buf, (1u << log2_floats) - 1u, iters);
  TSB_CHECK_LAUNCH("k_red_probe");
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

// ---------------------------------------------------------------------------
// Frame graph: K1-K6 of one view captured once as a CUDA graph; per view only
// the camera-dependent kernel parameters (K1, K5, K6) are rewritten and the
// graph is replayed — one host call instead of ~20 launches.
// ---------------------------------------------------------------------------
namespace tsb {
namespace {

template <int TILE>
const void* raster_fn_tile(int mode) {
  if (mode == TSB_MODE_HW) return reinterpret_cast<const void*>(k_raster_fwd<TILE, TSB_MODE_HW>);
  if (mode == TSB_MODE_VERIFY)
    return reinterpret_cast<const void*>(k_raster_fwd<TILE, TSB_MODE_VERIFY>);
  return reinterpret_cast<const void*>(k_raster_fwd<TILE, TSB_MODE_FLAT>);
}

const void* raster_fn(int tile, int mode) {
  if (tile == 8) return raster_fn_tile<8>(mode);
  if (tile == 16) return raster_fn_tile<16>(mode);
  return raster_fn_tile<32>(mode);
}

}  // namespace
}  // namespace tsb

struct tsb_frame_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t width = 0, height = 0;
  cudaGraphNode_t n_prep = nullptr, n_raster = nullptr, n_shade = nullptr;
  tsb::PrepParams prep;
  tsb::RasterParams raster;
  tsb::ShadeParams shade;
  cudaKernelNodeParams kp_prep, kp_raster, kp_shade;
};

extern "C" {

int tsb_frame_graph_destroy(tsb_frame_graph_t g) {
  if (!g) return TSB_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return TSB_OK;
}

int tsb_frame_graph_create(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                           int32_t mode, int32_t tile, void* ws, uint64_t ws_bytes, int64_t cap,
                           float* gbuf, const tsb_pixel_state* px, int64_t* entries_needed,
                           const tsb_environment* env, const float* background, float* color,
                           float* diffuse, float* specular, tsb_frame_graph_t* out) {
  return tsb_frame_graph_create_ev(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, gbuf, px,
                                   entries_needed, env, background, color, diffuse, specular,
                                   nullptr, out);
}

int tsb_frame_graph_create_ev(const tsb_scene* scene, const tsb_camera* camera,
                              const tsb_atlas* atlas, int32_t mode, int32_t tile, void* ws,
                              uint64_t ws_bytes, int64_t cap, float* gbuf,
                              const tsb_pixel_state* px, int64_t* entries_needed,
                              const tsb_environment* env, const float* background, float* color,
                              float* diffuse, float* specular, void* binned_event,
                              tsb_frame_graph_t* out) {
  if (!out || !camera) {
    set_error("tsb_frame_graph_create: null argument");
    return TSB_ERR_VALUE;
  }
  *out = nullptr;
  if (env && !color) {
    set_error("tsb_frame_graph_create: shading needs a colour buffer");
    return TSB_ERR_VALUE;
  }
  // one uncaptured frame first: validates the arguments and performs the
  // one-time attribute / occupancy queries outside the capture
  int rc = tsb_render_forward(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, gbuf, px,
                              entries_needed, nullptr);
  if (rc != TSB_OK) return rc;
  if (env) {
    rc = tsb_shade_forward(gbuf, camera, env, background, color, diffuse, specular, nullptr);
    if (rc != TSB_OK) return rc;
  }
  TSB_CUDA(cudaDeviceSynchronize());
  tsb_frame_graph* g = new tsb_frame_graph();
  g->width = camera->width;
  g->height = camera->height;
  cudaStream_t s;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete g; return cuda_fail("cudaStreamCreate", e); }
  e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    rc = tsb_render_binning(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, entries_needed,
                            s);
    if (rc == TSB_OK && binned_event) {  // an event-record node between binning and raster
      // (external: a real event-record node, not a capture-internal fork marker)
      const cudaError_t er =
          cudaEventRecordWithFlags((cudaEvent_t)binned_event, s, cudaEventRecordExternal);
      if (er != cudaSuccess) rc = cuda_fail("cudaEventRecord", er);
    }
    if (rc == TSB_OK)
      rc = tsb_render_composite(scene, camera, atlas, mode, tile, ws, ws_bytes, cap, gbuf, px, s);
    if (rc == TSB_OK && env)
      rc = tsb_shade_forward(gbuf, camera, env, background, color, diffuse, specular, s);
    cudaGraph_t graph = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(s, &graph);
    g->graph = graph;
    if (rc == TSB_OK && e2 != cudaSuccess) rc = cuda_fail("cudaStreamEndCapture", e2);
  } else {
    rc = cuda_fail("cudaStreamBeginCapture", e);
  }
  cudaStreamDestroy(s);
  if (rc != TSB_OK) { tsb_frame_graph_destroy(g); return rc; }
  // locate the camera-dependent kernel nodes
  size_t n = 0;
  TSB_CUDA(cudaGraphGetNodes(g->graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  TSB_CUDA(cudaGraphGetNodes(g->graph, nodes.data(), &n));
  const void* f_raster = raster_fn(tile, mode);
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    TSB_CUDA(cudaGraphNodeGetType(nd, &t));
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp;
    TSB_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
    if (kp.func == reinterpret_cast<void*>(k_preprocess)) {
      g->n_prep = nd; g->kp_prep = kp;
      g->prep = *static_cast<PrepParams*>(kp.kernelParams[0]);
    } else if (kp.func == f_raster) {
      g->n_raster = nd; g->kp_raster = kp;
      g->raster = *static_cast<RasterParams*>(kp.kernelParams[0]);
    } else if (kp.func == reinterpret_cast<void*>(k_shade)) {
      g->n_shade = nd; g->kp_shade = kp;
      g->shade = *static_cast<ShadeParams*>(kp.kernelParams[0]);
    }
  }
  const bool has_splats = scene && scene->num_splats > 0;
  if ((has_splats && !g->n_prep) || !g->n_raster || (env && !g->n_shade)) {
    tsb_frame_graph_destroy(g);
    set_error("tsb_frame_graph_create: kernel nodes not found in the capture");
    return TSB_ERR_CUDA;
  }
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) { tsb_frame_graph_destroy(g); return cuda_fail("cudaGraphInstantiate", e); }
  *out = g;
  return TSB_OK;
}

int tsb_frame_graph_launch(tsb_frame_graph_t g, const tsb_camera* camera, float* color,
                           void* stream) {
  if (!g || !camera) {
    set_error("tsb_frame_graph_launch: null argument");
    return TSB_ERR_VALUE;
  }
  if (camera->width != g->width || camera->height != g->height) {
    set_error("tsb_frame_graph_launch: camera size differs from the captured frame");
    return TSB_ERR_VALUE;
  }
  if (!(camera->near_z > 0.0) || !(camera->fx > 0.0) || !(camera->fy > 0.0)) {
    set_error("tsb_frame_graph_launch: invalid camera");
    return TSB_ERR_VALUE;
  }
  const tsb_cam_params cam = to_cam(camera);
  if (g->n_prep) {
    g->prep.cam = cam;
    g->prep.near_hi = (uint32_t)(tsb_f64_bits(camera->near_z) >> 32);
    void* args[] = {&g->prep};
    cudaKernelNodeParams kp = g->kp_prep;
    kp.kernelParams = args;
    kp.extra = nullptr;
    TSB_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->n_prep, &kp));
  }
  {
    g->raster.cam = cam;
    g->raster.near_f = (float)camera->near_z;
    void* args[] = {&g->raster};
    cudaKernelNodeParams kp = g->kp_raster;
    kp.kernelParams = args;
    kp.extra = nullptr;
    TSB_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->n_raster, &kp));
  }
  if (g->n_shade) {
    g->shade.cam = cam;
    g->shade.view = view_coeffs(camera);
    if (color) g->shade.color = color;
    void* args[] = {&g->shade};
    cudaKernelNodeParams kp = g->kp_shade;
    kp.kernelParams = args;
    kp.extra = nullptr;
    TSB_CUDA(cudaGraphExecKernelNodeSetParams(g->exec, g->n_shade, &kp));
  }
  TSB_CUDA(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
  return TSB_OK;
}

}  // extern "C"
