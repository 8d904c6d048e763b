/*
 * tsb_oracle.c — CPU oracle for the textured-2DGS render path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the CPU baseline — never as the product path.
 *
 * A plain-C restatement of the reference renderer's forward path
 * (/root/reference/pkg/src/texsplat, numpy):
 *   prepare / _cull_rects      rasterize.py:137-243
 *   draw order                 rasterize.py:178-182 (lexsort by (z, id))
 *   _tile_lists                rasterize.py:246-258
 *   _render_tile/_fetch_attrs  rasterize.py:261-385
 *   render_forward             rasterize.py:395-438
 *   shade_gbuffer              shading.py:126-183
 * It compiles the SAME decision math as the sm_100a kernels
 * (paper_2506_13348_b200/csrc/tsb_math.h) with -ffp-contract=off, so sort
 * keys, tile ranges, per-pixel contributor counts, transmittance and the
 * fp32 verify-mode G-buffer are bit-identical with the GPU. It is pinned to
 * the numpy reference by the golden fixtures in tests/golden (tolerance:
 * the reference computes in fp64).
 *
 * Threads: OpenMP over tiles (the reference's ThreadPoolExecutor over tiles,
 * rasterize.py:417-433); results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../paper_2506_13348_b200/csrc/tsb_math.h"

#define TSB_MODE_VERIFY_ORACLE 1
#define TSB_MODE_FLAT_ORACLE 2

typedef struct oracle_frame {
  int32_t P, W, H, tile, tiles_x, tiles_y, num_tiles;
  int32_t num_kept;
  int64_t num_entries;
  tsb_cam_params cam;
  /* per splat (by id) */
  float* lin;          /* P x TSB_LIN_WORDS linear intersection forms */
  double* m64;         /* P x 10 (M + opacity) */
  int32_t* rects;      /* P x 4 */
  float* frame;        /* P x 9 */
  float* l_ind;        /* P x 3 */
  double* view_z;      /* P */
  int32_t* keep;       /* P */
  int32_t* rank;       /* P */
  int32_t* boxes;      /* P x 4 test boxes (rect ∩ alpha-cut ellipse box) */
  /* draw order and tile lists */
  int32_t* sorted_ids; /* P: kept in (z, id) order, then culled in id order */
  /* two binnings: [0] by the reference rect (_tile_lists), [1] by the
   * test box (the GPU's binning); same draw order within each tile */
  int64_t n_ent[2];
  int32_t* ranges_b[2];   /* num_tiles x 2 */
  int32_t* entry_ids_b[2];
  int64_t* keys_b[2];     /* (tile << 32) | rank */
  int binning;            /* which one raster/export use (default 1) */
  int32_t* ranges;
  int32_t* entry_ids;
  int64_t* keys;
} oracle_frame;

static const double* g_sort_z;
static int cmp_z_id(const void* a, const void* b) {
  int32_t ia = *(const int32_t*)a, ib = *(const int32_t*)b;
  double za = g_sort_z[ia], zb = g_sort_z[ib];
  if (za < zb) return -1;
  if (za > zb) return 1;
  return (ia > ib) - (ia < ib);
}

void oracle_frame_free(oracle_frame* f) {
  if (!f) return;
  free(f->lin); free(f->m64); free(f->rects); free(f->frame);
  free(f->l_ind); free(f->view_z); free(f->keep); free(f->rank); free(f->sorted_ids);
  for (int b = 0; b < 2; ++b) { free(f->ranges_b[b]); free(f->entry_ids_b[b]); free(f->keys_b[b]); }
  free(f->boxes);
  free(f);
}

/* Select the tile lists raster/export use: 0 = reference rect binning
 * (rasterize.py:246-258), 1 = test-box binning (the GPU's). */
void oracle_frame_set_binning(oracle_frame* f, int32_t which) {
  f->binning = which ? 1 : 0;
  f->num_entries = f->n_ent[f->binning];
  f->ranges = f->ranges_b[f->binning];
  f->entry_ids = f->entry_ids_b[f->binning];
  f->keys = f->keys_b[f->binning];
}

/* prepare + sort + binning. cam: tsb_cam_params layout (== tsb_camera). */
oracle_frame* oracle_frame_new(int32_t P, int32_t sh_degree, const double* positions,
                               const double* tangent_u, const double* tangent_v,
                               const double* scales, const double* opacities,
                               const double* sh, const tsb_cam_params* cam, int32_t tile,
                               int32_t nthreads) {
  oracle_frame* f = (oracle_frame*)calloc(1, sizeof(oracle_frame));
  if (!f || tile <= 0) { free(f); return NULL; }
  f->P = P; f->W = cam->width; f->H = cam->height; f->tile = tile; f->cam = *cam;
  f->tiles_x = (f->W + tile - 1) / tile;
  f->tiles_y = (f->H + tile - 1) / tile;
  f->num_tiles = f->tiles_x * f->tiles_y;
  size_t Pn = P > 0 ? (size_t)P : 1;
  f->lin = (float*)malloc(Pn * TSB_LIN_WORDS * sizeof(float));
  f->m64 = (double*)malloc(Pn * 10 * sizeof(double));
  f->rects = (int32_t*)malloc(Pn * 4 * sizeof(int32_t));
  f->frame = (float*)malloc(Pn * 9 * sizeof(float));
  f->l_ind = (float*)malloc(Pn * 3 * sizeof(float));
  f->view_z = (double*)malloc(Pn * sizeof(double));
  f->keep = (int32_t*)malloc(Pn * sizeof(int32_t));
  f->rank = (int32_t*)malloc(Pn * sizeof(int32_t));
  f->sorted_ids = (int32_t*)malloc(Pn * sizeof(int32_t));
  const int K = (sh_degree + 1) * (sh_degree + 1);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
  for (int32_t id = 0; id < P; ++id) {
    tsb_prep r;
    tsb_preprocess_splat(cam, positions + 3 * (size_t)id, tangent_u + 3 * (size_t)id,
                         tangent_v + 3 * (size_t)id, scales + 2 * (size_t)id,
                         sh + (size_t)3 * K * id, sh_degree, &r);
    tsb_make_lin(r.m, opacities[id], f->lin + TSB_LIN_WORDS * (size_t)id);
    for (int k = 0; k < 9; ++k) {
      f->m64[10 * (size_t)id + k] = r.m[k];
      f->frame[9 * (size_t)id + k] = (float)r.frame[k];
    }
    f->m64[10 * (size_t)id + 9] = opacities[id];
    for (int k = 0; k < 3; ++k) f->l_ind[3 * (size_t)id + k] = (float)r.l_ind[k];
    f->rects[4 * (size_t)id] = r.x0; f->rects[4 * (size_t)id + 1] = r.x1;
    f->rects[4 * (size_t)id + 2] = r.y0; f->rects[4 * (size_t)id + 3] = r.y1;
    f->view_z[id] = r.view_z;
    f->keep[id] = r.keep;
  }
  /* draw order: kept ids sorted by (z, id), then culled ids ascending */
  int32_t nk = 0;
  for (int32_t id = 0; id < P; ++id) if (f->keep[id]) f->sorted_ids[nk++] = id;
  f->num_kept = nk;
  g_sort_z = f->view_z;
  qsort(f->sorted_ids, (size_t)nk, sizeof(int32_t), cmp_z_id);
  int32_t c = nk;
  for (int32_t id = 0; id < P; ++id) if (!f->keep[id]) f->sorted_ids[c++] = id;
  for (int32_t r = 0; r < P; ++r) f->rank[f->sorted_ids[r]] = r;

  /* boxes for the tighter binning (shared tsb_test_box) */
  f->boxes = (int32_t*)malloc(Pn * 4 * sizeof(int32_t));
  for (int32_t id = 0; id < P; ++id) {
    const int32_t* rc = f->rects + 4 * (size_t)id;
    tsb_test_box(cam, f->m64 + 10 * (size_t)id, f->lin[TSB_LIN_WORDS * (size_t)id + 11], rc[0],
                 rc[1], rc[2], rc[3], f->boxes + 4 * (size_t)id);
  }
  for (int bsel = 0; bsel < 2; ++bsel) {
    const int32_t* bx = bsel == 0 ? f->rects : f->boxes;
    /* stable counting sort of (tile, rank) entries == _tile_lists */
    int64_t* count = (int64_t*)calloc((size_t)f->num_tiles + 1, sizeof(int64_t));
    int64_t total = 0;
    for (int32_t r = 0; r < nk; ++r) {
      const int32_t* rc = bx + 4 * (size_t)f->sorted_ids[r];
      if (!(rc[1] > rc[0] && rc[3] > rc[2])) continue;
      for (int ty = rc[2] / tile; ty <= (rc[3] - 1) / tile; ++ty)
        for (int tx = rc[0] / tile; tx <= (rc[1] - 1) / tile; ++tx) {
          count[ty * f->tiles_x + tx]++;
          total++;
        }
    }
    f->n_ent[bsel] = total;
    f->ranges_b[bsel] = (int32_t*)calloc((size_t)f->num_tiles * 2, sizeof(int32_t));
    int32_t* rg = f->ranges_b[bsel];
    int64_t* pos = (int64_t*)malloc(((size_t)f->num_tiles + 1) * sizeof(int64_t));
    int64_t acc = 0;
    for (int t = 0; t < f->num_tiles; ++t) {
      pos[t] = acc;
      rg[2 * t] = (int32_t)acc;
      acc += count[t];
      rg[2 * t + 1] = (int32_t)acc;
      if (count[t] == 0) { rg[2 * t] = 0; rg[2 * t + 1] = 0; }
    }
    size_t Tn = total > 0 ? (size_t)total : 1;
    f->entry_ids_b[bsel] = (int32_t*)malloc(Tn * sizeof(int32_t));
    f->keys_b[bsel] = (int64_t*)malloc(Tn * sizeof(int64_t));
    for (int32_t r = 0; r < nk; ++r) {
      const int32_t id = f->sorted_ids[r];
      const int32_t* rc = bx + 4 * (size_t)id;
      if (!(rc[1] > rc[0] && rc[3] > rc[2])) continue;
      for (int ty = rc[2] / tile; ty <= (rc[3] - 1) / tile; ++ty)
        for (int tx = rc[0] / tile; tx <= (rc[1] - 1) / tile; ++tx) {
          int t = ty * f->tiles_x + tx;
          int64_t o = pos[t]++;
          f->entry_ids_b[bsel][o] = id;
          f->keys_b[bsel][o] = ((int64_t)t << 32) | (int64_t)(uint32_t)r;
        }
    }
    free(count);
    free(pos);
  }
  oracle_frame_set_binning(f, 1);
  return f;
}

int64_t oracle_frame_num_entries(const oracle_frame* f) { return f->num_entries; }
int32_t oracle_frame_num_kept(const oracle_frame* f) { return f->num_kept; }
int32_t oracle_frame_num_tiles(const oracle_frame* f) { return f->num_tiles; }

void oracle_frame_export(const oracle_frame* f, int32_t* sorted_ids, int64_t* keys,
                         int32_t* ranges, int32_t* rects, double* view_z) {
  if (sorted_ids) memcpy(sorted_ids, f->sorted_ids, (size_t)f->P * sizeof(int32_t));
  if (keys) memcpy(keys, f->keys, (size_t)f->num_entries * sizeof(int64_t));
  if (ranges) memcpy(ranges, f->ranges, (size_t)f->num_tiles * 2 * sizeof(int32_t));
  if (rects) memcpy(rects, f->rects, (size_t)f->P * 4 * sizeof(int32_t));
  if (view_z) memcpy(view_z, f->view_z, (size_t)f->P * sizeof(double));
}

/* Per-tile compositor. mode: 1 = fp32 verify bilinear, 2 = flat.
 * fam_a/fam_b: pages x page_h x page_w x 4 float32; entries: P x 3.
 * flat: P x 5. Outputs: gbuf planar 13 x H x W, per-pixel state. */
void oracle_frame_raster(const oracle_frame* f, int32_t mode, int32_t T, int32_t page_w,
                         int32_t page_h, const int32_t* entries, const float* fam_a,
                         const float* fam_b, const float* flat, int32_t nthreads, float* gbuf,
                         int32_t* n_contrib, int32_t* last_entry, float* final_T,
                         float* T_last) {
  const int W = f->W, H = f->H, tile = f->tile;
  const size_t HW = (size_t)W * H;
  const float near_f = (float)f->cam.near_z;
  const float teps = (float)TSB_TRANSMIT_EPS;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    const int npx = tile * tile;
    float* acc = (float*)malloc((size_t)npx * 13 * sizeof(float));
    float* Tp = (float*)malloc((size_t)npx * sizeof(float));
    float* Tl = (float*)malloc((size_t)npx * sizeof(float));
    int32_t* nc = (int32_t*)malloc((size_t)npx * sizeof(int32_t));
    int32_t* le = (int32_t*)malloc((size_t)npx * sizeof(int32_t));
    unsigned char* done = (unsigned char*)malloc((size_t)npx);
#pragma omp for schedule(dynamic, 1)
    for (int t = 0; t < f->num_tiles; ++t) {
      const int tx0 = (t % f->tiles_x) * tile, ty0 = (t / f->tiles_x) * tile;
      const int tx1 = tx0 + tile < W ? tx0 + tile : W;
      const int ty1 = ty0 + tile < H ? ty0 + tile : H;
      const int tw = tx1 - tx0;
      int live_px = (tx1 - tx0) * (ty1 - ty0);
      for (int k = 0; k < npx; ++k) {
        Tp[k] = 1.0f; Tl[k] = 1.0f; nc[k] = 0; le[k] = -1; done[k] = 0;
      }
      memset(acc, 0, (size_t)npx * 13 * sizeof(float));
      const int32_t start = f->ranges[2 * t], end = f->ranges[2 * t + 1];
      for (int32_t e = start; e < end && live_px > 0; ++e) {
        const int32_t id = f->entry_ids[e];
        const int32_t* rc = f->rects + 4 * (size_t)id;
        const int rx0 = rc[0] > tx0 ? rc[0] : tx0, rx1 = rc[1] < tx1 ? rc[1] : tx1;
        const int ry0 = rc[2] > ty0 ? rc[2] : ty0, ry1 = rc[3] < ty1 ? rc[3] : ty1;
        if (rx0 >= rx1 || ry0 >= ry1) continue;
        const float* lin = f->lin + TSB_LIN_WORDS * (size_t)id;
        const float* fr = f->frame + 9 * (size_t)id;
        for (int py = ry0; py < ry1; ++py) {
          const double yd = tsb_pixel_y(&f->cam, py);
          const float y = (float)yd;
          for (int px = rx0; px < rx1; ++px) {
            const int k = (py - ty0) * tw + (px - tx0);
            if (done[k]) continue;
            const double xd = tsb_pixel_x(&f->cam, px);
            const float x = (float)xd;
            float u, v, z, a;
            int r = tsb_eval_lin(lin, x, y, near_f, &u, &v, &z, &a);
            if (r == 0) continue;
            if (r == 2) {
              const double* m64 = f->m64 + 10 * (size_t)id;
              if (!tsb_live_f64(m64, m64[9], xd, yd, f->cam.near_z)) continue;
            }
            float xa[12];
            if (mode == TSB_MODE_FLAT_ORACLE) {
              const float* fl = flat + 5 * (size_t)id;
              xa[0] = fl[0]; xa[1] = fl[1]; xa[2] = fl[2]; xa[3] = fl[3]; xa[4] = fl[4];
              xa[5] = fr[6]; xa[6] = fr[7]; xa[7] = fr[8];
            } else {
              tsb_texc tc;
              tsb_texel_coords(u, v, T, &tc);
              const int32_t* en = entries + 3 * (size_t)id;
              const int64_t base = (int64_t)en[2] * page_h * page_w +
                                   (int64_t)en[1] * T * page_w + (int64_t)en[0] * T;
              const int64_t r0 = base + (int64_t)tc.j0 * page_w, r1 = base + (int64_t)tc.j1 * page_w;
              const float* a00 = fam_a + 4 * (r0 + tc.i0);
              const float* a01 = fam_a + 4 * (r0 + tc.i1);
              const float* a10 = fam_a + 4 * (r1 + tc.i0);
              const float* a11 = fam_a + 4 * (r1 + tc.i1);
              const float* b00 = fam_b + 4 * (r0 + tc.i0);
              const float* b01 = fam_b + 4 * (r0 + tc.i1);
              const float* b10 = fam_b + 4 * (r1 + tc.i0);
              const float* b11 = fam_b + 4 * (r1 + tc.i1);
              float A[4], B[3];
              for (int ch = 0; ch < 4; ++ch)
                A[ch] = tsb_lerp4(a00[ch], a01[ch], a10[ch], a11[ch], tc.fs, tc.ft);
              for (int ch = 0; ch < 3; ++ch)
                B[ch] = tsb_lerp4(b00[ch], b01[ch], b10[ch], b11[ch], tc.fs, tc.ft);
              xa[0] = A[0]; xa[1] = A[1]; xa[2] = A[2];
              xa[3] = B[2];
              xa[4] = A[3];
              tsb_decode_normal(B[0], B[1], fr, xa + 5);
            }
            const float* li = f->l_ind + 3 * (size_t)id;
            xa[8] = li[0]; xa[9] = li[1]; xa[10] = li[2];
            xa[11] = z;
            Tl[k] = Tp[k];
            Tp[k] = tsb_composite(acc + 13 * (size_t)k, xa, a, Tp[k]);
            nc[k]++;
            le[k] = e;
            if (!(Tp[k] > teps)) { done[k] = 1; live_px--; }
          }
        }
      }
      for (int py = ty0; py < ty1; ++py)
        for (int px = tx0; px < tx1; ++px) {
          const int k = (py - ty0) * tw + (px - tx0);
          const size_t pix = (size_t)py * W + px;
          for (int ch = 0; ch < 13; ++ch) gbuf[ch * HW + pix] = acc[13 * (size_t)k + ch];
          n_contrib[pix] = nc[k];
          last_entry[pix] = le[k];
          final_T[pix] = Tp[k];
          T_last[pix] = Tl[k];
        }
    }
    free(acc); free(Tp); free(Tl); free(nc); free(le); free(done);
  }
}

/* shade_gbuffer (mesh=None). mips: concatenated level grids; mip_hw: 2*levels ints. */
void oracle_shade(const float* gbuf, const tsb_cam_params* cam, int32_t levels,
                  const float* mips, const int32_t* mip_hw, const float* diffuse,
                  int32_t diff_h, int32_t diff_w, const float* lut, int32_t lut_res,
                  const float* bg, int32_t nthreads, float* color, float* dif, float* spe) {
  tsb_env_params env;
  memset(&env, 0, sizeof(env));
  env.levels = levels;
  size_t off = 0;
  for (int l = 0; l < levels && l < TSB_MAX_LEVELS; ++l) {
    env.mips[l].data = mips + off;
    env.mips[l].h = mip_hw[2 * l];
    env.mips[l].w = mip_hw[2 * l + 1];
    off += (size_t)mip_hw[2 * l] * mip_hw[2 * l + 1] * 3;
  }
  env.diffuse.data = diffuse; env.diffuse.h = diff_h; env.diffuse.w = diff_w;
  env.lut = lut; env.lut_res = lut_res;
  const int W = cam->width, H = cam->height;
  const size_t HW = (size_t)W * H;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
  for (int py = 0; py < H; ++py) {
    for (int px = 0; px < W; ++px) {
      const size_t pix = (size_t)py * W + px;
      float g[13];
      for (int c = 0; c < 13; ++c) g[c] = gbuf[c * HW + pix];
      float wo[3];
      tsb_view_dir(cam, tsb_pixel_x(cam, px), tsb_pixel_y(cam, py), wo);
      tsb_shade_pixel(g, wo, &env, bg, color + 3 * pix, dif + 3 * pix, spe + 3 * pix);
    }
  }
}

/* Entries under both binnings (diagnostics). */
void oracle_frame_entry_stats(const oracle_frame* f, int64_t* by_rect, int64_t* by_box) {
  *by_rect = f->n_ent[0];
  *by_box = f->n_ent[1];
}
