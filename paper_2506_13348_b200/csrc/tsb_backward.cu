// tsb_backward.cu — training backward pass for sm_100a.
//
//   K7 k_shade_bwd     per pixel: adjoint of the split-sum shading
//                      (shading.py:186-228, _shade_core_backward :72-109,
//                      environment.py:94-129 / 302-331 / 449-464); env grid
//                      gradients scattered with atomics.
//   K8 k_raster_bwd    per 8x4 pixel block (one warp): walks the tile list
//                      back to front from the block's last contributor,
//                      re-deciding fragments with the forward's exact math,
//                      and accumulates the reference's adjoint
//                      (rasterize.py:472-593): opacity, intersection (dM),
//                      SH radiance, frame and texel gradients. Per-splat
//                      terms are warp-reduced before one atomic per value.
//   K9 k_finish_grads  per splat, fp64: dM -> dH = W^T fold(dM) -> position /
//                      scale / tangent gradients, frame and SH chains
//                      (_finish_param_grads rasterize.py:642-676, sh.py:118-135).
//
// Back-to-front walk without a tape: the forward leaves, per pixel, the
// entry index of the last contributor and the transmittance T_last in front
// of it. Walking backward, T_i = T_{i+1} / (1 - alpha_i) is safe because
// every contributor except the last has T_{i+1} > 1e-4 >= (1-alpha_i)*0...
// i.e. 1 - alpha_i > 1e-4 (the T gate is tested before compositing), and
// the colour behind fragment i is carried by R <- alpha x + (1 - alpha) R,
// so alpha = 1 (allowed by the reference) never divides by zero:
//   dL/dalpha_i = T_i * sum_c g_c (x_ic - R_c)  ==  the reference's
//   sum_c g_c (T_i x_ic - S_ic / max(1 - alpha_i, 1e-30)).

#include <cuda_runtime.h>

#include <algorithm>

#include "tsb_internal.cuh"

namespace tsb {

constexpr int kAccWords = 24;  // per-splat accumulator stride (22 used)
// Deterministic backward: fixed-point scales of the int64 accumulators.
// Per-splat terms: resolution 2^-32 (2.3e-10), range +-2^31; texel
// gradients: resolution 2^-40 (9.1e-13), range +-2^23. Each contribution is
// rounded to the grid once; the sums are then exact, so bitwise repeatable.
constexpr int kAccFix = 32, kTexFix = 40;

// Diagnostics (tsb_debug_red_count): with a counter in the launch parameters,
// K8 counts the global atomic adds it issues (one warp-aggregated add per
// warp and site), for the training roofline's achieved RED rate.
__device__ unsigned long long g_red_count = 0ull;
static bool g_count_red_host = false;

__device__ __forceinline__ void count_red(unsigned long long* ctr, bool issued) {
  if (ctr) {
    const uint32_t b = __ballot_sync(__activemask(), issued);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && b)
      atomicAdd(ctr, (unsigned long long)__popc(b));
  }
}

__device__ __forceinline__ unsigned long long to_fix(float v, int shift) {
  return (unsigned long long)__double2ll_rn((double)v * (double)(1ull << shift));
}
// accumulator layout: [0..9) dWH rows 0..2 x cols (0,1,3); [9] dopacity;
// [10..13) dl_ind; [13..16) dframe_u; [16..19) dframe_v; [19..22) dn3.

// Reduce 32 per-lane values across the warp with a transpose butterfly:
// at each level a lane keeps one half of its vector and sends the other half
// to its partner, so after 31 shuffles lane l holds the warp total of v[l].
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// K7 shade backward
// ---------------------------------------------------------------------------
struct ShadeBwdParams {
  tsb_cam_params cam;
  ViewCoeffs view;
  tsb_env_params env;
  float bg[3];
  const float* gbuf;
  const float* dcolor;  // H x W x 3
  float* dgbuf;         // 13 x H x W
  float* gmips[TSB_MAX_LEVELS];  // shard 0 base of each level (shards contiguous)
  float* gdiffuse;
  int32_t shard_stride;          // floats between shards (0: no sharding)
};

constexpr int kEnvShards = 32;

// Bilinear equirect lookup with its taps (environment.py:57-91).
struct EqTaps {
  int i00, i01, i10, i11;  // flat texel indices
  float fr, fc;
  bool interior;
};

__device__ __forceinline__ EqTaps eq_taps(const tsb_grid& g, float dx, float dy, float dz) {
  const float PI_F = 3.14159265358979323846f, TWO_PI_F = 6.28318530717958647692f;
  const float zc = dz < -1.0f ? -1.0f : (dz > 1.0f ? 1.0f : dz);
  const float theta = acosf(zc);
  float phi = atan2f(dy, dx);
  if (phi < 0.0f) phi += TWO_PI_F;
  if (phi >= TWO_PI_F) phi -= TWO_PI_F;
  const int h = g.h, w = g.w;
  const float row = theta / PI_F * (float)h - 0.5f;
  const float col = phi / TWO_PI_F * (float)w - 0.5f;
  const float rowc = row < 0.0f ? 0.0f : (row > (float)(h - 1) ? (float)(h - 1) : row);
  const float r0f = floorf(rowc);
  const int r0 = (int)r0f;
  const int r1 = r0 + 1 < h - 1 ? r0 + 1 : h - 1;
  const float colf = floorf(col);
  int c0 = (int)colf;
  if (c0 < 0) c0 += w;
  if (c0 >= w) c0 -= w;
  const int c1 = c0 + 1 == w ? 0 : c0 + 1;
  EqTaps t;
  t.i00 = r0 * w + c0; t.i01 = r0 * w + c1; t.i10 = r1 * w + c0; t.i11 = r1 * w + c1;
  t.fr = rowc - r0f; t.fc = col - colf;
  t.interior = row > 0.0f && row < (float)(h - 1);
  return t;
}

// Adjoint of sample_equirect (environment.py:94-129): scatter `up` into the
// grid gradient and return d/d(direction). `rgba`: the gradient grid has 4
// floats per texel (the sharded scratch) and each tap is one 16-byte vector
// atomic instead of three scalar ones.
__device__ void eq_grad(const tsb_grid& g, float* ggrid, bool rgba, float dx, float dy,
                        float dz, const float* up, float* ddir) {
  const EqTaps t = eq_taps(g, dx, dy, dz);
  const float w00 = (1.0f - t.fc) * (1.0f - t.fr), w01 = t.fc * (1.0f - t.fr);
  const float w10 = (1.0f - t.fc) * t.fr, w11 = t.fc * t.fr;
  if (ggrid && rgba) {
    float4* g4 = reinterpret_cast<float4*>(ggrid);
    atomicAdd(g4 + t.i00, make_float4(up[0] * w00, up[1] * w00, up[2] * w00, 0.f));
    atomicAdd(g4 + t.i01, make_float4(up[0] * w01, up[1] * w01, up[2] * w01, 0.f));
    atomicAdd(g4 + t.i10, make_float4(up[0] * w10, up[1] * w10, up[2] * w10, 0.f));
    atomicAdd(g4 + t.i11, make_float4(up[0] * w11, up[1] * w11, up[2] * w11, 0.f));
  }
  float dfc = 0.f, dfr = 0.f;
  for (int ch = 0; ch < 3; ++ch) {
    const float u = up[ch];
    if (ggrid && !rgba) {
      atomicAdd(ggrid + 3 * t.i00 + ch, u * w00);
      atomicAdd(ggrid + 3 * t.i01 + ch, u * w01);
      atomicAdd(ggrid + 3 * t.i10 + ch, u * w10);
      atomicAdd(ggrid + 3 * t.i11 + ch, u * w11);
    }
    const float t00 = g.data[3 * t.i00 + ch], t01 = g.data[3 * t.i01 + ch];
    const float t10 = g.data[3 * t.i10 + ch], t11 = g.data[3 * t.i11 + ch];
    dfc += u * ((1.0f - t.fr) * (t01 - t00) + t.fr * (t11 - t10));
    dfr += u * ((t10 - t00) + t.fc * ((t11 - t10) - (t01 - t00)));
  }
  const float PI_F = 3.14159265358979323846f, TWO_PI_F = 6.28318530717958647692f;
  const float drow = t.interior ? dfr : 0.0f;
  const float dtheta = drow * ((float)g.h / PI_F);
  const float dphi = dfc * ((float)g.w / TWO_PI_F);
  const float zc = dz < -1.0f ? -1.0f : (dz > 1.0f ? 1.0f : dz);
  const bool at_pole = fabsf(dz) >= 1.0f;
  ddir[2] = at_pole ? 0.0f : -dtheta * rsqrtf(1.0f - zc * zc);
  const float ir2 = __fdividef(1.0f, fmaxf(dx * dx + dy * dy, 1e-30f));
  ddir[0] = -dy * ir2 * dphi;
  ddir[1] = dx * ir2 * dphi;
}

__global__ void __launch_bounds__(256) k_shade_bwd(ShadeBwdParams p) {
  const int W = p.cam.width, H = p.cam.height;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= W * H) return;
  // this CTA's private copy of the environment gradient grids
  const size_t shard = p.shard_stride ? (size_t)(blockIdx.x % kEnvShards) * p.shard_stride : 0;
  const bool rgba = p.shard_stride != 0;  // shards hold 4 floats per texel
  const size_t HW = (size_t)W * H;
  float g[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) g[c] = __ldg(p.gbuf + c * HW + pix);
  float dg[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) dg[c] = 0.f;
  const float a = g[12];
  if (a > TSB_COVER_EPS) {
    float wo[3];
    view_dir_pix(p.view, pix, W, wo);
    const tsb_env_params& env = p.env;
    const float ia = __fdividef(1.0f, a);
    const float alb[3] = {g[0] * ia, g[1] * ia, g[2] * ia};
    const float metal = g[3] * ia, rough = g[4] * ia;
    const float nb[3] = {g[5], g[6], g[7]};
    const float nn = sqrtf((nb[0] * nb[0] + nb[1] * nb[1]) + nb[2] * nb[2]);
    const bool degen = nn < 1e-12f;
    float n[3];
    const float rn = degen ? 0.0f : __fdividef(1.0f, nn);  // (tolerance-checked shading)
    for (int c = 0; c < 3; ++c) n[c] = degen ? wo[c] : nb[c] * rn;
    const float cos_raw = (n[0] * wo[0] + n[1] * wo[1]) + n[2] * wo[2];
    const float cos_cl = cos_raw < TSB_COS_MIN ? TSB_COS_MIN : (cos_raw > 1.0f ? 1.0f : cos_raw);
    float wr[3];
    for (int c = 0; c < 3; ++c) wr[c] = (2.0f * cos_raw) * n[c] - wo[c];
    float A, B;
    tsb_sample_lut(env.lut, env.lut_res, cos_cl, rough, &A, &B);
    // specular levels (environment.py:270-300)
    const int L = env.levels;
    const float rc = rough < 0.0f ? 0.0f : (rough > 1.0f ? 1.0f : rough);
    const float f = rc * (float)(L - 1);
    int l0 = (int)floorf(f);
    if (l0 > L - 1) l0 = L - 1;
    const float fl = f - (float)l0;
    const int l1 = l0 + 1 < L - 1 ? l0 + 1 : L - 1;
    float s0[3], s1[3], spec[3], irr[3];
    tsb_sample_equirect(&env.mips[l0], wr[0], wr[1], wr[2], s0);
    if (l1 != l0) tsb_sample_equirect(&env.mips[l1], wr[0], wr[1], wr[2], s1);
    else for (int c = 0; c < 3; ++c) s1[c] = s0[c];
    for (int c = 0; c < 3; ++c)
      spec[c] = l1 != l0 ? (1.0f - fl) * s0[c] + fl * s1[c] : ((1.0f - fl) + fl) * s0[c];
    tsb_sample_equirect(&env.diffuse, n[0], n[1], n[2], irr);
    const float INV_PI = 0.318309886183790671538f;
    float f0[3], ld[3], ls[3];
    for (int c = 0; c < 3; ++c) {
      f0[c] = 0.04f * (1.0f - metal) + alb[c] * metal;
      ls[c] = (f0[c] * A + B) * spec[c];
      ld[c] = (alb[c] * INV_PI) * (1.0f - metal) * irr[c];
    }
    // ---- adjoint (shading.py:186-228 with V = 1)
    float dl[3], da = 0.f;
    for (int c = 0; c < 3; ++c) {
      const float dc = __ldg(p.dcolor + 3 * (size_t)pix + c);
      dl[c] = a * dc;
      da += dc * ((ld[c] + ls[c]) - p.bg[c]);
    }
    float dalb[3], dirr[3], dspec[3];
    float dmetal = 0.f, dA = 0.f, dB = 0.f;
    for (int c = 0; c < 3; ++c) {
      dalb[c] = dl[c] * (1.0f - metal) * irr[c] * INV_PI;
      dmetal -= dl[c] * alb[c] * irr[c] * INV_PI;
      dirr[c] = dl[c] * alb[c] * (1.0f - metal) * INV_PI;
      const float df0 = dl[c] * A * spec[c];
      dA += dl[c] * f0[c] * spec[c];
      dB += dl[c] * spec[c];
      dspec[c] = dl[c] * (f0[c] * A + B);
      dalb[c] += df0 * metal;
      dmetal += df0 * (alb[c] - 0.04f);
    }
    float dn_diff[3];
    eq_grad(env.diffuse, p.gdiffuse ? p.gdiffuse + shard : nullptr, rgba, n[0], n[1], n[2],
            dirr, dn_diff);
    // LUT adjoint (environment.py:449-464)
    float dcos_cl, drough_lut;
    {
      const int res = env.lut_res;
      const float x = cos_cl * (float)res - 0.5f, y = rough * (float)res - 0.5f;
      const float hi = (float)(res - 1);
      const float xc = x < 0.0f ? 0.0f : (x > hi ? hi : x);
      const float yc = y < 0.0f ? 0.0f : (y > hi ? hi : y);
      const float xf = floorf(xc), yf = floorf(yc);
      const int i0 = (int)xf, j0 = (int)yf;
      const float fx = xc - xf, fy = yc - yf;
      const int i1 = i0 + 1 < res - 1 ? i0 + 1 : res - 1;
      const int j1 = j0 + 1 < res - 1 ? j0 + 1 : res - 1;
      const float* t00 = env.lut + 2 * (j0 * res + i0);
      const float* t01 = env.lut + 2 * (j0 * res + i1);
      const float* t10 = env.lut + 2 * (j1 * res + i0);
      const float* t11 = env.lut + 2 * (j1 * res + i1);
      float dfx = 0.f, dfy = 0.f;
      const float up[2] = {dA, dB};
      for (int q = 0; q < 2; ++q) {
        dfx += up[q] * ((1.0f - fy) * (t01[q] - t00[q]) + fy * (t11[q] - t10[q]));
        dfy += up[q] * ((t10[q] - t00[q]) + fx * ((t11[q] - t10[q]) - (t01[q] - t00[q])));
      }
      dcos_cl = (x > 0.0f && x < hi) ? dfx * (float)res : 0.0f;
      drough_lut = (y > 0.0f && y < hi) ? dfy * (float)res : 0.0f;
    }
    // specular adjoint (environment.py:302-331)
    float dwr[3] = {0.f, 0.f, 0.f};
    {
      float up[3], dd[3];
      const float w0 = l1 != l0 ? 1.0f - fl : (1.0f - fl) + fl;
      for (int c = 0; c < 3; ++c) up[c] = dspec[c] * w0;
      eq_grad(env.mips[l0], p.gmips[l0] ? p.gmips[l0] + shard : nullptr, rgba, wr[0], wr[1],
              wr[2], up, dd);
      for (int c = 0; c < 3; ++c) dwr[c] += dd[c];
      if (l1 != l0 && fl != 0.0f) {
        for (int c = 0; c < 3; ++c) up[c] = dspec[c] * fl;
        eq_grad(env.mips[l1], p.gmips[l1] ? p.gmips[l1] + shard : nullptr, rgba, wr[0],
                wr[1], wr[2], up, dd);
        for (int c = 0; c < 3; ++c) dwr[c] += dd[c];
      }
    }
    float dfl = 0.f;
    for (int c = 0; c < 3; ++c) dfl += dspec[c] * (s1[c] - s0[c]);
    const bool interior = rough > 0.0f && rough < 1.0f && l0 != l1;
    const float drough = drough_lut + (interior ? dfl * (float)(L - 1) : 0.0f);
    // normal adjoint
    float dn[3];
    const float dwn = (dwr[0] * n[0] + dwr[1] * n[1]) + dwr[2] * n[2];
    const float dcos = (cos_raw > TSB_COS_MIN && cos_raw < 1.0f) ? dcos_cl : 0.0f;
    for (int c = 0; c < 3; ++c)
      dn[c] = 2.0f * dwn * wo[c] + 2.0f * cos_raw * dwr[c] + dcos * wo[c] + dn_diff[c];
    if (!degen) {
      const float ndn = (n[0] * dn[0] + n[1] * dn[1]) + n[2] * dn[2];
      for (int c = 0; c < 3; ++c) dg[5 + c] = (dn[c] - n[c] * ndn) * rn;
    }
    // de-premultiply
    for (int c = 0; c < 3; ++c) {
      dg[c] = dalb[c] * ia;
      da -= dalb[c] * alb[c] * ia;
    }
    dg[3] = dmetal * ia;
    da -= dmetal * metal * ia;
    dg[4] = drough * ia;
    da -= drough * rough * ia;
    dg[12] = da;
  }
#pragma unroll
  for (int c = 0; c < 13; ++c) p.dgbuf[c * HW + pix] = dg[c];
}

// Sum the environment-gradient shards (4 floats per texel) into the caller's
// (h, w, 3) grids.
struct EnvShardPlan {
  float* dst[TSB_MAX_LEVELS + 1];   // caller grids: mips then diffuse
  int32_t off[TSB_MAX_LEVELS + 2];  // float offset of each grid in the caller layout (3/texel)
  int32_t off4[TSB_MAX_LEVELS + 2]; // ... and in a shard (4/texel)
  int32_t nseg;
};

__global__ void k_env_shard_reduce(const float* __restrict__ shards, int32_t n3, int32_t stride,
                                   EnvShardPlan plan) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n3) return;
  int seg = 0;
  while (seg + 1 < plan.nseg && plan.off[seg + 1] <= i) ++seg;
  const int li = i - plan.off[seg];
  const int j = plan.off4[seg] + 4 * (li / 3) + li % 3;
  float s = 0.f;
  for (int k = 0; k < kEnvShards; ++k) s += shards[(size_t)k * stride + j];
  float* d = plan.dst[seg];
  if (d) d[li] += s;
}

// ---------------------------------------------------------------------------
// K8 raster backward
// ---------------------------------------------------------------------------
struct RasterBwdParams {
  tsb_cam_params cam;
  int32_t W, H, tiles_x, tile;
  float near_f;
  const int32_t* ranges;
  const int32_t* evals;
  const GeomRec* geom;
  const MatRec* mat;
  const double* m64;
  int32_t T, page_w, tstride;
  const float4* fam_a;
  const float4* fam_b;
  const int32_t* last_entry;
  const float* T_last;
  const float* dgbuf;
  float* acc;          // P x kAccWords
  float* dtexels;      // P x T x T x tl
  // deterministic mode: fixed-point int64 accumulators instead of the float
  // atomics above (integer adds commute, so any order gives the same bits)
  unsigned long long* acc64;  // P x kAccWords, value * 2^kAccFix
  unsigned long long* tex64;  // P x T x T x tl, value * 2^kTexFix
  unsigned long long* red_count;  // diagnostics: atomic adds issued (or null)
  int32_t tl;          // channels per texel: 7 (combined) or 8 (interleaved)
  int32_t num_tiles;
  int32_t* work_counter;
  const int32_t* tile_order;
};

// Warp-private shared memory of the backward rasterizer (11 KB).
struct BwdWarpSmem {
  DecRec dec[32];          // staged step: decide records (AoS, broadcast reads)
  int32_t sid[32];         // splat ids
  float lin[11][32];       // intersection forms L0..L10 (SoA)
  float frame[9][32];      // t_u, t_v, t_u x t_v
  float lind[3][32];       // clamped SH radiance
  int32_t loff[32];        // chart offset in the linear atlas
  float mf[9][32];         // float M rows 0,1,2 x cols 0,1,3 (intersection adjoint)
  // reduction rows: first the per-splat terms of the live lanes (stride 28,
  // compacted), then per lane the 28 weighted texel values + cell offsets
  // (stride 36: conflict-free 128-bit stores)
  float red[32 * 36];
};

// Decode-normal adjoint (textures.py:290-322).
__device__ __forceinline__ void decode_grad(float ea, float eb, float gx, float gy, float gz,
                                            float* denc) {
  const float px = 2.0f * ea - 1.0f, py = 2.0f * eb - 1.0f;
  const float d2 = px * px + py * py;
  float dpx, dpy;
  if (d2 > 1.0f) {
    const float d = sqrtf(fmaxf(d2, 1e-12f));
    const float nx = px / d, ny = py / d;
    const float gdot = gx * nx + gy * ny;
    dpx = (gx - gdot * nx) / d;
    dpy = (gy - gdot * ny) / d;
  } else {
    const float nz = sqrtf(fmaxf(1e-12f, 1.0f - fminf(d2, 1.0f)));
    dpx = gx - gz * px / nz;
    dpy = gy - gz * py / nz;
  }
  denc[0] = 2.0f * dpx;
  denc[1] = 2.0f * dpy;
}

template <bool DET>
__global__ void __launch_bounds__(256, 2) k_raster_bwd(RasterBwdParams p) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  BwdWarpSmem& ws = *reinterpret_cast<BwdWarpSmem*>(s_raw + (size_t)warp * sizeof(BwdWarpSmem));
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int TILE = p.tile;
  const int wx = TILE / 8;
  const int nblk = TILE * TILE / 32;
  const int T = p.T;
  const int t_corner = lane / 7, t_ch = lane % 7;  // texel reducer lanes 0..27
  // combined channel -> slot of the texel layout (identity, or the 8-channel
  // interleaved atlas order [alb rgb, rough, nrm a, nrm b, metal, 0])
  const int t_slot = p.tl == 8 ? (t_ch == 4 ? 6 : (t_ch >= 5 ? t_ch - 1 : t_ch)) : t_ch;
  const int tl = p.tl;
  // persistent warps over (tile, 8x4 block) units, heaviest tiles first
  // (the forward's schedule order, left in the workspace)
  const int num_units = p.num_tiles * nblk;
  while (true) {
    int unit = 0;
    if (lane == 0) unit = atomicAdd(p.work_counter, 1);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= num_units) break;
    const int tile = p.tile_order ? p.tile_order[unit / nblk] : unit / nblk;
    const int blk = unit % nblk;
    const int start = p.ranges[2 * tile];
    const int bx0 = (tile % p.tiles_x) * TILE + (blk % wx) * 8;
    const int by0 = (tile / p.tiles_x) * TILE + (blk / wx) * 4;
    if (bx0 >= p.W || by0 >= p.H) continue;
    const int bx1 = min(bx0 + 8, p.W), by1 = min(by0 + 4, p.H);
    const BlockBox bb = tsb_block_box(p.cam, bx0, by0, bx1, by1);
    const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
    const bool inside = px < p.W && py < p.H;
    const int pix = py * p.W + px;
    const float x = (float)tsb_pixel_x(&p.cam, px), y = (float)tsb_pixel_y(&p.cam, py);
    const size_t HW = (size_t)p.W * p.H;
    const int last = inside ? p.last_entry[pix] : -1;
    float Tc = inside ? p.T_last[pix] : 0.f;
    float g[13], R[13];
#pragma unroll
    for (int c = 0; c < 13; ++c) {
      g[c] = inside ? __ldg(p.dgbuf + c * HW + pix) : 0.f;
      R[c] = 0.f;
    }
    bool first = true;  // next contributor met is the last one
    const int blk_last = __reduce_max_sync(0xffffffffu, last);
    for (int hi = blk_last; hi >= start; hi -= 32) {
      const int lo = max(start, hi - 31);
      const int cnt = hi - lo + 1;
      // ---- stage the step [lo, hi]
      __syncwarp();
      bool hit = false;
      uint32_t bflags = 0;
      if (lane < cnt) {
        const int rs = __ldg(p.evals + lo + lane);  // the entry's record slot
        float4 gv[4];
        hit = tsb_stage_geom(p.geom, rs, lane, bx0, by0, bx1, by1, ws.dec, bb, p.near_f, bflags,
                             gv) != 0;
        const int id = __float_as_int(gv[3].z);  // splat id (GeomRec.id)
        const float gl[11] = {gv[0].x, gv[0].y, gv[0].z, gv[0].w, gv[1].x, gv[1].y,
                              gv[1].z, gv[1].w, gv[2].x, gv[2].y, gv[2].z};
#pragma unroll
        for (int c = 0; c < 11; ++c) ws.lin[c][lane] = gl[c];
        ws.sid[lane] = id;
        const float4* mq = reinterpret_cast<const float4*>(p.mat + rs);
        const float4 m0 = __ldg(mq), m1 = __ldg(mq + 1), m2 = __ldg(mq + 2), m3 = __ldg(mq + 3);
        ws.frame[0][lane] = m0.x; ws.frame[1][lane] = m0.y; ws.frame[2][lane] = m0.z;
        ws.frame[3][lane] = m0.w; ws.frame[4][lane] = m1.x; ws.frame[5][lane] = m1.y;
        ws.frame[6][lane] = m1.z; ws.frame[7][lane] = m1.w; ws.frame[8][lane] = m2.x;
        ws.lind[0][lane] = m2.y; ws.lind[1][lane] = m2.z; ws.lind[2][lane] = m2.w;
        ws.loff[lane] = __float_as_int(m3.w);
        const double* m64 = p.m64 + (size_t)kM64Stride * id;
#pragma unroll
        for (int c = 0; c < 9; ++c) ws.mf[c][lane] = (float)__ldg(m64 + c);
      }
      const uint32_t cand = __ballot_sync(0xffffffffu, hit);
      const uint32_t fullm = __ballot_sync(0xffffffffu, (bflags & kBlockLive) != 0);
      const uint32_t zsm = __ballot_sync(0xffffffffu, (bflags & kBlockZSafe) != 0);
      __syncwarp();
      if (!cand) continue;
      // ---- decide: this pixel's contributors in the step (entries <= last)
      uint32_t live = 0;
      if (last >= lo) {
        const int nv = last - lo + 1;
        const uint32_t valid = nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u);
        // uniform candidate loop (broadcast reads), masked afterwards
        auto load_lin = [&](int k, float* L) {
#pragma unroll
          for (int c = 0; c < 11; ++c) L[c] = ws.lin[c][k];
          L[11] = ws.dec[k].r2hi;
        };
        auto dec_at = [&](int k) {
          const DecRec& d = ws.dec[k];
          return DecRef{d.lin, d.r2hi, d.pixmask};
        };
        live = (fullm | tsb_decide_step(dec_at, load_lin, ws.sid, cand & ~fullm, zsm, lane, x, y,
                                        p.near_f, p.cam, p.m64, px, py)) & valid;
      }
      // ---- adjoint, back to front over the entries with a live pixel
      for (uint32_t any = __reduce_or_sync(0xffffffffu, live); any;) {
        const int k = 31 - __clz(any);
        any &= ~(1u << k);
        const bool lk = (live >> k) & 1u;
        const uint32_t lm = __ballot_sync(0xffffffffu, lk);
        const int id = ws.sid[k];
        int tkey = -1 - lane;  // non-live lanes: singleton groups, never leaders
        int tdx = 0, tdy = 0;
        float tw[28];          // texel gradient: 4 corners x 7 channels
        if (lk) {
          float c_acc[24];
          float L[11];
#pragma unroll
          for (int c = 0; c < 11; ++c) L[c] = ws.lin[c][k];
          float u, v, z, a;
          tsb_uvza_lin(L, x, y, &u, &v, &z, &a);
          float fr[9];
#pragma unroll
          for (int c = 0; c < 9; ++c) fr[c] = ws.frame[c][k];
          // ---- recompute the fragment's attributes (verify sampler)
          tsb_texc tc;
          tsb_texel_coords(u, v, T, &tc);
          const int S = p.tstride;
          const int loff = ws.loff[k];
          const int r0 = loff + tc.j0 * p.page_w, r1 = loff + tc.j1 * p.page_w;
          const float4 a00 = __ldg(p.fam_a + S * (r0 + tc.i0)), a01 = __ldg(p.fam_a + S * (r0 + tc.i1));
          const float4 a10 = __ldg(p.fam_a + S * (r1 + tc.i0)), a11 = __ldg(p.fam_a + S * (r1 + tc.i1));
          const float4 b00 = __ldg(p.fam_b + S * (r0 + tc.i0)), b01 = __ldg(p.fam_b + S * (r0 + tc.i1));
          const float4 b10 = __ldg(p.fam_b + S * (r1 + tc.i0)), b11 = __ldg(p.fam_b + S * (r1 + tc.i1));
          // 7 combined channels: alb rgb, rough, metal, nrm a, b
          const float c00[7] = {a00.x, a00.y, a00.z, a00.w, b00.z, b00.x, b00.y};
          const float c01[7] = {a01.x, a01.y, a01.z, a01.w, b01.z, b01.x, b01.y};
          const float c10[7] = {a10.x, a10.y, a10.z, a10.w, b10.z, b10.x, b10.y};
          const float c11[7] = {a11.x, a11.y, a11.z, a11.w, b11.z, b11.x, b11.y};
          float t7[7];
#pragma unroll
          for (int c = 0; c < 7; ++c) t7[c] = tsb_lerp4(c00[c], c01[c], c10[c], c11[c], tc.fs, tc.ft);
          float xa[13];
          xa[0] = t7[0]; xa[1] = t7[1]; xa[2] = t7[2]; xa[3] = t7[4]; xa[4] = t7[3];
          tsb_decode_normal(t7[5], t7[6], fr, xa + 5);
          xa[8] = ws.lind[0][k]; xa[9] = ws.lind[1][k]; xa[10] = ws.lind[2][k];
          xa[11] = z;
          xa[12] = 1.0f;
          // transmittance in front of this fragment
          if (!first) Tc = Tc / (1.0f - a);
          first = false;
          const float w = a * Tc;
          // ---- alpha adjoint and the colour behind
          float dalpha = 0.f;
#pragma unroll
          for (int c = 0; c < 13; ++c) dalpha += g[c] * (xa[c] - R[c]);
          dalpha *= Tc;
#pragma unroll
          for (int c = 0; c < 13; ++c) R[c] = a * xa[c] + (1.0f - a) * R[c];
          float dx[12];
#pragma unroll
          for (int c = 0; c < 12; ++c) dx[c] = w * g[c];
          const float G = tsb_expf(-0.5f * fmaf(u, u, v * v));
          c_acc[9] = dalpha * G;
          float du = -dalpha * a * u, dv = -dalpha * a * v;
          const float dz = dx[11];
          c_acc[10] = dx[8]; c_acc[11] = dx[9]; c_acc[12] = dx[10];
          // ---- normal chain (rasterize.py:538-547)
          float nt[3];
          {
            float nx = 2.0f * t7[5] - 1.0f, ny = 2.0f * t7[6] - 1.0f;
            const float d2 = nx * nx + ny * ny;
            if (d2 > 1.0f) { const float sc = 1.0f / sqrtf(d2); nx *= sc; ny *= sc; }
            const float q = (1.0f - nx * nx) - ny * ny;
            nt[0] = nx; nt[1] = ny; nt[2] = sqrtf(q > 0.0f ? q : 0.0f);
          }
          const float dnw[3] = {dx[5], dx[6], dx[7]};
          const float gx = dnw[0] * fr[0] + dnw[1] * fr[1] + dnw[2] * fr[2];
          const float gy = dnw[0] * fr[3] + dnw[1] * fr[4] + dnw[2] * fr[5];
          const float gz = dnw[0] * fr[6] + dnw[1] * fr[7] + dnw[2] * fr[8];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            c_acc[13 + i] = dnw[i] * nt[0];
            c_acc[16 + i] = dnw[i] * nt[1];
            c_acc[19 + i] = dnw[i] * nt[2];
          }
          float denc[2];
          decode_grad(t7[5], t7[6], gx, gy, gz, denc);
          const float up7[7] = {dx[0], dx[1], dx[2], dx[4], dx[3], denc[0], denc[1]};
          float dfs = 0.f, dft = 0.f;
#pragma unroll
          for (int c = 0; c < 7; ++c) {
            dfs += up7[c] * ((1.0f - tc.ft) * (c01[c] - c00[c]) + tc.ft * (c11[c] - c10[c]));
            dft += up7[c] * ((c10[c] - c00[c]) + tc.fs * ((c11[c] - c10[c]) - (c01[c] - c00[c])));
          }
          // chart coordinate adjoint (textures.py:167-178, rasterize.py:563-587)
          {
            const float inv = (float)(1.0 / (2.0 * TSB_SUPPORT_SIGMA));
            const float half = 0.5f / (float)T;
            const float sup = (float)TSB_SUPPORT_SIGMA;
            const float s_raw = (u + sup) * inv, t_raw = (v + sup) * inv;
            const float s = s_raw < half ? half : (s_raw > 1.0f - half ? 1.0f - half : s_raw);
            const float t = t_raw < half ? half : (t_raw > 1.0f - half ? 1.0f - half : t_raw);
            const float xs = s * (float)T - 0.5f, yt = t * (float)T - 0.5f;
            const float ds = (xs > 0.0f && xs < (float)(T - 1)) ? dfs * (float)T : 0.0f;
            const float dtt = (yt > 0.0f && yt < (float)(T - 1)) ? dft * (float)T : 0.0f;
            if (s_raw > half && s_raw < 1.0f - half) du += ds * inv;
            if (t_raw > half && t_raw < 1.0f - half) dv += dtt * inv;
          }
          // ---- intersection adjoint (rasterize.py:605-639), fold to dWH
          {
            float M[9];
#pragma unroll
            for (int c = 0; c < 9; ++c) M[c] = ws.mf[c][k];  // rows 0,1,2 x cols 0,1,3
            const float hu0 = x * M[6] - M[0], hu1 = x * M[7] - M[1], hu3 = x * M[8] - M[2];
            const float hv0 = y * M[6] - M[3], hv1 = y * M[7] - M[4], hv3 = y * M[8] - M[5];
            const float D = hu0 * hv1 - hu1 * hv0;
            const float uu = (hu1 * hv3 - hu3 * hv1) / D, vv = (hu3 * hv0 - hu0 * hv3) / D;
            const float du2 = du + dz * M[6], dv2 = dv + dz * M[7];
            const float dNu = du2 / D, dNv = dv2 / D;
            const float dD = -(uu * du2 + vv * dv2) / D;
            const float dhu0 = dD * hv1 - dNv * hv3, dhu1 = dNu * hv3 - dD * hv0;
            const float dhu3 = dNv * hv0 - dNu * hv1;
            const float dhv0 = dNv * hu3 - dD * hu1, dhv1 = dD * hu0 - dNu * hu3;
            const float dhv3 = dNu * hu1 - dNv * hu0;
            c_acc[0] = -dhu0; c_acc[1] = -dhu1; c_acc[2] = -dhu3;
            c_acc[3] = -dhv0; c_acc[4] = -dhv1; c_acc[5] = -dhv3;
            // row 2 of WH receives dM[2] + dM[3] (PROJ_FLATTEN duplicates row 2)
            c_acc[6] = dz * uu + (x * dhu0 + y * dhv0);
            c_acc[7] = dz * vv + (x * dhu1 + y * dhv1);
            c_acc[8] = dz + (x * dhu3 + y * dhv3);
          }
          c_acc[22] = c_acc[23] = 0.f;
          // ---- per-splat terms: row at the lane's rank among the live lanes
          float4* rr = reinterpret_cast<float4*>(ws.red + 28 * __popc(lm & lt_mask));
#pragma unroll
          for (int q = 0; q < 6; ++q)
            rr[q] = make_float4(c_acc[4 * q], c_acc[4 * q + 1], c_acc[4 * q + 2], c_acc[4 * q + 3]);
#pragma unroll
          for (int c = 0; c < 7; ++c) {
            tw[c] = up7[c] * ((1.0f - tc.fs) * (1.0f - tc.ft));
            tw[7 + c] = up7[c] * (tc.fs * (1.0f - tc.ft));
            tw[14 + c] = up7[c] * ((1.0f - tc.fs) * tc.ft);
            tw[21 + c] = up7[c] * (tc.fs * tc.ft);
          }
          // cell key = the (i0, j0) corner's offset; corner steps to (i1, j1)
          tkey = tl * (tc.j0 * T + tc.i0);
          tdx = tl * (tc.i1 - tc.i0);
          tdy = tl * T * (tc.j1 - tc.j0);
        }
        __syncwarp();
        // ---- per-splat terms: lane c < 22 sums column c over the live rows
        if (lane < 22) {
          const int nl = __popc(lm);
          float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;  // four independent chains
          int i = 0;
          for (; i + 4 <= nl; i += 4) {
            t0 += ws.red[28 * i + lane];
            t1 += ws.red[28 * (i + 1) + lane];
            t2 += ws.red[28 * (i + 2) + lane];
            t3 += ws.red[28 * (i + 3) + lane];
          }
          for (; i < nl; ++i) t0 += ws.red[28 * i + lane];
          const float tot = (t0 + t1) + (t2 + t3);
          count_red(p.red_count, tot != 0.0f);
          if (tot != 0.0f) {
            if constexpr (DET)
              atomicAdd(p.acc64 + (size_t)kAccWords * id + lane, to_fix(tot, kAccFix));
            else
              atomicAdd(p.acc + (size_t)kAccWords * id + lane, tot);
          }
        }
        __syncwarp();
        if (lk) {
          float4* tr = reinterpret_cast<float4*>(ws.red + 36 * lane);
#pragma unroll
          for (int q = 0; q < 7; ++q)
            tr[q] = make_float4(tw[4 * q], tw[4 * q + 1], tw[4 * q + 2], tw[4 * q + 3]);
          tr[7] = make_float4(__int_as_float(tkey), __int_as_float(tdx), __int_as_float(tdy), 0.f);
        }
        __syncwarp();
        // ---- texel gradients (per-splat (T, T, 7) combined layout,
        // rasterize.py:548-562): live lanes grouped by bilinear cell
        // (match.any); for each group, reducer lane (corner, channel) sums
        // its weighted value over the members and issues one atomic
        {
          float* dt = p.dtexels + (size_t)id * T * T * tl;
          const uint32_t peers = __match_any_sync(0xffffffffu, tkey);
          uint32_t leaders = __ballot_sync(0xffffffffu, lk && lane == __ffs(peers) - 1);
          while (leaders) {
            const int l = __ffs(leaders) - 1;
            leaders &= leaders - 1;
            const uint32_t grp = __shfl_sync(0xffffffffu, peers, l);
            if (lane < 28) {
              float s0 = 0.f, s1 = 0.f;  // two independent chains over the members
              uint32_t m = grp;
              for (; __popc(m) >= 2;) {
                const int a = __ffs(m) - 1;
                m &= m - 1;
                const int b = __ffs(m) - 1;
                m &= m - 1;
                s0 += ws.red[36 * a + lane];
                s1 += ws.red[36 * b + lane];
              }
              if (m) s0 += ws.red[36 * (__ffs(m) - 1) + lane];
              const float tsum = s0 + s1;
              const int* lr = reinterpret_cast<const int*>(ws.red + 36 * l + 28);
              const int off = lr[0] + ((t_corner & 1) ? lr[1] : 0) + ((t_corner & 2) ? lr[2] : 0) + t_slot;
              count_red(p.red_count, tsum != 0.0f);
              if (tsum != 0.0f) {
                if constexpr (DET)
                  atomicAdd(p.tex64 + (size_t)id * T * T * tl + off, to_fix(tsum, kTexFix));
                else
                  atomicAdd(dt + off, tsum);
              }
            }
          }
        }
        __syncwarp();
      }
    }
  }
}

// Deterministic mode: fixed-point sums back to float (texel gradients are
// ADDED to the caller's buffer, like the atomic path).
__global__ void k_det_unfix(int64_t n_acc, const unsigned long long* __restrict__ acc64,
                            float* __restrict__ acc, int64_t n_tex,
                            const unsigned long long* __restrict__ tex64,
                            float* __restrict__ dtexels) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_acc; i += stride)
    acc[i] = (float)((double)(long long)acc64[i] * (1.0 / (double)(1ull << kAccFix)));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_tex; i += stride) {
    const long long v = (long long)tex64[i];
    if (v) dtexels[i] += (float)((double)v * (1.0 / (double)(1ull << kTexFix)));
  }
}

// ---------------------------------------------------------------------------
// K9 finish: per-splat parameter gradients in fp64
// ---------------------------------------------------------------------------
struct FinishParams {
  tsb_cam_params cam;
  int32_t P, sh_degree;
  const double* pos;
  const double* tu;
  const double* tv;
  const double* sc;
  const double* sh;
  const float* acc;
  double* g_pos;
  double* g_tu;
  double* g_tv;
  double* g_sc;
  double* g_op;
  double* g_sh;
};

// d(basis_k)/d(dir) for degree <= 3 (sh.py:64-101): out[k][3].
__device__ void sh_basis_grad(double x, double y, double z, int degree, double (*g)[3]) {
  for (int k = 0; k < 16; ++k) g[k][0] = g[k][1] = g[k][2] = 0.0;
  const double C1 = 0.4886025119029199;
  if (degree >= 1) { g[1][1] = -C1; g[2][2] = C1; g[3][0] = -C1; }
  if (degree >= 2) {
    const double c0 = 1.0925484305920792, c1 = -1.0925484305920792, c2 = 0.31539156525252005,
                 c3 = -1.0925484305920792, c4 = 0.5462742152960396;
    g[4][0] = c0 * y; g[4][1] = c0 * x;
    g[5][1] = c1 * z; g[5][2] = c1 * y;
    g[6][0] = c2 * (-2 * x); g[6][1] = c2 * (-2 * y); g[6][2] = c2 * (4 * z);
    g[7][0] = c3 * z; g[7][2] = c3 * x;
    g[8][0] = c4 * (2 * x); g[8][1] = c4 * (-2 * y);
  }
  if (degree >= 3) {
    const double xx = x * x, yy = y * y, zz = z * z;
    const double d0 = -0.5900435899266435, d1 = 2.890611442640554, d2 = -0.4570457994644658,
                 d3 = 0.3731763325901154, d4 = -0.4570457994644658, d5 = 1.445305721320277,
                 d6 = -0.5900435899266435;
    g[9][0] = d0 * (6 * x * y); g[9][1] = d0 * (3 * xx - 3 * yy);
    g[10][0] = d1 * (y * z); g[10][1] = d1 * (x * z); g[10][2] = d1 * (x * y);
    g[11][0] = d2 * (-2 * x * y); g[11][1] = d2 * (4 * zz - xx - 3 * yy); g[11][2] = d2 * (8 * y * z);
    g[12][0] = d3 * (-6 * x * z); g[12][1] = d3 * (-6 * y * z); g[12][2] = d3 * (6 * zz - 3 * xx - 3 * yy);
    g[13][0] = d4 * (4 * zz - 3 * xx - yy); g[13][1] = d4 * (-2 * x * y); g[13][2] = d4 * (8 * x * z);
    g[14][0] = d5 * (2 * x * z); g[14][1] = d5 * (-2 * y * z); g[14][2] = d5 * (xx - yy);
    g[15][0] = d6 * (3 * xx - 3 * yy); g[15][1] = d6 * (-6 * x * y);
  }
}

__global__ void __launch_bounds__(128) k_finish_grads(FinishParams p) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= p.P) return;
  const float* a = p.acc + (size_t)kAccWords * id;
  const double* W = p.cam.w2v;
  double tu[3], tv[3], pos[3];
  for (int j = 0; j < 3; ++j) {
    tu[j] = p.tu[3 * id + j]; tv[j] = p.tv[3 * id + j]; pos[j] = p.pos[3 * id + j];
  }
  const double s0 = p.sc[2 * id], s1 = p.sc[2 * id + 1];
  // dH[0:3][c] = R^T dWH[0:3][c] for c in (0, 1, 3)
  double dH[3][3];  // [col index 0,1,3][xyz]
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < 3; ++j)
      dH[c][j] = (W[0 + j] * (double)a[0 + c] + W[4 + j] * (double)a[3 + c]) +
                 W[8 + j] * (double)a[6 + c];
  double gp[3], gtu[3], gtv[3];
  for (int j = 0; j < 3; ++j) {
    gp[j] = dH[2][j];
    gtu[j] = s0 * dH[0][j] + (double)a[13 + j];
    gtv[j] = s1 * dH[1][j] + (double)a[16 + j];
  }
  double gs0 = (tu[0] * dH[0][0] + tu[1] * dH[0][1]) + tu[2] * dH[0][2];
  double gs1 = (tv[0] * dH[1][0] + tv[1] * dH[1][1]) + tv[2] * dH[1][2];
  // cross = t_u x t_v: dt_u += t_v x dn3, dt_v += dn3 x t_u
  const double dn3[3] = {a[19], a[20], a[21]};
  gtu[0] += tv[1] * dn3[2] - tv[2] * dn3[1];
  gtu[1] += tv[2] * dn3[0] - tv[0] * dn3[2];
  gtu[2] += tv[0] * dn3[1] - tv[1] * dn3[0];
  gtv[0] += dn3[1] * tu[2] - dn3[2] * tu[1];
  gtv[1] += dn3[2] * tu[0] - dn3[0] * tu[2];
  gtv[2] += dn3[0] * tu[1] - dn3[1] * tu[0];
  // SH chain (rasterize.py:659-676)
  const double dl[3] = {a[10], a[11], a[12]};
  const int K = (p.sh_degree + 1) * (p.sh_degree + 1);
  if (dl[0] != 0.0 || dl[1] != 0.0 || dl[2] != 0.0) {
    double cr[3] = {tu[1] * tv[2] - tu[2] * tv[1], tu[2] * tv[0] - tu[0] * tv[2],
                    tu[0] * tv[1] - tu[1] * tv[0]};
    const double cn = sqrt((cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]);
    const double cnd = cn > 1e-30 ? cn : 1e-30;
    const double n[3] = {cr[0] / cnd, cr[1] / cnd, cr[2] / cnd};
    double C[3];
    for (int j = 0; j < 3; ++j)
      C[j] = ((-W[0 + j] * W[3]) + (-W[4 + j] * W[7])) + (-W[8 + j] * W[11]);
    const double tc[3] = {C[0] - pos[0], C[1] - pos[1], C[2] - pos[2]};
    const double dist = sqrt((tc[0] * tc[0] + tc[1] * tc[1]) + tc[2] * tc[2]);
    const double dd = dist > 1e-30 ? dist : 1e-30;
    const double wo[3] = {tc[0] / dd, tc[1] / dd, tc[2] / dd};
    const double ndo = (n[0] * wo[0] + n[1] * wo[1]) + n[2] * wo[2];
    double wr[3];
    for (int j = 0; j < 3; ++j) wr[j] = (2.0 * ndo) * n[j] - wo[j];
    double b[16];
    tsb_sh_basis(wr[0], wr[1], wr[2], p.sh_degree, b);
    const double* sh = p.sh + (size_t)3 * K * id;
    double live[3];
    for (int c = 0; c < 3; ++c) {
      double raw = 0.0;
      for (int k = 0; k < K; ++k) raw += b[k] * sh[3 * k + c];
      live[c] = raw > 0.0 ? dl[c] : 0.0;
    }
    double* gsh = p.g_sh + (size_t)3 * K * id;
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < 3; ++c) gsh[3 * k + c] += b[k] * live[c];
    double gb[16][3];
    sh_basis_grad(wr[0], wr[1], wr[2], p.sh_degree, gb);
    double ddir[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < K; ++k) {
      const double s = (live[0] * sh[3 * k] + live[1] * sh[3 * k + 1]) + live[2] * sh[3 * k + 2];
      for (int j = 0; j < 3; ++j) ddir[j] += s * gb[k][j];
    }
    const double ndd = (n[0] * ddir[0] + n[1] * ddir[1]) + n[2] * ddir[2];
    const double nwo = ndo;
    double dn[3], dwo[3];
    for (int j = 0; j < 3; ++j) {
      dn[j] = 2.0 * ndd * wo[j] + 2.0 * nwo * ddir[j];
      dwo[j] = 2.0 * ndd * n[j] - ddir[j];
    }
    const double ndn = (n[0] * dn[0] + n[1] * dn[1]) + n[2] * dn[2];
    double dc[3];
    for (int j = 0; j < 3; ++j) dc[j] = (dn[j] - n[j] * ndn) / cnd;
    gtu[0] += tv[1] * dc[2] - tv[2] * dc[1];
    gtu[1] += tv[2] * dc[0] - tv[0] * dc[2];
    gtu[2] += tv[0] * dc[1] - tv[1] * dc[0];
    gtv[0] += dc[1] * tu[2] - dc[2] * tu[1];
    gtv[1] += dc[2] * tu[0] - dc[0] * tu[2];
    gtv[2] += dc[0] * tu[1] - dc[1] * tu[0];
    const double wdw = (wo[0] * dwo[0] + wo[1] * dwo[1]) + wo[2] * dwo[2];
    for (int j = 0; j < 3; ++j) gp[j] += -(dwo[j] - wo[j] * wdw) / dd;
  }
  for (int j = 0; j < 3; ++j) {
    p.g_pos[3 * id + j] += gp[j];
    p.g_tu[3 * id + j] += gtu[j];
    p.g_tv[3 * id + j] += gtv[j];
  }
  p.g_sc[2 * id] += gs0;
  p.g_sc[2 * id + 1] += gs1;
  p.g_op[id] += (double)a[9];
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_backward_scratch_size(int32_t P, uint64_t* bytes) {
  if (!bytes || P < 0) {
    set_error("tsb_backward_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *bytes = (uint64_t)(P > 0 ? P : 1) * kAccWords * sizeof(float);
  return TSB_OK;
}

int tsb_debug_red_count(int32_t enable, unsigned long long* count) {
  g_count_red_host = enable != 0;
  TSB_CUDA(cudaDeviceSynchronize());
  if (count) TSB_CUDA(cudaMemcpyFromSymbol(count, g_red_count, sizeof(unsigned long long)));
  const unsigned long long z = 0ull;
  TSB_CUDA(cudaMemcpyToSymbol(g_red_count, &z, sizeof(z)));
  return TSB_OK;
}

int tsb_backward_det_scratch_size(int32_t P, int32_t T, int32_t texel_layout, uint64_t* bytes) {
  if (!bytes || P < 0 || T < 1 ||
      (texel_layout != TSB_TEXELS_COMBINED && texel_layout != TSB_TEXELS_INTERLEAVED)) {
    set_error("tsb_backward_det_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  const uint64_t Pn = (uint64_t)(P > 0 ? P : 1);
  const uint64_t tl = texel_layout == TSB_TEXELS_INTERLEAVED ? 8 : 7;
  *bytes = Pn * kAccWords * 8 + Pn * (uint64_t)T * T * tl * 8;
  return TSB_OK;
}

// Floats of all environment grids at `ch` floats per texel (offsets per grid).
static int32_t env_floats(const tsb_environment* env, int32_t* off, int ch = 3) {
  int32_t o = 0;
  for (int l = 0; l < env->levels; ++l) {
    if (off) off[l] = o;
    o += env->mip_h[l] * env->mip_w[l] * ch;
  }
  if (off) off[env->levels] = o;
  o += env->diff_h * env->diff_w * ch;
  if (off) off[env->levels + 1] = o;
  return o;
}

int tsb_shade_backward_scratch_size(const tsb_environment* env, uint64_t* bytes) {
  if (!env || !bytes || env->levels < 1 || env->levels > TSB_ENV_MAX_LEVELS) {
    set_error("tsb_shade_backward_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *bytes = (uint64_t)kEnvShards * env_floats(env, nullptr, 4) * sizeof(float);
  return TSB_OK;
}

int tsb_shade_backward(const float* gbuf, const tsb_camera* camera, const tsb_environment* env,
                       const float* background, const float* dcolor, float* dgbuf,
                       tsb_env_grads* env_grads, void* scratch, uint64_t scratch_bytes,
                       void* stream) {
  if (!gbuf || !camera || !env || !dcolor || !dgbuf) {
    set_error("tsb_shade_backward: null argument");
    return TSB_ERR_VALUE;
  }
  if (env->levels < 1 || env->levels > TSB_ENV_MAX_LEVELS || !env->lut || !env->diffuse) {
    set_error("tsb_shade_backward: bad environment");
    return TSB_ERR_VALUE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  EnvShardPlan plan;
  const int32_t nfl3 = env_floats(env, plan.off);
  const int32_t nfl = env_floats(env, plan.off4, 4);
  const bool sharded = env_grads && scratch &&
                       scratch_bytes >= (uint64_t)kEnvShards * nfl * sizeof(float);
  ShadeBwdParams sp;
  sp.cam = to_cam(camera);
  sp.view = view_coeffs(camera);
  sp.env.levels = env->levels;
  float* sh = static_cast<float*>(scratch);
  for (int l = 0; l < TSB_MAX_LEVELS; ++l) {
    const bool on = l < env->levels;
    sp.env.mips[l].data = on ? env->spec_mips[l] : nullptr;
    sp.env.mips[l].h = on ? env->mip_h[l] : 0;
    sp.env.mips[l].w = on ? env->mip_w[l] : 0;
    float* caller = (on && env_grads) ? env_grads->spec_mips[l] : nullptr;
    sp.gmips[l] = sharded && caller ? sh + plan.off4[l] : caller;
    plan.dst[l] = on ? caller : nullptr;
  }
  sp.env.diffuse.data = env->diffuse;
  sp.env.diffuse.h = env->diff_h;
  sp.env.diffuse.w = env->diff_w;
  sp.env.lut = env->lut;
  sp.env.lut_res = env->lut_res;
  float* cdiff = env_grads ? env_grads->diffuse : nullptr;
  sp.gdiffuse = sharded && cdiff ? sh + plan.off4[env->levels] : cdiff;
  plan.dst[env->levels] = cdiff;
  plan.nseg = env->levels + 1;
  sp.shard_stride = sharded ? nfl : 0;
  for (int c = 0; c < 3; ++c) sp.bg[c] = background ? background[c] : 0.f;
  sp.gbuf = gbuf; sp.dcolor = dcolor; sp.dgbuf = dgbuf;
  if (sharded) TSB_CUDA(cudaMemsetAsync(sh, 0, (size_t)kEnvShards * nfl * sizeof(float), st));
  const int n = camera->width * camera->height;
  k_shade_bwd<<<(n + 255) / 256, 256, 0, st>>>(sp);
  TSB_CHECK_LAUNCH("k_shade_bwd");
  if (sharded) {
    k_env_shard_reduce<<<(nfl3 + 255) / 256, 256, 0, st>>>(sh, nfl3, nfl, plan);
    TSB_CHECK_LAUNCH("k_env_shard_reduce");
  }
  return TSB_OK;
}

int tsb_render_backward(const tsb_scene* scene, const tsb_camera* camera, const tsb_atlas* atlas,
                        int32_t tile, const void* ws, uint64_t ws_bytes, int64_t cap,
                        const tsb_pixel_state* px, const float* dgbuf, void* scratch,
                        tsb_scene_grads* grads, void* stream) {
  return tsb_render_backward_ex(scene, camera, atlas, tile, ws, ws_bytes, cap, px, dgbuf, scratch,
                                grads, 0, nullptr, 0, stream);
}

int tsb_render_backward_ex(const tsb_scene* scene, const tsb_camera* camera,
                           const tsb_atlas* atlas, int32_t tile, const void* ws,
                           uint64_t ws_bytes, int64_t cap, const tsb_pixel_state* px,
                           const float* dgbuf, void* scratch, tsb_scene_grads* grads,
                           int32_t deterministic, void* det_scratch, uint64_t det_scratch_bytes,
                           void* stream) {
  if (!scene || !camera || !atlas || !ws || !px || !dgbuf || !scratch || !grads) {
    set_error("tsb_render_backward: null argument");
    return TSB_ERR_VALUE;
  }
  if (deterministic) {
    uint64_t need = 0;
    const int rc = tsb_backward_det_scratch_size(scene->num_splats, atlas->resolution,
                                                 grads->texel_layout, &need);
    if (rc != TSB_OK) return rc;
    if (!det_scratch || det_scratch_bytes < need) {
      set_error("tsb_render_backward: deterministic mode needs tsb_backward_det_scratch_size "
                "bytes of det_scratch");
      return TSB_ERR_CAPACITY;
    }
  }
  if (!atlas->family_a || !atlas->family_b || !atlas->entries) {
    set_error("gradients require the per-primitive (linear atlas) texture path");
    return TSB_ERR_VALUE;
  }
  const int32_t P = scene->num_splats;
  WsLayout L;
  if (!ws_layout(P, camera->width, camera->height, tile, cap, &L)) {
    set_error("tsb_render_backward: invalid size/tile arguments");
    return TSB_ERR_VALUE;
  }
  if (ws_bytes < L.total) {
    set_error("tsb_render_backward: workspace too small");
    return TSB_ERR_CAPACITY;
  }
  if (P == 0) return TSB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  float* acc = static_cast<float*>(scratch);
  TSB_CUDA(cudaMemsetAsync(acc, 0, (size_t)P * kAccWords * sizeof(float), st));
  RasterBwdParams rp;
  rp.cam = to_cam(camera);
  rp.W = camera->width; rp.H = camera->height; rp.tiles_x = L.tiles_x; rp.tile = tile;
  rp.near_f = (float)camera->near_z;
  rp.ranges = ws_ptr<int32_t>(ws, L.ranges);
  rp.evals = ws_ptr<int32_t>(ws, L.evals_out);
  rp.geom = ws_ptr<GeomRec>(ws, L.geom);
  rp.mat = ws_ptr<MatRec>(ws, L.mat);
  rp.m64 = ws_ptr<double>(ws, L.m64);
  rp.T = atlas->resolution; rp.page_w = atlas->page_w;
  rp.tstride = atlas->texel_stride > 0 ? atlas->texel_stride : 1;
  rp.fam_a = reinterpret_cast<const float4*>(atlas->family_a);
  rp.fam_b = reinterpret_cast<const float4*>(atlas->family_b);
  rp.last_entry = px->last_entry;
  rp.T_last = px->T_last;
  rp.dgbuf = dgbuf;
  rp.acc = acc;
  rp.dtexels = grads->texels;
  rp.tl = grads->texel_layout == TSB_TEXELS_INTERLEAVED ? 8 : 7;
  const int64_t n_acc = (int64_t)P * kAccWords;
  const int64_t n_tex = (int64_t)P * atlas->resolution * atlas->resolution * rp.tl;
  rp.red_count = nullptr;
  if (g_count_red_host) TSB_CUDA(cudaGetSymbolAddress((void**)&rp.red_count, g_red_count));
  rp.acc64 = deterministic ? static_cast<unsigned long long*>(det_scratch) : nullptr;
  rp.tex64 = deterministic ? rp.acc64 + n_acc : nullptr;
  if (deterministic)
    TSB_CUDA(cudaMemsetAsync(det_scratch, 0, (size_t)(n_acc + n_tex) * 8, st));
  rp.num_tiles = L.num_tiles;
  rp.work_counter = reinterpret_cast<int32_t*>(const_cast<int64_t*>(ws_ptr<int64_t>(ws, L.counters)) + 2);
  rp.tile_order = ws_ptr<int32_t>(ws, L.torder_out);
  TSB_CUDA(cudaMemsetAsync(rp.work_counter, 0, 4, st));
  const size_t smem = 8 * sizeof(BwdWarpSmem);
  static PerDevice s_resident;  // per device: attributes set, persistent grid size
  int resident = 0;
  TSB_CUDA(s_resident.get(
      [smem](int dev) {
        int sms = 0, per_sm = 0;
        cudaError_t e = cudaFuncSetAttribute(k_raster_bwd<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(k_raster_bwd<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
          e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster_bwd<false>, 256,
                                                            smem);
        return e == cudaSuccess ? sms * (per_sm > 0 ? per_sm : 1) : -(int)e;
      },
      &resident));
  const int units = L.num_tiles * (tile * tile / 32);
  const int grid = std::min((units + 7) / 8, resident);
  if (deterministic) {
    k_raster_bwd<true><<<grid, 256, smem, st>>>(rp);
    TSB_CHECK_LAUNCH("k_raster_bwd<det>");
    k_det_unfix<<<1184, 256, 0, st>>>(n_acc, rp.acc64, acc, n_tex, rp.tex64, rp.dtexels);
    TSB_CHECK_LAUNCH("k_det_unfix");
  } else {
    k_raster_bwd<false><<<grid, 256, smem, st>>>(rp);
    TSB_CHECK_LAUNCH("k_raster_bwd");
  }
  FinishParams fp;
  fp.cam = to_cam(camera);
  fp.P = P; fp.sh_degree = scene->sh_degree;
  fp.pos = scene->positions; fp.tu = scene->tangent_u; fp.tv = scene->tangent_v;
  fp.sc = scene->scales; fp.sh = scene->sh; fp.acc = acc;
  fp.g_pos = grads->positions; fp.g_tu = grads->tangent_u; fp.g_tv = grads->tangent_v;
  fp.g_sc = grads->scales; fp.g_op = grads->opacities; fp.g_sh = grads->sh;
  k_finish_grads<<<(P + 127) / 128, 128, 0, st>>>(fp);
  TSB_CHECK_LAUNCH("k_finish_grads");
  return TSB_OK;
}

}  // extern "C"
