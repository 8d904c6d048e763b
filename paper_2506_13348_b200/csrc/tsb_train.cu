// tsb_train.cu — training-step glue for sm_100a: image loss, regularisers,
// fused Adam and the tangent-frame projection.
//
//   K10 image loss      display transform (losses.py:24-37), L1 and D-SSIM
//                       with the 11-tap separable Gaussian (losses.py:48-134)
//                       and their adjoints (ssim_backward :103-117,
//                       linear_to_display_grad :31-37): four passes
//                       (horizontal / vertical blur of the five SSIM moments,
//                       then of the three moment adjoints).
//   K11 regularisers    normal consistency against depth-derived normals and
//                       edge-aware normal smoothness (losses.py:147-277) with
//                       the compute_step chain into the G-buffer
//                       (training.py:152-172): a counting pass and a gradient
//                       pass (the means need the global valid counts).
//   K12 Adam            one launch over every parameter group
//                       (training.py:69-100), with the step's projections
//                       (opacity clip, scale floor, texel clip).
//   K13 tangents        Gram-Schmidt re-orthonormalisation (splats.py:382-392).
//
// Sums are accumulated in fp64 (device atomics); per-pixel math is fp32.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "tsb_internal.cuh"

namespace tsb {

namespace {

constexpr int kR = 5;  // SSIM window radius (11 taps, sigma 1.5)
__constant__ float c_win[2 * kR + 1];
constexpr float kDisplayToe = 1e-4f;
constexpr float kGammaInv = (float)(1.0 / 2.2);
constexpr float kSsimC1 = 0.01f * 0.01f;
constexpr float kSsimC2 = 0.03f * 0.03f;

__device__ __forceinline__ float display_of(float x) {
  x = fmaxf(x, 0.0f);
  const float toe_slope = powf(kDisplayToe, kGammaInv - 1.0f);
  return x >= kDisplayToe ? powf(fmaxf(x, kDisplayToe), kGammaInv) : toe_slope * x;
}

__device__ __forceinline__ float display_slope(float x) {
  const float toe_slope = powf(kDisplayToe, kGammaInv - 1.0f);
  float s = x >= kDisplayToe ? kGammaInv * powf(fmaxf(x, kDisplayToe), kGammaInv - 1.0f)
                             : toe_slope;
  return x < 0.0f ? 0.0f : s;
}

// Block-wide sums of K values (blockDim 256), one fp64 atomic per value per
// block (blocks cover several image rows, so a frame issues a few hundred).
template <int K>
__device__ __forceinline__ void block_sums_atomic(double (&v)[K], double* dst) {
  __shared__ double s_part[8][K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_part[warp][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w][threadIdx.x];
    if (t != 0.0) atomicAdd(dst + threadIdx.x, t);
  }
}

constexpr int kRowsPerBlock = 2;

// ---- K10 pass 1: display images, L1 / MSE sums, horizontal blur of the
// five SSIM moments (a, b, a^2, b^2, ab) per channel -> m5[15][H][W].
__global__ void __launch_bounds__(256) k_ssim_pass1(int W, int H, const float* __restrict__ color,
                                                    const float* __restrict__ target,
                                                    float* __restrict__ m5,
                                                    double* __restrict__ terms) {
  __shared__ float sa[3][256 + 2 * kR], sb[3][256 + 2 * kR];
  const int x0 = blockIdx.x * 256;
  const int x = x0 + threadIdx.x;
  const size_t HW = (size_t)W * H;
  double acc[3] = {0.0, 0.0, 0.0};  // L1, (SSIM: pass 2), squared error
  const int y1 = min(H, (int)(blockIdx.y + 1) * kRowsPerBlock);
  for (int y = blockIdx.y * kRowsPerBlock; y < y1; ++y) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256 + 2 * kR; i += 256) {
      const int xx = x0 - kR + i;
      const bool ok = xx >= 0 && xx < W;
      for (int c = 0; c < 3; ++c) {
        const size_t o = 3 * ((size_t)y * W + xx) + c;
        sa[c][i] = ok ? display_of(color[o]) : 0.0f;
        sb[c][i] = ok ? target[o] : 0.0f;
      }
    }
    __syncthreads();
    if (x < W) {
      const size_t pix = (size_t)y * W + x;
      for (int c = 0; c < 3; ++c) {
        const float a = sa[c][threadIdx.x + kR], b = sb[c][threadIdx.x + kR];
        acc[0] += fabsf(a - b);
        const float d = fminf(fmaxf(a, 0.f), 1.f) - fminf(fmaxf(b, 0.f), 1.f);
        acc[2] += d * d;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
        for (int t = 0; t <= 2 * kR; ++t) {
          const float w = c_win[t], av = sa[c][threadIdx.x + t], bv = sb[c][threadIdx.x + t];
          s0 += w * av;
          s1 += w * bv;
          s2 += w * av * av;
          s3 += w * bv * bv;
          s4 += w * av * bv;
        }
        float* o = m5 + (size_t)(5 * c) * HW + pix;
        o[0] = s0; o[HW] = s1; o[2 * HW] = s2; o[3 * HW] = s3; o[4 * HW] = s4;
      }
    }
  }
  block_sums_atomic(acc, terms);
}

// Vertical 11-tap blur of NP planes over a TX x TY tile staged in shared
// memory (rows [y0-5, y0+TY+5) of 32 columns): every input value is read
// from global once (+ the halo), taps come from conflict-free smem.
constexpr int kTX = 32, kTY = 48, kTR = kTY + 2 * kR;

template <int NP>
__device__ __forceinline__ void stage_vtile(float (*tile)[kTR][kTX + 1], const float* __restrict__ src,
                                            size_t HW, int W, int H, int x0, int y0) {
  for (int i = threadIdx.x; i < NP * kTR * kTX; i += blockDim.x) {
    const int pl = i / (kTR * kTX), r = (i / kTX) % kTR, cx = i % kTX;
    const int yy = y0 - kR + r, xx = x0 + cx;
    tile[pl][r][cx] = (yy >= 0 && yy < H && xx < W) ? src[pl * HW + (size_t)yy * W + xx] : 0.0f;
  }
}

// ---- K10 pass 2: vertical blur of the moments, SSIM map, its sum and the
// per-pixel moment adjoints (ssim_backward): part[9][H][W] =
// (g_mu_a, g_saa, g_sab) per channel, already scaled by upstream / N.
__global__ void __launch_bounds__(256) k_ssim_pass2(int W, int H, const float* __restrict__ m5,
                                                    float* __restrict__ part, float g,
                                                    double* __restrict__ terms) {
  __shared__ float tile[5][kTR][kTX + 1];
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x = x0 + tx;
  const size_t HW = (size_t)W * H;
  double msum[1] = {0.0};
  {
    const int c = blockIdx.z;  // one colour channel per CTA layer
    stage_vtile<5>(tile, m5 + (size_t)(5 * c) * HW, HW, W, H, x0, y0);
    __syncthreads();
    for (int r = ty; r < kTY; r += 8) {
      const int y = y0 + r;
      if (y >= H || x >= W) continue;
      float mom[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t <= 2 * kR; ++t) {
        const float w = c_win[t];
#pragma unroll
        for (int k = 0; k < 5; ++k) mom[k] += w * tile[k][r + t][tx];
      }
      const float mu_a = mom[0], mu_b = mom[1];
      const float saa = mom[2] - mu_a * mu_a, sbb = mom[3] - mu_b * mu_b;
      const float sab = mom[4] - mu_a * mu_b;
      const float p = 2.0f * mu_a * mu_b + kSsimC1, q = 2.0f * sab + kSsimC2;
      const float rr = mu_a * mu_a + mu_b * mu_b + kSsimC1, ss = saa + sbb + kSsimC2;
      const float m = (p * q) / (rr * ss);
      msum[0] += m;
      const float rs = rr * ss;
      const float g_p = g * q / rs, g_q = g * p / rs;
      const float g_r = -g * m / rr, g_s = -g * m / ss;
      const float g_sab = 2.0f * g_q, g_saa = g_s;
      const float g_mu_a = 2.0f * mu_b * g_p + 2.0f * mu_a * g_r - mu_b * g_sab - 2.0f * mu_a * g_saa;
      float* o = part + (size_t)(3 * c) * HW + (size_t)y * W + x;
      o[0] = g_mu_a; o[HW] = g_saa; o[2 * HW] = g_sab;
    }
  }
  block_sums_atomic(msum, terms + 1);
}

// ---- K10 passes 3+4 fused: the horizontal blur of the three adjoint planes
// of one channel goes to shared memory (rows with a 5-row halo) and the
// vertical blur reads it there, so the blurred planes never go through HBM.
// Same sums in the same order as separate passes (zero padding outside).
constexpr int kFTY = 32, kFR = kFTY + 2 * kR, kFX = 32, kFC = kFX + 2 * kR;
__global__ void __launch_bounds__(256) k_ssim_pass34(int W, int H, const float* __restrict__ part,
                                                     const float* __restrict__ color,
                                                     const float* __restrict__ target,
                                                     float l1_scale, float* __restrict__ dcolor) {
  __shared__ float raw[3][kFR][kFC + 1];
  __shared__ float hbt[3][kFR][kFX + 1];
  const int x0 = blockIdx.x * kFX, y0 = blockIdx.y * kFTY, c = blockIdx.z;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const size_t HW = (size_t)W * H;
  for (int i = threadIdx.x; i < 3 * kFR * kFC; i += blockDim.x) {
    const int pl = i / (kFR * kFC), r = (i / kFC) % kFR, cx = i % kFC;
    const int yy = y0 - kR + r, xx = x0 - kR + cx;
    raw[pl][r][cx] = (yy >= 0 && yy < H && xx >= 0 && xx < W)
                         ? part[(size_t)(3 * c + pl) * HW + (size_t)yy * W + xx] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * kFR * kFX; i += blockDim.x) {
    const int pl = i / (kFR * kFX), r = (i / kFX) % kFR, cx = i % kFX;
    float h = 0.f;
#pragma unroll
    for (int t = 0; t <= 2 * kR; ++t) h += c_win[t] * raw[pl][r][cx + t];
    const int yy = y0 - kR + r;
    hbt[pl][r][cx] = (yy >= 0 && yy < H) ? h : 0.0f;
  }
  __syncthreads();
  const int x = x0 + tx;
  for (int r = ty; r < kFTY; r += 8) {
    const int y = y0 + r;
    if (y >= H || x >= W) continue;
    float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t <= 2 * kR; ++t) {
      const float w = c_win[t];
      v[0] += w * hbt[0][r + t][tx];
      v[1] += w * hbt[1][r + t][tx];
      v[2] += w * hbt[2][r + t][tx];
    }
    const size_t pix = (size_t)y * W + x;
    const float cx = color[3 * pix + c];
    const float a = display_of(cx), b = target[3 * pix + c];
    const float d = a - b;
    const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    const float dpred = l1_scale * sg + v[0] + 2.0f * a * v[1] + b * v[2];
    dcolor[3 * pix + c] = dpred * display_slope(cx);
  }
}

// ---- K11 regularisers ------------------------------------------------------
struct RegParams {
  int W, H;
  double fx, fy, cx, cy;
  float R[9];          // camera rotation (world_to_view[:3,:3]), row-major
  const float* gbuf;   // 13 x H x W
  const float* target; // H x W x 3 display
  float* dgbuf;        // 13 x H x W (accumulated)
  double* terms;       // [3] normal sum, [4] normal count, [5] smooth sum, [6] smooth count
  float w_normal, w_smooth;
};

constexpr float kCoverAlpha = 0.5f;

struct PixReg {
  bool cover, n_ok;
  float zbar, a_safe;
  float P[3];     // back-projected view-space point
  float n[3];     // unit normal image
  float mag;      // |blended normal|
};

__device__ __forceinline__ PixReg reg_pixel(const RegParams& p, int x, int y) {
  PixReg r;
  const size_t HW = (size_t)p.W * p.H, pix = (size_t)y * p.W + x;
  const float alpha = p.gbuf[12 * HW + pix];
  r.cover = alpha > kCoverAlpha;
  r.a_safe = fmaxf(alpha, 1e-30f);
  r.zbar = r.cover ? p.gbuf[11 * HW + pix] / r.a_safe : 0.0f;
  const float xs = (float)((((double)x + 0.5) - p.cx) / p.fx);
  const float ys = (float)((((double)y + 0.5) - p.cy) / p.fy);
  r.P[0] = xs * r.zbar; r.P[1] = ys * r.zbar; r.P[2] = r.zbar;
  const float nb0 = p.gbuf[5 * HW + pix], nb1 = p.gbuf[6 * HW + pix], nb2 = p.gbuf[7 * HW + pix];
  r.mag = sqrtf(nb0 * nb0 + nb1 * nb1 + nb2 * nb2);
  r.n_ok = r.mag > 1e-12f;
  const float im = 1.0f / fmaxf(r.mag, 1e-30f);
  r.n[0] = r.n_ok ? nb0 * im : 0.f;
  r.n[1] = r.n_ok ? nb1 * im : 0.f;
  r.n[2] = r.n_ok ? nb2 * im : 0.f;
  return r;
}

__device__ __forceinline__ void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// Depth-derived normal at q (depth_to_normal, losses.py:147-180): needs q,
// q+x, q+y. Fills the view-space quantities the adjoint reuses.
struct DepthNrm {
  bool ok;
  float dx[3], dy[3];
  float unit_v[3];   // oriented unit view normal (0 if !ok)
  float mag;
  bool flip;
  float n_world[3];
};

__device__ __forceinline__ DepthNrm depth_normal(const RegParams& p, const PixReg& q,
                                                 const PixReg& qx, const PixReg& qy, bool interior) {
  DepthNrm d;
  float nv[3] = {0.f, 0.f, 0.f};
  for (int i = 0; i < 3; ++i) { d.dx[i] = 0.f; d.dy[i] = 0.f; }
  bool valid = false;
  if (interior) {
    for (int i = 0; i < 3; ++i) {
      d.dx[i] = qx.P[i] - q.P[i];
      d.dy[i] = qy.P[i] - q.P[i];
    }
    cross3(d.dx, d.dy, nv);
    valid = q.cover && qx.cover && qy.cover;
  }
  d.flip = (nv[0] * q.P[0] + nv[1] * q.P[1] + nv[2] * q.P[2]) > 0.0f;
  if (d.flip) { nv[0] = -nv[0]; nv[1] = -nv[1]; nv[2] = -nv[2]; }
  d.mag = sqrtf(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
  d.ok = valid && d.mag > 1e-12f;
  const float im = 1.0f / fmaxf(d.mag, 1e-30f);
  for (int i = 0; i < 3; ++i) d.unit_v[i] = d.ok ? nv[i] * im : 0.f;
  // n_world = unit_v @ R  (row vector times the rotation)
  for (int j = 0; j < 3; ++j)
    d.n_world[j] = d.unit_v[0] * p.R[0 * 3 + j] + d.unit_v[1] * p.R[1 * 3 + j] +
                   d.unit_v[2] * p.R[2 * 3 + j];
  return d;
}

__device__ __forceinline__ PixReg reg_pixel_or_empty(const RegParams& p, int x, int y) {
  if (x >= 0 && x < p.W && y >= 0 && y < p.H) return reg_pixel(p, x, y);
  PixReg r;
  r.cover = false; r.n_ok = false; r.zbar = 0.f; r.a_safe = 1e-30f; r.mag = 0.f;
  for (int i = 0; i < 3; ++i) { r.P[i] = 0.f; r.n[i] = 0.f; }
  return r;
}

__device__ __forceinline__ float tgt_diff_norm(const RegParams& p, int x0, int y0, int x1, int y1) {
  const float* a = p.target + 3 * ((size_t)y0 * p.W + x0);
  const float* b = p.target + 3 * ((size_t)y1 * p.W + x1);
  const float d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
  return sqrtf(d0 * d0 + d1 * d1 + d2 * d2);
}

// Smoothness pair term (q, q+e): weight, difference and its norm; valid
// when both pixels have a covered unit normal.
struct SmoothPair {
  bool v;
  float w, m;
  float d[3];
};

__device__ __forceinline__ SmoothPair smooth_pair(const RegParams& p, const PixReg& a,
                                                  const PixReg& b, int xa, int ya, int xb, int yb) {
  SmoothPair s;
  s.v = (a.n_ok && a.cover) && (b.n_ok && b.cover);
  for (int i = 0; i < 3; ++i) s.d[i] = b.n[i] - a.n[i];
  s.m = sqrtf(s.d[0] * s.d[0] + s.d[1] * s.d[1] + s.d[2] * s.d[2]);
  s.w = s.v ? expf(-tgt_diff_norm(p, xa, ya, xb, yb)) : 0.0f;
  return s;
}

// Pass A: loss sums and the valid counts.
__global__ void __launch_bounds__(256) k_reg_count(RegParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // normal sum, normal count, smooth sum, smooth count
  const int y1 = min(p.H, (int)(blockIdx.y + 1) * kRowsPerBlock);
  for (int y = blockIdx.y * kRowsPerBlock; y < y1 && x < p.W; ++y) {
    const PixReg q = reg_pixel(p, x, y);
    const bool has_x = x + 1 < p.W, has_y = y + 1 < p.H;
    const PixReg qx = reg_pixel_or_empty(p, x + 1, y);
    const PixReg qy = reg_pixel_or_empty(p, x, y + 1);
    if (p.w_normal > 0.0f) {
      const DepthNrm d = depth_normal(p, q, qx, qy, has_x && has_y);
      const bool valid = q.n_ok && d.ok && q.cover;
      if (valid) {
        acc[0] += 1.0 - (double)(q.n[0] * d.n_world[0] + q.n[1] * d.n_world[1] + q.n[2] * d.n_world[2]);
        acc[1] += 1.0;
      }
    }
    if (p.w_smooth > 0.0f) {
      if (has_x) {
        const SmoothPair s = smooth_pair(p, q, qx, x, y, x + 1, y);
        if (s.v) { acc[2] += (double)(s.w * s.m); acc[3] += 1.0; }
      }
      if (has_y) {
        const SmoothPair s = smooth_pair(p, q, qy, x, y, x, y + 1);
        if (s.v) { acc[2] += (double)(s.w * s.m); acc[3] += 1.0; }
      }
    }
  }
  block_sums_atomic(acc, p.terms + 3);
}

// G(q) of depth_to_normal_backward: the oriented view-normal adjoint of the
// normal-consistency term at q (0 outside [0,W-2] x [0,H-2] or invalid).
__device__ __forceinline__ void depth_adjoint_at(const RegParams& p, int x, int y, float scale_n,
                                                 float* G, float* dx, float* dy) {
  for (int i = 0; i < 3; ++i) { G[i] = 0.f; dx[i] = 0.f; dy[i] = 0.f; }
  if (x < 0 || y < 0 || x + 1 >= p.W || y + 1 >= p.H) return;
  const PixReg q = reg_pixel(p, x, y), qx = reg_pixel(p, x + 1, y), qy = reg_pixel(p, x, y + 1);
  const DepthNrm d = depth_normal(p, q, qx, qy, true);
  for (int i = 0; i < 3; ++i) { dx[i] = d.dx[i]; dy[i] = d.dy[i]; }
  const bool valid = q.n_ok && d.ok && q.cover;
  // upstream on n_ref: w_normal * (-1/n) * n_img; up_v = upstream @ R^T
  float upv[3];
  for (int i = 0; i < 3; ++i)
    upv[i] = -scale_n * (q.n[0] * p.R[i * 3 + 0] + q.n[1] * p.R[i * 3 + 1] + q.n[2] * p.R[i * 3 + 2]);
  const float dot = d.unit_v[0] * upv[0] + d.unit_v[1] * upv[1] + d.unit_v[2] * upv[2];
  const float im = 1.0f / fmaxf(d.mag, 1e-30f);
  for (int i = 0; i < 3; ++i) {
    const float g = (upv[i] - d.unit_v[i] * dot) * im;
    G[i] = valid ? (d.flip ? -g : g) : 0.0f;
  }
}

// smoothness adjoint of pair (q, q+e): gx = w/m * d / count (0 if m <= 1e-12)
__device__ __forceinline__ void smooth_adjoint(const RegParams& p, int xa, int ya, int xb, int yb,
                                               float inv_count, float* g) {
  g[0] = g[1] = g[2] = 0.f;
  if (xa < 0 || ya < 0 || xb >= p.W || yb >= p.H) return;
  const PixReg a = reg_pixel(p, xa, ya), b = reg_pixel(p, xb, yb);
  const SmoothPair s = smooth_pair(p, a, b, xa, ya, xb, yb);
  if (!(s.v && s.m > 1e-12f)) return;
  const float f = s.w / fmaxf(s.m, 1e-30f) * inv_count;
  for (int i = 0; i < 3; ++i) g[i] = f * s.d[i];
}

// Pass B: gradients into the G-buffer (normal channels 5..7, depth 11,
// alpha 12), compute_step's chain (training.py:152-172).
__global__ void __launch_bounds__(256) k_reg_grad(RegParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= p.W) return;
  const double ncnt = fmax(p.terms[4], 1.0), scnt = fmax(p.terms[6], 1.0);
  const float scale_n = (float)(1.0 / ncnt) * p.w_normal;  // w_normal / n
  const float inv_s = (float)(1.0 / scnt);
  const size_t HW = (size_t)p.W * p.H, pix = (size_t)y * p.W + x;
  const PixReg q = reg_pixel(p, x, y);
  float dn[3] = {0.f, 0.f, 0.f};
  if (p.w_normal > 0.0f) {
    // d/dn_img of the consistency term: -(w/n) n_ref on valid pixels
    if (x + 1 < p.W && y + 1 < p.H) {
      const PixReg qx = reg_pixel(p, x + 1, y), qy = reg_pixel(p, x, y + 1);
      const DepthNrm d = depth_normal(p, q, qx, qy, true);
      if (q.n_ok && d.ok && q.cover)
        for (int i = 0; i < 3; ++i) dn[i] += -scale_n * d.n_world[i];
    }
    // depth adjoint: dpx(p) = ddx(p-x) - ddx(p) + ddy(p-y) - ddy(p)
    float G[3], dx[3], dy[3], t[3], dpx[3] = {0.f, 0.f, 0.f};
    depth_adjoint_at(p, x, y, scale_n, G, dx, dy);
    cross3(dy, G, t);                      // ddx(p)
    for (int i = 0; i < 3; ++i) dpx[i] -= t[i];
    cross3(G, dx, t);                      // ddy(p)
    for (int i = 0; i < 3; ++i) dpx[i] -= t[i];
    depth_adjoint_at(p, x - 1, y, scale_n, G, dx, dy);
    cross3(dy, G, t);                      // ddx(p - x)
    for (int i = 0; i < 3; ++i) dpx[i] += t[i];
    depth_adjoint_at(p, x, y - 1, scale_n, G, dx, dy);
    cross3(G, dx, t);                      // ddy(p - y)
    for (int i = 0; i < 3; ++i) dpx[i] += t[i];
    const float xs = (float)((((double)x + 0.5) - p.cx) / p.fx);
    const float ys = (float)((((double)y + 0.5) - p.cy) / p.fy);
    const float dd = dpx[0] * xs + dpx[1] * ys + dpx[2];
    if (q.cover) {
      p.dgbuf[11 * HW + pix] += dd / q.a_safe;
      p.dgbuf[12 * HW + pix] -= dd * q.zbar / q.a_safe;
    }
  }
  if (p.w_smooth > 0.0f) {
    float g[3];
    const float ws = p.w_smooth;
    smooth_adjoint(p, x - 1, y, x, y, inv_s, g);   // gx(p - x): +
    for (int i = 0; i < 3; ++i) dn[i] += ws * g[i];
    smooth_adjoint(p, x, y, x + 1, y, inv_s, g);   // gx(p): -
    for (int i = 0; i < 3; ++i) dn[i] -= ws * g[i];
    smooth_adjoint(p, x, y - 1, x, y, inv_s, g);   // gy(p - y): +
    for (int i = 0; i < 3; ++i) dn[i] += ws * g[i];
    smooth_adjoint(p, x, y, x, y + 1, inv_s, g);   // gy(p): -
    for (int i = 0; i < 3; ++i) dn[i] -= ws * g[i];
  }
  // _normal_image_backward (training.py:121-126)
  if (q.n_ok) {
    const float dot = q.n[0] * dn[0] + q.n[1] * dn[1] + q.n[2] * dn[2];
    const float im = 1.0f / fmaxf(q.mag, 1e-30f);
    for (int i = 0; i < 3; ++i) p.dgbuf[(5 + i) * HW + pix] += (dn[i] - q.n[i] * dot) * im;
  }
}

// ---- K12 Adam over every parameter group in one launch ---------------------
constexpr int kAdamChunk = 256 * 8;  // elements per block

struct AdamLaunch {
  tsb_adam_group g[TSB_ADAM_MAX_GROUPS];
  int32_t blk_start[TSB_ADAM_MAX_GROUPS + 1];  // first block of each group
  int32_t n;
  double b1, b2, eps;
  double bc1, bc2;  // 1 - beta^t
  const int32_t* halt;  // optional: skip the update when *halt != 0 (divergence guard)
};

template <typename TP>
__device__ __forceinline__ void adam_chunk(const AdamLaunch& A, const tsb_adam_group& g,
                                           int64_t base) {
  TP* prm = static_cast<TP*>(g.param);
  TP* m = static_cast<TP*>(g.m);
  TP* v = static_cast<TP*>(g.v);
  const TP b1 = (TP)A.b1, b2 = (TP)A.b2, c1 = (TP)(1.0 - A.b1), c2 = (TP)(1.0 - A.b2);
  const TP ibc1 = (TP)(1.0 / A.bc1), ibc2 = (TP)(1.0 / A.bc2), lr = (TP)g.lr, eps = (TP)A.eps;
#pragma unroll 4
  for (int j = 0; j < kAdamChunk / 256; ++j) {
    const int64_t i = base + j * 256 + threadIdx.x;
    if (i >= g.count) break;
    const TP gr = (TP)__ldg(g.grad + i);
    const TP mi = b1 * m[i] + c1 * gr;
    const TP vi = b2 * v[i] + c2 * gr * gr;
    m[i] = mi;
    v[i] = vi;
    TP x = prm[i] - lr * (mi * ibc1) / (sqrt(vi * ibc2) + eps);
    if (g.clamp == TSB_CLAMP_UNIT) x = x < (TP)0 ? (TP)0 : (x > (TP)1 ? (TP)1 : x);
    else if (g.clamp == TSB_CLAMP_FLOOR) x = x < (TP)g.floor ? (TP)g.floor : x;
    prm[i] = x;
  }
}

__device__ __forceinline__ float adam_f(float p, float gr, float& m, float& v, float b1, float b2,
                                        float c1, float c2, float ibc1, float ibc2, float lr,
                                        float eps, const tsb_adam_group& g) {
  m = b1 * m + c1 * gr;
  v = b2 * v + c2 * gr * gr;
  float x = p - lr * (m * ibc1) / (sqrtf(v * ibc2) + eps);
  if (g.clamp == TSB_CLAMP_UNIT) x = fminf(fmaxf(x, 0.f), 1.f);
  else if (g.clamp == TSB_CLAMP_FLOOR) x = fmaxf(x, (float)g.floor);
  return x;
}

// float32 groups with 16-B aligned, multiple-of-4 arrays: 128-bit accesses
__device__ __forceinline__ void adam_chunk_f4(const AdamLaunch& A, const tsb_adam_group& g,
                                              int64_t base) {
  float4* prm = static_cast<float4*>(g.param);
  float4* m4 = static_cast<float4*>(g.m);
  float4* v4 = static_cast<float4*>(g.v);
  const float4* g4 = reinterpret_cast<const float4*>(g.grad);
  const float b1 = (float)A.b1, b2 = (float)A.b2, c1 = (float)(1.0 - A.b1), c2 = (float)(1.0 - A.b2);
  const float ibc1 = (float)(1.0 / A.bc1), ibc2 = (float)(1.0 / A.bc2), lr = (float)g.lr;
  const float eps = (float)A.eps;
  const int64_t n4 = g.count / 4;
#pragma unroll 2
  for (int j = 0; j < kAdamChunk / 1024; ++j) {
    const int64_t i = base / 4 + j * 256 + threadIdx.x;
    if (i >= n4) break;
    const float4 gr = __ldg(g4 + i);
    float4 p = prm[i], m = m4[i], v = v4[i];
    p.x = adam_f(p.x, gr.x, m.x, v.x, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
    p.y = adam_f(p.y, gr.y, m.y, v.y, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
    p.z = adam_f(p.z, gr.z, m.z, v.z, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
    p.w = adam_f(p.w, gr.w, m.w, v.w, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
    prm[i] = p; m4[i] = m; v4[i] = v;
  }
}

// One block = one contiguous chunk of one group (coalesced, no per-element
// group search).
// Texels as parameters in the 8-channel interleaved atlas order (what the
// verify-mode forward reads) with gradients in the 7-channel combined order
// (what K8 writes with TSB_TEXELS_COMBINED, and what the all-reduce carries:
// no always-zero 8th channel on the wire). Slot -> combined channel; the pad
// slot 7 stays untouched.
__device__ __forceinline__ void adam_chunk_tex87(const AdamLaunch& A, const tsb_adam_group& g,
                                                 int64_t base) {
  // one texel (8 parameter slots, 7 gradients) per thread: 128-bit parameter
  // and moment accesses (the group's arrays are 32-B aligned per texel)
  float4* prm = static_cast<float4*>(g.param);
  float4* m4 = static_cast<float4*>(g.m);
  float4* v4 = static_cast<float4*>(g.v);
  const float b1 = (float)A.b1, b2 = (float)A.b2, c1 = (float)(1.0 - A.b1), c2 = (float)(1.0 - A.b2);
  const float ibc1 = (float)(1.0 / A.bc1), ibc2 = (float)(1.0 / A.bc2), lr = (float)g.lr;
  const float eps = (float)A.eps;
  const int64_t q = base / 8 + threadIdx.x;  // texel
  if (q >= g.count / 8) return;
  const float* gr = g.grad + q * 7;  // combined: alb rgb, rough, metal, nrm a, nrm b
  float4 p0 = prm[2 * q], p1 = prm[2 * q + 1];
  float4 ma = m4[2 * q], mb = m4[2 * q + 1];
  float4 va = v4[2 * q], vb = v4[2 * q + 1];
  // slots: p0 = (alb r, g, b, rough), p1 = (nrm a, nrm b, metal, pad)
  p0.x = adam_f(p0.x, __ldg(gr + 0), ma.x, va.x, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p0.y = adam_f(p0.y, __ldg(gr + 1), ma.y, va.y, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p0.z = adam_f(p0.z, __ldg(gr + 2), ma.z, va.z, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p0.w = adam_f(p0.w, __ldg(gr + 3), ma.w, va.w, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p1.x = adam_f(p1.x, __ldg(gr + 5), mb.x, vb.x, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p1.y = adam_f(p1.y, __ldg(gr + 6), mb.y, vb.y, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  p1.z = adam_f(p1.z, __ldg(gr + 4), mb.z, vb.z, b1, b2, c1, c2, ibc1, ibc2, lr, eps, g);
  prm[2 * q] = p0; prm[2 * q + 1] = p1;
  m4[2 * q] = ma; m4[2 * q + 1] = mb;
  v4[2 * q] = va; v4[2 * q + 1] = vb;
}

__global__ void __launch_bounds__(256) k_adam(AdamLaunch A) {
  if (A.halt && *A.halt) return;
  int k = 0;
  while (k + 1 < A.n && A.blk_start[k + 1] <= (int)blockIdx.x) ++k;
  const tsb_adam_group& g = A.g[k];
  const int64_t base = (int64_t)(blockIdx.x - A.blk_start[k]) * kAdamChunk;
  if (g.dtype == TSB_F32_TEX87) {
    adam_chunk_tex87(A, g, base);
  } else if (g.dtype == TSB_F64) {
    adam_chunk<double>(A, g, base);
  } else if ((g.count & 3) == 0 && ((reinterpret_cast<uintptr_t>(g.param) |
                                     reinterpret_cast<uintptr_t>(g.m) |
                                     reinterpret_cast<uintptr_t>(g.v) |
                                     reinterpret_cast<uintptr_t>(g.grad)) & 15) == 0) {
    adam_chunk_f4(A, g, base);
  } else {
    adam_chunk<float>(A, g, base);
  }
}

// ---- K13 tangent frames ------------------------------------------------------
__global__ void k_orthonormalize(int32_t P, double* __restrict__ tu, double* __restrict__ tv,
                                 const int32_t* __restrict__ halt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P || (halt && *halt)) return;
  double u[3], v[3];
  for (int k = 0; k < 3; ++k) { u[k] = tu[3 * i + k]; v[k] = tv[3 * i + k]; }
  const double nu = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  for (int k = 0; k < 3; ++k) u[k] /= nu;
  const double d = u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
  for (int k = 0; k < 3; ++k) v[k] = v[k] - d * u[k];
  const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  for (int k = 0; k < 3; ++k) { tu[3 * i + k] = u[k]; tv[3 * i + k] = v[k] / nv; }
}

// ---- train loop glue (train(), training.py:224-322) ------------------------
// Divergence guard (training.py:263-265): halt = 1 once any loss term of a
// step is non-finite; the guarded Adam / orthonormalisation then skip, so the
// parameters stay those of the iteration that diverged (the reference raises
// before updating) while the host reads the flag at its next sync.
__global__ void k_guard_finite(const double* __restrict__ terms, int32_t n,
                               int32_t* __restrict__ halt) {
  const int i = threadIdx.x;
  if (i < n && !isfinite(terms[i])) *halt = 1;
}

// Stage-2 texel broadcast (broadcast_textures, training.py:201-221): charts of
// T0 x T0 texels grow to T x T by repeating each texel T/T0 times per axis,
// or (T not a multiple of T0) by repeating texel (0, 0). 8-channel layout.
__global__ void k_broadcast_texels(int64_t P, int32_t T0, int32_t T, const float4* __restrict__ src,
                                   float4* __restrict__ dst) {
  const int64_t n = P * T * T;
  const bool even = T % T0 == 0;
  const int reps = even ? T / T0 : 1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = q / ((int64_t)T * T);
    const int r = (int)(q % ((int64_t)T * T));
    const int j = r / T, i = r % T;
    const int64_t s = even ? p * T0 * T0 + (int64_t)(j / reps) * T0 + i / reps : p * T0 * T0;
    dst[2 * q] = src[2 * s];
    dst[2 * q + 1] = src[2 * s + 1];
  }
}

// Opacity pruning (_prune, training.py:187-198): rows with opacity > threshold
// are kept, in order, in every listed buffer (parameters, texels, Adam
// moments). Three launches: per-block keep counts, one CTA scanning them,
// then a stable gather of every buffer's rows.
constexpr int kPruneBlock = 1024;

__global__ void k_prune_count(int32_t P, const double* __restrict__ op, double thr,
                              int32_t* __restrict__ block_counts) {
  const int i = blockIdx.x * kPruneBlock + threadIdx.x;
  const bool k = i < P && op[i] > thr;
  const int c = __syncthreads_count(k);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = c;
}

__global__ void k_prune_scan(int32_t nb, int32_t* __restrict__ block_counts,
                             int32_t* __restrict__ kept) {
  __shared__ int32_t s_tot;
  if (threadIdx.x == 0) {
    int32_t run = 0;  // nb <= 2^31 / 1024: a serial scan by one thread is enough here
    for (int b = 0; b < nb; ++b) {
      const int32_t c = block_counts[b];
      block_counts[b] = run;
      run += c;
    }
    s_tot = run;
    *kept = run;
  }
}

__global__ void k_prune_gather(int32_t P, const double* __restrict__ op, double thr,
                               const int32_t* __restrict__ block_start, tsb_row_buffer buf) {
  __shared__ int32_t s_w[kPruneBlock / 32];
  const int i = blockIdx.x * kPruneBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool k = i < P && op[i] > thr;
  const uint32_t b = __ballot_sync(0xffffffffu, k);
  if (lane == 0) s_w[w] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int q = 0; q < kPruneBlock / 32; ++q) {
      const int c = s_w[q];
      s_w[q] = run;
      run += c;
    }
  }
  __syncthreads();
  if (!k) return;
  const int64_t dst_row = block_start[blockIdx.x] + s_w[w] + __popc(b & ((1u << lane) - 1u));
  const int64_t rb = buf.row_bytes;
  const unsigned char* src = static_cast<const unsigned char*>(buf.src) + (int64_t)i * rb;
  unsigned char* dst = static_cast<unsigned char*>(buf.dst) + dst_row * rb;
  if (((rb | (int64_t)(uintptr_t)buf.src | (int64_t)(uintptr_t)buf.dst) & 7) == 0) {
    for (int64_t q = 0; q < rb / 8; ++q)
      reinterpret_cast<uint64_t*>(dst)[q] = reinterpret_cast<const uint64_t*>(src)[q];
  } else {
    for (int64_t q = 0; q < rb; ++q) dst[q] = src[q];
  }
}

// The SSIM window lives in per-device __constant__ memory: uploaded once per
// device (a second GPU in the same process gets its own copy).
PerDevice g_win;

cudaError_t ensure_window() {
  int ok = 0;
  return g_win.get(
      [](int) {
        float w[2 * kR + 1];
        double s = 0.0, wd[2 * kR + 1];
        for (int i = 0; i <= 2 * kR; ++i) {
          const double x = (double)(i - kR);
          wd[i] = std::exp(-0.5 * (x / 1.5) * (x / 1.5));
          s += wd[i];
        }
        for (int i = 0; i <= 2 * kR; ++i) w[i] = (float)(wd[i] / s);
        const cudaError_t e = cudaMemcpyToSymbol(c_win, w, sizeof(w));
        return e == cudaSuccess ? 1 : -(int)e;
      },
      &ok);
}

}  // namespace
}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_loss_scratch_size(int32_t width, int32_t height, uint64_t* bytes) {
  if (width <= 0 || height <= 0 || !bytes) {
    set_error("tsb_loss_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *bytes = (uint64_t)(15 + 9) * width * height * sizeof(float);
  return TSB_OK;
}

int tsb_loss_image(const float* color, const float* target, int32_t width, int32_t height,
                   float dssim_weight, float* dcolor, double* terms, void* scratch,
                   uint64_t scratch_bytes, void* stream) {
  if (!color || !target || !dcolor || !terms || !scratch || width <= 0 || height <= 0) {
    set_error("tsb_loss_image: invalid arguments");
    return TSB_ERR_VALUE;
  }
  const size_t HW = (size_t)width * height;
  if (scratch_bytes < (15 + 9) * HW * sizeof(float)) {
    set_error("tsb_loss_image: scratch too small");
    return TSB_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  TSB_CUDA(ensure_window());
  float* m5 = static_cast<float*>(scratch);
  float* part = m5 + 15 * HW;
  const double N = 3.0 * (double)HW;
  const dim3 rows((width + 255) / 256, height);
  const dim3 strips((width + 255) / 256, (height + kRowsPerBlock - 1) / kRowsPerBlock);
  k_ssim_pass1<<<strips, 256, 0, st>>>(width, height, color, target, m5, terms);
  TSB_CHECK_LAUNCH("k_ssim_pass1");
  const dim3 vtiles((width + kTX - 1) / kTX, (height + kTY - 1) / kTY, 3);
  k_ssim_pass2<<<vtiles, 256, 0, st>>>(width, height, m5, part,
                                     (float)(-0.5 * dssim_weight / N), terms);
  TSB_CHECK_LAUNCH("k_ssim_pass2");
  k_ssim_pass34<<<dim3((width + kFX - 1) / kFX, (height + kFTY - 1) / kFTY, 3), 256, 0, st>>>(
      width, height, part, color, target, (float)((1.0 - dssim_weight) / N), dcolor);
  TSB_CHECK_LAUNCH("k_ssim_pass34");
  return TSB_OK;
}

int tsb_loss_regularizers(const float* gbuf, const float* target, const tsb_camera* camera,
                          float normal_weight, float smooth_weight, float* dgbuf, double* terms,
                          void* stream) {
  if (!gbuf || !target || !camera || !dgbuf || !terms || camera->width <= 0 ||
      camera->height <= 0) {
    set_error("tsb_loss_regularizers: invalid arguments");
    return TSB_ERR_VALUE;
  }
  if (!(normal_weight > 0.0f) && !(smooth_weight > 0.0f)) return TSB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  RegParams rp;
  rp.W = camera->width; rp.H = camera->height;
  rp.fx = camera->fx; rp.fy = camera->fy; rp.cx = camera->cx; rp.cy = camera->cy;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) rp.R[3 * i + j] = (float)camera->world_to_view[4 * i + j];
  rp.gbuf = gbuf; rp.target = target; rp.dgbuf = dgbuf; rp.terms = terms;
  rp.w_normal = normal_weight > 0.0f ? normal_weight : 0.0f;
  rp.w_smooth = smooth_weight > 0.0f ? smooth_weight : 0.0f;
  const dim3 rows((rp.W + 255) / 256, rp.H);
  k_reg_count<<<dim3(rows.x, (rp.H + kRowsPerBlock - 1) / kRowsPerBlock), 256, 0, st>>>(rp);
  TSB_CHECK_LAUNCH("k_reg_count");
  k_reg_grad<<<rows, 256, 0, st>>>(rp);
  TSB_CHECK_LAUNCH("k_reg_grad");
  return TSB_OK;
}

int tsb_adam_step(const tsb_adam_group* groups, int32_t num_groups, int32_t step, double beta1,
                  double beta2, double eps, void* stream) {
  return tsb_adam_step_ex(groups, num_groups, step, beta1, beta2, eps, nullptr, stream);
}

int tsb_adam_step_ex(const tsb_adam_group* groups, int32_t num_groups, int32_t step,
                     double beta1, double beta2, double eps, const int32_t* halt, void* stream) {
  if (!groups || num_groups <= 0 || num_groups > TSB_ADAM_MAX_GROUPS || step <= 0) {
    set_error("tsb_adam_step: invalid arguments");
    return TSB_ERR_VALUE;
  }
  AdamLaunch A;
  A.n = num_groups;
  A.blk_start[0] = 0;
  for (int k = 0; k < num_groups; ++k) {
    const tsb_adam_group& g = groups[k];
    if (g.count < 0 || (g.count > 0 && (!g.param || !g.grad || !g.m || !g.v)) ||
        (g.dtype != TSB_F32 && g.dtype != TSB_F64 && g.dtype != TSB_F32_TEX87) ||
        (g.dtype == TSB_F32_TEX87 && (g.count & 7) != 0)) {
      set_error("tsb_adam_step: invalid group");
      return TSB_ERR_VALUE;
    }
    A.g[k] = g;
    const int64_t nb = (g.count + kAdamChunk - 1) / kAdamChunk;
    if ((int64_t)A.blk_start[k] + nb > 0x7fffffff) {
      set_error("tsb_adam_step: too many elements");
      return TSB_ERR_VALUE;
    }
    A.blk_start[k + 1] = A.blk_start[k] + (int32_t)nb;
  }
  A.b1 = beta1; A.b2 = beta2; A.eps = eps;
  A.halt = halt;
  A.bc1 = 1.0 - std::pow(beta1, step);
  A.bc2 = 1.0 - std::pow(beta2, step);
  const int blocks = A.blk_start[num_groups];
  if (blocks == 0) return TSB_OK;
  k_adam<<<blocks, 256, 0, (cudaStream_t)stream>>>(A);
  TSB_CHECK_LAUNCH("k_adam");
  return TSB_OK;
}

int tsb_orthonormalize_tangents(int32_t num_splats, double* tangent_u, double* tangent_v,
                                void* stream) {
  return tsb_orthonormalize_tangents_ex(num_splats, tangent_u, tangent_v, nullptr, stream);
}

int tsb_orthonormalize_tangents_ex(int32_t num_splats, double* tangent_u, double* tangent_v,
                                   const int32_t* halt, void* stream) {
  if (num_splats < 0 || (num_splats > 0 && (!tangent_u || !tangent_v))) {
    set_error("tsb_orthonormalize_tangents: invalid arguments");
    return TSB_ERR_VALUE;
  }
  if (num_splats == 0) return TSB_OK;
  k_orthonormalize<<<(num_splats + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      num_splats, tangent_u, tangent_v, halt);
  TSB_CHECK_LAUNCH("k_orthonormalize");
  return TSB_OK;
}

int tsb_guard_finite(const double* terms, int32_t n, int32_t* halt, void* stream) {
  if (!terms || !halt || n <= 0 || n > 1024) {
    set_error("tsb_guard_finite: invalid arguments");
    return TSB_ERR_VALUE;
  }
  k_guard_finite<<<1, 32 * ((n + 31) / 32), 0, (cudaStream_t)stream>>>(terms, n, halt);
  TSB_CHECK_LAUNCH("k_guard_finite");
  return TSB_OK;
}

int tsb_broadcast_texels(int32_t num_splats, int32_t T0, int32_t T, const float* src, float* dst,
                         void* stream) {
  if (num_splats < 0 || T0 < 1 || T < 1 || (num_splats > 0 && (!src || !dst))) {
    set_error("tsb_broadcast_texels: invalid arguments");
    return TSB_ERR_VALUE;
  }
  if (num_splats == 0) return TSB_OK;
  k_broadcast_texels<<<1184, 256, 0, (cudaStream_t)stream>>>(
      num_splats, T0, T, reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst));
  TSB_CHECK_LAUNCH("k_broadcast_texels");
  return TSB_OK;
}

int tsb_prune_scratch_size(int32_t num_splats, uint64_t* bytes) {
  if (!bytes || num_splats < 0) {
    set_error("tsb_prune_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  *bytes = (uint64_t)((num_splats + kPruneBlock - 1) / kPruneBlock + 1) * 4;
  return TSB_OK;
}

int tsb_prune_rows(int32_t num_splats, const double* opacities, double threshold,
                   const tsb_row_buffer* bufs, int32_t num_bufs, int32_t* kept, void* scratch,
                   uint64_t scratch_bytes, void* stream) {
  uint64_t need = 0;
  if (tsb_prune_scratch_size(num_splats, &need) != TSB_OK) return TSB_ERR_VALUE;
  if (!opacities || !kept || !scratch || scratch_bytes < need || num_bufs < 0 ||
      (num_bufs > 0 && !bufs)) {
    set_error("tsb_prune_rows: invalid arguments");
    return TSB_ERR_VALUE;
  }
  for (int b = 0; b < num_bufs; ++b)
    if (!bufs[b].src || !bufs[b].dst || bufs[b].src == bufs[b].dst || bufs[b].row_bytes <= 0) {
      set_error("tsb_prune_rows: every buffer needs distinct src / dst and a row size");
      return TSB_ERR_VALUE;
    }
  cudaStream_t st = (cudaStream_t)stream;
  if (num_splats == 0) {
    TSB_CUDA(cudaMemsetAsync(kept, 0, 4, st));
    return TSB_OK;
  }
  const int nb = (num_splats + kPruneBlock - 1) / kPruneBlock;
  int32_t* counts = static_cast<int32_t*>(scratch);
  k_prune_count<<<nb, kPruneBlock, 0, st>>>(num_splats, opacities, threshold, counts);
  TSB_CHECK_LAUNCH("k_prune_count");
  k_prune_scan<<<1, 32, 0, st>>>(nb, counts, kept);
  TSB_CHECK_LAUNCH("k_prune_scan");
  for (int b = 0; b < num_bufs; ++b) {
    k_prune_gather<<<nb, kPruneBlock, 0, st>>>(num_splats, opacities, threshold, counts, bufs[b]);
    TSB_CHECK_LAUNCH("k_prune_gather");
  }
  return TSB_OK;
}

}  // extern "C"
