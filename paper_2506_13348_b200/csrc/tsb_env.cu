// tsb_env.cu — environment precompute on sm_100a.
//
//   K15 k_downsample2     2x2 box average of the base radiance map
//                         (environment.py:130-135), fp64
//   K15 k_env_quadrature  per output direction, one warp sums over the
//                         downsampled grid: GGX-weighted prefilter of a
//                         specular level (prefilter_specular :145-175) or the
//                         cosine-weighted diffuse irradiance
//                         (diffuse_irradiance :178-195), fp64
//   K16 k_brdf_lut        split-sum (A, B) per (cos, roughness) cell by GGX
//                         importance sampling over a Hammersley set
//                         (BrdfLut.integrate_cell / build :381-425), fp64
//
// Equirect directions and solid angles are evaluated on the fly with the
// reference's formulas (equirect_dirs / equirect_solid_angles :28-43).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "tsb_internal.cuh"

namespace tsb {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;

__device__ __forceinline__ void equirect_dir(int row, int col, int h, int w, double* d) {
  const double theta = ((double)row + 0.5) / h * kPi;
  const double phi = ((double)col + 0.5) / w * kTwoPi;
  const double st = sin(theta), ct = cos(theta);
  d[0] = st * cos(phi);
  d[1] = st * sin(phi);
  d[2] = ct;
}

__global__ void k_downsample2(const double* __restrict__ base, int h, int w,
                              double* __restrict__ src) {
  const int h2 = h / 2, w2 = w / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= h2 * w2) return;
  const int r = i / w2, c = i % w2;
  for (int k = 0; k < 3; ++k) {
    const double a = base[3 * ((size_t)(2 * r) * w + 2 * c) + k];
    const double b = base[3 * ((size_t)(2 * r) * w + 2 * c + 1) + k];
    const double cc = base[3 * ((size_t)(2 * r + 1) * w + 2 * c) + k];
    const double d = base[3 * ((size_t)(2 * r + 1) * w + 2 * c + 1) + k];
    src[3 * (size_t)i + k] = (((a + b) + cc) + d) * 0.25;
  }
}

// Per source texel: direction (3), solid angle, radiance (3) — 7 doubles.
__global__ void k_env_sources(const double* __restrict__ src, int sh, int sw,
                              double* __restrict__ table) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sh * sw) return;
  const int r = i / sw, c = i % sw;
  double d[3];
  equirect_dir(r, c, sh, sw, d);
  const double theta = ((double)r + 0.5) / sh * kPi;
  double* t = table + 7 * (size_t)i;
  t[0] = d[0]; t[1] = d[1]; t[2] = d[2];
  t[3] = sin(theta) * (kPi / sh) * (kTwoPi / sw);
  t[4] = src[3 * (size_t)i]; t[5] = src[3 * (size_t)i + 1]; t[6] = src[3 * (size_t)i + 2];
}

// One warp per output texel. alpha > 0: GGX prefilter with alpha =
// roughness^2; alpha == 0: diffuse irradiance.
__global__ void __launch_bounds__(256) k_env_quadrature(const double* __restrict__ table, int n_src,
                                                        int oh, int ow, double alpha,
                                                        float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (o >= oh * ow) return;
  double R[3];
  equirect_dir(o / ow, o % ow, oh, ow, R);
  const double a2 = alpha * alpha;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j = lane; j < n_src; j += 32) {
    const double* t = table + 7 * (size_t)j;
    const double cosw = R[0] * t[0] + R[1] * t[1] + R[2] * t[2];
    double wgt;
    if (alpha > 0.0) {
      const double c = cosw < -1.0 ? -1.0 : (cosw > 1.0 ? 1.0 : cosw);
      if (c > 0.0) {
        const double ch = sqrt(0.5 * (1.0 + c));
        const double d = ch * ch * (a2 - 1.0) + 1.0;
        wgt = a2 / (kPi * d * d) * c * t[3];
      } else {
        wgt = 0.0;
      }
    } else {
      wgt = (cosw > 0.0 ? cosw : 0.0) * t[3];
    }
    acc[0] += wgt * t[4];
    acc[1] += wgt * t[5];
    acc[2] += wgt * t[6];
    acc[3] += wgt;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
  if (lane == 0) {
    const double norm = alpha > 0.0 ? fmax(acc[3], 1e-30) : 1.0;
    for (int k = 0; k < 3; ++k) out[3 * (size_t)o + k] = (float)(acc[k] / norm);
  }
}

__global__ void k_cast_f32(const double* __restrict__ a, float* __restrict__ b, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

// One warp per LUT cell (j = roughness row, i = cos column).
__global__ void __launch_bounds__(256) k_brdf_lut(int res, int samples, double* __restrict__ table) {
  const int lane = threadIdx.x & 31;
  const int cell = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (cell >= res * res) return;
  const int j = cell / res, i = cell % res;
  const double rough = ((double)j + 0.5) / res, cos_theta = ((double)i + 0.5) / res;
  const double alpha = rough * rough;
  const double cos_v = fmax(cos_theta, 1e-8);
  const double sin_v = sqrt(fmax(0.0, 1.0 - cos_v * cos_v));
  const double k = alpha / 2.0;
  const double g1v = cos_v / (cos_v * (1.0 - k) + k);
  double sa = 0.0, sb = 0.0;
  for (int s = lane; s < samples; s += 32) {
    const double x0 = (double)s / samples;
    const double x1 = (double)__brev((unsigned)s) * 2.3283064365386963e-10;
    const double phi = kTwoPi * x0;
    const double cos_h = sqrt((1.0 - x1) / (1.0 + (alpha * alpha - 1.0) * x1));
    const double sin_h = sqrt(fmax(0.0, 1.0 - cos_h * cos_h));
    const double hx = sin_h * cos(phi), hz = cos_h;
    double voh = hx * sin_v + hz * cos_v;
    const double nol = 2.0 * voh * hz - cos_v;
    if (!(nol > 0.0)) continue;
    const double noh = fmax(cos_h, 1e-8);
    voh = fmax(voh, 1e-8);
    const double nl = fmax(nol, 1e-8);
    const double G = g1v * (nl / (nl * (1.0 - k) + k));
    const double g_vis = G * voh / (noh * cos_v);
    const double fc = pow(1.0 - voh, 5.0);
    sa += (1.0 - fc) * g_vis;
    sb += fc * g_vis;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, off);
    sb += __shfl_xor_sync(0xffffffffu, sb, off);
  }
  if (lane == 0) {
    table[2 * (size_t)cell] = sa / samples;
    table[2 * (size_t)cell + 1] = sb / samples;
  }
}

}  // namespace
}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_env_scratch_size(int32_t height, int32_t width, uint64_t* bytes) {
  if (height < 2 || width < 2 || !bytes) {
    set_error("tsb_env_scratch_size: invalid arguments");
    return TSB_ERR_VALUE;
  }
  const size_t n = (size_t)(height / 2) * (width / 2);
  *bytes = n * (3 + 7) * sizeof(double);
  return TSB_OK;
}

int tsb_env_prefilter(const double* base, int32_t height, int32_t width, int32_t levels,
                      float* const* spec_mips, const int32_t* mip_h, const int32_t* mip_w,
                      float* diffuse, int32_t diff_h, int32_t diff_w, void* scratch,
                      uint64_t scratch_bytes, void* stream) {
  if (!base || height < 2 || width < 2 || levels < 1 || levels > TSB_ENV_MAX_LEVELS ||
      !spec_mips || !mip_h || !mip_w || !scratch) {
    set_error("tsb_env_prefilter: invalid arguments");
    return TSB_ERR_VALUE;
  }
  uint64_t need = 0;
  tsb_env_scratch_size(height, width, &need);
  if (scratch_bytes < need) {
    set_error("tsb_env_prefilter: scratch too small");
    return TSB_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int sh = height / 2, sw = width / 2, n_src = sh * sw;
  double* src = static_cast<double*>(scratch);
  double* table = src + 3 * (size_t)n_src;
  k_downsample2<<<(n_src + 255) / 256, 256, 0, st>>>(base, height, width, src);
  TSB_CHECK_LAUNCH("k_downsample2");
  k_env_sources<<<(n_src + 255) / 256, 256, 0, st>>>(src, sh, sw, table);
  TSB_CHECK_LAUNCH("k_env_sources");
  // level 0 is the base itself (float32 copy)
  if (spec_mips[0]) {
    const size_t n = (size_t)height * width * 3;
    k_cast_f32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(base, spec_mips[0], n);
    TSB_CHECK_LAUNCH("k_cast_f32");
  }
  for (int l = 1; l < levels; ++l) {
    if (!spec_mips[l]) continue;
    const double r = (double)l / (double)(levels - 1);
    const int n_out = mip_h[l] * mip_w[l];
    k_env_quadrature<<<(n_out + 7) / 8, 256, 0, st>>>(table, n_src, mip_h[l], mip_w[l], r * r,
                                                     spec_mips[l]);
    TSB_CHECK_LAUNCH("k_env_quadrature(specular)");
  }
  if (diffuse) {
    const int n_out = diff_h * diff_w;
    k_env_quadrature<<<(n_out + 7) / 8, 256, 0, st>>>(table, n_src, diff_h, diff_w, 0.0,
                                                     diffuse);
    TSB_CHECK_LAUNCH("k_env_quadrature(diffuse)");
  }
  return TSB_OK;
}

int tsb_brdf_lut(int32_t resolution, int32_t samples, double* table, void* stream) {
  if (resolution <= 0 || samples <= 0 || !table) {
    set_error("tsb_brdf_lut: invalid arguments");
    return TSB_ERR_VALUE;
  }
  const int cells = resolution * resolution;
  k_brdf_lut<<<(cells + 7) / 8, 256, 0, (cudaStream_t)stream>>>(resolution, samples, table);
  TSB_CHECK_LAUNCH("k_brdf_lut");
  return TSB_OK;
}

}  // extern "C"
