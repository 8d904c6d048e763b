// tsb_image.cu — K14: the render command's decomposition images
// (cli.py:52-96 cmd_render --decompose; write_png imgio.py:13-21) computed
// on the device straight into 8-bit pixels.
//
// From the planar G-buffer and the shaded colour / diffuse / specular:
//   albedo    = cov ? albedo / a : 0               (3 channels)
//   normal    = cov ? 0.5 (n / max(|n|, 1e-12) + 1) : 0.5
//   roughness = cov ? roughness / a : 0            (1 channel)
//   metallic  = cov ? metallic / a : 0             (1 channel)
//   diffuse, specular, final = linear_to_display(...) (losses.py:24-29)
// with a = max(alpha, 1e-8), cov = alpha > 1e-8, each quantised as
// rint(clip(v, 0, 1) * 255) (round half to even, like numpy).

#include <cuda_runtime.h>

#include "tsb_internal.cuh"

namespace tsb {
namespace {

__device__ __forceinline__ float to_display(float x) {
  x = fmaxf(x, 0.0f);
  const float p = (float)(1.0 / 2.2);
  const float toe = 1e-4f;
  const float toe_slope = powf(toe, p - 1.0f);
  return x >= toe ? powf(fmaxf(x, toe), p) : toe_slope * x;
}

__device__ __forceinline__ uint8_t q8(float v) {
  v = fminf(fmaxf(v, 0.0f), 1.0f);
  return (uint8_t)rintf(v * 255.0f);
}

__global__ void k_decompose(int W, int H, const float* __restrict__ gbuf,
                            const float* __restrict__ color, const float* __restrict__ diffuse,
                            const float* __restrict__ specular, uint8_t* __restrict__ out) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t HW = (size_t)W * H;
  if (pix >= (int)HW) return;
  float g[13];
#pragma unroll
  for (int c = 0; c < 13; ++c) g[c] = gbuf[c * HW + pix];
  const bool cov = g[12] > 1e-8f;
  const float a = fmaxf(g[12], 1e-8f);
  uint8_t* albedo = out;
  uint8_t* normal = out + 3 * HW;
  uint8_t* rough = out + 6 * HW;
  uint8_t* metal = out + 7 * HW;
  uint8_t* dif = out + 8 * HW;
  uint8_t* spe = out + 11 * HW;
  uint8_t* fin = out + 14 * HW;
  const float nn = fmaxf(sqrtf(g[5] * g[5] + g[6] * g[6] + g[7] * g[7]), 1e-12f);
  for (int c = 0; c < 3; ++c) {
    albedo[3 * pix + c] = q8(cov ? g[c] / a : 0.0f);
    normal[3 * pix + c] = q8(cov ? 0.5f * (g[5 + c] / nn + 1.0f) : 0.5f);
    dif[3 * pix + c] = q8(to_display(diffuse[3 * pix + c]));
    spe[3 * pix + c] = q8(to_display(specular[3 * pix + c]));
    fin[3 * pix + c] = q8(to_display(color[3 * pix + c]));
  }
  rough[pix] = q8(cov ? g[4] / a : 0.0f);
  metal[pix] = q8(cov ? g[3] / a : 0.0f);
}

}  // namespace
}  // namespace tsb

using namespace tsb;

extern "C" int tsb_decompose(const float* gbuf, const float* color, const float* diffuse,
                             const float* specular, int32_t width, int32_t height, uint8_t* out,
                             void* stream) {
  if (!gbuf || !color || !diffuse || !specular || !out || width <= 0 || height <= 0) {
    set_error("tsb_decompose: invalid arguments");
    return TSB_ERR_VALUE;
  }
  const int n = width * height;
  k_decompose<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(width, height, gbuf, color,
                                                                 diffuse, specular, out);
  TSB_CHECK_LAUNCH("k_decompose");
  return TSB_OK;
}
