// TEX-unit microbenchmark (measurement tool, not product code): filtered
// tex2DLayered RGBA fetch rate vs the number of active lanes per warp and
// the texel format. Answers whether a warp-level TEX instruction with k of 32
// lanes active costs k/32 or a full instruction's TEX time.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/texprobe scripts/tex_lanes_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <vector>

__global__ void k_probe(cudaTextureObject_t tex, int window, int iters, int active, float* sink) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  float fx = 0.37f + (float)(t % window);
  float fy = 0.61f + (float)((t / window) % window);
  if (lane < active) {
    for (int k = 0; k < iters; ++k) {
      const float4 v = tex2DLayered<float4>(tex, fx, fy, 0);
      acc += v.x + v.y + v.z + v.w;
      fx += 1.13f; if (fx > (float)window) fx -= (float)window;
      fy += 0.71f; if (fy > (float)window) fy -= (float)window;
    }
  }
  sink[t] = acc;
}

static cudaTextureObject_t make(int fmt, int W, int H, cudaArray_t* arr) {
  cudaChannelFormatDesc cd = fmt ? cudaCreateChannelDescHalf4() : cudaCreateChannelDesc<float4>();
  cudaMalloc3DArray(arr, &cd, make_cudaExtent(W, H, 1), cudaArrayLayered);
  std::vector<float> h((size_t)W * H * 4);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 97) / 97.f;
  std::vector<__half> hh(h.size());
  for (size_t i = 0; i < h.size(); ++i) hh[i] = __float2half(h[i]);
  cudaMemcpy3DParms cp = {};
  cp.srcPtr = fmt ? make_cudaPitchedPtr(hh.data(), W * 8, W, H) : make_cudaPitchedPtr(h.data(), W * 16, W, H);
  cp.dstArray = *arr;
  cp.extent = make_cudaExtent(W, H, 1);
  cp.kind = cudaMemcpyHostToDevice;
  cudaMemcpy3D(&cp);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = *arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModeLinear;
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  return tex;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  const int blocks = sms * 8, threads = 256;
  cudaMalloc(&sink, (size_t)blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int fmt = 0; fmt < 2; ++fmt) {
    cudaArray_t arr;
    cudaTextureObject_t tex = make(fmt, 256, 256, &arr);
    for (int active : {32, 24, 16, 8, 4, 1}) {
      const int iters = 512;
      k_probe<<<blocks, threads>>>(tex, 32, iters, active, sink);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k_probe<<<blocks, threads>>>(tex, 32, iters, active, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double fetches = 5.0 * blocks * (threads / 32) * active * (double)iters;
      const double winst = 5.0 * blocks * (threads / 32) * (double)iters;
      printf("{\"fmt\": \"%s\", \"active\": %d, \"gfetch_s\": %.1f, \"gwarpinst_s\": %.2f}\n",
             fmt ? "rgba16f" : "rgba32f", active, fetches / ms * 1e-6, winst / ms * 1e-6);
    }
    cudaDestroyTextureObject(tex);
    cudaFreeArray(arr);
  }
  return 0;
}
