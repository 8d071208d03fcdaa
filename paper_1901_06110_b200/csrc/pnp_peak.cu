// FP32 (FFMA) and SFU (MUFU.EX2) throughput micro-benchmarks: the measured
// denominators of the DSG roofline (MEASURED_PEAKS.json has only HBM and
// tensor peaks; SURVEY.md §8(d) asks to verify the 16 ex2/clk/SM assumption).
#include <math.h>

#include "pnp_internal.h"

namespace pnp {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) peak_ffma_kernel(float* sink, int iters, float a, float b) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < kChains; ++c) v[c] = fmaf(v[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) peak_ex2_kernel(float* sink, int iters, float a) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = -1e-3f * (threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[c]));
        v[c] = y - a;  // keeps the argument in (-1, 0]
      }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

}  // namespace pnp

using namespace pnp;

extern "C" int pnp_peak_rates(int device, double* ffma_per_s, double* ex2_per_s) {
  if (!ffma_per_s || !ex2_per_s) return fail(PNP_EINVAL, "null argument");
  PNP_CUDA(cudaSetDevice(device));
  int sms = 0;
  PNP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  float* sink = nullptr;
  PNP_CUDA(cudaMalloc(&sink, 256 * sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  double best_f = 0, best_x = 0;
  for (int rep = 0; rep < 3; ++rep) {
    const int it_f = 4096, it_x = 512;
    cudaEventRecord(e0);
    peak_ffma_kernel<<<blocks, threads>>>(sink, it_f, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = (double)blocks * threads * it_f * 16 * kChains / (ms * 1e-3);
    cudaEventRecord(e0);
    peak_ex2_kernel<<<blocks, threads>>>(sink, it_x, 0.25f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double x = (double)blocks * threads * it_x * 16 * kChains / (ms * 1e-3);
    if (f > best_f) best_f = f;
    if (x > best_x) best_x = x;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (e != cudaSuccess) return cuda_fail(e, "peak kernels");
  *ffma_per_s = best_f;  // FFMA instructions per second (1 op each)
  *ex2_per_s = best_x;
  return PNP_OK;
}
