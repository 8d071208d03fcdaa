// FFMA2 operand-form throughput on sm_100a (development aid): which packed
// forms the DSG sweep can issue at full FP32 rate.  Each kernel runs CH
// independent accumulator chains; ops = FP32 FMAs (2 per FFMA2).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int IT = 2048;

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// 1: acc(pair) = x(pair) * u(uniform scalar) + acc(pair)     [H/V filter form]
__global__ void k_pair_ur(float* o, float u) {
  float2 acc[CH], x[CH];
  for (int c = 0; c < CH; ++c) { acc[c] = f2(threadIdx.x, c); x[c] = f2(1e-3f * c, 2e-3f * threadIdx.x); }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(x[(c + r) & (CH - 1)], f2(u, u), acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 2: acc(pair) = y(pair) * k(register scalar) + acc(pair)   [C=2 near/far]
__global__ void k_pair_rs(float* o, float u) {
  float2 acc[CH], y[CH];
  float k[CH];
  for (int c = 0; c < CH; ++c) {
    acc[c] = f2(threadIdx.x, c);
    y[c] = f2(1e-3f * c, 2e-3f * threadIdx.x);
    k[c] = u + 1e-7f * (threadIdx.x + c);
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(y[(c + r) & (CH - 1)], f2(k[c], k[c]), acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y + k[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 3: scalar acc = k * y + acc, all registers               [C=1 near]
__global__ void k_scalar_rrr(float* o, float u) {
  float acc[CH], y[CH], k[CH];
  for (int c = 0; c < CH; ++c) {
    acc[c] = threadIdx.x + c;
    y[c] = 1e-3f * c + threadIdx.x;
    k[c] = u + 1e-7f * (threadIdx.x + c);
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(k[(c + r) & (CH - 1)], y[c], acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c] + y[c] + k[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 4: scalar acc = k * y + acc, where k is shared by two chains (reuse cache)
__global__ void k_scalar_reuse(float* o, float u) {
  float acc[CH], y[CH], k[CH / 2];
  for (int c = 0; c < CH; ++c) { acc[c] = threadIdx.x + c; y[c] = 1e-3f * c + threadIdx.x; }
  for (int c = 0; c < CH / 2; ++c) k[c] = u + 1e-7f * (threadIdx.x + c);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __fmaf_rn(k[((c >> 1) + r) & (CH / 2 - 1)], y[c], acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c] + y[c];
  for (int c = 0; c < CH / 2; ++c) s += k[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 5: acc(pair) = k(pair) * y(scalar bcast) + acc(pair)      [C=1 far, offset pair]
__global__ void k_pair_pp_s(float* o, float u) {
  float2 acc[CH], k[CH];
  float y[CH];
  for (int c = 0; c < CH; ++c) {
    acc[c] = f2(threadIdx.x, c);
    k[c] = f2(u + 1e-7f * c, u - 1e-7f * threadIdx.x);
    y[c] = 1e-3f * c + threadIdx.x;
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(k[(c + r) & (CH - 1)], f2(y[c], y[c]), acc[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y + y[c] + k[c].x;
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 6: t = p(pair) + g(scalar bcast); t*t   [phase-1 squared difference]
__global__ void k_sqdiff(float* o, float u) {
  float2 acc[CH], p[CH];
  float g[CH];
  for (int c = 0; c < CH; ++c) {
    acc[c] = f2(0, 0);
    p[c] = f2(1e-3f * c, 2e-3f * threadIdx.x);
    g[c] = -u * c;
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const float2 t = __fadd2_rn(p[(c + r) & (CH - 1)], f2(g[c], g[c]));
        acc[c] = __fadd2_rn(acc[c], __fmul2_rn(t, t));
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y + g[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread_iter, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = (double)sms * 8 * 256 * IT * ops_per_thread_iter;
  printf("%-16s %8.3f ms  %7.2f T FMA/s  %6.1f /clk/SM  (%s)\n", name, best,
         ops / (best * 1e-3) / 1e12, ops / (best * 1e-3) / (clk * 1e3) / sms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 4096);
  dim3 g(sms * 8), b(256);
  run("pair*UR+pair", [&] { k_pair_ur<<<g, b>>>(o, 0.999f); }, 32.0 * CH, sms);
  run("pair*Rs+pair", [&] { k_pair_rs<<<g, b>>>(o, 0.999f); }, 32.0 * CH, sms);
  run("scalar rrr", [&] { k_scalar_rrr<<<g, b>>>(o, 0.999f); }, 16.0 * CH, sms);
  run("scalar k-reuse", [&] { k_scalar_reuse<<<g, b>>>(o, 0.999f); }, 16.0 * CH, sms);
  run("pairK*Ys+pair", [&] { k_pair_pp_s<<<g, b>>>(o, 0.999f); }, 32.0 * CH, sms);
  run("sqdiff f32x2", [&] { k_sqdiff<<<g, b>>>(o, 0.999f); }, 8.0 * CH * 6, sms);
  return 0;
}
