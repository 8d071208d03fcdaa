// FP32 issue micro-benchmarks on sm_100a (development aid, not product code):
// scalar FFMA (const / register operands), packed FFMA2/FMUL2/FADD2, and
// FFMA mixed with LDS / MUFU, to decide how the DSG sweep's inner loops
// should be written.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;
constexpr int IT = 2048;

__device__ __forceinline__ unsigned long long pk(float2 v) { return *(unsigned long long*)&v; }
__device__ __forceinline__ float2 up(unsigned long long v) { return *(float2*)&v; }

// 1: FFMA with a kernel-param (constant-bank) multiplier and addend
__global__ void k_ffma_c(float* o, float a, float b) {
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], a, b);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 2: FFMA with all-register operands (distinct registers per chain)
__global__ void k_ffma_r(float* o, float a0, float b0) {
  float v[CH], a[CH], b[CH];
  for (int c = 0; c < CH; ++c) {
    v[c] = threadIdx.x + c;
    a[c] = a0 + threadIdx.x * 1e-9f * c;
    b[c] = b0 - threadIdx.x * 1e-9f * c;
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) v[c] = fmaf(v[c], a[c], b[c]);
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c] + a[c] + b[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 3: FFMA2, register pairs
__global__ void k_ffma2_r(float* o, float a0, float b0) {
  unsigned long long v[CH], a[CH], b[CH];
  for (int c = 0; c < CH; ++c) {
    v[c] = pk(make_float2(threadIdx.x + c, c));
    a[c] = pk(make_float2(a0 + threadIdx.x * 1e-9f * c, a0));
    b[c] = pk(make_float2(b0 - threadIdx.x * 1e-9f * c, b0));
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(a[c]), "l"(b[c]));
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y + up(a[c]).x + up(b[c]).y;
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 4: FMUL2 / FADD2 alternating
__global__ void k_addmul2(float* o, float a0, float b0) {
  unsigned long long v[CH], a[CH];
  for (int c = 0; c < CH; ++c) {
    v[c] = pk(make_float2(threadIdx.x + c, c));
    a[c] = pk(make_float2(a0 + threadIdx.x * 1e-9f * c, b0));
  }
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(v[c]) : "l"(a[c]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v[c]) : "l"(a[c]));
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y + up(a[c]).x;
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 5: 2 FFMA (reg) + 1 LDS per chain step  (issue-mix test)
__global__ void k_ffma_lds(float* o, float a0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = p[(r * CH + c) * 32 & 1023];
        v[c] = fmaf(v[c], x, a0);
        v[c] = fmaf(v[c], x, x);
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 6: 1 FFMA2 (= 2 FMAs) + 1 LDS per chain step
__global__ void k_ffma2_lds(float* o, float a0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  unsigned long long v[CH];
  const unsigned long long aa = pk(make_float2(a0, a0));
  for (int c = 0; c < CH; ++c) v[c] = pk(make_float2(threadIdx.x + c, c));
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = p[(r * CH + c) * 32 & 1023];
        unsigned long long xx;
        asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(xx), "l"(aa));
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y;
  if (s == 1.5f) o[threadIdx.x] = s;
}

// 7: 8 FFMA2 + 1 MUFU.EX2
__global__ void k_ffma2_ex2(float* o, float a0) {
  unsigned long long v[CH];
  const unsigned long long aa = pk(make_float2(a0, a0)), bb = pk(make_float2(-1e-3f, -2e-3f));
  for (int c = 0; c < CH; ++c) v[c] = pk(make_float2(-1e-3f * threadIdx.x, -1e-3f * c));
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
      float y, x = up(v[r & 7]).x;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
      float2 t = up(v[(r + 1) & 7]);
      t.y = y;
      v[(r + 1) & 7] = pk(t);
    }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y;
  if (s == 1.5f) o[threadIdx.x] = s;
}


__device__ __forceinline__ float lds_v(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
// 8: 4 FFMA (const form) + 1 LDS per step (volatile LDS)
__global__ void k_4ffma_lds(float* o, float a0, float b0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  float v[CH];
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x + c;
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = lds_v(p + ((i + r * CH + c) & 31) * 32);
        v[c] = fmaf(v[c], a0, x);
        v[c] = fmaf(v[c], a0, b0);
        v[c] = fmaf(v[c], a0, b0);
        v[c] = fmaf(v[c], a0, b0);
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}
// 9: 2 FFMA2 (UR form) + 1 LDS per step
__global__ void k_2ffma2_lds(float* o, float a0, float b0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  unsigned long long v[CH];
  const unsigned long long aa = pk(make_float2(a0, a0)), bb = pk(make_float2(b0, b0));
  for (int c = 0; c < CH; ++c) v[c] = pk(make_float2(threadIdx.x + c, c));
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = lds_v(p + ((i + r * CH + c) & 31) * 32);
        unsigned long long xx;
        asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(xx));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y;
  if (s == 1.5f) o[threadIdx.x] = s;
}
// 10: 4 FFMA2 (UR) + 2 LDS + 1 MUFU + 2 FFMA 3-reg per step (sweep phase-2 like)
__global__ void k_mix(float* o, float a0, float b0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  unsigned long long v[CH];
  float nr[CH], fr[CH];
  const unsigned long long aa = pk(make_float2(a0, a0)), bb = pk(make_float2(b0, b0));
  for (int c = 0; c < CH; ++c) { v[c] = pk(make_float2(-1e-3f * threadIdx.x, c)); nr[c] = fr[c] = 0; }
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = lds_v(p + ((i + r * CH + c) & 31) * 32);
        float y = lds_v(p + ((i + r * CH + c + 7) & 31) * 32);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(aa), "l"(bb));
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(up(v[c]).x));
        nr[c] = fmaf(e, x, nr[c]);
        fr[c] = fmaf(e, y, fr[c]);
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += up(v[c]).x + up(v[c]).y + nr[c] + fr[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}
// 11: same as 10, scalar FFMA (const) x8
__global__ void k_mix_s(float* o, float a0, float b0) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  float v[CH], w[CH];
  float nr[CH], fr[CH];
  for (int c = 0; c < CH; ++c) { v[c] = -1e-3f * threadIdx.x; w[c] = c; nr[c] = fr[c] = 0; }
  const float* p = sm + (threadIdx.x & 31);
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float x = lds_v(p + ((i + r * CH + c) & 31) * 32);
        float y = lds_v(p + ((i + r * CH + c + 7) & 31) * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) { v[c] = fmaf(v[c], a0, b0); w[c] = fmaf(w[c], a0, b0); }
        float e;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(v[c]));
        nr[c] = fmaf(e, x, nr[c]);
        fr[c] = fmaf(e, y, fr[c]);
      }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += v[c] + w[c] + nr[c] + fr[c];
  if (s == 1.5f) o[threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread_iter, int sms, float* o) {
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
  int dev;
  cudaGetDevice(&dev);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double thr = (double)sms * 8 * 256;
  const double ops = thr * IT * ops_per_thread_iter;
  const double per_clk_sm = ops / (best * 1e-3) / (clk * 1e3) / sms;
  printf("%-14s %8.3f ms  %8.2f T FP32-op/s  %6.1f op/clk/SM  (err=%s)\n", name, best,
         ops / (best * 1e-3) / 1e12, per_clk_sm, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 4096);
  dim3 g(sms * 8), b(256);
  run("ffma_const", [&] { k_ffma_c<<<g, b>>>(o, 0.999f, 1e-3f); }, 16.0 * CH, sms, o);
  run("ffma_reg", [&] { k_ffma_r<<<g, b>>>(o, 0.999f, 1e-3f); }, 16.0 * CH, sms, o);
  run("ffma2_reg", [&] { k_ffma2_r<<<g, b>>>(o, 0.999f, 1e-3f); }, 32.0 * CH, sms, o);
  run("fmul2+fadd2", [&] { k_addmul2<<<g, b>>>(o, 0.999f, 1e-3f); }, 32.0 * CH, sms, o);
  run("2ffma+lds", [&] { k_ffma_lds<<<g, b>>>(o, 0.999f); }, 32.0 * CH, sms, o);
  run("ffma2+lds", [&] { k_ffma2_lds<<<g, b>>>(o, 0.999f); }, 32.0 * CH, sms, o);
  run("8ffma2+ex2", [&] { k_ffma2_ex2<<<g, b>>>(o, 0.999f); }, 16.0 * 16 * CH / 16 * 2, sms, o);
  run("4ffma+lds", [&] { k_4ffma_lds<<<g, b>>>(o, 0.999f, 1e-3f); }, 4.0 * CH * 4, sms, o);
  run("2ffma2+lds", [&] { k_2ffma2_lds<<<g, b>>>(o, 0.999f, 1e-3f); }, 4.0 * CH * 4, sms, o);
  run("mix ffma2", [&] { k_mix<<<g, b>>>(o, 0.999f, 1e-3f); }, 2.0 * CH * 10, sms, o);
  run("mix scalar", [&] { k_mix_s<<<g, b>>>(o, 0.999f, 1e-3f); }, 2.0 * CH * 10, sms, o);
  return 0;
}
