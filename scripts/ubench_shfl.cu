// Shared-memory load vs warp-shuffle throughput on sm_100a (development aid):
// does SHFL compete with LDS for the same per-SM datapath?  Each thread of a
// 128-thread CTA (3 CTAs/SM, like the DSG sweep) runs IT iterations of NL
// conflict-free 32-bit LDS (lane = row of an odd-pitch tile, as in phase 1)
// and NS shuffles; values are consumed by integer XORs (ALU pipe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubs scripts/ubench_shfl.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int IT = 4096;
constexpr int PITCH = 91;  // odd: lanes (rows) hit distinct banks

template <int NL, int NS>
__global__ void __launch_bounds__(128) k_mix(unsigned* o, int salt) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < 48 * PITCH; i += 128) sm[i] = (float)(i ^ salt);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* row = sm + lane * PITCH + warp * 16;
  unsigned acc0 = lane, acc1 = salt, reg[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) reg[j] = lane * 7 + j;
  for (int it = 0; it < IT; ++it) {
    const int off = (it * 3) & 7;
#pragma unroll
    for (int j = 0; j < NL; ++j) acc0 ^= __float_as_uint(row[off + (j % 22) + (j / 22) * PITCH]);
#pragma unroll
    for (int j = 0; j < NS; ++j) acc1 ^= __shfl_down_sync(0xffffffffu, reg[j & 7] ^ acc1 * 0u + it, 1 + (j & 3));
  }
  if ((acc0 ^ acc1) == 0x12345u) o[blockIdx.x] = acc0 ^ acc1;
}

template <int NL, int NS>
float run(unsigned* o) {
  const int smem = 70 * 1024;
  cudaFuncSetAttribute(k_mix<NL, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = 148 * 3 * 4;
  k_mix<NL, NS><<<grid, 128, smem>>>(o, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_mix<NL, NS><<<grid, 128, smem>>>(o, r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_ops = (double)grid * 4 * IT;  // warps x iterations
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("NL=%2d NS=%2d  %.3f ms  LDS warp-instr/clk/SM %.3f  SHFL warp-instr/clk/SM %.3f  total %.3f\n",
         NL, NS, ms, warp_ops * NL / 148 / cycles, warp_ops * NS / 148 / cycles,
         warp_ops * (NL + NS) / 148 / cycles);
  return ms;
}

int main() {
  unsigned* o;
  cudaMalloc(&o, 1 << 20);
  run<44, 0>(o);
  run<88, 0>(o);
  run<0, 44>(o);
  run<0, 88>(o);
  run<44, 44>(o);
  run<44, 22>(o);
  run<88, 44>(o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
