#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <stdint.h>
#include <vector>
struct Big { float a[4000]; int n; };
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const Big b, float* out, const __grid_constant__ CUtensorMap m, int x0, int y0) {
  extern __shared__ float sm[];
  float* buf = (float*)(((uintptr_t)sm + 127) & ~uintptr_t(127));
  uint64_t* bar = (uint64_t*)(sm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(92*43*4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(x0), "r"(y0), "r"(0), "r"(smem_u32(bar)) : "memory");
  }
  __syncthreads();
  unsigned ok = 0;
  do { asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory"); } while (!ok);
  for (int i = threadIdx.x; i < 92*43; i += blockDim.x) out[i] = buf[i] + b.a[0];
}
int main() {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  printf("entry %d\n", (int)cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q)); printf("q %d fn %p\n", (int)q, fn);
  int W = 256, H = 128;
  std::vector<float> h(W*H); for (int i = 0; i < W*H; ++i) h[i] = i;
  float *g, *out; cudaMalloc(&g, W*H*4); cudaMalloc(&out, 92*43*4); cudaMemcpy(g, h.data(), W*H*4, cudaMemcpyHostToDevice);
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}, str[2] = {(cuuint64_t)W*4, (cuuint64_t)W*H*4};
  cuuint32_t box[3] = {92, 43, 1}, es[3] = {1,1,1};
  CUresult r = ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  Big b; memset(&b, 0, sizeof b);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  k<<<1, 128, 4096*4 + 64>>>(b, out, m, 8, 5);
  printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> o(92*43); cudaMemcpy(o.data(), out, 92*43*4, cudaMemcpyDeviceToHost);
  int bad = 0; for (int r2 = 0; r2 < 43; ++r2) for (int c = 0; c < 92; ++c) if (o[r2*92+c] != h[(r2+5)*W + c + 8]) ++bad;
  printf("bad %d  o[0]=%g want %g\n", bad, o[0], h[5*W+8]);
}
