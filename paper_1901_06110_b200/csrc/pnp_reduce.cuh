// Deterministic reductions of per-CTA float64 partials, shared by the kernels
// that fold the former reduce_partials_kernel launch into their own tail.
#pragma once

#include <cuda_runtime.h>

namespace pnp {

// out[b*stride + k] = scale * sum_j partial[b][j][k] for one (b, k), computed
// by the calling CTA (blockDim.x == 256 for results identical to
// reduce_partials_kernel): thread t sums j = t, t + 256, ... in order, then a
// fixed shuffle / shared-memory tree.  `red` is 8 doubles of shared memory.
__device__ __forceinline__ void cta_reduce_partials(const double* partial, int nblk, int nvec,
                                                    int b, int k, double scale, double* out,
                                                    int stride, double* red) {
  double s = 0.0;
  for (int j = threadIdx.x; j < nblk; j += blockDim.x)
    s += __ldcg(partial + ((size_t)b * nblk + j) * nvec + k);
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[(size_t)b * stride + k] = scale * t;
  }
  __syncthreads();  // red is reused by the next call
}

// Three sums at once (k = 0..2 of nvec = 3 partials): per k exactly the
// arithmetic of cta_reduce_partials, with all loads of a thread in flight
// together.  `red` is 3 x 8 doubles of shared memory.
__device__ __forceinline__ void cta_reduce_partials3(const double* partial, int nblk, int b,
                                                     double scale, double* out, int stride,
                                                     double (*red)[8]) {
  double s[3] = {0.0, 0.0, 0.0};
  const double* base = partial + (size_t)b * nblk * 3;
  int j = threadIdx.x;
  for (; j + 3 * (int)blockDim.x < nblk; j += 4 * blockDim.x) {
    double v[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) v[i][k] = __ldcg(base + (size_t)(j + i * blockDim.x) * 3 + k);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) s[k] += v[i][k];
  }
  for (; j < nblk; j += blockDim.x)
#pragma unroll
    for (int k = 0; k < 3; ++k) s[k] += __ldcg(base + (size_t)j * 3 + k);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    for (int off = 16; off; off >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = s[k];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[k][w];
    out[(size_t)b * stride + k] = scale * t;
  }
  __syncthreads();
}

// Called by every CTA of a group of `total` CTAs after it wrote its partials:
// the last CTA to arrive (device-scope counter, reset by it for the next
// launch) reduces the group's sums.  Returns true in that CTA.
__device__ __forceinline__ bool cta_is_last_of(unsigned* counter, unsigned total) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == total - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
  return last;
}

// The whole grid as one group: the last CTA reduces all `batch` x `nvec` sums.
__device__ __forceinline__ bool cta_is_last(unsigned* counter) {
  return cta_is_last_of(counter, gridDim.x * gridDim.y * gridDim.z);
}

}  // namespace pnp
