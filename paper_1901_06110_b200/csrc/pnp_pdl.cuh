// Programmatic dependent launch (PDL) for the kernel chains of a denoise /
// ADMM iteration (sweep -> fixup -> adjoint -> sweep ...): a kernel launched
// with launch_pdl may be scheduled while its predecessor in the stream is
// still draining, so its CTAs are resident when the predecessor's last CTA
// retires instead of after a launch round trip.
//
// Contract: every kernel launched through launch_pdl calls pdl_begin() before
// it touches global memory.  griddepcontrol.wait returns once the whole
// predecessor grid has completed and its writes are visible; since each
// kernel of a chain waits the same way, that covers every earlier kernel too.
// A kernel launched without the attribute executes both instructions as
// no-ops.  PNP_PDL=0 in the environment turns the attribute off.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace pnp {

__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // dependents may launch as soon as every CTA of this grid has started
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PNP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace pnp

// ---- debug builds (scripts/build_variant.py ... -- -DPNP_CHECKS -DPNP_JITTER) ----
// PNP_CHECKS: device asserts on shared-memory indices and on every global
// write of the sweeps / fixups (partial blocks, k cache) against the buffer
// sizes the host passes; PNP_JITTER: every warp sleeps a pseudo-random
// 0-2 us before each block barrier of the sweeps, so warps reach the ordered
// flushes in a different order on every run -- any missing barrier shows up
// as a result that changes between runs (compute-sanitizer is not available
// on this pool; tests/test_checks_gpu.py drives both).
#include <assert.h>
#ifdef PNP_CHECKS
#define PNP_CHECK(cond) assert(cond)
#else
#define PNP_CHECK(cond) ((void)0)
#endif
namespace pnp {
__device__ __forceinline__ void jitter_sync() {
#ifdef PNP_JITTER
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned h = (unsigned)(t ^ (t >> 13)) * 2654435761u;
  h ^= (blockIdx.x * 977u + blockIdx.y * 131u + (threadIdx.x >> 5) * 40503u) * 2246822519u;
  __nanosleep((h >> 7) & 2047u);
#endif
  __syncthreads();
}
}  // namespace pnp

