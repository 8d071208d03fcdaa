// Launcher template for dsg_sweep_kernel; explicitly instantiated per patch
// side in pnp_sweep_p*.cu (compiled in parallel), dispatched in pnp_dsg.cu.
#pragma once

#include <atomic>
#include <cstring>

#include "dsg_sweep.cuh"

namespace pnp {

template <int P, int RB, int C, int MODE>
cudaError_t launch_sweep(const SweepArgs& a, const HostTab& t, dim3 grid, cudaStream_t st,
                         const CUtensorMap& gmap) {
  constexpr size_t smem = (size_t)Cfg<P, RB, C, MODE>::TOTAL * sizeof(float);
  static_assert(smem <= 227 * 1024, "sweep tile exceeds shared memory");
  // the opt-in shared-memory size is a per-device function attribute
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(dsg_sweep_kernel<P, RB, C, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  if (t.nch > max_chunks(RB) || t.ng > kMaxGroups) return cudaErrorInvalidValue;
  ChunkTab<RB> tab;
  memset(&tab, 0, sizeof(tab));
  memcpy(tab.c, t.ch, sizeof(Chunk) * t.nch);
  memcpy(tab.grp, t.grp, sizeof(int) * (t.ng + 1));
  return launch_pdl(dsg_sweep_kernel<P, RB, C, MODE>, grid, dim3(kThreads), smem, st, a, tab,
                    gmap);
}

#define PNP_INSTANTIATE_P(P) \
  template cudaError_t launch_sweep<P, 5, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 5, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 5, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 5, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 5, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 10, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 10, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 10, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 10, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 10, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 16, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 16, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 16, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 16, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 16, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 32, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 32, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 32, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 32, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  template cudaError_t launch_sweep<P, 32, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&);

#define PNP_DECLARE_P(P) \
  extern template cudaError_t launch_sweep<P, 5, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 5, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 5, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 5, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 5, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 10, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 10, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 10, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 10, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 10, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 16, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 16, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 16, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 16, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 16, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 32, 1, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 32, 1, 1>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 32, 1, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 32, 2, 0>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&); \
  extern template cudaError_t launch_sweep<P, 32, 2, 2>(const SweepArgs&, const HostTab&, dim3, cudaStream_t, const CUtensorMap&);

PNP_DECLARE_P(1)
PNP_DECLARE_P(3)
PNP_DECLARE_P(5)
PNP_DECLARE_P(7)
PNP_DECLARE_P(9)
PNP_DECLARE_P(11)
PNP_DECLARE_P(13)
PNP_DECLARE_P(15)

}  // namespace pnp
