// Instantiations + launcher of the general DSG sweep (dsg_generic.cuh).
#include <atomic>

#include "dsg_generic.cuh"

namespace pnp {

template <int C, bool BOX, bool SYM, int KG, int MODE, int NM = kGenNmax>
static cudaError_t launch_gen_t(const GenArgs& a, dim3 grid, cudaStream_t st) {
  if (a.TH / 2 > NM) return cudaErrorInvalidValue;
  const size_t smem =
      (size_t)gen_smem(a.TH, a.P, a.R, C, SYM, KG, MODE == MODE_CACHED).total * sizeof(float);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // opt in to the largest dynamic shared memory once per device
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(dsg_generic_kernel<C, BOX, SYM, KG, MODE, NM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  return launch_pdl(dsg_generic_kernel<C, BOX, SYM, KG, MODE, NM>, grid, dim3(kGenThreads), smem,
                    st, a);
}

template <int KG>
static cudaError_t launch_gen_kg(const GenArgs& a, int C, bool box, bool sym, int mode,
                                 dim3 grid, cudaStream_t st) {
  if (mode == MODE_CACHED) {  // no patch filter: box or not is the same kernel
    if (!sym) return cudaErrorInvalidValue;
    if (a.TH <= 8)
      return C == 1 ? launch_gen_t<1, false, true, KG, MODE_CACHED, 4>(a, grid, st)
                    : launch_gen_t<2, false, true, KG, MODE_CACHED, 4>(a, grid, st);
    if (a.TH <= 16)
      return C == 1 ? launch_gen_t<1, false, true, KG, MODE_CACHED, 8>(a, grid, st)
                    : launch_gen_t<2, false, true, KG, MODE_CACHED, 8>(a, grid, st);
    return C == 1 ? launch_gen_t<1, false, true, KG, MODE_CACHED>(a, grid, st)
                  : launch_gen_t<2, false, true, KG, MODE_CACHED>(a, grid, st);
  }
  if (mode == MODE_STORE) {  // sweep A (mass, one channel) writing the cache
    if (!sym || C != 1) return cudaErrorInvalidValue;
    return box ? launch_gen_t<1, true, true, KG, MODE_STORE>(a, grid, st)
               : launch_gen_t<1, false, true, KG, MODE_STORE>(a, grid, st);
  }
  if (C == 1) {
    if (box)
      return sym ? launch_gen_t<1, true, true, KG, MODE_RECOMPUTE>(a, grid, st)
                 : launch_gen_t<1, true, false, KG, MODE_RECOMPUTE>(a, grid, st);
    return sym ? launch_gen_t<1, false, true, KG, MODE_RECOMPUTE>(a, grid, st)
               : launch_gen_t<1, false, false, KG, MODE_RECOMPUTE>(a, grid, st);
  }
  if (box)
    return sym ? launch_gen_t<2, true, true, KG, MODE_RECOMPUTE>(a, grid, st)
               : launch_gen_t<2, true, false, KG, MODE_RECOMPUTE>(a, grid, st);
  return sym ? launch_gen_t<2, false, true, KG, MODE_RECOMPUTE>(a, grid, st)
             : launch_gen_t<2, false, false, KG, MODE_RECOMPUTE>(a, grid, st);
}

cudaError_t launch_generic(const GenArgs& a, int C, bool box, bool sym, int KG, int mode,
                           dim3 grid, cudaStream_t st) {
  if (KG == 4) return launch_gen_kg<4>(a, C, box, sym, mode, grid, st);
  if (KG == 2) return launch_gen_kg<2>(a, C, box, sym, mode, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace pnp
