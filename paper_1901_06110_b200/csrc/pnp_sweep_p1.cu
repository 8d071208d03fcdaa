// Explicit instantiations of the DSG sweep for patch side 1 (all R buckets, C = 1, 2).
#include "sweep_launch.cuh"

namespace pnp {
PNP_INSTANTIATE_P(1)
}  // namespace pnp
