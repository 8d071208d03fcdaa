// Explicit instantiations of the DSG sweep for patch side 5 (all R buckets, C = 1, 2).
#include "sweep_launch.cuh"

namespace pnp {
PNP_INSTANTIATE_P(5)
}  // namespace pnp
