// Explicit instantiations of the DSG sweep for patch side 13 (all R buckets, C = 1, 2).
#include "sweep_launch.cuh"

namespace pnp {
PNP_INSTANTIATE_P(13)
}  // namespace pnp
