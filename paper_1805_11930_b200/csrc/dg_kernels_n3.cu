// Degree p = 2 (n = 3) of the fp64 sm_100a kernels (see dg_kernels_impl.cuh).
#include "dg_kernels_impl.cuh"

namespace dg {
DG_INSTANTIATE_DEGREE(3)
}  // namespace dg
