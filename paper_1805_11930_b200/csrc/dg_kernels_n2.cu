// Degree p = 1 (n = 2) of the fp64 sm_100a kernels (see dg_kernels_impl.cuh).
#include "dg_kernels_impl.cuh"

namespace dg {
DG_INSTANTIATE_DEGREE(2)
}  // namespace dg
