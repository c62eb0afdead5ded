// Degree p = 4 (n = 5) of the fp64 sm_100a kernels (see dg_kernels_impl.cuh).
#include "dg_kernels_impl.cuh"

namespace dg {
DG_INSTANTIATE_DEGREE(5)
}  // namespace dg
