// Per-degree entry points of the kernels: one translation unit per n = p+1
// (dg_kernels_n<N>.cu), dispatched on p by dg_kernels.cu.
#pragma once
#include "dg_kernels.h"

namespace dg {

template <int N> struct Deg {
  static bool upload(const Tables1D& t, cudaError_t* err);
  static cudaError_t apply(const KParams& kp, const double* u, double* out, cudaStream_t s, int with_nbr);
  static cudaError_t solve(int method, bool sweep, const KParams& kp, const double* in,
                           const double* f, double* out, cudaStream_t s);
  static int solver_group_cells();   // cells per CTA of the plane solvers (0: line family)
  static int group_lcm();            // lcm of the cells per CTA of its apply / sweep kernels
};

}  // namespace dg
