// Internal interface of the stored-inverse block smoother (dg_pmf.cu).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

#include "dg_kernels.h"
#include "dg_tables.h"

namespace dg {

// exact 1D matrices of the nodal Gauss-Lobatto basis (Gauss rule with n points is exact)
struct Mat1D {
  int n;
  double M[kMaxN * kMaxN];   // int th_i th_j
  double S[kMaxN * kMaxN];   // int th_i' th_j'
  double C[kMaxN * kMaxN];   // int th_i' th_j  (row = test derivative)
  double e0[kMaxN], e1[kMaxN], d0[kMaxN], d1[kMaxN];
};

void pmf_tables(const Tables1D& tab, Mat1D* m);
size_t pmf_factor_smem(int nd);
// out[b] (nd x nd) = D_T row-major (invert = 0) or D_T^{-1} TRANSPOSED (invert = 1: out[J][I] =
// D_T^{-1}[I][J], partial pivoting) of cell cell_first + b
cudaError_t launch_pmf_factor(const KParams& kp, const Mat1D& t, int nd, int cell_first, int ncells,
                              int invert, double* out, cudaStream_t s);
// out = u + omega Dinv (f - Au) per cell (out may alias u)
cudaError_t launch_pmf_sweep(int nd, int ncells, const double* Dinv, const double* u, const double* f,
                             const double* Au, double omega, double* out, cudaStream_t s);

}  // namespace dg
