// Internal launch interface of the hybrid-multigrid kernels (dg_hybrid.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dg_kernels.h"

namespace dg {

constexpr int kMaxCoarseBlocks = 2048;    // cooperative coarse-PCG grid cap (partials buffer size)
constexpr int kPartials = 6 * kMaxCoarseBlocks;

int vec_blocks();
// A^ = P^T A P as 7 rows of a structure-of-arrays stencil: Ah[0..N) diagonal, Ah[(1+f)N..) the
// coupling to the face-f neighbour (f = 2 axis + hi), 0 where there is none.
cudaError_t launch_coarse_matrix(const KParams& kp, double* Ah, cudaStream_t s);
cudaError_t launch_restrict(const double* r, double* rh, int ncells, int nd, cudaStream_t s);
cudaError_t launch_prolongate_add(double* u, const double* uh, int64_t ndof, int nd, cudaStream_t s);
// x = (Jacobi-PCG) A^-1 rhs to ||r|| <= tol ||rhs||; work: 5N doubles; part: kPartials doubles;
// its[0] = iterations (| 1 << 30 when max_it was hit). One cooperative launch.
cudaError_t launch_coarse_pcg(const KParams& kp, const double* Ah, const double* rhs, double* x,
                              double* work, double* part, int* its, double tol, int max_it,
                              cudaStream_t s);
cudaError_t launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t s);
cudaError_t launch_sub(double* out, const double* x, const double* y, int64_t n, cudaStream_t s);
// out[k] = a_k . b_k for k < 3 (a1 / a2 may be NULL); part: kPartials doubles; device out[3]
cudaError_t launch_dots(const double* a0, const double* b0, const double* a1, const double* b1,
                        const double* a2, const double* b2, int64_t n, double* part, double* out,
                        cudaStream_t s);

}  // namespace dg
