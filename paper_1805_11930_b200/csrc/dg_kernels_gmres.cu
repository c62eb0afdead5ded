// The local GMRES kernels at p = 1..3 (n = 2..4), compiled with four-warp plane CTAs (the other
// plane kernels run two-warp CTAs): the Krylov basis fills 256 (n = 2, 3) or all 512 (n = 4)
// tensor-memory columns per CTA and a warp reaches only its own lane quadrant, so one CTA must
// span the four quadrants for the tensor memory of an SM to be used. Everything here lives in
// this unit's anonymous namespace, its own copy of the constant tables included (uploaded by
// upload_tables together with the degree's other unit).
#define DG_PL_WARPS2 4
#define DG_PL_WARPS3 4
#define DG_PL_WARPS4 4
#define DG_GMRES_TU 1
#include "dg_kernels_impl.cuh"

namespace dg {
bool upload_gmres(int p, const Tables1D& t, cudaError_t* err) {
  switch (p) {
    case 1: return upload_n<2>(t, err);
    case 2: return upload_n<3>(t, err);
    case 3: return upload_n<4>(t, err);
    default: *err = cudaErrorInvalidValue; return false;
  }
}
cudaError_t solve_gmres(int p, int method, bool sweep, const KParams& kp, const double* in,
                        const double* f, double* out, cudaStream_t s) {
  switch (p) {
    case 1: return sweep ? gmres_n<2, true>(method, kp, in, f, out, s) : gmres_n<2, false>(method, kp, in, f, out, s);
    case 2: return sweep ? gmres_n<3, true>(method, kp, in, f, out, s) : gmres_n<3, false>(method, kp, in, f, out, s);
    case 3: return sweep ? gmres_n<4, true>(method, kp, in, f, out, s) : gmres_n<4, false>(method, kp, in, f, out, s);
    default: return cudaErrorInvalidValue;
  }
}
int gmres_group_cells(int p) {
  return p == 1 ? pk::Geo<2>::C : (p == 2 ? pk::Geo<3>::C : (p == 3 ? pk::Geo<4>::C : 0));
}
}  // namespace dg
