// Degree dispatch of the fp64 sm_100a kernels (arXiv 1805.11930) and the DFMA microbenchmark.
// The kernels themselves are in dg_kernels_impl.cuh / dg_plane.cuh, compiled once per degree.
#include "dg_degree.h"

namespace dg {
namespace {

#define DG_DISPATCH(p, CALL)                          \
  switch (p) {                                        \
    case 1: { constexpr int N = 2; return CALL; }     \
    case 2: { constexpr int N = 3; return CALL; }     \
    case 3: { constexpr int N = 4; return CALL; }     \
    case 4: { constexpr int N = 5; return CALL; }     \
    case 5: { constexpr int N = 6; return CALL; }     \
    case 6: { constexpr int N = 7; return CALL; }     \
    case 7: { constexpr int N = 8; return CALL; }     \
    default: return cudaErrorInvalidValue;            \
  }

__global__ void __launch_bounds__(256) k_dfma(double* sink, int iters) {
  double a[16];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1e-3 * i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], x, y);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  sink[blockIdx.x * 256 + threadIdx.x] = s;
}

struct DVec { double d[kMaxN]; };

template <int N>
__global__ void __launch_bounds__(256) k_pack_traces(const double* __restrict__ layer, int ncol, int top,
                                                     DVec d, double* __restrict__ out) {
  constexpr int N2 = N * N, N3 = N * N * N;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;   // (col, face node)
  if (e >= ncol * N2) return;
  const int col = e / N2, node = e % N2;
  const double* c = layer + (size_t)col * N3 + node;
  double g = 0.0;
#pragma unroll
  for (int k = 0; k < N; ++k) g = fma(d.d[k], c[k * N2], g);   // the receivers' summation order
  out[(size_t)col * 2 * N2 + node] = c[(top ? N - 1 : 0) * N2];
  out[(size_t)col * 2 * N2 + N2 + node] = g;
}

}  // namespace

cudaError_t launch_pack_traces(int p, const Tables1D& t, const double* layer, int ncol, int top,
                               double* out, cudaStream_t s) {
  DVec d{};
  for (int i = 0; i < t.n; ++i) d.d[i] = top ? t.d1[i] : t.d0[i];
  const int n = p + 1, items = ncol * n * n;
  if (items == 0) return cudaSuccess;
  const int blocks = (items + 255) / 256;
  switch (p) {
    case 1: k_pack_traces<2><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 2: k_pack_traces<3><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 3: k_pack_traces<4><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 4: k_pack_traces<5><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 5: k_pack_traces<6><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 6: k_pack_traces<7><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    case 7: k_pack_traces<8><<<blocks, 256, 0, s>>>(layer, ncol, top, d, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_dfma_bench(double* sink, int blocks, int iters, cudaStream_t s) {
  k_dfma<<<blocks, 256, 0, s>>>(sink, iters);
  return cudaGetLastError();
}

int solver_group_cells(int p) {
  switch (p) {
    case 1: return Deg<2>::solver_group_cells();
    case 2: return Deg<3>::solver_group_cells();
    case 3: return Deg<4>::solver_group_cells();
    default: return 0;
  }
}

static int lcm_i(int a, int b) {
  int x = a, y = b;
  while (y) { const int t = x % y; x = y; y = t; }
  return a / x * b;
}
int range_group_cells(int p) {
  if (p >= 1 && p <= 3) {   // the GMRES translation unit's groups too
    const int a = p == 1 ? Deg<2>::group_lcm() : (p == 2 ? Deg<3>::group_lcm() : Deg<4>::group_lcm());
    return lcm_i(a, gmres_group_cells(p));
  }
  switch (p) {
    case 1: return Deg<2>::group_lcm();
    case 2: return Deg<3>::group_lcm();
    case 3: return Deg<4>::group_lcm();
    case 4: return Deg<5>::group_lcm();
    case 5: return Deg<6>::group_lcm();
    case 6: return Deg<7>::group_lcm();
    case 7: return Deg<8>::group_lcm();
    default: return 0;
  }
}

bool upload_tables(int p, const Tables1D& t, cudaError_t* err) {
  switch (p) {
    case 1: return Deg<2>::upload(t, err) && upload_gmres(p, t, err);
    case 2: return Deg<3>::upload(t, err) && upload_gmres(p, t, err);
    case 3: return Deg<4>::upload(t, err) && upload_gmres(p, t, err);
    case 4: return Deg<5>::upload(t, err);
    case 5: return Deg<6>::upload(t, err);
    case 6: return Deg<7>::upload(t, err);
    case 7: return Deg<8>::upload(t, err);
    default: *err = cudaErrorInvalidValue; return false;
  }
}

cudaError_t launch_apply(int p, const KParams& kp, const double* u, double* out, cudaStream_t s) {
  // without interior-face terms no neighbour data is needed (e.g. the volume-only hook)
  const int with_nbr = (kp.mask & 2u) ? 1 : 0;
  DG_DISPATCH(p, (Deg<N>::apply(kp, u, out, s, with_nbr)));
}

cudaError_t launch_block_diag_apply(int p, const KParams& kp, const double* u, double* out,
                                    cudaStream_t s) {
  KParams k2 = kp;
  k2.mask = 7u;
  DG_DISPATCH(p, (Deg<N>::apply(k2, u, out, s, 0)));
}

cudaError_t launch_local_solve(int p, int method, const KParams& kp0, const double* d, double* du,
                               cudaStream_t s) {
  KParams kp = kp0;
  kp.mask = 7u;
  DG_DISPATCH(p, (Deg<N>::solve(method, false, kp, d, nullptr, du, s)));
}

cudaError_t launch_sweep(int p, int method, const KParams& kp0, const double* u, const double* f,
                         double* u_new, cudaStream_t s) {
  KParams kp = kp0;
  kp.mask = 7u;
  DG_DISPATCH(p, (Deg<N>::solve(method, true, kp, u, f, u_new, s)));
}

}  // namespace dg
