// Hybrid multigrid with the P0 subspace (Alg. 1): the P0
// transfer kernels, the coarse matrix A^ = P^T A P as a 7-point stencil, its Jacobi-PCG solve
// in one cooperative kernel, and the vector kernels of the outer flexible CG.
//
//   prolongation  P|_T = (1,...,1)^T: u_i += u^_T for every DoF i of cell T
//   restriction   R = P^T: r^_T = sum_i r_i over the DoF of T
//   A^            P0 functions have zero gradient, so volume diffusion / convection and the
//                 consistency / symmetry face terms vanish in P^T A P (App. A.1, eq.
//                 p0_galerkin1); per face of T with outward normal nu:
//                   interior:  diag += (max(b.nu,0) + gamma_F) |F|,
//                              off  += (min(b.nu,0) - gamma_F) |F|,
//                              gamma_F = alpha p(p+2) <K_T, K_N> / h   (harmonic mean)
//                   Dirichlet: diag += (max(b.nu,0) + alpha p(p+2) K_T / h) |F|
//                   Neumann:   nothing;        reaction: diag += c |T|
//                 (the same face coefficients as the fine operator's setup).
//   coarse solve  the paper's AMG V-cycle is out of scope; A^ is solved by Jacobi-PCG to a
//                 relative tolerance inside one cooperative persistent kernel (grid-wide
//                 syncs between the stencil, the reductions and the updates).
#include <cooperative_groups.h>

#include "dg_hybrid.h"

namespace cg = cooperative_groups;

namespace dg {
namespace {

constexpr int kCoarseThreads = 1024;   // one 1024-thread block per SM for the cooperative coarse solve

__device__ __forceinline__ void cell_coords(const KParams& kp, int cell, int& cx, int& cy, int& cz) {
  cx = cell % kp.nx;
  cy = (cell / kp.nx) % kp.ny;
  cz = cell / (kp.nx * kp.ny);
}

// A^ rows, structure of arrays: Ah[0][T] diagonal, Ah[1 + f][T] coupling to the face-f
// neighbour (f = 2 axis + hi; 0 where there is none).
__global__ void k_coarse_matrix(KParams kp, double* __restrict__ Ah) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= kp.ncells) return;
  const int N = kp.ncells;
  const int nxy = kp.nx * kp.ny;
  int co[3];
  cell_coords(kp, cell, co[0], co[1], co[2]);
  const int dims[3] = {kp.nx, kp.ny, kp.nzl};
  const int step[3] = {1, kp.nx, nxy};
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
  double diag = kp.c ? kp.c[cell] * vol : 0.0;
  for (int f = 0; f < 6; ++f) {
    const int axis = f >> 1, hi = f & 1;
    const double bn = hi ? kp.b[axis] : -kp.b[axis];   // b . nu_T
    const double KT = kp.K[(size_t)(cell + nxy) * 3 + axis];
    const int nc = co[axis] + (hi ? 1 : -1);
    double off = 0.0;
    if (nc >= 0 && nc < dims[axis]) {
      const int nb = cell + (hi ? step[axis] : -step[axis]);
      const double KN = kp.K[(size_t)(nb + nxy) * 3 + axis];
      const double s = KT + KN;
      const double gam = kp.pen * (s > 0.0 ? 2.0 * KT * KN / s : 0.0) * kp.ih[axis];
      diag += (fmax(bn, 0.0) + gam) * kp.fa[axis];
      off = (fmin(bn, 0.0) - gam) * kp.fa[axis];
    } else if (kp.slab_face[f] == FK_DIRICHLET) {
      diag += (fmax(bn, 0.0) + kp.pen * KT * kp.ih[axis]) * kp.fa[axis];
    }
    Ah[(size_t)(1 + f) * N + cell] = off;
  }
  Ah[cell] = diag;
}

// r^_T = sum of the DoF values of cell T (one warp per cell, coalesced)
__global__ void k_restrict(const double* __restrict__ r, double* __restrict__ rh, int ncells, int nd) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int cell = warp; cell < ncells; cell += nwarps) {
    const double* p = r + (size_t)cell * nd;
    double s = 0.0;
    for (int i = lane; i < nd; i += 32) s += p[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rh[cell] = s;
  }
}

// u_i += u^_T(i)
__global__ void k_prolongate_add(double* __restrict__ u, const double* __restrict__ uh, int64_t ndof, int nd) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ndof; i += (int64_t)gridDim.x * blockDim.x)
    u[i] += uh[i / nd];
}

struct CoarseArgs {
  KParams kp;
  const double* Ah;   // [7][N]
  const double* rhs;  // [N]
  double* x;          // [N] out
  double* r;          // [N] work
  double* p;          // [N] work
  double* q;          // [N] work
  double* part;       // [2][3][gridDim.x] block partial sums
  int* its;           // [1] out: iterations (| 1 << 30 if not converged)
  double tol2;
  int max_it;
};

__device__ __forceinline__ double stencil(const CoarseArgs& a, const double* v, int cell) {
  const KParams& kp = a.kp;
  const int N = kp.ncells;
  const int nxy = kp.nx * kp.ny;
  double s = a.Ah[cell] * v[cell];
  // a zero coefficient marks a missing neighbour; its index is never formed
  const double cxl = a.Ah[(size_t)1 * N + cell], cxh = a.Ah[(size_t)2 * N + cell];
  const double cyl = a.Ah[(size_t)3 * N + cell], cyh = a.Ah[(size_t)4 * N + cell];
  const double czl = a.Ah[(size_t)5 * N + cell], czh = a.Ah[(size_t)6 * N + cell];
  if (cxl != 0.0) s = fma(cxl, v[cell - 1], s);
  if (cxh != 0.0) s = fma(cxh, v[cell + 1], s);
  if (cyl != 0.0) s = fma(cyl, v[cell - kp.nx], s);
  if (cyh != 0.0) s = fma(cyh, v[cell + kp.nx], s);
  if (czl != 0.0) s = fma(czl, v[cell - nxy], s);
  if (czh != 0.0) s = fma(czh, v[cell + nxy], s);
  return s;
}

// deterministic block sum of up to 3 values into part[k * gridDim.x + blockIdx.x]
template <int K>
__device__ __forceinline__ void block_partials(double (&v)[K], double* part) {
  __shared__ double red[K][kCoarseThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[k][w] = s;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int i = 0; i < kCoarseThreads / 32; ++i) s += red[threadIdx.x][i];
    part[threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
  __syncthreads();
}
// every block reduces the partials in the same order (same result everywhere)
__device__ __forceinline__ double sum_partials(const double* part, int k) {
  double s = 0.0;
  for (int i = 0; i < (int)gridDim.x; ++i) s += part[k * gridDim.x + i];
  return s;
}

// Jacobi-PCG on A^ x = rhs from x = 0 until ||r|| <= tol ||rhs|| or max_it, in the
// Chronopoulos-Gear form (one reduction phase per iteration: gamma = (r,u), delta = (w,u) and
// ||r||^2 together, w = A^ u), so each iteration costs two grid-wide barriers: after the vector
// updates (u complete before the stencil) and after the block partial sums.
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_pcg(CoarseArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int N = a.kp.ncells;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, ts = gridDim.x * blockDim.x;
  double* P0 = a.part;
  double* P1 = a.part + 3 * gridDim.x;
  double* u = a.r + 3 * (size_t)N;     // work: r, p, q(= z = A p), u, w
  double* w = a.r + 4 * (size_t)N;
  // x = 0, r = rhs, u = D^-1 r
  for (int i = t0; i < N; i += ts) {
    const double r = a.rhs[i];
    a.x[i] = 0.0;
    a.r[i] = r;
    u[i] = r / a.Ah[i];
  }
  grid.sync();
  double alpha = 0.0, gamma_old = 0.0, rr0 = 0.0;
  int it = 0;
  bool conv = false;
  double* part = P0;
  for (;;) {
    // w = A^ u and the three dot products
    {
      double v[3] = {0.0, 0.0, 0.0};
      for (int i = t0; i < N; i += ts) {
        const double wi = stencil(a, u, i);
        w[i] = wi;
        const double ri = a.r[i], ui = u[i];
        v[0] = fma(ri, ui, v[0]);
        v[1] = fma(wi, ui, v[1]);
        v[2] = fma(ri, ri, v[2]);
      }
      block_partials<3>(v, part);
    }
    grid.sync();
    const double gamma = sum_partials(part, 0), delta = sum_partials(part, 1), rr = sum_partials(part, 2);
    part = part == P0 ? P1 : P0;   // the next phase writes the other buffer
    if (it == 0) {
      rr0 = rr;
      if (rr0 == 0.0) { conv = true; break; }
    } else if (rr <= a.tol2 * rr0) {
      conv = true;
      break;
    }
    if (it >= a.max_it) break;
    double beta = 0.0, den = delta;
    if (it > 0) {
      beta = gamma / gamma_old;
      den = delta - beta * gamma / alpha;
    }
    if (!(den > 0.0)) break;   // breakdown: A^ or the preconditioner not SPD
    alpha = gamma / den;
    gamma_old = gamma;
    // q = w + beta q (= A p), p = u + beta p, x += alpha p, r -= alpha q, u = D^-1 r
    for (int i = t0; i < N; i += ts) {
      const double q = fma(beta, it > 0 ? a.q[i] : 0.0, w[i]);
      const double pp = fma(beta, it > 0 ? a.p[i] : 0.0, u[i]);
      a.q[i] = q;
      a.p[i] = pp;
      a.x[i] = fma(alpha, pp, a.x[i]);
      const double r = fma(-alpha, q, a.r[i]);
      a.r[i] = r;
      u[i] = r / a.Ah[i];
    }
    ++it;
    grid.sync();
  }
  if (t0 == 0) a.its[0] = conv ? it : (it | (1 << 30));
}

// y = a x + b y
__global__ void k_axpby(double* __restrict__ y, double a, const double* __restrict__ x, double b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}
// out = x - y
__global__ void k_sub(double* __restrict__ out, const double* __restrict__ x, const double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] - y[i];
}
// up to three dot products: block partials, then one block sums them in a fixed order
__global__ void __launch_bounds__(kCoarseThreads) k_dots(const double* a0, const double* b0, const double* a1,
                                                         const double* b1, const double* a2, const double* b2,
                                                         int64_t n, double* part) {
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    v[0] = fma(a0[i], b0[i], v[0]);
    if (a1) v[1] = fma(a1[i], b1[i], v[1]);
    if (a2) v[2] = fma(a2[i], b2[i], v[2]);
  }
  block_partials<3>(v, part);
}
// fixed-order final sum: thread t adds partials t, t + 256, ... (same order every call), then
// a fixed tree over the 256 thread sums
__global__ void __launch_bounds__(256) k_dots_final(const double* part, int nblocks, double* out) {
  __shared__ double sh[3][256];
  for (int k = 0; k < 3; ++k) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += 256) s += part[k * nblocks + i];
    sh[k][threadIdx.x] = s;
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < 3; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 3) out[threadIdx.x] = sh[threadIdx.x][0];
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

int vec_blocks() { return 4 * sm_count(); }

cudaError_t launch_coarse_matrix(const KParams& kp, double* Ah, cudaStream_t s) {
  if (kp.ncells == 0) return cudaSuccess;
  k_coarse_matrix<<<(kp.ncells + 255) / 256, 256, 0, s>>>(kp, Ah);
  return cudaGetLastError();
}

cudaError_t launch_restrict(const double* r, double* rh, int ncells, int nd, cudaStream_t s) {
  k_restrict<<<2 * sm_count(), 256, 0, s>>>(r, rh, ncells, nd);
  return cudaGetLastError();
}

cudaError_t launch_prolongate_add(double* u, const double* uh, int64_t ndof, int nd, cudaStream_t s) {
  k_prolongate_add<<<4 * sm_count(), 256, 0, s>>>(u, uh, ndof, nd);
  return cudaGetLastError();
}

cudaError_t launch_coarse_pcg(const KParams& kp, const double* Ah, const double* rhs, double* x,
                              double* work, double* part, int* its, double tol, int max_it,
                              cudaStream_t s) {
  static int blocks = 0;
  if (blocks == 0) {
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_pcg, kCoarseThreads, 0);
    if (e != cudaSuccess) return e;
    blocks = per_sm * sm_count();
    if (blocks > kMaxCoarseBlocks) blocks = kMaxCoarseBlocks;
  }
  const int N = kp.ncells;
  CoarseArgs a;
  a.kp = kp;
  a.Ah = Ah;
  a.rhs = rhs;
  a.x = x;
  a.r = work;
  a.p = work + N;
  a.q = work + 2 * (size_t)N;
  a.part = part;
  a.its = its;
  a.tol2 = tol * tol;
  a.max_it = max_it;
  // one block per SM (fewer blocks make the grid-wide barriers cheaper; measured on C2 / C3 / C5)
  int grid = (N + kCoarseThreads - 1) / kCoarseThreads;
  grid = grid < sm_count() ? grid : sm_count();
  grid = grid < blocks ? grid : blocks;
  if (grid < 1) grid = 1;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)k_coarse_pcg, dim3(grid), dim3(kCoarseThreads), args, 0, s);
}

cudaError_t launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t s) {
  k_axpby<<<vec_blocks(), 256, 0, s>>>(y, a, x, b, n);
  return cudaGetLastError();
}

cudaError_t launch_sub(double* out, const double* x, const double* y, int64_t n, cudaStream_t s) {
  k_sub<<<vec_blocks(), 256, 0, s>>>(out, x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_dots(const double* a0, const double* b0, const double* a1, const double* b1,
                        const double* a2, const double* b2, int64_t n, double* part, double* out,
                        cudaStream_t s) {
  const int nb = vec_blocks();
  k_dots<<<nb, kCoarseThreads, 0, s>>>(a0, b0, a1, b1, a2, b2, n, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_dots_final<<<1, 256, 0, s>>>(part, nb, out);
  return cudaGetLastError();
}

}  // namespace dg
