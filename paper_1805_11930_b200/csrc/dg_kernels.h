// Internal (non-ABI) launch interface of the fp64 sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dg_tables.h"

namespace dg {

enum FaceKind : int32_t { FK_DIRICHLET = 0, FK_NEUMANN = 1, FK_GHOST = 2 };
// kernel variant bits (= DG_VARIANT_* of dg.h)
enum : uint32_t { VAR_VOLUME_PREFETCH = 1u, VAR_LINE = 2u, VAR_NO_TMEM = 4u, VAR_LINE_CG_CTA = 8u,
                  VAR_APPLY_NOFOLD = 16u };

// Everything a kernel needs about the local slab (passed by value).
struct KParams {
  int32_t nx, ny, nzl, ncells;   // local slab: nzl z-layers, ncells = nx*ny*nzl
  double h[3];                   // cell sizes
  double ih[3];                  // 1 / h
  double sb[3];                  // |T| b_k / h_k  (volume advection scaling)
  double fa[3];                  // face areas |F| of x-, y-, z-faces: hy*hz, hx*hz, hx*hy
  double pen;                    // alpha * p * (p + d - 1), d = 3
  double b[3];                   // constant advection
  int32_t slab_face[6];          // x-,x+,y-,y+,z-,z+ of the slab: FaceKind
  const double* K;               // [(nzl+2)*nx*ny][3] diagonal K, z-shifted by one ghost layer
  const double* c;               // [ncells] reaction or nullptr
  const double* bc;              // [(nzl+2)*nx*ny][3] per-cell b (ghost layers as K) or nullptr:
                                 // constant kp.b; volume: the cell's b, faces: (b^- + b^+)/2 . nu
  const double* ghost_lo;        // [nx*ny][2][n^2] face traces of the lower rank's top layer (or nullptr)
  const double* ghost_hi;        // [nx*ny][2][n^2] face traces of the upper rank's bottom layer
                                 // (per column: the face values, then the normal-derivative sums
                                 // sum_k d[k] u_k, unscaled; see ghost_trace / launch_pack_traces)
  uint32_t mask;                 // 1 volume, 2 interior faces, 4 boundary faces
  int32_t max_it;
  int32_t krestart;              // GMRES restart length (0: the compiled basis size)
  double tol2;                   // local_tol^2
  double omega;
  int32_t* its;                  // [ncells] iterations of the last solve
  int32_t colour;                // -1: every cell; 0 / 1: only cells with (cx+cy+cz) % 2 == colour
                                 // are updated (multicolour block SOR), the others pass through
  int32_t zoff;                  // global z index of the slab's first layer (for the colour)
  const int32_t* gperm;          // order in which the solver CTAs take the cell groups (longest
                                 // first: groups with Dirichlet faces), nullptr = in order
  uint32_t variant;              // VAR_* kernel variant bits (0 = the measured defaults)
  int32_t gsplit;                // 0: every cell group; 1: the groups off the slab's ghost faces
                                 // (launched before the halo arrives); 2: the others (after it)
  int32_t gfirst, glast;         // the interior groups [gfirst, glast) of a split launch
  int32_t cfirst, clast;         // gsplit = 3 (dg_apply_range / dg_block_jacobi_sweep_range): the
                                 // cells [cfirst, clast), group-aligned (range_group_cells)
  int32_t cmap;                  // 1: the cell groups enumerate the cells of kp.colour only (nx even;
                                 // group_cell), the other colour is not touched
};

// The z-face of `cell` on side hi is a slab-boundary face whose neighbour is a ghost-layer
// trace record (2 n^2 doubles: the neighbour's face values and normal-derivative sums).
__host__ __device__ inline bool ghost_trace(const KParams& kp, int cell, int hi) {
  const int nxy = kp.nx * kp.ny;
  return hi ? (kp.slab_face[5] == FK_GHOST && cell >= kp.ncells - nxy)
            : (kp.slab_face[4] == FK_GHOST && cell >= 0 && cell < nxy);
}

// the cell is outside the colour of a multicolour half-sweep (kp.colour >= 0, masked mode)
__host__ __device__ inline bool skip_cell(const KParams& kp, int cell) {
  if (kp.colour < 0 || kp.cmap) return false;
  const int cx = cell % kp.nx, cy = (cell / kp.nx) % kp.ny, cz = cell / (kp.nx * kp.ny) + kp.zoff;
  return ((cx + cy + cz) & 1) != kp.colour;
}

// Cell group of this CTA: a split launch (interior groups, or the slab-boundary ones), else the
// solvers' longest-first order (perm, plane solvers only), else blockIdx.x.
#ifdef __CUDACC__
__device__ inline int block_group(const KParams& kp, bool perm) {
  const int b = blockIdx.x;
  if (kp.gsplit == 1 || kp.gsplit == 3) return kp.gfirst + b;
  if (kp.gsplit == 2) return b < kp.gfirst ? b : kp.glast + (b - kp.gfirst);
  return (perm && kp.gperm) ? kp.gperm[b] : b;
}
#endif

// Number of CTAs of a launch with C cells per group under kp.gsplit; sets gfirst / glast. The
// interior groups hold no cell of a layer next to a ghost (slab-boundary) face.
inline int split_groups(KParams& kp, int C) {
  const int items = kp.cmap ? kp.ncells / 2 : kp.ncells;
  const int ng = (items + C - 1) / C;
  if (kp.gsplit == 3 && !kp.cmap) {   // the groups of the cell range [cfirst, clast)
    kp.gfirst = kp.cfirst / C;
    kp.glast = (kp.clast + C - 1) / C;
    if (kp.glast > ng) kp.glast = ng;
    return kp.glast > kp.gfirst ? kp.glast - kp.gfirst : 0;
  }
  if (kp.gsplit == 0 || kp.cmap) {
    kp.gsplit = 0;
    return ng;
  }
  const int nxy = kp.nx * kp.ny;
  const int b0 = kp.slab_face[4] == FK_GHOST ? nxy : 0;
  const int b1 = kp.ncells - (kp.slab_face[5] == FK_GHOST ? nxy : 0);
  int gf = (b0 + C - 1) / C, gl = b1 / C;
  if (gl < gf) gl = gf;
  if (gl > ng) gl = ng;
  kp.gfirst = gf;
  kp.glast = gl;
  return kp.gsplit == 1 ? gl - gf : gf + (ng - gl);
}

// Cell of slot cs of the group starting at item g0: consecutive cells, or (kp.cmap) the
// (g0 + cs)-th cell of colour kp.colour in lexicographic order (nx even: nx / 2 per row);
// -1 past the end.
__host__ __device__ inline int group_cell(const KParams& kp, int g0, int cs) {
  const int m = g0 + cs;
  if (!kp.cmap) return m < kp.ncells ? m : -1;
  const int half = kp.nx >> 1;
  if (m >= kp.ncells / 2) return -1;
  const int row = m / half, i = m - row * half;
  const int cy = row % kp.ny, cz = row / kp.ny;
  return 2 * i + ((kp.colour + cy + cz + kp.zoff) & 1) + kp.nx * row;
}
__host__ __device__ inline int group_items(const KParams& kp) { return kp.cmap ? kp.ncells / 2 : kp.ncells; }

enum LocalMethod : int32_t { LM_CG = 1, LM_BICGSTAB = 2, LM_BICGSTAB_THOMAS = 3, LM_GMRES = 4, LM_GMRES_THOMAS = 5 };

bool upload_tables(int p, const Tables1D& t, cudaError_t* err);

// local GMRES at p = 1..3 (n <= 4): kernels of their own translation unit with four-warp plane
// CTAs (dg_kernels_gmres.cu); its table upload, launcher and cells per CTA
bool upload_gmres(int p, const Tables1D& t, cudaError_t* err);
cudaError_t solve_gmres(int p, int method, bool sweep, const KParams& kp, const double* in,
                        const double* f, double* out, cudaStream_t s);
int gmres_group_cells(int p);

// cells per CTA of the plane local solvers for degree p (0 when the line family runs them)
int solver_group_cells(int p);
// least common multiple of the cells per CTA of every kernel an apply or a sweep of degree p can
// launch (the granule of the cell ranges of dg_apply_range / dg_block_jacobi_sweep_range)
int range_group_cells(int p);

// Au (or selected parts) for all local cells.
cudaError_t launch_apply(int p, const KParams& kp, const double* u, double* out, cudaStream_t s);
// D_T u_T for all local cells.
cudaError_t launch_block_diag_apply(int p, const KParams& kp, const double* u, double* out,
                                    cudaStream_t s);
// du = D^{-1} d (iterative, per cell).
cudaError_t launch_local_solve(int p, int method, const KParams& kp, const double* d, double* du,
                               cudaStream_t s);
// u_new = u + omega D^{-1}(f - A u).
cudaError_t launch_sweep(int p, int method, const KParams& kp, const double* u, const double* f,
                         double* u_new, cudaStream_t s);

// Face traces of a z-layer for the neighbouring rank (the neighbour enters a face
// term only through its trace and its normal derivative): layer = ncol cells of n^3 DoF; out
// [ncol][2][n^2]: top = 0: node-0 values and sum_k d0[k] u_k (for the rank below), top = 1:
// node-(n-1) values and sum_k d1[k] u_k (for the rank above), summed in the kernels' order.
cudaError_t launch_pack_traces(int p, const Tables1D& t, const double* layer, int ncol, int top,
                               double* out, cudaStream_t s);

// fp64 FMA peak microbenchmark: blocks x 256 threads, 16 chains x iters DFMA each.
cudaError_t launch_dfma_bench(double* sink, int blocks, int iters, cudaStream_t s);

}  // namespace dg
