/*
 * dg.h — C ABI of the B200-native matrix-free DG hot path of arXiv 1805.11930.
 *
 * Problem: find u in V_h^p with a_h(u, v) = l_h(v), i.e. A u = f with
 * A_ij = a_h(psi_j, psi_i) (P:328-330, P:427-430 eq. linear_equation), a_h the WSIPG
 * form with upwind flux (P:333-360 eq. bilinear_form_split), on a
 * structured box of hexahedral cells with the nodal Gauss-Lobatto Q_p basis
 * (P:436-440). The library applies A matrix-free with sum factorisation
 * (§3.1) and runs the block-Jacobi smoother of Alg. 2 whose
 * diagonal blocks D_T = A_{T,T} (P:893-903 eq. block_diag_apply) are inverted
 * iteratively by a cell-local preconditioned Krylov solve (§2.2.1,
 * P:904-911 §3.2).
 *
 * Layout of every vector (u, f, Au, d, du): fp64, cell-major. Cell
 * c = cx + nx*(cy + ny*cz) (x fastest), DoF inside a cell I = i + n*j + n*n*k with
 * n = p+1 (x fastest), i.e. u[c*n^3 + I]. With nranks > 1 a rank holds the z-slab
 * cz in [z_begin, z_end) (dg_local_range), a contiguous range of the global vector,
 * and its pointers address that local range only.
 *
 * Pointers named u/f/Au/d/du are DEVICE pointers (e.g. torch CUDA tensors) on
 * desc.device, owned by the caller. Calls are stream ordered on `cuda_stream`
 * (a cudaStream_t, NULL = legacy default stream) and return before the GPU work
 * completes; statistics are valid after dg_get_stats (which synchronises).
 * The library owns all scratch, halo buffers and the NCCL communicator.
 * Errors: a dg_status; no exception crosses the ABI. dg_last_error() returns a
 * thread-local message for the last failing call on the calling thread.
 */
#ifndef DG_B200_H
#define DG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dg_ctx dg_ctx; /* opaque, owned by the library */

typedef enum {
  DG_OK = 0,
  DG_ERR_INVALID = 1,     /* bad sizes, p outside 1..7, non-positive L, negative K or c, NULL */
  DG_ERR_NOMEM = 2,       /* device allocation failed */
  DG_ERR_CUDA = 3,        /* CUDA runtime error (message in dg_last_error) */
  DG_ERR_NCCL = 4,        /* NCCL unavailable or failed */
  DG_ERR_STATE = 5,       /* call not valid in this context state */
  DG_ERR_UNSUPPORTED = 6  /* valid request outside this build (e.g. no sm_100a device) */
} dg_status;

enum { DG_BC_DIRICHLET = 0, DG_BC_NEUMANN = 1 };
/* local Krylov method; DG_LOCAL_BICGSTAB_THOMAS: BiCGStab right-preconditioned by the tridiagonal
 * part of D_T in DoF order (Thomas algorithm), for strongly convection-dominated
 * blocks where the diagonal fails; p <= 4. DG_LOCAL_GMRES / DG_LOCAL_GMRES_THOMAS:
 * restarted GMRES(k) (the paper's local method for the convection test; k <= 15 at
 * p = 1 and 3, 13 at p = 2, 9 at p = 4) with the diagonal or the tridiagonal right
 * preconditioner; p <= 4 (Krylov basis in tensor memory). dg_get_stats counts Arnoldi steps. */
enum { DG_LOCAL_AUTO = 0, DG_LOCAL_CG = 1, DG_LOCAL_BICGSTAB = 2, DG_LOCAL_BICGSTAB_THOMAS = 3,
       DG_LOCAL_GMRES = 4, DG_LOCAL_GMRES_THOMAS = 5 };
enum { DG_HALO_NCCL = 0, DG_HALO_EXTERNAL = 1 };
/* Kernel variants (dg_set_kernel_variant): the same operator / solver through another kernel of
 * the build, for A/B measurements and for parity tests of every kernel whose speed is reported.
 * 0 = the measured defaults. DG_VARIANT_VOLUME_PREFETCH: the register-prefetch persistent volume
 * kernel at p = 3 (default: the slim one); DG_VARIANT_LINE: line-per-thread kernels at every
 * degree; DG_VARIANT_NO_TMEM: shared-memory p = 3 BiCGStab (default: Krylov vectors in tensor
 * memory); DG_VARIANT_LINE_CG_CTA: the other line-solver kernel at p = 4..6 (defaults: CG one
 * warp per cell at p = 4, CTA-wide at p = 5, 6; BiCGStab one warp per cell at p = 4, 6, CTA-wide
 * at p = 5; the flag swaps them); DG_VARIANT_APPLY_NOFOLD: dg_apply at p = 4 through the warp-mode
 * nodal kernel with face arrays (default: the mass-folded kernel k_apply_fold). */
enum { DG_VARIANT_VOLUME_PREFETCH = 1, DG_VARIANT_LINE = 2, DG_VARIANT_NO_TMEM = 4,
       DG_VARIANT_LINE_CG_CTA = 8, DG_VARIANT_APPLY_NOFOLD = 16 };

typedef struct {
  int32_t nx, ny, nz;        /* GLOBAL cells per axis (uniform cells, D2 of SURVEY §2.1) */
  double Lx, Ly, Lz;         /* box [0,Lx]x[0,Ly]x[0,Lz], > 0 */
  int32_t bc[6];             /* x-, x+, y-, y+, z-, z+ : DG_BC_DIRICHLET / DG_BC_NEUMANN */
  int32_t p;                 /* polynomial degree 1..7 (n = p+1 GL nodes, m = p+1 Gauss points) */
  double alpha;              /* penalty parameter of gamma_F; configs use 2.0 */
  int32_t k_components;      /* 1: scalar K per cell; 3: diagonal (Kx,Ky,Kz) per cell */
  const double* K;           /* HOST, GLOBAL [nx*ny*nz][k_components], >= 0; copied at create */
  double b[3];               /* constant advection field b, used when b_cell is NULL */
  const double* b_cell;      /* HOST, GLOBAL [nx*ny*nz][3] per-cell advection b_T (b = b(x)),
                                finite, or NULL (constant b); copied at create. The volume term uses
                                the cell's b_T, a face b_nu = nu . (b^- + b^+)/2 (DESIGN reading #8) */
  const double* c;           /* HOST, GLOBAL [nx*ny*nz] reaction >= 0, or NULL (c = 0) */
  int32_t rank, nranks;      /* z-slab decomposition; nranks = 1 for a single GPU */
  int32_t halo_mode;         /* DG_HALO_NCCL or DG_HALO_EXTERNAL (caller fills ghost layers) */
  const void* nccl_id;       /* HOST, 128-byte ncclUniqueId (same on all ranks) if NCCL mode and
                                nranks > 1, else NULL */
  int32_t device;            /* CUDA device ordinal of this rank */
} dg_desc;

typedef struct {
  double it_mean, it_std;    /* local Krylov iterations per cell of the last sweep / solve */
  int32_t it_max, it_min;
  int64_t n_cells;           /* local cells */
  int64_t n_nonconverged;    /* cells that hit max_it before ||r|| <= tol ||d|| (not fatal) */
  int64_t it_sum;
} dg_stats;

/* Validates desc, builds the 1D tables (GL nodes, Gauss rule), copies this
 * rank's slice of K / c plus one ghost z-layer to the device, allocates scratch and
 * (NCCL mode, nranks > 1) creates the communicator. *out = NULL on failure. */
dg_status dg_create(const dg_desc* desc, dg_ctx** out);
dg_status dg_destroy(dg_ctx* ctx);

/* This rank's slab: global z-layers [z_begin, z_end) and its DoF count. */
dg_status dg_local_range(const dg_ctx* ctx, int32_t* z_begin, int32_t* z_end, int64_t* n_local_dof);

/* Au = A u, matrix-free: sum-factorised volume terms (Stages 1-3)
 * plus interior/boundary face terms. u, Au: device [n_local_dof], must not alias.
 * With nranks > 1 the face traces of the z-boundary layers are exchanged first (NCCL send/recv
 * of 2 n^2 doubles per column and side, or caller-filled in external mode). */
dg_status dg_apply(dg_ctx* ctx, const double* u, double* Au, void* cuda_stream);

/* One block-Jacobi sweep, Alg. 2 lines 2-4: d = f - A u; for every cell solve
 * D_T du_T = d_T by Jacobi-preconditioned CG (b = 0) or BiCGStab from du = 0 until
 * ||d_T - D_T du_T||_2 <= local_tol ||d_T||_2 or max_it; u <- u + omega du.
 * u: device [n_local_dof] in/out; f: device [n_local_dof]. */
dg_status dg_block_jacobi_sweep(dg_ctx* ctx, double* u, const double* f, double omega,
                                double local_tol, void* cuda_stream);

/* The same sweep out of place: u_new = u + omega D^{-1}(f - A u). u, f, u_new: device
 * [n_local_dof]; u_new must not alias u or f (callers ping-pong two buffers; the in-place form
 * above writes a library scratch vector and copies it back, +16 B/DoF of traffic). */
dg_status dg_block_jacobi_sweep_to(dg_ctx* ctx, const double* u, const double* f, double* u_new,
                                   double omega, double local_tol, void* cuda_stream);

/* z-layer ranges, for streaming (the host<->device copy of one chunk of layers under the compute
 * of another). Single slab only (nranks == 1, else DG_ERR_INVALID).
 * dg_range_granule: *layers = the smallest number of z-layers whose cells fill whole cell groups
 * of every kernel of this context; range bounds must be multiples of it (or the last local layer).
 * dg_apply_range: (A u)_T for the cells T of local z-layers [z_begin, z_end) only (the rows of
 * dg_apply, bit for bit); reads u of layers z_begin-1 .. z_end (the face neighbours,
 * P:345-350). Au elsewhere is untouched.
 * dg_block_jacobi_sweep_range: the out-of-place sweep (Alg. 2) for the cells of
 * [z_begin, z_end): u_new_T = u_T + omega D_T^{-1}(f - A u)_T, bit for bit the values of
 * dg_block_jacobi_sweep_to; reads u of layers z_begin-1 .. z_end and f of the range; u_new
 * elsewhere is untouched. dg_get_stats then reports, per cell, its last local solve.
 * Errors: DG_ERR_INVALID for a NULL pointer, aliasing as above, bounds outside
 * [0, local layers] or not multiples of the granule, nranks > 1; z_begin == z_end is a no-op. */
dg_status dg_range_granule(const dg_ctx* ctx, int32_t* layers);
dg_status dg_apply_range(dg_ctx* ctx, const double* u, double* Au, int32_t z_begin, int32_t z_end,
                         void* cuda_stream);
dg_status dg_block_jacobi_sweep_range(dg_ctx* ctx, const double* u, const double* f, double* u_new,
                                      double omega, double local_tol, int32_t z_begin, int32_t z_end,
                                      void* cuda_stream);

/* Block SOR / SSOR in the red-black cell order (Alg. 3): colour
 * (cx + cy + cz) mod 2 (global indices), red = 0 first. A forward sweep updates all red cells
 * from the current u, then all black cells from the updated u, each cell by
 * u_T <- u_T + omega D_T^{-1} (f - A u)_T with the same local Krylov solve as the block-Jacobi
 * sweep (equal to Alg. 3's (1 - omega) u + omega du with du the new block value, DESIGN reading
 * #17); symmetric != 0 adds the backward sweep (black, then red): block SSOR.
 * Every colour is ordered after all cells of the other colour, so each half-sweep is one fully
 * parallel launch (p <= 3 with nx even: only that colour's cells are launched, updated in place).
 * With nranks > 1 the z-halo is exchanged before every half-sweep (NCCL halo mode only;
 * DG_ERR_UNSUPPORTED in external-halo mode). The per-cell statistics (dg_get_stats) are those of
 * the last half-sweep (0 iterations for the cells it skipped, in either launch mode). */
dg_status dg_block_sor_sweep(dg_ctx* ctx, double* u, const double* f, double omega, double local_tol,
                             int32_t symmetric, void* cuda_stream);

/* Alg. 2 line 3 alone: du_T = (iterative) D_T^{-1} d_T for every local cell. */
dg_status dg_local_block_solve(dg_ctx* ctx, const double* d, double* du, double local_tol,
                               void* cuda_stream);

/* Local Krylov method (DG_LOCAL_AUTO: CG if b == 0 everywhere, else BiCGStab), iteration cap
 * (default 1000; reading #13 of SURVEY §8(c)) and GMRES restart length (0: the largest basis
 * the tensor memory holds: 15 at p = 1, 3, 13 at p = 2, 9 at p = 4; larger values are clamped to
 * it). A CG that breaks down (p^T D_T p <= 0: D_T not SPD) stops and counts as not converged. */
dg_status dg_set_local_solver(dg_ctx* ctx, int32_t method, int32_t max_it, int32_t gmres_restart);

/* Selects the kernel variant bits (DG_VARIANT_*) used by the later calls on ctx. At create they
 * default to the environment switches DG_VOLUME_SLIM=0, DG_KERNEL_FAMILY=line, DG_NO_TMEM=1,
 * DG_LINE_CG_CTA=1 (else 0). Unknown bits -> DG_ERR_INVALID. */
dg_status dg_set_kernel_variant(dg_ctx* ctx, uint32_t variant);

/* Synchronises the last sweep/solve stream and reduces its per-cell iteration counts. */
dg_status dg_get_stats(dg_ctx* ctx, dg_stats* st);

/* SURVEY 8(b)'s one-call forms: dg_block_jacobi_sweep / dg_local_block_solve followed by
 * dg_get_stats (they synchronise cuda_stream; the asynchronous calls above do not). st: host,
 * written on DG_OK; NULL = no statistics (then identical to the plain call). */
dg_status dg_block_jacobi_sweep_stats(dg_ctx* ctx, double* u, const double* f, double omega,
                                      double local_tol, dg_stats* st, void* cuda_stream);
dg_status dg_local_block_solve_stats(dg_ctx* ctx, const double* d, double* du, double local_tol,
                                     dg_stats* st, void* cuda_stream);

/* Component hooks for parity tests:
 *  dg_apply_parts: mask 1 = volume terms a^v, 2 = interior-face terms a^if,
 *                  4 = boundary-face terms a^bf (sums of the selected parts of A u);
 *  dg_block_diag_apply: Du_T = D_T u_T for every cell. */
dg_status dg_apply_parts(dg_ctx* ctx, const double* u, double* out, uint32_t mask, void* cuda_stream);
dg_status dg_block_diag_apply(dg_ctx* ctx, const double* u, double* Du, void* cuda_stream);

/* Ghost buffers (nranks > 1): per slab side the face traces of the neighbouring rank's adjacent
 * z-layer, [nx*ny][2][n^2] doubles: per column the n^2 face values (node n-1 of the lower rank's
 * top layer / node 0 of the upper rank's bottom layer, i + n j order) followed by the n^2 normal-
 * derivative sums sum_k d[k] u_k (d = theta'(1) resp. theta'(0), unscaled). A neighbour enters the
 * face terms only through these, so the halo is 2 n^2 instead of n^3 doubles per
 * column. *ghost_len = nx*ny*2n^2; NULL pointers where the slab touches the domain boundary. */
dg_status dg_ghost_layers(dg_ctx* ctx, double** ghost_lo, double** ghost_hi, int64_t* ghost_len);

/* External halo mode: fills the ghost buffers from the neighbouring ranks' adjacent LAYERS
 * (device, nx*ny cells of n^3 DoF each, the layout of u): lo = the lower rank's top layer,
 * hi = the upper rank's bottom layer; their traces are packed by the same kernel (and the same
 * arithmetic) the NCCL mode uses. Stream ordered; lo / hi may be NULL where there is no such
 * neighbour. */
dg_status dg_fill_ghosts(dg_ctx* ctx, const double* lo, const double* hi, void* cuda_stream);

/* The 1D tables used by the kernels, for parity with the oracle's own: out receives
 * z[n], xq[n], wq[n], A[n*n], D[n*n], M[n*n], d0[n], d1[n] (5n + 3n^2 doubles). */
dg_status dg_tables(int32_t p, double* out);

/* Host-only (no GPU): the z-slab of `rank` among `nranks` for nz global layers,
 * [floor(rank*nz/nranks), floor((rank+1)*nz/nranks)). */
dg_status dg_slab_range(int32_t nz, int32_t rank, int32_t nranks, int32_t* z_begin, int32_t* z_end);

/* Host-only (no GPU): the halo plan of desc's rank. out[0] = DoF offset (in the local vector) of
 * the layer sent to the lower neighbour (or -1), out[1] = offset of the layer sent to the upper
 * neighbour (or -1), out[2] = DoF per layer (nx*ny*n^3), out[3] = lower peer rank (or -1),
 * out[4] = upper peer rank (or -1), out[5] = local DoF count. The lower ghost layer receives the
 * lower peer's out[1] layer and the upper ghost its out[0] layer. */
dg_status dg_halo_plan(const dg_desc* desc, int64_t out[6]);

/* Writes a fresh 128-byte ncclUniqueId (rank 0 broadcasts it to the other ranks). */
dg_status dg_nccl_unique_id(void* out128);

/* ---- Hybrid multigrid with the P0 subspace (Alg. 1) ----------
 * Single rank (nranks = 1) and b = 0 only (the outer iteration is a CG; the paper solves the
 * convection-dominated case with FGMRES and block SSOR instead); otherwise
 * DG_ERR_UNSUPPORTED. The paper's AMG coarse solve (line 4) is replaced by Jacobi-PCG on A^ to
 * coarse_tol (reading #25 of DESIGN.md). Scratch (7 DoF vectors + O(cells)) is allocated on the
 * first call and owned by the context. */
typedef struct {
  int32_t n_pre, n_post;   /* block-Jacobi sweeps before / after the coarse correction */
  double omega;            /* sweep damping (Alg. 2 line 4) */
  double local_tol;        /* local Krylov tolerance of the sweeps */
  double coarse_tol;       /* relative residual tolerance of the coarse Jacobi-PCG */
  int32_t coarse_max_it;
  double rel_tol;          /* outer: ||f - A u||_2 <= rel_tol ||f - A u_0||_2 */
  int32_t max_it;          /* outer iteration cap */
} dg_hybrid_params;

typedef struct {
  int32_t iterations;      /* outer flexible-CG iterations */
  int32_t converged;       /* 1 if rel_tol was reached */
  double rel_residual;     /* final ||r|| / ||r_0|| (recursively updated residual) */
  int32_t vcycles;         /* preconditioner applications */
  int32_t coarse_it_max;   /* largest coarse PCG iteration count over the V-cycles */
  int32_t coarse_nonconverged;  /* V-cycles whose coarse solve hit coarse_max_it */
} dg_hybrid_stats;

/* A^ = P^T A P (eq. galerkin_product; App. A.1) for the local cells, copied to the
 * HOST array Ah[7][n_cells]: row 0 the diagonal, row 1 + f the coupling of cell T to its face-f
 * neighbour (f = 0..5: x-, x+, y-, y+, z-, z+), 0 where there is none. Synchronises. */
dg_status dg_coarse_matrix(dg_ctx* ctx, double* Ah_host);

/* One V-cycle of Alg. 1 from u_0 = 0 as a preconditioner: z = V(r). r, z: device
 * [n_local_dof], must not alias. Stream ordered. */
dg_status dg_hybrid_vcycle(dg_ctx* ctx, const double* r, double* z, const dg_hybrid_params* prm,
                           void* cuda_stream);

/* Solves A u = f by flexible CG (beta = z_new.(r_new - r_old) / z_old.r_old) preconditioned by
 * the V-cycle, from the initial guess in u (device, in/out). Synchronises once per iteration
 * (the scalars of the recurrence are read back); st may be NULL. */
dg_status dg_hybrid_solve(dg_ctx* ctx, double* u, const double* f, const dg_hybrid_params* prm,
                          dg_hybrid_stats* st, void* cuda_stream);

/* ---- Stored-inverse block-Jacobi smoother (the paper's partially
 * matrix-free variant, Table 2) -----------------------------------------------------
 * dg_pmf_setup assembles every D_T from the 1D matrices, inverts it (Gauss-Jordan
 * with partial pivoting in shared memory: the blocks are nonsymmetric for b != 0) and keeps the
 * inverses on the device: n_cells (p+1)^6 doubles. p <= 4 only (otherwise DG_ERR_UNSUPPORTED);
 * DG_ERR_NOMEM if they do not fit. Slab-boundary faces use the ghost-layer coefficients.
 * dg_pmf_sweep: one block-Jacobi sweep with exact local solves, u <- u + omega D^{-1}(f - A u),
 * u in place (device). dg_pmf_block: HOST copy of D_T (inverse = 0) or D_T^{-1} (inverse = 1)
 * of one local cell, nd x nd row-major (test index first), for parity tests (synchronises). */
dg_status dg_pmf_setup(dg_ctx* ctx);
dg_status dg_pmf_sweep(dg_ctx* ctx, double* u, const double* f, double omega, void* cuda_stream);
dg_status dg_pmf_block(dg_ctx* ctx, int64_t cell, int32_t inverse, double* host_out);

/* fp64 FMA-throughput microbenchmark: launches `blocks` x 256 threads,
 * each running 16 independent DFMA chains for `iters` steps on `cuda_stream`; *flops receives
 * the flop count (2 per DFMA). sink: device buffer of blocks*256 doubles (defeats DCE). */
dg_status dg_microbench_dfma(double* sink, int32_t blocks, int32_t iters, int64_t* flops,
                             void* cuda_stream);

/* Kernel launches issued by the last call on ctx (for launch accounting). */
int32_t dg_last_launch_count(const dg_ctx* ctx);

const char* dg_last_error(void);
const char* dg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DG_B200_H */
