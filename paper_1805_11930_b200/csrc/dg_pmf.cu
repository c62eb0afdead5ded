// Stored-inverse block-Jacobi smoother (the paper's partially matrix-free variant, P:966-972,
// P:1101-1120 Table 2), as a direct comparison point for the matrix-free
// iterative local solve on B200: D_T is assembled once per cell from the 1D matrices
// (volume + self-face terms, each a Kronecker product on the affine cell), inverted
// in shared memory by in-place Gauss-Jordan elimination with partial (row) pivoting (the blocks
// are nonsymmetric for b != 0), and stored TRANSPOSED in HBM; a sweep is then d = f - A u (the
// matrix-free apply) followed by one dense matvec per cell, u + omega D_T^{-1} d, whose warp
// reads row J of the stored transpose (= column J of the inverse) contiguously. Memory:
// n_cells (p+1)^6 doubles (C3: 33 GB), i.e. p <= 4 on a 180 GB B200.
#include "dg_pmf.h"

namespace dg {
namespace {

// per-cell coefficients of D_T: the volume scalings and the self-face parameters of each face
struct CellCoef {
  double vc[4];     // K_a |T| / h_a^2 (a = x, y, z), c |T|
  double vb[3];     // |T| b_a / h_a (the cell's advection, volume term)
  double sa[6];     // value test:      sa a + sg g / h_a  (a = trace, g = normal derivative)
  double sg[6];
  double ta[6];     // derivative test: ta a
};

__device__ void cell_coef(const KParams& kp, int cell, CellCoef& cc) {
  const int nxy = kp.nx * kp.ny;
  const int co[3] = {cell % kp.nx, (cell / kp.nx) % kp.ny, cell / nxy};
  const int dims[3] = {kp.nx, kp.ny, kp.nzl};
  const int step[3] = {1, kp.nx, nxy};
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
  const double* bT = kp.bc ? kp.bc + (size_t)(cell + nxy) * 3 : kp.b;
  for (int a = 0; a < 3; ++a) cc.vc[a] = kp.K[(size_t)(cell + nxy) * 3 + a] * vol * kp.ih[a] * kp.ih[a];
  for (int a = 0; a < 3; ++a) cc.vb[a] = vol * bT[a] * kp.ih[a];
  cc.vc[3] = kp.c ? kp.c[cell] * vol : 0.0;
  for (int f = 0; f < 6; ++f) {
    const int axis = f >> 1, hi = f & 1;
    const double KT = kp.K[(size_t)(cell + nxy) * 3 + axis];
    const double sgn = hi ? -1.0 : 1.0;                // the consistency terms carry nu_T
    const int nc = co[axis] + (hi ? 1 : -1);
    cc.sa[f] = cc.sg[f] = cc.ta[f] = 0.0;
    // interior face (in the slab, or across the slab boundary: the neighbour's K and b are in the
    // ghost layers of kp.K / kp.bc)
    long kidx = -1;
    if (nc >= 0 && nc < dims[axis]) kidx = cell + (hi ? step[axis] : -step[axis]) + nxy;
    else if (kp.slab_face[f] == FK_GHOST) kidx = hi ? (long)(kp.nzl + 1) * nxy + co[0] + kp.nx * co[1]
                                                    : co[0] + kp.nx * co[1];
    if (kidx >= 0) {
      const double KN = kp.K[(size_t)kidx * 3 + axis];
      const double bf = kp.bc ? 0.5 * (bT[axis] + kp.bc[(size_t)kidx * 3 + axis]) : bT[axis];
      const double bn = hi ? bf : -bf;                 // b_F . nu_T (reading #8)
      const double s = KT + KN;
      const double wT = s > 0.0 ? KN / s : 0.5;
      const double gam = kp.pen * (s > 0.0 ? 2.0 * KT * KN / s : 0.0) * kp.ih[axis];
      cc.sa[f] = fmax(bn, 0.0) + gam;
      cc.sg[f] = sgn * wT * KT;
      cc.ta[f] = sgn * wT * KT * kp.ih[axis];
    } else if (kp.slab_face[f] == FK_DIRICHLET) {
      const double bn = hi ? bT[axis] : -bT[axis];
      cc.sa[f] = fmax(bn, 0.0) + kp.pen * KT * kp.ih[axis];
      cc.sg[f] = sgn * KT;
      cc.ta[f] = sgn * KT * kp.ih[axis];
    }
  }
}

// 1D self-face block of axis a at (r, c): sum over the two faces of
// sa e_r e_c + sg/h e_r d_c + ta d_r e_c   (e, d: end-point values / derivatives of the basis)
__device__ __forceinline__ double face1d(const Mat1D& t, const CellCoef& cc, const KParams& kp, int a,
                                         int r, int c) {
  const double ih = kp.ih[a];
  const double lo = cc.sa[2 * a] * t.e0[r] * t.e0[c] + cc.sg[2 * a] * ih * t.e0[r] * t.d0[c] +
                    cc.ta[2 * a] * t.d0[r] * t.e0[c];
  const double hi = cc.sa[2 * a + 1] * t.e1[r] * t.e1[c] + cc.sg[2 * a + 1] * ih * t.e1[r] * t.d1[c] +
                    cc.ta[2 * a + 1] * t.d1[r] * t.e1[c];
  return lo + hi;
}

// D_T[I][J], I = i + n j + n^2 k (test), J likewise (trial)
__device__ double dt_entry(const Mat1D& t, const CellCoef& cc, const KParams& kp, int I, int J) {
  const int n = t.n;
  const int i = I % n, j = (I / n) % n, k = I / (n * n);
  const int ip = J % n, jp = (J / n) % n, kp_ = J / (n * n);
  const double Mx = t.M[i * n + ip], My = t.M[j * n + jp], Mz = t.M[k * n + kp_];
  double v = cc.vc[0] * t.S[i * n + ip] * My * Mz + cc.vc[1] * Mx * t.S[j * n + jp] * Mz +
             cc.vc[2] * Mx * My * t.S[k * n + kp_] + cc.vc[3] * Mx * My * Mz;
  v -= cc.vb[0] * t.C[i * n + ip] * My * Mz + cc.vb[1] * Mx * t.C[j * n + jp] * Mz +
       cc.vb[2] * Mx * My * t.C[k * n + kp_];
  v += kp.fa[0] * face1d(t, cc, kp, 0, i, ip) * My * Mz;
  v += kp.fa[1] * Mx * face1d(t, cc, kp, 1, j, jp) * Mz;
  v += kp.fa[2] * Mx * My * face1d(t, cc, kp, 2, k, kp_);
  return v;
}

// one CTA per cell: assemble D_T in shared memory, invert in place by Gauss-Jordan elimination
// with partial pivoting (the pivot row of column k is the largest |A_ik|, i >= k, found by warp 0;
// rows are swapped, and the inverse's columns are swapped back in reverse order at the end), and
// write the inverse TRANSPOSED (out[J][I] = D^{-1}[I][J]) — or, invert = 0, D_T itself, row-major
__global__ void k_pmf_factor(KParams kp, Mat1D t, int nd, int cell_first, int invert, double* __restrict__ out) {
  extern __shared__ double Am[];
  __shared__ CellCoef cc;
  __shared__ double piv;
  __shared__ int perm[kMaxN * kMaxN * kMaxN];
  const int cell = cell_first + blockIdx.x;
  if (threadIdx.x == 0) cell_coef(kp, cell, cc);
  __syncthreads();
  for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) Am[e] = dt_entry(t, cc, kp, e / nd, e % nd);
  __syncthreads();
  if (invert) {
    for (int k = 0; k < nd; ++k) {
      if (threadIdx.x < 32) {   // pivot search in column k, rows k..nd-1 (first maximum wins)
        double best = -1.0;
        int bi = k;
        for (int i = k + (int)threadIdx.x; i < nd; i += 32) {
          const double v = fabs(Am[i * nd + k]);
          if (v > best) { best = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (threadIdx.x == 0) perm[k] = bi;
      }
      __syncthreads();
      const int pr = perm[k];
      if (pr != k)
        for (int j = threadIdx.x; j < nd; j += blockDim.x) {
          const double a = Am[k * nd + j];
          Am[k * nd + j] = Am[pr * nd + j];
          Am[pr * nd + j] = a;
        }
      __syncthreads();
      if (threadIdx.x == 0) piv = 1.0 / Am[k * nd + k];
      __syncthreads();
      const double p = piv;
      // row k scaled (column k excluded)
      for (int j = threadIdx.x; j < nd; j += blockDim.x)
        if (j != k) Am[k * nd + j] *= p;
      __syncthreads();
      // eliminate column k from the other rows; column k becomes -A_ik p
      for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
        const int i = e / nd, j = e % nd;
        if (i != k && j != k) Am[e] = fma(-Am[i * nd + k], Am[k * nd + j], Am[e]);
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nd; i += blockDim.x)
        if (i != k) Am[i * nd + k] = -Am[i * nd + k] * p;
      if (threadIdx.x == 0) Am[k * nd + k] = p;
      __syncthreads();
    }
    // (P A)^{-1} = A^{-1} P^T: undo the row swaps as column swaps, last first
    for (int k = nd - 1; k >= 0; --k) {
      const int pr = perm[k];
      if (pr != k)
        for (int i = threadIdx.x; i < nd; i += blockDim.x) {
          const double a = Am[i * nd + k];
          Am[i * nd + k] = Am[i * nd + pr];
          Am[i * nd + pr] = a;
        }
      __syncthreads();
    }
  }
  double* o = out + (size_t)blockIdx.x * nd * nd;
  for (int e = threadIdx.x; e < nd * nd; e += blockDim.x)
    o[e] = invert ? Am[(e % nd) * nd + e / nd] : Am[e];
}

// u_new = u + omega Dinv (f - Au), one warp per cell: lane l accumulates rows l, l+32, ...; at
// step J the warp reads row J of the stored transpose, DinvT[J][l] = Dinv[l][J], coalesced.
// u and out may alias (each element is read by the lane that writes it): no __restrict__.
template <int ND>
__global__ void __launch_bounds__(256) k_pmf_sweep(int ncells, const double* __restrict__ Dinv,
                                                   const double* u, const double* __restrict__ f,
                                                   const double* __restrict__ Au, double omega,
                                                   double* out) {
  constexpr int R = (ND + 31) / 32;
  __shared__ double dsh[8][ND];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int cell = warp; cell < ncells; cell += nwarps) {
    const size_t base = (size_t)cell * ND;
    for (int I = lane; I < ND; I += 32) dsh[w][I] = f[base + I] - Au[base + I];
    __syncwarp();
    const double* D = Dinv + (size_t)cell * ND * ND;
    double y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = 0.0;
#pragma unroll 4
    for (int J = 0; J < ND; ++J) {
      const double dj = dsh[w][J];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int I = lane + 32 * r;
        if (I < ND) y[r] = fma(__ldcs(D + (size_t)J * ND + I), dj, y[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int I = lane + 32 * r;
      if (I < ND) out[base + I] = fma(omega, y[r], u[base + I]);
    }
    __syncwarp();
  }
}

int sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

void pmf_tables(const Tables1D& tab, Mat1D* m) {
  const int n = tab.n;
  m->n = n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0, c = 0.0;
      for (int q = 0; q < n; ++q) {
        s += tab.wq[q] * tab.G[q * n + i] * tab.G[q * n + j];   // int th_i' th_j'
        c += tab.wq[q] * tab.G[q * n + i] * tab.A[q * n + j];   // int th_i' th_j  (test derivative)
      }
      m->M[i * n + j] = tab.M[i * n + j];
      m->S[i * n + j] = s;
      m->C[i * n + j] = c;
    }
  for (int i = 0; i < n; ++i) {
    m->e0[i] = i == 0 ? 1.0 : 0.0;       // nodal basis on Gauss-Lobatto nodes: end values
    m->e1[i] = i == n - 1 ? 1.0 : 0.0;
    m->d0[i] = tab.d0[i];
    m->d1[i] = tab.d1[i];
  }
}

size_t pmf_factor_smem(int nd) { return sizeof(double) * (size_t)nd * nd; }

cudaError_t launch_pmf_factor(const KParams& kp, const Mat1D& t, int nd, int cell_first, int ncells,
                              int invert, double* out, cudaStream_t s) {
  if (ncells <= 0) return cudaSuccess;
  const size_t smem = pmf_factor_smem(nd);
  cudaError_t e = cudaFuncSetAttribute(k_pmf_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_pmf_factor<<<ncells, 256, smem, s>>>(kp, t, nd, cell_first, invert, out);
  return cudaGetLastError();
}

cudaError_t launch_pmf_sweep(int nd, int ncells, const double* Dinv, const double* u, const double* f,
                             const double* Au, double omega, double* out, cudaStream_t s) {
  const int blocks = 8 * sms();
  switch (nd) {
    case 8: k_pmf_sweep<8><<<blocks, 256, 0, s>>>(ncells, Dinv, u, f, Au, omega, out); break;
    case 27: k_pmf_sweep<27><<<blocks, 256, 0, s>>>(ncells, Dinv, u, f, Au, omega, out); break;
    case 64: k_pmf_sweep<64><<<blocks, 256, 0, s>>>(ncells, Dinv, u, f, Au, omega, out); break;
    case 125: k_pmf_sweep<125><<<blocks, 256, 0, s>>>(ncells, Dinv, u, f, Au, omega, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace dg
