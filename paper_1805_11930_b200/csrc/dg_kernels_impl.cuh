// fp64 sm_100a kernels of the matrix-free DG hot path (arXiv 1805.11930).
// Included once per degree by dg_kernels_n<N>.cu (one translation unit per n = p+1, so the
// degrees compile in parallel); each unit instantiates Deg<N> at the end of this file.
//
// One CTA owns a group of C consecutive cells (contiguous in the cell-major DoF
// vector, so tile loads/stores are fully coalesced). Each cell tensor lives in
// shared memory with a padded (bank-conflict-reduced) layout; every pass maps one
// thread to one 1D line of n values along x, y or z and applies an n x n 1D
// matrix held in __constant__ memory with compile-time indices (so the matrix
// entries are uniform constant-bank operands of DFMA, no shared-memory traffic).
//
//  Volume (§3.1), with collocation derivatives at the Gauss points:
//    Stage 1  U = (A_z A_y A_x) u                          passes P1-P3
//    Stage 2  F_k = W|T|(K_k/h_k^2 D_k U - b_k/h_k U), F_0 = W|T| c U
//    Stage 3  v = (A_x^T A_y^T A_z^T)(F_0 + sum_k D_k^T F_k)   passes P3-P7
//  Faces: per face node the value/normal-derivative traces
//    of the cell (and, for A, of the neighbour) are combined into a value-test
//    array S and a derivative-test array T, the tangential face mass
//    (h M^ x h M^, exact Gauss quadrature with m = n) is applied, and the result is
//    scattered with the 1D end-point profiles (e0/e1, d0/d1) in the last pass.
//  D_T = the same with only the cell's own face traces.
//  Local solves: Jacobi-preconditioned CG or BiCGStab per
//    cell, all C cells of a CTA iterating together with per-cell convergence masks
//    and deterministic per-cell reductions (no atomics).
#ifndef DG_NODAL_DT
#define DG_NODAL_DT 1   // local solvers: D_T in the nodal Kronecker-sum form
#endif
#ifndef DG_APPLY_SETUP_FIRST
#define DG_APPLY_SETUP_FIRST 0   // line apply: coefficient setup before the PDL wait (A/B)
#endif
#ifndef DG_NODAL_FLY
#define DG_NODAL_FLY 0   // local solvers: bit a = the nodal factor of direction a formed on the fly (else from shared memory)
#endif
#ifndef DG_NODAL_APPLY
#define DG_NODAL_APPLY 1   // line-family A u in the nodal Kronecker-sum form (apply_nodal)
#endif
#ifndef DG_PDL
#define DG_PDL 1
#endif
#include "dg_kernels.h"
#include "dg_degree.h"

#include <cstdio>
#include <cstdlib>

namespace dg {
namespace {

struct DevTab {
  double A[64], D[64], M[64], G[64];
  double w[8], d0[8], d1[8], Sd[8], Cd[8], Md[8];
  double E0[8], E1[8], F0[8], F1[8];  // A^-T e0, A^-T e1, A^-T d0, A^-T d1 (trace/derivative at 0/1 from Gauss values)
  // weight-folded variants for the unweighted quadrature residual of the plane kernels:
  double AW[64], GW[64];              // A[q][j] w_q, G[q][j] w_q
  double DW[64];                      // D[q][r] w_q / w_r
  double E0W[8], E1W[8], F0W[8], F1W[8];  // E0/w, E1/w, F0/w, F1/w
  // exact 1D stiffness and (test-derivative) convection matrices, for the bands of D_T
  double S[64], Cm[64];               // int th_i' th_j',  int th_i' th_j
  // Gauss-point line forms of the volume terms along one direction (collocation derivative D,
  // weights w): SG = D^T W D (stiffness), CG = D^T W (convection, test derivative)
  double SG[64], CG[64];
  double SGW[64];                     // SG[r][s] / w_r: the plane kernels' unweighted residual form
};
__constant__ DevTab c_tab[kMaxN + 1];
// mass-folded forms (k_apply_fold): Mhat^-1 Shat, Mhat^-1 Chat and Mhat^-1 applied to the face
// injection profiles e0, e1, d0, d1; one instance per translation unit (= per degree: the
// constant bank has no room for one per entry of c_tab)
struct FoldTab {
  double MiS[64], MiC[64];
  double mie0[8], mie1[8], mid0[8], mid1[8];
};
__constant__ FoldTab c_fold;

// Padded tensor layout per n: element (i,j,k) of cell slot cs at cs*CS + k*ZS + j*YS + i.
// Chosen offline to minimise shared-memory bank conflicts of x/y/z line passes.
template <int N> struct Lay;
template <> struct Lay<2> { static constexpr int YS = 2, ZS = 5, CS = 12; };
template <> struct Lay<3> { static constexpr int YS = 3, ZS = 9, CS = 27; };
template <> struct Lay<4> { static constexpr int YS = 4, ZS = 19, CS = 76; };
template <> struct Lay<5> { static constexpr int YS = 5, ZS = 25, CS = 125; };
template <> struct Lay<6> { static constexpr int YS = 9, ZS = 54, CS = 324; };
template <> struct Lay<7> { static constexpr int YS = 7, ZS = 52, CS = 369; };
template <> struct Lay<8> { static constexpr int YS = 9, ZS = 72, CS = 576; };

// cells per CTA
template <int N> struct Cells;
template <> struct Cells<2> { static constexpr int C = 32; };
template <> struct Cells<3> { static constexpr int C = 32; };
template <> struct Cells<4> { static constexpr int C = 16; };
template <> struct Cells<5> { static constexpr int C = 8; };
template <> struct Cells<6> { static constexpr int C = 4; };
template <> struct Cells<7> { static constexpr int C = 4; };
template <> struct Cells<8> { static constexpr int C = 2; };

// C_: cells per CTA (Cells<N>::C; the warp-per-cell solvers can run one cell per CTA)
template <int N_, int C_ = Cells<N_>::C> struct Geo {
  static constexpr int N = N_, N2 = N * N, N3 = N * N * N;
  static constexpr int C = C_;
  static constexpr int YS = Lay<N>::YS, ZS = Lay<N>::ZS, CS = Lay<N>::CS;
  static constexpr int LINES = C * N2;
  static constexpr int NT = ((LINES + 31) / 32) * 32;
  // one warp per cell: the thread count of k_cg_w / k_bicgstab_w, whose iterations then need no
  // CTA barrier (n = 5: 25 of 32 lanes hold a line; n >= 6: a lane holds up to two lines)
  static constexpr int NTW = C * 32;
  static constexpr int TENSOR = C * CS;
  static constexpr int FACE = C * 12 * N2;
};

// the solvers' face buffer fits in two tensors (it then aliases two the defect does not use)
template <int N, int CC = Cells<N>::C> __host__ __device__ constexpr bool fb_alias() {
  return 2 * Geo<N, CC>::TENSOR >= Geo<N, CC>::FACE;
}

// The leading members of Group (coefficients, face data, neighbour pointers, 1D rows): all the
// nodal apply uses, without the solvers' reduction and operator arrays (less static shared
// memory, one more resident CTA per SM at n = 5)
template <int N, int C_ = Cells<N>::C> struct GroupHead {
  static constexpr int C = C_;
  int cell[C];
  double vc[C][4];
  double vb[C][3];
  double fc[C][6][6];
  const double* nb[C][6];
  double tw[N], td0[N], td1[N];
};
template <int N, int C_ = Cells<N>::C> struct Group {
  static constexpr int C = C_;
  int cell[C];
  double vc[C][4];              // |T|K_x/h_x^2, |T|K_y/h_y^2, |T|K_z/h_z^2, |T|c
  double vb[C][3];              // |T| b_k / h_k (the cell's advection)
  double fc[C][6][6];           // per face: cs_a, cs_g, cn_a, cn_g, ct_a, ct_n
  const double* nb[C][6];       // neighbour cell base pointer (nullptr: none / not needed)
  double tw[N], td0[N], td1[N]; // runtime-indexed copies of w, d0, d1
  double red[2][C * N * N];     // per-line partial sums
  // self-face operators of D_T at the Gauss points, weighted residual form, per axis (x, y, z):
  // R_line += w_t1 w_t2 Bf U_line (the local solvers' D_T applications, no face passes)
  // rows padded to an even length (zero pad): the 16-byte aligned pairs are read with one
  // 128-bit broadcast load each (bterm)
  static constexpr int BR = (N + 1) & ~1;
  alignas(16) double Bf[C][3][N * BR];
  double sc[8][C];              // per-cell solver scalars
  int conv[C], its[C], rst[C];
};

enum { S_RR0 = 0, S_RZ, S_ALPHA, S_BETA, S_RHO, S_OMEGA, S_RHON, S_TMP };

// ---- table access with compile-time indices (constant-bank operands) ---------
template <int N, int W> __device__ __forceinline__ double tab(int idx) {
  if constexpr (W == 0) return c_tab[N].A[idx];
  else if constexpr (W == 1) return c_tab[N].D[idx];
  else return c_tab[N].M[idx];
}

// out[q] = sum_j M[q][j] in[j]
template <int N, int W> __device__ __forceinline__ void mv(const double* in, double* out) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(tab<N, W>(q * N + j), in[j], s);
    out[q] = s;
  }
}
// out[j] = sum_q M[q][j] in[q]
template <int N, int W> __device__ __forceinline__ void mtv(const double* in, double* out) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) s = fma(tab<N, W>(q * N + j), in[q], s);
    out[j] = s;
  }
}

template <int N, int S> __device__ __forceinline__ void ld(const double* p, double* v) {
#pragma unroll
  for (int e = 0; e < N; ++e) v[e] = p[e * S];
}
template <int N, int S> __device__ __forceinline__ void st(double* p, const double* v) {
#pragma unroll
  for (int e = 0; e < N; ++e) p[e * S] = v[e];
}
// global line access, 16-byte vectors where a line starts 16-byte aligned (n even)
template <int N> __device__ __forceinline__ void ldg_line(const double* p, double* v) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int e = 0; e < N; e += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + e);
      v[e] = t.x;
      v[e + 1] = t.y;
    }
  } else {
    ld<N, 1>(p, v);
  }
}
template <int N> __device__ __forceinline__ void stg_line(double* p, const double* v) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int e = 0; e < N; e += 2) *reinterpret_cast<double2*>(p + e) = make_double2(v[e], v[e + 1]);
  } else {
    st<N, 1>(p, v);
  }
}

// Stage 2 + the derivative half of stage 3 along one line of direction k:
// R += D^T ( Wl * w_q * (sK * (D U)_q - sb * U_q) )
// GEN = false (diffusion): the coefficient is constant along the line, so D^T W (sK D U) is the
// Gauss-point stiffness matvec sK (SG U), SG = D^T W D: one contraction instead of two
template <int N, bool GEN = true> __device__ __forceinline__ void dir_term(const double* U, double* R, double Wl,
                                                                           double sK, double sb) {
  if constexpr (!GEN) {
    const double f = Wl * sK;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) s = fma(c_tab[N].SG[r * N + q], U[q], s);
      R[r] = fma(f, s, R[r]);
    }
    return;
  }
  double du[N], F[N], t[N];
  mv<N, 1>(U, du);
#pragma unroll
  for (int q = 0; q < N; ++q) F[q] = Wl * c_tab[N].w[q] * fma(sK, du[q], -sb * U[q]);
  mtv<N, 1>(F, t);
#pragma unroll
  for (int r = 0; r < N; ++r) R[r] += t[r];
}

// R += Wl B U (B: a cell's D_T line operator along the line direction, from shared memory, rows
// of even stride BR, 16-byte aligned: read as pairs, one 128-bit broadcast load per pair)
template <int N> __device__ __forceinline__ void bterm(const double* B, const double* U, double* R, double Wl) {
  constexpr int BR = (N + 1) & ~1;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < N; r += 2) {
      const double2 b2 = *reinterpret_cast<const double2*>(B + q * BR + r);
      s = fma(b2.x, U[r], s);
      if (r + 1 < N) s = fma(b2.y, U[r + 1], s);
    }
    R[q] = fma(Wl, s, R[q]);
  }
}

// Degrees whose D_T applications fold the volume line terms into Bf (one matvec per direction
// from shared memory instead of the constant-table derivative pair; measured per degree,
// DESIGN.md §6): bit N of DG_FOLD_N.
#ifndef DG_FOLD_N
#define DG_FOLD_N 0x1fc   // every degree n = 2..8 (profiles/r02_fold_ab.txt)
#endif
template <int N> __host__ __device__ constexpr bool fold_volume() { return (DG_FOLD_N >> N) & 1; }

// Per cell and direction a, the D_T line operator at the Gauss points (weighted residual
// form, R_line += w_t1 w_t2 Bf U_line), so the local solvers' D_T applications need one matvec
// per direction instead of the derivative pair D^T W (.) D plus the face operator:
//   Bf[cs][a] = vc_a SG - vb_a CG + [a = z] diag(vc_3 w)                       (volume)
//             + |F_a| sum_{s = lo, hi} (E_s[q] (sa_s E_s[r] + sg_s F_s[r] / h_a) + F_s[q] ta_s E_s[r])
// (self faces: traces of a Gauss-value line u(s) = E_s.U, u'(s) = F_s.U, and the injection of
// the value- and derivative-test fluxes into the weighted Gauss residual).
// Needs g.fc, g.vc, g.vb; ends with a barrier.
template <int N, int NTH = Geo<N>::NT, int CC> __device__ void self_face_ops(const KParams& kp, Group<N, CC>& g) {
  using G = Geo<N, CC>;
  // one thread per row (cs, a, q), the row's entries unrolled (compile-time table columns: at
  // most n distinct constant-bank addresses per warp-wide load, see nodal_face_ops)
  for (int it = threadIdx.x; it < G::C * 3 * N; it += NTH) {
    const int cs = it / (3 * N), rem = it % (3 * N), a = rem / N, q = rem % N;
    const double* lo = g.fc[cs][2 * a];
    const double* hi = g.fc[cs][2 * a + 1];
    const double ih = kp.ih[a];   // 1 / h_a (host-computed, identical IEEE quotient)
    const double area = a == 0 ? kp.h[1] * kp.h[2] : (a == 1 ? kp.h[0] * kp.h[2] : kp.h[0] * kp.h[1]);
    const double e0q = c_tab[N].E0[q], f0q = c_tab[N].F0[q], e1q = c_tab[N].E1[q], f1q = c_tab[N].F1[q];
    const double vk = g.vc[cs][a], vb = g.vb[cs][a], vr = g.vc[cs][3], wq = c_tab[N].w[q];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double b = e0q * (lo[0] * c_tab[N].E0[r] + lo[1] * ih * c_tab[N].F0[r]) + f0q * lo[4] * c_tab[N].E0[r];
      b += e1q * (hi[0] * c_tab[N].E1[r] + hi[1] * ih * c_tab[N].F1[r]) + f1q * hi[4] * c_tab[N].E1[r];
      double t = area * b;
      if constexpr (fold_volume<N>()) {
        t = fma(vk, c_tab[N].SG[q * N + r], t);
        t = fma(-vb, c_tab[N].CG[q * N + r], t);
        if (a == 2 && q == r) t = fma(vr, wq, t);
      }
      g.Bf[cs][a][q * Group<N, CC>::BR + r] = t;
    }
    if (N & 1) g.Bf[cs][a][q * Group<N, CC>::BR + N] = 0.0;   // the pad
  }
  __syncthreads();
}

// Nodal D_T factors (warp-per-cell CG at n = 5): with per-cell constant coefficients on the
// affine cell, D_T = Kx (x) Mhat (x) Mhat + Mhat (x) Ky (x) Mhat + Mhat (x) Mhat (x) Kz (the
// Kronecker-sum form of the volume and self-face terms, P:343-357 restricted to T; tier B's
// diag_block), with the 1D matrices per cell and direction
//   K_a = |T|K_a/h_a^2 Shat - |T|b_a/h_a Chat + [a = z] |T| c Mhat
//       + |F_a| (e0 (s_a e0' + s_g/h d0') + t_a d0 e0' + e1 (.. hi ..))       (self faces)
// i.e. A^T Bf_a A of the Gauss-point line operators. Stored in g.Bf (rows of stride BR).
template <int N, int NTH = Geo<N>::NT, int CC> __device__ void nodal_face_ops(const KParams& kp, Group<N, CC>& g) {
  using G = Geo<N, CC>;
  // one thread per row (cs, a, i), the row's entries unrolled: the 1D tables are then read with
  // a compile-time column, i.e. at most n distinct constant-bank addresses per warp-wide load
  // (one thread per entry: up to 32, serialised by the constant cache; C3 D_T 490 -> 279 us)
  for (int it = threadIdx.x; it < G::C * 3 * N; it += NTH) {
    const int cs = it / (3 * N), rem = it % (3 * N), a = rem / N, i = rem % N;
    const double* lo = g.fc[cs][2 * a];
    const double* hi = g.fc[cs][2 * a + 1];
    const double ih = kp.ih[a];
    const double area = a == 0 ? kp.h[1] * kp.h[2] : (a == 1 ? kp.h[0] * kp.h[2] : kp.h[0] * kp.h[1]);
    const double e0i = i == 0, e1i = i == N - 1;
    const double d0i = c_tab[N].d0[i], d1i = c_tab[N].d1[i];
    const double vk = g.vc[cs][a], vb = g.vb[cs][a], vr = g.vc[cs][3];
#pragma unroll
    for (int ip = 0; ip < N; ++ip) {
      const double e0p = ip == 0, e1p = ip == N - 1;
      double f = e0i * (lo[0] * e0p + lo[1] * ih * c_tab[N].d0[ip]) + lo[4] * d0i * e0p;
      f += e1i * (hi[0] * e1p + hi[1] * ih * c_tab[N].d1[ip]) + hi[4] * d1i * e1p;
      double t = area * f;
      t = fma(vk, c_tab[N].S[i * N + ip], t);
      t = fma(-vb, c_tab[N].Cm[i * N + ip], t);
      if (a == 2) t = fma(vr, c_tab[N].M[i * N + ip], t);
      g.Bf[cs][a][i * Group<N, CC>::BR + ip] = t;
    }
    if (N & 1) g.Bf[cs][a][i * Group<N, CC>::BR + N] = 0.0;   // the pad
  }
  __syncthreads();
}

// v = K u along a line with K a per-cell nodal factor (rows of stride BR in shared memory, read
// as 128-bit broadcast pairs)
template <int N> __device__ __forceinline__ void kmv(const double* K, const double* u, double* v) {
  constexpr int BR = (N + 1) & ~1;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < N; r += 2) {
      const double2 b2 = *reinterpret_cast<const double2*>(K + q * BR + r);
      s = fma(b2.x, u[r], s);
      if (r + 1 < N) s = fma(b2.y, u[r + 1], s);
    }
    v[q] = s;
  }
}

// v = K_a u along a line with the nodal D_T factor of direction a (see nodal_face_ops) formed on
// the fly from the constant 1D tables (Shat, Chat, Mhat: constant-bank operands) and the cell's
// scalars: K_a = vc_a Shat - vb_a Chat + [a = z] vc_3 Mhat + |F_a| (self-face rank-2 terms)
template <int N, bool GEN, class CB>
__device__ __forceinline__ void kfly(const KParams& kp, const CB& g, int cs, int a, const double* u,
                                     double* v) {
  const double* lo = g.fc[cs][2 * a];
  const double* hi = g.fc[cs][2 * a + 1];
  const double vk = g.vc[cs][a];
  double g0 = 0.0, g1 = 0.0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
    g0 = fma(c_tab[N].d0[r], u[r], g0);
    g1 = fma(c_tab[N].d1[r], u[r], g1);
  }
  const double ih = kp.ih[a], fa = kp.fa[a];
  const double sl = fa * (lo[0] * u[0] + lo[1] * ih * g0), tl = fa * lo[4] * u[0];
  const double sh = fa * (hi[0] * u[N - 1] + hi[1] * ih * g1), th = fa * hi[4] * u[N - 1];
  double vb = 0.0, vr = 0.0;
  if constexpr (GEN) {
    vb = g.vb[cs][a];
    vr = a == 2 ? g.vc[cs][3] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double ss = 0.0, cc = 0.0, mm = 0.0;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      ss = fma(c_tab[N].S[q * N + r], u[r], ss);
      if constexpr (GEN) {
        cc = fma(c_tab[N].Cm[q * N + r], u[r], cc);
        mm = fma(c_tab[N].M[q * N + r], u[r], mm);
      }
    }
    double o = vk * ss;
    if constexpr (GEN) o = fma(-vb, cc, fma(vr, mm, o));
    o = fma(c_tab[N].d0[q], tl, fma(c_tab[N].d1[q], th, o));
    if (q == 0) o += sl;
    if (q == N - 1) o += sh;
    v[q] = o;
  }
}

// D_T p in the nodal Kronecker-sum form, one x-line per thread: WARP = the warp's own cell (lane
// l < n^2 owns x-line l), else the CTA's group (thread t < C n^2 owns x-line t):
// x-lines b = Mhat p, c = Kx p (registers) -> y-lines d = Mhat b, g = Ky b + Mhat c -> z-lines
// q = Mhat g + Kz d -> back to the thread's x-line. 7 one-direction contractions and 3 transposes
// (the Gauss-point form: 9 contractions, 6 transposes). pin: the thread's x-line of p.
template <int N, bool WARP, int FLY = 0, bool GEN = true, int CC>
__device__ __forceinline__ void dt_nodal(const Group<N, CC>& g, double* SA, double* SB, const double* pin,
                                         double* q, const KParams* kpp = nullptr) {
  using G = Geo<N, CC>;
  constexpr int N2 = G::N2;
  const int tid = threadIdx.x;
  const int cs = WARP ? tid >> 5 : tid / N2, l = WARP ? (tid & 31) : tid % N2;
  const bool act = WARP ? l < N2 : tid < G::LINES;
  const int a = l % N, b = l / N;
  const double* Kx = g.Bf[act ? cs : 0][0];
  const double* Ky = g.Bf[act ? cs : 0][1];
  const double* Kz = g.Bf[act ? cs : 0][2];
  const int base = cs * G::CS;
  auto sync = [] { if constexpr (WARP) __syncwarp(); else __syncthreads(); };
  if (act) {   // x-lines (j = a, k = b)
    double bv[N], cv[N];
    mv<N, 2>(pin, bv);
    if constexpr (FLY & 1) kfly<N, GEN>(*kpp, g, cs, 0, pin, cv); else kmv<N>(Kx, pin, cv);
    st<N, 1>(SA + base + b * G::ZS + a * G::YS, bv);
    st<N, 1>(SB + base + b * G::ZS + a * G::YS, cv);
  }
  sync();
  if (act) {   // y-lines (i = a, k = b)
    const int off = base + b * G::ZS + a;
    double bv[N], cv[N], dv[N], ev[N], fv[N];
    ld<N, G::YS>(SA + off, bv);
    ld<N, G::YS>(SB + off, cv);
    mv<N, 2>(bv, dv);
    if constexpr (FLY & 2) kfly<N, GEN>(*kpp, g, cs, 1, bv, ev); else kmv<N>(Ky, bv, ev);
    mv<N, 2>(cv, fv);
#pragma unroll
    for (int e = 0; e < N; ++e) ev[e] += fv[e];
    st<N, G::YS>(SA + off, dv);
    st<N, G::YS>(SB + off, ev);
  }
  sync();
  if (act) {   // z-lines (i = a, j = b)
    const int off = base + b * G::YS + a;
    double dv[N], gv[N], o1[N], o2[N];
    ld<N, G::ZS>(SA + off, dv);
    ld<N, G::ZS>(SB + off, gv);
    mv<N, 2>(gv, o1);
    if constexpr (FLY & 4) kfly<N, GEN>(*kpp, g, cs, 2, dv, o2); else kmv<N>(Kz, dv, o2);
#pragma unroll
    for (int e = 0; e < N; ++e) o1[e] += o2[e];
    st<N, G::ZS>(SA + off, o1);
  }
  sync();
  if (act) ld<N, 1>(SA + base + b * G::ZS + a * G::YS, q);
  else
#pragma unroll
    for (int e = 0; e < N; ++e) q[e] = 0.0;
}

// dst = D_T src in the nodal form for tensors in shared memory (CS layout), one x-line per thread
// (WARP: the warp's own cell); the callers synchronise around it
template <int N, bool WARP, int CC>
__device__ __forceinline__ void dt_nodal_smem(const Group<N, CC>& g, double* SA, double* SB, const double* src,
                                              double* dst) {
  using G = Geo<N, CC>;
  const int tid = threadIdx.x;
  const int cs = WARP ? tid >> 5 : tid / G::N2, l = WARP ? (tid & 31) : tid % G::N2;
  const bool act = WARP ? l < G::N2 : tid < G::LINES;
  const int off = cs * G::CS + (l / N) * G::ZS + (l % N) * G::YS;
  double pin[N], q[N];
  if (act) ld<N, 1>(src + off, pin);
  else
#pragma unroll
    for (int e = 0; e < N; ++e) pin[e] = 0.0;
  dt_nodal<N, WARP>(g, SA, SB, pin, q);
  if (act) st<N, 1>(dst + off, q);
}

// The y / z neighbours' lines through this thread's face nodes, loaded before the group setup:
// their addresses are integer arithmetic on the cell index (no coefficient), so their latency
// overlaps that of the setup's coefficient loads instead of following it. w[0], w[1]: y lo / hi
// (line (i = a, k = bb), stride n), w[2], w[3]: z lo / hi (line (i = a, j = bb), stride n^2); at a
// slab-boundary z face the ghost trace record's face value and derivative sum in w[.][0], w[.][1].
// Which faces have a neighbour is still read from the setup's pointers (the same decision).
template <int N> struct NbrLines { double w[4][N]; };
template <int N, int CC = Cells<N>::C>
__device__ __forceinline__ void nbr_lines_prefetch(const KParams& kp, const double* u, int cell0,
                                                   NbrLines<N>& W) {
  using G = Geo<N, CC>;
  constexpr int N2 = G::N2, N3 = G::N3;
  const int t = threadIdx.x;
  const int cs = t / N2, l = t % N2, a = l % N, bb = l / N;
  const int cell = cell0 + cs;
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int e = 0; e < N; ++e) W.w[f][e] = 0.0;
  if (u == nullptr || t >= G::LINES || cell >= kp.ncells) return;
  const int nxy = kp.nx * kp.ny;
  const int cy = (cell / kp.nx) % kp.ny, cz = cell / nxy;
  if (cy > 0) ld<N, N>(u + (size_t)(cell - kp.nx) * N3 + bb * N2 + a, W.w[0]);
  if (cy < kp.ny - 1) ld<N, N>(u + (size_t)(cell + kp.nx) * N3 + bb * N2 + a, W.w[1]);
  const int col = cell - cz * nxy, zo = bb * N + a;
  if (cz > 0) {
    ld<N, N2>(u + (size_t)(cell - nxy) * N3 + zo, W.w[2]);
  } else if (kp.slab_face[4] == FK_GHOST) {
    const double* rec = kp.ghost_lo + (size_t)col * 2 * N2;
    W.w[2][0] = rec[zo];
    W.w[2][1] = rec[N2 + zo];
  }
  if (cz < kp.nzl - 1) {
    ld<N, N2>(u + (size_t)(cell + nxy) * N3 + zo, W.w[3]);
  } else if (kp.slab_face[5] == FK_GHOST) {
    const double* rec = kp.ghost_hi + (size_t)col * 2 * N2;
    W.w[3][0] = rec[zo];
    W.w[3][1] = rec[N2 + zo];
  }
}

// A u (or the parts selected by kp.mask) for the CTA's group in the nodal Kronecker-sum form,
// one x-line per thread (C n^2 <= NTH):
//   (A u)_T = D_T u_T + sum over the interior faces F of (B_F (x) Mhat (x) Mhat) u_N
// D_T in the factored form of dt_nodal (K_a = g.Bf, nodal_face_ops: volume + self faces); the
// neighbour's face term depends on u_N only through its face values and normal-derivative sums
// (P:345-350), combined per face node into the value-test and derivative-test coefficients
// S, T (the fc neighbour coefficients, as face_line) and injected where the pipeline still
// applies the tangential masses: x faces into c = Kx u at the x stage (then Mhat_y, Mhat_z),
// y faces into g at the y stage after their Mhat_x (then Mhat_z), z faces at the z stage after
// Mhat_x and Mhat_y. Four barriers; no face passes. src: the group's tile (CS layout, shared),
// SA, SB: scratch tensors, FA: 12 C n^2 doubles (face arrays; the face buffer of cell_operator). out(cs, j, k, v[N]) receives x-line
// (j, k) of slot cs.
// INPLACE: src may be overwritten (A u alone): after the x stage has read a thread's own line, the
// z-face arrays after Mhat_x go there (4 < n entries per line) and FA shrinks to 8 C n^2
// W (optional): the y / z neighbour lines prefetched by nbr_lines_prefetch
// RS: row stride of the face arrays (N: the dense [n][n] layout; an even RS > N: 16-byte aligned
// rows read as 128-bit pairs, and the z-face arrays after Mhat_x stored transposed so that the y
// stage reads them as rows too)
template <int N> __device__ __forceinline__ void ld_row(const double* p, double* v) {
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    if (e + 1 < N) {
      const double2 t = *reinterpret_cast<const double2*>(p + e);
      v[e] = t.x;
      v[e + 1] = t.y;
    } else {
      v[e] = p[e];
    }
  }
}
// SHUF (WARP mode): the face arrays' tangential-mass contractions take the other face nodes' values
// from their lanes by warp shuffles instead of shared memory (the face arrays are not used)
template <int N, int NTH, bool GEN, bool INPLACE = false, bool WARP = false, int RS = N, bool SHUF = false, class Out, int CC>
__device__ __forceinline__ void apply_nodal(const KParams& kp, const Group<N, CC>& g, const double* src,
                                            double* SA, double* SB, double* FA, Out out,
                                            const NbrLines<N>* W = nullptr, const double* own = nullptr) {
  using G = Geo<N, CC>;
  constexpr int N2 = G::N2, C = G::C;
  static_assert(G::LINES <= NTH, "one x-line per thread");
  const int t = threadIdx.x;
  // WARP: warp w owns cell w (lanes < n^2 one x-line each; n <= 4: half-warps, two cells per
  // warp), the stages synchronise per warp
  constexpr int WL = N * N <= 16 ? 16 : 32;
  const bool act = WARP ? (t % WL) < N2 : t < G::LINES;
  const int cs = WARP ? t / WL : (act ? t / N2 : 0), l = WARP ? (t % WL) : t % N2, a = l % N, bb = l / N;
  auto sync = [] { if constexpr (WARP) __syncwarp(); else __syncthreads(); };
  constexpr bool ROWS = RS != N;
  static_assert(!ROWS || (RS % 2 == 0 && RS > N && !INPLACE), "padded rows: even, 16-byte aligned");
  constexpr int AS = N * RS;        // one face array
  double* FY = FA;                  // [C][4][n][RS]: y faces S_lo, T_lo, S_hi, T_hi at (i, k), row k
  double* FZ = FA + 4 * C * AS;     // [C][4][n][RS]: z faces at (i, j), row j; reused after Mhat_y
  double* FZb = FA + 8 * C * AS;    // [C][4][n][RS]: z faces after Mhat_x (not with INPLACE; ROWS: row i)
  static_assert(!INPLACE || N > 4, "INPLACE: the four face arrays fit in an x-line");
  // z-face entry (i, j) of array q after Mhat_x: in FZb, or (INPLACE) in the tile's x-line
  // (j' = i, k' = j), i.e. the line of the thread that produces the entry
  auto fzb = [&](int cs_, int q, int j, int i) -> double& {
    if constexpr (INPLACE) return const_cast<double*>(src)[cs_ * G::CS + j * G::ZS + i * G::YS + q];
    else if constexpr (ROWS) return FZb[cs_ * 4 * AS + q * AS + i * RS + j];
    else return FZb[cs_ * 4 * N2 + q * N2 + j * N + i];
  };
  const int base = cs * G::CS;
  // (the face sums are written as explicit fma: the ghost-record and in-slab branches then round
  // alike whatever the compiler contracts, so slab partitions stay bit for bit)
  double sxl = 0.0, txl = 0.0, sxh = 0.0, txh = 0.0;
  static_assert(!SHUF || WARP, "shuffles: one cell per (half-)warp");
  // SHUF: this lane's y- and z-face values (S_lo, T_lo, S_hi, T_hi), the lane of face node
  // (i, k) resp. (i, j) = (a, bb) being lb + bb n + a
  double yf[4] = {0.0, 0.0, 0.0, 0.0}, zf[4] = {0.0, 0.0, 0.0, 0.0};
  const int lb = (t & 31) & ~(WL - 1);
  // ---- stage 0: the neighbours' face data at this thread's face nodes
  if (act) {
    // x faces at (j = a, k = bb): the neighbours' x-lines (in the group: from the tile)
    {
      const double* nlo = g.nb[cs][0];
      const double* nhi = g.nb[cs][1];
      const double* clo = g.fc[cs][0];
      const double* chi = g.fc[cs][1];
      const int off = bb * G::ZS + a * G::YS, goff = bb * N2 + a * N;
      if (nlo) {
        double w[N];
        if (!WARP && cs > 0) ld<N, 1>(src + (cs - 1) * G::CS + off, w); else ldg_line<N>(nlo + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
        sxl = fma(clo[2], w[N - 1], (clo[3] * gn) * kp.ih[0]);
        txl = clo[5] * w[N - 1];
      }
      if (nhi) {
        double w[N];
        if (!WARP && cs < C - 1) ld<N, 1>(src + (cs + 1) * G::CS + off, w); else ldg_line<N>(nhi + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
        sxh = fma(chi[2], w[0], (chi[3] * gn) * kp.ih[0]);
        txh = chi[5] * w[0];
      }
    }
    // y faces at (i = a, k = bb)
    {
      const double* nlo = g.nb[cs][2];
      const double* nhi = g.nb[cs][3];
      const double* clo = g.fc[cs][2];
      const double* chi = g.fc[cs][3];
      const int goff = bb * N2 + a;
      double s0 = 0.0, t0 = 0.0, s1 = 0.0, t1 = 0.0;
      if (nlo) {
        double w[N];
        if (W) {
#pragma unroll
          for (int e = 0; e < N; ++e) w[e] = W->w[0][e];
        } else {
          ld<N, N>(nlo + goff, w);
        }
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
        s0 = fma(clo[2], w[N - 1], (clo[3] * gn) * kp.ih[1]);
        t0 = clo[5] * w[N - 1];
      }
      if (nhi) {
        double w[N];
        if (W) {
#pragma unroll
          for (int e = 0; e < N; ++e) w[e] = W->w[1][e];
        } else {
          ld<N, N>(nhi + goff, w);
        }
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
        s1 = fma(chi[2], w[0], (chi[3] * gn) * kp.ih[1]);
        t1 = chi[5] * w[0];
      }
      if constexpr (SHUF) {
        yf[0] = s0; yf[1] = t0; yf[2] = s1; yf[3] = t1;
      } else {
        double* fy = FY + cs * 4 * AS + bb * RS + a;
        fy[0] = s0; fy[AS] = t0; fy[2 * AS] = s1; fy[3 * AS] = t1;
      }
    }
    // z faces at (i = a, j = bb); at a slab boundary the neighbour is a ghost trace record
    {
      const double* nlo = g.nb[cs][4];
      const double* nhi = g.nb[cs][5];
      const double* clo = g.fc[cs][4];
      const double* chi = g.fc[cs][5];
      const int goff = bb * N + a;
      double s0 = 0.0, t0 = 0.0, s1 = 0.0, t1 = 0.0;
      if (nlo) {
        double av, gn = 0.0;
        if (ghost_trace(kp, g.cell[cs], 0)) {
          av = W ? W->w[2][0] : nlo[goff];
          gn = W ? W->w[2][1] : nlo[N2 + goff];
        } else {
          double w[N];
          if (W) {
#pragma unroll
            for (int e = 0; e < N; ++e) w[e] = W->w[2][e];
          } else {
            ld<N, N2>(nlo + goff, w);
          }
#pragma unroll
          for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
          av = w[N - 1];
        }
        s0 = fma(clo[2], av, (clo[3] * gn) * kp.ih[2]);
        t0 = clo[5] * av;
      }
      if (nhi) {
        double av, gn = 0.0;
        if (ghost_trace(kp, g.cell[cs], 1)) {
          av = W ? W->w[3][0] : nhi[goff];
          gn = W ? W->w[3][1] : nhi[N2 + goff];
        } else {
          double w[N];
          if (W) {
#pragma unroll
            for (int e = 0; e < N; ++e) w[e] = W->w[3][e];
          } else {
            ld<N, N2>(nhi + goff, w);
          }
#pragma unroll
          for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
          av = w[0];
        }
        s1 = fma(chi[2], av, (chi[3] * gn) * kp.ih[2]);
        t1 = chi[5] * av;
      }
      if constexpr (SHUF) {
        zf[0] = s0; zf[1] = t0; zf[2] = s1; zf[3] = t1;
      } else {
        double* fz = FZ + cs * 4 * AS + bb * RS + a;
        fz[0] = s0; fz[AS] = t0; fz[2 * AS] = s1; fz[3 * AS] = t1;
      }
    }
  }
  sync();
  // SHUF: the z-face arrays after Mhat_x at (i = a, j = bb), all lanes taking part
  double zx[4] = {0.0, 0.0, 0.0, 0.0};
  if constexpr (SHUF) {
    const int ia = act ? a : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double zs = 0.0;
#pragma unroll
      for (int ip = 0; ip < N; ++ip) {
        const double v = __shfl_sync(0xffffffffu, zf[q], lb + bb * N + ip);
        zs = fma(c_tab[N].M[ia * N + ip], v, zs);
      }
      zx[q] = zs;
    }
  }
  // ---- x stage (x-line j = a, k = bb): b = Mhat u, c = Kx u + x faces; z faces: Mhat_x
  if (act) {
    double u[N], bv[N], cv[N];
    if (own) {   // the thread's own x-line, loaded by the caller into registers
#pragma unroll
      for (int e = 0; e < N; ++e) u[e] = own[e];
    } else {
      ld<N, 1>(src + base + bb * G::ZS + a * G::YS, u);
    }
    mv<N, 2>(u, bv);
    kfly<N, GEN>(kp, g, cs, 0, u, cv);
    const double fa = kp.fa[0];
#pragma unroll
    for (int e = 0; e < N; ++e)
      cv[e] = fma(fa, fma(c_tab[N].d0[e], txl, fma(c_tab[N].d1[e], txh, (e == 0 ? sxl : 0.0) + (e == N - 1 ? sxh : 0.0))), cv[e]);
    st<N, 1>(SA + base + bb * G::ZS + a * G::YS, bv);
    st<N, 1>(SB + base + bb * G::ZS + a * G::YS, cv);
#pragma unroll
    for (int q = 0; q < 4 && !SHUF; ++q) {   // z-face arrays along x: entry (i = a, j = bb)
      const double* row = FZ + cs * 4 * AS + q * AS + bb * RS;
      double rv[N];
      if constexpr (ROWS) ld_row<N>(row, rv); else ld<N, 1>(row, rv);
      double zs = 0.0;
#pragma unroll
      for (int ip = 0; ip < N; ++ip) zs = fma(c_tab[N].M[a * N + ip], rv[ip], zs);
      fzb(cs, q, bb, a) = zs;
    }
  }
  sync();
  // SHUF: the y-face arrays after Mhat_x at (i = a, k = bb) and the z-face arrays after Mhat_x,
  // Mhat_y at (i = a, j = bb)
  double yqs[4] = {0.0, 0.0, 0.0, 0.0}, zy[4] = {0.0, 0.0, 0.0, 0.0};
  if constexpr (SHUF) {
    const int ia = act ? a : 0, ib = act ? bb : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double s = 0.0, z = 0.0;
#pragma unroll
      for (int ip = 0; ip < N; ++ip) {
        const double v = __shfl_sync(0xffffffffu, yf[q], lb + bb * N + ip);
        s = fma(c_tab[N].M[ia * N + ip], v, s);
      }
#pragma unroll
      for (int jp = 0; jp < N; ++jp) {
        const double v = __shfl_sync(0xffffffffu, zx[q], lb + jp * N + a);
        z = fma(c_tab[N].M[ib * N + jp], v, z);
      }
      yqs[q] = s;
      zy[q] = z;
    }
  }
  // ---- y stage (y-line i = a, k = bb): d = Mhat b, g = Ky b + Mhat c + y faces (after Mhat_x);
  // z faces: Mhat_y
  if (act) {
    const int off = base + bb * G::ZS + a;
    double bv[N], cv[N], dv[N], ev[N], fv[N];
    ld<N, G::YS>(SA + off, bv);
    ld<N, G::YS>(SB + off, cv);
    mv<N, 2>(bv, dv);
    kfly<N, GEN>(kp, g, cs, 1, bv, ev);
    mv<N, 2>(cv, fv);
    double yq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if constexpr (SHUF) {
        yq[q] = yqs[q];
        continue;
      }
      const double* row = FY + cs * 4 * AS + q * AS + bb * RS;
      double rv[N];
      if constexpr (ROWS) ld_row<N>(row, rv); else ld<N, 1>(row, rv);
      double s = 0.0;
#pragma unroll
      for (int ip = 0; ip < N; ++ip) s = fma(c_tab[N].M[a * N + ip], rv[ip], s);
      yq[q] = s;
    }
    const double fa = kp.fa[1];
#pragma unroll
    for (int e = 0; e < N; ++e)
      ev[e] += fv[e] + fa * (c_tab[N].d0[e] * yq[1] + c_tab[N].d1[e] * yq[3] + (e == 0 ? yq[0] : 0.0) +
                             (e == N - 1 ? yq[2] : 0.0));
    // z-face arrays along y (entry (i = a, j = bb)) -> FZ (free again)
#pragma unroll
    for (int q = 0; q < 4 && !SHUF; ++q) {
      double rv[N];
      if constexpr (ROWS) {
        ld_row<N>(FZb + cs * 4 * AS + q * AS + a * RS, rv);
      } else {
#pragma unroll
        for (int jp = 0; jp < N; ++jp) rv[jp] = fzb(cs, q, jp, a);
      }
      double s = 0.0;
#pragma unroll
      for (int jp = 0; jp < N; ++jp) s = fma(c_tab[N].M[bb * N + jp], rv[jp], s);
      FZ[cs * 4 * AS + q * AS + bb * RS + a] = s;
    }
    st<N, G::YS>(SA + off, dv);
    st<N, G::YS>(SB + off, ev);
  }
  sync();
  // ---- z stage (z-line i = a, j = bb): q = Mhat g + Kz d + z faces (after Mhat_x, Mhat_y)
  if (act) {
    const int off = base + bb * G::YS + a;
    double dv[N], gv[N], o1[N], o2[N];
    ld<N, G::ZS>(SA + off, dv);
    ld<N, G::ZS>(SB + off, gv);
    mv<N, 2>(gv, o1);
    kfly<N, GEN>(kp, g, cs, 2, dv, o2);
    const double* fz = FZ + cs * 4 * AS + bb * RS + a;
    const double z0 = SHUF ? zy[0] : fz[0], z1 = SHUF ? zy[1] : fz[AS], z2 = SHUF ? zy[2] : fz[2 * AS],
                 z3 = SHUF ? zy[3] : fz[3 * AS];
    const double fa = kp.fa[2];
#pragma unroll
    for (int e = 0; e < N; ++e)
      o1[e] += o2[e] + fa * (c_tab[N].d0[e] * z1 + c_tab[N].d1[e] * z3 + (e == 0 ? z0 : 0.0) +
                             (e == N - 1 ? z2 : 0.0));
    st<N, G::ZS>(SA + off, o1);
  }
  sync();
  if (act) {
    double v[N];
    ld<N, 1>(SA + base + bb * G::ZS + a * G::YS, v);
    out(cs, a, bb, v);
  }
}

// ---- group setup: coefficients, face parameters, neighbour pointers ------------
// Per cell of the group: volume scalings vc, face coefficients fc, neighbour pointers nb
// (nullptr when u == nullptr, i.e. for D_T-only operators). Ends with __syncthreads.
template <int N, int C, int NT>
__device__ void setup_cells(const KParams& kp, double (*vc_)[4], double (*vb_)[3], double (*fc_)[6][6],
                            const double* (*nb_)[6], int* cellv, int cell0, const double* u) {
  constexpr int N3 = N * N * N;
  const int t = threadIdx.x;
  const int nxy = kp.nx * kp.ny;
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
  const int c0x = cell0 % kp.nx, c0y = (cell0 / kp.nx) % kp.ny, c0z = cell0 / nxy;
  for (int it = t; it < C * 6; it += NT) {
    const int cs = it / 6, f = it % 6, axis = f >> 1, hi = f & 1;
    const int cell = cell0 + cs;
    const bool valid = cell < kp.ncells;
    double co[6] = {0, 0, 0, 0, 0, 0};
    const double* nbp = nullptr;
    if (f == 0) {
      if (cellv) cellv[cs] = valid ? cell : -1;
      double* vc = vc_[cs];
      if (valid && (kp.mask & 1u)) {
        const double* Kc = kp.K + (size_t)(cell + nxy) * 3;
        vc[0] = Kc[0] * vol * kp.ih[0] * kp.ih[0];
        vc[1] = Kc[1] * vol * kp.ih[1] * kp.ih[1];
        vc[2] = Kc[2] * vol * kp.ih[2] * kp.ih[2];
        vc[3] = kp.c ? vol * kp.c[cell] : 0.0;
        // (no pointer to the kernel parameter kp.b: that would copy KParams to local memory)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          vb_[cs][a] = vol * (kp.bc ? kp.bc[(size_t)(cell + nxy) * 3 + a] : kp.b[a]) * kp.ih[a];
      } else {
        vc[0] = vc[1] = vc[2] = vc[3] = 0.0;
        vb_[cs][0] = vb_[cs][1] = vb_[cs][2] = 0.0;
      }
    }
    if (valid) {
      // coordinates of cell0 + cs without per-item integer division (cs < C is small)
      int cx = c0x + cs, cy = c0y, cz = c0z;
      while (cx >= kp.nx) { cx -= kp.nx; ++cy; }
      while (cy >= kp.ny) { cy -= kp.ny; ++cz; }
      // (selects, not arrays indexed by the runtime axis: those went to local memory)
      const int crd = axis == 0 ? cx : (axis == 1 ? cy : cz);
      const int dim = axis == 0 ? kp.nx : (axis == 1 ? kp.ny : kp.nzl);
      const int dst = axis == 0 ? 1 : (axis == 1 ? kp.nx : nxy);
      const double ihk = kp.ih[axis];
      const double KT = kp.K[(size_t)(cell + nxy) * 3 + axis];
      const int ncoord = crd + (hi ? 1 : -1);
      int kind;  // 0 interior, 1 Dirichlet, 2 Neumann
      long kidx = 0;
      if (ncoord >= 0 && ncoord < dim) {
        kind = 0;
        const long nb = cell + (hi ? dst : -dst);
        kidx = nb + nxy;
        if (u) nbp = u + (size_t)nb * N3;
      } else {
        const int sk = kp.slab_face[f];
        if (sk == FK_GHOST) {
          kind = 0;
          const int col = cx + kp.nx * cy;
          kidx = hi ? (long)(kp.nzl + 1) * nxy + col : col;
          if (u) nbp = (hi ? kp.ghost_hi : kp.ghost_lo) + (size_t)col * 2 * N * N;   // trace record
        } else {
          kind = (sk == FK_DIRICHLET) ? 1 : 2;
        }
      }
      // b . nu_F on the face (reading #8: the mean of the two cells' b; exact for constant b)
      const double bT = kp.bc ? kp.bc[(size_t)(cell + nxy) * 3 + axis] : kp.b[axis];
      const double bn = kind == 0 ? 0.5 * (bT + (kp.bc ? kp.bc[(size_t)kidx * 3 + axis] : bT)) : bT;
      if (kind == 0 && (kp.mask & 2u)) {
        const double KN = kp.K[(size_t)kidx * 3 + axis];
        const double s = KT + KN;
        const double rs = s > 0.0 ? 1.0 / s : 0.0;   // the only division of the face setup
        const double wT = s > 0.0 ? KN * rs : 0.5, wN = s > 0.0 ? KT * rs : 0.5;
        const double gam = kp.pen * (2.0 * KT * KN * rs) * ihk;  // <dT,dN>|F|/|T|
        if (hi) {
          co[0] = fmax(bn, 0.0) + gam;  co[1] = -wT * KT;
          co[2] = fmin(bn, 0.0) - gam;  co[3] = -wN * KN;
          co[4] = -wT * KT * ihk;       co[5] = wT * KT * ihk;
        } else {
          co[0] = fmax(-bn, 0.0) + gam; co[1] = wT * KT;
          co[2] = fmin(-bn, 0.0) - gam; co[3] = wN * KN;
          co[4] = wT * KT * ihk;        co[5] = -wT * KT * ihk;
        }
      } else if (kind == 1 && (kp.mask & 4u)) {
        const double gam = kp.pen * KT * ihk;  // delta |F| / |T|
        if (hi) { co[0] = fmax(bn, 0.0) + gam;  co[1] = -KT; co[4] = -KT * ihk; }
        else    { co[0] = fmax(-bn, 0.0) + gam; co[1] = KT;  co[4] = KT * ihk; }
      }
      if (kind != 0) nbp = nullptr;
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) fc_[cs][f][e] = co[e];
    nb_[cs][f] = nbp;
  }
  __syncthreads();
}

template <int N, int NTH = Geo<N>::NT, int CC>
__device__ void group_setup(const KParams& kp, Group<N, CC>& g, int cell0, const double* u) {
  using G = Geo<N, CC>;
  const int t = threadIdx.x;
  if (t < N) {
    g.tw[t] = c_tab[N].w[t];
    g.td0[t] = c_tab[N].d0[t];
    g.td1[t] = c_tab[N].d1[t];
  }
  setup_cells<N, G::C, NTH>(kp, g.vc, g.vb, g.fc, g.nb, g.cell, cell0, u);
}

// ---- tiles ---------------------------------------------------------------------
template <int N, int NTH = Geo<N>::NT, int CC>
__device__ __forceinline__ void load_tile(const Group<N, CC>& g, int cell0, int ncells,
                                          const double* __restrict__ src, double* dst) {
  using G = Geo<N, CC>;
  const int nvalid = min(G::C, ncells - cell0);
  const double* s = src + (size_t)cell0 * G::N3;
  for (int e = threadIdx.x; e < G::C * G::N3; e += NTH) {
    const int cs = e / G::N3, r = e % G::N3;
    const int i = r % N, j = (r / N) % N, k = r / G::N2;
    dst[cs * G::CS + k * G::ZS + j * G::YS + i] = (cs < nvalid) ? s[e] : 0.0;
  }
}

// ---- faces, part 1: traces -> S/T arrays per face node (+ tangential mass) ------
// face buffer: FB[((cs*3 + axis)*4 + arr)*N2 + l], arr: 0 S_lo, 1 T_lo, 2 S_hi, 3 T_hi
// The neighbours' lines wlo / whi (the normal line through the face node, from the neighbour
// below / above; loaded by the caller ahead of time, see cell_operator) enter through their end
// value and end derivative. hlo / hhi: the neighbour exists (interior or ghost-layer face).
// tlo / thi: the neighbour is a ghost-layer trace record: w[0] is its face value and w[1] its
// normal-derivative sum (the sender's arithmetic, bit for bit the value computed here otherwise).
template <int N, int AX, int CC>
__device__ __forceinline__ void face_line(const Group<N, CC>& g, const double* src, double* FB,
                                          int cs, int a, int b, double inv_h, const double* wlo,
                                          const double* whi, bool hlo, bool hhi, bool tlo = false,
                                          bool thi = false) {
  using G = Geo<N, CC>;
  int off;
  constexpr int SS = AX == 0 ? 1 : (AX == 1 ? G::YS : G::ZS);   // smem stride along the line
  if (AX == 0) off = b * G::ZS + a * G::YS;
  else if (AX == 1) off = b * G::ZS + a;
  else off = b * G::YS + a;
  double v[N];
  ld<N, SS>(src + cs * G::CS + off, v);
  double glo = 0.0, ghi = 0.0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    glo = fma(c_tab[N].d0[e], v[e], glo);
    ghi = fma(c_tab[N].d1[e], v[e], ghi);
  }
  glo *= inv_h;
  ghi *= inv_h;
  const double* clo = g.fc[cs][2 * AX];
  const double* chi = g.fc[cs][2 * AX + 1];
  double Slo = clo[0] * v[0] + clo[1] * glo, Tlo = clo[4] * v[0];
  double Shi = chi[0] * v[N - 1] + chi[1] * ghi, Thi = chi[4] * v[N - 1];
  if (hlo) {  // neighbour below: its hi trace (node N-1) and d1 derivative
    double gn = 0.0, av;
    if (tlo) {
      av = wlo[0];
      gn = wlo[1];
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], wlo[e], gn);
      av = wlo[N - 1];
    }
    Slo += clo[2] * av + clo[3] * gn * inv_h;
    Tlo += clo[5] * av;
  }
  if (hhi) {  // neighbour above: its lo trace (node 0) and d0 derivative
    double gn = 0.0, av;
    if (thi) {
      av = whi[0];
      gn = whi[1];
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], whi[e], gn);
      av = whi[0];
    }
    Shi += chi[2] * av + chi[3] * gn * inv_h;
    Thi += chi[5] * av;
  }
  double* fb = FB + (cs * 3 + AX) * 4 * G::N2 + a + N * b;
  fb[0 * G::N2] = Slo;
  fb[1 * G::N2] = Tlo;
  fb[2 * G::N2] = Shi;
  fb[3 * G::N2] = Thi;
}

// ---- the full cell operator: faces + volume, result handed to `out` line by line ----
// src: input tensors (smem), SA/SB scratch tensors, FB face buffer.
// out(cs, j, k, v[N]) receives x-line (j,k) of cell slot cs.
// FACES = false: the volume terms alone (the face passes are skipped); USEB (with FACES = false):
// plus the self-face terms through g.Bf inside the Gauss-point passes (D_T without face passes)
// GEN = false: pure diffusion (b = 0, no reaction) with the convective and reaction terms compiled out
template <int N, bool FACES = true, bool USEB = false, bool WARP = false, int NTH = Geo<N>::NT,
          bool GEN = true, class Out, int CC>
__device__ __forceinline__ void cell_operator(const KParams& kp, const Group<N, CC>& g,
                                              const double* src, double* SA, double* SB,
                                              double* FB, bool vol, Out out,
                                              const double* pin = nullptr) {
  // pin (warp mode, one line per lane): the lane's own x-line of the input, from registers
  // instead of src
  using G = Geo<N, CC>;
  constexpr int C = G::C, N2 = G::N2, LINES = G::LINES, NT = NTH;   // NTH: the launch's thread count
  const int tid = threadIdx.x;
  static_assert(!WARP || !FACES, "warp mode: one cell per warp, no face passes");
  // WARP: the calling warp applies the operator to its own cell (cs = warp) alone, one line per
  // lane, __syncwarp between the passes; otherwise the whole CTA over all lines of the group
  const int lb = WARP ? (tid >> 5) * N2 + (tid & 31) : tid;
  const int le = WARP ? ((tid >> 5) + 1) * N2 : LINES;
  constexpr int ls = WARP ? 32 : NT;
  const double area[3] = {kp.h[1] * kp.h[2], kp.h[0] * kp.h[2], kp.h[0] * kp.h[1]};
  // advection scalings |T| b_k / h_k: in warp mode the warp's own cell's, read once (registers,
  // like the constant-b values they replace); otherwise per line item from shared memory
  double sbw[3] = {0.0, 0.0, 0.0};
  if constexpr (WARP && GEN)
#pragma unroll
    for (int a = 0; a < 3; ++a) sbw[a] = g.vb[tid >> 5][a];
  auto sbk = [&](int cs, int a) { return WARP ? sbw[a] : g.vb[cs][a]; };

  // pass 1: F1 (face traces, all axes) + P1 (x-lines: SA = A_x src); the neighbours' normal
  // lines: x neighbours inside the group from the tile in shared memory, the others from global
  // memory (prefetching them into registers cost more in occupancy than it saved in latency)
  for (int it = tid; FACES && it < 3 * LINES; it += NT) {
    const int ax = it / LINES, r = it % LINES, cs = r / N2, l = r % N2;
    const int a = l % N, b = l / N;
    const double* nlo = g.nb[cs][2 * ax];
    const double* nhi = g.nb[cs][2 * ax + 1];
    double wl[N], wh[N];
    if (ax == 0) {
      const int off = b * G::ZS + a * G::YS, goff = b * N2 + a * N;
      if (nlo) { if (cs > 0) ld<N, 1>(src + (cs - 1) * G::CS + off, wl); else ld<N, 1>(nlo + goff, wl); }
      if (nhi) { if (cs < C - 1) ld<N, 1>(src + (cs + 1) * G::CS + off, wh); else ld<N, 1>(nhi + goff, wh); }
      face_line<N, 0>(g, src, FB, cs, a, b, kp.ih[0], wl, wh, nlo != nullptr, nhi != nullptr);
    } else if (ax == 1) {
      const int goff = b * N2 + a;
      if (nlo) ld<N, N>(nlo + goff, wl);
      if (nhi) ld<N, N>(nhi + goff, wh);
      face_line<N, 1>(g, src, FB, cs, a, b, kp.ih[1], wl, wh, nlo != nullptr, nhi != nullptr);
    } else {
      // slab-boundary faces: the neighbour is a ghost trace record (face values, derivative sums)
      const int goff = b * N + a;
      const bool tl = nlo && ghost_trace(kp, g.cell[cs], 0), th = nhi && ghost_trace(kp, g.cell[cs], 1);
      if (tl) { wl[0] = nlo[goff]; wl[1] = nlo[N2 + goff]; }
      else if (nlo) ld<N, N2>(nlo + goff, wl);
      if (th) { wh[0] = nhi[goff]; wh[1] = nhi[N2 + goff]; }
      else if (nhi) ld<N, N2>(nhi + goff, wh);
      face_line<N, 2>(g, src, FB, cs, a, b, kp.ih[2], wl, wh, nlo != nullptr, nhi != nullptr, tl, th);
    }
  }
  if (vol) {
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;
      const int off = cs * G::CS + b * G::ZS + a * G::YS;
      double v[N], o[N];
      if ((WARP || LINES <= NT) && pin) {   // one line per thread: its own line, from registers
#pragma unroll
        for (int e = 0; e < N; ++e) v[e] = pin[e];
      } else {
        ld<N, 1>(src + off, v);
      }
      mv<N, 0>(v, o);
      st<N, 1>(SA + off, o);
    }
  }
  if constexpr (WARP) __syncwarp(); else __syncthreads();
  // pass 2: F2 (tangential mass along t1) + P2 (y-lines: SB = A_y SA)
  for (int it = tid; FACES && it < C * 12 * N; it += NT) {
    const int t2 = it % N, rest = it / N;
    double* fa = FB + rest * N2 + N * t2;
    double v[N], o[N];
    ld<N, 1>(fa, v);
    mv<N, 2>(v, o);
    st<N, 1>(fa, o);
  }
  if (vol) {
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;
      const int off = cs * G::CS + b * G::ZS + a;
      double v[N], o[N];
      ld<N, G::YS>(SA + off, v);
      mv<N, 0>(v, o);
      st<N, G::YS>(SB + off, o);
    }
  }
  if constexpr (WARP) __syncwarp(); else __syncthreads();
  // pass 3: F3 (tangential mass along t2, area scaling) + P3 (z-lines: U = A_z SB -> SA,
  //         R = reaction + z-term -> SB)
  for (int it = tid; FACES && it < C * 12 * N; it += NT) {
    const int t1 = it % N, rest = it / N;
    const int ax = (rest >> 2) % 3;
    double* fa = FB + rest * N2 + t1;
    double v[N], o[N];
    ld<N, N>(fa, v);
    mv<N, 2>(v, o);
#pragma unroll
    for (int e = 0; e < N; ++e) o[e] *= area[ax];
    st<N, N>(fa, o);
  }
  if (vol) {
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;  // a = qx, b = qy
      const int off = cs * G::CS + b * G::YS + a;
      double t[N], U[N], R[N];
      ld<N, G::ZS>(SB + off, t);
      mv<N, 0>(t, U);
      const double Wl = g.tw[a] * g.tw[b];
      constexpr bool FOLD = USEB && fold_volume<N>();
      if constexpr (FOLD) {   // the whole z-line operator of D_T (volume + self faces) at once
#pragma unroll
        for (int q = 0; q < N; ++q) R[q] = 0.0;
        bterm<N>(g.Bf[cs][2], U, R, Wl);
      } else {
        const double sc = g.vc[cs][3];
#pragma unroll
        for (int q = 0; q < N; ++q) R[q] = GEN ? Wl * c_tab[N].w[q] * sc * U[q] : 0.0;
        dir_term<N, GEN>(U, R, Wl, g.vc[cs][2], GEN ? sbk(cs, 2) : 0.0);
        if constexpr (USEB) bterm<N>(g.Bf[cs][2], U, R, Wl);
      }
      st<N, G::ZS>(SA + off, U);
      st<N, G::ZS>(SB + off, R);
    }
    if constexpr (WARP) __syncwarp(); else __syncthreads();
    // pass 4: x-lines, R += x-term
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;  // a = qy, b = qz
      const int off = cs * G::CS + b * G::ZS + a * G::YS;
      double U[N], R[N];
      ld<N, 1>(SA + off, U);
      ld<N, 1>(SB + off, R);
      if constexpr (!(USEB && fold_volume<N>()))
        dir_term<N, GEN>(U, R, g.tw[a] * g.tw[b], g.vc[cs][0], GEN ? sbk(cs, 0) : 0.0);
      if constexpr (USEB) bterm<N>(g.Bf[cs][0], U, R, g.tw[a] * g.tw[b]);
      st<N, 1>(SB + off, R);
    }
    if constexpr (WARP) __syncwarp(); else __syncthreads();
    // pass 5: y-lines, R += y-term, then A_y^T
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;  // a = qx, b = qz
      const int off = cs * G::CS + b * G::ZS + a;
      double U[N], R[N], o[N];
      ld<N, G::YS>(SA + off, U);
      ld<N, G::YS>(SB + off, R);
      if constexpr (!(USEB && fold_volume<N>()))
        dir_term<N, GEN>(U, R, g.tw[a] * g.tw[b], g.vc[cs][1], GEN ? sbk(cs, 1) : 0.0);
      if constexpr (USEB) bterm<N>(g.Bf[cs][1], U, R, g.tw[a] * g.tw[b]);
      mtv<N, 0>(R, o);
      st<N, G::YS>(SB + off, o);
    }
    if constexpr (WARP) __syncwarp(); else __syncthreads();
    // pass 6: z-lines, A_z^T
    for (int it = lb; it < le; it += ls) {
      const int cs = it / N2, l = it % N2, a = l % N, b = l / N;
      const int off = cs * G::CS + b * G::YS + a;
      double v[N], o[N];
      ld<N, G::ZS>(SB + off, v);
      mtv<N, 0>(v, o);
      st<N, G::ZS>(SB + off, o);
    }
  }
  if constexpr (WARP) __syncwarp(); else __syncthreads();
  // pass 7: x-lines, A_x^T + scatter of all face terms
  for (int it = lb; it < le; it += ls) {
    const int cs = it / N2, l = it % N2, j = l % N, k = l / N;
    double v[N];
    if (vol) {
      double t[N];
      ld<N, 1>(SB + cs * G::CS + k * G::ZS + j * G::YS, t);
      mtv<N, 0>(t, v);
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) v[e] = 0.0;
    }
    if constexpr (FACES) {
    const double* fx = FB + (cs * 3 + 0) * 4 * N2;
    const double* fy = FB + (cs * 3 + 1) * 4 * N2;
    const double* fz = FB + (cs * 3 + 2) * 4 * N2;
    // x faces: index (j,k)
    {
      const double Slo = fx[0 * N2 + l], Tlo = fx[1 * N2 + l], Shi = fx[2 * N2 + l], Thi = fx[3 * N2 + l];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = fma(c_tab[N].d0[i], Tlo, fma(c_tab[N].d1[i], Thi, v[i]));
      v[0] += Slo;
      v[N - 1] += Shi;
    }
    // y faces: index (i,k); profile in j.   z faces: index (i,j); profile in k.
    {
      const double e0j = (j == 0) ? 1.0 : 0.0, e1j = (j == N - 1) ? 1.0 : 0.0;
      const double d0j = g.td0[j], d1j = g.td1[j];
      const double e0k = (k == 0) ? 1.0 : 0.0, e1k = (k == N - 1) ? 1.0 : 0.0;
      const double d0k = g.td0[k], d1k = g.td1[k];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int iy = i + N * k, iz = i + N * j;
        double s = v[i];
        s = fma(e0j, fy[0 * N2 + iy], s);
        s = fma(d0j, fy[1 * N2 + iy], s);
        s = fma(e1j, fy[2 * N2 + iy], s);
        s = fma(d1j, fy[3 * N2 + iy], s);
        s = fma(e0k, fz[0 * N2 + iz], s);
        s = fma(d0k, fz[1 * N2 + iz], s);
        s = fma(e1k, fz[2 * N2 + iz], s);
        s = fma(d1k, fz[3 * N2 + iz], s);
        v[i] = s;
      }
    }
    }
    out(cs, j, k, v);
  }
}

// ---- diag(D_T) from 1D diagonals (Jacobi preconditioner) --------------
template <int N, int NTH = Geo<N>::NT, int CC>
__device__ void diag_setup(const KParams& kp, const Group<N, CC>& g, double* Dg) {
  using G = Geo<N, CC>;
  const double area[3] = {kp.h[1] * kp.h[2], kp.h[0] * kp.h[2], kp.h[0] * kp.h[1]};
  for (int e = threadIdx.x; e < G::C * G::N3; e += NTH) {
    const int cs = e / G::N3, r = e % G::N3;
    const int idx[3] = {r % N, (r / N) % N, r / G::N2};
    double Md[3], Sd[3], Cd[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Md[a] = c_tab[N].Md[idx[a]];
      Sd[a] = c_tab[N].Sd[idx[a]];
      Cd[a] = c_tab[N].Cd[idx[a]];
    }
    const double* vc = g.vc[cs];
    const double* sb = g.vb[cs];
    double d = vc[3] * Md[0] * Md[1] * Md[2];
    d += (vc[0] * Sd[0] - sb[0] * Cd[0]) * Md[1] * Md[2];
    d += (vc[1] * Sd[1] - sb[1] * Cd[1]) * Md[0] * Md[2];
    d += (vc[2] * Sd[2] - sb[2] * Cd[2]) * Md[0] * Md[1];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double tm = area[a] * Md[(a + 1) % 3] * Md[(a + 2) % 3];
      const double ih = kp.ih[a];   // 1 / h_a (host-computed, identical IEEE quotient)
      if (idx[a] == 0) {
        const double* c = g.fc[cs][2 * a];
        const double dd = c_tab[N].d0[0];
        d += tm * (c[0] + c[1] * dd * ih + c[4] * dd);
      }
      if (idx[a] == N - 1) {
        const double* c = g.fc[cs][2 * a + 1];
        const double dd = c_tab[N].d1[N - 1];
        d += tm * (c[0] + c[1] * dd * ih + c[4] * dd);
      }
    }
    // stored inverted: the solvers multiply (no division per element and iteration)
    Dg[cs * G::CS + idx[2] * G::ZS + idx[1] * G::YS + idx[0]] = d != 0.0 ? 1.0 / d : 1.0;
  }
}

// per-cell sum of the per-line partials red[q][cs*N2 + l] -> result[q][cs]
template <int N, int CC>
__device__ __forceinline__ double cell_sum(const Group<N, CC>& g, int q, int cs) {
  constexpr int N2 = N * N;
  double s = 0.0;
  for (int l = 0; l < N2; ++l) s += g.red[q][cs * N2 + l];
  return s;
}

// line iteration helper over x-lines of the group: f(cs, off, item)
#define DG_FOR_XLINES(...)                                                             \
  for (int it = threadIdx.x; it < G::LINES; it += G::NT) {                            \
    const int cs = it / G::N2, l_ = it % G::N2;                                      \
    const int off = cs * G::CS + (l_ / N) * G::ZS + (l_ % N) * G::YS;                 \
    (void)off;                                                                        \
    __VA_ARGS__                                                                       \
  }

// =============================== kernels ========================================

// ---- asynchronous tile staging (cp.async: no registers held while the copies are in flight) --
__device__ __forceinline__ void lcp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void lcp_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void lcp_async16(double* dst, const double* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
// the group's own tile (contiguous in global) into the padded CS layout, zero past the end.
// Unpadded layouts (n = 3, 5: CS = n^3) are the global block itself: 16-byte copies (the group's
// first DoF is 16-byte aligned); padded ones one x-line per thread, its indices computed once per
// line (per element they cost ~45 instructions per 8-byte copy: 30 % of the C3 apply's issued
// instructions, ncu)
template <int N, int CC = Cells<N>::C>
__device__ __forceinline__ void async_tile(double* dst, const double* src, int nvalid) {
  using G = Geo<N, CC>;
  if constexpr (G::CS == G::N3 && G::ZS == G::N2 && G::YS == N && (G::C * G::N3) % 2 == 0) {
    const int nel = nvalid * G::N3;
    for (int c = threadIdx.x; c < G::C * G::N3 / 2; c += G::NT) {
      const int e = 2 * c;
      const int bytes = e + 2 <= nel ? 16 : (e < nel ? 8 : 0);
      lcp_async16(dst + e, src + (bytes ? e : 0), bytes);
    }
  } else if constexpr (N == 8) {
    // n = 8 (128 threads, one line each): consecutive lanes on consecutive elements (per-line
    // copies: p = 7 volume 81 -> 87 us, apply 142 -> 147 us)
    for (int e = threadIdx.x; e < G::C * G::N3; e += G::NT) {
      const int cs = e / G::N3, r = e % G::N3;
      const int i = r % N, j = (r / N) % N, k = r / G::N2;
      lcp_async8(dst + cs * G::CS + k * G::ZS + j * G::YS + i, src + (cs < nvalid ? e : 0), cs < nvalid);
    }
  } else {
    for (int ln = threadIdx.x; ln < G::C * G::N2; ln += G::NT) {
      const int cs = ln / G::N2, l = ln % G::N2, j = l % N, k = l / N;
      const bool v = cs < nvalid;
      double* d = dst + cs * G::CS + k * G::ZS + j * G::YS;
      const double* sp = src + (v ? cs * G::N3 + k * G::N2 + j * N : 0);
#pragma unroll
      for (int i = 0; i < N; ++i) lcp_async8(d + i, sp + (v ? i : 0), v);
    }
  }
}

// FACES = false, USEB = true: D_T (self faces as Gauss-point operators, no face passes).
// The own tile is staged with cp.async while the face setup runs; programmatic dependent launch
// lets the setup (coefficients only) overlap the previous kernel's tail (griddepcontrol.wait
// before the first read of u).
// cells per CTA of the CTA-wide line CG at n = 6, 7, 8 (the group size Cells<N>::C = 4, 4, 2 of
// the other line kernels). Fewer cells: a CTA runs until its slowest cell has converged, so small
// groups idle less; at n = 6 one cell leaves 28 of 64 threads without a line. Poisson sweeps
// (~8M DoF): n = 6 2413 (4 cells) / 2091 (3) / 1985 (2) / 2465 us (1); n = 7 3568 (4) / 3814
// (2) / 3519 us (1); n = 8 3806 (2) / 3479 us (1)
#ifndef DG_CG_CELLS6
#define DG_CG_CELLS6 2
#endif
#ifndef DG_CG_CELLS7
#define DG_CG_CELLS7 1
#endif
#ifndef DG_CG_CELLS8
#define DG_CG_CELLS8 1
#endif
template <int N> constexpr int line_cg_cells() {
  return N == 6 ? DG_CG_CELLS6 : (N == 7 ? DG_CG_CELLS7 : (N == 8 ? DG_CG_CELLS8 : Cells<N>::C));
}
// cells per CTA of the warp-per-cell BiCGStab at n = 5, 7 (convection sweeps, ~8M DoF: n = 5
// 2834 (8 cells) / 2807 (2) / 2795 us (1); n = 7 8282 (4) / 6874 (2) / 7809 us (1))
#ifndef DG_BICGW_CELLS5
#define DG_BICGW_CELLS5 1
#endif
#ifndef DG_BICGW_CELLS7
#define DG_BICGW_CELLS7 2
#endif
template <int N> constexpr int bicgw_cells() {
  return N == 5 ? DG_BICGW_CELLS5 : (N == 7 ? DG_BICGW_CELLS7 : Cells<N>::C);
}
// cells per CTA of the CTA-wide line BiCGStab at n = 6, 8 (Cells<N>::C = 4, 2); convection
// sweeps, ~8M DoF: n = 6 4115 (4 cells) / 4537 (3) / 3881 (2) / 4487 us (1); n = 8 5520 (2) / 5270 us (1)
#ifndef DG_BICG_CELLS6
#define DG_BICG_CELLS6 2
#endif
#ifndef DG_BICG_CELLS8
#define DG_BICG_CELLS8 1
#endif
template <int N> constexpr int bicg_cells() {
  return N == 6 ? DG_BICG_CELLS6 : (N == 8 ? DG_BICG_CELLS8 : Cells<N>::C);
}
#ifndef DG_CGW_CELLS
#define DG_CGW_CELLS 1   // cells per CTA of the warp-per-cell CG at n = 5
#endif
#ifndef DG_APPLY_NBR_PREFETCH
// bit n: the nodal apply at n prefetches the neighbours' face lines (p = 6: 221 -> 200 us; at
// n = 5, 6, 8 the registers held across the setup cost more occupancy than they save: C3
// 596 -> 635 us with 4 CTAs per SM, 685 us with spills at 5; p = 5 136 -> 142; p = 7 142 -> 161)
#define DG_APPLY_NBR_PREFETCH 0x80
#endif
#ifndef DG_APPLY_INPLACE
#define DG_APPLY_INPLACE 1   // nodal A u: z-face arrays in the consumed tile (8 C n^2 face buffer)
#endif
template <int N> constexpr size_t apply_fb_doubles() {
  return (DG_APPLY_INPLACE && N > 4 ? 8 : 12) * (size_t)Geo<N>::C * Geo<N>::N2;
}
template <int N, bool FACES, bool USEB, bool GEN>
__device__ __forceinline__ void k_apply_body(const KParams& kp, const double* __restrict__ u,
                                             double* __restrict__ out, int with_nbr, Group<N>& g) {
  using G = Geo<N>;
  extern __shared__ double sm[];
  double* SRC = sm;
  double* SA = SRC + G::TENSOR;
  double* SB = SA + G::TENSOR;
  double* FB = SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(G::C, kp.ncells - cell0);
  asm volatile("griddepcontrol.launch_dependents;");
#if DG_APPLY_SETUP_FIRST
  group_setup<N>(kp, g, cell0, with_nbr ? u : nullptr);  // pointers only; ends with __syncthreads
  asm volatile("griddepcontrol.wait;" ::: "memory");
  async_tile<N>(SRC, u + (size_t)cell0 * G::N3, nvalid);
#else
  // the tile copy is in flight while the setup's coefficient loads wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  async_tile<N>(SRC, u + (size_t)cell0 * G::N3, nvalid);
#endif
  // A u (faces, not the D_T hook) in the nodal Kronecker-sum form
  constexpr bool NODAL = DG_NODAL_APPLY && FACES && !USEB;
  // the neighbours' face lines in flight together with the setup's coefficient loads
  constexpr bool PRE = NODAL && ((DG_APPLY_NBR_PREFETCH >> N) & 1);
  NbrLines<N> W;
  if constexpr (PRE) nbr_lines_prefetch<N>(kp, with_nbr ? u : nullptr, cell0, W);
#if !DG_APPLY_SETUP_FIRST
  group_setup<N>(kp, g, cell0, with_nbr ? u : nullptr);  // ends with __syncthreads
#endif
  if constexpr (USEB) self_face_ops<N>(kp, g);
  lcp_wait_all();
  __syncthreads();
  double* o = out + (size_t)cell0 * G::N3;
  if constexpr (NODAL) {
    apply_nodal<N, Geo<N>::NT, GEN, (DG_APPLY_INPLACE && N > 4)>(kp, g, SRC, SA, SB, FB, [&](int cs, int j, int k, const double* w) {
      if (cs < nvalid) stg_line<N>(o + cs * G::N3 + k * G::N2 + j * N, w);
    }, PRE ? &W : nullptr);
    return;
  }
  cell_operator<N, FACES, USEB, false, Geo<N>::NT, GEN>(kp, g, SRC, SA, SB, FB, (kp.mask & 1u) != 0,
                          [&](int cs, int j, int k, const double* v) {
                            if (cs < nvalid) stg_line<N>(o + cs * G::N3 + k * G::N2 + j * N, v);
                          });
}

// The nodal A u (apply_nodal) with CC cells per CTA: CC = 1 makes every barrier of the four
// stages a one-warp barrier (no CTA-wide waits behind the slowest cell's neighbour loads), at
// 25 of 32 lanes busy at n = 5
#ifndef DG_APPLY1_MINB
#define DG_APPLY1_MINB 0   // resident CTAs the one-cell apply is compiled for (0: no bound)
#endif
template <int N, bool GEN, int CC>
__global__ void __launch_bounds__(Geo<N, CC>::NT, (CC == 1 ? DG_APPLY1_MINB : 0))
k_apply_nodal(KParams kp, const double* __restrict__ u, double* __restrict__ out, int) {
  using G = Geo<N, CC>;
  using GR = Group<N, CC>;
  using GH = GroupHead<N, CC>;
  static_assert(offsetof(GR, td1) == offsetof(GH, td1), "GroupHead is a prefix of Group");
  __shared__ GH gh;
  Group<N, CC>& g = *reinterpret_cast<Group<N, CC>*>(&gh);
  extern __shared__ double sm[];
#ifndef DG_APPLY1_REGSRC
#define DG_APPLY1_REGSRC 1   // one cell per CTA: the own x-line straight into registers, no tile
#endif
  constexpr bool REGSRC = DG_APPLY1_REGSRC && CC == 1;
  double* SRC = sm;
  double* SA = REGSRC ? sm : SRC + G::TENSOR;
  double* SB = SA + G::TENSOR;
  double* FB = SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * CC;
  const int nvalid = min(CC, kp.ncells - cell0);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double ownl[N];
  if constexpr (REGSRC) {
    const int t = threadIdx.x;
    if (t < G::LINES && nvalid > 0) {
      ld<N, 1>(u + (size_t)cell0 * G::N3 + (t / N) * G::N2 + (t % N) * N, ownl);
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) ownl[e] = 0.0;
    }
  } else {
    async_tile<N, CC>(SRC, u + (size_t)cell0 * G::N3, nvalid);
  }
#ifndef DG_APPLY1_PREFETCH
#define DG_APPLY1_PREFETCH 0   // the y / z neighbour lines loaded before the setup (registers; C3 530 -> 578 us)
#endif
  NbrLines<N> W;
  if constexpr (DG_APPLY1_PREFETCH) nbr_lines_prefetch<N, CC>(kp, u, cell0, W);
  group_setup<N, G::NT>(kp, g, cell0, u);  // ends with __syncthreads
  lcp_wait_all();
  __syncthreads();
  double* o = out + (size_t)cell0 * G::N3;
  apply_nodal<N, G::NT, GEN, (DG_APPLY_INPLACE && N > 4 && !REGSRC)>(kp, g, SRC, SA, SB, FB, [&](int cs, int j, int k, const double* w) {
    if (cs < nvalid) stg_line<N>(o + cs * G::N3 + k * G::N2 + j * N, w);
  }, DG_APPLY1_PREFETCH ? &W : nullptr, REGSRC ? ownl : nullptr);
}
// Warp mode: CC independent cells per CTA, one warp each (apply_nodal<..., WARP = true>: the
// stages synchronise per warp, the x neighbours come from global memory, the own x-line straight
// into registers); the CTA barrier only after the coefficient setup. More resident warps than
// the 32 one-warp CTAs an SM can hold.
#ifndef DG_APPLYW_MINB
#define DG_APPLYW_MINB 0
#endif
template <int N> __host__ __device__ constexpr int warp_lanes() { return N * N <= 16 ? 16 : 32; }   // lanes per cell
#ifndef DG_APPLYW_ROWS
// bit n: the warp-mode apply's face arrays in padded 16-byte rows (apply_nodal RS). Off: the
// row reads are 2-wavefront LDS.64 with 5 distinct addresses per warp either way, and the 128-bit
// pairs did not halve them (C3 apply 493 -> 511 us; the face-row contractions are 36 % of the
// kernel's shared-memory wavefronts, ncu)
#define DG_APPLYW_ROWS 0
#endif
// face-array row stride of the warp-mode apply (N + 1 rounded up to even where enabled)
#ifndef DG_APPLYW_SHFL
// bit n: the warp-mode apply's face contractions by shuffles (apply_nodal SHUF). Off: the
// shuffles cost the same pipe as the shared-memory face arrays they replace and raise the
// registers (C3 apply 493 -> 529 us at 80 registers, 503 us capped at 64; C2 32.9 -> 34.2 us)
#define DG_APPLYW_SHFL 0
#endif
template <int N> __host__ __device__ constexpr bool apply_warps_shfl() { return (DG_APPLYW_SHFL >> N) & 1; }
template <int N> __host__ __device__ constexpr int apply_warps_rs() { return ((DG_APPLYW_ROWS >> N) & 1) ? ((N + 2) & ~1) : N; }
template <int N, bool GEN, int CC>
__global__ void __launch_bounds__(CC * warp_lanes<N>(), DG_APPLYW_MINB)
k_apply_warps(KParams kp, const double* __restrict__ u, double* __restrict__ out, int) {
  using G = Geo<N, CC>;
  using GR = Group<N, CC>;
  using GH = GroupHead<N, CC>;
  static_assert(offsetof(GR, td1) == offsetof(GH, td1), "GroupHead is a prefix of Group");
  static_assert(G::N2 <= 32, "one warp per cell");
  __shared__ GH gh;
  Group<N, CC>& g = *reinterpret_cast<Group<N, CC>*>(&gh);
  extern __shared__ double sm[];
  double* SA = sm;
  double* SB = SA + G::TENSOR;
  double* FB = SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * CC;
  const int nvalid = min(CC, kp.ncells - cell0);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int WL = warp_lanes<N>();
  static_assert((CC * WL) % 32 == 0, "whole warps");
  const int t = threadIdx.x, cs = t / WL, l = t % WL;
  double ownl[N];
  if (l < G::N2 && cs < nvalid) {
    ld<N, 1>(u + (size_t)(cell0 + cs) * G::N3 + (l / N) * G::N2 + (l % N) * N, ownl);
  } else {
#pragma unroll
    for (int e = 0; e < N; ++e) ownl[e] = 0.0;
  }
  group_setup<N, CC * WL>(kp, g, cell0, u);  // ends with __syncthreads
  double* o = out + (size_t)cell0 * G::N3;
  apply_nodal<N, CC * WL, GEN, false, true, apply_warps_rs<N>(), apply_warps_shfl<N>()>(kp, g, SA, SA, SB, FB, [&](int c, int j, int k, const double* w) {
    if (c < nvalid) stg_line<N>(o + c * G::N3 + k * G::N2 + j * N, w);
  }, nullptr, ownl);
}
template <int N, int CC> constexpr size_t apply_warps_smem() {
  return sizeof(double) * (2 * (size_t)Geo<N, CC>::TENSOR + (apply_warps_shfl<N>() ? 0 : 12 * (size_t)CC * N * apply_warps_rs<N>()));
}

// Mass-folded nodal A u, one warp per cell (n^2 <= 32 lanes, one line each). With exact 1D masses
// every term of (A u)_T carries Mhat in the directions it does not act on, so
//   (A u)_T = (Mhat (x) Mhat (x) Mhat) w,
//   w = sum_a [ vc_a Mhat^-1 Shat - vb_a Mhat^-1 Chat ]_a u + vc_3 u
//       + sum_a |F_a| [ (Mhat^-1 e0) S_lo + (Mhat^-1 d0) T_lo + (Mhat^-1 e1) S_hi + (Mhat^-1 d1) T_hi ]_a
// with S, T the value-test and derivative-test face sums (self and neighbour, the fc coefficients
// of group_setup) at the face node, which the lane that owns the normal line through
// that node forms in registers: no face arrays, no tangential-mass contractions of face data, no
// per-cell factor matrices (the 1D tables are constant-bank operands). Six line products
// (three derivative, three mass) instead of seven plus twelve face-array contractions.
// Stages: own x-line -> shared; z-lines: w_z; y-lines: += w_y; x-lines: += w_x, Mhat_x; y-lines:
// Mhat_y; z-lines: Mhat_z, stored to global memory as z-lines (n^2 consecutive doubles per k).
#ifndef DG_APPLY_FOLD5
#define DG_APPLY_FOLD5 4   // n = 5: cells (= warps) per CTA of the mass-folded apply (0: off)
#endif
#ifndef DG_APPLY_FOLD4
#define DG_APPLY_FOLD4 8   // n = 4: cells (half-warps) per CTA (0: off)
#endif
#ifndef DG_APPLY_FOLD3
// n = 3: cells per CTA, three per warp (27 of 32 lanes busy; half-warp cells: C5 580 us; 12 cells
// in 4 warps: 459 us, but a group size with a factor 3 triples the range granule). 20 cells in 7
// warps divide the other kernels' groups. (0: off)
#define DG_APPLY_FOLD3 20
#endif
template <int N, bool GEN>
__device__ __forceinline__ void fold_line(const KParams& kp, int a, const double* vc, const double* vb,
                                          const double* lo, const double* hi, const double (&u)[N],
                                          double sl, double tl, double sh, double th, double (&w)[N]) {
  double g0 = 0.0, g1 = 0.0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    g0 = fma(c_tab[N].d0[e], u[e], g0);
    g1 = fma(c_tab[N].d1[e], u[e], g1);
  }
  const double ih = kp.ih[a], fa = kp.fa[a];
  const double Sl = fa * (sl + fma(lo[0], u[0], (lo[1] * g0) * ih));
  const double Tl = fa * fma(lo[4], u[0], tl);
  const double Sh = fa * (sh + fma(hi[0], u[N - 1], (hi[1] * g1) * ih));
  const double Th = fa * fma(hi[4], u[N - 1], th);
  const double vk = vc[a], vbb = GEN ? vb[a] : 0.0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    double s = 0.0, c = 0.0;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      s = fma(c_fold.MiS[e * N + r], u[r], s);
      if constexpr (GEN) c = fma(c_fold.MiC[e * N + r], u[r], c);
    }
    double acc = fma(vk, s, w[e]);
    if constexpr (GEN) acc = fma(-vbb, c, acc);
    acc = fma(c_fold.mie0[e], Sl, acc);
    acc = fma(c_fold.mid0[e], Tl, acc);
    acc = fma(c_fold.mie1[e], Sh, acc);
    acc = fma(c_fold.mid1[e], Th, acc);
    w[e] = acc;
  }
}
#ifndef DG_APPLYF_PRE
// 1: the neighbours' traces loaded and reduced before the coefficient setup (12 scalars live across
// its barrier). Measured slower (72 registers, 7 CTAs per SM): C3 367 -> 380 us, C4 193 -> 199, C5 490 -> 513
#define DG_APPLYF_PRE 0
#endif
#ifndef DG_APPLYF_MINB
#define DG_APPLYF_MINB 0   // resident CTAs the mass-folded apply is compiled for (0: no bound)
#endif
// lanes per cell: a warp at n = 5 (25 busy), a half-warp at n = 4, 9 lanes at n = 3 (three cells per
// warp, 27 of 32 lanes busy)
template <int N> __host__ __device__ constexpr int fold_wl() { return N == 3 ? 9 : warp_lanes<N>(); }
template <int N, int CC> __host__ __device__ constexpr int fold_threads() {
  constexpr int CPW = 32 / fold_wl<N>();
  return (CC + CPW - 1) / CPW * 32;   // the last warp may hold fewer cells
}
template <int N, bool GEN, int CC>
__global__ void __launch_bounds__(fold_threads<N, CC>(), DG_APPLYF_MINB)
k_apply_fold(KParams kp, const double* __restrict__ u, double* __restrict__ out, int) {
  using G = Geo<N, CC>;
  using GR = Group<N, CC>;
  using GH = GroupHead<N, CC>;
  static_assert(offsetof(GR, td1) == offsetof(GH, td1), "GroupHead is a prefix of Group");
  static_assert(G::N2 <= 32, "one warp (n^2 <= 16: half-warp) per cell");
  constexpr int WL = fold_wl<N>(), CPW = 32 / WL, NTH = fold_threads<N, CC>();
  __shared__ GH gh;
  Group<N, CC>& g = *reinterpret_cast<Group<N, CC>*>(&gh);
  extern __shared__ double sm[];
  double* SU = sm;
  double* SA = SU + G::TENSOR;
  constexpr int N2 = G::N2;
  const int cell0 = block_group(kp, false) * CC;
  const int nvalid = min(CC, kp.ncells - cell0);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int t = threadIdx.x, ln = t & 31, cs = (t >> 5) * CPW + ln / WL, l = ln % WL, a = l % N, bb = l / N;
  const bool act = ln < CPW * WL && l < N2 && cs < nvalid;
  double own[N];
  if (act) {
    ld<N, 1>(u + (size_t)(cell0 + cs) * G::N3 + bb * N2 + a * N, own);
  } else {
#pragma unroll
    for (int e = 0; e < N; ++e) own[e] = 0.0;
  }
#if DG_APPLYF_PRE
  // the neighbours' face values and normal-derivative sums at this lane's face nodes, loaded and
  // reduced before the coefficient setup (their latency runs under the setup's own loads; 12
  // scalars live across the barrier). The neighbour of face f: the in-slab cell, the ghost trace
  // record at a slab boundary (FK_GHOST), or none (as setup_cells decides).
  double nav[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, ngn[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  unsigned nmask = 0;
  if (act) {
    const int cell = cell0 + cs, nxy = kp.nx * kp.ny;
    const int cx = cell % kp.nx, cy = (cell / kp.nx) % kp.ny, cz = cell / nxy;
    const double* uc = u + (size_t)cell * G::N3;
    if (cx > 0) {
      double w[N];
      ldg_line<N>(uc - G::N3 + bb * N2 + a * N, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d1[e], w[e], gsum);
      nav[0] = w[N - 1]; ngn[0] = gsum; nmask |= 1u;
    }
    if (cx < kp.nx - 1) {
      double w[N];
      ldg_line<N>(uc + G::N3 + bb * N2 + a * N, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d0[e], w[e], gsum);
      nav[1] = w[0]; ngn[1] = gsum; nmask |= 2u;
    }
    if (cy > 0) {
      double w[N];
      ld<N, N>(uc - (size_t)kp.nx * G::N3 + bb * N2 + a, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d1[e], w[e], gsum);
      nav[2] = w[N - 1]; ngn[2] = gsum; nmask |= 4u;
    }
    if (cy < kp.ny - 1) {
      double w[N];
      ld<N, N>(uc + (size_t)kp.nx * G::N3 + bb * N2 + a, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d0[e], w[e], gsum);
      nav[3] = w[0]; ngn[3] = gsum; nmask |= 8u;
    }
    const int col = cx + kp.nx * cy;
    if (cz > 0) {
      double w[N];
      ld<N, N2>(uc - (size_t)nxy * G::N3 + bb * N + a, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d1[e], w[e], gsum);
      nav[4] = w[N - 1]; ngn[4] = gsum; nmask |= 16u;
    } else if (kp.slab_face[4] == FK_GHOST) {
      const double* rec = kp.ghost_lo + (size_t)col * 2 * N2;
      nav[4] = rec[bb * N + a]; ngn[4] = rec[N2 + bb * N + a]; nmask |= 16u;
    }
    if (cz < kp.nzl - 1) {
      double w[N];
      ld<N, N2>(uc + (size_t)nxy * G::N3 + bb * N + a, w);
      double gsum = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) gsum = fma(c_tab[N].d0[e], w[e], gsum);
      nav[5] = w[0]; ngn[5] = gsum; nmask |= 32u;
    } else if (kp.slab_face[5] == FK_GHOST) {
      const double* rec = kp.ghost_hi + (size_t)col * 2 * N2;
      nav[5] = rec[bb * N + a]; ngn[5] = rec[N2 + bb * N + a]; nmask |= 32u;
    }
  }
  group_setup<N, NTH>(kp, g, cell0, u);  // ends with __syncthreads
  const int base = cs * G::CS;
  double sx[4] = {0.0, 0.0, 0.0, 0.0}, sy[4] = {0.0, 0.0, 0.0, 0.0}, sz[4] = {0.0, 0.0, 0.0, 0.0};
  if (act) {
    st<N, 1>(SU + base + bb * G::ZS + a * G::YS, own);
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (!((nmask >> f) & 1u)) continue;
      const double* cf = g.fc[cs][f];
      const double sv = fma(cf[2], nav[f], (cf[3] * ngn[f]) * kp.ih[f >> 1]);
      const double tv = cf[5] * nav[f];
      double* dst = (f >> 1) == 0 ? sx : ((f >> 1) == 1 ? sy : sz);
      dst[2 * (f & 1)] = sv;
      dst[2 * (f & 1) + 1] = tv;
    }
  }
#else
  group_setup<N, NTH>(kp, g, cell0, u);  // ends with __syncthreads
  const int base = cs * G::CS;
  // ---- stage 0: the neighbours' parts of the face sums at this lane's face nodes (as apply_nodal)
  double sx[4] = {0.0, 0.0, 0.0, 0.0}, sy[4] = {0.0, 0.0, 0.0, 0.0}, sz[4] = {0.0, 0.0, 0.0, 0.0};
  if (act) {
    st<N, 1>(SU + base + bb * G::ZS + a * G::YS, own);
    {
      const double* nlo = g.nb[cs][0];
      const double* nhi = g.nb[cs][1];
      const double* clo = g.fc[cs][0];
      const double* chi = g.fc[cs][1];
      const int goff = bb * N2 + a * N;
      if (nlo) {
        double w[N];
        ldg_line<N>(nlo + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
        sx[0] = fma(clo[2], w[N - 1], (clo[3] * gn) * kp.ih[0]);
        sx[1] = clo[5] * w[N - 1];
      }
      if (nhi) {
        double w[N];
        ldg_line<N>(nhi + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
        sx[2] = fma(chi[2], w[0], (chi[3] * gn) * kp.ih[0]);
        sx[3] = chi[5] * w[0];
      }
    }
    {
      const double* nlo = g.nb[cs][2];
      const double* nhi = g.nb[cs][3];
      const double* clo = g.fc[cs][2];
      const double* chi = g.fc[cs][3];
      const int goff = bb * N2 + a;
      if (nlo) {
        double w[N];
        ld<N, N>(nlo + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
        sy[0] = fma(clo[2], w[N - 1], (clo[3] * gn) * kp.ih[1]);
        sy[1] = clo[5] * w[N - 1];
      }
      if (nhi) {
        double w[N];
        ld<N, N>(nhi + goff, w);
        double gn = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
        sy[2] = fma(chi[2], w[0], (chi[3] * gn) * kp.ih[1]);
        sy[3] = chi[5] * w[0];
      }
    }
    {
      const double* nlo = g.nb[cs][4];
      const double* nhi = g.nb[cs][5];
      const double* clo = g.fc[cs][4];
      const double* chi = g.fc[cs][5];
      const int goff = bb * N + a;
      if (nlo) {
        double av, gn = 0.0;
        if (ghost_trace(kp, g.cell[cs], 0)) {
          av = nlo[goff];
          gn = nlo[N2 + goff];
        } else {
          double w[N];
          ld<N, N2>(nlo + goff, w);
#pragma unroll
          for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d1[e], w[e], gn);
          av = w[N - 1];
        }
        sz[0] = fma(clo[2], av, (clo[3] * gn) * kp.ih[2]);
        sz[1] = clo[5] * av;
      }
      if (nhi) {
        double av, gn = 0.0;
        if (ghost_trace(kp, g.cell[cs], 1)) {
          av = nhi[goff];
          gn = nhi[N2 + goff];
        } else {
          double w[N];
          ld<N, N2>(nhi + goff, w);
#pragma unroll
          for (int e = 0; e < N; ++e) gn = fma(c_tab[N].d0[e], w[e], gn);
          av = w[0];
        }
        sz[2] = fma(chi[2], av, (chi[3] * gn) * kp.ih[2]);
        sz[3] = chi[5] * av;
      }
    }
  }
#endif
  __syncwarp();
  const double* vc = g.vc[cs];
  const double* vb = g.vb[cs];
  // ---- z-lines (i = a, j = bb): w = w_z (+ reaction)
  if (act) {
    const int off = base + bb * G::YS + a;
    double v[N], w[N];
    ld<N, G::ZS>(SU + off, v);
#pragma unroll
    for (int e = 0; e < N; ++e) w[e] = GEN ? vc[3] * v[e] : 0.0;
    fold_line<N, GEN>(kp, 2, vc, vb, g.fc[cs][4], g.fc[cs][5], v, sz[0], sz[1], sz[2], sz[3], w);
    st<N, G::ZS>(SA + off, w);
  }
  __syncwarp();
  // ---- y-lines (i = a, k = bb): w += w_y
  if (act) {
    const int off = base + bb * G::ZS + a;
    double v[N], w[N];
    ld<N, G::YS>(SU + off, v);
    ld<N, G::YS>(SA + off, w);
    fold_line<N, GEN>(kp, 1, vc, vb, g.fc[cs][2], g.fc[cs][3], v, sy[0], sy[1], sy[2], sy[3], w);
    st<N, G::YS>(SA + off, w);
  }
  __syncwarp();
  // ---- x-lines (j = a, k = bb): w += w_x, then Mhat_x
  if (act) {
    const int off = base + bb * G::ZS + a * G::YS;
    double w[N], c[N];
    ld<N, 1>(SA + off, w);
    fold_line<N, GEN>(kp, 0, vc, vb, g.fc[cs][0], g.fc[cs][1], own, sx[0], sx[1], sx[2], sx[3], w);
    mv<N, 2>(w, c);
    st<N, 1>(SA + off, c);
  }
  __syncwarp();
  // ---- y-lines: Mhat_y
  if (act) {
    const int off = base + bb * G::ZS + a;
    double c[N], d[N];
    ld<N, G::YS>(SA + off, c);
    mv<N, 2>(c, d);
    st<N, G::YS>(SA + off, d);
  }
  __syncwarp();
  // ---- z-lines: Mhat_z, to global memory (lane (i, j): n^2 consecutive doubles per k)
  if (act) {
    double d[N], o[N];
    ld<N, G::ZS>(SA + base + bb * G::YS + a, d);
    mv<N, 2>(d, o);
    double* op = out + (size_t)(cell0 + cs) * G::N3 + bb * N + a;
#pragma unroll
    for (int k = 0; k < N; ++k) op[k * N2] = o[k];
  }
}
template <int N, int CC> constexpr size_t apply_fold_smem() { return sizeof(double) * 2 * (size_t)Geo<N, CC>::TENSOR; }

// D_T u (dg_block_diag_apply: the volume and self-face terms of each cell) with one
// warp per cell in the nodal Kronecker-sum form of the local CG's operator (dt_nodal, WARP mode;
// the factors K_a of nodal_face_ops): the own x-line from global memory straight into registers,
// the result from registers to global memory, two work tensors in shared memory. Replaces the
// Gauss-point line kernel k_apply<N, false, true> at n = 5 (C3 D_T: 569 us, 0.29 of the fp64 peak).
template <int N, bool GEN, int CC>
__global__ void __launch_bounds__(CC * 32)
k_dt_warps(KParams kp, const double* __restrict__ u, double* __restrict__ out, int) {
  using G = Geo<N, CC>;
  static_assert(G::N2 <= 32, "one warp per cell");
  __shared__ Group<N, CC> g;
  extern __shared__ double sm[];
  double* SA = sm;
  double* SB = SA + G::TENSOR;
  const int cell0 = block_group(kp, false) * CC;
  const int nvalid = min(CC, kp.ncells - cell0);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int t = threadIdx.x, cs = t >> 5, l = t & 31;
  const bool act = l < G::N2 && cs < nvalid;
  double ownl[N], q[N];
  if (act) {
    ld<N, 1>(u + (size_t)(cell0 + cs) * G::N3 + (l / N) * G::N2 + (l % N) * N, ownl);
  } else {
#pragma unroll
    for (int e = 0; e < N; ++e) ownl[e] = 0.0;
  }
  group_setup<N, CC * 32>(kp, g, cell0, nullptr);   // coefficients only; ends with __syncthreads
  nodal_face_ops<N, CC * 32>(kp, g);                // K_x, K_y, K_z per cell; ends with __syncthreads
  dt_nodal<N, true, 0, GEN>(g, SA, SB, ownl, q, &kp);
  if (act) stg_line<N>(out + (size_t)(cell0 + cs) * G::N3 + (l / N) * G::N2 + (l % N) * N, q);
}

template <int N, int CC> constexpr size_t apply_nodal_smem() {
  // REGSRC (one cell per CTA): no tile; the z-face arrays after Mhat_x in the face buffer
  return CC == 1 && DG_APPLY1_REGSRC ? sizeof(double) * (2 * (size_t)Geo<N, CC>::TENSOR + 12 * (size_t)N * N)
                                     : sizeof(double) * (3 * (size_t)Geo<N, CC>::TENSOR + (DG_APPLY_INPLACE && N > 4 ? 8 : 12) * (size_t)CC * N * N);
}

// resident CTAs the line apply is compiled for (n = 5: five by shared memory after INPLACE,
// registers capped at 56 so that the register file allows them too)
#ifndef DG_APPLY5_MINB
#define DG_APPLY5_MINB 5
#endif
template <int N> constexpr int apply_minb() { return N == 5 ? DG_APPLY5_MINB : 0; }   // 0: no .minnctapersm
template <int N, bool FACES = true, bool USEB = false, bool GEN = true>
__global__ void __launch_bounds__(Geo<N>::NT, apply_minb<N>())
k_apply(KParams kp, const double* __restrict__ u, double* __restrict__ out, int with_nbr) {
  if constexpr ((DG_NODAL_APPLY && FACES && !USEB) || (!FACES && !USEB)) {
    // the nodal apply and the volume terms alone touch only the head of the group block
    static_assert(offsetof(Group<N>, td1) == offsetof(GroupHead<N>, td1), "GroupHead is a prefix of Group");
    __shared__ GroupHead<N> gh;
    k_apply_body<N, FACES, USEB, GEN>(kp, u, out, with_nbr, *reinterpret_cast<Group<N>*>(&gh));
  } else {
    __shared__ Group<N> g;
    k_apply_body<N, FACES, USEB, GEN>(kp, u, out, with_nbr, g);
  }
}

// ---- the volume terms alone, lean line kernel (dg_apply_parts mask = volume, n >= 6) ----------
// The passes and arithmetic of cell_operator<N, FACES = false> (stage 1: A_x, A_y, A_z to the
// Gauss points; stage 2: reaction and the x / y / z direction terms at the Gauss points; stage 3:
// the transposed contractions), without its instruction overhead (ncu, p = 5: DFMA
// were 25 % of the issued instructions; the passes recomputed the line indices per loop, the
// tile copy spent ~45 instructions per 8-byte cp.async): each thread owns L x-lines with the same
// (j, k) in the cells cs and cs + CC / L (so the three line offsets and the Gauss weight are
// computed once and every constant-bank table entry loaded into a uniform register feeds L
// DFMA), the cells' scalars live in registers (loaded before the dependency wait), the own
// x-lines are read from global memory straight into registers and the result is written from
// registers, so only the two work tensors live in shared memory. Per line the FMA order is that
// of mv / mtv / dir_term (the results equal cell_operator's bit for bit).
template <int N, int W, int L> __device__ __forceinline__ void mvL(const double (&in)[L][N], double (&out)[L][N]) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double s[L];
#pragma unroll
    for (int m = 0; m < L; ++m) s[m] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double c = tab<N, W>(q * N + j);
#pragma unroll
      for (int m = 0; m < L; ++m) s[m] = fma(c, in[m][j], s[m]);
    }
#pragma unroll
    for (int m = 0; m < L; ++m) out[m][q] = s[m];
  }
}
template <int N, int W, int L> __device__ __forceinline__ void mtvL(const double (&in)[L][N], double (&out)[L][N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double s[L];
#pragma unroll
    for (int m = 0; m < L; ++m) s[m] = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const double c = tab<N, W>(q * N + j);
#pragma unroll
      for (int m = 0; m < L; ++m) s[m] = fma(c, in[m][q], s[m]);
    }
#pragma unroll
    for (int m = 0; m < L; ++m) out[m][j] = s[m];
  }
}
// dir_term for L lines (per-line scalings sK[m], sb[m]; the same FMA order per line)
template <int N, bool GEN, int L>
__device__ __forceinline__ void dir_termL(const double (&U)[L][N], double (&R)[L][N], double Wl,
                                          const double (&sK)[L], const double (&sb)[L]) {
  if constexpr (!GEN) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double s[L];
#pragma unroll
      for (int m = 0; m < L; ++m) s[m] = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const double c = c_tab[N].SG[r * N + q];
#pragma unroll
        for (int m = 0; m < L; ++m) s[m] = fma(c, U[m][q], s[m]);
      }
#pragma unroll
      for (int m = 0; m < L; ++m) R[m][r] = fma(Wl * sK[m], s[m], R[m][r]);
    }
    return;
  }
  double du[L][N], F[L][N], t[L][N];
  mvL<N, 1, L>(U, du);
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int m = 0; m < L; ++m) F[m][q] = Wl * c_tab[N].w[q] * fma(sK[m], du[m][q], -sb[m] * U[m][q]);
  mtvL<N, 1, L>(F, t);
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int m = 0; m < L; ++m) R[m][r] += t[m][r];
}
template <int N, int L, int CC> struct VolLine {
  static_assert(CC % L == 0, "L lines per thread: cells cs + i CC / L");
  static constexpr int LINES = CC / L * N * N;            // threads with lines
  static constexpr int NT = ((LINES + 31) / 32) * 32;
};
// TILE: the own x-lines from a tile staged in SA by coalesced cp.async (one element per lane)
// instead of per-lane line loads
template <int N, bool GEN, int L, int CC, bool TILE = false>
__global__ void __launch_bounds__(VolLine<N, L, CC>::NT)
k_volume_line(KParams kp, const double* __restrict__ u, double* __restrict__ out, int) {
  using G = Geo<N, CC>;
  using V = VolLine<N, L, CC>;
  constexpr int N2 = G::N2, N3 = G::N3, CL = CC / L;
  extern __shared__ double sm[];
  double* SA = sm;
  double* SB = SA + G::TENSOR;
  const int t = threadIdx.x;
  const int cell0 = block_group(kp, false) * CC;
  const bool act = t < V::LINES;
  const int cs = act ? t / N2 : 0, l = t % N2, a = l % N, b = l / N;
  const int ox = cs * G::CS + b * G::ZS + a * G::YS;   // x-line (j = a, k = b) of line 0
  const int oy = cs * G::CS + b * G::ZS + a;           // y-line (i = a, k = b)
  const int oz = cs * G::CS + b * G::YS + a;           // z-line (i = a, j = b)
  constexpr int LS = CL * G::CS;                        // line m: + m LS (cell cs + m CL)
  bool valid[L];
  int cell[L];
#pragma unroll
  for (int m = 0; m < L; ++m) {
    cell[m] = cell0 + cs + m * CL;
    valid[m] = act && cell[m] < kp.ncells;
  }
  asm volatile("griddepcontrol.launch_dependents;");
  // the cells' scalings (cell_operator: g.vc, g.vb from setup_cells), independent of u
  double sK[3][L], sb[3][L], sc[L];
#pragma unroll
  for (int m = 0; m < L; ++m) {
    sc[m] = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) sK[d][m] = sb[d][m] = 0.0;
    if (valid[m]) {
      const int nxy = kp.nx * kp.ny;
      const double vol = kp.h[0] * kp.h[1] * kp.h[2];
      const double* Kc = kp.K + (size_t)(cell[m] + nxy) * 3;
#pragma unroll
      for (int d = 0; d < 3; ++d) sK[d][m] = Kc[d] * vol * kp.ih[d] * kp.ih[d];
      if constexpr (GEN) {
        sc[m] = kp.c ? vol * kp.c[cell[m]] : 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d)
          sb[d][m] = vol * (kp.bc ? kp.bc[(size_t)(cell[m] + nxy) * 3 + d] : kp.b[d]) * kp.ih[d];
      }
    }
  }
  const double Wl = c_tab[N].w[a] * c_tab[N].w[b];   // (the same product in every pass)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double v[L][N], o[L][N];
  if constexpr (TILE) {
    const int nvalid = min(CC, kp.ncells - cell0);
    const double* src = u + (size_t)cell0 * N3;
    for (int e = t; e < CC * N3; e += V::NT) {
      const int c = e / N3, r = e % N3;
      const int i = r % N, j = (r / N) % N, k = r / N2;
      lcp_async8(SA + c * G::CS + k * G::ZS + j * G::YS + i, src + (c < nvalid ? e : 0), c < nvalid);
    }
    lcp_wait_all();
    __syncthreads();
#pragma unroll
    for (int m = 0; m < L; ++m) ld<N, 1>(SA + ox + m * LS, v[m]);
    __syncthreads();
  } else {
#pragma unroll
    for (int m = 0; m < L; ++m) {
      if (valid[m]) {
        ldg_line<N>(u + (size_t)cell[m] * N3 + b * N2 + a * N, v[m]);
      } else {
#pragma unroll
        for (int e = 0; e < N; ++e) v[m][e] = 0.0;
      }
    }
  }
  // pass 1: x-lines, SA = A_x u
  if (act) {
    mvL<N, 0, L>(v, o);
#pragma unroll
    for (int m = 0; m < L; ++m) st<N, 1>(SA + ox + m * LS, o[m]);
  }
  __syncthreads();
  // pass 2: y-lines, SB = A_y SA
  if (act) {
#pragma unroll
    for (int m = 0; m < L; ++m) ld<N, G::YS>(SA + oy + m * LS, v[m]);
    mvL<N, 0, L>(v, o);
#pragma unroll
    for (int m = 0; m < L; ++m) st<N, G::YS>(SB + oy + m * LS, o[m]);
  }
  __syncthreads();
  // pass 3: z-lines, U = A_z SB -> SA, R = reaction + z-term -> SB
  if (act) {
    double U[L][N], R[L][N];
#pragma unroll
    for (int m = 0; m < L; ++m) ld<N, G::ZS>(SB + oz + m * LS, v[m]);
    mvL<N, 0, L>(v, U);
#pragma unroll
    for (int m = 0; m < L; ++m)
#pragma unroll
      for (int q = 0; q < N; ++q) R[m][q] = GEN ? Wl * c_tab[N].w[q] * sc[m] * U[m][q] : 0.0;
    dir_termL<N, GEN, L>(U, R, Wl, sK[2], sb[2]);
#pragma unroll
    for (int m = 0; m < L; ++m) {
      st<N, G::ZS>(SA + oz + m * LS, U[m]);
      st<N, G::ZS>(SB + oz + m * LS, R[m]);
    }
  }
  __syncthreads();
  // pass 4: x-lines, R += x-term
  if (act) {
    double U[L][N], R[L][N];
#pragma unroll
    for (int m = 0; m < L; ++m) {
      ld<N, 1>(SA + ox + m * LS, U[m]);
      ld<N, 1>(SB + ox + m * LS, R[m]);
    }
    dir_termL<N, GEN, L>(U, R, Wl, sK[0], sb[0]);
#pragma unroll
    for (int m = 0; m < L; ++m) st<N, 1>(SB + ox + m * LS, R[m]);
  }
  __syncthreads();
  // pass 5: y-lines, R += y-term, then A_y^T
  if (act) {
    double U[L][N], R[L][N];
#pragma unroll
    for (int m = 0; m < L; ++m) {
      ld<N, G::YS>(SA + oy + m * LS, U[m]);
      ld<N, G::YS>(SB + oy + m * LS, R[m]);
    }
    dir_termL<N, GEN, L>(U, R, Wl, sK[1], sb[1]);
    mtvL<N, 0, L>(R, o);
#pragma unroll
    for (int m = 0; m < L; ++m) st<N, G::YS>(SB + oy + m * LS, o[m]);
  }
  __syncthreads();
  // pass 6: z-lines, A_z^T
  if (act) {
#pragma unroll
    for (int m = 0; m < L; ++m) ld<N, G::ZS>(SB + oz + m * LS, v[m]);
    mtvL<N, 0, L>(v, o);
#pragma unroll
    for (int m = 0; m < L; ++m) st<N, G::ZS>(SB + oz + m * LS, o[m]);
  }
  __syncthreads();
  // pass 7: x-lines, A_x^T, straight to global memory
  if (act) {
#pragma unroll
    for (int m = 0; m < L; ++m) ld<N, 1>(SB + ox + m * LS, v[m]);
    mtvL<N, 0, L>(v, o);
#pragma unroll
    for (int m = 0; m < L; ++m)
      if (valid[m]) stg_line<N>(out + (size_t)cell[m] * N3 + b * N2 + a * N, o[m]);
  }
}

// Jacobi-preconditioned CG on every cell of the group (SPD blocks, b = 0).
// SWEEP: in = u (defect d = f - A u formed first), result u + omega du; else in = d, result du.
template <int N, bool SWEEP, int CC = Cells<N>::C>
__global__ void __launch_bounds__(Geo<N, CC>::NT, (CC == Cells<N>::C ? 2 : 0))   // two CTAs per SM (n = 7: <= 146 registers)
k_cg(KParams kp, const double* __restrict__ in, const double* __restrict__ f,
     double* __restrict__ out) {
  using G = Geo<N, CC>;
  constexpr int C = G::C;
  extern __shared__ double sm[];
  __shared__ Group<N, CC> g;
  double* X = sm;
  double* R = X + G::TENSOR;
  double* P = R + G::TENSOR;
  double* Q = P + G::TENSOR;
  double* Dg = Q + G::TENSOR;
  double* SA = Dg + G::TENSOR;
  double* SB = SA + G::TENSOR;
  // the face buffer is only used by the defect (the loop's D_T takes the self faces through
  // g.Bf), before Q and Dg are: it aliases them when it fits
  double* FB = fb_alias<N, CC>() ? Q : SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(C, kp.ncells - cell0);
  const int tid = threadIdx.x;
  load_tile<N, G::NT>(g, cell0, kp.ncells, in, SWEEP ? P : R);
  const KParams& kq = kp;   // launched with mask = 7 (launch_local_solve / launch_sweep)
  group_setup<N, G::NT>(kq, g, cell0, SWEEP ? in : nullptr);
  constexpr bool NODAL = DG_NODAL_DT;   // D_T of the iterations in the nodal Kronecker-sum form
  if constexpr (NODAL) nodal_face_ops<N, G::NT>(kq, g);
  else self_face_ops<N, G::NT>(kq, g);   // D_T in the loop: self faces at the Gauss points
  if (SWEEP) {  // d = f - A u  (Alg. 2 line 2)
    const double* fb = f + (size_t)cell0 * G::N3;
    auto defect = [&](int cs, int j, int k, const double* v) {
      double fl[N] = {};
      if (cs < nvalid) ld<N, 1>(fb + cs * G::N3 + k * G::N2 + j * N, fl);
      double r[N];
#pragma unroll
      for (int e = 0; e < N; ++e) r[e] = (cs < nvalid) ? fl[e] - v[e] : 0.0;
      st<N, 1>(R + cs * G::CS + k * G::ZS + j * G::YS, r);
    };
    // d = f - A u: nodal form at n <= 6 (n = 7, 8: the Gauss-point passes measured faster)
    if constexpr (DG_NODAL_APPLY && N <= 6) apply_nodal<N, G::NT, true>(kq, g, P, SA, SB, FB, defect);
    else cell_operator<N, true, false, false, G::NT>(kq, g, P, SA, SB, FB, true, defect);
    __syncthreads();
    // D_T uses self faces only
    for (int it = tid; it < C * 6; it += G::NT) g.nb[it / 6][it % 6] = nullptr;
  }
  diag_setup<N, G::NT>(kp, g, Dg);
  __syncthreads();
  // Each thread owns one x-line of the group (LINES <= NT): the operator's first pass reads that
  // line of p and its last pass produces that line of q = D_T p, so r, p, x and diag(D_T)^-1 stay
  // in registers; only the per-cell scalars go through shared memory (reductions, alpha, beta).
  static_assert(G::LINES <= G::NT, "one line per thread");
  const bool own = tid < G::LINES;
  const int lcs = own ? tid / G::N2 : 0, ll = tid % G::N2;
  const int loff = lcs * G::CS + (ll / N) * G::ZS + (ll % N) * G::YS;
  double r[N], p[N], x[N], dgi[N];
#pragma unroll
  for (int e = 0; e < N; ++e) r[e] = p[e] = x[e] = dgi[e] = 0.0;
  {  // r0 = d, p = M^-1 r, x = 0
    double rr = 0.0, rz = 0.0;
    if (own) {
      ld<N, 1>(R + loff, r);
      ld<N, 1>(Dg + loff, dgi);
#pragma unroll
      for (int e = 0; e < N; ++e) { p[e] = r[e] * dgi[e]; rr = fma(r[e], r[e], rr); rz = fma(r[e], p[e], rz); }
      g.red[0][tid] = rr;
      g.red[1][tid] = rz;
    }
  }
  __syncthreads();
  if (tid < C) {
    const double rr0 = cell_sum<N>(g, 0, tid);
    g.sc[S_RR0][tid] = rr0;
    g.sc[S_RZ][tid] = cell_sum<N>(g, 1, tid);
    g.conv[tid] = (tid >= nvalid) || (rr0 == 0.0) || skip_cell(kp, cell0 + tid);
    g.its[tid] = 0;
  }
  for (int iter = 0;; ++iter) {
    const int done = __syncthreads_and(tid >= C || g.conv[tid]);
    if (done || iter >= kp.max_it) break;
    // q = D_T p (the thread's own line, in registers)
    double q[N];
#pragma unroll
    for (int e = 0; e < N; ++e) q[e] = 0.0;
    if constexpr (NODAL) {
      dt_nodal<N, false, DG_NODAL_FLY, true>(g, SA, SB, p, q, &kq);
    } else {
      cell_operator<N, false, true, false, G::NT>(kq, g, P, SA, SB, FB, true, [&](int, int, int, const double* v) {
#pragma unroll
        for (int e = 0; e < N; ++e) q[e] = v[e];
      }, p);
    }
    if (own) {
      double sp = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) sp = fma(p[e], q[e], sp);
      g.red[0][tid] = sp;
    }
    __syncthreads();
    if (tid < C) {
      const double pq = cell_sum<N>(g, 0, tid);
      double alpha = 0.0;
      if (!g.conv[tid]) {
        if (pq > 0.0) alpha = g.sc[S_RZ][tid] / pq;
        else g.conv[tid] = 2;  // breakdown (D_T not SPD): keep the last iterate, not converged
      }
      g.sc[S_ALPHA][tid] = alpha;
    }
    __syncthreads();
    double z[N];
    {
      const double alpha = g.sc[S_ALPHA][lcs];
      double rr = 0.0, rz = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) {
        x[e] = fma(alpha, p[e], x[e]);
        r[e] = fma(-alpha, q[e], r[e]);
        rr = fma(r[e], r[e], rr);
        z[e] = r[e] * dgi[e];
        rz = fma(r[e], z[e], rz);
      }
      if (own) {
        g.red[0][tid] = rr;
        g.red[1][tid] = rz;
      }
    }
    __syncthreads();
    if (tid < C && !g.conv[tid]) {
      const double rr = cell_sum<N>(g, 0, tid), rzn = cell_sum<N>(g, 1, tid);
      g.its[tid] += 1;
      if (rr <= kp.tol2 * g.sc[S_RR0][tid]) g.conv[tid] = 1;
      g.sc[S_BETA][tid] = rzn / g.sc[S_RZ][tid];
      g.sc[S_RZ][tid] = rzn;
    }
    __syncthreads();
    if (!g.conv[lcs]) {
      const double beta = g.sc[S_BETA][lcs];
#pragma unroll
      for (int e = 0; e < N; ++e) p[e] = fma(beta, p[e], z[e]);
    }
  }
  if (own) st<N, 1>(X + loff, x);
  __syncthreads();
  // write result (u + omega du for a sweep, du for a solve)
  const double* ib = in + (size_t)cell0 * G::N3;
  double* ob = out + (size_t)cell0 * G::N3;
  DG_FOR_XLINES({
    if (cs < nvalid) {
      const int j = l_ % N, k = l_ / N;
      double x[N];
      ld<N, 1>(X + off, x);
      if (SWEEP) {
        double uu[N];
        ld<N, 1>(ib + cs * G::N3 + k * G::N2 + j * N, uu);
#pragma unroll
        for (int e = 0; e < N; ++e) x[e] = fma(kp.omega, x[e], uu[e]);
      }
      st<N, 1>(ob + cs * G::N3 + k * G::N2 + j * N, x);
    }
  })
  if (tid < nvalid) kp.its[cell0 + tid] = g.conv[tid] == 1 ? g.its[tid] : (g.its[tid] | (1 << 30));
}

// Jacobi-preconditioned CG with one warp per cell (n = 5: 25 lanes hold the cell's lines).
// The group setup and the defect are CTA-wide; the iterations are warp-local (the operator in
// WARP mode, shuffle reductions, per-lane copies of the cell's scalars), so no CTA barrier is
// left in the loop and each warp leaves it when its own cell has converged.
// a / b as a * (1 / b) from rcp.approx + two Newton steps (~1 ulp), for Krylov scalars
__device__ __forceinline__ double quot_nr(double a, double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  double e = fma(-b, y, 1.0);
  y = fma(y, e, y);
  e = fma(-b, y, 1.0);
  return a * fma(y, e, y);
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// CC: cells (warps) per CTA. A CTA holds its registers until its slowest cell has converged, so
// with CC = 8 the warp slots of the early finishers idle (local iterations vary +-12 %, up to 1.8x
// the mean); CC = 1 releases each cell's slot as soon as that cell is done.
template <int N, bool SWEEP, bool GEN = true, int CC = Cells<N>::C>
__global__ void __launch_bounds__(Geo<N, CC>::NTW, (CC > 1 ? 2 : 0))
k_cg_w(KParams kp, const double* __restrict__ in, const double* __restrict__ f,
       double* __restrict__ out) {
  using G = Geo<N, CC>;
  constexpr int C = G::C;
  extern __shared__ double sm[];
  __shared__ Group<N, CC> g;
  double* X = sm;
  double* R = X + G::TENSOR;
  double* P = R + G::TENSOR;
  double* Q = P + G::TENSOR;
  double* Dg = Q + G::TENSOR;
  double* SA = Dg + G::TENSOR;
  double* SB = SA + G::TENSOR;
  double* FB = fb_alias<N, CC>() ? Q : SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(C, kp.ncells - cell0);
  const int tid = threadIdx.x;
  load_tile<N, G::NTW>(g, cell0, kp.ncells, in, SWEEP ? P : R);
  const KParams& kq = kp;   // launched with mask = 7 (launch_local_solve / launch_sweep)
  group_setup<N, G::NTW>(kq, g, cell0, SWEEP ? in : nullptr);
  constexpr int LPL0 = (G::N2 + 31) / 32;
  constexpr bool NODAL = DG_NODAL_DT && LPL0 == 1;   // D_T in the nodal Kronecker-sum form
  if constexpr (NODAL) nodal_face_ops<N, G::NTW>(kq, g);
  else self_face_ops<N, G::NTW>(kq, g);
  if (SWEEP) {  // d = f - A u  (Alg. 2 line 2), CTA-wide
    const double* fb = f + (size_t)cell0 * G::N3;
    auto defect = [&](int cs, int j, int k, const double* v) {
      double fl[N] = {};
      if (cs < nvalid) ld<N, 1>(fb + cs * G::N3 + k * G::N2 + j * N, fl);
      double r[N];
#pragma unroll
      for (int e = 0; e < N; ++e) r[e] = (cs < nvalid) ? fl[e] - v[e] : 0.0;
      st<N, 1>(R + cs * G::CS + k * G::ZS + j * G::YS, r);
    };
    if constexpr (DG_NODAL_APPLY && G::LINES <= G::NTW) apply_nodal<N, G::NTW, GEN>(kq, g, P, SA, SB, FB, defect);
    else cell_operator<N, true, false, false, G::NTW, GEN>(kq, g, P, SA, SB, FB, true, defect);
    __syncthreads();
    for (int it = tid; it < C * 6; it += G::NTW) g.nb[it / 6][it % 6] = nullptr;
  }
  diag_setup<N, G::NTW>(kp, g, Dg);
  __syncthreads();
  // from here on: warp w owns cell slot cs = w; lane l holds the x-lines l, l + 32, ... < n^2
  constexpr int LPL = (G::N2 + 31) / 32;   // lines per lane
  const int cs = tid >> 5, lane = tid & 31;
  int off[LPL];
  bool act[LPL];
#pragma unroll
  for (int m = 0; m < LPL; ++m) {
    const int l = lane + 32 * m;
    act[m] = l < G::N2;
    off[m] = cs * G::CS + (l / N) * G::ZS + (l % N) * G::YS;
  }
  double rr = 0.0, rz = 0.0;
#pragma unroll
  for (int m = 0; m < LPL; ++m)
    if (act[m]) {
      double r[N], dg[N], z[N], zero[N] = {};
      ld<N, 1>(R + off[m], r);
      ld<N, 1>(Dg + off[m], dg);
#pragma unroll
      for (int e = 0; e < N; ++e) { z[e] = r[e] * dg[e]; rr = fma(r[e], r[e], rr); rz = fma(r[e], z[e], rz); }
      st<N, 1>(P + off[m], z);
      st<N, 1>(X + off[m], zero);
    }
  const double rr0 = warp_sum(rr);
  rz = warp_sum(rz);
  bool conv = cs >= nvalid || rr0 == 0.0 || skip_cell(kp, cell0 + cs);
  int its = 0;
  if constexpr (LPL == 1) {
    // one line per lane (n = 5): every Krylov vector of the cell is lane-private line by line
    // (the operator's pass 1 reads the lane's own x-line of p, pass 7 produces the lane's own
    // line of q = D_T p), so r, p, x and diag(D_T)^-1 stay in registers and the iterations touch
    // shared memory only through the operator's transposes
    double r[N], p[N], x[N], dgi[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = p[e] = x[e] = dgi[e] = 0.0;
    if (act[0]) {
      ld<N, 1>(R + off[0], r);
      ld<N, 1>(P + off[0], p);
      ld<N, 1>(Dg + off[0], dgi);
    }
    for (int iter = 0; !conv && iter < kp.max_it; ++iter) {   // conv is warp-uniform
      __syncwarp();
      double q[N];
#pragma unroll
      for (int e = 0; e < N; ++e) q[e] = 0.0;
      if constexpr (NODAL) {
        dt_nodal<N, true, DG_NODAL_FLY, GEN>(g, SA, SB, p, q, &kq);
      } else {
        cell_operator<N, false, true, true, G::NT, GEN>(kq, g, P, SA, SB, FB, true,
                                                             [&](int, int, int, const double* v) {
#pragma unroll
          for (int e = 0; e < N; ++e) q[e] = v[e];
        }, p);
      }
      double pq = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) pq = fma(p[e], q[e], pq);
      pq = warp_sum(pq);
      if (!(pq > 0.0)) break;   // breakdown (D_T not SPD): keep the last iterate, not converged
      const double alpha = quot_nr(rz, pq);
      double r2 = 0.0, rzn = 0.0, z[N];
#pragma unroll
      for (int e = 0; e < N; ++e) {
        x[e] = fma(alpha, p[e], x[e]);
        r[e] = fma(-alpha, q[e], r[e]);
        r2 = fma(r[e], r[e], r2);
        z[e] = dgi[e] * r[e];   // z = M^-1 r
        rzn = fma(r[e], z[e], rzn);
      }
      r2 = warp_sum(r2);
      rzn = warp_sum(rzn);
      ++its;
      if (r2 <= kp.tol2 * rr0) {
        conv = true;
        break;
      }
      const double beta = quot_nr(rzn, rz);
      rz = rzn;
#pragma unroll
      for (int e = 0; e < N; ++e) p[e] = fma(beta, p[e], z[e]);
    }
    if (act[0]) st<N, 1>(X + off[0], x);
  } else {
  for (int iter = 0; !conv && iter < kp.max_it; ++iter) {   // conv is warp-uniform
    __syncwarp();
    cell_operator<N, false, true, true, G::NT, GEN>(kq, g, P, SA, SB, FB, true, [&](int c, int j, int k, const double* v) {
      st<N, 1>(Q + c * G::CS + k * G::ZS + j * G::YS, v);
    });
    __syncwarp();
    double pq = 0.0;
    double p[LPL][N], q[LPL][N], dg[LPL][N];
#pragma unroll
    for (int m = 0; m < LPL; ++m)
      if (act[m]) {
        ld<N, 1>(P + off[m], p[m]);
        ld<N, 1>(Q + off[m], q[m]);
#pragma unroll
        for (int e = 0; e < N; ++e) pq = fma(p[m][e], q[m][e], pq);
      }
    pq = warp_sum(pq);
    if (!(pq > 0.0)) {   // breakdown (D_T not SPD): keep the last iterate, not converged
      break;
    }
    const double alpha = quot_nr(rz, pq);
    double r2 = 0.0, rzn = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m)
      if (act[m]) {
        double x[N], r[N];
        ld<N, 1>(X + off[m], x);
        ld<N, 1>(R + off[m], r);
        ld<N, 1>(Dg + off[m], dg[m]);
#pragma unroll
        for (int e = 0; e < N; ++e) {
          x[e] = fma(alpha, p[m][e], x[e]);
          r[e] = fma(-alpha, q[m][e], r[e]);
          r2 = fma(r[e], r[e], r2);
          dg[m][e] *= r[e];   // z = M^-1 r
          rzn = fma(r[e], dg[m][e], rzn);
        }
        st<N, 1>(X + off[m], x);
        st<N, 1>(R + off[m], r);
      }
    r2 = warp_sum(r2);
    rzn = warp_sum(rzn);
    ++its;
    if (r2 <= kp.tol2 * rr0) {
      conv = true;
      break;
    }
    const double beta = quot_nr(rzn, rz);
    rz = rzn;
#pragma unroll
    for (int m = 0; m < LPL; ++m)
      if (act[m]) {
#pragma unroll
        for (int e = 0; e < N; ++e) p[m][e] = fma(beta, p[m][e], dg[m][e]);
        st<N, 1>(P + off[m], p[m]);
      }
  }
  }
  __syncwarp();
  // write result (u + omega du for a sweep, du for a solve), warp by warp
#pragma unroll
  for (int m = 0; m < LPL; ++m)
    if (act[m] && cs < nvalid) {
      const int l = lane + 32 * m, j = l % N, k = l / N;
      double x[N];
      ld<N, 1>(X + off[m], x);
      if (SWEEP) {
        double uu[N];
        ld<N, 1>(in + (size_t)(cell0 + cs) * G::N3 + k * G::N2 + j * N, uu);
#pragma unroll
        for (int e = 0; e < N; ++e) x[e] = fma(kp.omega, x[e], uu[e]);
      }
      st<N, 1>(out + (size_t)(cell0 + cs) * G::N3 + k * G::N2 + j * N, x);
    }
  if (lane == 0 && cs < nvalid) kp.its[cell0 + cs] = conv ? its : (its | (1 << 30));
}

// Jacobi right-preconditioned BiCGStab with one warp per cell (n = 5), the same scheme as k_cg_w:
// CTA-wide setup and defect, warp-local iterations without CTA barriers.
template <int N, bool SWEEP, int CC = Cells<N>::C>
__global__ void __launch_bounds__(Geo<N, CC>::NTW, (CC == Cells<N>::C ? 2 : 0))
k_bicgstab_w(KParams kp, const double* __restrict__ in, const double* __restrict__ f,
             double* __restrict__ out) {
  using G = Geo<N, CC>;
  constexpr int C = G::C;
  extern __shared__ double sm[];
  __shared__ Group<N, CC> g;
  double* X = sm;
  double* R = X + G::TENSOR;
  double* RH = R + G::TENSOR;
  double* P = RH + G::TENSOR;
  double* V = P + G::TENSOR;
  double* PS = V + G::TENSOR;
  double* T = PS + G::TENSOR;
  double* Dg = T + G::TENSOR;
  double* SA = Dg + G::TENSOR;
  double* SB = SA + G::TENSOR;
  double* FB = fb_alias<N, CC>() ? T : SB + G::TENSOR;
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(C, kp.ncells - cell0);
  const int tid = threadIdx.x;
  load_tile<N, G::NTW>(g, cell0, kp.ncells, in, SWEEP ? P : R);
  const KParams& kq = kp;   // launched with mask = 7 (launch_local_solve / launch_sweep)
  group_setup<N, G::NTW>(kq, g, cell0, SWEEP ? in : nullptr);
  constexpr bool NODAL = DG_NODAL_DT && G::N2 <= 32;   // one line per lane: D_T in the nodal form
  if constexpr (NODAL) nodal_face_ops<N, G::NTW>(kq, g);
  else self_face_ops<N, G::NTW>(kq, g);
  if (SWEEP) {
    const double* fb = f + (size_t)cell0 * G::N3;
    auto defect = [&](int cs, int j, int k, const double* v) {
      double fl[N] = {};
      if (cs < nvalid) ld<N, 1>(fb + cs * G::N3 + k * G::N2 + j * N, fl);
      double r[N];
#pragma unroll
      for (int e = 0; e < N; ++e) r[e] = (cs < nvalid) ? fl[e] - v[e] : 0.0;
      st<N, 1>(R + cs * G::CS + k * G::ZS + j * G::YS, r);
    };
    if constexpr (DG_NODAL_APPLY && G::LINES <= G::NTW) apply_nodal<N, G::NTW, true>(kq, g, P, SA, SB, FB, defect);
    else cell_operator<N, true, false, false, G::NTW>(kq, g, P, SA, SB, FB, true, defect);
    __syncthreads();
    for (int it = tid; it < C * 6; it += G::NTW) g.nb[it / 6][it % 6] = nullptr;
  }
  diag_setup<N, G::NTW>(kp, g, Dg);
  __syncthreads();
  constexpr int LPL = (G::N2 + 31) / 32;   // x-lines per lane
  const int cs = tid >> 5, lane = tid & 31;
  int offs[LPL];
  bool acts[LPL];
#pragma unroll
  for (int m = 0; m < LPL; ++m) {
    const int l = lane + 32 * m;
    acts[m] = l < G::N2;
    offs[m] = cs * G::CS + (l / N) * G::ZS + (l % N) * G::YS;
  }
  auto op = [&](double* dst) {   // dst = D_T PS on this warp's cell
    __syncwarp();
    if constexpr (NODAL) {
      dt_nodal_smem<N, true>(g, SA, SB, PS, dst);
    } else {
      cell_operator<N, false, true, true, G::NT>(kq, g, PS, SA, SB, FB, true, [&](int c, int j, int k, const double* v) {
        st<N, 1>(dst + c * G::CS + k * G::ZS + j * G::YS, v);
      });
    }
    __syncwarp();
  };
  double rr = 0.0;
#pragma unroll
  for (int m = 0; m < LPL; ++m) if (acts[m]) {
    const int off = offs[m];
    double r[N], zero[N] = {};
    ld<N, 1>(R + off, r);
#pragma unroll
    for (int e = 0; e < N; ++e) rr = fma(r[e], r[e], rr);
    st<N, 1>(RH + off, r);
    st<N, 1>(X + off, zero);
    st<N, 1>(P + off, zero);
    st<N, 1>(V + off, zero);
  }
  const double rr0 = warp_sum(rr);
  bool conv = cs >= nvalid || rr0 == 0.0 || skip_cell(kp, cell0 + cs);
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  bool rst = false;
  int its = 0;
  for (int iter = 0; !conv && iter < kp.max_it; ++iter) {   // conv is warp-uniform
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double r[N], rh[N];
      ld<N, 1>(R + off, r);
      ld<N, 1>(RH + off, rh);
#pragma unroll
      for (int e = 0; e < N; ++e) { a = fma(rh[e], r[e], a); b = fma(r[e], r[e], b); }
    }
    double rhon = warp_sum(a);
    const double r2 = warp_sum(b);
    if (fabs(rhon) <= 1e-24 * r2) rst = true;   // breakdown: restart with rh = r
    if (rst) rhon = r2;
    const double beta = rst ? 0.0 : quot_nr(rhon * alpha, rho * omega);
    // p = r + beta (p - omega v); ps = M^-1 p
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double r[N], p[N], v[N], dg[N], ps[N];
      ld<N, 1>(R + off, r);
      ld<N, 1>(P + off, p);
      ld<N, 1>(V + off, v);
      ld<N, 1>(Dg + off, dg);
#pragma unroll
      for (int e = 0; e < N; ++e) {
        p[e] = rst ? r[e] : fma(beta, fma(-omega, v[e], p[e]), r[e]);
        ps[e] = p[e] * dg[e];
      }
      if (rst) st<N, 1>(RH + off, r);
      st<N, 1>(P + off, p);
      st<N, 1>(PS + off, ps);
    }
    rst = false;
    op(V);
    double rvl = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double rh[N], v[N];
      ld<N, 1>(RH + off, rh);
      ld<N, 1>(V + off, v);
#pragma unroll
      for (int e = 0; e < N; ++e) rvl = fma(rh[e], v[e], rvl);
    }
    const double rv = warp_sum(rvl);
    alpha = 0.0;
    if (rv != 0.0) alpha = quot_nr(rhon, rv);
    else rst = true;
    // x += alpha ps; s = r - alpha v (in R); ps <- M^-1 s
    double ss = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double x[N], r[N], v[N], ps[N], dg[N];
      ld<N, 1>(X + off, x);
      ld<N, 1>(R + off, r);
      ld<N, 1>(V + off, v);
      ld<N, 1>(PS + off, ps);
      ld<N, 1>(Dg + off, dg);
#pragma unroll
      for (int e = 0; e < N; ++e) {
        x[e] = fma(alpha, ps[e], x[e]);
        r[e] = fma(-alpha, v[e], r[e]);
        ss = fma(r[e], r[e], ss);
        ps[e] = r[e] * dg[e];
      }
      st<N, 1>(X + off, x);
      st<N, 1>(R + off, r);
      st<N, 1>(PS + off, ps);
    }
    ss = warp_sum(ss);
    if (ss <= kp.tol2 * rr0) {
      ++its;
      conv = true;
      break;
    }
    op(T);
    double tsl = 0.0, ttl = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double t[N], sv[N];
      ld<N, 1>(T + off, t);
      ld<N, 1>(R + off, sv);
#pragma unroll
      for (int e = 0; e < N; ++e) { tsl = fma(t[e], sv[e], tsl); ttl = fma(t[e], t[e], ttl); }
    }
    const double ts = warp_sum(tsl), tt = warp_sum(ttl);
    const double om = tt > 0.0 ? quot_nr(ts, tt) : 0.0;
    if (om == 0.0) rst = true;
    // x += omega s^; r = s - omega t
    double r2n = 0.0;
#pragma unroll
    for (int m = 0; m < LPL; ++m) if (acts[m]) {
      const int off = offs[m];
      double x[N], r[N], t[N], ps[N];
      ld<N, 1>(X + off, x);
      ld<N, 1>(R + off, r);
      ld<N, 1>(T + off, t);
      ld<N, 1>(PS + off, ps);
#pragma unroll
      for (int e = 0; e < N; ++e) {
        x[e] = fma(om, ps[e], x[e]);
        r[e] = fma(-om, t[e], r[e]);
        r2n = fma(r[e], r[e], r2n);
      }
      st<N, 1>(X + off, x);
      st<N, 1>(R + off, r);
    }
    r2n = warp_sum(r2n);
    ++its;
    if (r2n <= kp.tol2 * rr0) conv = true;
    rho = rhon;
    omega = om == 0.0 ? 1.0 : om;
  }
  __syncwarp();
#pragma unroll
  for (int m = 0; m < LPL; ++m) if (acts[m] && cs < nvalid) {
    const int off = offs[m], l = lane + 32 * m, j = l % N, k = l / N;
    double x[N];
    ld<N, 1>(X + off, x);
    if (SWEEP) {
      double uu[N];
      ld<N, 1>(in + (size_t)(cell0 + cs) * G::N3 + k * G::N2 + j * N, uu);
#pragma unroll
      for (int e = 0; e < N; ++e) x[e] = fma(kp.omega, x[e], uu[e]);
    }
    st<N, 1>(out + (size_t)(cell0 + cs) * G::N3 + k * G::N2 + j * N, x);
  }
  if (lane == 0 && cs < nvalid) kp.its[cell0 + cs] = conv ? its : (its | (1 << 30));
}

// Jacobi right-preconditioned BiCGStab per cell (nonsymmetric blocks, b != 0).
template <int N, bool SWEEP, int CC = Cells<N>::C>
__global__ void __launch_bounds__(Geo<N, CC>::NT, (CC == Cells<N>::C ? 2 : 0))   // two CTAs per SM (n = 7: <= 146 registers)
k_bicgstab(KParams kp, const double* __restrict__ in, const double* __restrict__ f,
           double* __restrict__ out) {
  using G = Geo<N, CC>;
  constexpr int C = G::C;
  extern __shared__ double sm[];
  __shared__ Group<N, CC> g;
  double* X = sm;
  double* R = X + G::TENSOR;
  double* RH = R + G::TENSOR;
  double* P = RH + G::TENSOR;
  double* V = P + G::TENSOR;
  double* PS = V + G::TENSOR;
  double* T = PS + G::TENSOR;
  double* Dg = T + G::TENSOR;
  double* SA = Dg + G::TENSOR;
  double* SB = SA + G::TENSOR;
  double* FB = fb_alias<N, CC>() ? T : SB + G::TENSOR;   // defect only: aliases T and Dg when it fits
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(C, kp.ncells - cell0);
  const int tid = threadIdx.x;
  load_tile<N, G::NT>(g, cell0, kp.ncells, in, SWEEP ? P : R);
  const KParams& kq = kp;   // launched with mask = 7 (launch_local_solve / launch_sweep)
  group_setup<N, G::NT>(kq, g, cell0, SWEEP ? in : nullptr);
  constexpr bool NODAL = DG_NODAL_DT;   // D_T of the iterations in the nodal form
  if constexpr (NODAL) nodal_face_ops<N, G::NT>(kq, g);
  else self_face_ops<N, G::NT>(kq, g);   // D_T in the loop: self faces at the Gauss points
  if (SWEEP) {
    const double* fb = f + (size_t)cell0 * G::N3;
    auto defect = [&](int cs, int j, int k, const double* v) {
      double fl[N] = {};
      if (cs < nvalid) ld<N, 1>(fb + cs * G::N3 + k * G::N2 + j * N, fl);
      double r[N];
#pragma unroll
      for (int e = 0; e < N; ++e) r[e] = (cs < nvalid) ? fl[e] - v[e] : 0.0;
      st<N, 1>(R + cs * G::CS + k * G::ZS + j * G::YS, r);
    };
    // d = f - A u: nodal form at n <= 6 (n = 7, 8: the Gauss-point passes measured faster)
    if constexpr (DG_NODAL_APPLY && N <= 6) apply_nodal<N, G::NT, true>(kq, g, P, SA, SB, FB, defect);
    else cell_operator<N, true, false, false, G::NT>(kq, g, P, SA, SB, FB, true, defect);
    __syncthreads();
    for (int it = tid; it < C * 6; it += G::NT) g.nb[it / 6][it % 6] = nullptr;
  }
  diag_setup<N, G::NT>(kp, g, Dg);
  __syncthreads();
  DG_FOR_XLINES({
    double r[N], zero[N] = {};
    ld<N, 1>(R + off, r);
    double rr = 0.0;
#pragma unroll
    for (int e = 0; e < N; ++e) rr = fma(r[e], r[e], rr);
    st<N, 1>(RH + off, r);
    st<N, 1>(X + off, zero);
    st<N, 1>(P + off, zero);
    st<N, 1>(V + off, zero);
    g.red[0][it] = rr;
  })
  __syncthreads();
  if (tid < C) {
    const double rr0 = cell_sum<N>(g, 0, tid);
    g.sc[S_RR0][tid] = rr0;
    g.sc[S_RHO][tid] = 1.0;
    g.sc[S_ALPHA][tid] = 1.0;
    g.sc[S_OMEGA][tid] = 1.0;
    g.conv[tid] = (tid >= nvalid) || (rr0 == 0.0) || skip_cell(kp, cell0 + tid);
    g.its[tid] = 0;
    g.rst[tid] = 0;
  }
  for (int iter = 0;; ++iter) {
    const int done = __syncthreads_and(tid >= C || g.conv[tid]);
    if (done || iter >= kp.max_it) break;
    // rho_new = <rh, r>, rr = <r, r>
    DG_FOR_XLINES({
      double r[N], rh[N];
      ld<N, 1>(R + off, r);
      ld<N, 1>(RH + off, rh);
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) { a = fma(rh[e], r[e], a); b = fma(r[e], r[e], b); }
      g.red[0][it] = a;
      g.red[1][it] = b;
    })
    __syncthreads();
    if (tid < C && !g.conv[tid]) {
      double rhon = cell_sum<N>(g, 0, tid);
      const double rr = cell_sum<N>(g, 1, tid);
      int rst = g.rst[tid];
      if (fabs(rhon) <= 1e-24 * rr) rst = 1;  // breakdown: restart with rh = r
      if (rst) rhon = rr;
      g.rst[tid] = rst;
      g.sc[S_BETA][tid] = rst ? 0.0 : (rhon / g.sc[S_RHO][tid]) * (g.sc[S_ALPHA][tid] / g.sc[S_OMEGA][tid]);
      g.sc[S_RHON][tid] = rhon;
    }
    __syncthreads();
    // p = r + beta (p - omega v); ps = M^-1 p
    DG_FOR_XLINES({
      if (!g.conv[cs]) {
        const double beta = g.sc[S_BETA][cs], om = g.sc[S_OMEGA][cs];
        const int rst = g.rst[cs];
        double r[N], p[N], v[N], dg[N], ps[N];
        ld<N, 1>(R + off, r);
        ld<N, 1>(P + off, p);
        ld<N, 1>(V + off, v);
        ld<N, 1>(Dg + off, dg);
#pragma unroll
        for (int e = 0; e < N; ++e) {
          p[e] = rst ? r[e] : fma(beta, fma(-om, v[e], p[e]), r[e]);
          ps[e] = p[e] * dg[e];
        }
        if (rst) st<N, 1>(RH + off, r);
        st<N, 1>(P + off, p);
        st<N, 1>(PS + off, ps);
      }
    })
    __syncthreads();
    if constexpr (NODAL) {
      dt_nodal_smem<N, false>(g, SA, SB, PS, V);
    } else {
      cell_operator<N, false, true, false, G::NT>(kq, g, PS, SA, SB, FB, true, [&](int cs, int j, int k, const double* v) {
        st<N, 1>(V + cs * G::CS + k * G::ZS + j * G::YS, v);
      });
    }
    __syncthreads();
    DG_FOR_XLINES({
      double rh[N], v[N];
      ld<N, 1>(RH + off, rh);
      ld<N, 1>(V + off, v);
      double a = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) a = fma(rh[e], v[e], a);
      g.red[0][it] = a;
    })
    __syncthreads();
    if (tid < C) {
      g.rst[tid] = 0;
      double alpha = 0.0;
      if (!g.conv[tid]) {
        const double rv = cell_sum<N>(g, 0, tid);
        if (rv != 0.0) alpha = g.sc[S_RHON][tid] / rv;
        else g.rst[tid] = 1;
      }
      g.sc[S_ALPHA][tid] = alpha;
    }
    __syncthreads();
    // x += alpha ps; s = r - alpha v (stored in R); ps <- M^-1 s
    DG_FOR_XLINES({
      if (!g.conv[cs]) {
        const double alpha = g.sc[S_ALPHA][cs];
        double x[N], r[N], v[N], ps[N], dg[N];
        ld<N, 1>(X + off, x);
        ld<N, 1>(R + off, r);
        ld<N, 1>(V + off, v);
        ld<N, 1>(PS + off, ps);
        ld<N, 1>(Dg + off, dg);
        double ss = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) {
          x[e] = fma(alpha, ps[e], x[e]);
          r[e] = fma(-alpha, v[e], r[e]);
          ss = fma(r[e], r[e], ss);
          ps[e] = r[e] * dg[e];
        }
        st<N, 1>(X + off, x);
        st<N, 1>(R + off, r);
        st<N, 1>(PS + off, ps);
        g.red[0][it] = ss;
      } else {
        g.red[0][it] = 0.0;
      }
    })
    __syncthreads();
    if (tid < C && !g.conv[tid]) {
      const double ss = cell_sum<N>(g, 0, tid);
      if (ss <= kp.tol2 * g.sc[S_RR0][tid]) { g.conv[tid] = 1; g.its[tid] += 1; }
    }
    __syncthreads();
    if constexpr (NODAL) {
      dt_nodal_smem<N, false>(g, SA, SB, PS, T);
    } else {
      cell_operator<N, false, true, false, G::NT>(kq, g, PS, SA, SB, FB, true, [&](int cs, int j, int k, const double* v) {
        st<N, 1>(T + cs * G::CS + k * G::ZS + j * G::YS, v);
      });
    }
    __syncthreads();
    DG_FOR_XLINES({
      double t[N], s[N];
      ld<N, 1>(T + off, t);
      ld<N, 1>(R + off, s);
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int e = 0; e < N; ++e) { a = fma(t[e], s[e], a); b = fma(t[e], t[e], b); }
      g.red[0][it] = a;
      g.red[1][it] = b;
    })
    __syncthreads();
    if (tid < C && !g.conv[tid]) {
      const double ts = cell_sum<N>(g, 0, tid), tt = cell_sum<N>(g, 1, tid);
      const double om = tt > 0.0 ? ts / tt : 0.0;
      g.sc[S_OMEGA][tid] = om;
      if (om == 0.0) g.rst[tid] = 1;
    }
    __syncthreads();
    // x += omega s^; r = s - omega t
    DG_FOR_XLINES({
      if (!g.conv[cs]) {
        const double om = g.sc[S_OMEGA][cs];
        double x[N], r[N], t[N], ps[N];
        ld<N, 1>(X + off, x);
        ld<N, 1>(R + off, r);
        ld<N, 1>(T + off, t);
        ld<N, 1>(PS + off, ps);
        double rr = 0.0;
#pragma unroll
        for (int e = 0; e < N; ++e) {
          x[e] = fma(om, ps[e], x[e]);
          r[e] = fma(-om, t[e], r[e]);
          rr = fma(r[e], r[e], rr);
        }
        st<N, 1>(X + off, x);
        st<N, 1>(R + off, r);
        g.red[0][it] = rr;
      } else {
        g.red[0][it] = 0.0;
      }
    })
    __syncthreads();
    if (tid < C && !g.conv[tid]) {
      const double rr = cell_sum<N>(g, 0, tid);
      g.its[tid] += 1;
      if (rr <= kp.tol2 * g.sc[S_RR0][tid]) g.conv[tid] = 1;
      g.sc[S_RHO][tid] = g.sc[S_RHON][tid];
      if (g.sc[S_OMEGA][tid] == 0.0) { g.sc[S_OMEGA][tid] = 1.0; }
    }
  }
  const double* ib = in + (size_t)cell0 * G::N3;
  double* ob = out + (size_t)cell0 * G::N3;
  DG_FOR_XLINES({
    if (cs < nvalid) {
      const int j = l_ % N, k = l_ / N;
      double x[N];
      ld<N, 1>(X + off, x);
      if (SWEEP) {
        double uu[N];
        ld<N, 1>(ib + cs * G::N3 + k * G::N2 + j * N, uu);
#pragma unroll
        for (int e = 0; e < N; ++e) x[e] = fma(kp.omega, x[e], uu[e]);
      }
      st<N, 1>(ob + cs * G::N3 + k * G::N2 + j * N, x);
    }
  })
  if (tid < nvalid) kp.its[cell0 + tid] = g.conv[tid] ? g.its[tid] : (g.its[tid] | (1 << 30));
}

}  // namespace

#include "dg_plane.cuh"

namespace {

// ---- host-side launch helpers ------------------------------------------------------
template <int N> constexpr size_t smem_bytes(int tensors) {
  return sizeof(double) * ((size_t)tensors * Geo<N>::TENSOR + Geo<N>::FACE);
}

// Dynamic shared memory limit + the maximum shared-memory carveout (the kernels are sized by
// shared memory per resident cell; a smaller carveout would cap the resident CTAs per SM).
template <class K> cudaError_t set_smem(K kernel, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                              (int)cudaSharedmemCarveoutMaxShared);
}

template <class K>
cudaError_t launch(K kernel, int grid, int block, size_t smem, cudaStream_t s, const KParams& kp,
                   const double* a, const double* b, double* c) {
  if (grid <= 0) return cudaSuccess;   // an empty split launch (no interior / boundary groups)
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  kernel<<<grid, block, smem, s>>>(kp, a, b, c);
  return cudaGetLastError();
}

// Kernel variants (KParams::variant, dg_set_kernel_variant; defaults are the measured winners):
// VAR_NO_TMEM: shared-memory n = 4 BiCGStab instead of Krylov vectors in tensor memory;
// VAR_LINE: the line-per-thread kernels for every degree.
inline bool use_tmem(const KParams& kp) { return (kp.variant & VAR_NO_TMEM) == 0; }
inline bool force_line(const KParams& kp) { return (kp.variant & VAR_LINE) != 0; }

// Kernel family of the operator application per degree, chosen by measurement on C1-C5
// (profiles/r01_kernel_family.md, profiles/r01_ab.md): the plane kernels for n = 2, 3, 4;
// at n = 5 the line kernels' higher occupancy wins for A u and D_T u (the volume-only hook uses
// the persistent plane kernel k_volume for every n <= 5). The local solvers always use the plane
// kernels for n <= 5 (register-resident Krylov vectors).
#ifndef DG_PLANE_APPLY3
#define DG_PLANE_APPLY3 1   // n = 3: plane kernels (C5: D_T 832 -> 351 us, A 900 -> 847 us)
#endif
#ifndef DG_PLANE_APPLY5
#define DG_PLANE_APPLY5 0
#endif
template <int N> constexpr bool plane_apply() {
  return N == 2 || N == 4 || (N == 3 && DG_PLANE_APPLY3) || (N == 5 && DG_PLANE_APPLY5);
}

// convective or reaction terms present (else the pure-diffusion instantiations, GEN = false)
inline bool gen_terms(const KParams& kp) {
  return kp.c != nullptr || kp.bc != nullptr || kp.b[0] != 0.0 || kp.b[1] != 0.0 || kp.b[2] != 0.0;
}

#ifndef DG_VOLUME_LINE_N
#define DG_VOLUME_LINE_N 0xc0   // bit n: the volume terms alone by the lean k_volume_line (n = 8: 80 -> 116 us, off)
#endif
#ifndef DG_VOLUME_LINE_GEN_N
// the same for the convective / reaction kernels: n = 5 too (p = 4 cube 77 -> 64 us: the plane
// k_volume<5, true> spills; for diffusion the plane kernel stays, 55 vs 61 us)
#define DG_VOLUME_LINE_GEN_N 0xe0
#endif
template <int N> inline bool volume_line(const KParams& kp) {
  return (((gen_terms(kp) ? DG_VOLUME_LINE_GEN_N : DG_VOLUME_LINE_N) >> N) & 1) != 0;
}
#ifndef DG_APPLY_WARPS4
// n = 4: cells per CTA of the warp-mode nodal apply, two per warp (0: off), pure diffusion only
// (C2 apply: plane 36.9 us, 4 / 8 / 16 cells 32.8 / 32.8 / 34.9; C4 with convection: plane 308,
// warp mode 317 / 323 / 341 us)
#define DG_APPLY_WARPS4 4
#endif
#ifndef DG_APPLY_WARPS3
#define DG_APPLY_WARPS3 0   // n = 3: the same (9 of 16 lanes; C5: plane 643 us, 4 / 8 cells 721 / 711 us: off)
#endif
template <int N> inline bool warp_apply(const KParams& kp, int with_nbr) {
  constexpr int W = N == 4 ? DG_APPLY_WARPS4 : (N == 3 ? DG_APPLY_WARPS3 : 0);
  return W > 0 && DG_NODAL_APPLY && kp.mask == 7u && with_nbr && !gen_terms(kp);
}
inline bool warp_apply4(const KParams& kp, int with_nbr) { return warp_apply<4>(kp, with_nbr); }
// the full A u goes through the mass-folded kernel k_apply_fold (n = 3, 4, 5; any term set)
template <int N> inline bool fold_apply(const KParams& kp, int with_nbr) {
  constexpr int F = N == 5 ? DG_APPLY_FOLD5 : (N == 4 ? DG_APPLY_FOLD4 : (N == 3 ? DG_APPLY_FOLD3 : 0));
  return F > 0 && DG_NODAL_APPLY && kp.mask == 7u && with_nbr && !force_line(kp) && !(kp.variant & VAR_APPLY_NOFOLD);
}
template <int N>
cudaError_t apply_n(const KParams& kp0, const double* u, double* out, cudaStream_t s, int with_nbr) {
  KParams kp = kp0;   // split_groups fills the split range of this kernel's group size
#ifndef DG_VOL_PERSIST
#define DG_VOL_PERSIST 1
#endif
#ifndef DG_PLANE_VOL67
#define DG_PLANE_VOL67 0   // measured slower: p = 6 volume 105 -> 130 us (255 registers, 8 warps per SM)
#endif
  if constexpr (N >= 6 && N <= 7 && DG_PLANE_VOL67) {
    // n = 6, 7: the plane-per-lane volume kernel without register prefetch (k_volume_s)
    if (kp.mask == 1u && !force_line(kp)) {
      using G = pk::Geo<N>;
      const int grid = (kp.ncells + G::C - 1) / G::C;
      if (grid == 0) return cudaSuccess;
      static int sslots = 0;
      const size_t ssm = sizeof(double) * (size_t)G::TB;
      if (sslots == 0) {
        cudaError_t e = set_smem(pk::k_volume_s<N, true>, ssm);
        if (e == cudaSuccess) e = set_smem(pk::k_volume_s<N, false>, ssm);
        int per_sm = 0, dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pk::k_volume_s<N>, G::NT, ssm);
        if (e != cudaSuccess) return e;
        sslots = max(1, per_sm) * nsm;
      }
      if (gen_terms(kp)) pk::k_volume_s<N, true><<<min(grid, sslots), G::NT, ssm, s>>>(kp, u, out);
      else pk::k_volume_s<N, false><<<min(grid, sslots), G::NT, ssm, s>>>(kp, u, out);
      return cudaGetLastError();
    }
  }
  if constexpr (N <= 5) {
    if (kp.mask == 1u && DG_VOL_PERSIST && N <= 5 && !volume_line<N>(kp)) {
      using G = pk::Geo<N>;
      const int grid = (kp.ncells + G::C - 1) / G::C;
      if (grid == 0) return cudaSuccess;
      // persistent volume kernel: one CTA per resident slot
      static int slots = 0;
      const size_t vsm = pk::smem_apply<N>(false, false);
      if (slots == 0) {
        cudaError_t e = set_smem(pk::k_volume<N, true>, vsm);
        if (e == cudaSuccess) e = set_smem(pk::k_volume<N, false>, vsm);
        if (e != cudaSuccess) return e;
        int per_sm = 0, dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pk::k_volume<N>, G::NT, vsm);
        if (e != cudaSuccess) return e;
        slots = max(1, per_sm) * nsm;
      }
      if constexpr (N == 4) {
        // slim variant (no register prefetch, 4 CTAs per SM); VAR_VOLUME_PREFETCH: k_volume
        if (!(kp.variant & VAR_VOLUME_PREFETCH)) {
          static int sslots = 0;
          const size_t ssm = sizeof(double) * (size_t)G::TB;
          if (sslots == 0) {
            cudaError_t e = set_smem(pk::k_volume_s<N, true>, ssm);
            if (e == cudaSuccess) e = set_smem(pk::k_volume_s<N, false>, ssm);
            int per_sm = 0, dev = 0, nsm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pk::k_volume_s<N>, G::NT, ssm);
            if (e != cudaSuccess) return e;
            sslots = max(1, per_sm) * nsm;
          }
          if (gen_terms(kp)) pk::k_volume_s<N, true><<<min(grid, sslots), G::NT, ssm, s>>>(kp, u, out);
          else pk::k_volume_s<N, false><<<min(grid, sslots), G::NT, ssm, s>>>(kp, u, out);
          return cudaGetLastError();
        }
      }
      if (gen_terms(kp)) pk::k_volume<N, true><<<min(grid, slots), G::NT, vsm, s>>>(kp, u, out);
      else pk::k_volume<N, false><<<min(grid, slots), G::NT, vsm, s>>>(kp, u, out);
      return cudaGetLastError();
    }
  }
#ifndef DG_VOLUME_LPT
#define DG_VOLUME_LPT 1         // x-lines per thread of k_volume_line (the convective n = 7 kernel: 2)
#endif
#ifndef DG_VOLUME_CELLS
#define DG_VOLUME_CELLS 4       // cells per CTA of k_volume_line
#endif
#ifndef DG_VOLUME_TILE_N
#define DG_VOLUME_TILE_N 0      // bit n: k_volume_line reads its lines from a cp.async tile (p = 5: 48 -> 56 us)
#endif
  // lines per thread x cells per CTA, ~8M DoF cubes, diffusion / convective-reaction us
  // (scripts/vol_times.py): p = 5: 1 x 4 55.9 / 64.1, 2 x 4 55.7 / 78.9, 2 x 8 58.5 / 80.0,
  // 2 x 16 104 / 128; p = 6: 1 x 4 72.9 / 111.7, 2 x 4 74.8 / 94.3, 2 x 8 85.9 / 152
  if (kp.mask == 1u && volume_line<N>(kp)) {
    constexpr int CC = DG_VOLUME_CELLS;
    constexpr int LG = N == 7 ? 2 : (N == 8 ? 1 : DG_VOLUME_LPT);   // lines per thread, convective kernel
    using GV = Geo<N, CC>;
    KParams kv_p = kp0;
    const int gridv = split_groups(kv_p, CC);
    if (gridv == 0) return cudaSuccess;
    const size_t smem = sizeof(double) * 2 * (size_t)GV::TENSOR;
    const bool gen = gen_terms(kp);
    constexpr bool TL = (DG_VOLUME_TILE_N >> N) & 1;
    auto kv = gen ? k_volume_line<N, true, LG, CC, TL> : k_volume_line<N, false, DG_VOLUME_LPT, CC, TL>;
    cudaError_t e = set_smem(kv, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gridv);
    cfg.blockDim = dim3(gen ? VolLine<N, LG, CC>::NT : VolLine<N, DG_VOLUME_LPT, CC>::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kv, kv_p, u, out, with_nbr);
  }
  if constexpr (plane_apply<N>()) {
    // (n = 4 with DG_APPLY_WARPS4: A u by the warp-mode line kernel below)
    if (!force_line(kp) && !((N == 4 || N == 3) && warp_apply<N>(kp, with_nbr)) && !fold_apply<N>(kp, with_nbr)) {
      using G = pk::Geo<N>;
      const int grid = split_groups(kp, G::C);
      if (grid == 0) return cudaSuccess;
      const bool faces = kp.mask != 1u;   // mask = volume: the volume terms alone
      const size_t smem = pk::smem_apply<N>(with_nbr, faces);
      const bool gen = gen_terms(kp);
      auto kern = with_nbr ? (gen ? pk::k_apply<N, true, true, true> : pk::k_apply<N, true, true, false>)
                           : (gen ? pk::k_apply<N, false, true, true> : pk::k_apply<N, false, true, false>);
      if (!faces) kern = gen ? pk::k_apply<N, false, false, true> : pk::k_apply<N, false, false, false>;
      cudaError_t e = set_smem(kern, smem);
      if (e != cudaSuccess) return e;
      // programmatic dependent launch (the kernel waits on griddepcontrol before touching u)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(G::NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kern, kp, u, out);
    }
  }
  using G = Geo<N>;
#ifndef DG_APPLY_CELLS5
// cells per CTA of the nodal A u at n = 5 (C3 apply: 8 567 us, 4 561, 2 574, 1 546; staging the
// six neighbour cells of a one-cell CTA with cp.async before the setup: 769 us, 7 KB of L2 reads
// and shared-memory writes per cell)
#define DG_APPLY_CELLS5 1
#endif
#ifndef DG_APPLY_WARPS5
#define DG_APPLY_WARPS5 4   // n = 5: cells (= warps) per CTA of the warp-mode nodal apply (0: off; C3 1 cell per CTA 515 us, 2 / 4 / 8 warps 500 / 490 / 504 us)
#endif
  constexpr int FCELLS = N == 5 ? DG_APPLY_FOLD5 : (N == 4 ? DG_APPLY_FOLD4 : (N == 3 ? DG_APPLY_FOLD3 : 0));
  if constexpr (DG_NODAL_APPLY && FCELLS > 0) {
    if (fold_apply<N>(kp, with_nbr)) {
      constexpr int CC = FCELLS;
      KParams ka = kp0;
      const int grida = split_groups(ka, CC);
      if (grida == 0) return cudaSuccess;
      const size_t smem = apply_fold_smem<N, CC>();
      auto ke = gen_terms(kp) ? k_apply_fold<N, true, CC> : k_apply_fold<N, false, CC>;
      cudaError_t e = set_smem(ke, smem);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grida);
      cfg.blockDim = dim3(fold_threads<N, CC>());
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, ke, ka, u, out, with_nbr);
    }
  }
  constexpr int WCELLS = N == 5 ? DG_APPLY_WARPS5 : (N == 4 ? DG_APPLY_WARPS4 : (N == 3 ? DG_APPLY_WARPS3 : 0));
  if constexpr ((N == 5 || N == 4 || N == 3) && DG_NODAL_APPLY && WCELLS > 0) {
    if (kp.mask == 7u && with_nbr && !force_line(kp) && (N == 5 || warp_apply<N>(kp, with_nbr))) {
      constexpr int CC = WCELLS;
      KParams ka = kp0;
      const int grida = split_groups(ka, CC);
      if (grida == 0) return cudaSuccess;
      const size_t smem = apply_warps_smem<N, CC>();
      auto ke = gen_terms(kp) ? k_apply_warps<N, true, CC> : k_apply_warps<N, false, CC>;
      cudaError_t e = set_smem(ke, smem);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grida);
      cfg.blockDim = dim3(CC * warp_lanes<N>());
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, ke, ka, u, out, with_nbr);
    }
  }
  if constexpr (N == 5 && DG_NODAL_APPLY && DG_APPLY_CELLS5 != Cells<5>::C) {
    if (kp.mask == 7u && with_nbr) {
      constexpr int CC = DG_APPLY_CELLS5;
      KParams ka = kp0;
      const int grida = split_groups(ka, CC);
      if (grida == 0) return cudaSuccess;
      const size_t smem = apply_nodal_smem<N, CC>();
      auto ke = gen_terms(kp) ? k_apply_nodal<N, true, CC> : k_apply_nodal<N, false, CC>;
      cudaError_t e = set_smem(ke, smem);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grida);
      cfg.blockDim = dim3(Geo<N, CC>::NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, ke, ka, u, out, with_nbr);
    }
  }
#ifndef DG_DT_WARPS5
#define DG_DT_WARPS5 4   // n = 5: cells (= warps) per CTA of the warp-mode nodal D_T (0: off)
#endif
  if constexpr (N == 5 && DG_DT_WARPS5 > 0) {
    if (kp.mask == 7u && !with_nbr && !force_line(kp)) {
      constexpr int CC = DG_DT_WARPS5;
      KParams ka = kp0;
      const int grida = split_groups(ka, CC);
      if (grida == 0) return cudaSuccess;
      const size_t smem = sizeof(double) * 2 * (size_t)Geo<N, CC>::TENSOR;
      auto ke = gen_terms(kp) ? k_dt_warps<N, true, CC> : k_dt_warps<N, false, CC>;
      cudaError_t e = set_smem(ke, smem);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grida);
      cfg.blockDim = dim3(CC * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, ke, ka, u, out, with_nbr);
    }
  }
  // (each kernel above splits the groups by its own group size: an early return on the group
  // count of G::C would skip its launch when that count is 0)
  const int grid = split_groups(kp, G::C);
  if (grid == 0) return cudaSuccess;
  // mask = volume: no face passes; D_T (all parts, no neighbours): self faces as Gauss-point
  // operators. Neither has face passes, so neither gets the face buffer (more resident CTAs)
  const bool nofb = kp.mask == 1u || (!with_nbr && kp.mask == 7u);   // kernels without face passes
  const size_t smem = sizeof(double) * (3 * (size_t)G::TENSOR +
                                        (nofb ? 0 : (DG_NODAL_APPLY ? apply_fb_doubles<N>() : (size_t)G::FACE)));
  const bool gen = gen_terms(kp);
  auto kl = kp.mask == 1u ? (gen ? k_apply<N, false> : k_apply<N, false, false, false>)
                          : (!with_nbr && kp.mask == 7u ? (gen ? k_apply<N, false, true> : k_apply<N, false, true, false>)
                                                        : (gen ? k_apply<N, true> : k_apply<N, true, false, false>));
  const size_t smem_n = smem;
  cudaError_t e = set_smem(kl, smem_n);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(G::NT);
  cfg.dynamicSmemBytes = smem_n;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = DG_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kl, kp, u, out, with_nbr);
}

#ifndef DG_GMRES_TU
#define DG_GMRES_TU 0
#endif
// restarted GMRES(KR) on the plane kernels, Krylov basis + diagonal in TMEM (compact colour maps
// not supported: the SOR half-sweeps run masked). KR fills 256 TMEM columns at n = 2, 3 (two CTAs
// per SM) and all 512 at n = 4 (one CTA per SM: GMRES(7) with two CTAs was faster on C4, 13.3 vs
// 14.8 ms, but stalls at cell Peclet 1.8e4; profiles/r01_ab.md); n = 5: 9 basis vectors + the
// diagonal = 500 of the 512 columns (one CTA per SM). The CTAs take the groups in order (the
// longest-first permutation is made for the other solvers' group size).
template <int N, bool SWEEP>
cudaError_t gmres_n(int method, const KParams& kp0, const double* in, const double* f, double* out,
                    cudaStream_t s) {
  if constexpr (N <= 5) {
    KParams kp = kp0;
    kp.gperm = nullptr;
    using G = pk::Geo<N>;
    const int grid = split_groups(kp, G::C);
    if (grid == 0) return cudaSuccess;
    constexpr int KR = N == 5 ? 9 : N == 4 ? 15 : N == 3 ? 13 : 15;
    if (method == LM_GMRES)
      return launch(pk::k_gmres<N, SWEEP, false, KR>, grid, G::NT, pk::smem_gmres<N, KR>(false), s, kp, in, f, out);
    if (method == LM_GMRES_THOMAS)
      return launch(pk::k_gmres<N, SWEEP, true, KR>, grid, G::NT, pk::smem_gmres<N, KR>(true), s, kp, in, f, out);
  }
  return cudaErrorInvalidValue;
}

template <int N, bool SWEEP>
cudaError_t solve_n(int method, const KParams& kp0, const double* in, const double* f, double* out,
                    cudaStream_t s) {
  KParams kp = kp0;   // split_groups fills the split range of this kernel's group size
  // plane solvers for n <= 4; at n = 5 the line solvers (self faces as Gauss-point operators,
  // two CTAs per SM) beat the register-starved plane ones (C3 sweep 32.7 -> 20.1 ms), except
  // for the tridiagonal preconditioner, which exists in the plane family only
  if constexpr (N <= 5) {
    if (!force_line(kp) && (N <= 4 || method == LM_BICGSTAB_THOMAS || method == LM_GMRES ||
                            method == LM_GMRES_THOMAS)) {
      using G = pk::Geo<N>;
      const int grid = split_groups(kp, G::C);
      if (grid == 0) return cudaSuccess;
      constexpr size_t cg_smem = pk::smem_solve<N>(2);
      // compact colour map (red-black SOR half-sweeps, n <= 4 sweeps only): own instantiations
      if constexpr (SWEEP && N <= 4) {
        if (kp.cmap) {
          if (method == LM_BICGSTAB_THOMAS)
            return launch(pk::k_bicgstab<N, true, true, true>, grid, G::NT, pk::smem_solve<N>(7), s, kp, in, f, out);
          if (method == LM_BICGSTAB) {
            if constexpr (N == 4)
              if (use_tmem(kp))
                return launch(pk::k_bicgstab<N, true, false, true, true>, grid, G::NT, pk::smem_solve<N>(2), s, kp, in, f, out);
            return launch(pk::k_bicgstab<N, true, false, true>, grid, G::NT, pk::smem_solve<N>(5), s, kp, in, f, out);
          }
          if (gen_terms(kp))
            return launch(pk::k_cg<N, true, true, true>, grid, G::NT, cg_smem, s, kp, in, f, out);
          return launch(pk::k_cg<N, true, false, true>, grid, G::NT, cg_smem, s, kp, in, f, out);
        }
      }
      if (method == LM_BICGSTAB_THOMAS)
        return launch(pk::k_bicgstab<N, SWEEP, true>, grid, G::NT, pk::smem_solve<N>(7), s, kp, in, f, out);
      if (method == LM_GMRES || method == LM_GMRES_THOMAS) {
        // n <= 4: the GMRES kernels come from their own translation unit (dg_kernels_gmres.cu),
        // compiled with four-warp plane CTAs: the basis fills 256 / 512 TMEM columns, and a
        // CTA's warps reach only their own lane quadrants, so a CTA must span all four
        if constexpr (N <= 4 && !DG_GMRES_TU) return solve_gmres(N - 1, method, SWEEP, kp0, in, f, out, s);
        else return gmres_n<N, SWEEP>(method, kp0, in, f, out, s);
      }
      if constexpr (N <= 4) {
        if (method == LM_BICGSTAB) {
          if constexpr (N == 4)
            if (use_tmem(kp))
              return launch(pk::k_bicgstab<N, SWEEP, false, false, true>, grid, G::NT, pk::smem_solve<N>(2), s, kp, in, f, out);
          return launch(pk::k_bicgstab<N, SWEEP>, grid, G::NT, pk::smem_solve<N>(5), s, kp, in, f, out);
        }
        if (gen_terms(kp))
          return launch(pk::k_cg<N, SWEEP, true>, grid, G::NT, cg_smem, s, kp, in, f, out);
        return launch(pk::k_cg<N, SWEEP, false>, grid, G::NT, cg_smem, s, kp, in, f, out);
      }
    }
  }
  if (method == LM_BICGSTAB_THOMAS) return cudaErrorInvalidValue;   // plane kernels (p <= 4) only
  if constexpr (N == 5 && DG_CGW_CELLS != Cells<N>::C) {
    // warp-per-cell CG with DG_CGW_CELLS cells per CTA (its own group size, hence its own split)
    if (method == LM_CG && !(kp.variant & VAR_LINE_CG_CTA)) {
      constexpr int CC = DG_CGW_CELLS;
      using G1 = Geo<N, CC>;
      const int grid1 = split_groups(kp, CC);
      if (grid1 == 0) return cudaSuccess;
      const size_t sm1 = sizeof(double) * (7 * (size_t)G1::TENSOR + (fb_alias<N, CC>() ? 0 : (size_t)G1::FACE));
      return launch(gen_terms(kp) ? k_cg_w<N, SWEEP, true, CC> : k_cg_w<N, SWEEP, false, CC>, grid1, G1::NTW,
                    sm1, s, kp, in, f, out);
    }
  }
  if constexpr (N >= 6 && line_cg_cells<N>() != Cells<N>::C) {
    // CTA-wide CG with its own group size (hence its own split), n >= 6
    if (method == LM_CG && !(N <= 7 && (kp.variant & VAR_LINE_CG_CTA))) {
      constexpr int CC = line_cg_cells<N>();
      using G1 = Geo<N, CC>;
      const int grid1 = split_groups(kp, CC);
      if (grid1 == 0) return cudaSuccess;
      const size_t sm1 = sizeof(double) * (7 * (size_t)G1::TENSOR + (fb_alias<N, CC>() ? 0 : (size_t)G1::FACE));
      return launch(k_cg<N, SWEEP, CC>, grid1, G1::NT, sm1, s, kp, in, f, out);
    }
  }
  // (each kernel below has its own group size and split; launch() skips an empty grid)
  using G = Geo<N>;
  const int grid = split_groups(kp, G::C);
  // line solvers per degree (measured after the D_T fold and the register-resident CTA CG,
  // profiles/r02_ab.md): CG one warp per cell at n = 5, CTA-wide at n = 6..8; BiCGStab one warp
  // per cell at n = 5 and 7, CTA-wide at n = 6 and 8; VAR_LINE_CG_CTA selects the other kernel
  constexpr bool warp_cg = N == 5, warp_bicg = N == 5 || N == 7;
  if constexpr (N >= 5 && N <= 7) {
    const bool cta = ((kp.variant & VAR_LINE_CG_CTA) != 0) == warp_bicg;
    if (method == LM_BICGSTAB && !cta) {
      if constexpr (bicgw_cells<N>() != Cells<N>::C) {   // its own group size, hence its own split
        constexpr int CC = bicgw_cells<N>();
        using G1 = Geo<N, CC>;
        const int grid1 = split_groups(kp, CC);
        if (grid1 == 0) return cudaSuccess;
        const size_t sm1 = sizeof(double) * (10 * (size_t)G1::TENSOR + (fb_alias<N, CC>() ? 0 : (size_t)G1::FACE));
        return launch(k_bicgstab_w<N, SWEEP, CC>, grid1, G1::NTW, sm1, s, kp, in, f, out);
      }
      return launch(k_bicgstab_w<N, SWEEP>, grid, G::NTW,
                    fb_alias<N>() ? sizeof(double) * 10 * (size_t)G::TENSOR : smem_bytes<N>(10), s, kp, in, f, out);
    }
  }
  if (method == LM_BICGSTAB) {
    if constexpr (bicg_cells<N>() != Cells<N>::C) {   // its own group size, hence its own split
      constexpr int CC = bicg_cells<N>();
      using G1 = Geo<N, CC>;
      const int grid1 = split_groups(kp, CC);
      const size_t sm1 = sizeof(double) * (10 * (size_t)G1::TENSOR + (fb_alias<N, CC>() ? 0 : (size_t)G1::FACE));
      return launch(k_bicgstab<N, SWEEP, CC>, grid1, G1::NT, sm1, s, kp, in, f, out);
    }
    return launch(k_bicgstab<N, SWEEP>, grid, G::NT,
                  fb_alias<N>() ? sizeof(double) * 10 * (size_t)G::TENSOR : smem_bytes<N>(10), s, kp, in, f, out);
  }
  if constexpr (N >= 5 && N <= 7) {   // n = 8: 255 registers with spills, the CTA version is faster
    const bool cta = ((kp.variant & VAR_LINE_CG_CTA) != 0) == warp_cg;
    if (!cta)
      return launch(gen_terms(kp) ? k_cg_w<N, SWEEP, true> : k_cg_w<N, SWEEP, false>, grid, G::NTW,
                    fb_alias<N>() ? sizeof(double) * 7 * (size_t)G::TENSOR : smem_bytes<N>(7), s, kp, in, f, out);
  }
  return launch(k_cg<N, SWEEP>, grid, G::NT,
                fb_alias<N>() ? sizeof(double) * 7 * (size_t)G::TENSOR : smem_bytes<N>(7), s, kp, in, f, out);
}

// ---- per-degree entry points (dg_degree.h) ---------------------------------------------
template <int N> bool upload_n(const Tables1D& t, cudaError_t* err) {
  DevTab d{};
  const int n = t.n;
  for (int i = 0; i < n * n; ++i) { d.A[i] = t.A[i]; d.D[i] = t.D[i]; d.M[i] = t.M[i]; d.G[i] = t.G[i]; }
  for (int i = 0; i < n; ++i) {
    d.w[i] = t.wq[i]; d.d0[i] = t.d0[i]; d.d1[i] = t.d1[i];
    d.Sd[i] = t.Sdiag[i]; d.Cd[i] = t.Cdiag[i]; d.Md[i] = t.Mdiag[i];
    d.E0[i] = t.E0[i]; d.E1[i] = t.E1[i]; d.F0[i] = t.F0[i]; d.F1[i] = t.F1[i];
    d.E0W[i] = t.E0[i] / t.wq[i]; d.E1W[i] = t.E1[i] / t.wq[i];
    d.F0W[i] = t.F0[i] / t.wq[i]; d.F1W[i] = t.F1[i] / t.wq[i];
  }
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) {
      d.AW[q * n + j] = t.A[q * n + j] * t.wq[q];
      d.GW[q * n + j] = t.G[q * n + j] * t.wq[q];
      d.DW[q * n + j] = t.D[q * n + j] * t.wq[q] / t.wq[j];
    }
  for (int q = 0; q < n; ++q)
    for (int r = 0; r < n; ++r) {
      double sg = 0.0;
      for (int k = 0; k < n; ++k) sg += t.D[k * n + q] * t.wq[k] * t.D[k * n + r];
      d.SG[q * n + r] = sg;
      d.SGW[q * n + r] = sg / t.wq[q];
      d.CG[q * n + r] = t.D[r * n + q] * t.wq[r];
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double sv = 0.0, cv = 0.0;
      for (int q = 0; q < n; ++q) {
        sv += t.wq[q] * t.G[q * n + i] * t.G[q * n + j];
        cv += t.wq[q] * t.G[q * n + i] * t.A[q * n + j];
      }
      d.S[i * n + j] = sv;
      d.Cm[i * n + j] = cv;
    }
  {
    // Mhat^-1 [Shat | Chat | e0 | e1 | d0 | d1] by Gauss-Jordan with partial pivoting (long double)
    const int m = 2 * n + 4;
    FoldTab ft{};
    long double a[8][8], b[8][20];
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) {
        a[i][j] = t.M[i * n + j];
        b[i][j] = d.S[i * n + j];
        b[i][n + j] = d.Cm[i * n + j];
      }
      b[i][2 * n] = i == 0;
      b[i][2 * n + 1] = i == n - 1;
      b[i][2 * n + 2] = t.d0[i];
      b[i][2 * n + 3] = t.d1[i];
    }
    for (int c = 0; c < n; ++c) {
      int pv = c;
      for (int r = c + 1; r < n; ++r)
        if (fabsl(a[r][c]) > fabsl(a[pv][c])) pv = r;
      for (int j = 0; j < n; ++j) { const long double x = a[c][j]; a[c][j] = a[pv][j]; a[pv][j] = x; }
      for (int j = 0; j < m; ++j) { const long double x = b[c][j]; b[c][j] = b[pv][j]; b[pv][j] = x; }
      const long double ip = 1.0L / a[c][c];
      for (int j = 0; j < n; ++j) a[c][j] *= ip;
      for (int j = 0; j < m; ++j) b[c][j] *= ip;
      for (int r = 0; r < n; ++r) {
        if (r == c) continue;
        const long double f = a[r][c];
        for (int j = 0; j < n; ++j) a[r][j] -= f * a[c][j];
        for (int j = 0; j < m; ++j) b[r][j] -= f * b[c][j];
      }
    }
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) {
        ft.MiS[i * n + j] = (double)b[i][j];
        ft.MiC[i * n + j] = (double)b[i][n + j];
      }
      ft.mie0[i] = (double)b[i][2 * n];
      ft.mie1[i] = (double)b[i][2 * n + 1];
      ft.mid0[i] = (double)b[i][2 * n + 2];
      ft.mid1[i] = (double)b[i][2 * n + 3];
    }
    *err = cudaMemcpyToSymbol(c_fold, &ft, sizeof(FoldTab));
    if (*err != cudaSuccess) return false;
  }
  *err = cudaMemcpyToSymbol(c_tab, &d, sizeof(DevTab), sizeof(DevTab) * N);
  return *err == cudaSuccess;
}

}  // namespace

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
constexpr int lcm_c(int a, int b) { return a / gcd_c(a, b) * b; }
// every group size split_groups is called with at degree N (plane kernels n <= 5, line apply /
// solvers, the warp / CTA CG and BiCGStab variants, the lean volume kernel)
template <int N> constexpr int group_lcm_n() {
  int l = lcm_c(Cells<N>::C, line_cg_cells<N>());
  l = lcm_c(l, bicgw_cells<N>());
  l = lcm_c(l, bicg_cells<N>());
  l = lcm_c(l, DG_CGW_CELLS);
  l = lcm_c(l, DG_VOLUME_CELLS);
  if constexpr (N == 5) l = lcm_c(l, DG_APPLY_CELLS5);
  if constexpr (N == 5 && DG_APPLY_WARPS5 > 0) l = lcm_c(l, DG_APPLY_WARPS5);
  if constexpr (N == 5 && DG_APPLY_FOLD5 > 0) l = lcm_c(l, DG_APPLY_FOLD5);
  if constexpr (N == 4 && DG_APPLY_FOLD4 > 0) l = lcm_c(l, DG_APPLY_FOLD4);
  if constexpr (N == 3 && DG_APPLY_FOLD3 > 0) l = lcm_c(l, DG_APPLY_FOLD3);
  if constexpr (N == 5 && DG_DT_WARPS5 > 0) l = lcm_c(l, DG_DT_WARPS5);
  if constexpr (N == 4 && DG_APPLY_WARPS4 > 0) l = lcm_c(l, DG_APPLY_WARPS4);
  if constexpr (N == 3 && DG_APPLY_WARPS3 > 0) l = lcm_c(l, DG_APPLY_WARPS3);
  if constexpr (N <= 5) l = lcm_c(l, pk::Geo<N>::C);
  return l;
}

#define DG_INSTANTIATE_DEGREE(NN)                                                              \
  template <> bool Deg<NN>::upload(const Tables1D& t, cudaError_t* err) { return upload_n<NN>(t, err); } \
  template <> cudaError_t Deg<NN>::apply(const KParams& kp, const double* u, double* out,        \
                                         cudaStream_t s, int with_nbr) {                         \
    return apply_n<NN>(kp, u, out, s, with_nbr);                                                 \
  }                                                                                              \
  template <> int Deg<NN>::solver_group_cells() { return NN <= 4 ? pk::Geo<(NN <= 5 ? NN : 5)>::C : 0; } \
  template <> int Deg<NN>::group_lcm() { return group_lcm_n<NN>(); }                          \
  template <> cudaError_t Deg<NN>::solve(int method, bool sweep, const KParams& kp,              \
                                         const double* in, const double* f, double* out,         \
                                         cudaStream_t s) {                                       \
    return sweep ? solve_n<NN, true>(method, kp, in, f, out, s)                                  \
                 : solve_n<NN, false>(method, kp, in, f, out, s);                                \
  }

}  // namespace dg
