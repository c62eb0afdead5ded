// Plane-per-thread fp64 kernels for n = p+1 <= 5 (included by dg_kernels.cu).
//
// Each cell is owned by n consecutive lanes of one warp; lane t holds one n x n plane of
// the cell in registers, so two of the three 1D contractions of every sum-factorisation
// stage run in registers and only the third goes through shared memory. One operator
// application (A or D_T) is three register phases separated by two transposes:
//
//   Q1 (lane = z node k, plane (j,i)):  a = A_x u;  t2 = A_y a;  t2y = G_y a     (Stage 1)
//        y-face traces of the nodal plane -> S/T arrays, interpolated along x
//   Q2 (lane = y Gauss point qy, plane (qz,qx)):  U = A_z t2, Uy = A_z t2y;
//        Stage 2 at the Gauss points; x- and z-direction terms D^T(W(K D U - b U));
//        x- and z-face traces straight from the Gauss values (E/F end-point vectors),
//        face fluxes injected back through A^-T (so the later A^T contractions give the
//        tangential face mass); then A_z^T on R and on F_y                     (Stage 3, part)
//   Q3 (lane = z node k, plane (qy,qx)):  V' = A_y^T R + G_y^T F_y;  y-face terms with the
//        z face mass;  V = A_x^T V'                                              (Stage 3)
//
// The output plane has the same ownership as the input plane, so the per-cell Krylov
// vectors of the local solves stay in registers; dot products are n-lane shuffles.
// Neighbour traces (A only) are staged tile by tile through shared memory with coalesced
// loads in a prologue and enter Q1/Q2 as extra face arrays.

#ifndef DG_RESTRICT
#define DG_RESTRICT
#endif
namespace pk {

#ifndef DG_PLANE_NODAL_APPLY
#define DG_PLANE_NODAL_APPLY 1   // plane-family A u in the nodal Kronecker-sum form
#endif
#ifndef DG_NODAL_BICG
#define DG_NODAL_BICG 1
#endif
#ifndef DG_PLANE5_ASYNC
#define DG_PLANE5_ASYNC 0
#endif
#ifndef DG_VOL_MINB
#define DG_VOL_MINB 3   // resident CTAs per SM the persistent volume kernel is compiled for
#endif

template <int N> struct PL;
// KS/CTB: transpose-buffer plane / cell strides; QS/PS: plane / cell strides of the per-lane
// plane storage (X, diag, ...). All chosen by an offline search for conflict-free lane patterns.
// warps (cell groups of 32 / n cells each) per plane CTA: two (measured: C4 BiCGStab sweep
// 5490 / 4306 / 4155 us with 4 / 3 / 2 warps, C2 CG sweep 340 / 304 / 276, C5 apply 644 / - / 587,
// p = 1 apply 192 / - / 178; four warps needed 119 KB of shared memory per CTA at n = 4: one CTA,
// 4 warps per SM); the local GMRES keeps four (dg_kernels_gmres.cu: tensor-memory lane quadrants)
#ifndef DG_PL_WARPS2
#define DG_PL_WARPS2 2
#endif
#ifndef DG_PL_WARPS3
#define DG_PL_WARPS3 2
#endif
#ifndef DG_PL_WARPS4
#define DG_PL_WARPS4 2
#endif
#ifndef DG_PL_WARPS5
#define DG_PL_WARPS5 2
#endif
#ifndef DG_PL3_KS
// n = 3 transpose strides (A/B: KS = 10, CTB = 71 gives the apply 3 instead of 2 CTAs per SM,
// C5 apply 739 -> 662 us, but 2-way half-warp conflicts cost the sweep 3960 -> 4264 us)
#define DG_PL3_KS 19
#define DG_PL3_CTB 121
#endif
template <> struct PL<2> { static constexpr int WARPS = DG_PL_WARPS2, KS = 5, CTB = 22, QS = 8, PS = 17; };
template <> struct PL<3> { static constexpr int WARPS = DG_PL_WARPS3, KS = DG_PL3_KS, CTB = DG_PL3_CTB, QS = 13, PS = 39; };
template <> struct PL<4> { static constexpr int WARPS = DG_PL_WARPS4, KS = 20, CTB = 161, QS = 17, PS = 68; };
template <> struct PL<5> { static constexpr int WARPS = DG_PL_WARPS5, KS = 25, CTB = 253, QS = 25, PS = 125; };
// n = 6, 7: the volume-only kernel k_volume_s alone (one n x n plane per lane, 5 / 4 cells per
// warp); strides from the same search restricted to its two lane patterns (read_plane and the
// Q2 columns): 2 + 3 and 2 + 2 wavefronts per warp-wide 8-byte access
template <> struct PL<6> { static constexpr int WARPS = 2, KS = 37, CTB = 447, QS = 36, PS = 216; };
template <> struct PL<7> { static constexpr int WARPS = 2, KS = 49, CTB = 692, QS = 49, PS = 343; };

template <int N_> struct Geo {
  static constexpr int N = N_, N2 = N * N, N3 = N * N * N;
  static constexpr int CPW = 32 / N, WARPS = PL<N>::WARPS, C = CPW * WARPS, NT = 32 * WARPS;
  static constexpr int KS = PL<N>::KS, ARR = N * KS, CTB = PL<N>::CTB;
  // per-cell stride of a block of 4 face arrays; even at n = 4 so that staged neighbour tiles
  // can be copied with 16-byte cp.async (see async_nbr)
  // DG_PLANE5_ASYNC: at n = 5 too a face region holds a whole neighbour tile (cp.async staging)
  static constexpr int FS = (N == 5 && DG_PLANE5_ASYNC) ? N3 : 4 * N2 + (N == 4 ? 2 : 1);
  static constexpr int QS = PL<N>::QS, PS = PL<N>::PS;  // plane storage (X, Dg, ...)
  static_assert(PS >= N * QS && PS >= FS, "plane storage must hold a cell and a face block");
  static constexpr int PER = (C * N3 + NT - 1) / NT;      // tile elements per thread
  // dynamic shared memory (doubles)
  static constexpr int TB = C * CTB;      // transposes / tile staging
  static constexpr int FY = C * FS;       // y-face arrays (k, qx)
  static constexpr int FX = C * FS;       // x-neighbour arrays (k, qy)
  static constexpr int FZ = C * FS;       // z-neighbour arrays (j, qx)
};

// WB: with the per-cell self-face operators B (local solvers); the apply kernels omit them.
template <int N, bool WB = true> struct Cells {
  static constexpr int C = Geo<N>::C;
  // odd stride (the cells of a half-warp hit distinct banks), room for the x / z Gauss-point
  // self-face operators (2 n^2) or the three nodal D_T factors (3 n^2, setup_K3)
  static constexpr int BS = 3 * N * N + (N % 2 == 0 ? 1 : 2);
  double vc[C][4];
  double vb[C][3];   // |T| b_k / h_k of the cell (volume advection)
  double fc[C][6][6];
  const double* nb[C][6];
  int cell[C];
  // per face: bit cs set when cell cs has an in-slab neighbour there (its tile is then at
  // tile +- step n^3, contiguous); nbg[f] != 0 when some cell's neighbour is a ghost-layer cell
  static_assert(C <= 64, "neighbour masks hold 64 cells");
  unsigned int nbm[6][2];
  int nbg[6];
  // per-cell self-face operators at the Gauss points: B[cs][0] acts on x-rows, B[cs][1] on z-columns
  double B[WB ? C : 1][BS];
};

// per-lane identity
struct Lane {
  int lane, cs, t;
  bool active;
};
template <int N> __device__ __forceinline__ Lane lane_id() {
  using G = Geo<N>;
  Lane L;
  L.lane = threadIdx.x & 31;
  L.active = L.lane < G::CPW * N;
  L.cs = (threadIdx.x >> 5) * G::CPW + (L.active ? L.lane / N : 0);
  L.t = L.lane % N;
  return L;
}

// sum over the n lanes of the cell (identical order, hence identical result, in every lane)
template <int N> __device__ __forceinline__ double cell_sum(double v, int lane) {
  const int base = (lane / N) * N;
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) s += __shfl_sync(0xffffffffu, v, base + m);
  return s;
}

template <int N> __device__ __forceinline__ double T_A(int i) { return c_tab[N].A[i]; }
template <int N> __device__ __forceinline__ double T_G(int i) { return c_tab[N].G[i]; }
template <int N> __device__ __forceinline__ double T_D(int i) { return c_tab[N].D[i]; }
template <int N> __device__ __forceinline__ double T_W(int i) { return c_tab[N].w[i]; }

// runtime-indexed rows held in registers
template <int N> struct Rows {
  double Arow[N];   // A[t][.]   (y interpolation of z-neighbour traces)
  double Mrow[N];   // Mhat[t][.] (z face mass of the y faces)
  double Md, Sd, Cd;
};
template <int N> __device__ __forceinline__ void load_rows(Rows<N>& r, int t) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    r.Arow[j] = c_tab[N].A[t * N + j];
    r.Mrow[j] = c_tab[N].M[t * N + j];
  }
  r.Md = c_tab[N].Md[t];
  r.Sd = c_tab[N].Sd[t];
  r.Cd = c_tab[N].Cd[t];
}
template <int N> __device__ __forceinline__ double T_AW(int i) { return c_tab[N].AW[i]; }
template <int N> __device__ __forceinline__ double T_GW(int i) { return c_tab[N].GW[i]; }
template <int N> __device__ __forceinline__ double T_DW(int i) { return c_tab[N].DW[i]; }
template <int N> __device__ __forceinline__ double T_SGW(int i) { return c_tab[N].SGW[i]; }

// ---- coalesced tile staging: C cells x n^3 (contiguous in global) -> TB layout ---------
// element (k, j, i) of cell slot cs at cs*CTB + k*KS + j*N + i
template <int N>
__device__ __forceinline__ void stage_tile(double* TB, const double* __restrict__ src, int nvalid) {
  using G = Geo<N>;
  double v[G::PER];
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    v[m] = (e < G::C * G::N3 && e / G::N3 < nvalid) ? src[e] : 0.0;
  }
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    const int cs = e / G::N3, r = e % G::N3;
    if (e < G::C * G::N3) TB[cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2)] = v[m];
  }
}
// the group's own tile / a neighbour tile into registers (coalesced, all loads in flight)
template <int N>
__device__ __forceinline__ void load_own(double (&v)[Geo<N>::PER], const double* __restrict__ src,
                                         int nvalid) {
  using G = Geo<N>;
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    v[m] = (e < G::C * G::N3 && e / G::N3 < nvalid) ? __ldg(src + e) : 0.0;
  }
}
// neighbour tile: per-cell base pointers (nullptr -> zeros), loaded into registers
// (z faces at a slab boundary: the neighbour is a trace record of 2 n^2 doubles, which lands in
// planes 0 and 1 of the staged tile; the ghost buffers are padded so the full n^3 read stays in
// bounds)
template <int N, bool WB>
__device__ __forceinline__ void load_nbr(double (&v)[Geo<N>::PER], const Cells<N, WB>& cl, int f,
                                         const KParams& kp) {
  using G = Geo<N>;
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    const int cs = e / G::N3, r = e % G::N3;
    const double* p = (e < G::C * G::N3) ? cl.nb[cs][f] : nullptr;
    v[m] = p ? __ldg(p + r) : 0.0;
  }
}
template <int N>
__device__ __forceinline__ void store_tile(double* TB, const double (&v)[Geo<N>::PER]) {
  using G = Geo<N>;
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    const int cs = e / G::N3, r = e % G::N3;
    if (e < G::C * G::N3) TB[cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2)] = v[m];
  }
}
template <int N>
__device__ __forceinline__ void unstage_tile(const double* TB, double* __restrict__ dst, int nvalid) {
  using G = Geo<N>;
  for (int e = threadIdx.x; e < nvalid * G::N3; e += G::NT) {
    const int cs = e / G::N3, r = e % G::N3;
    dst[e] = TB[cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2)];
  }
}
template <int N>
__device__ __forceinline__ void read_plane(const double* TB, const Lane& L, double (&p)[N][N]) {
  using G = Geo<N>;
  const double* b = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) p[j][i] = b[j * N + i];
}
template <int N>
__device__ __forceinline__ void write_plane(double* TB, const Lane& L, const double (&p)[N][N]) {
  using G = Geo<N>;
  double* b = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) b[j * N + i] = p[j][i];
}

// ---- neighbour prologue: traces of the 6 face neighbours -> FY (nodal), FX, FZ ----------
// Must be called by all threads; leaves TB free. Face order f = 2*axis + hi.
template <int N, bool WB>
__device__ void nbr_prologue(const KParams& kp, const Cells<N, WB>& cl, const Lane& L, double* TB,
                             double* FY, double* FX, double* FZ, const double* tile,
                             double (&pv0)[Geo<N>::PER], double (&pv1)[Geo<N>::PER]) {
  using G = Geo<N>;
  const int k = L.t;
  // x faces: the neighbour is usually the next / previous cell of the group, whose tile is
  // still in TB (staged by the caller); otherwise its plane k is read from global memory.
  if (L.active) {
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const double* c = cl.fc[L.cs][hi];
      const double cna = c[2], cng = c[3], ctn = c[5];
      const double* nbp = cl.nb[L.cs][hi];
      const int ncs = L.cs + (hi ? 1 : -1);
      const double* plane = nullptr;
      if (nbp) {
        if (ncs >= 0 && ncs < G::C && nbp == tile + (size_t)ncs * G::N3)
          plane = TB + ncs * G::CTB + k * G::KS;
        else
          plane = nbp + k * G::N2;
      }
      double S[N], T[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double row[N];
#pragma unroll
        for (int i = 0; i < N; ++i) row[i] = plane ? plane[j * N + i] : 0.0;
        double g = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) g = fma(hi ? c_tab[N].d0[i] : c_tab[N].d1[i], row[i], g);
        const double a = hi ? row[0] : row[N - 1];
        S[j] = cna * a + cng * g * kp.ih[0];
        T[j] = ctn * a;
      }
      double* fx = FX + L.cs * G::FS + (hi ? 2 : 0) * G::N2 + k * N;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double s = 0.0, tt = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          s = fma(T_A<N>(q * N + j), S[j], s);
          tt = fma(T_A<N>(q * N + j), T[j], tt);
        }
        fx[q] = s;
        fx[G::N2 + q] = tt;
      }
    }
  }
  // y / z neighbours: two tiles per round (the y pair, then the z pair) staged into the two
  // halves of TB; the z pair's global loads are in flight while the y traces are extracted.
#pragma unroll 1
  for (int axis = 1; axis < 3; ++axis) {
    __syncthreads();
    store_tile<N>(TB, pv0);
    store_tile<N>(TB + G::ARR, pv1);
    __syncthreads();
    if (axis == 1) {
      load_nbr<N>(pv0, cl, 4, kp);
      load_nbr<N>(pv1, cl, 5, kp);
    }
    if (!L.active) continue;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const int f = 2 * axis + hi;
      const double* c = cl.fc[L.cs][f];
      const double cna = c[2], cng = c[3], ctn = c[5];
      const double* nb = TB + L.cs * G::CTB + hi * G::ARR;   // layout k*KS + j*N + i
      if (axis == 1) {
        // lane k: columns i of the neighbour's plane k (nodal in i; interpolated in Q1)
        double* fy = FY + L.cs * G::FS + (hi ? 2 : 0) * G::N2 + k * N;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double g = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j)
            g = fma(hi ? c_tab[N].d0[j] : c_tab[N].d1[j], nb[k * G::KS + j * N + i], g);
          const double a = nb[k * G::KS + (hi ? 0 : N - 1) * N + i];
          fy[i] = cna * a + cng * g * kp.ih[1];
          fy[G::N2 + i] = ctn * a;
        }
      } else {
        // lane t = y node j: the neighbour's z-lines (kk, i) at fixed j (a ghost trace record:
        // plane 0 the face values, plane 1 the normal-derivative sums)
        const int j = L.t;
        const bool tr = ghost_trace(kp, cl.cell[L.cs], hi);
        double S[N], T[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double g = 0.0;
          if (tr) {
            g = nb[G::KS + j * N + i];
          } else {
#pragma unroll
            for (int kk = 0; kk < N; ++kk)
              g = fma(hi ? c_tab[N].d0[kk] : c_tab[N].d1[kk], nb[kk * G::KS + j * N + i], g);
          }
          const double a = nb[(tr ? 0 : (hi ? 0 : N - 1)) * G::KS + j * N + i];
          S[i] = cna * a + cng * g * kp.ih[2];
          T[i] = ctn * a;
        }
        double* fz = FZ + L.cs * G::FS + (hi ? 2 : 0) * G::N2 + j * N;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double s = 0.0, tt = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            s = fma(T_A<N>(q * N + i), S[i], s);
            tt = fma(T_A<N>(q * N + i), T[i], tt);
          }
          fz[q] = s;
          fz[G::N2 + q] = tt;
        }
      }
    }
  }
  __syncthreads();
}

// ---- asynchronous neighbour staging (cp.async, no registers held while in flight) --------
// All five tiles a cell group needs for A u (own, y-lo, y-hi, z-lo, z-hi) are copied global ->
// shared with 8-byte cp.async as soon as their addresses are known, so their latencies overlap
// each other and the coefficient setup; missing neighbours (domain boundary) are zero-filled.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  // no "memory" clobber: the copies may be issued in any order relative to other smem reads
  // (the destination is read only after cp_async_wait_all + a barrier)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
// The own tile and the four y / z neighbour tiles of the apply's prologue in one loop, when every
// neighbour tile is on the fast path (no ghost-layer neighbour) and none of them goes by 16-byte
// pairs: the element's cell, plane and in-plane offset are computed once for the five copies
// (separately they were ~30 % of the C5 apply's warp samples, ncu). Same copies, same order of
// arrival per destination: the result is bitwise that of async_own + async_nbr.
#ifndef DG_FUSED_TILES
#define DG_FUSED_TILES 2   // 1: the four neighbour tiles fused, 2: the own tile too (C5 apply 742 / 700 / 643 us)
#endif
template <int N> __host__ __device__ constexpr bool fused_tiles() {
  return !(N % 2 == 0 && Geo<N>::FS % 2 == 0) && N <= 3;
}
template <int N, bool OWN, bool WB>
__device__ __forceinline__ void async_tiles5(double* TB, double* FY, double* FX, double* FZ,
                                             const Cells<N, WB>& cl, const KParams& kp,
                                             const double* tile, int nvalid) {
  using G = Geo<N>;
  const long sy = (long)kp.nx * G::N3, sz = (long)kp.nx * kp.ny * G::N3;
  const double* s2 = tile - sy;
  const double* s3 = tile + sy;
  const double* s4 = tile - sz;
  const double* s5 = tile + sz;
  const unsigned m20 = cl.nbm[2][0], m21 = cl.nbm[2][1], m30 = cl.nbm[3][0], m31 = cl.nbm[3][1];
  const unsigned m40 = cl.nbm[4][0], m41 = cl.nbm[4][1], m50 = cl.nbm[5][0], m51 = cl.nbm[5][1];
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    if (e < G::C * G::N3) {
      const int cs = e / G::N3, r = e % G::N3;
      const int oT = cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2);
      const int oF = cs * G::FS + r;
      auto bit = [&](unsigned a, unsigned b) { return ((cs < 32 ? a >> cs : b >> (cs - 32)) & 1u) != 0; };
      const bool own = cs < nvalid, k2 = bit(m20, m21), k3 = bit(m30, m31), k4 = bit(m40, m41), k5 = bit(m50, m51);
      if (OWN) cp_async8(TB + oT, tile + (own ? e : 0), own);
      cp_async8(TB + G::ARR + oT, k2 ? s2 + e : tile, k2);
      cp_async8(FY + oF, k3 ? s3 + e : tile, k3);
      cp_async8(FX + oF, k4 ? s4 + e : tile, k4);
      cp_async8(FZ + oF, k5 ? s5 + e : tile, k5);
    }
  }
}

// own tile (contiguous in global) -> TB layout, half h
template <int N, bool ROLL = false>
__device__ __forceinline__ void async_own(double* TB, const double* __restrict__ src, int nvalid) {
  using G = Geo<N>;
#pragma unroll (ROLL ? 1 : 64)
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    if (e < G::C * G::N3) {
      const int cs = e / G::N3, r = e % G::N3;
      cp_async8(TB + cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2), src + (cs < nvalid ? e : 0), cs < nvalid);
    }
  }
}
// solvers: a tile into the TB layout; at n = 4 through rolled cp.async copies (code size: the
// solver prologue / epilogue share the instruction cache with the iteration loop)
template <int N>
__device__ __forceinline__ void stage_tile_s(double* TB, const double* __restrict__ src, int nvalid) {
  if constexpr (N == 4) {
    async_own<N, true>(TB, src, nvalid);
    cp_async_wait_all();
  } else {
    stage_tile<N>(TB, src, nvalid);
  }
}
// face-f neighbour tiles: into TB layout (KSX = KS, cell stride CTB) or into a face region
// (KSX = N2, cell stride FS >= N3)
// fast path (no ghost-layer neighbour on face f): the neighbour tile is the group's own tile
// shifted by +- step cells, so the sources are contiguous and no per-cell pointer is loaded
template <int N, int KSX, int CSX, bool ROLL = false, bool WB>
__device__ __forceinline__ void async_nbr(double* dst, const Cells<N, WB>& cl, int f, const double* any,
                                          const KParams& kp, const double* tile) {
  using G = Geo<N>;
  if (cl.nbg[f] == 0) {
    const unsigned m0 = cl.nbm[f][0], m1 = cl.nbm[f][1];
    const long step = (f >> 1) == 0 ? 1 : ((f >> 1) == 1 ? kp.nx : (long)kp.nx * kp.ny);
    const double* src = tile + ((f & 1) ? step : -step) * (long)G::N3;
    if constexpr (N % 2 == 0 && CSX % 2 == 0 && KSX % 2 == 0) {
      // element pairs (same cell and plane, 16-byte aligned on both sides)
      static_assert((G::C * G::N3 / 2) % G::NT == 0, "pairs tile the group evenly");
#pragma unroll (ROLL ? 1 : 64)
      for (int m = 0; m < G::C * G::N3 / 2 / G::NT; ++m) {
        const int e = 2 * (threadIdx.x + m * G::NT);
        const int cs = e / G::N3, r = e % G::N3;
        const bool ok = ((cs < 32 ? m0 >> cs : m1 >> (cs - 32)) & 1u) != 0;
        cp_async16(dst + cs * CSX + (r / G::N2) * KSX + (r % G::N2), ok ? src + e : any, ok);
      }
      return;
    }
#pragma unroll (ROLL ? 1 : 64)
    for (int m = 0; m < G::PER; ++m) {
      const int e = threadIdx.x + m * G::NT;
      if (e < G::C * G::N3) {
        const int cs = e / G::N3, r = e % G::N3;
        const bool ok = ((cs < 32 ? m0 >> cs : m1 >> (cs - 32)) & 1u) != 0;
        cp_async8(dst + cs * CSX + (r / G::N2) * KSX + (r % G::N2), ok ? src + e : any, ok);
      }
    }
    return;
  }
#pragma unroll (ROLL ? 1 : 64)
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    if (e < G::C * G::N3) {
      const int cs = e / G::N3, r = e % G::N3;
      // (a ghost trace record, z faces at a slab boundary, fills planes 0 and 1; the rest of the
      // n^3 copy reads the next record or the buffer's padding and is never used)
      const double* p = cl.nb[cs][f];
      cp_async8(dst + cs * CSX + (r / G::N2) * KSX + (r % G::N2), p ? p + r : any, p != nullptr);
    }
  }
}

// y-face traces of the neighbour on side `hi` (plane k of the neighbour, nodal in i), lane k:
// out[0..N) = S row (k, i), out[N..2N) = T row (k, i)
template <int N, int KSX>
__device__ __forceinline__ void ytrace(const double* nb, const double* c, double ih, int hi, int k,
                                       double (&S)[N], double (&T)[N]) {
  const double cna = c[2], cng = c[3], ctn = c[5];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double g = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) g = fma(hi ? c_tab[N].d0[j] : c_tab[N].d1[j], nb[k * KSX + j * N + i], g);
    const double a = nb[k * KSX + (hi ? 0 : N - 1) * N + i];
    S[i] = cna * a + cng * g * ih;
    T[i] = ctn * a;
  }
}
// z-face traces (lane t = y node j): rows (kk, i) of the neighbour at fixed j, interpolated in x
// tr: nb is a ghost trace record (plane 0 the face values, plane 1 the derivative sums); both
// paths share the flux arithmetic below, so a slab-boundary face is bitwise the in-slab one
template <int N, int KSX>
__device__ __forceinline__ void ztrace(const double* nb, const double* c, double ih, int hi, int j,
                                       double (&S)[N], double (&T)[N], bool tr = false) {
  const double cna = c[2], cng = c[3], ctn = c[5];
  double s0[N], t0[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double g = 0.0;
    if (tr) {
      g = nb[KSX + j * N + i];
    } else {
#pragma unroll
      for (int kk = 0; kk < N; ++kk) g = fma(hi ? c_tab[N].d0[kk] : c_tab[N].d1[kk], nb[kk * KSX + j * N + i], g);
    }
    const double a = nb[(tr ? 0 : (hi ? 0 : N - 1)) * KSX + j * N + i];
    s0[i] = cna * a + cng * g * ih;
    t0[i] = ctn * a;
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double ss = 0.0, tt = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      ss = fma(T_A<N>(q * N + i), s0[i], ss);
      tt = fma(T_A<N>(q * N + i), t0[i], tt);
    }
    S[q] = ss;
    T[q] = tt;
  }
}
// x-face traces (lane k): rows (k, j) of the neighbour's plane k, interpolated in y
template <int N>
__device__ __forceinline__ void xtrace(const double* plane, const double* c, double ih, int hi,
                                       double (&S)[N], double (&T)[N]) {
  const double cna = c[2], cng = c[3], ctn = c[5];
  double s0[N], t0[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double row[N];
#pragma unroll
    for (int i = 0; i < N; ++i) row[i] = plane ? plane[j * N + i] : 0.0;
    double g = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) g = fma(hi ? c_tab[N].d0[i] : c_tab[N].d1[i], row[i], g);
    const double a = hi ? row[0] : row[N - 1];
    s0[j] = cna * a + cng * g * ih;
    t0[j] = ctn * a;
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    double ss = 0.0, tt = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      ss = fma(T_A<N>(q * N + j), s0[j], ss);
      tt = fma(T_A<N>(q * N + j), t0[j], tt);
    }
    S[q] = ss;
    T[q] = tt;
  }
}

// Neighbour prologue over the asynchronously staged tiles: own in TB half 0, y-lo in TB half 1,
// y-hi / z-lo / z-hi in the FY / FX / FZ regions (cell stride FS, plane stride N2). The z and x
// traces are taken first and written over the z staging, then the y traces over the y-hi
// staging. Leaves TB free. All threads must call it (three barriers).
template <int N, bool GH, bool WB>
__device__ void nbr_prologue_async(const KParams& kp, const Cells<N, WB>& cl, const Lane& L,
                                   double* TB, double* FY, double* FX, double* FZ, const double* tile) {
  using G = Geo<N>;
  static_assert(G::FS >= G::N3, "a face region must hold one staged tile");
  const int t = L.t;
  {
    double xs[2][2][N], zs[2][2][N];
    if (L.active) {
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        // x: the neighbour is the next / previous cell of the group (its tile is in TB half 0)
        // unless the group ends there; then its plane t is read from global memory
        const double* nbp = cl.nb[L.cs][hi];
        const int ncs = L.cs + (hi ? 1 : -1);
        const double* plane = nullptr;
        if (nbp) {
          if (ncs >= 0 && ncs < G::C && nbp == tile + (size_t)ncs * G::N3)
            plane = TB + ncs * G::CTB + t * G::KS;
          else
            plane = nbp + t * G::N2;
        }
        xtrace<N>(plane, cl.fc[L.cs][hi], kp.ih[0], hi, xs[hi][0], xs[hi][1]);
        ztrace<N, G::N2>((hi ? FZ : FX) + L.cs * G::FS, cl.fc[L.cs][4 + hi], kp.ih[2], hi, t,
                         zs[hi][0], zs[hi][1], GH && ghost_trace(kp, cl.cell[L.cs], hi));
      }
    }
    __syncthreads();   // z staging consumed
    if (L.active) {
#pragma unroll
      for (int hi = 0; hi < 2; ++hi)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            FX[L.cs * G::FS + (2 * hi + a) * G::N2 + t * N + q] = xs[hi][a][q];
            FZ[L.cs * G::FS + (2 * hi + a) * G::N2 + t * N + q] = zs[hi][a][q];
          }
    }
  }
  {
    double ys[2][2][N];
    if (L.active) {
      ytrace<N, G::KS>(TB + L.cs * G::CTB + G::ARR, cl.fc[L.cs][2], kp.ih[1], 0, t, ys[0][0], ys[0][1]);
      ytrace<N, G::N2>(FY + L.cs * G::FS, cl.fc[L.cs][3], kp.ih[1], 1, t, ys[1][0], ys[1][1]);
    }
    __syncthreads();   // y-hi staging consumed
    if (L.active) {
#pragma unroll
      for (int hi = 0; hi < 2; ++hi)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int i = 0; i < N; ++i) FY[L.cs * G::FS + (2 * hi + a) * G::N2 + t * N + i] = ys[hi][a][i];
    }
  }
  __syncthreads();
}

// ---- the operator: out = A u (NBR) or D_T u (self faces only) on the lane's plane ---------
// All lanes of the warp must call it (two __syncwarp inside: a cell's n lanes are in one warp,
// so both transposes are warp-local). The cell's TB / FY slots must be free on entry.
// The quadrature-point residual R is kept UNWEIGHTED: the Gauss weights (and |T|, face
// areas through kp) are folded into the transposed 1D tables AW = A w, GW = G w,
// DW = D w_q / w_r and the end-point injection vectors E/w, F/w.
// GEN = false: pure diffusion (b = 0, no reaction), the convective and reaction terms are
// compiled out (the b = 0 / c = 0 configurations C1-C3, C5).
template <int N, bool NBR, bool USEB, bool FACES = true, bool GEN = true, bool WB>
__device__ __forceinline__ void plane_op(const KParams& kp, const Cells<N, WB>& cl, const Lane& L,
                                         const Rows<N>& rw, bool vol, const double (&in)[N][N],
                                         double (&out)[N][N], double* TB, double* FY,
                                         const double* FX, const double* FZ) {
  using G = Geo<N>;
  double* tb = TB + L.cs * G::CTB;
  double* fy = FY + L.cs * G::FS;
  const double* fc = &cl.fc[L.cs][0][0];
  __syncwarp();   // the previous call's Q3 reads of TB / FY (other lanes of the cell) are done
  // ---------------- Q1: lane = z node k ----------------
  if (L.active) {
    const int k = L.t;
    {  // Stage 1 in the plane: a = A_x u; t2 = A_y a (always, for the face traces); t2y = G_y a
      double a[N][N];
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) s = fma(T_A<N>(q * N + i), in[j][i], s);
          a[j][q] = s;
        }
      // the y terms of the volume (constant coefficients on the affine cell): the exact 1D
      // stiffness / convection matrices along y, nodal to nodal (Shat = G^T W G,
      // Chat = G^T W A), scaled by the cell's |T| K_y / h_y^2 and |T| b_y / h_y; Q2 adds the
      // z mass and Q3 the result without a G_y^T contraction (index qy stands for node j there)
      const double cKy = cl.vc[L.cs][1], cBy = cl.vb[L.cs][1];
#pragma unroll
      for (int qx = 0; qx < N; ++qx)
#pragma unroll
        for (int qy = 0; qy < N; ++qy) {
          double s = 0.0, sy = 0.0, cy = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            s = fma(T_A<N>(qy * N + j), a[j][qx], s);
            sy = fma(c_tab[N].S[qy * N + j], a[j][qx], sy);
            if constexpr (GEN) cy = fma(c_tab[N].Cm[qy * N + j], a[j][qx], cy);
          }
          tb[k * G::KS + qy * N + qx] = s;
          if (vol) tb[G::ARR + k * G::KS + qy * N + qx] = GEN ? fma(cKy, sy, -cBy * cy) : cKy * sy;
        }
    }
    // y faces (normal y; tangential z = this lane, x): nodal S/T combos, then A_x
    if constexpr (FACES) {
    const double* clo = fc + 2 * 6;
    const double* chi = fc + 3 * 6;
    double X0[N], X1[N], X2[N], X3[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double glo = 0.0, ghi = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        glo = fma(c_tab[N].d0[j], in[j][i], glo);
        ghi = fma(c_tab[N].d1[j], in[j][i], ghi);
      }
      const double alo = in[0][i], ahi = in[N - 1][i];
      X0[i] = fma(clo[0], alo, clo[1] * glo * kp.ih[1]);
      X1[i] = clo[4] * alo;
      X2[i] = fma(chi[0], ahi, chi[1] * ghi * kp.ih[1]);
      X3[i] = chi[4] * ahi;
      if (NBR) {
        X0[i] += fy[0 * G::N2 + k * N + i];
        X1[i] += fy[1 * G::N2 + k * N + i];
        X2[i] += fy[2 * G::N2 + k * N + i];
        X3[i] += fy[3 * G::N2 + k * N + i];
      }
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double A = T_A<N>(q * N + i);
        s0 = fma(A, X0[i], s0);
        s1 = fma(A, X1[i], s1);
        s2 = fma(A, X2[i], s2);
        s3 = fma(A, X3[i], s3);
      }
      fy[0 * G::N2 + k * N + q] = s0;
      fy[1 * G::N2 + k * N + q] = s1;
      fy[2 * G::N2 + k * N + q] = s2;
      fy[3 * G::N2 + k * N + q] = s3;
    }
    }
  }
  __syncwarp();   // the transposes stay inside the cell's own warp
  // ---------------- Q2: lane = y Gauss point qy ----------------
  if (L.active) {
    const int qy = L.t;
    const double* vcell = cl.vc[L.cs];
    const double* vbc = cl.vb[L.cs];
    double U[N][N], R[N][N];   // [qz][qx], unweighted
    if (vol) {
      // U = A_z t2, Uy = A_z t2y; Stage 2 for the reaction and the y flux pointwise; the y flux
      // column goes straight through (A w)_z^T into TB (its t2y column has just been read)
      const double cR = vcell[3];
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double c0[N], c1[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          c0[k] = tb[k * G::KS + qy * N + qx];
          c1[k] = tb[G::ARR + k * G::KS + qy * N + qx];
        }
        // U at the Gauss points (+ the reaction), and the y terms (c1: (K_y Shat - b_y Chat)_y a
        // from Q1) through the exact z mass: (Mhat_z (x) (K_y Shat - b_y Chat)_y) on the
        // x-Gauss / y,z-nodal values; Q3 adds them without a G_y^T contraction
#pragma unroll
        for (int qz = 0; qz < N; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(T_A<N>(qz * N + k), c0[k], s);
          U[qz][qx] = s;
          R[qz][qx] = GEN ? cR * s : 0.0;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double s = 0.0;
#pragma unroll
          for (int kk = 0; kk < N; ++kk) s = fma(c_tab[N].M[k * N + kk], c1[kk], s);
          tb[G::ARR + k * G::KS + qy * N + qx] = s;
        }
      }
      if constexpr (!GEN) {
        // pure diffusion: the coefficient is constant along each line, so the derivative pair
        // DW^T (sK D U) is one Gauss-point stiffness matvec sK (SGW U), SGW = DW^T D
#pragma unroll
        for (int qz = 0; qz < N; ++qz)
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s = fma(T_SGW<N>(r * N + q), U[qz][q], s);
            R[qz][r] = fma(vcell[0], s, R[qz][r]);
          }
#pragma unroll
        for (int qx = 0; qx < N; ++qx)
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s = fma(T_SGW<N>(r * N + q), U[q][qx], s);
            R[r][qx] = fma(vcell[2], s, R[r][qx]);
          }
      } else {
      // x direction: rows qz;  R += DW^T (sK D U - sb U)
#pragma unroll
      for (int qz = 0; qz < N; ++qz) {
        double F[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double du = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r) du = fma(T_D<N>(q * N + r), U[qz][r], du);
          F[q] = fma(vcell[0], du, -vbc[0] * U[qz][q]);
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double s = R[qz][r];
#pragma unroll
          for (int q = 0; q < N; ++q) s = fma(T_DW<N>(q * N + r), F[q], s);
          R[qz][r] = s;
        }
      }
      // z direction: columns qx
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double F[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double du = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r) du = fma(T_D<N>(q * N + r), U[r][qx], du);
          F[q] = fma(vcell[2], du, -vbc[2] * U[q][qx]);
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double s = R[r][qx];
#pragma unroll
          for (int q = 0; q < N; ++q) s = fma(T_DW<N>(q * N + r), F[q], s);
          R[r][qx] = s;
        }
      }
      }
    } else {
      // faces only: U still needed for the traces
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double c0[N];
#pragma unroll
        for (int k = 0; k < N; ++k) c0[k] = tb[k * G::KS + qy * N + qx];
#pragma unroll
        for (int qz = 0; qz < N; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(T_A<N>(qz * N + k), c0[k], s);
          U[qz][qx] = s;
          R[qz][qx] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) tb[G::ARR + k * G::KS + qy * N + qx] = 0.0;
      }
    }
    if constexpr (!FACES) {
    } else if (!USEB) {
      // x faces at the face Gauss points (qz, qy): traces from the x-rows of U
      const double* clo = fc + 0 * 6;
      const double* chi = fc + 1 * 6;
      const double* fx = FX + L.cs * G::FS;
#pragma unroll
      for (int qz = 0; qz < N; ++qz) {
        double alo = 0.0, ahi = 0.0, glo = 0.0, ghi = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          alo = fma(c_tab[N].E0[q], U[qz][q], alo);
          ahi = fma(c_tab[N].E1[q], U[qz][q], ahi);
          glo = fma(c_tab[N].F0[q], U[qz][q], glo);
          ghi = fma(c_tab[N].F1[q], U[qz][q], ghi);
        }
        double Slo = fma(clo[0], alo, clo[1] * glo * kp.ih[0]), Tlo = clo[4] * alo;
        double Shi = fma(chi[0], ahi, chi[1] * ghi * kp.ih[0]), Thi = chi[4] * ahi;
        if (NBR) {  // neighbour traces at (k, qy) -> interpolate in z
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double A = T_A<N>(qz * N + k);
            Slo = fma(A, fx[0 * G::N2 + k * N + qy], Slo);
            Tlo = fma(A, fx[1 * G::N2 + k * N + qy], Tlo);
            Shi = fma(A, fx[2 * G::N2 + k * N + qy], Shi);
            Thi = fma(A, fx[3 * G::N2 + k * N + qy], Thi);
          }
        }
        const double fa = kp.fa[0];
        Slo *= fa; Tlo *= fa; Shi *= fa; Thi *= fa;
#pragma unroll
        for (int q = 0; q < N; ++q)
          R[qz][q] += fma(c_tab[N].E0W[q], Slo,
                          fma(c_tab[N].F0W[q], Tlo, fma(c_tab[N].E1W[q], Shi, c_tab[N].F1W[q] * Thi)));
      }
      // z faces at the face Gauss points (qy, qx): traces from the z-columns of U
      const double* zlo = fc + 4 * 6;
      const double* zhi = fc + 5 * 6;
      const double* fz = FZ + L.cs * G::FS;
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double alo = 0.0, ahi = 0.0, glo = 0.0, ghi = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          alo = fma(c_tab[N].E0[q], U[q][qx], alo);
          ahi = fma(c_tab[N].E1[q], U[q][qx], ahi);
          glo = fma(c_tab[N].F0[q], U[q][qx], glo);
          ghi = fma(c_tab[N].F1[q], U[q][qx], ghi);
        }
        double Slo = fma(zlo[0], alo, zlo[1] * glo * kp.ih[2]), Tlo = zlo[4] * alo;
        double Shi = fma(zhi[0], ahi, zhi[1] * ghi * kp.ih[2]), Thi = zhi[4] * ahi;
        if (NBR) {  // neighbour traces at (j, qx) -> interpolate in y (row qy of A)
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double A = rw.Arow[j];
            Slo = fma(A, fz[0 * G::N2 + j * N + qx], Slo);
            Tlo = fma(A, fz[1 * G::N2 + j * N + qx], Tlo);
            Shi = fma(A, fz[2 * G::N2 + j * N + qx], Shi);
            Thi = fma(A, fz[3 * G::N2 + j * N + qx], Thi);
          }
        }
        const double fb = kp.fa[2];
        Slo *= fb; Tlo *= fb; Shi *= fb; Thi *= fb;
#pragma unroll
        for (int q = 0; q < N; ++q)
          R[q][qx] += fma(c_tab[N].E0W[q], Slo,
                          fma(c_tab[N].F0W[q], Tlo, fma(c_tab[N].E1W[q], Shi, c_tab[N].F1W[q] * Thi)));
      }
    } else {
      // x and z self faces: the per-cell Gauss-point operators B (rows / columns of U), read
      // from shared memory at the point of use (broadcast within the cell's lanes)
      const double* Bc = cl.B[L.cs];
#pragma unroll
      for (int q = 0; q < N; ++q)
#pragma unroll
        for (int r = 0; r < N; ++r) {
          const double bx = Bc[q * N + r];
#pragma unroll
          for (int qz = 0; qz < N; ++qz) R[qz][q] = fma(bx, U[qz][r], R[qz][q]);
        }
#pragma unroll
      for (int q = 0; q < N; ++q)
#pragma unroll
        for (int r = 0; r < N; ++r) {
          const double bz = Bc[G::N2 + q * N + r];
#pragma unroll
          for (int qx = 0; qx < N; ++qx) R[q][qx] = fma(bz, U[r][qx], R[q][qx]);
        }
    if (NBR) {
      // neighbour traces of the x faces at (k, qy) -> interpolate in z; inject through A^-T / w
      const double* fx = FX + L.cs * G::FS;
      const double fa = kp.fa[0];
#pragma unroll
      for (int qz = 0; qz < N; ++qz) {
        double Slo = 0.0, Tlo = 0.0, Shi = 0.0, Thi = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double A = T_A<N>(qz * N + k);
          Slo = fma(A, fx[0 * G::N2 + k * N + qy], Slo);
          Tlo = fma(A, fx[1 * G::N2 + k * N + qy], Tlo);
          Shi = fma(A, fx[2 * G::N2 + k * N + qy], Shi);
          Thi = fma(A, fx[3 * G::N2 + k * N + qy], Thi);
        }
        Slo *= fa; Tlo *= fa; Shi *= fa; Thi *= fa;
#pragma unroll
        for (int q = 0; q < N; ++q)
          R[qz][q] += fma(c_tab[N].E0W[q], Slo,
                          fma(c_tab[N].F0W[q], Tlo, fma(c_tab[N].E1W[q], Shi, c_tab[N].F1W[q] * Thi)));
      }
      // neighbour traces of the z faces at (j, qx) -> interpolate in y (row qy of A)
      const double* fz = FZ + L.cs * G::FS;
      const double fb = kp.fa[2];
#pragma unroll
      for (int qx = 0; qx < N; ++qx) {
        double Slo = 0.0, Tlo = 0.0, Shi = 0.0, Thi = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double A = rw.Arow[j];
          Slo = fma(A, fz[0 * G::N2 + j * N + qx], Slo);
          Tlo = fma(A, fz[1 * G::N2 + j * N + qx], Tlo);
          Shi = fma(A, fz[2 * G::N2 + j * N + qx], Shi);
          Thi = fma(A, fz[3 * G::N2 + j * N + qx], Thi);
        }
        Slo *= fb; Tlo *= fb; Shi *= fb; Thi *= fb;
#pragma unroll
        for (int q = 0; q < N; ++q)
          R[q][qx] += fma(c_tab[N].E0W[q], Slo,
                          fma(c_tab[N].F0W[q], Tlo, fma(c_tab[N].E1W[q], Shi, c_tab[N].F1W[q] * Thi)));
      }
    }
    }
    // (A w)_z^T on R, stored in place of t2 (same index set (., qy, .))
#pragma unroll
    for (int qx = 0; qx < N; ++qx)
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double s = 0.0;
#pragma unroll
        for (int qz = 0; qz < N; ++qz) s = fma(T_AW<N>(qz * N + k), R[qz][qx], s);
        tb[k * G::KS + qy * N + qx] = s;
      }
  }
  __syncwarp();
  // ---------------- Q3: lane = z node k ----------------
  if (L.active) {
    const int k = L.t;
    double Vq[N][N];   // [j][qx]
#pragma unroll
    for (int qx = 0; qx < N; ++qx) {
      double r[N], f[N];
#pragma unroll
      for (int qy = 0; qy < N; ++qy) {
        r[qy] = tb[k * G::KS + qy * N + qx];
        f[qy] = tb[G::ARR + k * G::KS + qy * N + qx];
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s = f[j];   // the y terms are already nodal in j
#pragma unroll
        for (int qy = 0; qy < N; ++qy) s = fma(T_AW<N>(qy * N + j), r[qy], s);
        Vq[j][qx] = s;
      }
    }
    // y faces: z face mass (row k of Mhat) on the (k', qx) arrays, end profiles in j
#pragma unroll
    for (int qx = 0; qx < N && FACES; ++qx) {
      double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        const double M = rw.Mrow[kk];
        z0 = fma(M, fy[0 * G::N2 + kk * N + qx], z0);
        z1 = fma(M, fy[1 * G::N2 + kk * N + qx], z1);
        z2 = fma(M, fy[2 * G::N2 + kk * N + qx], z2);
        z3 = fma(M, fy[3 * G::N2 + kk * N + qx], z3);
      }
      const double fa = kp.fa[1];
      z0 *= fa; z1 *= fa; z2 *= fa; z3 *= fa;
      Vq[0][qx] += z0;
      Vq[N - 1][qx] += z2;
#pragma unroll
      for (int j = 0; j < N; ++j) Vq[j][qx] = fma(c_tab[N].d0[j], z1, fma(c_tab[N].d1[j], z3, Vq[j][qx]));
    }
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int qx = 0; qx < N; ++qx) s = fma(T_AW<N>(qx * N + i), Vq[j][qx], s);
        out[j][i] = s;
      }
  }
}

// 1 / diag(D_T) on the lane's plane (Jacobi preconditioner), from 1D diagonals
// 1 / d from the hardware approximation and two Newton steps (a handful of instructions where
// an IEEE division expands to ~35): used for the Jacobi preconditioners only, where any fixed
// diagonal scaling is valid and the last bit does not matter (the solvers' code size does).
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
// Krylov scalars of the plane solvers: a * (1 / b) with rcp_nr (~1 ulp; the IEEE division is
// ~35 instructions inside loops that must stay within the instruction cache). DG_EXACT_QUOT=1:
// IEEE division (A/B).
#ifndef DG_EXACT_QUOT
#define DG_EXACT_QUOT 0
#endif
#if DG_EXACT_QUOT
#define DG_QUOT(a, b) ((a) / (b))
#else
#define DG_QUOT(a, b) ((a) * rcp_nr(b))
#endif
template <int N>
__device__ __forceinline__ void plane_inv_diag(const KParams& kp, const Cells<N>& cl, const Lane& L,
                                               const Rows<N>& rw, double (&dg)[N][N]) {
  const double* vc = cl.vc[L.cs];
  const double* vb = cl.vb[L.cs];
  const double* fc = &cl.fc[L.cs][0][0];
  const int k = L.t;
  const double dd0 = c_tab[N].d0[0], dd1 = c_tab[N].d1[N - 1];
  auto fd = [&](int f, double dd, double ih) {
    const double* c = fc + f * 6;
    return c[0] + c[1] * dd * ih + c[4] * dd;
  };
  const double zlo = (k == 0) ? fd(4, dd0, kp.ih[2]) : 0.0;
  const double zhi = (k == N - 1) ? fd(5, dd1, kp.ih[2]) : 0.0;
  const double xlo = fd(0, dd0, kp.ih[0]), xhi = fd(1, dd1, kp.ih[0]);
  const double ylo = fd(2, dd0, kp.ih[1]), yhi = fd(3, dd1, kp.ih[1]);
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double Mi = c_tab[N].Md[i], Mj = c_tab[N].Md[j], Mk = rw.Md;
      double d = vc[3] * Mi * Mj * Mk;
      d += (vc[0] * c_tab[N].Sd[i] - vb[0] * c_tab[N].Cd[i]) * Mj * Mk;
      d += (vc[1] * c_tab[N].Sd[j] - vb[1] * c_tab[N].Cd[j]) * Mi * Mk;
      d += (vc[2] * rw.Sd - vb[2] * rw.Cd) * Mi * Mj;
      if (i == 0) d += kp.fa[0] * Mj * Mk * xlo;
      if (i == N - 1) d += kp.fa[0] * Mj * Mk * xhi;
      if (j == 0) d += kp.fa[1] * Mi * Mk * ylo;
      if (j == N - 1) d += kp.fa[1] * Mi * Mk * yhi;
      d += kp.fa[2] * Mi * Mj * (zlo + zhi);
      dg[j][i] = rcp_nr(d);
    }
}

// ---- group setup in two halves ------------------------------------------------------------
// setup_issue: one thread per (cell, axis) writes the two neighbour pointers of that axis and
// issues the loads of K_T, K of both neighbours (and c) into registers; after a barrier the
// caller issues its neighbour-tile loads, which are then in flight together with these;
// setup_finish turns the registers into the volume scalings vc and face coefficients fc
// (harmonic weights, penalty gamma_F = alpha p(p+2) <delta>|F|/|T|, upwind b_nu).
template <int N> struct SetupRegs {
  static constexpr int C = Geo<N>::C, NT = Geo<N>::NT;
  static constexpr int IT = (3 * C + NT - 1) / NT;   // (cell, axis) items per thread
  double KT[IT], Kn[IT][2], cR[IT];
  double bT[IT], bN[IT][2];   // b_axis of the cell and of its two neighbours along the axis
  int kind[IT][2];   // 0 interior (or ghost), 1 Dirichlet, 2 Neumann; -1: item not valid
};

// zero the neighbour masks (call before setup_issue, followed by a barrier)
template <int N, bool WB> __device__ __forceinline__ void clear_masks(Cells<N, WB>& cl) {
  if (threadIdx.x < 12) (&cl.nbm[0][0])[threadIdx.x] = 0u;
  if (threadIdx.x < 6) cl.nbg[threadIdx.x] = 0;
}

template <int N, bool CMAP = false, bool WB>
__device__ __forceinline__ void setup_issue(const KParams& kp, Cells<N, WB>& cl, SetupRegs<N>& sr,
                                            int cell0, const double* u) {
  using G = Geo<N>;
  const int nxy = kp.nx * kp.ny;
  const int c0x = cell0 % kp.nx, c0y = (cell0 / kp.nx) % kp.ny, c0z = cell0 / nxy;
#pragma unroll
  for (int r = 0; r < SetupRegs<N>::IT; ++r) {
    const int it = threadIdx.x + r * G::NT;
    const int cs = it / 3, axis = it % 3;
    const int cell = CMAP ? group_cell(kp, cell0, cs) : (cell0 + cs < kp.ncells ? cell0 + cs : -1);
    sr.kind[r][0] = sr.kind[r][1] = -1;
    if (it >= 3 * G::C) continue;
    if (axis == 0) cl.cell[cs] = cell;
    if (cell < 0) {
      cl.nb[cs][2 * axis] = cl.nb[cs][2 * axis + 1] = nullptr;
      continue;
    }
    int cx, cy, cz;
    if (CMAP) {
      cx = cell % kp.nx;
      cy = (cell / kp.nx) % kp.ny;
      cz = cell / nxy;
    } else {
      cx = c0x + cs; cy = c0y; cz = c0z;
      while (cx >= kp.nx) { cx -= kp.nx; ++cy; }
      while (cy >= kp.ny) { cy -= kp.ny; ++cz; }
    }
    const int co = axis == 0 ? cx : (axis == 1 ? cy : cz);
    const int dim = axis == 0 ? kp.nx : (axis == 1 ? kp.ny : kp.nzl);
    const int step = axis == 0 ? 1 : (axis == 1 ? kp.nx : nxy);
    sr.KT[r] = __ldg(kp.K + (size_t)(cell + nxy) * 3 + axis);
    sr.cR[r] = (axis == 0 && kp.c) ? __ldg(kp.c + cell) : 0.0;
    sr.bT[r] = kp.bc ? __ldg(kp.bc + (size_t)(cell + nxy) * 3 + axis) : kp.b[axis];
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const int f = 2 * axis + hi;
      const int nc = co + (hi ? 1 : -1);
      const double* nbp = nullptr;
      long kidx = -1;
      int kind;
      if (nc >= 0 && nc < dim) {
        kind = 0;
        const long nb = cell + (hi ? step : -step);
        kidx = nb + nxy;
        if (u) nbp = u + (size_t)nb * G::N3;
      } else if (kp.slab_face[f] == FK_GHOST) {
        kind = 0;
        const int col = cx + kp.nx * cy;
        kidx = hi ? (long)(kp.nzl + 1) * nxy + col : col;
        if (u) nbp = (hi ? kp.ghost_hi : kp.ghost_lo) + (size_t)col * 2 * G::N2;   // trace record
      } else {
        kind = kp.slab_face[f] == FK_DIRICHLET ? 1 : 2;
      }
      sr.kind[r][hi] = kind;
      sr.Kn[r][hi] = kidx >= 0 ? __ldg(kp.K + (size_t)kidx * 3 + axis) : 0.0;
      sr.bN[r][hi] = (kp.bc && kidx >= 0) ? __ldg(kp.bc + (size_t)kidx * 3 + axis) : sr.bT[r];
      cl.nb[cs][f] = nbp;
      if (nc >= 0 && nc < dim) atomicOr(&cl.nbm[f][cs >> 5], 1u << (cs & 31));
      if ((kind == 0 && !(nc >= 0 && nc < dim)) || CMAP) cl.nbg[f] = 1;   // per-cell pointers
    }
  }
}

template <int N, bool WB>
__device__ __forceinline__ void setup_finish(const KParams& kp, Cells<N, WB>& cl,
                                             const SetupRegs<N>& sr) {
  using G = Geo<N>;
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
#pragma unroll
  for (int r = 0; r < SetupRegs<N>::IT; ++r) {
    const int it = threadIdx.x + r * G::NT;
    const int cs = it / 3, axis = it % 3;
    if (it >= 3 * G::C) continue;
    const bool valid = sr.kind[r][0] >= 0;
    const double ihk = kp.ih[axis];
    const double KT = valid ? sr.KT[r] : 0.0;
    cl.vc[cs][axis] = (valid && (kp.mask & 1u)) ? KT * vol * ihk * ihk : 0.0;
    if (axis == 0) cl.vc[cs][3] = (valid && (kp.mask & 1u)) ? vol * sr.cR[r] : 0.0;
    cl.vb[cs][axis] = (valid && (kp.mask & 1u)) ? vol * sr.bT[r] * ihk : 0.0;
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      double co[6] = {0, 0, 0, 0, 0, 0};
      const int kind = sr.kind[r][hi];
      // b . nu_F on the face (reading #8: the mean of the two cells' b; exact for constant b)
      const double bn = kind == 0 ? 0.5 * (sr.bT[r] + sr.bN[r][hi]) : sr.bT[r];
      if (kind == 0 && (kp.mask & 2u)) {
        const double KN = sr.Kn[r][hi];
        const double sum = KT + KN;
        const double rs = sum > 0.0 ? rcp_nr(sum) : 0.0;   // ~1 ulp (code size: see rcp_nr)
        const double wT = sum > 0.0 ? KN * rs : 0.5, wN = sum > 0.0 ? KT * rs : 0.5;
        const double gam = kp.pen * (2.0 * KT * KN * rs) * ihk;   // <dT,dN>|F|/|T|
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
        const double gam = kp.pen * KT * ihk;   // delta |F| / |T|
        if (hi) { co[0] = fmax(bn, 0.0) + gam;  co[1] = -KT; co[4] = -KT * ihk; }
        else    { co[0] = fmax(-bn, 0.0) + gam; co[1] = KT;  co[4] = KT * ihk; }
      }
#pragma unroll
      for (int e = 0; e < 6; ++e) cl.fc[cs][2 * axis + hi][e] = co[e];
    }
  }
}

// =============================== kernels ================================================
// Self-face operator of the x (z) faces at the Gauss points, unweighted quadrature level:
//   B[q][r] = |F| sum_{s=lo,hi} ( E_s^w[q] (cs_a E_s[r] + cs_g F_s[r] / h) + F_s^w[q] ct_a E_s[r] ),
// i.e. traces a_s = E_s.U, g_s = F_s.U of a Gauss-value line U, the flux combinations
// S = cs_a a + cs_g g / h, T = ct_a a, and their injection through A^-T / w (see plane_op).
template <int N, bool WB> __device__ __forceinline__ void setup_B(const KParams& kp, Cells<N, WB>& cl);

template <int N, bool USEB = true, bool WB>
__device__ __forceinline__ void setup(const KParams& kp, Cells<N, WB>& cl, int cell0, const double* u) {
  using G = Geo<N>;
  setup_cells<N, G::C, G::NT>(kp, cl.vc, cl.vb, cl.fc, cl.nb, cl.cell, cell0, u);
  if constexpr (!USEB || !WB) return;
  setup_B<N>(kp, cl);
}

// the x / z self-face operators B of every cell (needs fc complete); ends with a barrier
template <int N, bool WB>
__device__ __forceinline__ void setup_B(const KParams& kp, Cells<N, WB>& cl) {
  using G = Geo<N>;
  for (int it = threadIdx.x; it < G::C * 2 * G::N2; it += G::NT) {
    const int cs = it / (2 * G::N2), rem = it % (2 * G::N2), d = rem / G::N2;
    const int q = (rem % G::N2) / N, r = rem % N;
    const int axis = d == 0 ? 0 : 2;
    const double* lo = cl.fc[cs][2 * axis];
    const double* hi = cl.fc[cs][2 * axis + 1];
    const double ih = kp.ih[axis];
    double b = c_tab[N].E0W[q] * (lo[0] * c_tab[N].E0[r] + lo[1] * ih * c_tab[N].F0[r]) +
               c_tab[N].F0W[q] * lo[4] * c_tab[N].E0[r];
    b += c_tab[N].E1W[q] * (hi[0] * c_tab[N].E1[r] + hi[1] * ih * c_tab[N].F1[r]) +
         c_tab[N].F1W[q] * hi[4] * c_tab[N].E1[r];
    cl.B[cs][d * G::N2 + q * N + r] = b * kp.fa[axis];
  }
  __syncthreads();
}

// out = A u (with_nbr) or D_T u, selected parts by kp.mask
// FACES = false: the volume terms alone (dg_apply_parts with mask = volume), no face code.
// A u (kp.mask parts) for the lane's plane in the nodal Kronecker-sum form:
//   (A u)_T = Kx (x) Mhat (x) Mhat u_T + Mhat (x) Ky (x) Mhat u_T + Mhat (x) Mhat (x) Kz u_T
//           + sum over the interior faces of (B_F (x) Mhat (x) Mhat) u_N
// (K_a: volume + self faces, formed on the fly by kfly; B_F: the neighbour coupling, through the
// neighbour's face values and normal-derivative sums). In the plane (lane = z node
// k): b = Mhat_x u, c = Kx u + x faces, d = Mhat_y b, g = Ky b + Mhat_y c + y faces (after
// Mhat_x); transpose; (lane = y node j) q = Mhat_z g + Kz d + z faces (after Mhat_x, Mhat_y);
// transpose back. The neighbours come from the tiles staged by the caller (TB half 1: y-lo,
// FY: y-hi, FX: z-lo, FZ: z-hi; x: the group's own tile or global memory); FX then holds the
// contracted z-face arrays. res: the lane's plane of the result.
template <int N, bool GEN, bool WB>
__device__ __forceinline__ void plane_apply_nodal(const KParams& kp, const Cells<N, WB>& cl, const Lane& L,
                                                  double* TB, double* FY, double* FX, double* FZ,
                                                  const double* tile, double (&res)[N][N]) {
  using G = Geo<N>;
  constexpr int N2 = G::N2;
  static_assert(G::FS >= 4 * G::N2, "a face region holds the four contracted z-face arrays");
  constexpr int ZQ = (4 + N - 1) / N;   // z-face arrays per lane
  const int k = L.t, cs = L.cs;
  double u[N][N], xs[4][N], ys[4][N], zs[ZQ][N][N];
  if (L.active) {
    read_plane<N>(TB, L, u);
    // x faces at (j, k): the neighbours' plane k (in the group: the own tile; else global)
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const double* c = cl.fc[cs][hi];
      const double* nbp = cl.nb[cs][hi];
      const int ncs = cs + (hi ? 1 : -1);
      const double* plane = nullptr;
      if (nbp) plane = (ncs >= 0 && ncs < G::C && nbp == tile + (size_t)ncs * G::N3) ? TB + ncs * G::CTB + k * G::KS
                                                                                     : nbp + k * G::N2;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double row[N];
#pragma unroll
        for (int i = 0; i < N; ++i) row[i] = plane ? plane[j * N + i] : 0.0;
        double gn = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) gn = fma(hi ? c_tab[N].d0[i] : c_tab[N].d1[i], row[i], gn);
        const double av = hi ? row[0] : row[N - 1];
        xs[2 * hi][j] = c[2] * av + c[3] * gn * kp.ih[0];
        xs[2 * hi + 1][j] = c[5] * av;
      }
    }
    // y faces at (i, k): the staged y tiles' plane k, then Mhat_x along i
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
      const double* c = cl.fc[cs][2 + hi];
      double S[N], T[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double gn = 0.0, av;
        if (hi) {
          const double* nb = FY + cs * G::FS + k * G::N2;
#pragma unroll
          for (int j = 0; j < N; ++j) gn = fma(c_tab[N].d0[j], nb[j * N + i], gn);
          av = nb[i];
        } else {
          const double* nb = TB + cs * G::CTB + G::ARR + k * G::KS;
#pragma unroll
          for (int j = 0; j < N; ++j) gn = fma(c_tab[N].d1[j], nb[j * N + i], gn);
          av = nb[(N - 1) * N + i];
        }
        S[i] = c[2] * av + c[3] * gn * kp.ih[1];
        T[i] = c[5] * av;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0, t = 0.0;
#pragma unroll
        for (int ip = 0; ip < N; ++ip) {
          s = fma(c_tab[N].M[i * N + ip], S[ip], s);
          t = fma(c_tab[N].M[i * N + ip], T[ip], t);
        }
        ys[2 * hi][i] = s;
        ys[2 * hi + 1][i] = t;
      }
    }
    // z faces: array q = k + N qq (S_lo, T_lo, S_hi, T_hi) over (j, i), then Mhat_x, Mhat_y
#pragma unroll
    for (int qq = 0; qq < ZQ; ++qq) {
      const int q = k + N * qq;
      if (q < 4) {
        const int side = q >> 1, isT = q & 1;
        const double* c = cl.fc[cs][4 + side];
        const double* nb = (side ? FZ : FX) + cs * G::FS;   // layout kk*N2 + j*N + i
        const bool tr = ghost_trace(kp, cl.cell[cs], side);
        double A[N][N];
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double gn = 0.0, av;
            if (tr) {
              av = nb[j * N + i];
              gn = nb[G::N2 + j * N + i];
            } else {
#pragma unroll
              for (int kk = 0; kk < N; ++kk) gn = fma(side ? c_tab[N].d0[kk] : c_tab[N].d1[kk], nb[kk * G::N2 + j * N + i], gn);
              av = nb[(side ? 0 : N - 1) * G::N2 + j * N + i];
            }
            A[j][i] = isT ? c[5] * av : c[2] * av + c[3] * gn * kp.ih[2];
          }
        double B[N][N];
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int ip = 0; ip < N; ++ip) s = fma(c_tab[N].M[i * N + ip], A[j][ip], s);
            B[j][i] = s;
          }
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int jp = 0; jp < N; ++jp) s = fma(c_tab[N].M[j * N + jp], B[jp][i], s);
            zs[qq][j][i] = s;
          }
      }
    }
  }
  __syncthreads();   // every read of the staged tiles and of the own tile is done
  double* tb = TB + cs * G::CTB;
  if (L.active) {
    double b[N][N], c[N][N];
    const double fa0 = kp.fa[0];
#pragma unroll
    for (int j = 0; j < N; ++j) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int ip = 0; ip < N; ++ip) s = fma(c_tab[N].M[i * N + ip], u[j][ip], s);
        b[j][i] = s;
      }
      kfly<N, GEN>(kp, cl, cs, 0, u[j], c[j]);
#pragma unroll
      for (int i = 0; i < N; ++i)
        c[j][i] = fma(fa0, fma(c_tab[N].d0[i], xs[1][j], fma(c_tab[N].d1[i], xs[3][j],
                               (i == 0 ? xs[0][j] : 0.0) + (i == N - 1 ? xs[2][j] : 0.0))), c[j][i]);
    }
    const double fa1 = kp.fa[1];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double cb[N], cc[N], e[N];
#pragma unroll
      for (int j = 0; j < N; ++j) { cb[j] = b[j][i]; cc[j] = c[j][i]; }
      kfly<N, GEN>(kp, cl, cs, 1, cb, e);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double sd = 0.0, sf = 0.0;
#pragma unroll
        for (int jp = 0; jp < N; ++jp) {
          sd = fma(c_tab[N].M[j * N + jp], cb[jp], sd);
          sf = fma(c_tab[N].M[j * N + jp], cc[jp], sf);
        }
        const double yf = c_tab[N].d0[j] * ys[1][i] + c_tab[N].d1[j] * ys[3][i] +
                          (j == 0 ? ys[0][i] : 0.0) + (j == N - 1 ? ys[2][i] : 0.0);
        tb[k * G::KS + j * N + i] = sd;
        tb[G::ARR + k * G::KS + j * N + i] = e[j] + sf + fa1 * yf;
      }
    }
#pragma unroll
    for (int qq = 0; qq < ZQ; ++qq) {
      const int q = k + N * qq;
      if (q < 4)
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) FX[cs * G::FS + q * G::N2 + j * N + i] = zs[qq][j][i];
    }
  }
  __syncwarp();
  if (L.active) {   // lane = y node j
    const int j = k;
    const double fa2 = kp.fa[2];
    double dz[N][N], gz[N][N];   // [kk][i]
#pragma unroll
    for (int kk = 0; kk < N; ++kk)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        dz[kk][i] = tb[kk * G::KS + j * N + i];
        gz[kk][i] = tb[G::ARR + kk * G::KS + j * N + i];
      }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double cd[N], o[N];
#pragma unroll
      for (int kk = 0; kk < N; ++kk) cd[kk] = dz[kk][i];
      kfly<N, GEN>(kp, cl, cs, 2, cd, o);
      const double* z = FX + cs * G::FS + j * N + i;
      const double z0 = z[0], z1 = z[G::N2], z2 = z[2 * G::N2], z3 = z[3 * G::N2];
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        double s = o[kk];
#pragma unroll
        for (int kp2 = 0; kp2 < N; ++kp2) s = fma(c_tab[N].M[kk * N + kp2], gz[kp2][i], s);
        s += fa2 * (c_tab[N].d0[kk] * z1 + c_tab[N].d1[kk] * z3 + (kk == 0 ? z0 : 0.0) + (kk == N - 1 ? z2 : 0.0));
        tb[kk * G::KS + j * N + i] = s;
      }
    }
  }
  __syncwarp();
  if (L.active) read_plane<N>(TB, L, res);
}

template <int N, bool NBR, bool FACES = true, bool GEN = true>
__global__ void __launch_bounds__(Geo<N>::NT)
k_apply(KParams kp, const double* __restrict__ u, double* __restrict__ out) {
  using G = Geo<N>;
  extern __shared__ double sm[];
  __shared__ Cells<N, false> cl;
  double* TB = sm;
  double* FY = TB + G::TB;
  double* FX = FY + G::FY;
  double* FZ = FX + G::FX;
  const int cell0 = block_group(kp, false) * G::C;
  const int nvalid = min(G::C, kp.ncells - cell0);
  const Lane L = lane_id<N>();
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  // programmatic dependent launch: the next kernel in the stream may start launching now; this
  // one's coefficient setup (K, c: constant) runs before it waits for the previous kernel's
  // results (u, the ghost layers), so the setup overlaps the previous kernel's tail
  asm volatile("griddepcontrol.launch_dependents;");
  const double* tile = u + (size_t)cell0 * G::N3;
  clear_masks<N>(cl);
  __syncthreads();
  SetupRegs<N> sr;
  setup_issue<N>(kp, cl, sr, cell0, NBR ? u : nullptr);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // DG_FUSED_TILES = 2: the own tile in the fused loop too (issued after the setup barrier)
  constexpr bool FUSED = DG_FUSED_TILES && NBR && fused_tiles<N>();
  constexpr bool FOWN = FUSED && DG_FUSED_TILES == 2;
  if (!FOWN) async_own<N>(TB, tile, nvalid);
  __syncthreads();   // neighbour pointers and masks
  if (FUSED && (cl.nbg[2] | cl.nbg[3] | cl.nbg[4] | cl.nbg[5]) == 0) {
    async_tiles5<N, FOWN>(TB, FY, FX, FZ, cl, kp, tile, nvalid);
  } else if (NBR) {
    if (FOWN) async_own<N>(TB, tile, nvalid);
    async_nbr<N, G::KS, G::CTB>(TB + G::ARR, cl, 2, u, kp, tile);   // y-lo -> TB half 1
    async_nbr<N, G::N2, G::FS>(FY, cl, 3, u, kp, tile);             // y-hi, z-lo, z-hi -> FY, FX, FZ
    async_nbr<N, G::N2, G::FS>(FX, cl, 4, u, kp, tile);
    async_nbr<N, G::N2, G::FS>(FZ, cl, 5, u, kp, tile);
  }
  setup_finish<N>(kp, cl, sr);
  cp_async_wait_all();
  __syncthreads();
  double in[N][N], o[N][N];
  // nodal form (C5 apply 815 -> 739 us, C2 37.8 -> 36.3 us); at n = 4 with convection it spills
  // (C4 301 -> 330 us) and the Gauss-point form stays
  if constexpr (DG_PLANE_NODAL_APPLY && NBR && FACES && !(N == 4 && GEN)) {
    plane_apply_nodal<N, GEN>(kp, cl, L, TB, FY, FX, FZ, tile, o);
  } else {
    read_plane<N>(TB, L, in);
    if (NBR) nbr_prologue_async<N, true>(kp, cl, L, TB, FY, FX, FZ, tile);
    else __syncthreads();
    plane_op<N, NBR, false, FACES, GEN>(kp, cl, L, rw, FACES ? (kp.mask & 1u) != 0 : true, in, o, TB, FY, FX, FZ);
  }
  if (L.active) write_plane<N>(TB, L, o);  // same TB slots this lane read in Q3
  __syncthreads();
  unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
}

// Tile transfers through the group's cell list (cl.cell; compact colour map): each cell's n^3
// values are contiguous in global memory, the cells are not.
template <int N, bool WB>
__device__ __forceinline__ void async_own_map(double* TB, const double* __restrict__ src, const Cells<N, WB>& cl) {
  using G = Geo<N>;
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    if (e < G::C * G::N3) {
      const int cs = e / G::N3, r = e % G::N3;
      const int cell = cl.cell[cs];
      cp_async8(TB + cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2), src + (cell >= 0 ? (size_t)cell * G::N3 + r : 0),
                cell >= 0);
    }
  }
}
template <int N, bool WB>
__device__ __forceinline__ void stage_tile_map(double* TB, const double* __restrict__ src, const Cells<N, WB>& cl) {
  using G = Geo<N>;
  double v[G::PER];
#pragma unroll
  for (int m = 0; m < G::PER; ++m) {
    const int e = threadIdx.x + m * G::NT;
    const int cell = e < G::C * G::N3 ? cl.cell[e / G::N3] : -1;
    v[m] = cell >= 0 ? src[(size_t)cell * G::N3 + e % G::N3] : 0.0;
  }
  store_tile<N>(TB, v);
}
template <int N, bool WB>
__device__ __forceinline__ void unstage_tile_map(const double* TB, double* __restrict__ dst, const Cells<N, WB>& cl) {
  using G = Geo<N>;
  for (int e = threadIdx.x; e < G::C * G::N3; e += G::NT) {
    const int cs = e / G::N3, r = e % G::N3;
    const int cell = cl.cell[cs];
    if (cell >= 0) dst[(size_t)cell * G::N3 + r] = TB[cs * G::CTB + (r / G::N2) * G::KS + (r % G::N2)];
  }
}

// Solver prologue: coefficients, self-face operators and (SWEEP) the defect's neighbour tiles
// staged with cp.async exactly as in the apply kernel; the own tile lands in TB half 0.
// The nodal D_T factors of every cell (the Kronecker-sum form, see plane_dt_nodal): per direction
//   K_a = |T|K_a/h_a^2 Shat - |T|b_a/h_a Chat + [a = z] |T| c Mhat + |F_a| (self-face 1D terms)
// in cl.B[cs][a n^2 + i n + i']. Needs fc, vc, vb complete; ends with a barrier.
template <int N, bool WB> __device__ __forceinline__ void setup_K3(const KParams& kp, Cells<N, WB>& cl) {
  using G = Geo<N>;
  for (int it = threadIdx.x; it < G::C * 3 * G::N2; it += G::NT) {
    const int cs = it / (3 * G::N2), rem = it % (3 * G::N2), a = rem / G::N2;
    const int i = (rem % G::N2) / N, ip = rem % N;
    const double* lo = cl.fc[cs][2 * a];
    const double* hi = cl.fc[cs][2 * a + 1];
    const double ih = kp.ih[a];
    const double e0i = i == 0, e0p = ip == 0, e1i = i == N - 1, e1p = ip == N - 1;
    double f = e0i * (lo[0] * e0p + lo[1] * ih * c_tab[N].d0[ip]) + lo[4] * c_tab[N].d0[i] * e0p;
    f += e1i * (hi[0] * e1p + hi[1] * ih * c_tab[N].d1[ip]) + hi[4] * c_tab[N].d1[i] * e1p;
    double t = kp.fa[a] * f;
    t = fma(cl.vc[cs][a], c_tab[N].S[i * N + ip], t);
    t = fma(-cl.vb[cs][a], c_tab[N].Cm[i * N + ip], t);
    if (a == 2) t = fma(cl.vc[cs][3], c_tab[N].M[i * N + ip], t);
    cl.B[cs][a * G::N2 + i * N + ip] = t;
  }
  __syncthreads();
}

// out = D_T in for the lane's plane in the nodal Kronecker-sum form
//   D_T = Kx (x) Mhat (x) Mhat + Mhat (x) Ky (x) Mhat + Mhat (x) Mhat (x) Kz
// (per-cell constant coefficients on the affine cell): in the plane (lane = z node k)
// b = Mhat_x p, c = Kx p, d = Mhat_y b, g = Ky b + Mhat_y c; one transpose; (lane = y node j)
// q = Mhat_z g + Kz d; one transpose back. 7 contractions per lane (the Gauss-point form: ~14).
template <int N, bool WB>
__device__ __forceinline__ void plane_dt_nodal(const Cells<N, WB>& cl, const Lane& L, const double (&in)[N][N],
                                               double (&out)[N][N], double* TB) {
  using G = Geo<N>;
  double* tb = TB + L.cs * G::CTB;
  const double* K = cl.B[L.cs];
  __syncwarp();   // the previous call's reads of TB (other lanes of the cell) are done
  if (L.active) {
    const int k = L.t;
    double b[N][N], c[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double kr[N];
#pragma unroll
      for (int ip = 0; ip < N; ++ip) kr[ip] = K[i * N + ip];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double sb = 0.0, sc = 0.0;
#pragma unroll
        for (int ip = 0; ip < N; ++ip) {
          sb = fma(c_tab[N].M[i * N + ip], in[j][ip], sb);
          sc = fma(kr[ip], in[j][ip], sc);
        }
        b[j][i] = sb;
        c[j][i] = sc;
      }
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double kr[N];
#pragma unroll
      for (int jp = 0; jp < N; ++jp) kr[jp] = K[G::N2 + j * N + jp];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double sd = 0.0, sg = 0.0;
#pragma unroll
        for (int jp = 0; jp < N; ++jp) {
          sd = fma(c_tab[N].M[j * N + jp], b[jp][i], sd);
          sg = fma(kr[jp], b[jp][i], sg);
          sg = fma(c_tab[N].M[j * N + jp], c[jp][i], sg);
        }
        tb[k * G::KS + j * N + i] = sd;
        tb[G::ARR + k * G::KS + j * N + i] = sg;
      }
    }
  }
  __syncwarp();
  if (L.active) {
    const int j = L.t;
    double dz[N][N], gz[N][N];   // [k][i]
#pragma unroll
    for (int kk = 0; kk < N; ++kk)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        dz[kk][i] = tb[kk * G::KS + j * N + i];
        gz[kk][i] = tb[G::ARR + kk * G::KS + j * N + i];
      }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double kr[N];
#pragma unroll
      for (int kk = 0; kk < N; ++kk) kr[kk] = K[2 * G::N2 + k * N + kk];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int kk = 0; kk < N; ++kk) {
          s = fma(c_tab[N].M[k * N + kk], gz[kk][i], s);
          s = fma(kr[kk], dz[kk][i], s);
        }
        tb[k * G::KS + j * N + i] = s;
      }
    }
  }
  __syncwarp();
  if (L.active) read_plane<N>(TB, L, out);
}

template <int N, bool SWEEP, bool CMAP, bool WB, bool NODAL = false>
__device__ __forceinline__ void solver_setup(const KParams& kp, Cells<N, WB>& cl, double* TB, double* FY,
                                             double* FX, double* FZ, const double* in, int cell0, int nvalid) {
  using G = Geo<N>;
  const double* tile = in + (size_t)cell0 * G::N3;
  // n = 4 solvers: the copy loops rolled (the fused sweep kernel's prologue code shrinks by
  // ~20 KB; C2 sweep 433 -> 416 us, C4 7.40 -> 7.33 ms; n = 3 and the applies lose with it)
  constexpr bool RL = N == 4;
  // the fused staging of the apply's prologue (async_tiles5), for the sweeps' defect
  constexpr bool FUSED = DG_FUSED_TILES && SWEEP && !CMAP && fused_tiles<N>();
  constexpr bool FOWN = FUSED && DG_FUSED_TILES == 2;
  if (!CMAP && !FOWN) async_own<N, RL>(TB, tile, nvalid);
  clear_masks<N>(cl);
  __syncthreads();
  SetupRegs<N> sr;
  setup_issue<N, CMAP>(kp, cl, sr, cell0, SWEEP ? in : nullptr);
  __syncthreads();   // neighbour pointers and masks
  if (CMAP) async_own_map<N>(TB, in, cl);
  if (FUSED && (cl.nbg[2] | cl.nbg[3] | cl.nbg[4] | cl.nbg[5]) == 0) {
    async_tiles5<N, FOWN>(TB, FY, FX, FZ, cl, kp, tile, nvalid);
  } else if (SWEEP) {
    if (FOWN) async_own<N, RL>(TB, tile, nvalid);
    async_nbr<N, G::KS, G::CTB, RL>(TB + G::ARR, cl, 2, in, kp, tile);
    async_nbr<N, G::N2, G::FS, RL>(FY, cl, 3, in, kp, tile);
    async_nbr<N, G::N2, G::FS, RL>(FX, cl, 4, in, kp, tile);
    async_nbr<N, G::N2, G::FS, RL>(FZ, cl, 5, in, kp, tile);
  }
  setup_finish<N>(kp, cl, sr);
  __syncthreads();   // fc of every cell
  if constexpr (NODAL) setup_K3<N>(kp, cl);
  else setup_B<N>(kp, cl);
  cp_async_wait_all();
  __syncthreads();
}

// The volume terms alone, A^v u (Stages 1-3; dg_apply_parts with mask = volume):
// a persistent kernel, one CTA per resident slot, walking the cell groups with a stride of the
// grid; the next group's tile and coefficients are loaded into registers while the current
// group is computed, so the HBM/L2 latency is hidden behind the fp64 work.
template <int N, bool GEN = true>
__global__ void __launch_bounds__(Geo<N>::NT, DG_VOL_MINB)
k_volume(KParams kp, const double* __restrict__ u, double* __restrict__ out) {
  using G = Geo<N>;
  extern __shared__ double sm[];
  __shared__ Cells<N, false> cl;
  double* TB = sm;
  const int ngroups = (kp.ncells + G::C - 1) / G::C;
  const Lane L = lane_id<N>();
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
  const int nxy = kp.nx * kp.ny;
  double nxt[G::PER], kn[3] = {0.0, 0.0, 0.0}, cn = 0.0, bnx[3] = {0.0, 0.0, 0.0};
  auto prefetch = [&](int g) {
    const int cell0 = g * G::C;
    load_own<N>(nxt, u + (size_t)cell0 * G::N3, min(G::C, kp.ncells - cell0));
    const int cell = cell0 + (int)threadIdx.x;
    if (threadIdx.x < G::C && cell < kp.ncells) {
      const double* Kc = kp.K + (size_t)(cell + nxy) * 3;
      kn[0] = __ldg(Kc); kn[1] = __ldg(Kc + 1); kn[2] = __ldg(Kc + 2);
      cn = kp.c ? __ldg(kp.c + cell) : 0.0;
      if (GEN)
#pragma unroll
        for (int a = 0; a < 3; ++a) bnx[a] = kp.bc ? __ldg(kp.bc + (size_t)(cell + nxy) * 3 + a) : kp.b[a];
    }
  };
  int g = blockIdx.x;
  if (g < ngroups) prefetch(g);
  for (; g < ngroups; g += gridDim.x) {
    const int cell0 = g * G::C;
    const int nvalid = min(G::C, kp.ncells - cell0);
    __syncthreads();   // the previous group's TB and vc reads are done
    store_tile<N>(TB, nxt);
    if (threadIdx.x < G::C) {
      const int cs = threadIdx.x;
      const bool ok = cs < nvalid;
      cl.vc[cs][0] = ok ? kn[0] * vol * kp.ih[0] * kp.ih[0] : 0.0;
      cl.vc[cs][1] = ok ? kn[1] * vol * kp.ih[1] * kp.ih[1] : 0.0;
      cl.vc[cs][2] = ok ? kn[2] * vol * kp.ih[2] * kp.ih[2] : 0.0;
      cl.vc[cs][3] = ok ? vol * cn : 0.0;
      if (GEN)
#pragma unroll
        for (int a = 0; a < 3; ++a) cl.vb[cs][a] = ok ? vol * bnx[a] * kp.ih[a] : 0.0;
    }
    __syncthreads();
    if (g + (int)gridDim.x < ngroups) prefetch(g + gridDim.x);
    double in[N][N], o[N][N];
    read_plane<N>(TB, L, in);
    plane_op<N, false, false, false, GEN>(kp, cl, L, rw, true, in, o, TB, nullptr, nullptr, nullptr);
    if (L.active) write_plane<N>(TB, L, o);
    __syncthreads();
    unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
  }
}

// Variant without register prefetch (n = 4): the group's tile is copied with cp.async straight
// into TB and the coefficients into a slim shared array, so the kernel needs ~130 instead of 166
// registers and 42 KB instead of 54 KB of shared memory: four CTAs (16 warps) per SM hide the
// load latency instead of the prefetch.
#ifndef DG_VOL4_MINB
#define DG_VOL4_MINB 4
#endif
#ifndef DG_VOL4_MINB_GEN
// the convective / reaction instantiation with two-warp CTAs: eight per SM (C4 volume 97.9 ->
// 95.4 us, 0.51); the same bound for diffusion costs the L2-resident C2 (14.0 -> 17.6 us)
#define DG_VOL4_MINB_GEN 8
#endif
template <int N, bool GEN = true>
__global__ void __launch_bounds__(Geo<N>::NT, GEN ? DG_VOL4_MINB_GEN : DG_VOL4_MINB)
k_volume_s(KParams kp, const double* __restrict__ u, double* __restrict__ out) {
  using G = Geo<N>;
  extern __shared__ double sm[];
  double* TB = sm;
  // only vc and vb (the leading members) of the cell block are read by the volume-only operator
  using CellsV = Cells<N, false>;
  static_assert(offsetof(CellsV, vc) == 0, "vc leads the cell block");
  static_assert(offsetof(CellsV, vb) == sizeof(double) * 4 * G::C, "vb follows vc");
  __shared__ double vcb[G::C * 7];   // [C][4] vc, then [C][3] vb
  const Cells<N, false>& cl = *reinterpret_cast<const Cells<N, false>*>(vcb);
  double (*vcs)[4] = reinterpret_cast<double (*)[4]>(vcb);
  double (*vbs)[3] = reinterpret_cast<double (*)[3]>(vcb + 4 * G::C);
  const int ngroups = (kp.ncells + G::C - 1) / G::C;
  const Lane L = lane_id<N>();
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  const double vol = kp.h[0] * kp.h[1] * kp.h[2];
  const int nxy = kp.nx * kp.ny;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int cell0 = g * G::C;
    const int nvalid = min(G::C, kp.ncells - cell0);
    async_own<N>(TB, u + (size_t)cell0 * G::N3, nvalid);
    if (threadIdx.x < G::C) {
      const int cs = threadIdx.x;
      const bool ok = cs < nvalid;
      const double* Kc = kp.K + (size_t)(cell0 + (ok ? cs : 0) + nxy) * 3;
      vcs[cs][0] = ok ? __ldg(Kc) * vol * kp.ih[0] * kp.ih[0] : 0.0;
      vcs[cs][1] = ok ? __ldg(Kc + 1) * vol * kp.ih[1] * kp.ih[1] : 0.0;
      vcs[cs][2] = ok ? __ldg(Kc + 2) * vol * kp.ih[2] * kp.ih[2] : 0.0;
      vcs[cs][3] = ok && kp.c ? vol * __ldg(kp.c + cell0 + cs) : 0.0;
      if (GEN)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          vbs[cs][a] = ok ? vol * (kp.bc ? __ldg(kp.bc + (size_t)(cell0 + cs + nxy) * 3 + a) : kp.b[a]) * kp.ih[a] : 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    double in[N][N], o[N][N];
    read_plane<N>(TB, L, in);
    plane_op<N, false, false, false, GEN>(kp, cl, L, rw, true, in, o, TB, nullptr, nullptr, nullptr);
    if (L.active) write_plane<N>(TB, L, o);
    __syncthreads();
    unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
    __syncthreads();   // TB and vcs are reused by the next group
  }
}

// Jacobi-PCG per cell; SWEEP: defect d = f - A u first, result u + omega du.
// Registers: r, p (and the operator's planes); shared: x and diag(D_T) planes.
template <int N, bool SWEEP, bool GEN = true, bool CMAP = false>
__global__ void __launch_bounds__(Geo<N>::NT)
k_cg(KParams kp, const double* DG_RESTRICT in, const double* __restrict__ f,
     double* DG_RESTRICT out) {
  using G = Geo<N>;
  extern __shared__ double sm[];
  __shared__ Cells<N> cl;
  double* TB = sm;
  double* FY = TB + G::TB;
  double* XS = FY + G::FY;          // FX / FZ (defect prologue only) alias XS / DS
  double* DS = XS + G::C * G::PS;
  double* FX = XS;
  double* FZ = DS;
  const int cell0 = (CMAP ? (int)blockIdx.x : block_group(kp, true)) * G::C;
  const int nvalid = min(G::C, (CMAP ? kp.ncells / 2 : kp.ncells) - cell0);
  const Lane L = lane_id<N>();
  const bool valid = L.active && L.cs < nvalid;
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  // n <= 4: neighbour tiles staged with cp.async (a face region holds a tile); n = 5: through
  // registers, one pair of tiles at a time
  constexpr bool ASYNC = G::FS >= G::N3;
  // D_T of the iterations in the nodal Kronecker-sum form (plane_dt_nodal): C5 sweep
  // 5339 -> 3960 us; at n = 4 equal to the Gauss-point form (C2 339 vs 342 us), which with the
  // cell block sized for the nodal factors (BiCGStab) loses occupancy (437 us)
  constexpr bool NODAL = DG_NODAL_DT && ASYNC;
  if constexpr (ASYNC) {
    solver_setup<N, SWEEP, CMAP, true, NODAL>(kp, cl, TB, FY, FX, FZ, in, cell0, nvalid);
  } else {
    stage_tile<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
    setup<N>(kp, cl, cell0, SWEEP ? in : nullptr);
  }
  double R[N][N], P[N][N];
  read_plane<N>(TB, L, P);
  if (SWEEP) {
    double Q[N][N];
    if constexpr (ASYNC) {
      nbr_prologue_async<N, true>(kp, cl, L, TB, FY, FX, FZ, CMAP ? nullptr : in + (size_t)cell0 * G::N3);
    } else {
      double pv0[G::PER], pv1[G::PER];
      load_nbr<N>(pv0, cl, 2, kp);
      load_nbr<N>(pv1, cl, 3, kp);
      nbr_prologue<N>(kp, cl, L, TB, FY, FX, FZ, in + (size_t)cell0 * G::N3, pv0, pv1);
    }
    // Q = A u (with the nodal D_T factors in cl.B, the self faces come from the traces)
    plane_op<N, true, !NODAL, true, GEN>(kp, cl, L, rw, true, P, Q, TB, FY, FX, FZ);
    __syncthreads();
    if (CMAP) stage_tile_map<N>(TB, f, cl);
    else stage_tile_s<N>(TB, f + (size_t)cell0 * G::N3, nvalid);
    __syncthreads();
    read_plane<N>(TB, L, R);
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? R[j][i] - Q[j][i] : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? P[j][i] : 0.0;
  }
  const int po = L.cs * G::PS + L.t * G::QS;
  double* xs = XS + po;
  double* ds = DS + po;
  __syncthreads();   // the prologue's FX / FZ (aliasing XS / DS) are consumed
  {
    double dg[N][N];
    plane_inv_diag<N>(kp, cl, L, rw, dg);
    if (L.active)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) ds[j * N + i] = valid ? dg[j][i] : 1.0;
  }
  int its_out = 0;
  double rr = 0.0, rz = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double z = L.active ? R[j][i] * ds[j * N + i] : 0.0;
      P[j][i] = z;
      rr = fma(R[j][i], R[j][i], rr);
      rz = fma(R[j][i], z, rz);
      if (L.active) xs[j * N + i] = 0.0;
    }
  const double rr0 = cell_sum<N>(rr, L.lane);
  rz = cell_sum<N>(rz, L.lane);
  bool conv = !valid || rr0 == 0.0 || skip_cell(kp, cell0 + L.cs);
  bool brk = false;
  int its = 0;
  for (int iter = 0;; ++iter) {
    const int done = __all_sync(0xffffffffu, conv || !L.active);  // per-warp lock-step
    if (done || iter >= kp.max_it) break;
    double Q[N][N];
    if constexpr (NODAL) plane_dt_nodal<N>(cl, L, P, Q, TB);                       // Q = D_T P
    else plane_op<N, false, true, true, GEN>(kp, cl, L, rw, true, P, Q, TB, FY, FX, FZ);
    double pq = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) pq = fma(P[j][i], Q[j][i], pq);
    pq = cell_sum<N>(pq, L.lane);
    double alpha = 0.0;
    if (!conv) {
      if (pq > 0.0) alpha = DG_QUOT(rz, pq);
      else conv = brk = true;   // breakdown (D_T not SPD): stop, reported as not converged
    }
    double r2 = 0.0, rzn = 0.0;
    double Z[N][N];   // M^-1 r, formed once (reused by the direction update)
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (L.active) xs[j * N + i] = fma(alpha, P[j][i], xs[j * N + i]);
        R[j][i] = fma(-alpha, Q[j][i], R[j][i]);
        r2 = fma(R[j][i], R[j][i], r2);
        Z[j][i] = L.active ? R[j][i] * ds[j * N + i] : 0.0;
        rzn = fma(R[j][i], Z[j][i], rzn);
      }
    r2 = cell_sum<N>(r2, L.lane);
    rzn = cell_sum<N>(rzn, L.lane);
    if (!conv) {
      ++its;
      if (r2 <= kp.tol2 * rr0) conv = true;
      const double beta = DG_QUOT(rzn, rz);
      rz = rzn;
      if (!conv && L.active) {
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) P[j][i] = fma(beta, P[j][i], Z[j][i]);
      }
    }
  }
  its_out = (conv && !brk) ? its : (its | (1 << 30));
  // result: X (+ u) -> TB -> global
  __syncthreads();
  if (SWEEP) {
    if (CMAP) stage_tile_map<N>(TB, in, cl);
    else stage_tile_s<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
  }
  __syncthreads();
  if (L.active) {
    double* b = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i)
        b[j * N + i] = SWEEP ? fma(kp.omega, xs[j * N + i], b[j * N + i]) : xs[j * N + i];
  }
  __syncthreads();
  if (CMAP) unstage_tile_map<N>(TB, out, cl);
  else unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
  if (valid && L.t == 0) kp.its[CMAP ? cl.cell[L.cs] : cell0 + L.cs] = its_out;
}

// ---- tridiagonal (Thomas) local preconditioner -------------
// D_T[I][J] from the 1D matrices (volume + self faces as Kronecker products on the
// affine cell; the same coefficients as the operator), I = i + n j + n^2 k test, J trial.
template <int N, bool WB>
__device__ __forceinline__ double dt_entry(const KParams& kp, const Cells<N, WB>& cl, int cs, int I, int J) {
  const int i = I % N, j = (I / N) % N, k = I / (N * N);
  const int a = J % N, b = (J / N) % N, c = J / (N * N);
  const double* M = c_tab[N].M;
  const double* S = c_tab[N].S;
  const double* C = c_tab[N].Cm;
  const double* vc = cl.vc[cs];
  const double Mx = M[i * N + a], My = M[j * N + b], Mz = M[k * N + c];
  double v = vc[0] * S[i * N + a] * My * Mz + vc[1] * Mx * S[j * N + b] * Mz +
             vc[2] * Mx * My * S[k * N + c] + vc[3] * Mx * My * Mz;
  const double* vb = cl.vb[cs];
  v -= vb[0] * C[i * N + a] * My * Mz + vb[1] * Mx * C[j * N + b] * Mz + vb[2] * Mx * My * C[k * N + c];
  const int r3[3] = {i, j, k}, c3[3] = {a, b, c};
  const double m3[3] = {Mx, My, Mz};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const int r = r3[ax], q = c3[ax];
    const double* lo = cl.fc[cs][2 * ax];
    const double* hi = cl.fc[cs][2 * ax + 1];
    const double ih = kp.ih[ax];
    const double e0r = r == 0, e0q = q == 0, e1r = r == N - 1, e1q = q == N - 1;
    double bf = lo[0] * e0r * e0q + lo[1] * ih * e0r * c_tab[N].d0[q] + lo[4] * c_tab[N].d0[r] * e0q;
    bf += hi[0] * e1r * e1q + hi[1] * ih * e1r * c_tab[N].d1[q] + hi[4] * c_tab[N].d1[r] * e1q;
    double t = kp.fa[ax] * bf;
#pragma unroll
    for (int o = 0; o < 3; ++o)
      if (o != ax) t *= m3[o];
    v += t;
  }
  return v;
}

// Bands of D_T in DoF order and their LU (Thomas) factors, per cell: lane t writes the sub-,
// main and super-diagonal entries of its plane, then the cell's lane 0 eliminates sequentially:
// SB = sub, IP = 1 / pivot, CP = super / pivot.
template <int N, bool WB>
__device__ void thomas_factor(const KParams& kp, const Cells<N, WB>& cl, const Lane& L, double* SB,
                              double* IP, double* CP, bool valid) {
  using G = Geo<N>;
  constexpr int ND = G::N3;
  double* sb = SB + L.cs * G::PS;
  double* ip = IP + L.cs * G::PS;
  double* cp = CP + L.cs * G::PS;
  if (L.active) {
    for (int q = 0; q < G::N2; ++q) {
      const int I = L.t * G::N2 + q, o = L.t * G::QS + q;
      sb[o] = (valid && I > 0) ? dt_entry<N>(kp, cl, L.cs, I, I - 1) : 0.0;
      ip[o] = valid ? dt_entry<N>(kp, cl, L.cs, I, I) : 1.0;
      cp[o] = (valid && I < ND - 1) ? dt_entry<N>(kp, cl, L.cs, I, I + 1) : 0.0;
    }
  }
  __syncwarp();
  if (L.active && L.t == 0) {
    double c_prev = 0.0;
    for (int I = 0; I < ND; ++I) {
      const int o = (I / G::N2) * G::QS + I % G::N2;
      const double inv = 1.0 / (ip[o] - sb[o] * c_prev);
      ip[o] = inv;
      c_prev = cp[o] * inv;
      cp[o] = c_prev;
    }
  }
  __syncwarp();
}

// v <- M^-1 v with M the tridiagonal part of D_T (forward / back substitution by the cell's
// lane 0 through the cell's TB slot, which is free between two operator applications)
template <int N>
__device__ void thomas_apply(const Lane& L, double* TB, const double* SB, const double* IP, const double* CP,
                             double (&v)[N][N]) {
  using G = Geo<N>;
  double* sc = TB + L.cs * G::CTB;
  const double* sb = SB + L.cs * G::PS;
  const double* ip = IP + L.cs * G::PS;
  const double* cp = CP + L.cs * G::PS;
  __syncwarp();
  if (L.active)
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) sc[L.t * G::KS + j * N + i] = v[j][i];
  __syncwarp();
  if (L.active && L.t == 0) {
    double y = 0.0;
    for (int I = 0; I < G::N3; ++I) {
      const int o = (I / G::N2) * G::QS + I % G::N2, s = (I / G::N2) * G::KS + I % G::N2;
      y = (sc[s] - sb[o] * y) * ip[o];
      sc[s] = y;
    }
    double x = 0.0;
    for (int I = G::N3 - 1; I >= 0; --I) {
      const int o = (I / G::N2) * G::QS + I % G::N2, s = (I / G::N2) * G::KS + I % G::N2;
      x = fma(-cp[o], x, sc[s]);
      sc[s] = x;
    }
  }
  __syncwarp();
  if (L.active)
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) v[j][i] = sc[L.t * G::KS + j * N + i];
}


// ---- tensor memory (TMEM) as per-lane storage of Krylov vectors ------------------------------
// The fp64 local solvers never issue tcgen05.mma, so the SM's 256 KB of TMEM is otherwise idle.
// The BiCGStab kernel keeps three of its per-lane vectors there (x, p, v: each lane owns one TMEM
// lane, a row of N doubles = 2N 32-bit columns), which takes them out of shared memory and lets
// two CTAs (8 warps) share an SM instead of one. Warp w of the CTA owns TMEM lanes 32w..32w+31
// (the tcgen05.ld/st lane-quadrant rule), so the CTA must have at most 4 warps.
template <int NCOL> __device__ __forceinline__ uint32_t tm_alloc(uint32_t* slot) {
  static_assert(NCOL == 32 || NCOL == 64 || NCOL == 128 || NCOL == 256 || NCOL == 512, "TMEM allocation: power of 2");
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 ::"r"((unsigned)__cvta_generic_to_shared(slot)), "n"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  return *slot;
}
// all warps' TMEM accesses are complete (tcgen05.wait inside the row helpers) before the call
template <int NCOL> __device__ __forceinline__ void tm_free(uint32_t base) {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(NCOL));
}
// one row of N doubles of the lane's plane at TMEM address a (warp-collective: every lane of the
// warp executes it; the load waits for its data inside the same asm block)
template <int N> struct TmRow;
template <> struct TmRow<4> {
  static __device__ __forceinline__ void ld(uint32_t a, double (&v)[4]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(a));
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
  }
  static __device__ __forceinline__ void st(uint32_t a, const double (&v)[4]) {
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      r[2 * i] = (uint32_t)__double2loint(v[i]);
      r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                 ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                   "r"(r[7]));
  }
};
template <> struct TmRow<2> {
  static __device__ __forceinline__ void ld(uint32_t a, double (&v)[2]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
#pragma unroll
    for (int i = 0; i < 2; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
  }
  static __device__ __forceinline__ void st(uint32_t a, const double (&v)[2]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n"
                 ::"r"(a), "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])),
                   "r"(__double2hiint(v[1])));
  }
};
template <> struct TmRow<3> {
  static __device__ __forceinline__ void ld(uint32_t a, double (&v)[3]) {
    uint32_t r[6];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%6];\n"
                 "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%4,%5}, [%7];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5])
                 : "r"(a), "r"(a + 4));
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
  }
  static __device__ __forceinline__ void st(uint32_t a, const double (&v)[3]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%2,%3,%4,%5};\n"
                 "tcgen05.st.sync.aligned.32x32b.x2.b32 [%1], {%6,%7};\n"
                 ::"r"(a), "r"(a + 4), "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])),
                   "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])),
                   "r"(__double2hiint(v[2])));
  }
};
template <> struct TmRow<5> {
  static __device__ __forceinline__ void ld(uint32_t a, double (&v)[5]) {
    uint32_t r[10];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%10];\n"
                 "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%8,%9}, [%11];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9])
                 : "r"(a), "r"(a + 8));
#pragma unroll
    for (int i = 0; i < 5; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
  }
  static __device__ __forceinline__ void st(uint32_t a, const double (&v)[5]) {
    uint32_t r[10];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      r[2 * i] = (uint32_t)__double2loint(v[i]);
      r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%2,%3,%4,%5,%6,%7,%8,%9};\n"
                 "tcgen05.st.sync.aligned.32x32b.x2.b32 [%1], {%10,%11};\n"
                 ::"r"(a), "r"(a + 8), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                   "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]));
  }
};
// stores of this thread are complete (before TMEM data is read back or freed)
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }

// Jacobi right-preconditioned BiCGStab per cell (nonsymmetric blocks).
// Registers: r and the operator input/output planes; shared: x, r^, p, v, diag planes.
// THOMAS: right preconditioner = the tridiagonal part of D_T in DoF order (NEXT-3) instead of
// its diagonal; two more shared planes (the band factors) per cell.
// TM: x, p and v in tensor memory (see tm_alloc), r^ and the inverse diagonal in shared memory;
// the dynamic shared memory drops from 5 planes to 2, two CTAs per SM.
template <int N, bool SWEEP, bool THOMAS = false, bool CMAP = false, bool TM = false>
__global__ void __launch_bounds__(Geo<N>::NT)
k_bicgstab(KParams kp, const double* DG_RESTRICT in, const double* __restrict__ f,
           double* DG_RESTRICT out) {
  using G = Geo<N>;
  static_assert(!TM || (N == 4 && !THOMAS && G::WARPS <= 4), "TMEM vectors: n = 4, one lane quadrant per warp");
  constexpr int PLN = G::C * G::PS;
  extern __shared__ double sm[];
  __shared__ Cells<N> cl;
  __shared__ uint32_t tm_slot;
  double* TB = sm;
  double* FY = TB + G::TB;
  double* XS = FY + G::FY;          // FX / FZ (defect prologue only) alias the first two planes
  double* RHS = TM ? XS : XS + PLN;
  double* PSM = RHS + PLN;
  double* VSM = PSM + PLN;
  double* DS = TM ? RHS + PLN : VSM + PLN;
  double* SBM = DS + PLN;            // THOMAS: sub-diagonal; DS then holds 1 / pivot
  double* CPM = SBM + PLN;           // THOMAS: super-diagonal / pivot
  double* FX = XS;
  double* FZ = XS + PLN;
  // TMEM: columns [0, 2N^2) x, [32, ...) p, [64, ...) v; this warp's lane quadrant
  const int cell0 = (CMAP ? (int)blockIdx.x : block_group(kp, true)) * G::C;
  const int nvalid = min(G::C, (CMAP ? kp.ncells / 2 : kp.ncells) - cell0);
  const Lane L = lane_id<N>();
  const bool valid = L.active && L.cs < nvalid;
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  // n <= 4: neighbour tiles staged with cp.async (a face region holds a tile); n = 5: through
  // registers, one pair of tiles at a time
  constexpr bool ASYNC = G::FS >= G::N3;
  // D_T of the iterations in the nodal Kronecker-sum form (plane_dt_nodal)
  constexpr bool NODAL = DG_NODAL_DT && DG_NODAL_BICG && ASYNC;
  if constexpr (ASYNC) {
    solver_setup<N, SWEEP, CMAP, true, NODAL>(kp, cl, TB, FY, FX, FZ, in, cell0, nvalid);
  } else {
    stage_tile<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
    setup<N>(kp, cl, cell0, SWEEP ? in : nullptr);
  }
  double R[N][N], W[N][N];
  read_plane<N>(TB, L, W);
  if (SWEEP) {
    double T[N][N];
    if constexpr (ASYNC) {
      nbr_prologue_async<N, true>(kp, cl, L, TB, FY, FX, FZ, CMAP ? nullptr : in + (size_t)cell0 * G::N3);
    } else {
      double pv0[G::PER], pv1[G::PER];
      load_nbr<N>(pv0, cl, 2, kp);
      load_nbr<N>(pv1, cl, 3, kp);
      nbr_prologue<N>(kp, cl, L, TB, FY, FX, FZ, in + (size_t)cell0 * G::N3, pv0, pv1);
    }
    plane_op<N, true, !NODAL>(kp, cl, L, rw, true, W, T, TB, FY, FX, FZ);   // A u
    __syncthreads();
    if (CMAP) stage_tile_map<N>(TB, f, cl);
    else stage_tile_s<N>(TB, f + (size_t)cell0 * G::N3, nvalid);
    __syncthreads();
    read_plane<N>(TB, L, R);
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? R[j][i] - T[j][i] : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? W[j][i] : 0.0;
  }
  const int po = L.cs * G::PS + L.t * G::QS;
  double* xs = XS + po;
  double* rh = RHS + po;
  double* ps = PSM + po;
  double* vs = VSM + po;
  double* ds = DS + po;
  // the prologue's FX / FZ (aliasing the first two planes) are consumed; the TMEM allocation
  // (TM) comes with its own barrier, late so that its address is not live through the prologue
  if constexpr (TM) tm_alloc<128>(&tm_slot);
  else __syncthreads();
  // TMEM addresses re-derived at each use (no register held through the operator)
#define tx (*(volatile uint32_t*)&tm_slot + ((uint32_t)((threadIdx.x >> 5) * 32) << 16))
#define tp (tx + 32)
#define tv (tx + 64)
#define tr (tx + 96)
  // TM: the residual waits in TMEM while the operator runs (frees 2 N^2 registers there)
  auto park = [&](double (&R_)[N][N]) {
    if constexpr (TM) {
#pragma unroll
      for (int j = 0; j < N; ++j) TmRow<N>::st(tr + 2 * N * j, R_[j]);
      tm_wait_st();
    }
  };
  auto unpark = [&](double (&R_)[N][N]) {
    if constexpr (TM) {
#pragma unroll
      for (int j = 0; j < N; ++j) TmRow<N>::ld(tr + 2 * N * j, R_[j]);
    }
  };
  if constexpr (THOMAS) {
    thomas_factor<N>(kp, cl, L, SBM, DS, CPM, valid);
  } else {
    double dg[N][N];
    plane_inv_diag<N>(kp, cl, L, rw, dg);
    if (L.active)
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) ds[j * N + i] = valid ? dg[j][i] : 1.0;
  }
  double rr = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      rr = fma(R[j][i], R[j][i], rr);
      if (L.active) {
        rh[j * N + i] = R[j][i];
        if constexpr (!TM) {
          xs[j * N + i] = 0.0;
          ps[j * N + i] = 0.0;
          vs[j * N + i] = 0.0;
        }
      }
    }
  if constexpr (TM) {
    const double z[N] = {};
#pragma unroll
    for (int j = 0; j < N; ++j) {
      TmRow<N>::st(tx + 2 * N * j, z);
      TmRow<N>::st(tp + 2 * N * j, z);
      TmRow<N>::st(tv + 2 * N * j, z);
    }
    tm_wait_st();
  }
  const double rr0 = cell_sum<N>(rr, L.lane);
  bool conv = !valid || rr0 == 0.0 || skip_cell(kp, cell0 + L.cs);
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  bool rst = false;
  int its = 0;
  // one operator call site per loop pass (the two half-steps of BiCGStab alternate), so the
  // loop body holds a single copy of the operator's code: the instruction-cache footprint
  // halves (the unrolled two-call loop was 77 KB against a 32 KB L1.5 instruction cache)
  double rhon = 0.0;
  double T[N][N];
  bool half = false;   // false: v = D_T p^ next; true: t = D_T s^ next
  for (int iter = 0;;) {
    if (!half) {
      const int done = __all_sync(0xffffffffu, conv || !L.active);  // per-warp lock-step
      if (done || iter >= kp.max_it) break;
      ++iter;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if (L.active) a = fma(rh[j * N + i], R[j][i], a);
          b = fma(R[j][i], R[j][i], b);
        }
      rhon = cell_sum<N>(a, L.lane);
      const double r2 = cell_sum<N>(b, L.lane);
      if (fabs(rhon) <= 1e-24 * r2) rst = true;   // breakdown: restart with r^ = r
      if (rst) rhon = r2;
      const double beta = rst ? 0.0 : DG_QUOT(rhon * alpha, rho * omega);
      // p = r + beta (p - omega v);  W = M^-1 p
      if constexpr (TM) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double pr[N], vr[N];
          TmRow<N>::ld(tp + 2 * N * j, pr);
          TmRow<N>::ld(tv + 2 * N * j, vr);
#pragma unroll
          for (int i = 0; i < N; ++i) {
            if (!conv) {
              pr[i] = rst ? R[j][i] : fma(beta, fma(-omega, vr[i], pr[i]), R[j][i]);
              if (rst && L.active) rh[j * N + i] = R[j][i];
            }
            W[j][i] = L.active ? pr[i] * ds[j * N + i] : 0.0;
          }
          TmRow<N>::st(tp + 2 * N * j, pr);
        }
        tm_wait_st();
      } else {
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double p = 0.0;
          if (L.active) {
            p = ps[j * N + i];
            if (!conv) {
              p = rst ? R[j][i] : fma(beta, fma(-omega, vs[j * N + i], p), R[j][i]);
              ps[j * N + i] = p;
              if (rst) rh[j * N + i] = R[j][i];
            }
            if (!THOMAS) p *= ds[j * N + i];
          }
          W[j][i] = p;
        }
      }
      if constexpr (THOMAS) thomas_apply<N>(L, TB, SBM, DS, CPM, W);
      rst = false;
    }
    park(R);
    if constexpr (NODAL) plane_dt_nodal<N>(cl, L, W, T, TB);                  // v = D_T p^ / t = D_T s^
    else plane_op<N, false, true>(kp, cl, L, rw, true, W, T, TB, FY, FX, FZ);
    unpark(R);
    if (!half) {
      double rv = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if constexpr (TM) TmRow<N>::st(tv + 2 * N * j, T[j]);
#pragma unroll
        for (int i = 0; i < N; ++i)
          if (L.active) {
            if constexpr (!TM) vs[j * N + i] = T[j][i];
            rv = fma(rh[j * N + i], T[j][i], rv);
          }
      }
      rv = cell_sum<N>(rv, L.lane);
      alpha = 0.0;
      if (!conv) {
        if (rv != 0.0) alpha = DG_QUOT(rhon, rv);
        else rst = true;
      }
      // x += alpha p^;  s = r - alpha v (in R);  W = M^-1 s
      double ss = 0.0;
      if constexpr (TM) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double xr[N];
          TmRow<N>::ld(tx + 2 * N * j, xr);
#pragma unroll
          for (int i = 0; i < N; ++i) xr[i] = fma(alpha, W[j][i], xr[i]);
          TmRow<N>::st(tx + 2 * N * j, xr);
        }
        tm_wait_st();
      }
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if (!TM && L.active) xs[j * N + i] = fma(alpha, W[j][i], xs[j * N + i]);
          R[j][i] = fma(-alpha, T[j][i], R[j][i]);
          ss = fma(R[j][i], R[j][i], ss);
          W[j][i] = L.active ? (THOMAS ? R[j][i] : R[j][i] * ds[j * N + i]) : 0.0;
        }
      if constexpr (THOMAS) thomas_apply<N>(L, TB, SBM, DS, CPM, W);
      ss = cell_sum<N>(ss, L.lane);
      if (!conv && ss <= kp.tol2 * rr0) {
        conv = true;
        ++its;
      }
    } else {
      double ts = 0.0, tt = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          ts = fma(T[j][i], R[j][i], ts);
          tt = fma(T[j][i], T[j][i], tt);
        }
      ts = cell_sum<N>(ts, L.lane);
      tt = cell_sum<N>(tt, L.lane);
      const double om = (!conv && tt > 0.0) ? DG_QUOT(ts, tt) : 0.0;
      double r2n = 0.0;
      if constexpr (TM) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double xr[N];
          TmRow<N>::ld(tx + 2 * N * j, xr);
#pragma unroll
          for (int i = 0; i < N; ++i) xr[i] = fma(om, W[j][i], xr[i]);
          TmRow<N>::st(tx + 2 * N * j, xr);
        }
        tm_wait_st();
      }
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if (!TM && L.active) xs[j * N + i] = fma(om, W[j][i], xs[j * N + i]);
          R[j][i] = fma(-om, T[j][i], R[j][i]);
          r2n = fma(R[j][i], R[j][i], r2n);
        }
      r2n = cell_sum<N>(r2n, L.lane);
      if (!conv) {
        ++its;
        if (r2n <= kp.tol2 * rr0) conv = true;
        rho = rhon;
        omega = om;
        if (omega == 0.0) {
          rst = true;
          omega = 1.0;
        }
      }
    }
    half = !half;
  }
  __syncthreads();
  if (SWEEP) {
    if (CMAP) stage_tile_map<N>(TB, in, cl);
    else stage_tile_s<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
  }
  __syncthreads();
  if constexpr (TM) {
    double* bb = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double xr[N];
      TmRow<N>::ld(tx + 2 * N * j, xr);
      if (L.active)
#pragma unroll
        for (int i = 0; i < N; ++i) bb[j * N + i] = SWEEP ? fma(kp.omega, xr[i], bb[j * N + i]) : xr[i];
    }
    tm_free<128>(tm_slot);   // includes the barrier below
  } else {
  if (L.active) {
    double* bb = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i)
        bb[j * N + i] = SWEEP ? fma(kp.omega, xs[j * N + i], bb[j * N + i]) : xs[j * N + i];
  }
  __syncthreads();
  }
  if (CMAP) unstage_tile_map<N>(TB, out, cl);
  else unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
  if (valid && L.t == 0) kp.its[CMAP ? cl.cell[L.cs] : cell0 + L.cs] = conv ? its : (its | (1 << 30));
#undef tx
#undef tp
#undef tv
#undef tr
}


// ---- restarted GMRES(KR) per cell (the paper's local GMRES with the
// tridiagonal preconditioner for convection-dominated blocks) -------
// Right preconditioning (M = diag(D_T), or its tridiagonal part in DoF order with THOMAS),
// Arnoldi with modified Gram-Schmidt, Givens rotations on the Hessenberg columns, restart
// after KR steps: x += M^-1 V y, r -= D_T M^-1 V y (one operator application per cycle).
// The Krylov basis V (KR vectors) and, for Jacobi, M^-1 live in tensor memory: each lane owns
// a TMEM lane and keeps its plane of every basis vector there (2N^2 columns per vector).
// Per-cell scalars (the rotated Hessenberg columns R, g, the rotations) in shared memory,
// written by the cell's lane 0. All lanes of a warp run the same number of steps (lock-step);
// a cell that has converged inside a cycle freezes its column count jl.
template <int N, int KR> struct Gm {
  static constexpr int PSZ = 2 * N * N;                           // TMEM columns per vector
  static constexpr int COLS = (KR + 1) * PSZ;                     // basis + M^-1
  static constexpr int ALLOC = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
  static_assert(COLS <= 512, "GMRES basis must fit the SM's 512 TMEM columns");
  static constexpr int RT = KR * (KR + 1) / 2;                     // packed upper triangle
  static constexpr int SCS = RT + (KR + 1) + 2 * KR + 1;           // per-cell scalar stride (odd)
};
template <int N, int KR> constexpr size_t smem_gmres(bool thomas) {
  using G = Geo<N>;
  constexpr int PLN = G::C * G::PS;
  const int tail = (thomas ? 4 * PLN : PLN) + G::C * Gm<N, KR>::SCS;
  return sizeof(double) * (size_t)(G::TB + G::FY + (tail > 2 * PLN ? tail : 2 * PLN));
}

template <int N, bool SWEEP, bool THOMAS, int KR>
__global__ void __launch_bounds__(Geo<N>::NT)
k_gmres(KParams kp, const double* DG_RESTRICT in, const double* __restrict__ f,
        double* DG_RESTRICT out) {
  using G = Geo<N>;
  using M = Gm<N, KR>;
  static_assert(G::WARPS <= 4, "one TMEM lane quadrant per warp");
  constexpr int PLN = G::C * G::PS;
  extern __shared__ double sm[];
  __shared__ Cells<N> cl;
  __shared__ uint32_t tm_slot;
  double* TB = sm;
  double* FY = TB + G::TB;
  double* XS = FY + G::FY;           // FX / FZ (defect prologue only) alias XS and what follows
  double* SBM = XS + PLN;            // THOMAS: sub-diagonal, 1 / pivot, super-diagonal / pivot
  double* IPM = SBM + PLN;
  double* CPM = IPM + PLN;
  double* SC = THOMAS ? CPM + PLN : XS + PLN;
  double* FX = XS;
  double* FZ = XS + PLN;
  const int cell0 = block_group(kp, true) * G::C;
  const int nvalid = min(G::C, kp.ncells - cell0);
  const Lane L = lane_id<N>();
  const bool valid = L.active && L.cs < nvalid;
  Rows<N> rw;
  load_rows<N>(rw, L.t);
  // n <= 4: neighbour tiles staged with cp.async; n = 5: through registers (as in k_bicgstab)
  constexpr bool ASYNC = G::FS >= G::N3;
  if constexpr (ASYNC) {
    solver_setup<N, SWEEP, false>(kp, cl, TB, FY, FX, FZ, in, cell0, nvalid);
  } else {
    stage_tile<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
    setup<N>(kp, cl, cell0, SWEEP ? in : nullptr);
  }
  double R[N][N], W[N][N], T[N][N];
  read_plane<N>(TB, L, W);
  if (SWEEP) {
    if constexpr (ASYNC) {
      nbr_prologue_async<N, true>(kp, cl, L, TB, FY, FX, FZ, in + (size_t)cell0 * G::N3);
    } else {
      double pv0[G::PER], pv1[G::PER];
      load_nbr<N>(pv0, cl, 2, kp);
      load_nbr<N>(pv1, cl, 3, kp);
      nbr_prologue<N>(kp, cl, L, TB, FY, FX, FZ, in + (size_t)cell0 * G::N3, pv0, pv1);
    }
    plane_op<N, true, true>(kp, cl, L, rw, true, W, T, TB, FY, FX, FZ);
    __syncthreads();
    stage_tile_s<N>(TB, f + (size_t)cell0 * G::N3, nvalid);
    __syncthreads();
    read_plane<N>(TB, L, R);
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? R[j][i] - T[j][i] : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) R[j][i] = valid ? W[j][i] : 0.0;
  }
  const int po = L.cs * G::PS + L.t * G::QS;
  double* xs = XS + po;
  double* sc = SC + L.cs * M::SCS;    // [0, RT) R packed by columns, then g[KR+1], c[KR], s[KR]
  double* gv = sc + M::RT;
  double* cv = gv + KR + 1;
  double* sv = cv + KR;
  // the prologue's FX / FZ are consumed (barrier inside the TMEM allocation)
  tm_alloc<M::ALLOC>(&tm_slot);
#define tq (*(volatile uint32_t*)&tm_slot + ((uint32_t)((threadIdx.x >> 5) * 32) << 16))
  // M^-1: Jacobi in TMEM (vector slot KR), or the Thomas factors in shared memory
  if constexpr (THOMAS) {
    thomas_factor<N>(kp, cl, L, SBM, IPM, CPM, valid);
  } else {
    double dg[N][N];
    plane_inv_diag<N>(kp, cl, L, rw, dg);
#pragma unroll
    for (int j = 0; j < N; ++j) {
#pragma unroll
      for (int i = 0; i < N; ++i) dg[j][i] = valid ? dg[j][i] : 1.0;
      TmRow<N>::st(tq + KR * M::PSZ + 2 * N * j, dg[j]);
    }
  }
  double rr = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      rr = fma(R[j][i], R[j][i], rr);
      if (L.active) xs[j * N + i] = 0.0;
    }
  const double rr0 = cell_sum<N>(rr, L.lane);
  bool conv = !valid || rr0 == 0.0 || skip_cell(kp, cell0 + L.cs);
  const double lim = kp.tol2 * rr0;
  int its = 0;     // Arnoldi steps of this cell
  int steps = 0;   // Arnoldi steps of the warp (warp-uniform: the cap must not split the warp)
  // restart length: kp.krestart (dg_set_local_solver) up to the compiled basis size KR
  const int kr = (kp.krestart > 0 && kp.krestart < KR) ? kp.krestart : KR;
  // M^-1 applied to W in place
  auto precond = [&]() {
    if constexpr (THOMAS) {
      thomas_apply<N>(L, TB, SBM, IPM, CPM, W);
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double d[N];
        TmRow<N>::ld(tq + KR * M::PSZ + 2 * N * j, d);
#pragma unroll
        for (int i = 0; i < N; ++i) W[j][i] = L.active ? W[j][i] * d[i] : 0.0;
      }
    }
  };
  for (int cycle = 0;; ++cycle) {
    double b2 = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) b2 = fma(R[j][i], R[j][i], b2);
    b2 = cell_sum<N>(b2, L.lane);
    if (!conv && b2 <= lim) conv = true;
    if (__all_sync(0xffffffffu, conv || !L.active) || steps >= kp.max_it) break;
    // v_0 = r / |r|
    const double beta = sqrt(b2);
    const double ib = conv ? 0.0 : rcp_nr(beta);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = R[j][i] * ib;
      TmRow<N>::st(tq + 2 * N * j, v);
    }
    tm_wait_st();
    if (L.active && L.t == 0) gv[0] = beta;
    bool live = !conv;
    int jl = -1;
    for (int j = 0; j < kr; ++j) {
      if (__all_sync(0xffffffffu, !live || !L.active) || steps >= kp.max_it) break;
      ++steps;
      // W = M^-1 v_j;  T = D_T W
#pragma unroll
      for (int r = 0; r < N; ++r) TmRow<N>::ld(tq + j * M::PSZ + 2 * N * r, W[r]);
      precond();
      plane_op<N, false, true>(kp, cl, L, rw, true, W, T, TB, FY, FX, FZ);
      // modified Gram-Schmidt against v_0 .. v_j; h_i -> column j of R (lane 0)
      for (int i = 0; i <= j; ++i) {
        double V[N][N], h = 0.0;
#pragma unroll
        for (int r = 0; r < N; ++r) TmRow<N>::ld(tq + i * M::PSZ + 2 * N * r, V[r]);
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) h = fma(T[r][q], V[r][q], h);
        h = cell_sum<N>(h, L.lane);
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) T[r][q] = fma(-h, V[r][q], T[r][q]);
        if (live && L.active && L.t == 0) sc[j * (j + 1) / 2 + i] = h;
      }
      double hn = 0.0;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int q = 0; q < N; ++q) hn = fma(T[r][q], T[r][q], hn);
      hn = sqrt(cell_sum<N>(hn, L.lane));
      if (j + 1 < kr) {
        const double ih = (live && hn > 0.0) ? rcp_nr(hn) : 0.0;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double v[N];
#pragma unroll
          for (int q = 0; q < N; ++q) v[q] = T[r][q] * ih;
          TmRow<N>::st(tq + (j + 1) * M::PSZ + 2 * N * r, v);
        }
        tm_wait_st();
      }
      // Givens: previous rotations on column j, then the new one zeroing hn (lane 0 of the cell)
      if (live && L.active && L.t == 0) {
        double* col = sc + j * (j + 1) / 2;
        for (int i = 0; i < j; ++i) {
          const double a = col[i], b = col[i + 1];
          col[i] = cv[i] * a + sv[i] * b;
          col[i + 1] = -sv[i] * a + cv[i] * b;
        }
        const double a = col[j];
        const double rn = sqrt(a * a + hn * hn);
        const double irn = rn > 0.0 ? rcp_nr(rn) : 0.0;
        const double c = rn > 0.0 ? a * irn : 1.0, s_ = hn * irn;
        col[j] = rn;
        cv[j] = c;
        sv[j] = s_;
        const double g = gv[j];
        gv[j] = c * g;
        gv[j + 1] = -s_ * g;
      }
      __syncwarp();
      if (live) {
        jl = j;
        ++its;
        const double gn = gv[j + 1];
        if (gn * gn <= lim || hn == 0.0) live = false;
      }
    }
    // y = R^-1 g (lane 0, into g), then W = V y, W = M^-1 W, x += W, R -= D_T W
    if (L.active && L.t == 0)
      for (int i = jl; i >= 0; --i) {
        double y = gv[i];
        for (int k = i + 1; k <= jl; ++k) y = fma(-sc[k * (k + 1) / 2 + i], gv[k], y);
        gv[i] = DG_QUOT(y, sc[i * (i + 1) / 2 + i]);
      }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int q = 0; q < N; ++q) W[r][q] = 0.0;
    const int jw = __reduce_max_sync(0xffffffffu, L.active ? jl : -1);
    for (int i = 0; i <= jw; ++i) {
      double V[N][N];
#pragma unroll
      for (int r = 0; r < N; ++r) TmRow<N>::ld(tq + i * M::PSZ + 2 * N * r, V[r]);
      if (i <= jl) {
        const double y = gv[i];
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) W[r][q] = fma(y, V[r][q], W[r][q]);
      }
    }
    precond();
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int q = 0; q < N; ++q)
        if (L.active) xs[r * N + q] += W[r][q];
    plane_op<N, false, true>(kp, cl, L, rw, true, W, T, TB, FY, FX, FZ);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int q = 0; q < N; ++q) R[r][q] -= T[r][q];
  }
  tm_free<M::ALLOC>(tm_slot);
#undef tq
  if (SWEEP) stage_tile_s<N>(TB, in + (size_t)cell0 * G::N3, nvalid);
  __syncthreads();
  if (L.active) {
    double* bb = TB + L.cs * G::CTB + L.t * G::KS;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i)
        bb[j * N + i] = SWEEP ? fma(kp.omega, xs[j * N + i], bb[j * N + i]) : xs[j * N + i];
  }
  __syncthreads();
  unstage_tile<N>(TB, out + (size_t)cell0 * G::N3, nvalid);
  if (valid && L.t == 0) kp.its[cell0 + L.cs] = conv ? its : (its | (1 << 30));
}

template <int N> constexpr size_t smem_apply(bool nbr, bool faces) {
  using G = Geo<N>;
  return sizeof(double) * (size_t)(G::TB + (faces ? G::FY : 0) + (nbr ? G::FX + G::FZ : 0));
}
template <int N> constexpr size_t smem_solve(int planes) {
  using G = Geo<N>;
  return sizeof(double) * (size_t)(G::TB + G::FY + planes * G::C * G::PS);
}

}  // namespace pk
