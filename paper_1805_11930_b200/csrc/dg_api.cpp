// C ABI of the matrix-free DG hot path (include/dg.h): validation, the z-slab
// partition, coefficient upload with ghost layers, the halo exchange (NCCL loaded
// at run time, or caller-filled ghost layers) and kernel dispatch.
#include "dg.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <numeric>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <utility>
#include <string>
#include <vector>

#include "dg_hybrid.h"
#include "dg_pmf.h"
#include "dg_kernels.h"
#include "dg_tables.h"

namespace {

// NVTX range over one ABI call (the host-side enqueue of its kernels; SURVEY §5 phase tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

bool getenv_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && *v && *v != '0';
}


thread_local std::string g_err;

dg_status fail(dg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

dg_status cuda_fail(cudaError_t e, const char* where) {
  return fail(DG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---- minimal NCCL binding, resolved with dlopen so single-GPU use needs no NCCL ----
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat64 = 8 };
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load(std::string* why) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { *why = std::string("dlopen libnccl failed: ") + dlerror(); return false; }
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    send = (decltype(send))dlsym(h, "ncclSend");
    recv = (decltype(recv))dlsym(h, "ncclRecv");
    groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
    groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    if (!commInitRank || !commDestroy || !send || !recv || !groupStart || !groupEnd) {
      *why = "libnccl is missing required symbols";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;

}  // namespace

struct dg_ctx {
  dg_desc desc{};
  int n = 0, nd = 0;
  int z_begin = 0, z_end = 0, nzl = 0;
  int64_t ncells = 0, ndof = 0, layer_dof = 0;
  dg::Tables1D tab{};
  dg::KParams kp{};
  double* d_K = nullptr;
  double* d_bc = nullptr;      // per-cell b with ghost layers (or nullptr)
  bool has_b = false;          // any non-zero advection (selects BiCGStab for DG_LOCAL_AUTO)
  double* d_c = nullptr;
  double* d_ghost_lo = nullptr;   // [nxy][2][n^2] trace records of the lower rank's top layer
  double* d_ghost_hi = nullptr;   // ... of the upper rank's bottom layer
  double* d_send = nullptr;       // NCCL mode: [2][nxy][2][n^2] this rank's bottom / top traces
  int64_t ghost_len = 0;          // doubles per ghost buffer: nxy * 2 n^2
  cudaStream_t comm_stream = nullptr;   // NCCL mode: the halo runs here, under the interior groups
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  double* d_unew = nullptr;
  int32_t* d_its = nullptr;
  int32_t* d_gperm = nullptr;  // solver CTA -> cell group, boundary-heavy groups first
  // hybrid multigrid scratch (allocated on first use)
  double* d_Ah = nullptr;      // [7][ncells]
  double* d_cvec = nullptr;    // rh, uh, 5 coarse work vectors: [7][ncells]
  double* d_part = nullptr;    // [kPartials]
  double* d_dots = nullptr;    // [3]
  int* d_cits = nullptr;       // [1]
  double* d_hv = nullptr;      // t, r0, r1, z, p, q: [6][ndof]
  double* d_pmf = nullptr;     // stored inverses [ncells][nd][nd] (dg_pmf_setup)
  double* d_pmf_au = nullptr;  // A u of a stored-inverse sweep [ndof]
  int method = 0;  // resolved local method
  int32_t max_it = 1000;
  int32_t krestart = 0;   // GMRES restart (0: the kernel's basis size)
  ncclComm_t comm = nullptr;
  cudaStream_t last_stream = nullptr;
  bool have_stats = false;
  int32_t launches = 0;
  int64_t plan[6] = {-1, -1, 0, -1, -1, 0};  // dg_halo_plan
};

namespace {

dg_status validate(const dg_desc* d) {
  if (!d) return fail(DG_ERR_INVALID, "desc is NULL");
  if (d->nx < 1 || d->ny < 1 || d->nz < 1) return fail(DG_ERR_INVALID, "nx, ny, nz must be >= 1");
  if (!(d->Lx > 0) || !(d->Ly > 0) || !(d->Lz > 0)) return fail(DG_ERR_INVALID, "Lx, Ly, Lz must be > 0");
  if (d->p < 1 || d->p > 7) return fail(DG_ERR_INVALID, "p must be in 1..7");
  if (!(d->alpha >= 0) || !std::isfinite(d->alpha)) return fail(DG_ERR_INVALID, "alpha must be >= 0");
  for (int i = 0; i < 6; ++i)
    if (d->bc[i] != DG_BC_DIRICHLET && d->bc[i] != DG_BC_NEUMANN)
      return fail(DG_ERR_INVALID, "bc[i] must be DG_BC_DIRICHLET or DG_BC_NEUMANN");
  if (d->k_components != 1 && d->k_components != 3)
    return fail(DG_ERR_INVALID, "k_components must be 1 or 3");
  if (!d->K) return fail(DG_ERR_INVALID, "K is NULL");
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(d->b[i])) return fail(DG_ERR_INVALID, "b must be finite");
  if (d->b_cell)
    for (int64_t i = 0; i < (int64_t)d->nx * d->ny * d->nz * 3; ++i)
      if (!std::isfinite(d->b_cell[i])) return fail(DG_ERR_INVALID, "b_cell must be finite");
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks)
    return fail(DG_ERR_INVALID, "need 0 <= rank < nranks");
  if (d->nranks > d->nz) return fail(DG_ERR_INVALID, "nranks must not exceed nz (empty slab)");
  if (d->halo_mode != DG_HALO_NCCL && d->halo_mode != DG_HALO_EXTERNAL)
    return fail(DG_ERR_INVALID, "halo_mode must be DG_HALO_NCCL or DG_HALO_EXTERNAL");
  if (d->nranks > 1 && d->halo_mode == DG_HALO_NCCL && !d->nccl_id)
    return fail(DG_ERR_INVALID, "nccl_id required for nranks > 1 in NCCL halo mode");
  const int64_t N = (int64_t)d->nx * d->ny * d->nz;
  for (int64_t i = 0; i < N * d->k_components; ++i)
    if (!(d->K[i] >= 0) || !std::isfinite(d->K[i])) return fail(DG_ERR_INVALID, "K must be finite and >= 0");
  if (d->c)
    for (int64_t i = 0; i < N; ++i)
      if (!(d->c[i] >= 0) || !std::isfinite(d->c[i])) return fail(DG_ERR_INVALID, "c must be finite and >= 0");
  return DG_OK;
}

void release(dg_ctx* c) {
  if (!c) return;
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  cudaFree(c->d_K);
  cudaFree(c->d_bc);
  cudaFree(c->d_c);
  cudaFree(c->d_ghost_lo);
  cudaFree(c->d_ghost_hi);
  cudaFree(c->d_send);
  cudaFree(c->d_unew);
  cudaFree(c->d_its);
  cudaFree(c->d_gperm);
  cudaFree(c->d_Ah);
  cudaFree(c->d_cvec);
  cudaFree(c->d_part);
  cudaFree(c->d_dots);
  cudaFree(c->d_cits);
  cudaFree(c->d_hv);
  cudaFree(c->d_pmf);
  cudaFree(c->d_pmf_au);
  delete c;
}

// Halo exchange of the face traces (a neighbour enters the face terms only through
// its trace and normal derivative): each rank packs its bottom and top layers' traces (2 n^2
// doubles per column instead of the n^3 of the layer) on the call's stream, and the NCCL
// send/recv to the ranks below / above runs on the context's comm stream; the returned event
// (ev_halo) marks the arrival of both ghost buffers.
dg_status halo_start(dg_ctx* c, const double* u, cudaStream_t s) {
  NvtxRange nv("halo_traces");
  const int64_t* pl = c->plan;
  const size_t L = (size_t)c->ghost_len;
  const int ncol = c->desc.nx * c->desc.ny;
  cudaError_t ce = cudaSuccess;
  if (pl[3] >= 0) ce = dg::launch_pack_traces(c->desc.p, c->tab, u + pl[0], ncol, 0, c->d_send, s);
  if (ce == cudaSuccess && pl[4] >= 0)
    ce = dg::launch_pack_traces(c->desc.p, c->tab, u + pl[1], ncol, 1, c->d_send + L, s);
  if (ce == cudaSuccess) ce = cudaEventRecord(c->ev_pack, s);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0);
  if (ce != cudaSuccess) return cuda_fail(ce, "pack traces");
  ncclResult_t e = g_nccl.groupStart();
  if (pl[3] >= 0) {
    e |= g_nccl.send(c->d_send, L, ncclFloat64, (int)pl[3], c->comm, c->comm_stream);
    e |= g_nccl.recv(c->d_ghost_lo, L, ncclFloat64, (int)pl[3], c->comm, c->comm_stream);
  }
  if (pl[4] >= 0) {
    e |= g_nccl.send(c->d_send + L, L, ncclFloat64, (int)pl[4], c->comm, c->comm_stream);
    e |= g_nccl.recv(c->d_ghost_hi, L, ncclFloat64, (int)pl[4], c->comm, c->comm_stream);
  }
  e |= g_nccl.groupEnd();
  if (e != 0) return fail(DG_ERR_NCCL, "NCCL halo exchange failed");
  ce = cudaEventRecord(c->ev_halo, c->comm_stream);
  if (ce != cudaSuccess) return cuda_fail(ce, "halo event");
  return DG_OK;
}

// A launch over the slab that reads neighbour data: with nranks > 1 the cell groups off the
// ghost faces run first (while the halo is in flight, NCCL mode), then, once the ghost traces are
// there, the slab-boundary groups. Per cell the arithmetic is that of one launch (bitwise).
template <class F>
dg_status run_split(dg_ctx* c, const double* u, cudaStream_t s, const dg::KParams& kp0, F&& launch,
                    const char* what) {
  dg::KParams kp = kp0;
  if (c->desc.nranks == 1) {
    kp.gsplit = 0;
    cudaError_t e = launch(kp);
    if (e != cudaSuccess) return cuda_fail(e, what);
    c->launches += 1;
    return DG_OK;
  }
  const bool nccl = c->desc.halo_mode == DG_HALO_NCCL;
  if (nccl) {
    dg_status st = halo_start(c, u, s);
    if (st != DG_OK) return st;
  }
  kp.gsplit = 1;
  cudaError_t e = launch(kp);
  if (e == cudaSuccess && nccl) e = cudaStreamWaitEvent(s, c->ev_halo, 0);
  if (e == cudaSuccess) {
    kp.gsplit = 2;
    e = launch(kp);
  }
  if (e != cudaSuccess) return cuda_fail(e, what);
  c->launches += 2 + (nccl ? 2 : 0);
  return DG_OK;
}

// the whole halo before a launch (block SOR half-sweeps: one launch per colour)
dg_status halo_exchange(dg_ctx* c, const double* u, cudaStream_t s) {
  if (c->desc.nranks == 1 || c->desc.halo_mode == DG_HALO_EXTERNAL) return DG_OK;
  dg_status st = halo_start(c, u, s);
  if (st != DG_OK) return st;
  cudaError_t e = cudaStreamWaitEvent(s, c->ev_halo, 0);
  if (e != cudaSuccess) return cuda_fail(e, "halo wait");
  return DG_OK;
}

}  // namespace

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }
const char* dg_version(void) { return "dg-b200 0.1 (sm_100a, fp64)"; }

dg_status dg_tables(int32_t p, double* out) {
  dg::Tables1D t;
  if (!out) return fail(DG_ERR_INVALID, "out is NULL");
  if (!dg::build_tables(p, &t)) return fail(DG_ERR_INVALID, "p must be in 1..7");
  const int n = t.n;
  double* o = out;
  for (int i = 0; i < n; ++i) *o++ = t.z[i];
  for (int i = 0; i < n; ++i) *o++ = t.xq[i];
  for (int i = 0; i < n; ++i) *o++ = t.wq[i];
  for (int i = 0; i < n * n; ++i) *o++ = t.A[i];
  for (int i = 0; i < n * n; ++i) *o++ = t.D[i];
  for (int i = 0; i < n * n; ++i) *o++ = t.M[i];
  for (int i = 0; i < n; ++i) *o++ = t.d0[i];
  for (int i = 0; i < n; ++i) *o++ = t.d1[i];
  return DG_OK;
}

dg_status dg_create(const dg_desc* desc, dg_ctx** out) {
  if (!out) return fail(DG_ERR_INVALID, "out is NULL");
  *out = nullptr;
  dg_status st = validate(desc);
  if (st != DG_OK) return st;
  cudaError_t e = cudaSetDevice(desc->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, desc->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(DG_ERR_UNSUPPORTED, "this build targets sm_100a (B200); device is sm_" +
                                        std::to_string(prop.major) + std::to_string(prop.minor));
  dg_ctx* c = new dg_ctx();
  c->desc = *desc;
  c->desc.K = nullptr;
  c->desc.b_cell = nullptr;
  c->desc.c = nullptr;
  c->desc.nccl_id = nullptr;
  c->n = desc->p + 1;
  c->nd = c->n * c->n * c->n;
  const int G = desc->nranks, r = desc->rank;
  dg_slab_range(desc->nz, r, G, &c->z_begin, &c->z_end);
  dg_halo_plan(desc, c->plan);
  c->nzl = c->z_end - c->z_begin;
  const int64_t nxy = (int64_t)desc->nx * desc->ny;
  c->ncells = nxy * c->nzl;
  c->ndof = c->ncells * c->nd;
  c->layer_dof = nxy * c->nd;
  dg::build_tables(desc->p, &c->tab);
  if (!dg::upload_tables(desc->p, c->tab, &e)) { release(c); return cuda_fail(e, "upload tables"); }

  // K with one ghost z-layer on each side, always 3 components
  std::vector<double> K3((size_t)(c->nzl + 2) * nxy * 3, 0.0);
  for (int zl = -1; zl <= c->nzl; ++zl) {
    const int zg = c->z_begin + zl;
    if (zg < 0 || zg >= desc->nz) continue;
    for (int64_t col = 0; col < nxy; ++col) {
      const int64_t gc = (int64_t)zg * nxy + col;
      for (int a = 0; a < 3; ++a)
        K3[((size_t)(zl + 1) * nxy + col) * 3 + a] =
            desc->k_components == 1 ? desc->K[gc] : desc->K[gc * 3 + a];
    }
  }
  auto alloc = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes ? bytes : 8); };
  if ((e = alloc((void**)&c->d_K, K3.size() * 8)) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc K"); }
  if ((e = cudaMemcpy(c->d_K, K3.data(), K3.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) { release(c); return cuda_fail(e, "copy K"); }
  c->has_b = desc->b[0] != 0.0 || desc->b[1] != 0.0 || desc->b[2] != 0.0;
  if (desc->b_cell) {
    // per-cell b, one ghost z-layer on each side like K (the faces average both cells' b)
    c->has_b = false;
    for (int64_t i = 0; i < (int64_t)desc->nx * desc->ny * desc->nz * 3; ++i)
      if (desc->b_cell[i] != 0.0) { c->has_b = true; break; }
    std::vector<double> B3((size_t)(c->nzl + 2) * nxy * 3, 0.0);
    for (int zl = -1; zl <= c->nzl; ++zl) {
      const int zg = c->z_begin + zl;
      if (zg < 0 || zg >= desc->nz) continue;
      std::memcpy(&B3[(size_t)(zl + 1) * nxy * 3], desc->b_cell + (size_t)zg * nxy * 3, (size_t)nxy * 3 * 8);
    }
    if ((e = alloc((void**)&c->d_bc, B3.size() * 8)) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc b_cell"); }
    if ((e = cudaMemcpy(c->d_bc, B3.data(), B3.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) { release(c); return cuda_fail(e, "copy b_cell"); }
  }
  if (desc->c) {
    if ((e = alloc((void**)&c->d_c, (size_t)c->ncells * 8)) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc c"); }
    if ((e = cudaMemcpy(c->d_c, desc->c + (size_t)c->z_begin * nxy, (size_t)c->ncells * 8, cudaMemcpyHostToDevice)) != cudaSuccess) { release(c); return cuda_fail(e, "copy c"); }
  }
  c->ghost_len = nxy * 2 * c->n * c->n;
  if (G > 1) {
    // + n^3 doubles of padding: the kernels stage a neighbour as n^3 doubles from its record
    const size_t gbytes = ((size_t)c->ghost_len + (size_t)c->nd) * 8;
    if (alloc((void**)&c->d_ghost_lo, gbytes) != cudaSuccess ||
        alloc((void**)&c->d_ghost_hi, gbytes) != cudaSuccess ||
        alloc((void**)&c->d_send, (size_t)c->ghost_len * 2 * 8) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc ghosts"); }
    cudaMemset(c->d_ghost_lo, 0, gbytes);
    cudaMemset(c->d_ghost_hi, 0, gbytes);
  }
  if (alloc((void**)&c->d_unew, (size_t)c->ndof * 8) != cudaSuccess ||
      alloc((void**)&c->d_its, (size_t)c->ncells * 4) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc scratch"); }
  cudaMemset(c->d_its, 0, (size_t)c->ncells * 4);

  dg::KParams& kp = c->kp;
  kp.nx = desc->nx; kp.ny = desc->ny; kp.nzl = c->nzl; kp.ncells = (int32_t)c->ncells;
  kp.h[0] = desc->Lx / desc->nx; kp.h[1] = desc->Ly / desc->ny; kp.h[2] = desc->Lz / desc->nz;
  for (int a = 0; a < 3; ++a) kp.ih[a] = 1.0 / kp.h[a];
  {
    const double T3 = kp.h[0] * kp.h[1] * kp.h[2];
    for (int a = 0; a < 3; ++a) kp.sb[a] = T3 * desc->b[a] / kp.h[a];
    kp.fa[0] = kp.h[1] * kp.h[2];
    kp.fa[1] = kp.h[0] * kp.h[2];
    kp.fa[2] = kp.h[0] * kp.h[1];
  }
  kp.pen = desc->alpha * desc->p * (desc->p + 2);
  for (int a = 0; a < 3; ++a) kp.b[a] = desc->b[a];
  for (int f = 0; f < 4; ++f) kp.slab_face[f] = desc->bc[f] == DG_BC_DIRICHLET ? dg::FK_DIRICHLET : dg::FK_NEUMANN;
  kp.slab_face[4] = r > 0 ? dg::FK_GHOST : (desc->bc[4] == DG_BC_DIRICHLET ? dg::FK_DIRICHLET : dg::FK_NEUMANN);
  kp.slab_face[5] = r < G - 1 ? dg::FK_GHOST : (desc->bc[5] == DG_BC_DIRICHLET ? dg::FK_DIRICHLET : dg::FK_NEUMANN);
  kp.K = c->d_K;
  kp.bc = c->d_bc;
  kp.c = c->d_c;
  kp.ghost_lo = r > 0 ? c->d_ghost_lo : nullptr;
  kp.ghost_hi = r < G - 1 ? c->d_ghost_hi : nullptr;
  kp.mask = 7u;
  kp.its = c->d_its;
  kp.colour = -1;
  kp.cmap = 0;
  kp.zoff = c->z_begin;
  kp.gperm = nullptr;
  kp.variant = 0;
  {
    const char* v = std::getenv("DG_VOLUME_SLIM");
    if (v && v[0] == '0') kp.variant |= dg::VAR_VOLUME_PREFETCH;
    v = std::getenv("DG_KERNEL_FAMILY");
    if (v && v[0] == 'l') kp.variant |= dg::VAR_LINE;
  }
  if (getenv_flag("DG_NO_TMEM")) kp.variant |= dg::VAR_NO_TMEM;
  if (getenv_flag("DG_LINE_CG_CTA")) kp.variant |= dg::VAR_LINE_CG_CTA;
  if (getenv_flag("DG_APPLY_NOFOLD")) kp.variant |= dg::VAR_APPLY_NOFOLD;
  if (const int C = dg::solver_group_cells(desc->p); C > 0 && !getenv_flag("DG_NO_GPERM")) {
    // Longest-processing-time-first order for the local-solver CTAs: cells with Dirichlet faces
    // take more local iterations (the penalty stiffens their block), so the groups holding them
    // start first and the ragged tail of the launch is made of cheap groups.
    const int ng = (int)((c->ncells + C - 1) / C);
    std::vector<int> weight(ng, 0), perm(ng);
    const int64_t nx = desc->nx, ny = desc->ny, nzl = c->ncells / (nx * ny);
    for (int64_t cell = 0; cell < c->ncells; ++cell) {
      const int64_t co[3] = {cell % nx, (cell / nx) % ny, cell / (nx * ny)};
      const int64_t dims[3] = {nx, ny, nzl};
      int w = 0;
      for (int f = 0; f < 6; ++f) {
        const int64_t cc = co[f >> 1] + ((f & 1) ? 1 : -1);
        if ((cc < 0 || cc >= dims[f >> 1]) && kp.slab_face[f] == dg::FK_DIRICHLET) ++w;
      }
      weight[cell / C] += w;
    }
    for (int g = 0; g < ng; ++g) perm[g] = g;
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return weight[a] > weight[b]; });
    if (alloc((void**)&c->d_gperm, (size_t)ng * 4) != cudaSuccess) { release(c); return fail(DG_ERR_NOMEM, "cudaMalloc gperm"); }
    cudaMemcpy(c->d_gperm, perm.data(), (size_t)ng * 4, cudaMemcpyHostToDevice);
    kp.gperm = c->d_gperm;
  }
  c->method = c->has_b ? dg::LM_BICGSTAB : dg::LM_CG;
  c->max_it = 1000;

  if (G > 1 && desc->halo_mode == DG_HALO_NCCL) {
    std::string why;
    if (!g_nccl.load(&why)) { release(c); return fail(DG_ERR_NCCL, why); }
    if ((e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming)) != cudaSuccess) {
      release(c);
      return cuda_fail(e, "comm stream");
    }
    ncclUniqueId id;
    std::memcpy(&id, desc->nccl_id, sizeof(id));
    ncclResult_t ne = g_nccl.commInitRank(&c->comm, G, id, r);
    if (ne != 0) {
      c->comm = nullptr;
      release(c);
      return fail(DG_ERR_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(ne) : "error"));
    }
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { release(c); return cuda_fail(e, "create"); }
  *out = c;
  return DG_OK;
}

dg_status dg_destroy(dg_ctx* ctx) {
  if (!ctx) return fail(DG_ERR_INVALID, "ctx is NULL");
  cudaSetDevice(ctx->desc.device);
  cudaDeviceSynchronize();
  release(ctx);
  return DG_OK;
}

dg_status dg_local_range(const dg_ctx* c, int32_t* zb, int32_t* ze, int64_t* nd) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (zb) *zb = c->z_begin;
  if (ze) *ze = c->z_end;
  if (nd) *nd = c->ndof;
  return DG_OK;
}

dg_status dg_ghost_layers(dg_ctx* c, double** lo, double** hi, int64_t* ghost_len) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (lo) *lo = (double*)c->kp.ghost_lo;
  if (hi) *hi = (double*)c->kp.ghost_hi;
  if (ghost_len) *ghost_len = c->ghost_len;
  return DG_OK;
}

dg_status dg_fill_ghosts(dg_ctx* c, const double* lo, const double* hi, void* stream) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (c->desc.halo_mode != DG_HALO_EXTERNAL) return fail(DG_ERR_STATE, "context is not in external halo mode");
  cudaStream_t s = (cudaStream_t)stream;
  const int ncol = c->desc.nx * c->desc.ny;
  // the traces the neighbouring rank would send: the lower rank's top layer, the upper's bottom
  if (lo && c->kp.ghost_lo) {
    cudaError_t e = dg::launch_pack_traces(c->desc.p, c->tab, lo, ncol, 1, c->d_ghost_lo, s);
    if (e != cudaSuccess) return cuda_fail(e, "fill ghost lo");
  }
  if (hi && c->kp.ghost_hi) {
    cudaError_t e = dg::launch_pack_traces(c->desc.p, c->tab, hi, ncol, 0, c->d_ghost_hi, s);
    if (e != cudaSuccess) return cuda_fail(e, "fill ghost hi");
  }
  return DG_OK;
}

dg_status dg_set_local_solver(dg_ctx* c, int32_t method, int32_t max_it, int32_t gmres_restart) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (max_it < 1) return fail(DG_ERR_INVALID, "max_it must be >= 1");
  if (gmres_restart < 0) return fail(DG_ERR_INVALID, "gmres_restart must be >= 0");
  int m;
  if (method == DG_LOCAL_AUTO) {
    m = c->has_b ? dg::LM_BICGSTAB : dg::LM_CG;
  } else if (method == DG_LOCAL_CG) {
    m = dg::LM_CG;
  } else if (method == DG_LOCAL_BICGSTAB) {
    m = dg::LM_BICGSTAB;
  } else if (method == DG_LOCAL_BICGSTAB_THOMAS) {
    if (c->desc.p > 4) return fail(DG_ERR_UNSUPPORTED, "the tridiagonal preconditioner needs p <= 4 (plane kernels)");
    m = dg::LM_BICGSTAB_THOMAS;
  } else if (method == DG_LOCAL_GMRES || method == DG_LOCAL_GMRES_THOMAS) {
    if (c->desc.p > 4) return fail(DG_ERR_UNSUPPORTED, "local GMRES needs p <= 4 (Krylov basis in tensor memory)");
    if (c->kp.variant & dg::VAR_LINE) return fail(DG_ERR_UNSUPPORTED, "local GMRES exists in the plane kernels only");
    m = method == DG_LOCAL_GMRES ? dg::LM_GMRES : dg::LM_GMRES_THOMAS;
  } else {
    return fail(DG_ERR_INVALID, "unknown local method");
  }
  c->method = m;
  c->max_it = max_it;
  c->krestart = gmres_restart;
  return DG_OK;
}

dg_status dg_set_kernel_variant(dg_ctx* c, uint32_t variant) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (variant & ~31u) return fail(DG_ERR_INVALID, "unknown kernel variant bits");
  c->kp.variant = variant;
  return DG_OK;
}

static dg_status check_vec(const void* p, const char* name) {
  if (!p) return fail(DG_ERR_INVALID, std::string(name) + " is NULL");
  return DG_OK;
}

dg_status dg_apply_parts(dg_ctx* c, const double* u, double* Au, uint32_t mask, void* stream) {
  NvtxRange nv("dg_apply");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(Au, "Au")) return DG_ERR_INVALID;
  if (u == Au) return fail(DG_ERR_INVALID, "u and Au must not alias");
  if (mask == 0 || mask > 7) return fail(DG_ERR_INVALID, "mask must be in 1..7");
  cudaStream_t s = (cudaStream_t)stream;
  c->launches = 0;
  dg::KParams kp = c->kp;
  kp.mask = mask;
  const int p = c->desc.p;
  if (!(mask & 2u)) {   // no interior-face terms: no neighbour data, one launch
    cudaError_t e = dg::launch_apply(p, kp, u, Au, s);
    if (e != cudaSuccess) return cuda_fail(e, "apply");
    c->launches = 1;
    return DG_OK;
  }
  return run_split(c, u, s, kp, [&](const dg::KParams& k) { return dg::launch_apply(p, k, u, Au, s); }, "apply");
}

dg_status dg_apply(dg_ctx* c, const double* u, double* Au, void* stream) {
  return dg_apply_parts(c, u, Au, 7u, stream);
}

dg_status dg_block_diag_apply(dg_ctx* c, const double* u, double* Du, void* stream) {
  NvtxRange nv("dg_block_diag_apply");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(Du, "Du")) return DG_ERR_INVALID;
  if (u == Du) return fail(DG_ERR_INVALID, "u and Du must not alias");
  cudaError_t e = dg::launch_block_diag_apply(c->desc.p, c->kp, u, Du, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "block_diag_apply");
  c->launches = 1;
  return DG_OK;
}

dg_status dg_local_block_solve(dg_ctx* c, const double* d, double* du, double tol, void* stream) {
  NvtxRange nv("dg_local_block_solve");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(d, "d") || check_vec(du, "du")) return DG_ERR_INVALID;
  if (d == du) return fail(DG_ERR_INVALID, "d and du must not alias");
  if (!(tol >= 0) || !std::isfinite(tol)) return fail(DG_ERR_INVALID, "local_tol must be >= 0");
  dg::KParams kp = c->kp;
  kp.tol2 = tol * tol;
  kp.max_it = c->max_it;
  kp.krestart = c->krestart;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = dg::launch_local_solve(c->desc.p, c->method, kp, d, du, s);
  if (e != cudaSuccess) return cuda_fail(e, "local_block_solve");
  c->last_stream = s;
  c->have_stats = true;
  c->launches = 1;
  return DG_OK;
}

static dg_status sweep_impl(dg_ctx* c, const double* u, const double* f, double* u_new, double omega,
                            double tol, cudaStream_t s) {
  NvtxRange nv("dg_block_jacobi_sweep");
  if (!(tol >= 0) || !std::isfinite(tol)) return fail(DG_ERR_INVALID, "local_tol must be >= 0");
  if (!std::isfinite(omega)) return fail(DG_ERR_INVALID, "omega must be finite");
  c->launches = 0;
  dg::KParams kp = c->kp;
  kp.tol2 = tol * tol;
  kp.max_it = c->max_it;
  kp.krestart = c->krestart;
  kp.omega = omega;
  const int p = c->desc.p, m = c->method;
  dg_status st = run_split(c, u, s, kp,
                           [&](const dg::KParams& k) { return dg::launch_sweep(p, m, k, u, f, u_new, s); }, "sweep");
  if (st != DG_OK) return st;
  c->last_stream = s;
  c->have_stats = true;
  return DG_OK;
}

dg_status dg_block_jacobi_sweep(dg_ctx* c, double* u, const double* f, double omega, double tol,
                                void* stream) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f")) return DG_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  dg_status st = sweep_impl(c, u, f, c->d_unew, omega, tol, s);
  if (st != DG_OK) return st;
  // in place: the kernel reads the neighbours' u, so it writes a scratch vector copied back
  cudaError_t e = cudaMemcpyAsync(u, c->d_unew, (size_t)c->ndof * 8, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "sweep copy-back");
  return DG_OK;
}

dg_status dg_block_jacobi_sweep_to(dg_ctx* c, const double* u, const double* f, double* u_new,
                                   double omega, double tol, void* stream) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f") || check_vec(u_new, "u_new")) return DG_ERR_INVALID;
  if (u_new == u || u_new == f) return fail(DG_ERR_INVALID, "u_new must not alias u or f");
  return sweep_impl(c, u, f, u_new, omega, tol, (cudaStream_t)stream);
}

// ---- z-layer ranges (streaming: host<->device copies of one chunk under the compute of another)
dg_status dg_range_granule(const dg_ctx* c, int32_t* layers) {
  if (!c || !layers) return fail(DG_ERR_INVALID, "ctx or layers is NULL");
  const int64_t g = dg::range_group_cells(c->desc.p);
  const int64_t nxy = (int64_t)c->desc.nx * c->desc.ny;
  *layers = (int32_t)(g / std::gcd(g, nxy));
  return DG_OK;
}

static dg_status range_check(dg_ctx* c, int32_t zb, int32_t ze) {
  if (c->desc.nranks != 1) return fail(DG_ERR_INVALID, "range calls need a single slab (nranks == 1)");
  if (zb < 0 || ze > c->nzl || zb > ze) return fail(DG_ERR_INVALID, "z range outside [0, local layers]");
  int32_t g = 1;
  dg_range_granule(c, &g);
  if (zb % g != 0 || (ze % g != 0 && ze != c->nzl))
    return fail(DG_ERR_INVALID, "z range bounds must be multiples of dg_range_granule (or the last layer)");
  return DG_OK;
}

dg_status dg_apply_range(dg_ctx* c, const double* u, double* Au, int32_t z_begin, int32_t z_end,
                         void* stream) {
  NvtxRange nv("dg_apply_range");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(Au, "Au")) return DG_ERR_INVALID;
  if (u == Au) return fail(DG_ERR_INVALID, "u and Au must not alias");
  dg_status st = range_check(c, z_begin, z_end);
  if (st != DG_OK) return st;
  c->launches = 0;
  if (z_begin == z_end) return DG_OK;
  const int64_t nxy = (int64_t)c->desc.nx * c->desc.ny;
  dg::KParams kp = c->kp;
  kp.mask = 7u;
  kp.gsplit = 3;
  kp.cfirst = (int32_t)(z_begin * nxy);
  kp.clast = (int32_t)(z_end * nxy);
  cudaError_t e = dg::launch_apply(c->desc.p, kp, u, Au, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "apply_range");
  c->launches = 1;
  return DG_OK;
}

dg_status dg_block_jacobi_sweep_range(dg_ctx* c, const double* u, const double* f, double* u_new,
                                      double omega, double tol, int32_t z_begin, int32_t z_end,
                                      void* stream) {
  NvtxRange nv("dg_block_jacobi_sweep_range");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f") || check_vec(u_new, "u_new")) return DG_ERR_INVALID;
  if (u_new == u || u_new == f) return fail(DG_ERR_INVALID, "u_new must not alias u or f");
  if (!(tol >= 0) || !std::isfinite(tol)) return fail(DG_ERR_INVALID, "local_tol must be >= 0");
  if (!std::isfinite(omega)) return fail(DG_ERR_INVALID, "omega must be finite");
  dg_status st = range_check(c, z_begin, z_end);
  if (st != DG_OK) return st;
  c->launches = 0;
  if (z_begin == z_end) return DG_OK;
  const int64_t nxy = (int64_t)c->desc.nx * c->desc.ny;
  dg::KParams kp = c->kp;
  kp.tol2 = tol * tol;
  kp.max_it = c->max_it;
  kp.krestart = c->krestart;
  kp.omega = omega;
  kp.gsplit = 3;
  kp.cfirst = (int32_t)(z_begin * nxy);
  kp.clast = (int32_t)(z_end * nxy);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = dg::launch_sweep(c->desc.p, c->method, kp, u, f, u_new, s);
  if (e != cudaSuccess) return cuda_fail(e, "sweep_range");
  c->last_stream = s;
  c->have_stats = true;
  c->launches = 1;
  return DG_OK;
}

dg_status dg_block_sor_sweep(dg_ctx* c, double* u, const double* f, double omega, double tol,
                             int32_t symmetric, void* stream) {
  NvtxRange nv("dg_block_sor_sweep");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f")) return DG_ERR_INVALID;
  if (!(tol >= 0) || !std::isfinite(tol)) return fail(DG_ERR_INVALID, "local_tol must be >= 0");
  if (!std::isfinite(omega)) return fail(DG_ERR_INVALID, "omega must be finite");
  if (c->desc.nranks > 1 && c->desc.halo_mode == DG_HALO_EXTERNAL)
    return fail(DG_ERR_UNSUPPORTED, "block SOR with external halos: the ghost layers would have to be "
                                    "refreshed between the colour half-sweeps (use the NCCL halo mode)");
  cudaStream_t s = (cudaStream_t)stream;
  const int order[4] = {0, 1, 1, 0};   // forward: red, black; backward: black, red
  const int halves = symmetric ? 4 : 2;
  // p <= 3 (plane solvers with cp.async staging) and nx even: the launch enumerates the cells of
  // one colour only and updates them in place (their neighbours are of the other colour and are
  // not written); otherwise every cell is launched and the other colour passes through
  const bool compact = c->desc.p <= 3 && c->desc.nx % 2 == 0 && c->method != dg::LM_GMRES &&
                       c->method != dg::LM_GMRES_THOMAS;
  c->launches = 0;
  for (int h = 0; h < halves; ++h) {
    dg_status st = halo_exchange(c, u, s);
    if (st != DG_OK) return st;
    dg::KParams kp = c->kp;
    kp.tol2 = tol * tol;
    kp.max_it = c->max_it;
    kp.krestart = c->krestart;
    kp.omega = omega;
    kp.colour = order[h];
    kp.cmap = compact ? 1 : 0;
    cudaError_t e = cudaSuccess;
    // compact mode launches one colour only: clear the counts so that the skipped colour reads
    // 0 iterations, as in masked mode (dg_get_stats = the last half-sweep)
    if (compact) e = cudaMemsetAsync(c->d_its, 0, (size_t)c->ncells * 4, s);
    if (e == cudaSuccess) e = dg::launch_sweep(c->desc.p, c->method, kp, u, f, compact ? u : c->d_unew, s);
    if (e != cudaSuccess) return cuda_fail(e, "sor half-sweep");
    if (!compact) {
      e = cudaMemcpyAsync(u, c->d_unew, (size_t)c->ndof * 8, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return cuda_fail(e, "sor copy-back");
    }
    ++c->launches;
  }
  c->last_stream = s;
  c->have_stats = true;
  return DG_OK;
}

dg_status dg_get_stats(dg_ctx* c, dg_stats* st) {
  if (!c || !st) return fail(DG_ERR_INVALID, "NULL argument");
  if (!c->have_stats) return fail(DG_ERR_STATE, "no sweep or local solve has run");
  cudaError_t e = cudaStreamSynchronize(c->last_stream);
  if (e != cudaSuccess) return cuda_fail(e, "stats sync");
  std::vector<int32_t> its((size_t)c->ncells);
  e = cudaMemcpy(its.data(), c->d_its, its.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "stats copy");
  double s = 0, s2 = 0;
  int32_t mx = 0, mn = its.empty() ? 0 : (its[0] & ~(1 << 30));
  int64_t nonconv = 0, sum = 0;
  for (int32_t raw : its) {
    const int32_t v = raw & ~(1 << 30);
    if (raw & (1 << 30)) ++nonconv;
    s += v;
    s2 += (double)v * v;
    sum += v;
    mx = v > mx ? v : mx;
    mn = v < mn ? v : mn;
  }
  const double n = its.empty() ? 1.0 : (double)its.size();
  st->it_mean = s / n;
  st->it_std = std::sqrt(std::fmax(0.0, s2 / n - (s / n) * (s / n)));
  st->it_max = mx;
  st->it_min = mn;
  st->n_cells = c->ncells;
  st->n_nonconverged = nonconv;
  st->it_sum = sum;
  return DG_OK;
}

dg_status dg_block_jacobi_sweep_stats(dg_ctx* c, double* u, const double* f, double omega, double tol,
                                      dg_stats* st, void* stream) {
  const dg_status s = dg_block_jacobi_sweep(c, u, f, omega, tol, stream);
  return (s != DG_OK || !st) ? s : dg_get_stats(c, st);
}

dg_status dg_local_block_solve_stats(dg_ctx* c, const double* d, double* du, double tol, dg_stats* st,
                                     void* stream) {
  const dg_status s = dg_local_block_solve(c, d, du, tol, stream);
  return (s != DG_OK || !st) ? s : dg_get_stats(c, st);
}

int32_t dg_last_launch_count(const dg_ctx* c) { return c ? c->launches : 0; }

dg_status dg_slab_range(int32_t nz, int32_t rank, int32_t nranks, int32_t* zb, int32_t* ze) {
  if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || nranks > nz || !zb || !ze)
    return fail(DG_ERR_INVALID, "need nz >= nranks >= 1, 0 <= rank < nranks, non-NULL outputs");
  *zb = (int32_t)((int64_t)rank * nz / nranks);
  *ze = (int32_t)((int64_t)(rank + 1) * nz / nranks);
  return DG_OK;
}

dg_status dg_halo_plan(const dg_desc* d, int64_t out[6]) {
  if (!d || !out) return fail(DG_ERR_INVALID, "NULL argument");
  if (d->p < 1 || d->p > 7 || d->nx < 1 || d->ny < 1) return fail(DG_ERR_INVALID, "bad desc");
  int32_t zb, ze;
  dg_status st = dg_slab_range(d->nz, d->rank, d->nranks, &zb, &ze);
  if (st != DG_OK) return st;
  const int64_t n = d->p + 1, layer = (int64_t)d->nx * d->ny * n * n * n;
  const int64_t nzl = ze - zb;
  out[0] = d->rank > 0 ? 0 : -1;
  out[1] = d->rank < d->nranks - 1 ? (nzl - 1) * layer : -1;
  out[2] = layer;
  out[3] = d->rank > 0 ? d->rank - 1 : -1;
  out[4] = d->rank < d->nranks - 1 ? d->rank + 1 : -1;
  out[5] = nzl * layer;
  return DG_OK;
}

dg_status dg_nccl_unique_id(void* out128) {
  if (!out128) return fail(DG_ERR_INVALID, "out is NULL");
  std::string why;
  if (!g_nccl.load(&why)) return fail(DG_ERR_NCCL, why);
  auto get = (ncclResult_t(*)(ncclUniqueId*))dlsym(g_nccl.h, "ncclGetUniqueId");
  if (!get) return fail(DG_ERR_NCCL, "ncclGetUniqueId missing");
  ncclUniqueId id;
  if (get(&id) != 0) return fail(DG_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof(id));
  return DG_OK;
}

dg_status dg_microbench_dfma(double* sink, int32_t blocks, int32_t iters, int64_t* flops, void* stream) {
  if (!sink || !flops || blocks < 1 || iters < 1) return fail(DG_ERR_INVALID, "bad microbench arguments");
  cudaError_t e = dg::launch_dfma_bench(sink, blocks, iters, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "dfma bench");
  *flops = (int64_t)blocks * 256 * 16 * 2 * (int64_t)iters;
  return DG_OK;
}

}  // extern "C"

// ---- hybrid multigrid (Alg. 1) -------------------------------------------------------------
namespace {

dg_status hybrid_prepare(dg_ctx* c, cudaStream_t s) {
  if (c->desc.nranks != 1)
    return fail(DG_ERR_UNSUPPORTED, "hybrid multigrid: single rank only (the coarse solve is not distributed)");
  if (c->has_b) return fail(DG_ERR_UNSUPPORTED, "hybrid multigrid: b = 0 only (outer CG)");
  if (c->d_Ah) return DG_OK;   // set only once everything below has succeeded
  const size_t N = (size_t)c->ncells, nd = (size_t)c->ndof;
  double *Ah = nullptr, *cvec = nullptr, *part = nullptr, *dts = nullptr, *hv = nullptr;
  int* cits = nullptr;
  auto drop = [&]() {
    cudaFree(Ah); cudaFree(cvec); cudaFree(part); cudaFree(dts); cudaFree(cits); cudaFree(hv);
  };
  cudaError_t e = cudaMalloc(&Ah, 7 * N * 8);
  if (e == cudaSuccess) e = cudaMalloc(&cvec, 7 * N * 8);
  if (e == cudaSuccess) e = cudaMalloc(&part, (size_t)dg::kPartials * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dts, 3 * 8);
  if (e == cudaSuccess) e = cudaMalloc(&cits, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&hv, 6 * nd * 8);
  if (e != cudaSuccess) {
    cudaGetLastError();   // clear the allocation error so later launches do not report it
    drop();
    return fail(DG_ERR_NOMEM, "hybrid multigrid scratch");
  }
  dg::KParams kp = c->kp;
  kp.mask = 7u;
  e = dg::launch_coarse_matrix(kp, Ah, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    drop();
    return cuda_fail(e, "coarse matrix");
  }
  c->d_Ah = Ah; c->d_cvec = cvec; c->d_part = part; c->d_dots = dts; c->d_cits = cits; c->d_hv = hv;
  return DG_OK;
}

dg_status check_params(const dg_hybrid_params* p) {
  if (!p) return fail(DG_ERR_INVALID, "params is NULL");
  if (p->n_pre < 0 || p->n_post < 0 || p->coarse_max_it < 1 || p->max_it < 0)
    return fail(DG_ERR_INVALID, "need n_pre, n_post, max_it >= 0 and coarse_max_it >= 1");
  if (!std::isfinite(p->omega) || !(p->local_tol >= 0) || !(p->coarse_tol >= 0) || !(p->rel_tol >= 0))
    return fail(DG_ERR_INVALID, "omega finite, tolerances >= 0");
  return DG_OK;
}

// z = V(r), Alg. 1 with u_0 = 0; *coarse_its = the coarse PCG's raw iteration word (or NULL)
dg_status vcycle(dg_ctx* c, const double* r, double* z, const dg_hybrid_params* p, cudaStream_t s,
                 int* coarse_its) {
  const int64_t nd = c->ndof;
  const int N = (int)c->ncells, n = c->desc.p + 1;
  double* t = c->d_hv;
  double* rh = c->d_cvec;
  double* uh = c->d_cvec + N;
  cudaError_t e = cudaMemsetAsync(z, 0, (size_t)nd * 8, s);
  if (e != cudaSuccess) return cuda_fail(e, "vcycle memset");
  for (int i = 0; i < p->n_pre; ++i) {   // line 1: presmooth
    dg_status st = dg_block_jacobi_sweep(c, z, r, p->omega, p->local_tol, s);
    if (st != DG_OK) return st;
  }
  dg_status st = dg_apply(c, z, t, s);   // line 2: residual
  if (st != DG_OK) return st;
  if ((e = dg::launch_sub(t, r, t, nd, s)) != cudaSuccess) return cuda_fail(e, "residual");
  if ((e = dg::launch_restrict(t, rh, N, n * n * n, s)) != cudaSuccess) return cuda_fail(e, "restrict");   // line 3
  dg::KParams kp = c->kp;
  if ((e = dg::launch_coarse_pcg(kp, c->d_Ah, rh, uh, c->d_cvec + 2 * (size_t)N, c->d_part, c->d_cits,
                                 p->coarse_tol, p->coarse_max_it, s)) != cudaSuccess)
    return cuda_fail(e, "coarse solve");   // line 4
  if ((e = dg::launch_prolongate_add(z, uh, nd, n * n * n, s)) != cudaSuccess) return cuda_fail(e, "prolongate");  // line 5
  for (int i = 0; i < p->n_post; ++i) {   // line 6: postsmooth
    st = dg_block_jacobi_sweep(c, z, r, p->omega, p->local_tol, s);
    if (st != DG_OK) return st;
  }
  if (coarse_its) {
    e = cudaMemcpyAsync(coarse_its, c->d_cits, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "coarse its");
  }
  return DG_OK;
}

dg_status dots(dg_ctx* c, const double* a0, const double* b0, const double* a1, const double* b1,
               const double* a2, const double* b2, double out[3], cudaStream_t s) {
  cudaError_t e = dg::launch_dots(a0, b0, a1, b1, a2, b2, c->ndof, c->d_part, c->d_dots, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, c->d_dots, 3 * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "dot products");
  return DG_OK;
}

}  // namespace

extern "C" {

dg_status dg_coarse_matrix(dg_ctx* c, double* Ah_host) {
  if (!c || !Ah_host) return fail(DG_ERR_INVALID, "NULL argument");
  dg_status st = hybrid_prepare(c, nullptr);
  if (st != DG_OK) return st;
  cudaError_t e = cudaMemcpy(Ah_host, c->d_Ah, 7 * (size_t)c->ncells * 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "coarse matrix copy");
  return DG_OK;
}

dg_status dg_hybrid_vcycle(dg_ctx* c, const double* r, double* z, const dg_hybrid_params* p, void* stream) {
  NvtxRange nv("dg_hybrid_vcycle");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(r, "r") || check_vec(z, "z")) return DG_ERR_INVALID;
  if (r == z) return fail(DG_ERR_INVALID, "r and z must not alias");
  dg_status st = check_params(p);
  if (st != DG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = hybrid_prepare(c, s)) != DG_OK) return st;
  return vcycle(c, r, z, p, s, nullptr);
}

dg_status dg_hybrid_solve(dg_ctx* c, double* u, const double* f, const dg_hybrid_params* p,
                          dg_hybrid_stats* out, void* stream) {
  NvtxRange nv("dg_hybrid_solve");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f")) return DG_ERR_INVALID;
  if ((const double*)u == f) return fail(DG_ERR_INVALID, "u and f must not alias");
  dg_status st = check_params(p);
  if (st != DG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = hybrid_prepare(c, s)) != DG_OK) return st;
  const int64_t nd = c->ndof;
  double* t = c->d_hv;   // used inside the V-cycle
  double* r0 = c->d_hv + nd;
  double* r1 = c->d_hv + 2 * nd;
  double* z = c->d_hv + 3 * nd;
  double* pv = c->d_hv + 4 * nd;
  double* q = c->d_hv + 5 * nd;
  dg_hybrid_stats hs{};
  int cits = 0;
  auto note_coarse = [&]() {
    const int v = cits & ~(1 << 30);
    if (v > hs.coarse_it_max) hs.coarse_it_max = v;
    if (cits & (1 << 30)) ++hs.coarse_nonconverged;
    ++hs.vcycles;
  };
  cudaError_t e;
  if ((st = dg_apply(c, u, q, s)) != DG_OK) return st;
  if ((e = dg::launch_sub(r0, f, q, nd, s)) != cudaSuccess) return cuda_fail(e, "initial residual");
  double d[3];
  if ((st = dots(c, r0, r0, nullptr, nullptr, nullptr, nullptr, d, s)) != DG_OK) return st;
  const double rr0 = d[0];
  hs.rel_residual = rr0 > 0.0 ? 1.0 : 0.0;
  if (rr0 > 0.0 && p->max_it > 0) {
    if ((st = vcycle(c, r0, z, p, s, &cits)) != DG_OK) return st;
    if ((e = cudaMemcpyAsync(pv, z, (size_t)nd * 8, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "p = z");
    if ((st = dots(c, z, r0, nullptr, nullptr, nullptr, nullptr, d, s)) != DG_OK) return st;
    note_coarse();
    double zr = d[0];
    for (int it = 1; it <= p->max_it; ++it) {
      if ((st = dg_apply(c, pv, q, s)) != DG_OK) return st;
      if ((st = dots(c, pv, q, nullptr, nullptr, nullptr, nullptr, d, s)) != DG_OK) return st;
      if (!(d[0] > 0.0)) break;   // breakdown (A or the preconditioner not SPD)
      const double alpha = zr / d[0];
      if ((e = dg::launch_axpby(u, alpha, pv, 1.0, nd, s)) != cudaSuccess) return cuda_fail(e, "u update");
      if ((e = cudaMemcpyAsync(r1, r0, (size_t)nd * 8, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "r copy");
      if ((e = dg::launch_axpby(r1, -alpha, q, 1.0, nd, s)) != cudaSuccess) return cuda_fail(e, "r update");
      if ((st = dots(c, r1, r1, nullptr, nullptr, nullptr, nullptr, d, s)) != DG_OK) return st;
      hs.iterations = it;
      hs.rel_residual = std::sqrt(d[0] / rr0);
      if (hs.rel_residual <= p->rel_tol) {
        hs.converged = 1;
        std::swap(r0, r1);
        break;
      }
      if ((st = vcycle(c, r1, z, p, s, &cits)) != DG_OK) return st;
      if ((st = dots(c, z, r1, z, r0, nullptr, nullptr, d, s)) != DG_OK) return st;
      note_coarse();
      const double beta = (d[0] - d[1]) / zr;
      zr = d[0];
      if ((e = dg::launch_axpby(pv, 1.0, z, beta, nd, s)) != cudaSuccess) return cuda_fail(e, "p update");
      std::swap(r0, r1);
    }
  } else if (rr0 == 0.0) {
    hs.converged = 1;
  }
  (void)t;
  if (out) *out = hs;
  c->launches = 0;
  return DG_OK;
}

}  // extern "C"

// ---- stored-inverse block-Jacobi smoother (NEXT-4) -------------------------------------------
namespace {
dg_status pmf_check(dg_ctx* c) {
  if (c->desc.p > 4) return fail(DG_ERR_UNSUPPORTED, "stored inverses: p <= 4 only ((p+1)^6 doubles per cell)");
  return DG_OK;
}
}  // namespace

extern "C" {

dg_status dg_pmf_setup(dg_ctx* c) {
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  dg_status st = pmf_check(c);
  if (st != DG_OK) return st;
  const int n = c->desc.p + 1, nd = n * n * n;
  if (!c->d_pmf) {
    cudaError_t e = cudaMalloc(&c->d_pmf, (size_t)c->ncells * nd * nd * 8);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_pmf_au, (size_t)c->ndof * 8);
    if (e != cudaSuccess) {
      cudaGetLastError();
      cudaFree(c->d_pmf);
      c->d_pmf = nullptr;
      return fail(DG_ERR_NOMEM, "stored inverses do not fit in device memory");
    }
  }
  dg::Mat1D m;
  dg::pmf_tables(c->tab, &m);
  dg::KParams kp = c->kp;
  kp.mask = 7u;
  cudaError_t e = dg::launch_pmf_factor(kp, m, nd, 0, (int)c->ncells, 1, c->d_pmf, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "pmf factor");
  return DG_OK;
}

dg_status dg_pmf_sweep(dg_ctx* c, double* u, const double* f, double omega, void* stream) {
  NvtxRange nv("dg_pmf_sweep");
  if (!c) return fail(DG_ERR_INVALID, "ctx is NULL");
  if (check_vec(u, "u") || check_vec(f, "f")) return DG_ERR_INVALID;
  if (!c->d_pmf) return fail(DG_ERR_STATE, "dg_pmf_setup has not run");
  if (!std::isfinite(omega)) return fail(DG_ERR_INVALID, "omega must be finite");
  cudaStream_t s = (cudaStream_t)stream;
  dg_status st = dg_apply(c, u, c->d_pmf_au, s);
  if (st != DG_OK) return st;
  const int n = c->desc.p + 1;
  cudaError_t e = dg::launch_pmf_sweep(n * n * n, (int)c->ncells, c->d_pmf, u, f, c->d_pmf_au, omega, u, s);
  if (e != cudaSuccess) return cuda_fail(e, "pmf sweep");
  c->launches = 2;
  return DG_OK;
}

dg_status dg_pmf_block(dg_ctx* c, int64_t cell, int32_t inverse, double* host_out) {
  if (!c || !host_out) return fail(DG_ERR_INVALID, "NULL argument");
  if (cell < 0 || cell >= c->ncells) return fail(DG_ERR_INVALID, "cell out of range");
  const int n = c->desc.p + 1, nd = n * n * n;
  if (nd * nd * 8 > 200 * 1024) return fail(DG_ERR_UNSUPPORTED, "block too large for shared memory (p <= 4)");
  if (inverse) {
    dg_status st = pmf_check(c);
    if (st != DG_OK) return st;
  }
  double* tmp = nullptr;
  cudaError_t e = cudaMalloc(&tmp, (size_t)nd * nd * 8);
  if (e != cudaSuccess) return fail(DG_ERR_NOMEM, "block scratch");
  dg::Mat1D m;
  dg::pmf_tables(c->tab, &m);
  dg::KParams kp = c->kp;
  kp.mask = 7u;
  e = dg::launch_pmf_factor(kp, m, nd, (int)cell, 1, inverse ? 1 : 0, tmp, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(host_out, tmp, (size_t)nd * nd * 8, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  if (e != cudaSuccess) return cuda_fail(e, "pmf block");
  if (inverse)   // the device keeps the inverse transposed (coalesced sweep reads)
    for (int i = 0; i < nd; ++i)
      for (int j = i + 1; j < nd; ++j) std::swap(host_out[(size_t)i * nd + j], host_out[(size_t)j * nd + i]);
  return DG_OK;
}

}  // extern "C"
