"""Thin ctypes binding of the C ABI in include/dg.h (argument marshalling only).

Every step of the hot path runs in libdg_b200.so; this module only converts a
`synth.Problem` into a `dg_desc`, passes torch CUDA tensors as raw device
pointers plus the current CUDA stream, and maps error codes to exceptions. There
is no CPU fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
# DG_LIB overrides the library path (A/B builds of the same sources); default: the in-tree build
LIB_PATH = os.environ.get("DG_LIB") or os.path.join(HERE, "libdg_b200.so")

DG_OK, DG_ERR_INVALID, DG_ERR_NOMEM, DG_ERR_CUDA, DG_ERR_NCCL, DG_ERR_STATE, DG_ERR_UNSUPPORTED = range(7)
DG_LOCAL_AUTO, DG_LOCAL_CG, DG_LOCAL_BICGSTAB, DG_LOCAL_BICGSTAB_THOMAS = 0, 1, 2, 3
DG_LOCAL_GMRES, DG_LOCAL_GMRES_THOMAS = 4, 5
DG_HALO_NCCL, DG_HALO_EXTERNAL = 0, 1
DG_VARIANT_VOLUME_PREFETCH, DG_VARIANT_LINE, DG_VARIANT_NO_TMEM, DG_VARIANT_LINE_CG_CTA = 1, 2, 4, 8
DG_VARIANT_APPLY_NOFOLD = 16
MASK_VOLUME, MASK_INTERIOR_FACES, MASK_BOUNDARY_FACES = 1, 2, 4

# every symbol include/dg.h declares (checked by the CPU tests)
EXPORTS = ["dg_create", "dg_destroy", "dg_local_range", "dg_apply", "dg_block_jacobi_sweep",
           "dg_local_block_solve", "dg_set_local_solver", "dg_get_stats", "dg_apply_parts",
           "dg_block_diag_apply", "dg_ghost_layers", "dg_fill_ghosts", "dg_tables",
           "dg_last_launch_count", "dg_last_error", "dg_version", "dg_nccl_unique_id",
           "dg_microbench_dfma", "dg_slab_range", "dg_halo_plan", "dg_coarse_matrix",
           "dg_hybrid_vcycle", "dg_hybrid_solve", "dg_block_sor_sweep", "dg_pmf_setup",
           "dg_pmf_sweep", "dg_pmf_block", "dg_block_jacobi_sweep_to", "dg_set_kernel_variant",
           "dg_range_granule", "dg_apply_range", "dg_block_jacobi_sweep_range",
           "dg_block_jacobi_sweep_stats", "dg_local_block_solve_stats"]


class DGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dg error {code}: {msg}")
        self.code = code


class dg_desc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("Lx", ctypes.c_double), ("Ly", ctypes.c_double), ("Lz", ctypes.c_double),
                ("bc", ctypes.c_int32 * 6), ("p", ctypes.c_int32), ("alpha", ctypes.c_double),
                ("k_components", ctypes.c_int32), ("K", ctypes.POINTER(ctypes.c_double)),
                ("b", ctypes.c_double * 3), ("b_cell", ctypes.POINTER(ctypes.c_double)),
                ("c", ctypes.POINTER(ctypes.c_double)),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("halo_mode", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("device", ctypes.c_int32)]


class dg_stats(ctypes.Structure):
    _fields_ = [("it_mean", ctypes.c_double), ("it_std", ctypes.c_double),
                ("it_max", ctypes.c_int32), ("it_min", ctypes.c_int32),
                ("n_cells", ctypes.c_int64), ("n_nonconverged", ctypes.c_int64),
                ("it_sum", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class dg_hybrid_params(ctypes.Structure):
    _fields_ = [("n_pre", ctypes.c_int32), ("n_post", ctypes.c_int32), ("omega", ctypes.c_double),
                ("local_tol", ctypes.c_double), ("coarse_tol", ctypes.c_double),
                ("coarse_max_it", ctypes.c_int32), ("rel_tol", ctypes.c_double),
                ("max_it", ctypes.c_int32)]


class dg_hybrid_stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("vcycles", ctypes.c_int32),
                ("coarse_it_max", ctypes.c_int32), ("coarse_nonconverged", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def hybrid_params(n_pre=1, n_post=1, omega=1.0, local_tol=1e-12, coarse_tol=1e-12,
                  coarse_max_it=10000, rel_tol=1e-8, max_it=200) -> dg_hybrid_params:
    return dg_hybrid_params(n_pre, n_post, omega, local_tol, coarse_tol, coarse_max_it, rel_tol, max_it)


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads libdg_b200.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, i32, i64, u32, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
    sig = {
        "dg_create": ([ctypes.POINTER(dg_desc), ctypes.POINTER(P)], i32),
        "dg_destroy": ([P], i32),
        "dg_local_range": ([P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i64)], i32),
        "dg_apply": ([P, P, P, P], i32),
        "dg_apply_parts": ([P, P, P, u32, P], i32),
        "dg_block_diag_apply": ([P, P, P, P], i32),
        "dg_block_jacobi_sweep": ([P, P, P, dbl, dbl, P], i32),
        "dg_local_block_solve": ([P, P, P, dbl, P], i32),
        "dg_block_sor_sweep": ([P, P, P, dbl, dbl, i32, P], i32),
        "dg_pmf_setup": ([P], i32),
        "dg_pmf_sweep": ([P, P, P, dbl, P], i32),
        "dg_pmf_block": ([P, i64, i32, ctypes.POINTER(dbl)], i32),
        "dg_set_local_solver": ([P, i32, i32, i32], i32),
        "dg_set_kernel_variant": ([P, u32], i32),
        "dg_block_jacobi_sweep_to": ([P, P, P, P, dbl, dbl, P], i32),
        "dg_range_granule": ([P, ctypes.POINTER(i32)], i32),
        "dg_apply_range": ([P, P, P, i32, i32, P], i32),
        "dg_block_jacobi_sweep_range": ([P, P, P, P, dbl, dbl, i32, i32, P], i32),
        "dg_get_stats": ([P, ctypes.POINTER(dg_stats)], i32),
        "dg_block_jacobi_sweep_stats": ([P, P, P, dbl, dbl, ctypes.POINTER(dg_stats), P], i32),
        "dg_local_block_solve_stats": ([P, P, P, dbl, ctypes.POINTER(dg_stats), P], i32),
        "dg_ghost_layers": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(i64)], i32),
        "dg_fill_ghosts": ([P, P, P, P], i32),
        "dg_tables": ([i32, ctypes.POINTER(dbl)], i32),
        "dg_last_launch_count": ([P], i32),
        "dg_last_error": ([], ctypes.c_char_p),
        "dg_version": ([], ctypes.c_char_p),
        "dg_nccl_unique_id": ([P], i32),
        "dg_microbench_dfma": ([P, i32, i32, ctypes.POINTER(i64), P], i32),
        "dg_slab_range": ([i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "dg_halo_plan": ([ctypes.POINTER(dg_desc), ctypes.POINTER(i64)], i32),
        "dg_coarse_matrix": ([P, ctypes.POINTER(dbl)], i32),
        "dg_hybrid_vcycle": ([P, P, P, ctypes.POINTER(dg_hybrid_params), P], i32),
        "dg_hybrid_solve": ([P, P, P, ctypes.POINTER(dg_hybrid_params),
                             ctypes.POINTER(dg_hybrid_stats), P], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(code):
    if code != DG_OK:
        raise DGError(code, _lib.dg_last_error().decode())


def tables(p: int):
    """The 1D tables the kernels use: dict of z, xq, wq, A, D, M, d0, d1 (numpy)."""
    import numpy as np
    lib = load_library()
    n = p + 1
    buf = (ctypes.c_double * (5 * n + 3 * n * n))()
    _check(lib.dg_tables(p, buf))
    a = np.frombuffer(buf, dtype=np.float64).copy()
    out, o = {}, 0
    for name, size in (("z", n), ("xq", n), ("wq", n), ("A", n * n), ("D", n * n), ("M", n * n),
                       ("d0", n), ("d1", n)):
        out[name] = a[o:o + size].reshape((n, n) if size == n * n else (n,))
        o += size
    return out


def slab_range(nz: int, rank: int, nranks: int):
    """Host-only: this rank's z-layers [z_begin, z_end)."""
    lib = load_library()
    zb, ze = ctypes.c_int32(), ctypes.c_int32()
    _check(lib.dg_slab_range(nz, rank, nranks, ctypes.byref(zb), ctypes.byref(ze)))
    return zb.value, ze.value


def make_desc(problem, rank: int = 0, nranks: int = 1, device: int = 0, halo_mode: int = DG_HALO_NCCL):
    """dg_desc for a synth.Problem (the arrays it points to are returned to keep them alive)."""
    import numpy as np
    P = problem
    K = np.ascontiguousarray(np.asarray(P.K, dtype=np.float64))
    c = None if P.c is None else np.ascontiguousarray(np.asarray(P.c, dtype=np.float64))
    bcl = (None if getattr(P, "b_cells", None) is None
           else np.ascontiguousarray(np.asarray(P.b_cells, dtype=np.float64).reshape(-1, 3)))
    d = dg_desc()
    d.nx, d.ny, d.nz = P.nx, P.ny, P.nz
    d.Lx, d.Ly, d.Lz = P.Lx, P.Ly, P.Lz
    d.bc[:] = list(P.bc)
    d.p = P.p
    d.alpha = P.alpha
    d.k_components = 1 if K.ndim == 1 else 3
    d.K = K.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    d.b[:] = list(P.b)
    d.b_cell = bcl.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if bcl is not None else None
    d.c = c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if c is not None else None
    d.rank, d.nranks, d.halo_mode, d.device = rank, nranks, halo_mode, device
    return d, (K, c, bcl)


def halo_plan(problem, rank: int, nranks: int) -> dict:
    """Host-only: the halo plan of dg_halo_plan as a dict."""
    lib = load_library()
    d, keep = make_desc(problem, rank, nranks)
    out = (ctypes.c_int64 * 6)()
    _check(lib.dg_halo_plan(ctypes.byref(d), out))
    keys = ["send_lo_offset", "send_hi_offset", "layer_dof", "peer_lo", "peer_hi", "n_local_dof"]
    return dict(zip(keys, list(out)))


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.dg_nccl_unique_id(buf))
    return buf.raw


def microbench_dfma(sink, blocks: int, iters: int, stream=None) -> int:
    """Launches the DFMA-throughput kernel; returns its flop count (time it with CUDA events)."""
    lib = load_library()
    flops = ctypes.c_int64()
    _check(lib.dg_microbench_dfma(_ptr(sink), blocks, iters, ctypes.byref(flops), _stream(stream)))
    return flops.value


def _ptr(t, numel=None, device=None):
    """Device pointer of a contiguous float64 CUDA tensor; with numel / device given, the size
    and the device are checked too (an undersized tensor would be read out of bounds)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("expected a contiguous float64 CUDA tensor")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"expected {numel} elements, got {t.numel()}")
    if device is not None and t.device.index != device:
        raise ValueError(f"tensor on cuda:{t.device.index}, context on cuda:{device}")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class DGContext:
    """One rank's view of the DG operator / smoother on its z-slab (dg_create ... dg_destroy)."""

    def __init__(self, problem, rank: int = 0, nranks: int = 1, device: Optional[int] = None,
                 halo_mode: int = DG_HALO_NCCL, nccl_id: Optional[bytes] = None):
        import numpy as np
        import torch
        lib = load_library()
        self.lib = lib
        self.problem = problem
        P = problem
        if device is None:
            device = torch.cuda.current_device()
        d, self._keep = make_desc(P, rank, nranks, device, halo_mode)
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        d.nccl_id = ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None
        self.device = device
        h = ctypes.c_void_p()
        _check(lib.dg_create(ctypes.byref(d), ctypes.byref(h)))
        self.h = h
        zb, ze, nd = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _check(lib.dg_local_range(h, ctypes.byref(zb), ctypes.byref(ze), ctypes.byref(nd)))
        self.z_begin, self.z_end, self.n_local_dof = zb.value, ze.value, nd.value
        nxy = P.nx * P.ny
        self.cell_begin, self.cell_end = self.z_begin * nxy, self.z_end * nxy

    def close(self):
        if getattr(self, "h", None):
            _check(self.lib.dg_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- calls ---------------------------------------------------------------
    def _v(self, t):
        """A local DoF vector of this context (size and device checked)."""
        return _ptr(t, self.n_local_dof, self.device)

    def apply(self, u, out, stream=None):
        _check(self.lib.dg_apply(self.h, self._v(u), self._v(out), _stream(stream)))
        return out

    def apply_parts(self, u, out, mask: int, stream=None):
        _check(self.lib.dg_apply_parts(self.h, self._v(u), self._v(out), mask, _stream(stream)))
        return out

    def block_diag_apply(self, u, out, stream=None):
        _check(self.lib.dg_block_diag_apply(self.h, self._v(u), self._v(out), _stream(stream)))
        return out

    def local_block_solve(self, d, du, tol: float, stream=None):
        _check(self.lib.dg_local_block_solve(self.h, self._v(d), self._v(du), float(tol), _stream(stream)))
        return du

    def sweep(self, u, f, omega: float = 1.0, tol: float = 1e-12, stream=None):
        _check(self.lib.dg_block_jacobi_sweep(self.h, self._v(u), self._v(f), float(omega), float(tol),
                                              _stream(stream)))
        return u

    def sweep_stats(self, u, f, omega: float = 1.0, tol: float = 1e-12, stream=None) -> dict:
        """dg_block_jacobi_sweep_stats: the in-place sweep and its statistics in one (synchronising) call."""
        st = dg_stats()
        _check(self.lib.dg_block_jacobi_sweep_stats(self.h, self._v(u), self._v(f), float(omega), float(tol),
                                                    ctypes.byref(st), _stream(stream)))
        return st.as_dict()

    def local_block_solve_stats(self, d, du, tol: float, stream=None) -> dict:
        st = dg_stats()
        _check(self.lib.dg_local_block_solve_stats(self.h, self._v(d), self._v(du), float(tol),
                                                   ctypes.byref(st), _stream(stream)))
        return st.as_dict()

    def sweep_to(self, u, f, u_new, omega: float = 1.0, tol: float = 1e-12, stream=None):
        """Out-of-place sweep: u_new = u + omega D^-1 (f - A u) (u_new must not alias u or f)."""
        _check(self.lib.dg_block_jacobi_sweep_to(self.h, self._v(u), self._v(f), self._v(u_new),
                                                 float(omega), float(tol), _stream(stream)))
        return u_new

    # ---- z-layer ranges (streaming chunks; single slab) ------------------------
    def range_granule(self) -> int:
        """Range bounds must be multiples of this many local z-layers (or the last layer)."""
        g = ctypes.c_int32()
        _check(self.lib.dg_range_granule(self.h, ctypes.byref(g)))
        return g.value

    def apply_range(self, u, out, z_begin: int, z_end: int, stream=None):
        """(A u) for the cells of local z-layers [z_begin, z_end) only (reads layers z_begin-1..z_end)."""
        _check(self.lib.dg_apply_range(self.h, self._v(u), self._v(out), int(z_begin), int(z_end),
                                       _stream(stream)))
        return out

    def sweep_range_to(self, u, f, u_new, z_begin: int, z_end: int, omega: float = 1.0,
                       tol: float = 1e-12, stream=None):
        """Out-of-place sweep for the cells of local z-layers [z_begin, z_end) only."""
        _check(self.lib.dg_block_jacobi_sweep_range(self.h, self._v(u), self._v(f), self._v(u_new),
                                                    float(omega), float(tol), int(z_begin), int(z_end),
                                                    _stream(stream)))
        return u_new

    def set_kernel_variant(self, variant: int = 0):
        _check(self.lib.dg_set_kernel_variant(self.h, int(variant)))

    # ---- hybrid multigrid (Alg. 1, P0 subspace) ------------------------------
    def coarse_matrix(self):
        """A^ = P^T A P as a (7, n_cells) numpy array (diagonal, then x-, x+, y-, y+, z-, z+)."""
        import numpy as np
        n = self.cell_end - self.cell_begin
        out = np.empty(7 * n, dtype=np.float64)
        _check(self.lib.dg_coarse_matrix(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out.reshape(7, n)

    def hybrid_vcycle(self, r, z, params: Optional[dg_hybrid_params] = None, stream=None):
        prm = params if params is not None else hybrid_params()
        _check(self.lib.dg_hybrid_vcycle(self.h, self._v(r), self._v(z), ctypes.byref(prm), _stream(stream)))
        return z

    def hybrid_solve(self, u, f, params: Optional[dg_hybrid_params] = None, stream=None) -> dict:
        prm = params if params is not None else hybrid_params()
        st = dg_hybrid_stats()
        _check(self.lib.dg_hybrid_solve(self.h, self._v(u), self._v(f), ctypes.byref(prm), ctypes.byref(st),
                                        _stream(stream)))
        return st.as_dict()

    def sor_sweep(self, u, f, omega: float = 1.0, tol: float = 1e-12, symmetric: bool = False, stream=None):
        """Red-black block SOR (symmetric: SSOR) sweep, u in place (Alg. 3)."""
        _check(self.lib.dg_block_sor_sweep(self.h, self._v(u), self._v(f), float(omega), float(tol),
                                           1 if symmetric else 0, _stream(stream)))
        return u

    # ---- stored-inverse block-Jacobi smoother (NEXT-4) ------------------------
    def pmf_setup(self):
        _check(self.lib.dg_pmf_setup(self.h))

    def pmf_sweep(self, u, f, omega: float = 1.0, stream=None):
        _check(self.lib.dg_pmf_sweep(self.h, self._v(u), self._v(f), float(omega), _stream(stream)))
        return u

    def pmf_block(self, cell: int, inverse: bool = False):
        import numpy as np
        nd = (self.problem.p + 1) ** 3
        out = np.empty(nd * nd, dtype=np.float64)
        _check(self.lib.dg_pmf_block(self.h, int(cell), 1 if inverse else 0,
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out.reshape(nd, nd)

    def set_local_solver(self, method: int = DG_LOCAL_AUTO, max_it: int = 1000, gmres_restart: int = 0):
        _check(self.lib.dg_set_local_solver(self.h, method, max_it, gmres_restart))

    def stats(self) -> dict:
        st = dg_stats()
        _check(self.lib.dg_get_stats(self.h, ctypes.byref(st)))
        return st.as_dict()

    def fill_ghosts(self, lo=None, hi=None, stream=None):
        _check(self.lib.dg_fill_ghosts(self.h, _ptr(lo) if lo is not None else None,
                                       _ptr(hi) if hi is not None else None, _stream(stream)))

    def launch_count(self) -> int:
        return int(self.lib.dg_last_launch_count(self.h))
