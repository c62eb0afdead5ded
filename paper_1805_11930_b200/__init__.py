"""B200-native matrix-free DG operator + block-Jacobi smoother (arXiv 1805.11930 hot path).

The compute lives in libdg_b200.so (hand-written fp64 CUDA for sm_100a behind the C
ABI of include/dg.h); this package is the ctypes binding.
"""
from .dg import (halo_plan, hybrid_params, make_desc, slab_range, microbench_dfma, nccl_unique_id, DG_HALO_EXTERNAL, DG_HALO_NCCL, DG_LOCAL_AUTO, DG_LOCAL_BICGSTAB, DG_LOCAL_BICGSTAB_THOMAS, DG_LOCAL_CG, DG_LOCAL_GMRES, DG_LOCAL_GMRES_THOMAS,
                 DGContext, DGError, EXPORTS, LIB_PATH, MASK_BOUNDARY_FACES, MASK_INTERIOR_FACES,
                 MASK_VOLUME, load_library, tables)

__all__ = ["halo_plan", "hybrid_params", "make_desc", "slab_range", "microbench_dfma", "nccl_unique_id", "DGContext", "DGError", "EXPORTS", "LIB_PATH", "load_library", "tables",
           "DG_HALO_EXTERNAL", "DG_HALO_NCCL", "DG_LOCAL_AUTO", "DG_LOCAL_BICGSTAB", "DG_LOCAL_BICGSTAB_THOMAS", "DG_LOCAL_CG", "DG_LOCAL_GMRES", "DG_LOCAL_GMRES_THOMAS",
           "MASK_BOUNDARY_FACES", "MASK_INTERIOR_FACES", "MASK_VOLUME"]
