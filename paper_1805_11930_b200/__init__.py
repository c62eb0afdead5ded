"""B200-native matrix-free DG operator + block-Jacobi smoother (arXiv 1805.11930 hot path).

The compute lives in libdg_b200.so (hand-written fp64 CUDA for sm_100a behind the C
ABI of include/dg.h); this package is the ctypes binding.
"""
from .dg import (DG_HALO_EXTERNAL, DG_HALO_NCCL, DG_LOCAL_AUTO, DG_LOCAL_BICGSTAB,
                 DG_LOCAL_BICGSTAB_THOMAS, DG_LOCAL_CG, DG_LOCAL_GMRES, DG_LOCAL_GMRES_THOMAS,
                 DG_VARIANT_APPLY_NOFOLD, DG_VARIANT_LINE, DG_VARIANT_LINE_CG_CTA, DG_VARIANT_NO_TMEM,
                 DG_VARIANT_VOLUME_PREFETCH, EXPORTS, LIB_PATH, MASK_BOUNDARY_FACES,
                 MASK_INTERIOR_FACES, MASK_VOLUME, DGContext, DGError, halo_plan, hybrid_params,
                 load_library, make_desc, microbench_dfma, nccl_unique_id, slab_range, tables)

__all__ = ["halo_plan", "hybrid_params", "make_desc", "slab_range", "microbench_dfma", "nccl_unique_id",
           "DGContext", "DGError", "EXPORTS", "LIB_PATH", "load_library", "tables",
           "DG_HALO_EXTERNAL", "DG_HALO_NCCL", "DG_LOCAL_AUTO", "DG_LOCAL_BICGSTAB",
           "DG_LOCAL_BICGSTAB_THOMAS", "DG_LOCAL_CG", "DG_LOCAL_GMRES", "DG_LOCAL_GMRES_THOMAS",
           "DG_VARIANT_APPLY_NOFOLD", "DG_VARIANT_LINE", "DG_VARIANT_LINE_CG_CTA", "DG_VARIANT_NO_TMEM", "DG_VARIANT_VOLUME_PREFETCH",
           "MASK_BOUNDARY_FACES", "MASK_INTERIOR_FACES", "MASK_VOLUME"]
