"""Builds the in-tree C-ABI library libdg_b200.so for sm_100a with nvcc (no GPU needed)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libdg_b200.so")
# one translation unit per degree n = p+1 (compiled in parallel), the dispatch, the C ABI, tables
SOURCES = [f"dg_kernels_n{n}.cu" for n in range(2, 9)] + ["dg_kernels_gmres.cu", "dg_kernels.cu", "dg_hybrid.cu",
                                                            "dg_pmf.cu", "dg_api.cpp", "dg_tables.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "dg.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    """Builds `out` (default: the in-tree libdg_b200.so). `extra` nvcc flags with another `out`
    give A/B variants of the same sources (e.g. -DDG_PL_WARPS4=1), loaded through DG_LIB."""
    if out == LIB and not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build") if out == LIB else os.path.join("/tmp", "dg_objs_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-I", INCLUDE, "-I", CSRC,
              *ARCH, *extra]
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *common, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd), flush=True)
        jobs.append((cmd, obj))
    # the biggest units first; each nvcc is single-threaded
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for r in ex.map(lambda j: subprocess.run(j[0], capture_output=not verbose, text=True), jobs):
            if r.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(r.args) + "\n" + (r.stderr or "")[-4000:])
    objs = [o for _, o in jobs]
    tmp = out + ".tmp"
    cmd = [nvcc(), "-shared", *ARCH, "-o", tmp, *objs, "-lcudart", "-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
