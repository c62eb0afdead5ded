"""Times the hybrid-multigrid-preconditioned flexible CG (Alg. 1, P0 subspace) on b = 0 configs.

usage: python scripts/hybrid_solve.py [C2 C3 C5 ...] [--coarse-tol X] [--local-tol Y]
Prints one JSON line per config: outer iterations, coarse PCG iterations, wall time of the solve
(CUDA events around dg_hybrid_solve, which synchronises per iteration), true relative residual.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

args = sys.argv[1:]
def opt(name, default):
    if name in args:
        i = args.index(name)
        v = float(args[i + 1])
        del args[i:i + 2]
        return v
    return default
ctol = opt("--coarse-tol", 1e-2)
ltol = opt("--local-tol", 1e-2)
for name in args or ["C2"]:
    P = make_config(name)
    _, f = make_vectors(P)
    ctx = dg.DGContext(P)
    ft = torch.from_numpy(f).cuda()
    prm = dg.hybrid_params(n_pre=1, n_post=1, omega=1.0, local_tol=ltol, coarse_tol=ctol,
                           coarse_max_it=20000, rel_tol=1e-8, max_it=500)
    u = torch.zeros_like(ft)
    ctx.hybrid_solve(u, ft, dg.hybrid_params(max_it=1))   # warm-up (scratch, coarse matrix)
    u.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    st = ctx.hybrid_solve(u, ft, prm)
    b.record()
    torch.cuda.synchronize()
    Au = torch.empty_like(u)
    ctx.apply(u, Au)
    res = float(torch.linalg.norm(ft - Au) / torch.linalg.norm(ft))
    ms = a.elapsed_time(b)
    print(json.dumps({"config": name, "p": P.p, "n_dof": P.n_dof, "ms": round(ms, 2),
                      "dof_per_s": P.n_dof / (ms * 1e-3), "true_rel_residual": res,
                      "local_tol": prm.local_tol, "coarse_tol": prm.coarse_tol, **st}), flush=True)
    ctx.close()
