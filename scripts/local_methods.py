"""One block-Jacobi sweep with each local Krylov method (BiCGStab / GMRES(7), diagonal or
tridiagonal preconditioner) on the convection configuration C4 (64^3, Q3, eps = 1e-3, cell
Peclet ~18) and on C4 with eps = 1e-6 (cell Peclet ~1.8e4, the NEXT-3 regime): sweep time
(CUDA events, 3 calls after one warm-up), local iteration counts (operator applications per
cell: BiCGStab 2 per iteration, GMRES 1 per Arnoldi step + 1 per restart cycle)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

METHODS = (("bicgstab", dg.DG_LOCAL_BICGSTAB), ("bicgstab-thomas", dg.DG_LOCAL_BICGSTAB_THOMAS),
           ("gmres", dg.DG_LOCAL_GMRES), ("gmres-thomas", dg.DG_LOCAL_GMRES_THOMAS))

for eps_scale, label in ((1.0, "C4"), (1e-3, "C4 eps=1e-6")):
    P = make_config("C4")
    P.K = np.asarray(P.K) * eps_scale
    u, f = make_vectors(P)
    ut0, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    ref = None
    for name, m in METHODS:
        with dg.DGContext(P) as ctx:
            ctx.set_local_solver(m, 1000)
            ut = ut0.clone()
            ctx.sweep(ut, ft, 1.0, 1e-12)
            st = ctx.stats()
            if ref is None:
                ref = ut.clone()
            diff = float(torch.linalg.norm(ut - ref) / torch.linalg.norm(ref))
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            uu = ut0.clone()
            a.record()
            for _ in range(3):
                ctx.sweep(uu, ft, 1.0, 1e-12)
            e.record()
            torch.cuda.synchronize()
            print(json.dumps({"case": label, "method": name, "sweep_us": a.elapsed_time(e) * 1e3 / 3,
                              "it_mean": round(st["it_mean"], 2), "it_max": st["it_max"],
                              "n_nonconverged": st["n_nonconverged"], "rel_diff_vs_bicgstab": diff}), flush=True)
