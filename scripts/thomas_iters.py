"""Local iteration counts of one sweep, diagonal vs tridiagonal (Thomas) preconditioned BiCGStab,
on strongly convection-dominated blocks (eps = 1e-6, h = 1/16, Q3): the NEXT-3 regime."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import random_problem, uniform_pm1

for b in [(1.0, 0.0, 0.0), (1.0, 0.5, 0.3)]:
    P = random_problem(16, 16, 16, 3, seed=850, b=b, spread=0.0)
    P.K = np.asarray(P.K) * 1e-6
    u, f = uniform_pm1(851, 0, P.n_dof), uniform_pm1(852, 0, P.n_dof)
    row = {"b": b, "cell_peclet": float(np.linalg.norm(b) / 16 / 1e-6)}
    for name, m in (("jacobi", dg.DG_LOCAL_BICGSTAB), ("thomas", dg.DG_LOCAL_BICGSTAB_THOMAS)):
        with dg.DGContext(P) as ctx:
            ctx.set_local_solver(m, 1000)
            ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.sweep(ut, ft, 1.0, 1e-12)
            e.record()
            st = ctx.stats()
            row[name] = {"it_mean": st["it_mean"], "it_max": st["it_max"],
                         "n_nonconverged": st["n_nonconverged"], "sweep_ms": a.elapsed_time(e)}
    print(json.dumps(row), flush=True)
