"""One block-Jacobi sweep on a convection-diffusion cube (C4's coefficients: eps = 1e-3,
b = (1, 0.5, 0.25), Dirichlet) at a given degree: sweep time (CUDA events, 3 calls after a
warm-up) and local BiCGStab iterations. usage: python scripts/conv_sweep.py P MESH"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import random_problem, uniform_pm1

p, m = int(sys.argv[1]), int(sys.argv[2])
P = random_problem(m, m, m, p, seed=77, b=(1.0, 0.5, 0.25), spread=0.0, aniso=False)
P.K = np.full(P.n_cells, 1e-3)
u, f = uniform_pm1(78, 0, P.n_dof), uniform_pm1(79, 0, P.n_dof)
with dg.DGContext(P) as ctx:
    ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    w = ut.clone()
    ctx.sweep(w, ft, 1.0, 1e-12)
    st = ctx.stats()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        ctx.sweep(w, ft, 1.0, 1e-12)
    e.record()
    torch.cuda.synchronize()
    print(json.dumps({"p": p, "mesh": m, "n_dof": P.n_dof, "sweep_us": a.elapsed_time(e) * 1e3 / 3,
                      "it_mean": st["it_mean"], "n_nonconverged": st["n_nonconverged"]}), flush=True)
