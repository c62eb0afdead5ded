"""Diagnostic: run each hot-path call once with synchronisation after every call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors, random_problem

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
if name.startswith("C"):
    P = make_config(name)
    u, f = make_vectors(P)
else:
    P = random_problem(5, 4, 3, 3, seed=1)
    rng = np.random.default_rng(0)
    u, f = rng.uniform(-1, 1, P.n_dof), rng.uniform(-1, 1, P.n_dof)
ctx = dg.DGContext(P)
ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
Au = torch.empty_like(ut)
for step in ("apply", "solve", "sweep"):
    if step == "apply":
        ctx.apply(ut, Au)
    elif step == "solve":
        ctx.local_block_solve(ft, Au, 1e-12)
    else:
        ctx.sweep(ut, ft, 1.0, 1e-12)
    torch.cuda.synchronize()
    print(step, "ok", flush=True)
print(ctx.stats())
