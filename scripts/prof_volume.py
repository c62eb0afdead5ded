"""Short run for ncu: the volume-only operator (dg_apply_parts, mask = volume) on the ~8M DoF
Poisson cube of degree p (as scripts/p_sweep.py), three calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import Problem, uniform_pm1

p = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = p + 1
m = int(round((8e6 / n ** 3) ** (1 / 3)))
P = Problem(m, m, m, p, K=np.ones(m ** 3))
ctx = dg.DGContext(P)
ut = torch.from_numpy(uniform_pm1(900 + p, 0, P.n_dof)).cuda()
out = torch.empty_like(ut)
for _ in range(3):
    ctx.apply_parts(ut, out, dg.MASK_VOLUME)
torch.cuda.synchronize()
print("ok")
