"""One hybrid solve of C2 for an ncu launch list (where the solver time goes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

P = make_config("C2")
_, f = make_vectors(P)
ctx = dg.DGContext(P)
ft = torch.from_numpy(f).cuda()
u = torch.zeros_like(ft)
st = ctx.hybrid_solve(u, ft, dg.hybrid_params(local_tol=1e-2, coarse_tol=1e-6, rel_tol=1e-8, max_it=10))
torch.cuda.synchronize()
print(st)
