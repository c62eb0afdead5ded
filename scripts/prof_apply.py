"""Short run for ncu: a few dg_apply of one config (warm-up included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

P = make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
u, _ = make_vectors(P)
ctx = dg.DGContext(P)
ut = torch.from_numpy(u).cuda()
Au = torch.empty_like(ut)
for _ in range(3):
    ctx.apply(ut, Au)
torch.cuda.synchronize()
print("ok")
