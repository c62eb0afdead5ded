"""Short C2 run for ncu: a few applies and sweeps (warm-up included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
P = make_config(name)
u, f = make_vectors(P)
ctx = dg.DGContext(P)
ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
Au = torch.empty_like(ut)
for _ in range(3):
    ctx.apply(ut, Au)
for _ in range(2):
    ctx.sweep_to(ut, ft, Au, 1.0, 1e-12)
torch.cuda.synchronize()
print("ok", ctx.stats())
# the volume kernel alone (dg_apply_parts, mask = volume)
for _ in range(2):
    ctx.apply_parts(ut, Au, dg.MASK_VOLUME)
torch.cuda.synchronize()
