"""Short run for ncu: the volume-only operator (dg_apply_parts, mask = volume) of a named config
(C1-C5), three calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

P = make_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
u, _ = make_vectors(P)
ctx = dg.DGContext(P)
ut = torch.from_numpy(u).cuda()
out = torch.empty_like(ut)
for _ in range(3):
    ctx.apply_parts(ut, out, dg.MASK_VOLUME)
torch.cuda.synchronize()
print("ok")
