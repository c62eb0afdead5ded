"""dg_apply_parts timings per mask on one config (A/B of the apply's volume / face split)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_times import timed   # noqa: E402

for name in (sys.argv[1:] or ["C3"]):
    P = make_config(name)
    u, _ = make_vectors(P)
    ctx = dg.DGContext(P)
    ut = torch.from_numpy(u).cuda()
    out = torch.empty_like(ut)
    r = {"config": name}
    for mask in (1, 2, 4, 6, 7):
        r[f"mask{mask}_us"] = timed(lambda: ctx.apply_parts(ut, out, mask))
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    ctx.close()
