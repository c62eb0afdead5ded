"""dg_apply us per call on the named configs (default C3), for A/B of library variants (DG_LIB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_times import timed   # noqa: E402

for name in [a for a in sys.argv[1:] if not a.startswith("--")] or ["C3"]:
    P = make_config(name)
    u, _ = make_vectors(P)
    ctx = dg.DGContext(P)
    ut = torch.from_numpy(u).cuda()
    out = torch.empty_like(ut)
    t = timed(lambda: ctx.apply(ut, out), calls=30)
    print(json.dumps({"lib": os.path.basename(os.environ.get("DG_LIB", "default")), "config": name,
                      "apply_us": round(t, 2)}), flush=True)
    ctx.close()
