"""Volume-only operator (dg_apply_parts, mask = volume) per degree on the ~8M DoF Poisson cube of
scripts/p_sweep.py, pure diffusion and (--gen) with a zero reaction array (the general kernels);
us per call and the SURVEY 8(d) model fraction. For A/B of library variants (DG_LIB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_11930_b200 as dg
from synth import Problem, uniform_pm1

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_times import PEAK, timed   # noqa: E402

ps = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or range(1, 8)
for p in ps:
    n = p + 1
    m = int(round((8e6 / n ** 3) ** (1 / 3)))
    P = Problem(m, m, m, p, K=np.ones(m ** 3))
    if "--gen" in sys.argv:
        P.c = np.zeros(m ** 3)
    ctx = dg.DGContext(P)
    ut = torch.from_numpy(uniform_pm1(900 + p, 0, P.n_dof)).cuda()
    out = torch.empty_like(ut)
    t = timed(lambda: ctx.apply_parts(ut, out, dg.MASK_VOLUME), calls=50)
    vol = 24 * n ** 4 + 8 * n ** 3
    print(json.dumps({"lib": os.environ.get("DG_LIB", "default"), "p": p, "gen": "--gen" in sys.argv,
                      "volume_us": round(t, 2), "frac": round(P.n_cells * vol / (t * 1e-6) / PEAK, 4)}))
    ctx.close()
