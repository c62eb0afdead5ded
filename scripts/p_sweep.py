"""Throughput per polynomial degree p = 1..7 on one B200: Poisson (K = 1, alpha = 2, Dirichlet)
on a cube of ~8M DoF per degree; dg_apply, the volume kernel, D_T and one sweep (local CG to
1e-12), with the SURVEY 8(d) model fractions of the fp64 peak (scripts/kernel_times.py model)."""
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

ARGS = [a for i, a in enumerate(sys.argv[1:]) if not a.startswith('--') and sys.argv[i] != '--variant']
for p in ([int(a) for a in ARGS] or range(1, 8)):
    n = p + 1
    m = int(round((8e6 / n ** 3) ** (1 / 3)))
    P = Problem(m, m, m, p, K=np.ones(m ** 3))
    if "--gen" in sys.argv:   # a zero reaction array: the general (convection / reaction) kernels
        P.c = np.zeros(m ** 3)
    u, f = uniform_pm1(900 + p, 0, P.n_dof), uniform_pm1(910 + p, 0, P.n_dof)
    ctx = dg.DGContext(P)
    VAR = int(sys.argv[sys.argv.index("--variant") + 1]) if "--variant" in sys.argv else 0
    ctx.set_kernel_variant(VAR)
    ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    out = torch.empty_like(ut)
    nc = P.n_cells
    vol = 24 * n ** 4 + 8 * n ** 3
    sf, nf = 8 * n ** 3 + 12 * n ** 2, 10 * n ** 3
    r = {"p": p, "mesh": m, "n_dof": P.n_dof}
    t = timed(lambda: ctx.apply_parts(ut, out, dg.MASK_VOLUME))
    r["volume_us"], r["volume_frac"] = t, nc * vol / (t * 1e-6) / PEAK
    t = timed(lambda: ctx.apply(ut, out))
    r["apply_us"], r["apply_frac"] = t, nc * (vol + 6 * sf + 6 * nf) / (t * 1e-6) / PEAK
    r["apply_gdof_s"] = P.n_dof / (t * 1e-6) / 1e9
    uu = torch.empty_like(ut)
    t = timed(lambda: ctx.sweep_to(ut, ft, uu, 1.0, 1e-12), calls=2)
    st = ctx.stats()
    fl = nc * (vol + 6 * sf + 6 * nf + 4 * n ** 3) + st["it_sum"] * (vol + 6 * sf + 12 * n ** 3)
    r["sweep_us"], r["sweep_frac"], r["it_mean"] = t, fl / (t * 1e-6) / PEAK, st["it_mean"]
    r["sweep_gdof_s"] = P.n_dof / (t * 1e-6) / 1e9
    if "--conv" in sys.argv:
        # convection-diffusion (K = 1e-2, b = (1, .5, .25)): local BiCGStab, 2 D_T per iteration
        ctx.close()
        Pc = Problem(m, m, m, p, K=np.full(m ** 3, 1e-2), b=(1.0, 0.5, 0.25))
        ctx = dg.DGContext(Pc)
        ctx.set_kernel_variant(VAR)
        t = timed(lambda: ctx.sweep_to(ut, ft, uu, 1.0, 1e-12), calls=2)
        st = ctx.stats()
        volc = vol + 4 * n ** 3
        fl = nc * (volc + 6 * sf + 6 * nf + 4 * n ** 3) + st["it_sum"] * 2 * (volc + 6 * sf + 10 * n ** 3)
        r["conv_sweep_us"], r["conv_sweep_frac"], r["conv_it_mean"] = t, fl / (t * 1e-6) / PEAK, st["it_mean"]
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
    ctx.close()
