"""Per-kernel timings on one GPU for A/B work: dg_apply, the volume kernel alone, D_T, one sweep.

usage: python scripts/kernel_times.py [C2 C3 ...]   (DG_LIB selects the library build)
Prints one JSON line per config: microseconds per call (CUDA events, 20 calls after warm-up,
inputs resident) and the model fraction of the derived fp64 peak (SURVEY 8(d) flop model).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1805_11930_b200 as dg
from synth import make_config, make_vectors

PEAK = 148 * 64 * 2 * 1.965e9


def timed(fn, calls=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(calls):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / calls


def main(names):
    for name in names:
        P = make_config(name)
        u, f = make_vectors(P)
        ctx = dg.DGContext(P)
        ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
        out = torch.empty_like(ut)
        n = P.p + 1
        nc = P.n_cells
        # + 4 n^3 with convection, + 2 n^3 with a reaction term
        vol = 24 * n ** 4 + 8 * n ** 3 + (4 * n ** 3 if any(P.b) else 0) + (2 * n ** 3 if P.c is not None else 0)
        sf, nf = 8 * n ** 3 + 12 * n ** 2, 10 * n ** 3
        r = {"config": name, "p": P.p}
        t = timed(lambda: ctx.apply_parts(ut, out, dg.MASK_VOLUME))
        r["volume_us"], r["volume_frac"] = t, nc * vol / (t * 1e-6) / PEAK
        t = timed(lambda: ctx.apply(ut, out))
        r["apply_us"], r["apply_frac"] = t, nc * (vol + 6 * sf + 6 * nf) / (t * 1e-6) / PEAK
        t = timed(lambda: ctx.block_diag_apply(ut, out))
        r["dt_us"], r["dt_frac"] = t, nc * (vol + 6 * sf) / (t * 1e-6) / PEAK
        uu = torch.empty_like(ut)
        t = timed(lambda: ctx.sweep_to(ut, ft, uu, 1.0, 1e-12), calls=3)
        st = ctx.stats()
        it = 12 if P.local_solver == "cg" else 20
        per_it = (vol + 6 * sf + it * n ** 3) * (1 if P.local_solver == "cg" else 2)
        fl = nc * (vol + 6 * sf + 6 * nf + 4 * n ** 3) + st["it_sum"] * per_it
        r["sweep_us"], r["sweep_frac"], r["it_mean"] = t, fl / (t * 1e-6) / PEAK, st["it_mean"]
        if P.p <= 4 and not any(P.b) and "--pmf" in sys.argv:
            import time
            t0 = time.perf_counter()
            ctx.pmf_setup()
            r["pmf_setup_s"] = time.perf_counter() - t0
            uu.copy_(ut)
            t = timed(lambda: ctx.pmf_sweep(uu, ft, 1.0), calls=5)
            nd = n ** 3
            r["pmf_sweep_us"] = t
            r["pmf_inverse_GB"] = nc * nd * nd * 8 / 1e9
            # stored inverses + (u, f, Au, u_new) of the matvec kernel, over the whole sweep
            r["pmf_sweep_GBps"] = (nc * nd * nd * 8 + 4 * nc * nd * 8) / (t * 1e-6) / 1e9
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if not a.startswith("--")] or ["C2"])
