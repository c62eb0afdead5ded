"""The N>1 (z-slab) path's host logic on CPU with torch.distributed gloo, world_size 2 and 3:
slab partition from the library, the halo plan, a face-layer exchange that follows the plan,
and the NCCL unique-id broadcast the bench uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1805_11930_b200 as dg
        from synth import make_config, make_vectors, random_problem
        P = random_problem(3, 2, 7, 2, seed=3) if name == "small" else make_config(name)
        zb, ze = dg.slab_range(P.nz, rank, world)
        plan = dg.halo_plan(P, rank, world)
        nxy, nd = P.nx * P.ny, P.nd
        # this rank's slab of the seeded global input (counter-based streams)
        u_loc, _ = make_vectors(P, seed=77, cell_begin=zb * nxy, cell_end=ze * nxy)
        assert plan["n_local_dof"] == u_loc.size
        L = plan["layer_dof"]
        ghost_lo = np.zeros(L)
        ghost_hi = np.zeros(L)
        reqs = []
        t_lo, t_hi = torch.from_numpy(ghost_lo), torch.from_numpy(ghost_hi)
        if plan["peer_lo"] >= 0:
            reqs.append(dist.isend(torch.from_numpy(u_loc[plan["send_lo_offset"]:plan["send_lo_offset"] + L].copy()),
                                   plan["peer_lo"]))
            reqs.append(dist.irecv(t_lo, plan["peer_lo"]))
        if plan["peer_hi"] >= 0:
            reqs.append(dist.isend(torch.from_numpy(u_loc[plan["send_hi_offset"]:plan["send_hi_offset"] + L].copy()),
                                   plan["peer_hi"]))
            reqs.append(dist.irecv(t_hi, plan["peer_hi"]))
        for r in reqs:
            r.wait()
        # the ghosts must equal the global vector's z-layers just outside the slab
        if plan["peer_lo"] >= 0:
            ref, _ = make_vectors(P, seed=77, cell_begin=(zb - 1) * nxy, cell_end=zb * nxy)
            assert np.array_equal(t_lo.numpy(), ref)
        if plan["peer_hi"] >= 0:
            ref, _ = make_vectors(P, seed=77, cell_begin=ze * nxy, cell_end=(ze + 1) * nxy)
            assert np.array_equal(t_hi.numpy(), ref)
        # slabs tile the global z range
        got = [None] * world
        dist.all_gather_object(got, (zb, ze))
        assert got[0][0] == 0 and got[-1][1] == P.nz
        assert all(got[i][1] == got[i + 1][0] for i in range(world - 1))
        # NCCL unique id broadcast (as bench.py does); skipped if libnccl cannot be loaded
        try:
            obj = [dg.nccl_unique_id() if rank == 0 else None]
        except Exception:
            obj = [b"no-nccl" if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(x == ids[0] for x in ids) and len(ids[0]) in (128, 7)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,name", [(2, "small"), (3, "small"), (2, "C5")])
def test_slab_halo_exchange_gloo(world, name):
    from paper_1805_11930_b200.build import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res


def test_slab_range_edges():
    import paper_1805_11930_b200 as dg
    assert dg.slab_range(85, 0, 8) == (0, 10)
    assert dg.slab_range(85, 7, 8) == (74, 85)
    sizes = [dg.slab_range(85, r, 8)[1] - dg.slab_range(85, r, 8)[0] for r in range(8)]
    assert sum(sizes) == 85 and set(sizes) <= {10, 11}
    with pytest.raises(Exception):
        dg.slab_range(4, 0, 5)


def _trace_worker(rank, world, port, p, q):
    """The trace-record contract of include/dg.h (dg_ghost_layers) over gloo: each rank packs its
    bottom / top layers' face traces (face values at node 0 / n-1, normal-derivative sums with
    theta'(0) / theta'(1) from the oracle's basis), exchanges them with the ranks below / above,
    and rebuilds from the received records alone the coupling of its boundary cells to the other
    rank's cells; that must equal the oracle's full neighbour blocks (tier B) applied to the
    neighbours' complete n^3 data."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1805_11930_b200 as dg
        from oracle.basis import lagrange_derivs, lobatto_nodes
        from oracle.tier_b import TierB
        from synth import make_vectors, random_problem
        P = random_problem(3, 2, 2 * world + 1, p, seed=40 + p, b=(0.4, -0.2, 0.7), c=True)
        n, nxy, nd = p + 1, P.nx * P.ny, P.nd
        zb, ze = dg.slab_range(P.nz, rank, world)
        plan = dg.halo_plan(P, rank, world)
        u_glob, _ = make_vectors(P, seed=5)
        u_loc = u_glob[zb * nxy * nd:ze * nxy * nd]
        z = lobatto_nodes(p)
        d0, d1 = lagrange_derivs(z, [0.0])[0], lagrange_derivs(z, [1.0])[0]

        def pack(layer, top):
            U = layer.reshape(nxy, n, n * n)          # [col][k][j*n + i]
            vals = U[:, n - 1 if top else 0, :]
            ders = np.einsum("k,ckf->cf", d1 if top else d0, U)
            return np.concatenate([vals, ders], axis=1).reshape(-1)   # [col][2][n^2]

        L = nxy * 2 * n * n
        got_lo, got_hi = torch.zeros(L, dtype=torch.float64), torch.zeros(L, dtype=torch.float64)
        reqs = []
        if plan["peer_lo"] >= 0:
            lay = u_loc[plan["send_lo_offset"]:plan["send_lo_offset"] + plan["layer_dof"]]
            reqs.append(dist.isend(torch.from_numpy(pack(lay, top=False)), plan["peer_lo"]))
            reqs.append(dist.irecv(got_lo, plan["peer_lo"]))
        if plan["peer_hi"] >= 0:
            lay = u_loc[plan["send_hi_offset"]:plan["send_hi_offset"] + plan["layer_dof"]]
            reqs.append(dist.isend(torch.from_numpy(pack(lay, top=True)), plan["peer_hi"]))
            reqs.append(dist.irecv(got_hi, plan["peer_hi"]))
        for r_ in reqs:
            r_.wait()
        tb = TierB(P)
        U = u_glob.reshape(-1, nd)
        Mx, My = tb.M1(0), tb.M1(1)
        MM = np.kron(My, Mx)                             # tangential face mass of a z face
        e0, e1 = np.eye(n)[0], np.eye(n)[n - 1]
        hz = tb.h[2]
        for hi, rec in ((False, got_lo.numpy()), (True, got_hi.numpy())):
            if (not hi and plan["peer_lo"] < 0) or (hi and plan["peer_hi"] < 0):
                continue
            R = rec.reshape(nxy, 2, n * n)
            zc = zb if not hi else ze - 1                # the slab's boundary layer
            for col in range(nxy):
                c = zc * nxy + col
                kind, wT, wN, g, bn, KT, KN, nb = tb.face_params(c, 2, hi)
                V, D = R[col, 0], R[col, 1]              # neighbour face values, derivative sums
                if hi:   # neighbour above: F_z (x) [min(bn,0) e1 e0' - wN KN e1 d0'/h + wT KT d1 e0'/h - g e1 e0']
                    a = MM @ ((min(bn, 0.0) - g) * V - wN * KN * D / hz)
                    b = MM @ (wT * KT * V / hz)
                    got = np.outer(e1, a) + np.outer(d1, b)
                else:    # neighbour below: F_z (x) [min(-bn,0) e0 e1' + wN KN e0 d1'/h - wT KT d0 e1'/h - g e0 e1']
                    a = MM @ ((min(-bn, 0.0) - g) * V + wN * KN * D / hz)
                    b = MM @ (-wT * KT * V / hz)
                    got = np.outer(e0, a) + np.outer(d0, b)
                nb2, B = tb.nbr_face_1d(c, 2, hi)
                ref = tb.embed(2, B) @ U[nb2]
                err = np.abs(got.reshape(-1) - ref).max() / max(np.abs(ref).max(), 1e-300)
                assert err < 1e-12, (rank, hi, col, err)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,p", [(2, 1), (2, 3), (3, 2)])
def test_trace_halo_contract_gloo(world, p):
    from paper_1805_11930_b200.build import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_trace_worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res
