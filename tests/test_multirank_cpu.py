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
