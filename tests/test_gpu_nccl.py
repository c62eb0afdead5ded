"""NCCL halo mode (one process per GPU, z-slabs, face traces by ncclSend/ncclRecv on the comm
stream under the interior launch): dg_apply and a sweep on 2 GPUs reproduce the single-GPU
result bit for bit. Runs only where at least two GPUs are visible; the same
kernels and split launches are covered on one GPU by the external-halo partition tests."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, p, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import paper_1805_11930_b200 as dg
        from synth import make_vectors, random_problem
        P = random_problem(6, 5, 8, p, seed=70 + p, spread=1.0)
        obj = [dg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = dg.DGContext(P, rank=rank, nranks=world, device=rank, nccl_id=obj[0])
        u, f = make_vectors(P, seed=9, cell_begin=ctx.cell_begin, cell_end=ctx.cell_end)
        ut, ft = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
        Au, un = torch.empty_like(ut), torch.empty_like(ut)
        ctx.apply(ut, Au)
        ctx.sweep_to(ut, ft, un, 0.9, 1e-12)
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, (Au.cpu().numpy(), un.cpu().numpy()))
        if rank == 0:
            one = dg.DGContext(P, device=0)
            ug, fg = make_vectors(P, seed=9)
            ug_t, fg_t = torch.from_numpy(ug).cuda(), torch.from_numpy(fg).cuda()
            A1, u1 = torch.empty_like(ug_t), torch.empty_like(ug_t)
            one.apply(ug_t, A1)
            one.sweep_to(ug_t, fg_t, u1, 0.9, 1e-12)
            assert np.array_equal(np.concatenate([a for a, _ in parts]), A1.cpu().numpy())
            assert np.array_equal(np.concatenate([s for _, s in parts]), u1.cpu().numpy())
            one.close()
        ctx.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
@pytest.mark.parametrize("p", [2, 4])
def test_nccl_two_gpus_bitwise(p):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
