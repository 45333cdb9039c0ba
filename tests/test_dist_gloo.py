"""The slab decomposition's communication layer (dist.TorchComm) with
world_size 2 over gloo on CPU: the four collectives of the native step
program (include/walldist_b200.h: wd_comm_callbacks) -- ghost-plane ring
exchange, slab <-> pencil all_to_all, per-line carry all_gather and the
all_reduce(max) of the convergence words -- reassemble the global field
exactly and arrive in rank order."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, q):
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_09859_b200 import dist
        n0, n1, n2 = dims
        G = dist.GHOST
        glob = np.arange(n0 * n1 * n2, dtype=float).reshape(dims)
        slab = dist.Slab(n0, world, rank)
        slab.check()
        nl = slab.nl
        interior = dist.split_global(glob, world)[rank]
        ghosted = np.zeros((nl + 2 * G, n1 * n2))
        ghosted[G:G + nl] = interior.reshape(nl, -1)
        t = torch.from_numpy(ghosted)
        comm = dist.TorchComm()
        assert (comm.P, comm.rank) == (world, rank)
        comm._halo(t, nl, G)
        flat = glob.reshape(n0, -1)
        lo_expect = np.take(flat, range(slab.lo - G, slab.lo), axis=0, mode="wrap")
        hi_expect = np.take(flat, range(slab.hi, slab.hi + G), axis=0, mode="wrap")
        ok_halo = np.array_equal(t[:G].numpy(), lo_expect) and \
            np.array_equal(t[nl + G:].numpy(), hi_expect)
        # slab (nl, n1, n2) -> (P, nl, n1/P, n2) as k_pack_slab, all_to_all -> pencil
        m1 = n1 // world
        packed = interior.reshape(nl, world, m1, n2).transpose(1, 0, 2, 3).copy()
        send = torch.from_numpy(packed.ravel())
        recv = torch.empty_like(send)
        comm._alltoall(send, recv)
        pencil = recv.numpy().reshape(n0, m1, n2)
        ok_pencil = np.array_equal(pencil, glob[:, rank * m1:(rank + 1) * m1, :])
        back = torch.empty_like(send)
        comm._alltoall(torch.from_numpy(pencil.ravel().copy()), back)
        unpacked = back.numpy().reshape(world, nl, m1, n2).transpose(1, 0, 2, 3).reshape(nl, n1, n2)
        ok_back = np.array_equal(unpacked, interior)
        mine = torch.full((6,), float(rank + 1), dtype=torch.float64)
        gath = torch.empty(6 * world, dtype=torch.float64)
        comm._allgather(mine, gath)
        ok_gather = gath.view(world, 6)[:, 0].tolist() == [float(r + 1) for r in range(world)]
        stats = torch.tensor([rank * 10 + 3, 7 - rank, rank], dtype=torch.int64)
        comm._allreduce_max(stats)
        ok_red = stats.tolist() == [(world - 1) * 10 + 3, 7, world - 1]
        q.put((rank, ok_halo, ok_pencil, ok_back, ok_red, ok_gather))
        comm.close()
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("dims", [(16, 8, 5), (32, 6, 3)])
def test_torchcomm_gloo_world2(dims):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert all(r[1:]), r


def test_slab_partition_bookkeeping():
    from paper_2111_09859_b200 import dist
    s = dist.Slab(64, 4, 3)
    assert (s.nl, s.lo, s.hi, s.left, s.right) == (16, 48, 64, 2, 0)
    parts = dist.split_global(np.arange(64 * 4 * 2, dtype=float).reshape(64, 4, 2), 4)
    assert len(parts) == 4 and parts[0].shape == (16, 4, 2)
    with pytest.raises(ValueError):
        dist.Slab(30, 4, 0).check()
    with pytest.raises(ValueError):
        dist.split_global(np.zeros((30, 4)), 4)
