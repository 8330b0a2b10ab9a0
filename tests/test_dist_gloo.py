"""Row E host plumbing under a real process group (gloo, world size 2, CPU):
the NCCL unique id made by rank 0 reaches every rank intact, and the local
batches / LWW key bases the ranks compute tile the global batch."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_15113_b200.dist import share_nccl_id
        from paper_2402_15113_b200.shard import key_base, local_range
        uid = share_nccl_id(rank)
        got = [None] * world
        dist.all_gather_object(got, uid)
        E, B = 5003, 100
        mine = []
        for i in range(1, 30):
            j0, j1 = local_range(i, rank, world, B, E)
            mine.append((i, j0, j1, key_base(i, rank, world, B)))
        allm = [None] * world
        dist.all_gather_object(allm, mine)
        out[rank] = (got, allm)
    finally:
        dist.destroy_process_group()


def test_nccl_id_broadcast_and_partition_world2():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        got, allm = out[r]
        assert len(got[0]) == 128 and got[0] == got[1]  # same id on every rank
        events = []
        for i in range(1, 30):
            for g in range(world):
                _, j0, j1, kb = allm[g][i - 1]
                assert kb == 2 * j0 or j0 == j1
                events.extend(range(j0, j1))
        assert events == list(range(min(5003, 29 * world * 100)))
