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


def _train_worker(rank, world, port, out):
    """Row F4, T7: every rank computes the oracle gradient of its local batch,
    packs it into the library's flat layout and all-reduces it through the
    product's allreduce_grads; the mean must equal the mean of all ranks' grads."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        import oracle
        from oracle import train as ot
        from paper_2402_15113_b200.train import allreduce_grads, flat_params
        from synth import CONFIGS, edge_features, gru_params, make_events, train_params
        cfg = CONFIGS["tiny"]
        src, dst, ts, neg = make_events(cfg, 0, 2000)
        M, B = cfg.mem_dim, 50
        gp = gru_params(M, cfg.mail_dim, cfg.time_dim)
        tp = train_params(M, cfg.time_dim, 16)
        graph = oracle.Graph(cfg.num_nodes, src, dst, ts)
        st = oracle.new_state(cfg.num_nodes, M, cfg.edge_dim)
        flats = []
        for r in range(world):  # the global batch of iteration 1: rank r takes events [r B, (r+1) B)
            b = slice(1000 + r * B, 1000 + (r + 1) * B)
            g = ot.train_step(cfg.num_nodes, src[b], dst[b], neg[b], ts[b], edge_features(0, b.start, B, cfg.edge_dim),
                              st["mem"], st["mem_ts"], graph, gp, tp, fanout=cfg.fanout)["grads"]
            flats.append(flat_params(g, g, M, cfg.edge_dim, cfg.time_dim, 16)[0].astype(np.float64))
        mine = torch.from_numpy(flats[rank].copy())
        n = allreduce_grads(mine)
        out[rank] = (n, (mine / n).numpy(), sum(flats) / world)
    finally:
        dist.destroy_process_group()


def test_train_gradient_allreduce_world2():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_train_worker, args=(world, port, out), nprocs=world, join=True)
    import numpy as np
    for r in range(world):
        n, got, want = out[r]
        assert n == world
        assert np.allclose(got, want, rtol=1e-12, atol=1e-15)
        assert np.abs(want).max() > 0
