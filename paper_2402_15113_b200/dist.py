"""Process-group plumbing for row E (one process per GPU).

torch.distributed is used only at setup: to hand the library's NCCL unique id
from rank 0 to every rank, and to all-gather the ranks' receive-window IPC
handles.  The data path (stores into the peers' windows, NCCL barriers) runs
inside the library, in mspipe_memory_fetch / mspipe_memory_writeback_keyed.
"""
from __future__ import annotations

import torch.distributed as dist

from . import _C


def share_nccl_id(rank: int) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId; every rank returns the same bytes."""
    obj = [_C.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def all_gather_bytes(blob: bytes) -> list:
    """Every rank's blob, in rank order (the window handles of mspipe_shard_connect)."""
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, blob)
    return out


def connect_shards(memory) -> None:
    """Export this rank's window, gather every rank's, open the peers' (collective)."""
    _C.shard_connect(memory, all_gather_bytes(_C.shard_window_handle(memory)))
