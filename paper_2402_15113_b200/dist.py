"""Process-group plumbing for row E (one process per GPU).

torch.distributed is used only to hand the library's NCCL unique id from
rank 0 to every rank; the data-path all-to-alls run on the library-owned
NCCL communicator inside mspipe_memory_fetch / mspipe_memory_writeback_keyed.
"""
from __future__ import annotations

import torch.distributed as dist

from . import _C


def share_nccl_id(rank: int) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId; every rank returns the same bytes."""
    obj = [_C.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
