"""Host-side input preparation (not a per-batch step): the temporal CSR the
sampler reads, and the γ hyperparameter of MSPipe-S.

T-CSR: per node its incident events in stream order (ts non-decreasing, ties
by eid), a self-loop once.  γ: the p-quantile (nearest rank,
S:L107-L115) of Δt, the gap between consecutive incident events of a node
("set γ to p quantile (e.g., 99% quantile) of the Δt distribution", P:L317;
reading G16).  Both are computed once per stream, before the timed stage.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _C


def build_tcsr_host(num_nodes, src, dst, ts):
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    ts = np.asarray(ts, np.float64)
    E = len(src)
    eid = np.arange(E, dtype=np.int64)
    keep2 = dst != src
    node = np.concatenate([src, dst[keep2]])
    other = np.concatenate([dst, src[keep2]])
    e = np.concatenate([eid, eid[keep2]])
    order = np.lexsort((e, node))
    node, other, e = node[order], other[order], e[order]
    indptr = np.zeros(num_nodes + 1, np.int64)
    np.cumsum(np.bincount(node, minlength=num_nodes), out=indptr[1:])
    return dict(indptr=indptr, nbr=other.astype(np.int32), eid=e.astype(np.int32), ts=ts[e])


def build_tcsr_torch(num_nodes, src, dst, ts, device):
    """The same T-CSR built on `device`: entries in stream order (event j's src
    entry, then its dst entry unless j is a self-loop), stably sorted by node,
    so each row is in (eid, role) order — GDELT's 382M entries in well under a
    second on the GPU, where the host lexsort takes minutes."""
    dev = torch.device(device)
    s = torch.as_tensor(np.asarray(src, np.int32)).to(dev)
    d = torch.as_tensor(np.asarray(dst, np.int32)).to(dev)
    t = torch.as_tensor(np.asarray(ts, np.float64)).to(dev)
    E = s.numel()
    keep = torch.ones((E, 2), dtype=torch.bool, device=dev)
    keep[:, 1] = s != d  # a self-loop is one entry
    keep = keep.reshape(-1)
    node = torch.stack([s, d], 1).reshape(-1)[keep]
    order = torch.sort(node, stable=True).indices
    del node
    other = torch.stack([d, s], 1).reshape(-1)[keep][order]
    e = torch.arange(E, dtype=torch.int32, device=dev).repeat_interleave(2)[keep][order]
    del order, keep
    cnt = torch.bincount(torch.cat([s, d[s != d]]).long(), minlength=num_nodes)
    indptr = torch.zeros(num_nodes + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt, 0, out=indptr[1:])
    return dict(indptr=indptr, nbr=other.contiguous(), eid=e.contiguous(), ts=t[e.long()].contiguous())


def build_tcsr(num_nodes, src, dst, ts, device) -> _C.TcsrHandle:
    t = build_tcsr_torch(num_nodes, src, dst, ts, device)
    return _C.TcsrHandle(num_nodes, t["indptr"], t["nbr"], t["eid"], t["ts"])


def gamma_quantile(num_nodes, src, dst, ts, p=0.99):
    h = build_tcsr_host(num_nodes, src, dst, ts)
    d = np.diff(h["ts"])
    first = np.zeros(len(h["ts"]), bool)
    first[h["indptr"][:-1][h["indptr"][:-1] < len(first)]] = True
    gaps = d[~first[1:]]
    if len(gaps) == 0:
        raise ValueError("no Δt observations")
    gaps.sort()
    r = min(max(int(math.ceil(p * len(gaps))), 1), len(gaps))
    return float(gaps[r - 1])
