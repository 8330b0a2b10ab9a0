"""Row F4 driver: the MTGNN training stage after each commit ("the
memory updater computes the updated memory, the MTGNN layer computes the
embeddings, and the loss and backward steps are performed (including
all-reduce)").  Argument marshalling only — forward, backward and SGD run in
libmspipe (mspipe_train_step / mspipe_train_sgd); the data-parallel gradient
all-reduce (reading T7) is one NCCL collective on the flat
gradient buffer through torch.distributed.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _C


def flat_params(gru_params: dict, train_params: dict, mem_dim, edge_dim, time_dim, emb_dim):
    """The flat f32 buffer of mspipe_train_layout (host), filled from the tensors."""
    total, off = _C.train_layout(mem_dim, edge_dim, time_dim, emb_dim)
    flat = np.zeros(total, np.float32)
    src = {**train_params, **{k: gru_params[k] for k in ("w_ih", "w_hh", "b_ih", "b_hh")}}
    for name in _C.TRAIN_TENSORS:
        a = np.asarray(src[name], np.float32).ravel()
        flat[off[name]:off[name] + a.size] = a
    return flat, off


def allreduce_grads(grads: torch.Tensor, group=None) -> int:
    """T7: sum the flat gradient buffer over the data-parallel ranks (one
    collective); returns the world size (the SGD step divides the rate by it)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world > 1:
        dist.all_reduce(grads, group=group)
    return world


class TrainStage:
    """Owns the flat parameter / gradient buffers (device), the gate sink of the
    updater's GEMM and a per-batch loss ring."""

    def __init__(self, gru: _C.GruHandle, gru_params: dict, train_params: dict, num_nodes, mem_dim, edge_dim,
                 time_dim, fanout, batch, lr, device, emb_dim=None, group=None, ring=4096):
        emb_dim = emb_dim or int(np.asarray(train_params["w_q"]).shape[0])
        self.dims = (mem_dim, edge_dim, time_dim, emb_dim)
        flat, self.off = flat_params(gru_params, train_params, mem_dim, edge_dim, time_dim, emb_dim)
        self.params = torch.from_numpy(flat).to(device)
        self.grads = torch.zeros_like(self.params)
        self.gru = gru
        self.lr = float(lr)
        self.group = group
        self.h = _C.TrainHandle(gru, num_nodes, emb_dim, fanout, batch, self.params, self.grads)
        self.gates = torch.empty((2 * batch, 4 * mem_dim), dtype=torch.float32, device=device)
        _C.gru_save_gates(gru, self.gates)
        self.losses = torch.zeros((ring,), dtype=torch.float64, device=device)
        self.logits = torch.zeros((2 * batch,), dtype=torch.float32, device=device)

    def close(self):
        """Detach the gate sink from the updater (its GEMM stops writing self.gates)."""
        if getattr(self, "gru", None) is not None and getattr(self.gru, "h", None):
            _C.gru_save_gates(self.gru, None)

    def __del__(self):  # self.gru outlives this object (it holds the reference)
        try:
            self.close()
        except Exception:
            pass

    def shape(self, name):
        M, He, Dt, H = self.dims
        Dx = 2 * M + He + Dt
        return dict(w_q=(H, M), w_k=(H, M + Dt), w_v=(H, M + Dt), w_o=(H, H + M), b_o=(H,), w_1=(H, 2 * H),
                    b_1=(H,), w_2=(H,), b_2=(1,), w_ih=(3 * M, Dx), w_hh=(3 * M, M), b_ih=(3 * M,),
                    b_hh=(3 * M,))[name]

    def tensor(self, name, which="params"):
        buf = self.params if which == "params" else self.grads
        shp = self.shape(name)
        n = int(np.prod(shp))
        return buf[self.off[name]:self.off[name] + n].view(shp)

    def step(self, i, num_events, samp, snap_mem, upd, workspace, sgd=True):
        """Forward + backward of batch i (after its commit), then the DP mean and SGD."""
        _C.train_step(self.h, self.gru, num_events, samp, snap_mem, upd["nodes"], upd["num"], upd["mem"], workspace,
                      self.gates, self.losses[(i - 1) % self.losses.numel():][:1], self.logits[: 2 * num_events])
        if not sgd:
            return
        world = allreduce_grads(self.grads, self.group) if self.group is not None else 1  # sum; lr / world: mean
        _C.train_sgd(self.h, self.gru, self.lr / world)
