"""Row F1 driver: minimal-staleness planning for the stage (MSPipe §3.2).

The arithmetic lives in libmspipe (host: mspipe_plan_timeline,
mspipe_plan_min_staleness; GPU: mspipe_stale_histogram).  This module only
marshals: the C3 cap k_max from the stream, a plan k_i from stage durations,
and the StageConfig that runs it (schedule "plan": prep(i) is enqueued right
after commit(i - k_i), the Alg. 1 gate as stream order).

Paper staleness k_i >= 1 throughout (k = 1: no staleness); the stage's
ring size is k = max k_i - 1 in build units.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import _C
from .stage import MemoryStage, StageConfig


def stale_fractions(hist, k_values):
    """Share of (batch, node) updates read stale under paper staleness k
    (reading F6), computed by mspipe_plan_stale_fractions."""
    return _C.plan_stale_fractions(hist, k_values)


def k_max_for_stream(g, src, dst, batch, limit=0.5, max_d=64):
    """C3: k_max = 1 + the largest k whose stale share is <= limit (F5)."""
    hist = _C.stale_histogram(g, src, dst, batch, max_d)
    ks = list(range(1, max_d + 1))
    fr = stale_fractions(hist, ks)
    ok = [k for k, f in zip(ks, fr) if f <= limit]
    return (1 + max(ok) if ok else 1), hist


def plan(tau, num_iters, k_max):
    """Minimal k_i under C1-C3 (mspipe_plan_min_staleness); raises when C2 cannot
    be met past warm-up."""
    k, bad = _C.plan_min_staleness(tau, num_iters, k_max)
    if bad:
        raise ValueError(f"no staleness bound < k_max={k_max} keeps iteration {bad} from stalling training (C2)")
    return k


def stage_config_for_plan(base: StageConfig, k_plan) -> StageConfig:
    """The stage configuration that runs a plan: schedule "plan", ring k = max_i (i - v(i)) - 1."""
    k_plan = [int(x) for x in k_plan]
    ring = max(min(kk, i) for i, kk in enumerate(k_plan, start=1))
    return dataclasses.replace(base, schedule="plan", plan=tuple(k_plan), k=max(ring - 1, 0))


@dataclasses.dataclass
class StageProfile:
    """tau^(j) in ms for j = sample, fetch feature, fetch memory, train, update memory."""
    tau: tuple

    @classmethod
    def from_stage_timing(cls, op_ms: dict, train_ms: float, feature_ms: float = 0.0):
        """Map the library's measured ops onto the paper's five stages.  The fused
        prep does A1 (sample) and A3 (fetch memory) in one launch, so its time is
        split between stages 1 and 3 by `sample_share`; the update stage is the
        message build plus the GRU + commit.  Training (F4) and feature fetching
        (F2) are not in this library: their durations are inputs."""
        prep = op_ms.get("prep", op_ms.get("sample", 0.0) + op_ms.get("fetch", 0.0))
        sample = op_ms.get("sample", 0.5 * prep)
        fetch = prep - sample
        update = op_ms.get("build", 0.0) + op_ms.get("update", 0.0) + op_ms.get("writeback", 0.0)
        return cls((sample, feature_ms, fetch, train_ms, update))


def staleness_error_series(cfg: StageConfig, params: dict, tcsr, device, src, dst, ts, neg, ef):
    """Row F1 analytics (MSPipe §5.5, Fig. `fig:staleness_error`):
    the stage under `cfg` (staleness k, MSPipe-S if cfg.mitigation) and a k = 0
    reference stage of the same stream run in lockstep, one step each; after
    step t both still hold batch t's fetched rows, and mspipe_staleness_error
    writes ‖x − s‖_F over batch t's update targets (x = the GRU hidden input
    the stale stage consumed, s = the reference's S_{t-1} rows; reading F7).
    Returns the device f64 series [num_batches]."""
    ref_cfg = dataclasses.replace(cfg, k=0, mitigation=None, schedule="exact", plan=None, double_buffer=None)
    a, b = MemoryStage(cfg, params, tcsr, device), MemoryStage(ref_cfg, params, tcsr, device)
    for st in (a, b):
        st.bind_resident(src, dst, ts, neg, ef)
    sa, sb = a.step_ops(), b.step_ops()
    if len(sa) != len(sb):
        raise ValueError("the two schedules must commit one batch per step")
    out = torch.zeros(len(sa), dtype=torch.float64, device=device)
    F1, B, E = cfg.fanout + 1, cfg.batch, src.numel()
    for t, (oa, ob) in enumerate(zip(sa, sb), start=1):
        a.run_ops(oa)
        b.run_ops(ob)
        la, lb = a._slot(t), b._slot(t)
        n = min(B, E - (t - 1) * B)
        rows_a, stride_a = (la.h, 1) if cfg.mitigation else (la.mem, F1)
        _C.staleness_error(la.dd["winner"], la.dd["num"], n, rows_a, stride_a, lb.mem, F1, cfg.mem_dim,
                           out[t - 1:t])
    return out
