"""The per-batch node-memory stage as a stream-ordered schedule of ABI calls.

For batch (iteration) i, 1-based:
    prep(i)   = A1 sampler + A2 dedup + A3 snapshot fetch of the 3B(𝒩+1) subgraph
                rows [+ A4 MSPipe-S of the 2B targets, P:L317]
                [+ F2 feature fetch on its own stream] + A5 message build;
                fused: mspipe_memory_prep + mspipe_message_build
    commit(i) = A6 GRU + A7 write-back of version i (i_upd <- i);
                fused: mspipe_gru_apply_commit (one kernel)

The staleness bound becomes an ORDER on the streams (no host waits): with the
exact schedule prep(i) is enqueued right after commit(i-1-k), so it reads
version v(i) = i-1-k (Eq. 2; the gate of Alg. 1 L8-L11 is the
library's staleness check).  k+1 snapshot slots hold the prepared batches in
flight — the paper's "K additional subgraphs".  The
grouped schedule fetches k+1 batches after one commit; the "plan" schedule
(row F1) follows per-iteration k_i.  With k >= 1 the state tables are double-
buffered, so prep(t+k) and commit(t) run concurrently on two streams.

A *step* (bench.py) is one commit and the preps enqueued with it.  Steps are
captured once into CUDA graphs and replayed (µs-scale batches are launch-bound
otherwise).
"""
from __future__ import annotations

import dataclasses
import os

import torch

from . import _C


@dataclasses.dataclass
class StageConfig:
    num_nodes: int
    mem_dim: int
    edge_dim: int
    time_dim: int
    fanout: int
    batch: int
    k: int
    schedule: str = "exact"        # "exact" | "grouped"
    mitigation: dict | None = None  # dict(lam, gamma, n_sim) or None
    fetch_mail: bool = False        # also fetch mail rows of the subgraph nodes
    precision: int = _C.FP32_3XTF32  # tcgen05 3xTF32 (fp32 parity); _C.FP32_SIMT = CUDA-core baseline
    fused: bool | None = None  # mspipe_memory_prep + message_build/gru_apply (default: when supported)
    double_buffer: bool | None = None  # two table sets (mspipe_memory_double_buffer); default: k >= 1
    plan: tuple | None = None  # schedule "plan": paper staleness k_i per iteration (row F1)
    cell: str = "gru"           # row F3: "gru" (TGN, APAN) | "rnn" (JODIE's RNNCell updater)
    mailbox: str = "immediate"  # row F3: "immediate" (G14) | "deferred" (TGL's TGN; needs fetch_mail) | "apan"
    apan: dict | None = None    # row F3, mailbox="apan": dict(w_q [M, M], w_k [M, Dm], slots=10); k = 0
    features: bool = False     # row F2: fetch node / edge features of the sampled subgraphs (bind_features)
    node_dim: int = 0          # |d_v| (GDELT 413); rows padded to a multiple of 4 floats on the device
    train: dict | None = None  # row F4: dict(params=train weights, lr, [group]) — training stage after each commit

    def use_fused(self) -> bool:
        ok = self.precision in (_C.FP32_3XTF32, _C.BF16) and self.fanout <= 31 and self.batch <= 8192
        return ok if self.fused is None else (self.fused and ok)

    def use_double_buffer(self) -> bool:
        if self.mailbox == "apan":  # one table set: the commit waits for the fetch and the APAN build
            return False
        return self.k >= 1 if self.double_buffer is None else bool(self.double_buffer)


# timing diagnostics (scripts/exp_overlap.py): "prep" or "commit" runs only that half of every
# step (results are meaningless); unset in every real run
_DEBUG_ONLY = os.environ.get("MSPIPE_DEBUG_ONLY", "")
_E2E_SKIP = os.environ.get("MSPIPE_E2E_SKIP", "")  # "h2d" | "d2h": drop that copy (e2e timing diagnostics)


def plan_versions(plan, nb):
    """v(i) = max(0, i - k_i) for a plan of paper staleness values k_i (row F1)."""
    return [max(0, i - int(plan[i - 1])) for i in range(1, nb + 1)]


def schedule_ops(nb: int, k: int, schedule: str = "exact", plan=None):
    """Stream order of prep/commit ops for batches 1..nb.  "plan": prep(i) is
    enqueued right after commit(v(i)), v(i) = max(0, i - k_i) — the Alg. 1
    gate as stream order; needs k >= max(i - v(i)) - 1."""
    ops = []
    if schedule == "plan":
        v = plan_versions(plan, nb)
        if any(i - vi > k + 1 or vi > i - 1 for i, vi in zip(range(1, nb + 1), v)):
            raise ValueError("plan needs k_i >= 1 and i - v(i) <= k + 1 (the slots in flight)")
        after = {}
        for i, vi in enumerate(v, start=1):
            after.setdefault(vi, []).append(i)
        ops += [("prep", i) for i in after.get(0, [])]
        for t in range(1, nb + 1):
            ops.append(("commit", t))
            ops += [("prep", i) for i in after.get(t, [])]
        return ops
    if schedule == "exact":
        for i in range(1, min(k, nb) + 1):
            ops.append(("prep", i))
        for t in range(1, nb + 1):
            if t + k <= nb:
                ops.append(("prep", t + k))
            ops.append(("commit", t))
    elif schedule == "grouped":
        for g0 in range(1, nb + 1, k + 1):
            grp = list(range(g0, min(g0 + k, nb) + 1))
            ops += [("prep", i) for i in grp]
            ops += [("commit", i) for i in grp]
    else:
        raise ValueError(schedule)
    return ops


def snapshot_versions(nb: int, k: int, schedule: str = "exact", plan=None):
    """v(i) the schedule reads (for checks): committed count at prep(i)."""
    v, committed = {}, 0
    for op, i in schedule_ops(nb, k, schedule, plan):
        if op == "prep":
            v[i] = committed
        else:
            committed = i
    return [v[i] for i in range(1, nb + 1)]


def _pad4(n):
    return (n + 3) // 4 * 4


class _Slot:
    def __init__(self, cfg: StageConfig, mail_stride: int, device, staged: bool, ws_bytes: int = 0):
        B, F, M = cfg.batch, cfg.fanout, cfg.mem_dim
        self.samp = _C.alloc_sample(3 * B, F, device, sub=True)
        n = 3 * B * (F + 1)
        self.mem = torch.empty((n, M), dtype=torch.float32, device=device)
        self.mem_ts = torch.empty((n,), dtype=torch.float64, device=device)
        self.mail = torch.empty((n, mail_stride), dtype=torch.float32, device=device) if cfg.fetch_mail else None
        self.mail_ts = torch.empty((n,), dtype=torch.float64, device=device) if cfg.fetch_mail else None
        self.h = torch.empty((2 * B, M), dtype=torch.float32, device=device) if cfg.mitigation else None
        self.omega = (torch.empty((2 * B, cfg.mitigation["n_sim"]), dtype=torch.int32, device=device)
                      if cfg.mitigation else None)
        self.elig = torch.empty((2 * B,), dtype=torch.uint8, device=device) if cfg.mitigation else None
        self.dd = _C.alloc_dedup(B, device)
        if cfg.features:  # row F2 outputs
            self.nfeat = (torch.empty((3 * B, F + 1, _pad4(cfg.node_dim)), dtype=torch.float32, device=device)
                          if cfg.node_dim else None)
            self.efeat = torch.empty((3 * B, F, cfg.edge_dim), dtype=torch.float32, device=device)
        if ws_bytes:  # fused path: message_build(t+k) runs ahead of gru_apply(t), so its outputs are per slot
            self.ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=device)
            self.uts = torch.empty((2 * B,), dtype=torch.float64, device=device)
            self.umail = torch.empty((2 * B, mail_stride), dtype=torch.float32, device=device)
        self.version = -1
        if staged:
            self.inp = dict(src=torch.empty(B, dtype=torch.int32, device=device),
                            dst=torch.empty(B, dtype=torch.int32, device=device),
                            neg=torch.empty(B, dtype=torch.int32, device=device),
                            ts=torch.empty(B, dtype=torch.float64, device=device),
                            ef=torch.empty((B, cfg.edge_dim), dtype=torch.float32, device=device))


class _TimedOps:
    """Optional per-op CUDA timing events (also valid under graph capture)."""

    timing = None

    def reserve_timing_events(self, n):
        """Materialise n timing events outside any stream capture (torch
        creates the CUDA event lazily at its first record)."""
        self._pool = []
        for _ in range(n):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self._pool.append(e)
        torch.cuda.synchronize()
        self.timing = {}

    timing_only = None  # optional set of op names to bracket (the others get no event nodes)

    def _ev_pair(self, name):
        """Two timing events for the library to record (name, name + '_end')."""
        if not getattr(self, "_pool", None) or len(self._pool) < 2:
            return None
        b, e = self._pool.pop(), self._pool.pop()
        self.timing.setdefault(name, []).append(b)
        self.timing.setdefault(name + "_end", []).append(e)
        return b, e

    def _ev(self, name):
        if self.timing is None:
            return None
        if self.timing_only is not None and name.removesuffix("_end") not in self.timing_only:
            return None
        if getattr(self, "_pool", None):
            e = self._pool.pop()
        else:
            e = torch.cuda.Event(enable_timing=True)
            e.record()  # materialise (not allowed under capture: reserve_timing_events first)
        _C.event_record(e)
        self.timing.setdefault(name, []).append(e)
        return e


class MemoryStage(_TimedOps):
    """Drives libmspipe over an event stream.  Inputs are either resident in
    HBM (``bind_resident``) or staged per batch from pinned host memory
    (``bind_host``: the H2D copy of the batch happens inside prep(i))."""

    def __init__(self, cfg: StageConfig, params: dict, tcsr: _C.TcsrHandle, device="cuda"):
        self.cfg = cfg
        self.device = torch.device(device)
        self.tcsr = tcsr
        self.memory = _C.MemoryHandle(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.k, self.device,
                                      double_buffer=cfg.use_double_buffer())
        self.deferred = cfg.mailbox == "deferred"
        self.apan = None
        if cfg.mailbox == "apan":  # row F3: APAN (multi-slot mailbox, attention message, propagation)
            if cfg.cell != "gru" or cfg.precision != _C.FP32_3XTF32 or cfg.apan is None or cfg.schedule != "exact":
                raise ValueError("mailbox='apan' runs on the 3xTF32 GRUCell path, exact schedule, with cfg.apan weights")
            if cfg.mitigation:
                raise ValueError("mailbox='apan' with MSPipe-S is not built (the APAN build takes h = S.mem[w])")
            self.apan = _C.ApanHandle(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.apan.get("slots", 10), cfg.batch,
                                      cfg.apan["w_q"], cfg.apan["w_k"], self.device)
        self.gru = _C.GruHandle(cfg.mem_dim, cfg.edge_dim, cfg.time_dim, params, self.device, cfg.precision,
                                max_events=cfg.batch, cell=_C.CELL_RNN if cfg.cell == "rnn" else _C.CELL_GRU,
                                mailbox=(_C.MAILBOX_DEFERRED if (self.deferred or self.apan is not None)
                                         else _C.MAILBOX_IMMEDIATE))
        self.upd = _C.alloc_update(cfg.batch, cfg.mem_dim, self.memory.mail_stride, self.device)
        self.fused = cfg.use_fused()
        self._dbg_one = torch.zeros(1, device=self.device) if _DEBUG_ONLY else None  # timing diagnostics
        if self.apan is not None and not self.fused:
            raise ValueError("mailbox='apan' runs on the fused tensor-core path")
        if self.deferred and not (self.fused and cfg.fetch_mail):
            raise ValueError("mailbox='deferred' runs on the fused tensor-core path with fetch_mail=True")
        self.ws_bytes = _C.gru_workspace_size(self.gru, cfg.batch) if self.fused else 0
        self.trainer = None
        if cfg.train is not None:  # row F4
            if not self.fused or self.deferred or cfg.cell != "gru" or cfg.precision != _C.FP32_3XTF32:
                raise ValueError("the training stage runs on the fused 3xTF32 GRUCell path (immediate mailbox)")
            from .train import TrainStage
            self.trainer = TrainStage(self.gru, params, cfg.train["params"], cfg.num_nodes, cfg.mem_dim,
                                      cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, cfg.train.get("lr", 1e-4),
                                      self.device, group=cfg.train.get("group"))
        self.staged = False
        self.slots = None
        self.timing = None  # optional dict name -> list of (start, end) events per op
        self.versions = {}

    # -- inputs ---------------------------------------------------------------
    def bind_resident(self, src, dst, ts, neg, ef):
        self.E = src.numel()
        self.res = dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef)
        self.staged = False
        self.slots = [_Slot(self.cfg, self.memory.mail_stride, self.device, False, self.ws_bytes)
                      for _ in range(self._nslots())]

    def bind_host(self, src, dst, ts, neg, ef):
        """e2e path: the stream in pinned host memory, one packed record per
        batch ([src | dst | neg | ts | ef]), copied H2D with ONE memcpy per batch
        on a copy stream a step ahead of its prep (a ring of k+2 device
        records); each commit's result (unique count, node ids, h' rows — one
        packed record) is read back D2H on a second copy stream during the next
        step."""
        cfg, dev, B = self.cfg, self.device, self.cfg.batch
        self.E = int(src.shape[0])
        nb = -(-self.E // B)
        He = cfg.edge_dim
        self._rec = [("src", 4 * B, torch.int32, (B,)), ("dst", 4 * B, torch.int32, (B,)),
                     ("neg", 4 * B, torch.int32, (B,)), ("ts", 8 * B, torch.float64, (B,)),
                     ("ef", 4 * B * He, torch.float32, (B, He))]
        rec_bytes = sum(r[1] for r in self._rec)
        host = torch.zeros((nb, rec_bytes), dtype=torch.uint8).pin_memory()
        arrays = dict(src=src, dst=dst, neg=neg, ts=ts, ef=ef)
        for i in range(nb):
            j0, j1 = i * B, min((i + 1) * B, self.E)
            for name, view in self._views(host[i]).items():
                view[: j1 - j0].copy_(torch.as_tensor(arrays[name][j0:j1]))
        self.host_rec = host
        self.staged = True
        self.slots = [_Slot(cfg, self.memory.mail_stride, dev, False, self.ws_bytes) for _ in range(self._nslots())]
        self.inp_ring = [torch.empty(rec_bytes, dtype=torch.uint8, device=dev) for _ in range(cfg.k + 2)]
        # result records: [num (16 B) | nodes 2B x 4 | h' 2B x M x 4]; the GEMM writes h' in place
        M = cfg.mem_dim
        self._out_mem_off = 16 + (8 * B + 15) // 16 * 16  # h' rows 16-byte aligned (float4 stores)
        self._out_bytes = self._out_mem_off + 8 * B * M
        # result records: record i % 2 is written by commit(i) and read back during the next step
        self._nout = 2
        self.out_ring = [torch.empty(self._out_bytes, dtype=torch.uint8, device=dev) for _ in range(self._nout)]
        self.upd_ring = []
        for o in self.out_ring:
            u = _C.alloc_update(B, M, self.memory.mail_stride, dev)
            u["mem"] = o[self._out_mem_off:].view(torch.float32).view(2 * B, M)
            self.upd_ring.append(u)
        self.out_host = torch.empty(self._out_bytes, dtype=torch.uint8).pin_memory()
        self.h2d = self.d2h = None
        self._h2d_pending, self._d2h_pending = {}, {}  # copies not yet joined (multi-step graphs)
        self._loaded = set()      # batches whose H2D is enqueued
        self._pending_out = None  # commit whose result awaits its D2H

    def _views(self, rec):
        out, off = {}, 0
        for name, nbytes, dt, shape in self._rec:
            out[name] = rec[off:off + nbytes].view(dt).view(shape)
            off += nbytes
        return out

    def result(self):
        """The last result read back (e2e): (unique count, node ids, h' rows) of a commit."""
        B, M = self.cfg.batch, self.cfg.mem_dim
        o = self.out_host
        U = int(o[:4].view(torch.int32)[0])
        return (U, o[16:16 + 8 * B].view(torch.int32)[:U],
                o[self._out_mem_off:].view(torch.float32).view(2 * B, M)[:U])

    @property
    def num_batches(self):
        return -(-self.E // self.cfg.batch)

    def _range(self, i):
        B = self.cfg.batch
        j0 = (i - 1) * B
        return j0, min(j0 + B, self.E)

    def inputs(self, i):
        j0, j1 = self._range(i)
        if not self.staged:
            return {k: v[j0:j1] for k, v in self.res.items()}
        n = j1 - j0
        return {k: v[:n] for k, v in self._views(self.inp_ring[(i - 1) % (self.cfg.k + 2)]).items()}

    def _load(self, i):
        """H2D of batch i's packed record into its ring buffer, on the current stream."""
        _C.record_to_device(self.inp_ring[(i - 1) % (self.cfg.k + 2)], self.host_rec[i - 1])

    # -- ops ------------------------------------------------------------------
    def _nslots(self):
        """k + 1 snapshot slots in flight; with the training stage one more,
        so prep(t+k+1) need not wait for train(t), which still reads slot t."""
        return self.cfg.k + 1 + (1 if self.trainer is not None and self.cfg.k >= 1 else 0)

    def _slot(self, i):
        return self.slots[(i - 1) % len(self.slots)]

    def prep(self, i):
        """A1 sampler, A2 dedup, A3 fetch (+A4 mitigation) of batch i into its slot."""
        cfg, sl = self.cfg, self._slot(i)
        if self.staged and i not in self._loaded:  # not prefetched (the first steps): load here
            self._load(i)
            self._loaded.add(i)
        self._wait_h2d(i)
        x = self.inputs(i)
        n = x["src"].numel()
        samp = {k: v[: 3 * n] for k, v in sl.samp.items()}
        if self.fused:
            self._prep_fused(i, sl, x, n, samp)
            return
        self._ev("sample")
        _C.sample_batch(self.tcsr, x["src"], x["dst"], x["neg"], x["ts"], cfg.fanout, samp)
        self._ev("sample_end")
        self._features(sl, samp)
        self._ev("dedup")
        _C.memory_dedup(self.memory, x["src"], x["dst"], sl.dd)
        self._ev("dedup_end")
        ids = samp["sub"].reshape(-1)
        m = ids.numel()
        mit = None
        if cfg.mitigation:
            mit = _C.make_mitigation(self.tcsr, cfg.mitigation["lam"], cfg.mitigation["gamma"],
                                     cfg.mitigation["n_sim"], cfg.fanout, x["src"], x["dst"], x["ts"],
                                     sl.h[: 2 * n], sl.omega[: 2 * n], sl.elig[: 2 * n])
        self._ev("fetch")
        sl.version = _C.memory_fetch(self.memory, i, ids, sl.mem[:m], sl.mem_ts[:m],
                                     sl.mail[:m] if sl.mail is not None else None,
                                     sl.mail_ts[:m] if sl.mail_ts is not None else None, mit)
        self._ev("fetch_end")
        self.versions[i] = sl.version

    def bind_features(self, node_feat=None, edge_feat=None):
        """Row F2 tables, resident in HBM: node features [N, node_dim] (padded to a
        multiple of 4 floats) and the edge features of the whole stream [E, He]."""
        dev = self.device
        self.feat_tables = {"node": None, "edge": None}
        if node_feat is not None and self.cfg.node_dim:
            nf = torch.as_tensor(node_feat, dtype=torch.float32)
            t = torch.zeros((nf.shape[0], _pad4(nf.shape[1])), dtype=torch.float32, device=dev)
            t[:, : nf.shape[1]] = nf.to(dev)
            self.feat_tables["node"] = t
        if edge_feat is not None:
            self.feat_tables["edge"] = torch.as_tensor(edge_feat, dtype=torch.float32).to(dev).contiguous()
        self.fstream = None
        self._feat_done = []

    def _features(self, sl, samp):
        """F2 on its own stream, forked after the sampler: it reads only the sample."""
        if not self.cfg.features:
            return
        if not hasattr(self, "feat_tables"):
            raise RuntimeError("StageConfig.features needs bind_features(node_feat, edge_feat) first")
        cur = torch.cuda.current_stream()
        if self.fstream is None or self.fstream.device != cur.device:
            self.fstream = torch.cuda.Stream(device=cur.device)
        fork = torch.cuda.Event()
        fork.record(cur)
        self.fstream.wait_event(fork)
        R = samp["sub"].shape[0]
        with torch.cuda.stream(self.fstream):
            self._ev("features")
            _C.feature_fetch(samp["sub"], samp["eid"], self.cfg.fanout, self.feat_tables["node"],
                             self.feat_tables["edge"], sl.nfeat[:R] if sl.nfeat is not None else None,
                             sl.efeat[:R] if self.feat_tables["edge"] is not None else None)
            self._ev("features_end")
            done = torch.cuda.Event()
            done.record(self.fstream)
        self._feat_done.append(done)

    def _join_features(self):
        main = torch.cuda.current_stream()
        for e in getattr(self, "_feat_done", []):
            main.wait_event(e)
        if getattr(self, "_feat_done", None):
            self._feat_done = []

    def _mitigation(self, sl, x, n):
        cfg = self.cfg
        if not cfg.mitigation:
            return None
        return _C.make_mitigation(self.tcsr, cfg.mitigation["lam"], cfg.mitigation["gamma"], cfg.mitigation["n_sim"],
                                  cfg.fanout, x["src"], x["dst"], x["ts"], sl.h[: 2 * n], sl.omega[: 2 * n],
                                  sl.elig[: 2 * n])

    def _prep_fused(self, i, sl, x, n, samp):
        """mspipe_memory_prep (A1+A2+A3[+A4], one launch) then mspipe_message_build (A5) of batch i."""
        cfg = self.cfg
        m = 3 * n * (cfg.fanout + 1)
        self._ev("prep")
        sl.version = _C.memory_prep(self.memory, self.tcsr, i, x["src"], x["dst"], x["neg"], x["ts"], cfg.fanout,
                                    samp, sl.dd, sl.mem[:m], sl.mem_ts[:m],
                                    sl.mail[:m] if sl.mail is not None else None,
                                    sl.mail_ts[:m] if sl.mail_ts is not None else None, self._mitigation(sl, x, n))
        self._ev("prep_end")
        self._features(sl, samp)
        self.versions[i] = sl.version
        if not self.memory.double_buffer and self.apan is None:
            self._fetched = torch.cuda.Event()  # the state tables have been read for batch i
            self._fetched.record()
        self._ev("build")
        if self.apan is not None:  # row F3 APAN: attention over the node's mailbox slots
            _C.message_build_apan(self.apan, self.gru, x["ts"], sl.mem, sl.mem_ts, cfg.fanout + 1, sl.dd["nodes"][: 2 * n],
                                  sl.dd["winner"][: 2 * n], sl.dd["num"], sl.uts[: 2 * n], sl.ws)
        elif self.deferred:  # row F3: the message is the stored mail of the snapshot
            _C.message_build_deferred(self.gru, x["ts"], sl.mem, sl.mem_ts, sl.mail, cfg.fanout + 1,
                                      sl.dd["winner"][: 2 * n], sl.dd["num"], sl.uts[: 2 * n], sl.ws)
        else:
            _C.message_build(self.gru, x["ts"], x["ef"], sl.mem, sl.mem_ts, cfg.fanout + 1, sl.dd["winner"][: 2 * n],
                             sl.dd["num"], sl.uts[: 2 * n], sl.umail[: 2 * n], sl.ws,
                             snap_h=sl.h[: 2 * n] if sl.h is not None else None)
        self._ev("build_end")
        if self.apan is not None:  # the APAN build read the mailbox rings: commits of later batches wait for it
            self._fetched = torch.cuda.Event()
            self._fetched.record()

    def _upd(self, i):
        n = self.inputs(i)["src"].numel()
        sl = self._slot(i)
        base = self.upd_ring[i % self._nout] if self.staged else self.upd
        upd = {k: v[: 2 * n] for k, v in base.items() if k not in ("nodes", "winner", "num")}
        upd.update(nodes=sl.dd["nodes"][: 2 * n], winner=sl.dd["winner"][: 2 * n], num=sl.dd["num"])
        if self.fused:
            upd.update(ts=sl.uts[: 2 * n], mail=None if (self.deferred or self.apan is not None) else sl.umail[: 2 * n])
        return upd

    def update(self, i):
        """A5+A6 of batch i from its slot (touches no state table)."""
        cfg, sl = self.cfg, self._slot(i)
        x = self.inputs(i)
        n = x["src"].numel()
        self._ev("update")
        if self.fused:
            upd = self._upd(i)
            _C.gru_apply(self.gru, n, sl.mem, cfg.fanout + 1, upd["winner"], upd["num"], upd["mem"], sl.ws,
                         snap_h=sl.h[: 2 * n] if sl.h is not None else None)
        else:
            _C.memory_update(self.memory, self.gru, x["src"], x["dst"], x["ts"], x["ef"], sl.mem, sl.mem_ts,
                             cfg.fanout + 1, self._upd(i), snap_h=sl.h[: 2 * n] if sl.h is not None else None)
        self._ev("update_end")

    def writeback(self, i):
        """A7: commit version i."""
        upd = self._upd(i)
        self._ev("writeback")
        _C.memory_writeback(self.memory, i, upd)
        self._ev("writeback_end")
        self._stash_result(i, upd)

    def commit(self, i):
        if self.fused:
            self.apply_commit(i)
            return
        self._wait_d2h(i)
        self.update(i)
        self.writeback(i)

    def apply_commit(self, i):
        """Fused A6 + A7 (mspipe_gru_apply_commit): GRU of batch i, write-back in its epilogue."""
        self._wait_d2h(i)
        cfg, sl = self.cfg, self._slot(i)
        n = self.inputs(i)["src"].numel()
        upd = self._upd(i)
        self._ev("update")
        # e2e: the GEMM also writes the result record's winner ids and U (no copies after it)
        rec = {}
        if self.staged:
            o = self.out_ring[i % self._nout]
            rec = dict(out_nodes=o[16:16 + 4 * 2 * n].view(torch.int32), out_num=o[:4].view(torch.int32))
        if self.timing is not None and (self.timing_only is None or "gemm" in self.timing_only):
            pair = self._ev_pair("gemm")  # the GEMM kernel alone, recorded by the library around its launch
            if pair is not None:
                _C.kernel_events(*pair)
        _C.gru_apply_commit(self.gru, self.memory, i, n, sl.mem, cfg.fanout + 1, upd, sl.ws,
                            snap_h=sl.h[: 2 * n] if sl.h is not None else None, **rec)
        if self.deferred:  # row F3: new mails from the committed memories of both endpoints
            x = self.inputs(i)
            _C.memory_mail_deferred(self.memory, i, x["src"], x["dst"], x["ts"], x["ef"], upd["nodes"], upd["winner"],
                                    upd["num"])
        if self.apan is not None:  # row F3 APAN: mails from the committed memories, to the node and its neighbours
            x = self.inputs(i)
            _C.apan_deliver(self.apan, self.memory, i, x["src"], x["dst"], x["ts"], x["ef"], upd["nodes"], upd["winner"],
                            upd["num"], sl.samp["nbr"], sl.samp["cnt"], cfg.fanout)
        self._ev("update_end")
        if self.trainer is not None:  # row F4: embeddings, loss, backward, (all-reduce,) SGD of batch i
            # the next step's preps fork from here, not after the training step: MSPipe's
            # fetch of later batches overlaps the training stage (Fig. pipeline (c))
            ev = torch.cuda.Event()
            ev.record()
            self._after_commit = (ev, _C.capture_seq())
            self._ev("train")
            self.trainer.step(i, n, sl.samp, sl.mem, upd, sl.ws, sgd=cfg.train.get("sgd", True))
            self._ev("train_end")
        if self.staged:
            self._pending_out = i  # the GEMM filled the result record
        else:
            self._stash_result(i, upd)

    # -- e2e copies (staged inputs) ---------------------------------------
    def _stash_result(self, i, upd):
        """After commit i: keep its node ids / count (the slot is reused by the
        next prep) for the D2H the next step issues."""
        if not self.staged:
            return
        o = self.out_ring[i % self._nout]  # on the commit's stream, right behind it (two small copies)
        n2 = upd["nodes"].numel()
        o[16:16 + 4 * n2].view(torch.int32).copy_(upd["nodes"], non_blocking=True)
        o[:4].view(torch.int32).copy_(upd["num"], non_blocking=True)
        self._pending_out = i

    def _copy_streams(self):
        cur = torch.cuda.current_stream()
        if self.h2d is None or self.h2d.device != cur.device:
            self.h2d = torch.cuda.Stream(device=cur.device)
            self.d2h = torch.cuda.Stream(device=cur.device)
        return self.h2d, self.d2h

    def _copies_begin(self, ops):
        """Step start (e2e): remember the step's start; the copies themselves are
        captured after the step's kernels (_copies_issue) so that in the graph
        the kernel nodes come first, but depend only on this start."""
        if not self.staged:
            return
        self._step_start = torch.cuda.Event()
        self._step_start.record()
        self._read_back = self._pending_out  # the previous commit (this step's commit re-sets _pending_out)
        self._pending_out = None

    def _copies_issue(self, ops):
        """On the copy streams, from the step start: read back the previous
        commit's result (only its U rows cross PCIe: a zero-copy kernel into the
        pinned record) and prefetch the inputs of the next step's preps."""
        h2d, d2h = self._copy_streams()
        d2h.wait_event(self._step_start)
        with torch.cuda.stream(d2h):
            c = self._read_back
            if _E2E_SKIP == "d2h":  # timing diagnostics only
                c = None
            if c is not None:
                o, B, M = self.out_ring[c % self._nout], self.cfg.batch, self.cfg.mem_dim
                _C.rows_to_host(o[:4].view(torch.int32), self.out_host[:4].view(torch.int32),
                                o[16:16 + 8 * B].view(torch.int32).view(2 * B, 1),
                                self.out_host[16:16 + 8 * B].view(torch.int32).view(2 * B, 1),
                                o[self._out_mem_off:].view(torch.float32).view(2 * B, M),
                                self.out_host[self._out_mem_off:].view(torch.float32).view(2 * B, M), 2 * B)
        h2d.wait_event(self._step_start)
        with torch.cuda.stream(h2d):
            commits = [i for op, i in ops if op == "commit"]
            preps = [i for op, i in ops if op == "prep"]
            done_before = (min(commits) - 1) if commits else 0  # committed in earlier steps
            j = max(preps + [max(self._loaded, default=0)]) + 1
            for _ in range(max(1, len(preps))):
                # its ring buffer last held batch j-(k+2): that one must be committed already
                if j > self.num_batches or j - (self.cfg.k + 2) > done_before:
                    break
                if j not in self._loaded:
                    if _E2E_SKIP != "h2d":  # timing diagnostics only
                        self._load(j)
                    self._loaded.add(j)
                    ev = torch.cuda.Event()
                    ev.record(h2d)
                    self._h2d_pending[j] = ev
                j += 1
        if c is not None:
            ev = torch.cuda.Event()
            ev.record(d2h)
            self._d2h_pending[c] = ev

    def _copies_end(self, ops, join=True):
        """join=False (inside a multi-step graph): no join of the copy streams at
        the step's end; the prep of a prefetched batch waits for its H2D and the
        commit that reuses a result record waits for that record's read-back."""
        if self.staged:
            self._copies_issue(ops)
        if self.staged and self.h2d is not None and join:
            torch.cuda.current_stream().wait_stream(self.h2d)
            torch.cuda.current_stream().wait_stream(self.d2h)
            self._h2d_pending.clear()
            self._d2h_pending.clear()

    def _wait_h2d(self, i):
        ev = self._h2d_pending.pop(i, None) if self.staged else None
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def _wait_d2h(self, i):
        # commit i rewrites result record i % 2, last read back for commit i - 2
        ev = self._d2h_pending.pop(i - self._nout, None) if self.staged else None
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)

    def run_ops(self, ops, overlap=None, join_copies=True):
        """Enqueue ops in order.  With overlap (default when k >= 1) every prep
        goes to a side stream, in order (preps share the handle's scratch); a
        commit of the same group waits for its own prep.  Preps only read the
        T-CSR and the state tables, so prep(t+k) runs concurrently with
        commit(t) — the paper's pipelining of fetch with update,
        moved onto the GPU.  One table set: the commit waits for that fetch
        (its write would change rows the fetch of version t-1 reads), which
        keeps the exact staleness order of Eq. 2.  Double-buffered tables:
        fetch(t+k) reads version t-1 from the other set than the one commit t
        writes, so the commit does not wait at all; the join at the end of the
        group keeps that fetch ahead of commit t+1 (which rewrites its set)."""
        overlap = (self.cfg.k >= 1) if overlap is None else overlap
        self._copies_begin(ops)
        if not overlap:
            for op, i in ops:
                (self.prep if op == "prep" else self.commit)(i)
            self._join_features()
            self._copies_end(ops, join_copies)
            return
        main = torch.cuda.current_stream()
        if getattr(self, "side", None) is None or self.side.device != main.device:
            self.side = torch.cuda.Stream(device=main.device, priority=int(os.environ.get("MSPIPE_SIDE_PRIO", "0")))
        commits = {i for op, i in ops if op == "commit"}
        db = self.memory.double_buffer
        forked = joined = False
        for op, i in ops:
            if op == "prep" and _DEBUG_ONLY in ("commit", "none"):  # timing diagnostics only: no prep
                continue
            if op == "prep":
                # every prep goes to the side stream, in order (preps of one handle
                # share its scratch); a commit of this group waits for its own prep
                if not forked:
                    ac = getattr(self, "_after_commit", None)
                    if ac is not None and ac[1] == _C.capture_seq() and len(self.slots) > self.cfg.k + 1:
                        self.side.wait_event(ac[0])  # the previous commit, not its training step
                    else:
                        self.side.wait_stream(main)
                    forked = True
                with torch.cuda.stream(self.side):
                    self.prep(i)
                if i in commits:
                    done = torch.cuda.Event()
                    done.record(self.side)
                    main.wait_event(done)
            elif self.fused:
                # the epilogue writes the tables: wait only for the side stream's
                # fetch (not its message build, which overlaps this GEMM)
                if forked and not db:
                    main.wait_event(self._fetched)
                if _DEBUG_ONLY in ("prep", "none"):  # timing diagnostics only: the commit is not run
                    self.memory.set_committed(i)
                    if _DEBUG_ONLY == "none":  # one trivial kernel: the step's fixed cost
                        self._dbg_one.add_(1.0)
                    continue
                self.apply_commit(i)
            else:
                self.update(i)
                if forked and not joined and not db:
                    main.wait_stream(self.side)
                    joined = True
                self.writeback(i)
        if forked and not joined:
            main.wait_stream(self.side)
        self._join_features()
        self._copies_end(ops, join_copies)

    def run(self, nb=None):
        """All batches (or the first nb) in schedule order, one step at a time."""
        nb = self.num_batches if nb is None else nb
        for ops in self.step_ops(nb):
            self.run_ops(ops)

    def step_ops(self, nb=None):
        """Ops grouped per step (one commit per step; prologue preps in step 0)."""
        nb = self.num_batches if nb is None else nb
        steps, cur = [], []
        for op in schedule_ops(nb, self.cfg.k, self.cfg.schedule, self.cfg.plan):
            cur.append(op)
            if op[0] == "commit":
                steps.append(cur)
                cur = []
        return steps

    def h2d_bytes_per_batch(self):
        B = self.cfg.batch
        return B * (4 + 4 + 4 + 8 + 4 * self.cfg.edge_dim)

    def d2h_bytes_per_batch(self, mean_unique=None):
        """Bytes read back per step: the count and the U committed rows (ids + h');
        mean_unique = the mean U of the timed batches (None: the 2B upper bound)."""
        U = 2 * self.cfg.batch if mean_unique is None else mean_unique
        return 4 + U * (4 + 4 * self.cfg.mem_dim)
