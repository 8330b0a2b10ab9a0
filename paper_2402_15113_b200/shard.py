"""Row E driver: the node-memory stage with memory sharded by node id.

Global iteration i covers G·B consecutive events; rank g takes the local batch
[(i-1)GB + gB, (i-1)GB + (g+1)B) ("each GPU worker retrieves a local batch",
P:L817).  Each rank samples and deduplicates its local batch against the
replicated T-CSR, fetches the snapshot rows it needs from their owners
(v mod G), runs the GRU for its local winners, and sends keyed write-back
records to the owners, which keep the largest key per node: the result equals
the single-GPU stage at batch G·B (pin P10, tests/test_gpu_shard.py).

Transport: the sending phases store straight into the peers' receive windows
(only the real entries); a barrier follows.  One process per GPU
(``ShardRank`` with an ``nccl_id``: CUDA IPC windows, NCCL barriers), or G
in-process ranks on one device (``LoopbackShards``: the whole protocol on one
GPU, the stream orders the phases).  With k >= 1 the process driver runs
prep(t+k) (sampler, dedup, fetch) on a side stream concurrently with
commit(t) on the main stream; the commit's merge waits only for the fetch's
serve phase, the one that reads this rank's tables.
"""
from __future__ import annotations

import torch

from . import _C
from .stage import StageConfig, _Slot, _TimedOps, schedule_ops


def local_range(i, rank, world, batch, num_events):
    """Events of rank's local batch in global iteration i (1-based): [j0, j1)."""
    j0 = (i - 1) * world * batch + rank * batch
    return min(j0, num_events), min(j0 + batch, num_events)


def key_base(i, rank, world, batch):
    """LWW key of local pair p is key_base + p = 2 * (global event index) + role."""
    return 2 * ((i - 1) * world * batch + rank * batch)


def num_global_batches(num_events, world, batch):
    return -(-num_events // (world * batch))


class ShardRank(_TimedOps):
    """One rank's handles, slots and ops (ordinary or NCCL-collective calls)."""

    def __init__(self, cfg: StageConfig, params: dict, tcsr: _C.TcsrHandle, device, rank: int, world: int,
                 nccl_id: bytes | None = None):
        self.cfg, self.rank, self.world = cfg, rank, world
        self.device = torch.device(device)
        self.tcsr = tcsr
        self.memory = _C.MemoryHandle(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.k, self.device, rank, world,
                                      nccl_id)
        if nccl_id is not None:  # collective: every rank's window handle, then open the peers'
            from .dist import connect_shards
            connect_shards(self.memory)
        self.side = None
        self._served = None
        if cfg.mitigation:  # MSPipe-S (A4): candidate list and a node-indexed table of the fetched rows
            B, F = cfg.batch, cfg.fanout
            self.cand = torch.empty((2 * B, 1 + F * F), dtype=torch.int32, device=self.device)
            self.tab_mem = torch.zeros((cfg.num_nodes, cfg.mem_dim), dtype=torch.float32, device=self.device)
            self.tab_ts = torch.zeros((cfg.num_nodes,), dtype=torch.float64, device=self.device)
        self.gru = _C.GruHandle(cfg.mem_dim, cfg.edge_dim, cfg.time_dim, params, self.device, cfg.precision,
                                max_events=cfg.batch)
        self.slots = [_Slot(cfg, self.memory.mail_stride, self.device, False) for _ in range(cfg.k + 1)]
        self.upd = _C.alloc_update(cfg.batch, cfg.mem_dim, self.memory.mail_stride, self.device)
        self.versions = {}
        self.staged = False

    def bind_resident(self, src, dst, ts, neg, ef):
        self.E = src.numel()
        self.res = dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef)

    def bind_host(self, src, dst, ts, neg, ef):
        """e2e: pinned host stream; each prep copies its local batch H2D, each commit
        reads its h' rows back."""
        self.E = int(src.shape[0])
        self.host = {k: torch.as_tensor(v).pin_memory() for k, v in
                     dict(src=src, dst=dst, ts=ts, neg=neg, ef=ef).items()}
        self.staged = True
        self.slots = [_Slot(self.cfg, self.memory.mail_stride, self.device, True) for _ in range(self.cfg.k + 1)]
        B = self.cfg.batch
        self.out_host = dict(num=torch.empty(1, dtype=torch.int32).pin_memory(),
                             nodes=torch.empty(2 * B, dtype=torch.int32).pin_memory(),
                             mem=torch.empty((2 * B, self.cfg.mem_dim), dtype=torch.float32).pin_memory())

    def h2d_bytes_per_batch(self):
        return self.cfg.batch * (4 + 4 + 4 + 8 + 4 * self.cfg.edge_dim)

    def d2h_bytes_per_batch(self):
        B = self.cfg.batch
        return 4 + 2 * B * 4 + 2 * B * self.cfg.mem_dim * 4

    def _slot(self, i):
        return self.slots[(i - 1) % (self.cfg.k + 1)]

    def inputs(self, i):
        j0, j1 = local_range(i, self.rank, self.world, self.cfg.batch, self.E)
        if not self.staged:
            return {k: v[j0:j1] for k, v in self.res.items()}
        return {k: v[: j1 - j0] for k, v in self._slot(i).inp.items()}

    # -- prep -------------------------------------------------------------
    def prep_local(self, i):
        """A1 + A2 on the local batch (no state access)."""
        sl = self._slot(i)
        if self.staged:
            j0, j1 = local_range(i, self.rank, self.world, self.cfg.batch, self.E)
            for key in ("src", "dst", "neg", "ts", "ef"):
                sl.inp[key][: j1 - j0].copy_(self.host[key][j0:j1], non_blocking=True)
        x = self.inputs(i)
        n = x["src"].numel()
        samp = {k: v[: 3 * n] for k, v in sl.samp.items()}
        _C.sample_batch(self.tcsr, x["src"], x["dst"], x["neg"], x["ts"], self.cfg.fanout, samp)
        _C.memory_dedup(self.memory, x["src"], x["dst"], sl.dd)
        self._ids = (i, samp["sub"].reshape(-1))

    def _fetch_out(self, i):
        sl = self._slot(i)
        ids = self._ids[1]
        m = ids.numel()
        return ids, sl.mem[:m], sl.mem_ts[:m], (sl.mail[:m] if sl.mail is not None else None), \
            (sl.mail_ts[:m] if sl.mail_ts is not None else None)

    def fetch_plan(self, i):
        ids, _, _, mail, _ = self._fetch_out(i)
        _C.shard_fetch_plan(self.memory, i, ids, with_mail=mail is not None)

    def fetch_serve(self):
        _C.shard_fetch_serve(self.memory)

    def fetch_finish(self, i):
        ids, mem, mem_ts, mail, mail_ts = self._fetch_out(i)
        self.versions[i] = _C.shard_fetch_finish(self.memory, ids, mem, mem_ts, mail, mail_ts)

    # -- MSPipe-S (A4) with sharded memory: a second fetch of the candidates' rows
    def _mit(self, i):
        cfg, sl, x = self.cfg, self._slot(i), self.inputs(i)
        n = x["src"].numel()
        m = cfg.mitigation
        return _C.make_mitigation(self.tcsr, m["lam"], m["gamma"], m["n_sim"], cfg.fanout, x["src"], x["dst"],
                                  x["ts"], sl.h[: 2 * n], sl.omega[: 2 * n], sl.elig[: 2 * n])

    def mit_plan(self, i):
        """Candidates of the eligible targets (their roots' mem_ts came with the
        subgraph fetch), then the fetch plan of that list."""
        sl = self._slot(i)
        n = self.inputs(i)["src"].numel()
        cand = self.cand[: 2 * n]
        _C.shard_mitigation_candidates(self.memory, self._mit(i), sl.mem_ts, self.cfg.fanout + 1, cand)
        _C.shard_fetch_plan(self.memory, i, cand.reshape(-1))

    def mit_finish(self, i):
        """The candidates' rows into the node table, then the blend (k_mitigate)."""
        n = self.inputs(i)["src"].numel()
        _C.shard_fetch_finish_table(self.memory, self.cand[: 2 * n].reshape(-1), self.tab_mem, self.tab_ts)
        _C.shard_mitigate(self.memory, self._mit(i), self.tab_mem, self.tab_ts)

    def fetch_collective(self, i):
        """NCCL: plan, all-to-all, serve, all-to-all, finish inside mspipe_memory_fetch."""
        ids, mem, mem_ts, mail, mail_ts = self._fetch_out(i)
        self.versions[i] = _C.memory_fetch(self.memory, i, ids, mem, mem_ts, mail, mail_ts)

    # -- commit -----------------------------------------------------------
    def _upd(self, i):
        n = self.inputs(i)["src"].numel()
        sl = self._slot(i)
        upd = {k: v[: 2 * n] for k, v in self.upd.items() if k not in ("nodes", "winner", "num")}
        upd.update(nodes=sl.dd["nodes"][: 2 * n], winner=sl.dd["winner"][: 2 * n], num=sl.dd["num"])
        return upd

    def update(self, i):
        """A5 + A6 for the local winners (rank-local); h = MSPipe-S's blend when mitigating."""
        sl, x = self._slot(i), self.inputs(i)
        n = x["src"].numel()
        _C.memory_update(self.memory, self.gru, x["src"], x["dst"], x["ts"], x["ef"], sl.mem, sl.mem_ts,
                         self.cfg.fanout + 1, self._upd(i), snap_h=sl.h[: 2 * n] if sl.h is not None else None)

    def commit_pack(self, i):
        _C.shard_commit_pack(self.memory, i, self._upd(i), key_base(i, self.rank, self.world, self.cfg.batch))

    def commit_merge(self, i):
        _C.shard_commit_merge(self.memory, i)

    def writeback_collective(self, i):
        _C.memory_writeback_keyed(self.memory, i, self._upd(i), key_base(i, self.rank, self.world, self.cfg.batch))

    # -- process driver (one rank per GPU) -----------------------------------
    def prep(self, i):
        """A1 + A2 local, then the fetch phases with their barriers; the event
        after the serve phase (the one that reads this rank's tables) lets a
        concurrent commit's merge start as early as possible."""
        self._ev("prep")
        self.prep_local(i)
        self.fetch_plan(i)
        _C.shard_exchange(self.memory, _C.XCHG_FETCH_IDS)
        self.fetch_serve()
        self._served = torch.cuda.Event()
        self._served.record()
        _C.shard_exchange(self.memory, _C.XCHG_FETCH_ROWS)
        self.fetch_finish(i)
        if self.cfg.mitigation:  # same iteration, same window parity: the barriers above separate the rounds
            self.mit_plan(i)
            _C.shard_exchange(self.memory, _C.XCHG_FETCH_IDS)
            self.fetch_serve()
            self._served = torch.cuda.Event()
            self._served.record()
            _C.shard_exchange(self.memory, _C.XCHG_FETCH_ROWS)
            self.mit_finish(i)
        self._ev("prep_end")

    def commit(self, i, served=None):
        self._ev("update")
        self.update(i)
        self._ev("update_end")
        self._ev("writeback")
        self.commit_pack(i)
        _C.shard_exchange(self.memory, _C.XCHG_COMMIT)
        if served is not None:  # a concurrent fetch still reads the rows the merge rewrites
            torch.cuda.current_stream().wait_event(served)
        self.commit_merge(i)
        self._ev("writeback_end")
        if self.staged:
            self.copy_out(i)

    def copy_out(self, i):
        """e2e: D2H of this batch's result (unique count, winners' node ids, h')."""
        upd = self._upd(i)
        n2 = upd["nodes"].numel()
        self.out_host["num"].copy_(upd["num"], non_blocking=True)
        self.out_host["nodes"][:n2].copy_(upd["nodes"], non_blocking=True)
        self.out_host["mem"][:n2].copy_(upd["mem"], non_blocking=True)

    @property
    def num_batches(self):
        return num_global_batches(self.E, self.world, self.cfg.batch)

    def step_ops(self, nb=None):
        nb = self.num_batches if nb is None else nb
        steps, cur = [], []
        for op in schedule_ops(nb, self.cfg.k, self.cfg.schedule, self.cfg.plan):
            cur.append(op)
            if op[0] == "commit":
                steps.append(cur)
                cur = []
        return steps

    def run_ops(self, ops, overlap=None, join_copies=True):
        """One step.  overlap (default k >= 1): the step's preps on a side stream
        (forked after the previous step's commit, so they read its version),
        the commit on the current stream; its merge waits for the side
        stream's serve phase, then the step joins the side stream."""
        overlap = (self.cfg.k >= 1) if overlap is None else overlap
        if not overlap:
            for op, i in ops:
                (self.prep if op == "prep" else self.commit)(i)
            return
        main = torch.cuda.current_stream()
        if self.side is None or self.side.device != main.device:
            self.side = torch.cuda.Stream(device=main.device)
        self.side.wait_stream(main)
        served = None
        for op, i in ops:
            if op == "prep":
                with torch.cuda.stream(self.side):
                    self.prep(i)
                served = self._served
                if any(o == "commit" and j == i for o, j in ops):  # its own commit in this step
                    main.wait_stream(self.side)
            else:
                self.commit(i, served=served)
        main.wait_stream(self.side)

    def run(self, nb=None):
        for ops in self.step_ops(nb):
            self.run_ops(ops)

    def exchange_bytes(self):
        """(fetch ids, reply rows, commit records) bytes this rank stored since the last reset."""
        return _C.shard_sent_bytes(self.memory)


class LoopbackShards:
    """G in-process ranks on one device, phases interleaved on one stream (the
    stream orders each phase's stores into the windows before the phase that
    reads them): the whole sharded protocol without NCCL."""

    def __init__(self, cfg: StageConfig, params: dict, tcsr: _C.TcsrHandle, device, world: int):
        self.cfg, self.world = cfg, world
        self.ranks = [ShardRank(cfg, params, tcsr, device, r, world, None) for r in range(world)]
        _C.shard_connect_local([r.memory for r in self.ranks])

    def bind_resident(self, src, dst, ts, neg, ef):
        for r in self.ranks:
            r.bind_resident(src, dst, ts, neg, ef)
        self.E = src.numel()

    def bind_host(self, src, dst, ts, neg, ef):
        for r in self.ranks:
            r.bind_host(src, dst, ts, neg, ef)
        self.E = int(src.shape[0])

    def step_ops(self, nb=None):
        return self.ranks[0].step_ops(nb)

    def run_ops(self, ops):
        for op, i in ops:
            (self.prep if op == "prep" else self.commit)(i)

    def reset(self):
        for r in self.ranks:
            r.memory.reset()

    def _xchg(self, kind):
        _C.shard_loopback([r.memory for r in self.ranks], kind)

    def prep(self, i):
        for r in self.ranks:
            r.prep_local(i)
            r.fetch_plan(i)
        self._xchg(_C.XCHG_FETCH_IDS)
        for r in self.ranks:
            r.fetch_serve()
        self._xchg(_C.XCHG_FETCH_ROWS)
        for r in self.ranks:
            r.fetch_finish(i)
        if self.cfg.mitigation:
            for r in self.ranks:
                r.mit_plan(i)
            self._xchg(_C.XCHG_FETCH_IDS)
            for r in self.ranks:
                r.fetch_serve()
            self._xchg(_C.XCHG_FETCH_ROWS)
            for r in self.ranks:
                r.mit_finish(i)

    def commit(self, i):
        for r in self.ranks:
            r.update(i)
            r.commit_pack(i)
        self._xchg(_C.XCHG_COMMIT)
        for r in self.ranks:
            r.commit_merge(i)
            if r.staged:
                r.copy_out(i)

    def run(self, nb=None):
        for ops in self.step_ops(nb):
            self.run_ops(ops)

    def gather(self):
        """Global tables assembled from the shards (row v lives at rank v % G, row v // G)."""
        N, G = self.cfg.num_nodes, self.world
        out = {}
        for key in ("mem", "mem_ts", "mail", "mail_ts"):
            parts = [getattr(r.memory, key) for r in self.ranks]
            full = torch.empty((N,) + tuple(parts[0].shape[1:]), dtype=parts[0].dtype, device=parts[0].device)
            for g, p in enumerate(parts):
                full[g::G] = p
            out[key] = full
        return out
