#!/usr/bin/env python
"""bench.py — MSPipe node-memory stage on B200: events/s + roofline.

A *step* is one batch through the whole hot path (A1-A7):
the prep of batch t+k (sampler, dedup, fetch, message build) and the commit
of batch t (GRU GEMM + write-back).  At N = 1, 8 consecutive steps
(--graph-steps; the largest divisor of K up to it) are captured as ONE CUDA
graph and replayed; L2 is flushed (a 256 MiB write) before every replay,
outside the timed events, and exactly K steps are timed.  One graph per step
pays the ~6 us graph-launch gap per step (measured the same with and without
the flush, so it is launch latency, not cache); that per-step protocol is
timed as well and reported in `per_step_graphs`.  Inputs are resident in HBM
for `value`; `e2e` copies each batch from pinned host memory and reads each
commit's result back.  Default workload: the GDELT-shaped stream (BASELINE.json
configs[4], the largest single-GPU configuration: B = 4000, build k = 3), its
first 1,000 batches (4M events, the prefix the GPU tests check against the
oracle) run over a T-CSR built from the WHOLE 191M-event stream, so the
sampler searches rows of full-stream length.  The K timed steps are repeated
as whole K-step blocks until >= 0.1 s is timed (each block bracketed by
synchronisation; `value` is the median block).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config wiki] [--impl mspipe|reference]

N > 1 (torchrun): node memory sharded by node id over the ranks with NCCL
all-to-all fetch and write-back (row E; MSPIPE_BENCH_REPLICAS=1: independent
replicas), one graph per step; value = events of all ranks / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "memory-stage events/sec"
UNIT = "events/s"
FLUSH_BYTES = 256 << 20
FP32_FMA_LANES_PER_SM = 128  # B200 SM: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md / guide unit counts)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm_gbs=float(d.get("hbm_gbs", 6650.0)), bf16_tflops=float(d.get("bf16_tflops", 1590.0)),
                    bf16_tflops_sustained=float(d.get("bf16_tflops_sustained", 1400.0)), source="measured")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, source="fallback")


class ClockSampler:
    """SM clock + throttle reasons during the timed region: an NVML poll thread
    (every ~2 ms, so even a 20 ms timed region has samples) plus the recipe's
    nvidia-smi record (gpurun_out/clocks_<pid>.csv) running alongside."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.samples = []
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self.nv, self.h
        while True:
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                return
            if self.stop.wait(0.002):
                return

    def __enter__(self):
        import threading
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        self.thread = None
        try:
            self.nv, self.h = self._nvml_handle()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        rows = [(float(c), float(m), {n for n, bit in self.REASONS.items() if r & bit}) for c, m, r in self.samples]
        if self.proc is not None:
            names = list(self.REASONS)
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 7:
                        try:
                            rows.append((float(parts[0]), float(parts[1]),
                                         {names[i] for i, v in enumerate(parts[3:7]) if v.lower() == "active"}))
                        except ValueError:
                            pass
        if not rows:
            return None
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(set().union(*(r[2] for r in rows))), "samples": len(rows),
                "source": "NVML poll every 2 ms + nvidia-smi -lms 100 during the timed region"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _unique_counts(src, dst, B):
    """U per batch (host arithmetic on the inputs, for the algorithmic-bytes model)."""
    out = []
    for j0 in range(0, len(src), B):
        out.append(len(np.unique(np.concatenate([src[j0:j0 + B], dst[j0:j0 + B]]))))
    return np.array(out)


def algorithmic(cfg, stage_cfg, U):
    """Bytes (or FLOPs) each op must move per batch."""
    B, F, M, He = cfg.batch, cfg.fanout, cfg.mem_dim, cfg.edge_dim
    Dm = 2 * M + He
    Dx = Dm + cfg.time_dim
    stride = (Dm + 3) // 4 * 4
    R = 3 * B
    n_sub = R * (F + 1)
    sample = R * (4 + 8 + 16 + F * 16 + F * 20 + 4 + (F + 1) * 4)
    row = 4 * M + 8
    fetch = n_sub * (4 + 2 * row) + (n_sub * 2 * (4 * stride + 8) if stage_cfg.fetch_mail else 0)
    upd_bytes = 2 * B * 8 + U * (2 * 4 * M + 8 + 8 + 4 * He + 4 * M + 8 + 4 * stride + 8)
    upd_flops = U * 2 * 3 * M * (Dx + M)
    wb = U * (4 + 2 * (4 * M + 8 + 4 * stride))
    dedup = 2 * B * 8
    # fused ops: prep = A1 + A2 + A3 in one launch; build = the A5 half of update (its bytes); the
    # apply half (A6) keeps the name "update" and its FLOPs
    nstride = (cfg.node_dim + 3) // 4 * 4
    feats = R * (F + 1) * (4 + 8 * nstride) * (1 if cfg.node_dim else 0) + R * F * (4 + 8 * He)
    return dict(sample=sample, dedup=dedup, fetch=fetch, prep=sample + dedup + fetch, build=upd_bytes,
                update=upd_bytes, update_flops=upd_flops, writeback=wb, features=feats)


def train_flops(cfg, H=100):
    """FLOPs of the row F4 step's contractions (2 m n k each):
    forward projections / embedding / decoder, their weight and input
    gradients, the GRU weight gradient over the 2B rows the GEMMs run on."""
    B, F, M, Dt = cfg.batch, cfg.fanout, cfg.mem_dim, cfg.time_dim
    Dx = 2 * M + cfg.edge_dim + Dt
    R, RF, Z = 3 * B, 3 * B * F, M + Dt
    mnk = [(R, H, M), (RF, 2 * H, Z), (R, H, H + M), (2 * B, H, 2 * H),            # forward
           (H, 2 * H, 2 * B), (2 * B, 2 * H, H), (H, H + M, R), (R, H + M, H),     # decoder / W_o grads
           (H, M, R), (R, M, H), (2 * H, Z, RF), (RF, M, 2 * H),                   # attention grads
           (3 * M, Dx, 2 * B), (2 * M, M, 2 * B), (M, M, 2 * B)]                   # GRU weight grads
    return float(sum(2 * m * n * k for m, n, k in mnk))


def fp32_simt_peak_tflops(sm_mhz):
    """CUDA-core fp32 peak: 148 SMs x 128 FMA lanes x 2 FLOP x clock (B200_PROFILING.md unit counts)."""
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12


def run_mspipe(args):
    import torch
    import torch.distributed as dist

    from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr, gamma_quantile
    from synth import make_workload

    ws, rank, local = _dist()
    # the device first: NCCL collectives of the process group (the unique-id
    # broadcast, barriers, the max over ranks) run on the current device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        # NCCL: connect peers at communicator init, not lazily inside a graph capture
        os.environ.setdefault("NCCL_RUNTIME_CONNECT", "0")
        dist.init_process_group("nccl", device_id=dev)
    events, tcsr_events = _window(args)
    w = make_workload(args.config, seed=args.seed, num_events=events, tcsr_events=tcsr_events)
    cfg = w["cfg"]
    k = cfg.staleness_k if args.k is None else args.k
    mit = None
    if cfg.mitigation and not args.no_mitigation:
        mit = dict(lam=cfg.lam, gamma=gamma_quantile(cfg.num_nodes, w["src"], w["dst"], w["ts"], cfg.quantile_p),
                   n_sim=cfg.n_sim)
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     schedule=args.schedule, mitigation=mit, fetch_mail=args.fetch_mail,
                     precision={"tc": _C.FP32_3XTF32, "bf16": _C.BF16, "simt": _C.FP32_SIMT}[args.gru],
                     features=args.features, node_dim=cfg.node_dim)
    g = build_tcsr(cfg.num_nodes, *w.get("tcsr", (w["src"], w["dst"], w["ts"])), dev)
    nnz = int(g.nbr.numel())
    w.pop("tcsr", None)
    # N > 1: node-id-sharded memory over NCCL (row E); MSPIPE_BENCH_REPLICAS=1 runs
    # N independent single-GPU replicas instead (ablation)
    sharded = ws > 1 and os.environ.get("MSPIPE_BENCH_REPLICAS", "0") != "1"
    G = ws if sharded else 1
    E = len(w["src"])
    nb = -(-E // (G * cfg.batch))
    U_host = _unique_counts(w["src"], w["dst"], G * cfg.batch)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    resident = {}

    def make_stage(staged):
        if sharded:
            # every stage owns its communicator: a fresh unique id each time (collective)
            from paper_2402_15113_b200 import ShardRank
            from paper_2402_15113_b200.dist import share_nccl_id
            st = ShardRank(sc, w["params"], g, dev, rank, ws, share_nccl_id(rank))
        else:
            st = MemoryStage(sc, w["params"], g, dev)
        if staged:
            st.bind_host(w["src"], w["dst"], w["ts"], w["neg"], w["ef"])
        else:  # the device copy of the inputs is made once and shared by every stage
            if not resident:
                resident.update({kk: torch.from_numpy(w[kk]).to(dev) for kk in ("src", "dst", "ts", "neg", "ef")})
            t = resident
            st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        if args.features:  # row F2: feature tables resident in HBM (the stream's edge features, node features)
            from synth import node_features
            st.bind_features(node_features(args.seed, cfg.num_nodes, cfg.node_dim) if cfg.node_dim else None,
                             torch.from_numpy(w["ef"]).to(dev))
        return st

    def capture(st):
        """One CUDA graph per step (the per-step protocol)."""
        s = torch.cuda.Stream(device=dev)
        st.timing = None
        graphs = [_C.StepGraph().capture(lambda ops=ops: st.run_ops(ops), s) for ops in st.step_ops()]
        st.memory.reset(stream=s)
        return graphs, s

    def timed_run(st, graphs, s, W, K):
        """One K-step block from an epoch start: reset, W warm-up steps, K timed
        steps (wrapping over epochs), L2 flushed before every step; per-step ms."""
        step_ms, pending = [], []
        with torch.cuda.stream(s):
            st.memory.reset(stream=s)
            for n in range(W + K):
                t = n % nb
                if t == 0 and n > 0:
                    torch.cuda.synchronize()
                    step_ms += [e0.elapsed_time(e1) for e0, e1 in pending]
                    pending.clear()
                    st.memory.reset(stream=s)
                if args.l2 == "flush":
                    flush.fill_(float(n))
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                graphs[t].replay(s)
                e1.record(s)
                if n >= W:
                    pending.append((e0, e1))
            torch.cuda.synchronize()
        step_ms += [e0.elapsed_time(e1) for e0, e1 in pending]
        return step_ms

    def capture_groups(st, gs, op=None, serial=False):
        """One CUDA graph per gs consecutive steps (the epoch's last group may be
        shorter).  op: bracket that op (and nothing else) with event nodes; the
        group's events are st.timing[op][a:b] / st.timing[op + '_end'][a:b].
        serial: the step's ops one after another on one stream (each kernel
        alone on the GPU, L2 warm from the ops before it)."""
        s = torch.cuda.Stream(device=dev)
        st.timing = None
        st.timing_only = None
        sops = st.step_ops()
        if op is not None:
            st.timing_only = {op}
            st.reserve_timing_events(2 * 2 * len(sops) + 16)
        groups = []
        for j in range(0, len(sops), gs):
            idx = list(range(j, min(j + gs, len(sops))))

            def run_group(idx=idx):
                for t in idx:  # e2e copies join only at the graph's end
                    st.run_ops(sops[t], overlap=False if serial else None, join_copies=(t == idx[-1]))
            a = len((st.timing or {}).get(op, []))
            gr = _C.StepGraph().capture(run_group, s)
            groups.append((gr, idx, a, len((st.timing or {}).get(op, []))))
        st.memory.reset(stream=s)
        return groups, s

    def timed_run_groups(st, groups, s, W, K, gs, op=None):
        """One K-step block from an epoch start: reset, warm-up replays until >= W
        steps ran, then replays of full gs-step groups until exactly K steps are
        timed (an epoch's shorter last group runs untimed); L2 flushed before
        every replay, one event pair per replay.  op: also returns the bracketed
        op's durations (the host waits after every timed replay to read them)."""
        ms, timed, pending, op_ms = [], [], [], []
        warm, r = 0, 0
        with torch.cuda.stream(s):
            st.memory.reset(stream=s)
            while len(timed) + len(pending) * gs < K:
                j = r % len(groups)
                if j == 0 and r > 0:
                    torch.cuda.synchronize()
                    st.memory.reset(stream=s)
                graph, idx, a, b = groups[j]
                if args.l2 == "flush":
                    flush.fill_(float(r))
                if warm >= W and len(idx) == gs:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    graph.replay(s)
                    e1.record(s)
                    pending.append((e0, e1, idx))
                    if op is not None:
                        e1.synchronize()
                        op_ms += [st.timing[op][q].elapsed_time(st.timing[op + "_end"][q]) for q in range(a, b)]
                else:
                    graph.replay(s)
                    warm += len(idx)
                r += 1
            torch.cuda.synchronize()
        for e0, e1, idx in pending:
            ms.append(e0.elapsed_time(e1))
            timed.extend(idx)
        return ms, timed, op_ms

    def max_over_ranks(x):
        if ws == 1:
            return x
        tt = torch.tensor([x], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    W, K = args.warmup, args.steps
    # steps per captured graph: launch latency between graphs (~6 us, the same
    # with or without the L2 flush) is paid once per graph, not once per step
    gs = 1
    if ws == 1 and not args.profile:  # the largest divisor of K up to --graph-steps (exactly K steps timed)
        gs = max(d for d in range(1, max(1, min(args.graph_steps, nb - 1)) + 1) if K % d == 0)

    def run_blocks(staged):
        """K-step blocks (each from an epoch start, W warm-up steps untimed) until
        >= MIN_TIMED_MS is timed: the block count comes from the first block's
        max-over-ranks time, so every rank runs the same number.  Returns a list
        of (max-over-ranks ms of the block, timed batch indices) and the clocks."""
        st = make_stage(staged)
        if gs > 1:
            groups, s = capture_groups(st, gs)
        else:
            graphs, s = capture(st)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        blocks, nblocks = [], 1
        with ClockSampler(local) as clk:
            while len(blocks) < nblocks:
                if gs > 1:
                    step_ms, tb, _ = timed_run_groups(st, groups, s, W, K, gs)
                else:
                    step_ms = timed_run(st, graphs, s, W, K)
                    tb = [(W + q) % nb for q in range(K)]
                if ws > 1:
                    dist.barrier()
                blocks.append((max_over_ranks(float(sum(step_ms))), tb))
                if len(blocks) == 1 and not args.profile:
                    nblocks = int(min(MAX_BLOCKS, max(1, -(-MIN_TIMED_MS // max(blocks[0][0], 1e-3)))))
        _C.check(s)
        return blocks, clk.summary(), st

    def block_value(blocks):
        """(median block rate, its ms per step, every block's rate)."""
        rates = [sum(min(G * cfg.batch, E - b * G * cfg.batch) for b in tb) * (ws if not sharded else 1) / (ms / 1e3)
                 for ms, tb in blocks]
        order = sorted(range(len(rates)), key=rates.__getitem__)
        med = order[len(order) // 2]
        return rates[med], blocks[med][0] / K, rates, blocks[med][1]

    def train_measurement():
        """Memory stage + training stage (forward, backward, SGD) per step, the
        same grouped graphs and flush protocol; the train op alone (bracketed,
        in the two-stream step) against the CUDA-core fp32 peak."""
        import dataclasses

        from synth import train_params
        sct = dataclasses.replace(sc, train=dict(params=train_params(cfg.mem_dim, cfg.time_dim, 100), lr=1e-4))

        def mk():
            stt = MemoryStage(sct, w["params"], g, dev)
            t = resident
            stt.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
            return stt
        stt = mk()
        gr_t, s_t = capture_groups(stt, gs)
        torch.cuda.synchronize()
        with ClockSampler(local) as clk_t:
            ms_t, tb_t, _ = timed_run_groups(stt, gr_t, s_t, W, K, gs)
        _C.check(s_t)
        loss = stt.trainer.losses[: min(nb, stt.trainer.losses.numel())]
        finite = bool(torch.isfinite(loss).all().item())
        ev_t = sum(min(cfg.batch, E - b * cfg.batch) for b in tb_t)
        del gr_t, stt
        sti = mk()
        gi, si = capture_groups(sti, gs, op="train")
        _, _, opm = timed_run_groups(sti, gi, si, W, K, gs, op="train")
        _C.check(si)
        del gi, sti
        t_ms = float(np.mean(opm))
        fl = train_flops(cfg)
        clk = clk_t.summary()
        simt = fp32_simt_peak_tflops((clk or {}).get("sm_mhz") or 1965.0)
        peak = peaks["bf16_tflops_sustained"] * (1.1 / 2.25) / 3.0  # 3xTF32 tensor peak (the big contractions)
        ach = fl / (t_ms / 1e3) / 1e12
        return {"metric": "memory stage + MTGNN training stage (row F4) events/s", "unit": UNIT,
                "value": ev_t / (sum(ms_t) / 1e3), "ms_per_step": float(sum(ms_t)) / K,
                "train_ms_in_step": t_ms, "losses_finite": finite,
                "roofline": {"kernel": "row F4 step (3xTF32 tensor-core GEMMs for the neighbour-slot K|V "
                                       "projection and its two gradients, SGEMM for the rest, attention / "
                                       "decoder / scatter / GRU-backward kernels)",
                             "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                             "flops_per_step": fl, "frac_of_fp32_simt_peak": ach / simt,
                             "peak_source": "measured bf16 sustained x 1.1/2.25 (tf32) / 3 (3xTF32 passes); "
                                            "fp32 CUDA-core peak = 148 SMs x 128 lanes x 2 x median SM clock"},
                "config": {"emb_dim": 100, "lr": 1e-4, "attention": "single-head, 10 neighbours",
                           "decoder": "TGN link MLP", "optimizer": "SGD"},
                "clocks": clk}

    def apan_measurement():
        """Row F3, APAN: the stage with the multi-slot mailbox (attention message,
        GRU GEMM, propagation to sampled neighbours) at the config's staleness k,
        grouped graphs and the same flush protocol; events/s beside the TGN stage's."""
        import dataclasses

        rng = np.random.default_rng(args.seed + 77)
        M, Dm = cfg.mem_dim, cfg.mail_dim
        ap = dict(w_q=(rng.uniform(-1, 1, (M, M)) / np.sqrt(M)).astype(np.float32),
                  w_k=(rng.uniform(-1, 1, (M, Dm)) / np.sqrt(Dm)).astype(np.float32), slots=10)
        sca = dataclasses.replace(sc, mailbox="apan", apan=ap, mitigation=None, double_buffer=False)
        sta = MemoryStage(sca, w["params"], g, dev)
        t = resident
        sta.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        gr_a, s_a = capture_groups(sta, gs)
        torch.cuda.synchronize()
        with ClockSampler(local) as clk_a:
            ms_a, tb_a, _ = timed_run_groups(sta, gr_a, s_a, W, K, gs)
        _C.check(s_a)
        ev_a = sum(min(cfg.batch, E - b * cfg.batch) for b in tb_a)
        filled = float(sta.apan.mb_cnt.float().mean().item())
        del gr_a, sta
        return {"metric": "APAN memory stage (row F3) events/s", "unit": UNIT, "value": ev_a / (sum(ms_a) / 1e3),
                "ms_per_step": float(sum(ms_a)) / K,
                "config": {"staleness_k": sca.k, "slots": 10, "message": "attention over the filled mailbox slots",
                           "tables": "one set (the commit waits for the fetch and the APAN build of the later batch)",
                           "propagation": "node + its sampled neighbours, latest key wins",
                           "mean_filled_slots_at_end": filled},
                "note": "the mailbox epoch reset is the caller's (not between timed blocks)",
                "clocks": clk_a.summary()}

    # ---- device-resident run (the `value`) ---------------------------------
    blocks, clocks, st = run_blocks(False)
    value, ms_step, rates, timed_batches = block_value(blocks)
    per_step = None
    if gs > 1:
        # the same steps with one graph per step (L2 flushed before each): the
        # per-step protocol, reported beside the grouped headline
        st1 = make_stage(False)
        graphs1, s1 = capture(st1)
        ms1 = timed_run(st1, graphs1, s1, W, K)
        _C.check(s1)
        del graphs1, st1
        tb1 = [(W + q) % nb for q in range(K)]
        ev1 = sum(min(cfg.batch, E - b * cfg.batch) for b in tb1)
        per_step = {"value": ev1 / (sum(ms1) / 1e3), "unit": UNIT, "ms_per_step": sum(ms1) / K,
                    "l2": "flushed (256 MiB write) before every step, one CUDA graph per step"}
    # ---- per-op durations: the same grouped steps, ONE op bracketed per run --
    # alone: the step's ops serialised on one stream, one op bracketed per run
    # (its own duration, L2 warm from the ops before it); in_step: the timed
    # configuration (two streams), the op's duration while it shares the GPU
    op_mean, op_instr_step, op_in_step = {}, {}, {}
    if ws == 1 and getattr(st, "fused", False) and not args.profile:
        for op, serial in (("prep", True), ("build", True), ("update", True), ("gemm", True), ("prep", False),
                           ("update", False), ("gemm", False)):
            sti = make_stage(False)
            gi, si = capture_groups(sti, gs, op=op, serial=serial)
            ms_i, _, opm = timed_run_groups(sti, gi, si, W, K, gs, op=op)
            _C.check(si)
            del gi, sti
            if opm and serial:
                op_mean[op] = float(np.mean(opm))
                op_instr_step[op] = float(sum(ms_i)) / K
            elif opm:
                op_in_step[op] = float(np.mean(opm))
    # ---- roofline of the dominant op ---------------------------------------
    peaks = _peaks()
    mean_U = float(np.mean(U_host[timed_batches]))
    alg = algorithmic(cfg, sc, mean_U)
    traffic = _ncu_traffic(args.config)
    # the dominant KERNEL: k_prep (prep), k_build_x (build) or k_gru_tc (gemm, timed alone by the
    # library's events); the 'update' op is the GEMM plus its forked write-back branch (two kernels),
    # kept in dominant_of for reference
    kernel_ops = [o for o in op_mean if o != "update"] if "gemm" in op_mean else [o for o in op_mean if o != "gemm"]
    dom = max(kernel_ops, key=op_mean.get) if op_mean else "update"
    rooflines = {}
    for op, t_ms in op_mean.items():
        if op in ("update", "gemm"):
            r = _tensor_roofline(args.gru, alg["update_flops"], t_ms, peaks, st, burst=True)
            if op == "gemm":
                r["kernel"] = "k_gru_tc alone (events recorded by the library around the GEMM launch inside " \
                              "mspipe_gru_apply_commit; the write-back branch excluded)"
        else:
            ach = alg[op] / (t_ms / 1e3) / 1e9
            r = {"kernel": {"prep": "k_prep (A1 sampler + A2 dedup + A3 subgraph gather)",
                            "build": "k_build_x (A5 message + time encoding -> GEMM operand, mail rows)"}[op],
                 "bound": "hbm", "achieved": ach,
                 "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                 "peak_source": peaks["source"] + " copy bandwidth", "bytes_per_launch": alg[op]}
        r["launch_ms_mean"] = t_ms
        r["launch_ms_source"] = ("CUDA events around this op only, on its launching stream, in the same grouped "
                                 "step graphs with the step's ops serialised (the kernel alone on the GPU, L2 warm "
                                 "from the ops before it); instrumented serial ms/step %.4f" % op_instr_step[op])
        if op in op_in_step:
            r["launch_ms_in_step"] = op_in_step[op]
        kname = {"prep": "k_prep", "update": "k_gru_tc", "gemm": "k_gru_tc", "build": "k_build_x"}[op]
        ncu = (traffic or {}).get(kname)
        r["traffic"] = ncu["dram_bytes"] if ncu else None
        if ncu:
            r["ncu"] = ncu
        rooflines[op] = r
    roof = rooflines.get(dom) or _tensor_roofline(args.gru, alg["update_flops"], ms_step, peaks, st)
    roof["dominant_of"] = {k2: v for k2, v in op_mean.items()}
    roof["in_step_ms"] = op_in_step
    roof["gru_flops_per_launch"] = alg["update_flops"]
    roof_gather = rooflines.get("prep")
    roof_features = None
    if "build" in rooflines and dom != "build":
        roof["build"] = rooflines["build"]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
           "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "bf16-gemm/f32" if args.gru == "bf16" else "f32", "data": "synthetic",
           "config": {"workload": args.config, "events": int(E), "tcsr_events": int(tcsr_events or E),
                      "tcsr_nnz": nnz, "num_nodes": cfg.num_nodes,
                      "batch": cfg.batch, "staleness_k": k, "schedule": args.schedule, "fanout": cfg.fanout,
                      "mem_dim": cfg.mem_dim, "edge_dim": cfg.edge_dim, "time_dim": cfg.time_dim,
                      "mitigation": bool(mit), "features": args.features, "fetch_mail": args.fetch_mail,
                      "gru": {"tc": "fp32-3xtf32-tcgen05", "bf16": "bf16-operands-tcgen05 (fp32 accumulate/state)",
                              "simt": "fp32-simt"}[args.gru],
                      "l2": (("flushed (256 MiB write) between timed steps, outside the timed events" if gs == 1 else
                              f"flushed (256 MiB write) before every replay of a {gs}-step CUDA graph, outside "
                              f"the timed events; the per-step-flushed protocol is in per_step_graphs")
                             if args.l2 == "flush" else "warm: steps back to back, state tables L2-resident"),
                      "steps_per_graph": gs,
                      "parallelism": ("single" if ws == 1 else
                                      f"shard{ws}: node-id-sharded memory, window transport (stores into peers' "
                                      f"windows + NCCL barriers), global batch {G * cfg.batch}" if sharded
                                      else f"replicas{ws}")},
           "blocks": {"count": len(blocks), "timed_ms_total": float(sum(b[0] for b in blocks)),
                      "rates": rates, "rule": f"K-step blocks (reset + W warm-up each) until >= {MIN_TIMED_MS} ms; "
                                              "value = the median block"},
           "roofline": roof, "roofline_gather": roof_gather,
           "roofline_gemm": (rooflines.get("gemm") if dom != "gemm" else None) or
                            (rooflines.get("update") if dom != "update" else None),
           "roofline_features": roof_features,
           "per_step_graphs": per_step,
           "gpu_launches": _launches(st.step_ops(), timed_batches, bool(mit), getattr(st, "fused", False), sharded,
                                     args.features),
           "clocks": clocks}
    if sharded:
        out["exchange"] = _exchange_report(st, W + K, ms_step)
    if args.profile:
        if rank == 0:
            print(json.dumps(out))
        return
    del st
    # ---- row F4: the same steps with the training stage after every commit ----
    if ws == 1 and not args.no_train and getattr(sc, "use_fused")() and args.gru == "tc" and not args.features:
        try:
            out["train"] = train_measurement()
        except Exception as ex:  # reported, never hides the headline
            out["train"] = {"error": f"{type(ex).__name__}: {ex}"}
    if ws == 1 and not args.no_apan and getattr(sc, "use_fused")() and args.gru == "tc" and not args.features:
        try:
            out["apan"] = apan_measurement()
        except Exception as ex:  # reported, never hides the headline
            out["apan"] = {"error": f"{type(ex).__name__}: {ex}"}
    # ---- e2e: host buffers through the same C-ABI calls ---------------------
    blocks2, _, st2 = run_blocks(True)
    v2, ms2, _, _ = block_value(blocks2)
    out["e2e"] = {"value": v2, "unit": UNIT, "h2d_bytes_per_step": st2.h2d_bytes_per_batch(),
                  "d2h_bytes_per_step": (st2.d2h_bytes_per_batch(mean_U) if not sharded
                                         else st2.d2h_bytes_per_batch()),
                  "ms_per_step": ms2, "blocks": len(blocks2)}
    del st2
    # ---- HBM probe: A3 / A7 kernels on a table that misses L2
    if rank == 0 and ws == 1 and not args.no_probe:
        out["hbm_probe"] = hbm_probe(dev, cfg, peaks, flush, args.seed)
    # ---- CPU oracle beside it (rank 0, N = 1 only) ---------------------------
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(w, cfg, k, args.schedule, mit, args.cpu_events)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


MIN_TIMED_MS = 100.0
MAX_BLOCKS = 50


def _window(args):
    """(events the batches run over, events the T-CSR is built from)."""
    if args.config == "gdelt":
        ev = args.events if args.events is not None else GDELT_WINDOW
        tev = args.tcsr_events if args.tcsr_events is not None else None  # None: the whole stream
        from synth import CONFIGS
        return ev, (CONFIGS["gdelt"].num_events if tev is None else max(tev, ev))
    return args.events, (max(args.tcsr_events, args.events or 0) if args.tcsr_events else None)


GDELT_WINDOW = 4_000_000  # the first 1,000 batches, parity-tested against the oracle


def _tensor_roofline(gru, flops, t_ms, peaks, st, burst=False):
    """burst: the kernel timed alone (MEASURED_PEAKS burst figure); else inside a
    long step (the sustained figure)."""
    ach = flops / (t_ms / 1e3) / 1e12
    bf16 = peaks["bf16_tflops"] if burst else peaks["bf16_tflops_sustained"]
    which = "burst" if burst else "sustained"
    if gru == "bf16":
        peak = bf16
        return {"kernel": "k_gru_tc<bf16> via mspipe_gru_apply_commit (GEMM + gates + LWW commit epilogue)",
                "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": f"{peaks['source']} bf16 {which}"}
    if gru == "tc":
        # 3xTF32: each useful fp32 MAC costs 3 tf32 MACs; tf32 dense = bf16 x (1.1 / 2.25)
        # nominal ratio (B200_PROFILING.md); sustained bf16 figure (kernel timed inside a long step)
        peak = bf16 * (1.1 / 2.25) / 3.0
        kname = ("k_gru_tc via mspipe_gru_apply_commit (GEMM + gates + LWW commit epilogue)"
                 if getattr(st, "fused", False) else "k_build_x + k_gru_tc via mspipe_memory_update")
        return {"kernel": kname, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak,
                "peak_source": f"{peaks['source']} bf16 {which} x 1.1/2.25 (tf32) / 3 (3xTF32 passes)"}
    peak = 148 * FP32_FMA_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    return {"kernel": "k_build_x + k_gru_simt via mspipe_memory_update", "bound": "alu", "achieved": ach,
            "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1965 MHz (guide unit counts, max clock)"}


def _exchange_report(st, steps, ms_step):
    """Row E: bytes this rank stored into peers' windows per global iteration
    (fetch request ids, reply rows, commit records: the real entries only) over
    the last block (reset, then `steps` steps), and that rate against NVLink
    5's 900 GB/s per direction."""
    try:
        ids, rows, recs = st.exchange_bytes()
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}
    per = (ids + rows + recs) / max(steps, 1)
    return {"bytes_per_iter_per_rank": per, "fetch_id_bytes": ids / steps, "reply_bytes": rows / steps,
            "commit_bytes": recs / steps, "nvlink_gbs": per / (ms_step / 1e3) / 1e9 if ms_step > 0 else None,
            "nvlink_peak_gbs": 900.0,
            "note": "bytes over the whole step time (an upper bound on the exchange time), so the rate is a lower "
                    "bound on the link rate; the owner's own rows are stored locally but counted too"}


def hbm_probe(dev, cfg, peaks, flush, seed):
    """the product's A3 gather (mspipe_memory_fetch ->
    k_fetch_gather) and A7 scatter (mspipe_memory_writeback -> k_writeback) on
    N = 10^7-row tables (mem 4 GB + mail ~15 GB) with uniform ids, so rows miss
    the 126 MB L2: effective GB/s (algorithmic bytes / CUDA-event time, L2
    flushed before every launch) against the measured copy bandwidth."""
    import torch
    from paper_2402_15113_b200 import _C
    N, M, He = 10_000_000, cfg.mem_dim, cfg.edge_dim
    try:
        h = _C.MemoryHandle(N, M, He, 0, dev)
    except Exception as e:  # noqa: BLE001
        return {"error": f"tables: {e}"}
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed + 77)
    stride = h.mail_stride
    row = 4 * M + 8
    res = {"num_nodes": N, "table_bytes": N * (4 * M + 8 + 4 * stride + 8), "ids": "uniform over [0, N)",
           "l2": "flushed (256 MiB write) before every launch"}

    def timeit(fn, reps=20):
        ts_ = []
        for r in range(reps + 2):
            flush.fill_(float(r))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            if r >= 2:
                ts_.append(e0.elapsed_time(e1))
        return float(np.median(ts_))

    for n, tag in ((3 * cfg.batch * (cfg.fanout + 1), "batch"), (1 << 20, "large")):
        ids = torch.randint(0, N, (n,), generator=gen, device=dev, dtype=torch.int32)
        om = torch.empty((n, M), device=dev)
        ots = torch.empty(n, dtype=torch.float64, device=dev)
        t = timeit(lambda: _C.memory_fetch(h, 1, ids, om, ots))
        b = n * (4 + 2 * row)
        res[f"fetch_{tag}"] = {"kernel": "k_fetch_gather (A3, mem rows + mem_ts)", "rows": n, "bytes": b, "ms": t,
                               "achieved_gbs": b / (t / 1e3) / 1e9, "frac": b / (t / 1e3) / 1e9 / peaks["hbm_gbs"]}
        del om, ots
    for U, tag in ((2 * cfg.batch, "batch"), (1 << 18, "large")):
        upd = _C.alloc_update(U // 2, M, stride, dev)
        upd["nodes"][:U] = torch.randperm(N, generator=gen, device=dev)[:U].int()
        upd["num"].fill_(U)
        upd["mem"].uniform_(-1, 1, generator=gen)
        upd["mail"].uniform_(-1, 1, generator=gen)
        upd["ts"].fill_(1.0)
        t = timeit(lambda: _C.memory_writeback(h, h.committed + 1, upd))
        b = U * (4 + 2 * (4 * M + 8 + 4 * stride + 8))
        res[f"writeback_{tag}"] = {"kernel": "k_writeback (A7, mem + mem_ts + mail + mail_ts rows)", "rows": U,
                                   "bytes": b, "ms": t, "achieved_gbs": b / (t / 1e3) / 1e9,
                                   "frac": b / (t / 1e3) / 1e9 / peaks["hbm_gbs"]}
        del upd
    _C.check()
    del h
    torch.cuda.empty_cache()
    res["peak_gbs"] = peaks["hbm_gbs"]
    return res


def _launches(steps, timed_batches, mit, fused, sharded=False, features=False):
    """Kernels of this library per timed step.  fused: prep = k_prep + k_build_x
    (+ k_mitigate), commit = k_gru_tc (h' rows) + k_writeback (mem_ts / mail); otherwise prep = sampler +
    dedup + gather (+ mitigation), commit = build + GEMM (or SIMT GRU) + write-back.  Sharded:
    prep = sampler + dedup + mark + plan + serve + finish, commit = build + GEMM + pack-plan + pack
    + merge-key + merge-apply (NCCL barrier kernels not counted)."""
    if sharded:
        per = {"prep": 6, "commit": 6}
        return int(sum(per[op] for t in timed_batches for op, _ in steps[t]))
    # fused commit: k_gru_tc (+ the k_writeback branch of mem_ts / mail unless MSPIPE_SPLIT_COMMIT=0)
    split = fused and os.environ.get("MSPIPE_SPLIT_COMMIT", "1") != "0"
    per = {"prep": (2 if fused else 3) + (1 if mit else 0) + (1 if features else 0),
           "commit": (2 if split else 1) if fused else 3}
    return int(sum(per[op] for t in timed_batches for op, _ in steps[t]))


def _ncu_traffic(config):
    """Per-launch DRAM bytes and L2 hit rate of each kernel from ONE committed
    `ncu --set full` capture of this config (profiles/ncu_traffic.json, written
    by scripts/make_profiles.py from the .ncu-rep summaries), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(config)


CPU_MIN_S = 10.0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(w, cfg, k, schedule, mit, n_events):
    """The oracle as it stands on the host's cores (T = all usable threads), on a
    bounded sample of the same workload: whole passes over its first n_events
    events until >= CPU_MIN_S; plus one pass of a smaller sample at T = 1."""
    import oracle
    threads = len(os.sched_getaffinity(0))
    E = min(n_events, len(w["src"]))
    sl = slice(0, E)

    def one(sl_):
        oracle.run_stream(cfg.num_nodes, w["src"][sl_], w["dst"][sl_], w["ts"][sl_], w["ef"][sl_], w["params"],
                          cfg.batch, k, schedule, mitigation=mit, fanout=cfg.fanout, neg=w["neg"][sl_])

    oracle.set_threads(threads)
    # whole epochs of the sample (each from the initial state, as the GPU epochs)
    # until at least CPU_MIN_S of CPU work
    passes, t0 = 0, time.perf_counter()
    while True:
        one(sl)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= CPU_MIN_S or passes >= 50:
            break
    E1 = min(E, 20 * cfg.batch)
    oracle.set_threads(1)
    t1 = time.perf_counter()
    one(slice(0, E1))
    dt1 = time.perf_counter() - t1
    oracle.set_threads(threads)
    return {"value": passes * E / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"first {E} events ({-(-E // cfg.batch)} batches) of the same stream x {passes} epoch(s), "
                      f"full per-batch path (sampler, subgraph gather, dedup, {'mitigation, ' if mit else ''}"
                      f"message, f64 GRU, commit), {dt:.1f} s",
            "t1": {"value": E1 / dt1, "unit": UNIT, "cores": 1,
                   "sample": f"first {E1} events ({-(-E1 // cfg.batch)} batches), one pass, {dt1:.1f} s"}}


def run_reference(args):
    """The base contract's reference arm = the CPU oracle, as it stands."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import oracle
    from paper_2402_15113_b200.graph import gamma_quantile
    from synth import make_workload
    # the batches' window only: the oracle's sampler needs no events past it
    # (strict ts < t_q), so its prefix-built graph answers as the full T-CSR does
    w = make_workload(args.config, seed=args.seed, num_events=_window(args)[0])
    cfg = w["cfg"]
    k = cfg.staleness_k if args.k is None else args.k
    mit = None
    if cfg.mitigation and not args.no_mitigation:
        mit = dict(lam=cfg.lam, gamma=gamma_quantile(cfg.num_nodes, w["src"], w["dst"], w["ts"], cfg.quantile_p),
                   n_sim=cfg.n_sim)
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads)
    W, K = args.warmup, args.steps
    nb = -(-len(w["src"]) // cfg.batch)
    W = min(W, nb - 1)
    K = min(K, nb - W)
    E_w = min(W * cfg.batch, len(w["src"]))
    E_t = min((W + K) * cfg.batch, len(w["src"]))

    def timed(E):
        sl = slice(0, E)
        t0 = time.perf_counter()
        oracle.run_stream(cfg.num_nodes, w["src"][sl], w["dst"][sl], w["ts"][sl], w["ef"][sl], w["params"],
                          cfg.batch, k, args.schedule, mitigation=mit, fanout=cfg.fanout, neg=w["neg"][sl])
        return time.perf_counter() - t0

    # the W warm-up batches are replayed untimed inside each run (the oracle starts
    # from S_0): time W+K and W batches (best of 3 each, after one call that absorbs
    # one-time costs) and take the difference; if noise swamps it (K small), the
    # full run's mean rate stands in for the K steps
    timed(min(E_t, cfg.batch))
    t_w = min(timed(E_w) for _ in range(3)) if E_w > 0 else 0.0
    t_all = min(timed(E_t) for _ in range(3))
    dt = t_all - t_w
    if dt <= 0.05 * t_all:
        dt = t_all * (E_t - E_w) / E_t
    value = (E_t - E_w) / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
           "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64-accumulate/f32-state", "data": "synthetic",
           # the same keys as the mspipe arm's config (values of the oracle's run)
           "config": {"workload": args.config, "events": int(len(w["src"])), "tcsr_events": int(len(w["src"])),
                      "tcsr_nnz": None, "num_nodes": cfg.num_nodes,
                      "batch": cfg.batch, "staleness_k": k, "schedule": args.schedule, "fanout": cfg.fanout,
                      "mem_dim": cfg.mem_dim, "edge_dim": cfg.edge_dim, "time_dim": cfg.time_dim,
                      "mitigation": bool(mit), "features": False, "fetch_mail": False,
                      "gru": "f64-oracle", "l2": "host", "steps_per_graph": None, "parallelism": "host cores"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": _cpu_model(),
                            "sample": f"batches {W + 1}..{W + K} of the stream (after {W} untimed), full per-batch path"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="mspipe", choices=["mspipe", "reference"])
    ap.add_argument("--config", default="gdelt",
                    help="workload (synth.CONFIGS); default gdelt, the largest single-GPU configuration")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--schedule", default="exact", choices=["exact", "grouped"])
    ap.add_argument("--fetch-mail", action="store_true")
    ap.add_argument("--gru", default="tc", choices=["tc", "bf16", "simt"],
                    help="tc: 3xTF32 tcgen05 (fp32 parity, default); bf16: tcgen05 bf16 operands "
                         "(2e-2 tolerance); simt: CUDA-core fp32 baseline")
    ap.add_argument("--no-mitigation", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--l2", default="flush", choices=["flush", "warm"],
                    help="flush: 256 MiB write between timed steps (default); warm: back-to-back steps")
    ap.add_argument("--cpu-events", type=int, default=157_474)
    ap.add_argument("--features", action="store_true",
                    help="also run row F2 (feature fetch of the sampled subgraphs) in every step")
    ap.add_argument("--events", type=int, default=None,
                    help="first N events of the config's stream the batches run over (default: all; GDELT: the "
                         "first 4,000,000 = 1,000 batches)")
    ap.add_argument("--tcsr-events", type=int, default=None,
                    help="events the sampler's T-CSR is built from (default: the whole stream for GDELT, else "
                         "--events)")
    ap.add_argument("--no-probe", action="store_true", help="skip the N = 10^7 HBM probe of the A3/A7 kernels")
    ap.add_argument("--no-train", action="store_true", help="skip the row F4 (training stage) measurement")
    ap.add_argument("--no-apan", action="store_true", help="skip the row F3 APAN stage measurement")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no flush/e2e/cpu")
    ap.add_argument("--graph-steps", type=int, default=8,
                    help="consecutive steps captured per CUDA graph (1: one graph per step); N = 1 only")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mspipe(args)


if __name__ == "__main__":
    main()
