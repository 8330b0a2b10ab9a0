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
commit's result back.  Default workload: the Wikipedia-shaped stream
(BASELINE.json configs[1]) at its build staleness k=1.

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
    w = make_workload(args.config, seed=args.seed, num_events=args.events)
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
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    # N > 1: node-id-sharded memory over NCCL (row E); MSPIPE_BENCH_REPLICAS=1 runs
    # N independent single-GPU replicas instead (ablation)
    sharded = ws > 1 and os.environ.get("MSPIPE_BENCH_REPLICAS", "0") != "1"
    G = ws if sharded else 1
    E = len(w["src"])
    nb = -(-E // (G * cfg.batch))
    U_host = _unique_counts(w["src"], w["dst"], G * cfg.batch)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

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
        else:
            t = {kk: torch.from_numpy(w[kk]).to(dev) for kk in ("src", "dst", "ts", "neg", "ef")}
            st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
        if args.features:  # row F2: feature tables resident in HBM (the stream's edge features, node features)
            from synth import node_features
            st.bind_features(node_features(args.seed, cfg.num_nodes, cfg.node_dim) if cfg.node_dim else None,
                             torch.from_numpy(w["ef"]).to(dev))
        return st

    def capture(st, timing):
        s = torch.cuda.Stream(device=dev)
        st.timing = None
        if timing:
            st.reserve_timing_events(8 * sum(len(o) for o in st.step_ops()) + 16)
        graphs, marks = [], []
        for ops in st.step_ops():
            before = {kk: len(v) for kk, v in (st.timing or {}).items()}
            graphs.append(_C.StepGraph().capture(lambda: st.run_ops(ops), s))
            marks.append({kk: (before.get(kk, 0), len(v)) for kk, v in (st.timing or {}).items()})
        st.memory.reset()
        return graphs, marks, s

    def timed_run(st, graphs, marks, s, W, K, profile=False):
        """W warm-up + K timed steps (wrapping over epochs); returns per-step ms and per-op ms."""
        step_ms, op_ms = [], {}
        pending = []
        total = W + K
        with torch.cuda.stream(s):
            for n in range(total):
                t = n % nb
                if t == 0 and n > 0:
                    torch.cuda.synchronize()
                    _collect(pending, step_ms, op_ms, st, marks)
                    st.memory.reset()
                if not profile and args.l2 == "flush":
                    flush.fill_(float(n))
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                graphs[t].replay(s)
                e1.record(s)
                if n >= W:
                    pending.append((t, e0, e1))
            torch.cuda.synchronize()
        _collect(pending, step_ms, op_ms, st, marks)
        return step_ms, op_ms

    def capture_groups(st, gs):
        """One CUDA graph per gs consecutive steps (the epoch's last group may be shorter)."""
        s = torch.cuda.Stream(device=dev)
        st.timing = None
        sops = st.step_ops()
        groups = []
        for j in range(0, len(sops), gs):
            idx = list(range(j, min(j + gs, len(sops))))

            def run_group(idx=idx):
                for t in idx:  # e2e copies join only at the graph's end
                    st.run_ops(sops[t], join_copies=(t == idx[-1]))
            groups.append((_C.StepGraph().capture(run_group, s), idx))
        st.memory.reset()
        return groups, s

    def timed_run_groups(st, groups, s, W, K, gs):
        """Warm-up replays until >= W steps ran, then replays of full gs-step groups
        until exactly K steps are timed (an epoch's shorter last group runs untimed);
        L2 flushed before every replay, one event pair per replay.  Returns
        (per-replay ms list, timed step indices)."""
        ms, timed, pending = [], [], []
        warm, r = 0, 0
        with torch.cuda.stream(s):
            while len(timed) + len(pending) * gs < K:
                j = r % len(groups)
                if j == 0 and r > 0:
                    torch.cuda.synchronize()
                    st.memory.reset()
                graph, idx = groups[j]
                if args.l2 == "flush":
                    flush.fill_(float(r))
                if warm >= W and len(idx) == gs:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    graph.replay(s)
                    e1.record(s)
                    pending.append((e0, e1, idx))
                else:
                    graph.replay(s)
                    warm += len(idx)
                r += 1
            torch.cuda.synchronize()
        for e0, e1, idx in pending:
            ms.append(e0.elapsed_time(e1))
            timed.extend(idx)
        return ms, timed

    def _collect(pending, step_ms, op_ms, st, marks):
        for t, e0, e1 in pending:
            step_ms.append(e0.elapsed_time(e1))
            if st.timing:
                for name in ("prep", "build", "sample", "dedup", "fetch", "update", "writeback", "features"):
                    a, b = marks[t].get(name, (0, 0))
                    ends = st.timing.get(name + "_end", [])
                    for q in range(a, b):
                        op_ms.setdefault(name, []).append(st.timing[name][q].elapsed_time(ends[q]))
                        # offsets inside the step (diagnostic timeline)
                        op_ms.setdefault(name + "@start", []).append(e0.elapsed_time(st.timing[name][q]))
                        op_ms.setdefault(name + "@end", []).append(e0.elapsed_time(ends[q]))
        pending.clear()

    W, K = args.warmup, args.steps
    # ---- device-resident run (the `value`) ---------------------------------
    # The timed graphs carry no per-op event nodes (each one is an extra graph
    # node on the critical path); the per-op breakdown for the roofline comes
    # from a second, instrumented replay of the same steps right after.
    # steps per captured graph: launch latency between graphs (~6 us, the same
    # with or without the L2 flush) is paid once per graph, not once per step
    gs = 1
    if ws == 1 and not args.profile:  # the largest divisor of K up to --graph-steps (exactly K steps timed)
        gs = max(d for d in range(1, max(1, min(args.graph_steps, nb - 1)) + 1) if K % d == 0)
    st = make_stage(False)
    if gs > 1:
        groups, s = capture_groups(st, gs)
    else:
        graphs, marks, s = capture(st, timing=False)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        if gs > 1:
            step_ms, timed_batches = timed_run_groups(st, groups, s, W, K, gs)
        else:
            step_ms, _ = timed_run(st, graphs, marks, s, W, K, profile=args.profile)
            timed_batches = [(W + q) % nb for q in range(K)]
    _C.check(s)
    per_step = None
    if gs > 1:
        # the same steps with one graph per step (L2 flushed before each): the
        # per-step protocol, reported beside the grouped headline
        del groups
        st1 = make_stage(False)
        graphs1, marks1, s1 = capture(st1, timing=False)
        ms1, _ = timed_run(st1, graphs1, marks1, s1, W, K)
        _C.check(s1)
        del graphs1
        tb1 = [(W + q) % nb for q in range(K)]
        ev1 = sum(min(cfg.batch, E - b * cfg.batch) for b in tb1)
        per_step = {"value": ev1 / (sum(ms1) / 1e3), "unit": UNIT, "ms_per_step": sum(ms1) / K,
                    "l2": "flushed (256 MiB write) before every step, one CUDA graph per step"}
    else:
        del graphs
    st_i = make_stage(False)
    graphs_i, marks_i, s_i = capture(st_i, timing=True)
    step_ms_instr, op_ms = timed_run(st_i, graphs_i, marks_i, s_i, W, K, profile=args.profile)
    _C.check(s_i)
    del graphs_i
    tot_ms = float(sum(step_ms))
    if ws > 1:
        tt = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot_ms = float(tt.item())
        dist.barrier()
    # events of all ranks in the timed global batches (replicas: every rank its own copy)
    events = sum(min(G * cfg.batch, E - b * G * cfg.batch) for b in timed_batches) * (ws if not sharded else 1)
    value = events / (tot_ms / 1e3)
    # ---- roofline of the dominant op ---------------------------------------
    peaks = _peaks()
    mean_U = float(np.mean(U_host[timed_batches]))
    alg = algorithmic(cfg, sc, mean_U)
    op_mean = {kk: float(np.mean(v)) for kk, v in op_ms.items() if v and "@" not in kk}
    timeline = {kk: float(np.mean(v)) for kk, v in op_ms.items() if v and "@" in kk}
    dom = max(op_mean, key=op_mean.get) if op_mean else "update"
    clocks = clk.summary()
    if dom == "update" and args.gru == "bf16":
        peak_tc = peaks["bf16_tflops_sustained"]
        ach = alg["update_flops"] / (op_mean[dom] / 1e3) / 1e12
        roof = {"kernel": "k_gru_tc<bf16> via mspipe_gru_apply_commit (GEMM + gates + LWW commit epilogue)",
                "bound": "tensor", "achieved": ach, "peak": peak_tc, "unit": "TFLOP/s", "frac": ach / peak_tc,
                "peak_source": f"{peaks['source']} bf16 sustained"}
    elif dom == "update" and args.gru == "tc":
        # 3xTF32: each useful fp32 MAC costs 3 tf32 MACs; tf32 dense = bf16 x (1.1 / 2.25)
        # nominal ratio (B200_PROFILING.md); sustained bf16 figure (kernel timed inside a long step)
        peak_tc = peaks["bf16_tflops_sustained"] * (1.1 / 2.25) / 3.0
        ach = alg["update_flops"] / (op_mean[dom] / 1e3) / 1e12
        kname = ("k_gru_tc via mspipe_gru_apply_commit (GEMM + gates + LWW commit epilogue)"
                 if getattr(st, "fused", False) else "k_build_x + k_gru_tc via mspipe_memory_update")
        roof = {"kernel": kname, "bound": "tensor", "achieved": ach,
                "peak": peak_tc, "unit": "TFLOP/s", "frac": ach / peak_tc,
                "peak_source": f"{peaks['source']} bf16 sustained x 1.1/2.25 (tf32) / 3 (3xTF32 passes)"}
    elif dom == "update":
        sm_clock = 1965.0
        peak_alu = 148 * FP32_FMA_LANES_PER_SM * 2 * sm_clock * 1e6 / 1e12
        ach = alg["update_flops"] / (op_mean[dom] / 1e3) / 1e12
        roof = {"kernel": "k_build_x + k_gru_simt via mspipe_memory_update", "bound": "alu", "achieved": ach,
                "peak": peak_alu, "unit": "TFLOP/s", "frac": ach / peak_alu,
                "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1965 MHz (guide unit counts, max clock)"}
    else:
        ach = alg[dom] / (op_mean[dom] / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "peak_source": peaks["source"]}
    roof["traffic"] = _ncu_traffic(args.config, dom)
    if roof.get("bound") == "tensor":
        roof["note"] = (f"{mean_U:.0f} GEMM rows per batch ({int(-(-mean_U // 128))} M tiles of 128): the contraction "
                        "is a few us of tensor work; the launch is bound by dependent latency (operand chunk "
                        "loads, the K-split partial exchange, the commit epilogue), DESIGN.md section 5")
    roof["op_ms_mean"] = op_mean
    roof["op_share"] = {kk: v / sum(op_mean.values()) for kk, v in op_mean.items()} if op_mean else None
    roof["step_timeline_ms"] = dict(sorted(timeline.items(), key=lambda kv: kv[1]))
    roof["instrumented_ms_per_step"] = float(np.mean(step_ms_instr)) if step_ms_instr else None
    roof["alg_bytes_per_launch"] = {kk: alg[kk] for kk in op_mean if kk in alg}
    roof["gru_flops_per_launch"] = alg["update_flops"]
    gather_op = "prep" if "prep" in op_mean else ("fetch" if "fetch" in op_mean else None)
    if gather_op and dom != gather_op:
        # the gather/scatter kernel against HBM (north star: >= 60 % of the HBM roofline)
        ach_g = alg[gather_op] / (op_mean[gather_op] / 1e3) / 1e9
        roof_gather = {"kernel": "k_prep (A1 sampler + A2 dedup + A3 gather)" if gather_op == "prep"
                       else "k_fetch_gather", "bound": "hbm", "achieved": ach_g, "peak": peaks["hbm_gbs"],
                       "unit": "GB/s", "frac": ach_g / peaks["hbm_gbs"], "bytes_per_launch": alg[gather_op],
                       "traffic": _ncu_traffic(args.config, gather_op)}
    else:
        roof_gather = None
    roof_features = None
    if "features" in op_mean:
        ach_f = alg["features"] / (op_mean["features"] / 1e3) / 1e9
        roof_features = {"kernel": "k_feature_fetch (row F2)", "bound": "hbm", "achieved": ach_f,
                         "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach_f / peaks["hbm_gbs"],
                         "bytes_per_launch": alg["features"]}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
           "ms_per_step": tot_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "bf16-gemm/f32" if args.gru == "bf16" else "f32", "data": "synthetic",
           "config": {"workload": args.config, "events": int(len(w["src"])), "num_nodes": cfg.num_nodes,
                      "batch": cfg.batch, "staleness_k": k, "schedule": args.schedule, "fanout": cfg.fanout,
                      "mem_dim": cfg.mem_dim, "edge_dim": cfg.edge_dim, "time_dim": cfg.time_dim,
                      "mitigation": bool(mit), "features": args.features, "fetch_mail": args.fetch_mail, "gru": {"tc": "fp32-3xtf32-tcgen05", "bf16": "bf16-operands-tcgen05 (fp32 accumulate/state)",
                              "simt": "fp32-simt"}[args.gru],
                      "l2": (("flushed (256 MiB write) between timed steps, outside the timed events" if gs == 1 else
                              f"flushed (256 MiB write) before every replay of a {gs}-step CUDA graph, outside "
                              f"the timed events; the per-step-flushed protocol is in per_step_graphs")
                             if args.l2 == "flush" else "warm: steps back to back, state tables L2-resident"),
                      "steps_per_graph": gs,
                      "parallelism": ("single" if ws == 1 else
                                      f"shard{ws}: node-id-sharded memory, NCCL all-to-all fetch + write-back, "
                                      f"global batch {G * cfg.batch}" if sharded else f"replicas{ws}")},
           "roofline": roof, "roofline_gather": roof_gather, "roofline_features": roof_features, "per_step_graphs": per_step, "gpu_launches": _launches(st.step_ops(), timed_batches, bool(mit),
                                                       getattr(st, "fused", False), sharded, args.features,
                                                       getattr(st, "gemm_build", False)), "clocks": clocks}
    if args.profile:
        if rank == 0:
            print(json.dumps(out))
        return
    # ---- e2e: host buffers through the same C-ABI calls ---------------------
    st2 = make_stage(True)
    if gs > 1:
        groups2, s2 = capture_groups(st2, gs)
    else:
        graphs2, marks2, s2 = capture(st2, timing=False)
    if ws > 1:
        dist.barrier()
    if gs > 1:
        step2, tb2 = timed_run_groups(st2, groups2, s2, W, K, gs)
        graphs2 = groups2
    else:
        step2, _ = timed_run(st2, graphs2, marks2, s2, W, K)
        tb2 = timed_batches
    _C.check(s2)
    events2 = sum(min(G * cfg.batch, E - b * G * cfg.batch) for b in tb2) * (ws if not sharded else 1)
    tot2 = float(sum(step2))
    if ws > 1:
        tt = torch.tensor([tot2], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot2 = float(tt.item())
    out["e2e"] = {"value": events2 / (tot2 / 1e3), "unit": UNIT,
                  "h2d_bytes_per_step": st2.h2d_bytes_per_batch(), "d2h_bytes_per_step": (st2.d2h_bytes_per_batch(mean_U) if not sharded
                                                                         else st2.d2h_bytes_per_batch()),
                  "ms_per_step": tot2 / K}
    del graphs2
    # ---- CPU oracle beside it (rank 0, N = 1 only) ---------------------------
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(w, cfg, k, args.schedule, mit, args.cpu_events)
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


def _launches(steps, timed_batches, mit, fused, sharded=False, features=False, gemm_build=False):
    """Kernels of this library per timed step.  fused: prep = k_prep + k_build_x
    (+ k_mitigate), commit = k_gru_tc (h' rows) + k_writeback (mem_ts / mail); otherwise prep = sampler +
    dedup + gather (+ mitigation), commit = build + GEMM (or SIMT GRU) + write-back.  Sharded:
    prep = sampler + dedup + mark + plan + serve + finish, commit = build + GEMM + clear + pack-plan
    + pack + merge-key + merge-apply (NCCL kernels not counted)."""
    if sharded:
        per = {"prep": 6, "commit": 7}
        return int(sum(per[op] for t in timed_batches for op, _ in steps[t]))
    # fused commit: k_gru_tc (+ the k_writeback branch of mem_ts / mail unless MSPIPE_SPLIT_COMMIT=0;
    # gemm_build's k_gru_fb writes everything itself)
    split = fused and not gemm_build and os.environ.get("MSPIPE_SPLIT_COMMIT", "1") != "0"
    per = {"prep": (1 if gemm_build else 2 if fused else 3) + (1 if mit else 0) + (1 if features else 0),
           "commit": (2 if split else 1) if fused else 3}
    return int(sum(per[op] for t in timed_batches for op, _ in steps[t]))


def _ncu_traffic(config, dom):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(config, {}).get(dom)


CPU_MIN_S = 10.0


def cpu_baseline(w, cfg, k, schedule, mit, n_events):
    import oracle
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads)
    E = min(n_events, len(w["src"]))
    sl = slice(0, E)
    # whole epochs of the sample (each from the initial state, as the GPU epochs)
    # until at least CPU_MIN_S of CPU work
    passes, t0 = 0, time.perf_counter()
    while True:
        oracle.run_stream(cfg.num_nodes, w["src"][sl], w["dst"][sl], w["ts"][sl], w["ef"][sl], w["params"],
                          cfg.batch, k, schedule, mitigation=mit, fanout=cfg.fanout, neg=w["neg"][sl])
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= CPU_MIN_S or passes >= 50:
            break
    return {"value": passes * E / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"first {E} events ({-(-E // cfg.batch)} batches) of the same stream x {passes} epoch(s), "
                      f"full per-batch path (sampler, subgraph gather, dedup, {'mitigation, ' if mit else ''}"
                      f"message, f64 GRU, commit), {dt:.1f} s"}


def run_reference(args):
    """The base contract's reference arm = the CPU oracle, as it stands."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import oracle
    from paper_2402_15113_b200.graph import gamma_quantile
    from synth import make_workload
    w = make_workload(args.config, seed=args.seed, num_events=args.events)
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
           "config": {"workload": args.config, "batch": cfg.batch, "staleness_k": k, "schedule": args.schedule,
                      "fanout": cfg.fanout, "mem_dim": cfg.mem_dim, "edge_dim": cfg.edge_dim,
                      "mitigation": bool(mit), "parallelism": "host cores"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": f"batches {W + 1}..{W + K} of the stream (after {W} untimed), full per-batch path"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="mspipe", choices=["mspipe", "reference"])
    ap.add_argument("--config", default="wiki")
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
                    help="first N events of the config's stream (default: all; GDELT's 191M needs a cap)")
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
