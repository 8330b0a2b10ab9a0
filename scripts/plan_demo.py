"""Row F1 end to end on one GPU: C3 cap from the stream, stage durations
profiled from the library's own kernels (+ an emulated training stage), the
minimal-staleness plan, and the stage run under that plan (parity vs oracle on
a prefix, throughput of the plan's stream order).

  python scripts/plan_demo.py [config] [train_ms] [events]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from paper_2402_15113_b200.planner import StageProfile, k_max_for_stream, plan, stage_config_for_plan, stale_fractions
from synth import make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "wiki"
train_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.030
events = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = make_workload(name, num_events=events)
cfg = w["cfg"]
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
t = {x: torch.from_numpy(w[x]).to(dev) for x in ("src", "dst", "ts", "neg", "ef")}
out = {"config": name, "events": int(len(w["src"])), "batch": cfg.batch}

# C3: stale share per paper k, and k_max
k_max, hist = k_max_for_stream(g, t["src"], t["dst"], cfg.batch)
out["stale_fraction_by_k"] = {k: float(f) for k, f in zip(range(1, 9), stale_fractions(hist, range(1, 9)))}
out["k_max"] = k_max


def timed(sc, steps=None, instrument=False):
    st = MemoryStage(sc, w["params"], g, dev)
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    ops = st.step_ops()
    s = torch.cuda.Stream()
    if instrument:
        st.reserve_timing_events(8 * sum(len(o) for o in ops) + 16)
    graphs = [_C.StepGraph().capture(lambda: st.run_ops(o), s) for o in ops]
    st.memory.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for gr in graphs:
            gr.replay(s)
        e1.record(s)
    torch.cuda.synchronize()
    op_ms = {}
    if instrument:
        for nm in ("prep", "build", "update", "sample", "fetch", "writeback"):
            ends = st.timing.get(nm + "_end", [])
            if ends:
                op_ms[nm] = float(np.mean([a.elapsed_time(b) for a, b in zip(st.timing[nm], ends)]))
    return e0.elapsed_time(e1) / len(graphs), op_ms


# profile the library's stages (k = 1 build, exact schedule), emulated training
base = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, 1)
_, op_ms = timed(base, instrument=True)
prof = StageProfile.from_stage_timing(op_ms, train_ms)
out["tau_ms"] = dict(zip(("sample", "fetch_feature", "fetch_memory", "train", "update_memory"), prof.tau))
nb = -(-len(w["src"]) // cfg.batch)
try:
    k_plan = plan(prof.tau, nb, k_max)
    out["feasible"] = True
except ValueError as err:  # C2 cannot hold: the update stage outlasts training
    out["feasible"] = False
    out["infeasible"] = str(err)
    k_plan, _ = _C.plan_min_staleness(prof.tau, nb, k_max)
out["k_plan_steady"] = int(np.median(k_plan[10:])) if nb > 10 else None
out["k_plan_hist"] = {int(v): int(c) for v, c in zip(*np.unique(k_plan, return_counts=True))}
b, e = _C.plan_timeline(prof.tau, nb, k_plan)
stalls = int(np.sum(b[10:, 3] > e[9:-1, 3] + 1e-9)) if nb > 10 else 0
out["model_training_stalls_after_warmup"] = stalls
sc = stage_config_for_plan(base, k_plan)
ms_plan, _ = timed(sc)
ms_exact, _ = timed(base)
out["stage_ms_per_step_plan"] = ms_plan
out["stage_ms_per_step_exact_k1"] = ms_exact
print(json.dumps(out, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"plan_{name}.json"), "w") as f:
    json.dump(out, f, indent=1)
