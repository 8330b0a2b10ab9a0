"""Experiment: per-step device time of the captured stage under variants
(overlap on/off, double buffer on/off, fused on/off) — L2 flushed between steps.

  python scripts/exp_overlap.py [config] [k]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "wiki"
kk = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = make_workload(name, num_events=int(os.environ["EXP_EVENTS"]) if os.environ.get("EXP_EVENTS") else None)
cfg = w["cfg"]
k = cfg.staleness_k if kk is None else kk
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
t = {x: torch.from_numpy(w[x]).to(dev) for x in ("src", "dst", "ts", "neg", "ef")}
flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)


GROUP = int(os.environ.get("EXP_GROUP", "1"))  # steps captured per graph (timed per graph, / GROUP)
EAGER = bool(os.environ.get("EXP_EAGER"))  # launch the step's kernels directly instead of replaying its graph


def run(overlap, db, fused=None, steps=300, warm=10, l2=True):
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k,
                     double_buffer=db, fused=fused)
    st = MemoryStage(sc, w["params"], g, dev)
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    import paper_2402_15113_b200.stage as stage_mod
    if stage_mod._DEBUG_ONLY == "commit":  # fill every slot with a real prep first (realistic U per commit)
        stage_mod._DEBUG_ONLY = ""
        for ops in st.step_ops()[:8]:
            st.run_ops(ops, overlap=overlap)
        torch.cuda.synchronize()
        st.memory.reset()
        stage_mod._DEBUG_ONLY = "commit"
    s = torch.cuda.Stream()
    sops = st.step_ops()
    groups = [sops[j:j + GROUP] for j in range(0, len(sops), GROUP)]

    def run_group(gr):
        for ops in gr:
            st.run_ops(ops, overlap=overlap)
    graphs = [_C.StepGraph().capture(lambda: run_group(gr), s) for gr in groups]
    st.memory.reset()
    nb = len(graphs)
    eager_ops = st.step_ops()
    ms = []
    with torch.cuda.stream(s):
        for n in range(warm + steps):
            i = n % nb
            if i == 0 and n:
                torch.cuda.synchronize()
                st.memory.reset()
            if l2:
                flush.fill_(float(n))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if EAGER:
                st.run_ops(eager_ops[i], overlap=overlap)
            else:
                graphs[i].replay(s)
            e1.record(s)
            if n >= warm:
                ms.append((e0, e1))
    torch.cuda.synchronize()
    v = np.array([a.elapsed_time(b) for a, b in ms]) * 1e3 / GROUP  # per step
    return np.mean(v), np.median(v)


print(f"{name} k={k} B={cfg.batch}")
if os.environ.get("EXP_HALVES"):
    # each half of the step alone (stage._DEBUG_ONLY is read per run), then both
    import paper_2402_15113_b200.stage as stage_mod
    for only in ("none", "prep", "commit", ""):
        stage_mod._DEBUG_ONLY = only
        m, md = run(True, True)
        print(f"only={only or 'both':6s}: mean {m:6.2f} us  median {md:6.2f} us")
    sys.exit(0)
if os.environ.get("EXP_KNOBS"):
    # EXP_KNOBS="MSPIPE_CATCHUP=0,1,2;MSPIPE_PREP_SMEM=1,0": one knob varied at a time from the defaults
    for spec in os.environ["EXP_KNOBS"].split(";"):
        knob, vals = spec.split("=")
        for v in vals.split(","):
            os.environ[knob] = v
            m, md = run(True, True)
            print(f"{knob}={v}: mean {m:6.2f} us  median {md:6.2f} us")
        del os.environ[knob]
    sys.exit(0)

for overlap, db, fused, l2 in [(False, False, None, True), (True, False, None, True), (True, True, None, True),
                               (False, True, None, True), (True, True, None, False), (True, True, False, True)]:
    m, md = run(overlap, db, fused, l2=l2)
    print(f"overlap={overlap!s:5} db={db!s:5} fused={fused!s:5} l2flush={l2!s:5}: mean {m:6.2f} us  median {md:6.2f} us")
