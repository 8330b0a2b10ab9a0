"""Experiment: per-op timeline inside a step, resident vs staged (e2e) inputs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload
w = make_workload("wiki"); cfg = w["cfg"]; dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
for staged in (False, True):
    st = MemoryStage(StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, 1), w["params"], g, dev)
    if staged:
        st.bind_host(w["src"], w["dst"], w["ts"], w["neg"], w["ef"])
    else:
        t = {k: torch.from_numpy(w[k]).to(dev) for k in ("src", "dst", "ts", "neg", "ef")}
        st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    ops = st.step_ops()
    st.reserve_timing_events(8 * sum(len(o) for o in ops) + 16)
    s = torch.cuda.Stream()
    marks, graphs = [], []
    for o in ops:
        before = {k: len(v) for k, v in st.timing.items()}
        graphs.append(_C.StepGraph().capture(lambda: st.run_ops(o), s))
        marks.append({k: (before.get(k, 0), len(v)) for k, v in st.timing.items()})
    st.memory.reset()
    rec = {}
    with torch.cuda.stream(s):
        e = []
        for n, gr in enumerate(graphs[:200]):
            flush.fill_(float(n))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); gr.replay(s); e1.record(s)
            e.append((n, e0, e1))
    torch.cuda.synchronize()
    tot = []
    for n, e0, e1 in e[10:]:
        tot.append(e0.elapsed_time(e1))
        for name in ("prep", "build", "update"):
            a, b = marks[n].get(name, (0, 0))
            for q in range(a, b):
                rec.setdefault(name + "@start", []).append(e0.elapsed_time(st.timing[name][q]))
                rec.setdefault(name + "@end", []).append(e0.elapsed_time(st.timing[name + "_end"][q]))
    print("staged" if staged else "resident", "step", round(np.mean(tot) * 1e3, 2), {k: round(np.mean(v) * 1e3, 2) for k, v in sorted(rec.items(), key=lambda kv: np.mean(kv[1]))})
