"""Debug experiment: per-block phase times of k_prep (built with -DMSPIPE_PHASES).
Phases: 0 entry, 1 roots done (block 0: dedup done), 5 build-wait start, 2 flag seen, 3 build done, 4 exit."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MSPIPE_LIB"] = "/tmp/libmspipe_dbg.so"
from paper_2402_15113_b200.build import build
dbg = build(force=True, extra_flags=["-DMSPIPE_PHASES"], out="/tmp/libmspipe_dbg.so")
import numpy as np, torch
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload
name = sys.argv[1] if len(sys.argv) > 1 else "wiki"
w = make_workload(name, num_events=int(os.environ.get("EXP_EVENTS", "200000" if name == "gdelt" else "60000")),
                  tcsr_events=None if not os.environ.get("EXP_FULL") else 10 ** 12)
cfg = w["cfg"]
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, *w.get("tcsr", (w["src"], w["dst"], w["ts"])), dev)
w.pop("tcsr", None)
st = MemoryStage(StageConfig(cfg.num_nodes, 100, cfg.edge_dim, 100, 10, cfg.batch, cfg.staleness_k), w["params"], g, dev)
t = {k: torch.from_numpy(w[k]).to(dev) for k in ("src", "dst", "ts", "neg", "ef")}
st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
ops = st.step_ops()
L = ctypes.CDLL(dbg)
for i in range(10):
    st.run_ops(ops[i])
torch.cuda.synchronize()
L.mspipe_debug_prep_phases(None, 0, 1)
st.run_ops(ops[10])
torch.cuda.synchronize()
buf = np.zeros((8192, 6), np.uint64)
L.mspipe_debug_prep_phases(buf.ctypes.data_as(ctypes.c_void_p), 8192, 0)
used = buf[:, 0] > 0
ph = buf[used].astype(np.int64)
t0 = ph[:, 0].min()
print("blocks", used.sum())
names = {0: "entry", 1: "roots/dedup done", 5: "wait start", 2: "flag seen", 3: "build done", 4: "exit"}
print("block0:", {k: round((ph[0, k] - t0) / 1e3, 2) for k in (0, 3, 4, 5, 2, 1)},
      "(0 entry, 3 table cleared + ids loaded, 4 atomicMax done, 5 counts scanned, 2 dedup done, 1 stamps)")
for k in (0, 1, 5, 2, 3, 4):
    col = ph[1:, k]
    col = col[col > 0] - t0
    if len(col):
        print(f"{names[k]:18s} min {col.min()/1e3:7.2f} med {np.median(col)/1e3:7.2f} max {col.max()/1e3:7.2f} us")
