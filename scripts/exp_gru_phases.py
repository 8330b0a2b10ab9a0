"""Debug experiment: per-CTA phase timestamps of k_gru_tc (built with -DMSPIPE_PHASES)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MSPIPE_LIB"] = "/tmp/libmspipe_dbg.so"  # before the package import
from paper_2402_15113_b200.build import build
dbg = build(force=True, extra_flags=["-DMSPIPE_PHASES"] + os.environ.get("EXP_FLAGS", "").split(),
            out="/tmp/libmspipe_dbg.so")
os.environ["MSPIPE_LIB"] = dbg
import numpy as np, torch
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload
name = sys.argv[1] if len(sys.argv) > 1 else "wiki"
w = make_workload(name, num_events=int(os.environ.get("EXP_EVENTS", "200000" if name == "gdelt" else "60000")))
cfg = w["cfg"]
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
prec = _C.BF16 if (len(sys.argv) > 2 and sys.argv[2] == "bf16") else _C.FP32_3XTF32
st = MemoryStage(StageConfig(cfg.num_nodes, 100, cfg.edge_dim, 100, 10, cfg.batch, cfg.staleness_k, precision=prec),
                 w["params"], g, dev)
t = {k: torch.from_numpy(w[k]).to(dev) for k in ("src", "dst", "ts", "neg", "ef")}
st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
ops = st.step_ops()
for i in range(20):
    st.run_ops(ops[i])
torch.cuda.synchronize()
if os.environ.get("EXP_COLD"):  # the recorded step alone (its prep skipped), after an L2 flush
    import paper_2402_15113_b200.stage as stage_mod
    flush = torch.empty(256 << 18, dtype=torch.float32, device=dev)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    stage_mod._DEBUG_ONLY = "commit"
    st.run_ops(ops[20])
    torch.cuda.synchronize()
    stage_mod._DEBUG_ONLY = ""
L = ctypes.CDLL(dbg)
buf = np.zeros((8192, 16), np.uint64)
print("copy rc", L.mspipe_debug_phases(buf.ctypes.data_as(ctypes.c_void_p), 8192))
U = int(st.upd["num"].item())
used = buf[:, 9] > 0
ph = buf[used].astype(np.int64)
print("U", U, "CTAs recorded", used.sum())
t0 = ph[:, 9].min()
names = {9: "entry", 0: "setup", 2: "mma_done", 3: "acc_full", 4: "tmem_sum", 1: "pushed", 5: "sync", 7: "arrived", 6: "cluster1", 11: "sum_done", 10: "gates_done", 8: "end"}
act = ph[:, 3] > 0
one = act & (ph[:, 8] - ph[:, 9] < np.median(ph[act, 8] - ph[act, 9]) * 1.3)  # CTAs with one tile (the marks are the last tile's)
print("one-tile CTAs", one.sum())
print("active CTAs", act.sum())
for k in [9, 0, 2, 3, 4, 1, 5, 6, 11, 10, 8]:
    col = ph[one, k] - ph[one, 9]
    print(f"{names[k]:10s} min {col.min()/1e3:8.2f} med {np.median(col)/1e3:8.2f} max {col.max()/1e3:8.2f} us")
dead = ~act
if dead.any():
    col = ph[dead, 9] - t0
    print(f"dead entry min {col.min()/1e3:8.2f} med {np.median(col)/1e3:8.2f} max {col.max()/1e3:8.2f} us  n={dead.sum()}")
# kernel-level spread: every CTA's entry and end against the earliest entry
ent = ph[:, 9] - t0
end = ph[act, 8] - t0
print(f"entry spread (all CTAs)  min {ent.min()/1e3:8.2f} med {np.median(ent)/1e3:8.2f} max {ent.max()/1e3:8.2f} us")
print(f"end   (active CTAs)      min {end.min()/1e3:8.2f} med {np.median(end)/1e3:8.2f} max {end.max()/1e3:8.2f} us")
