"""Debug: the stage with the row F4 training step, eager (no graphs), on a workload prefix."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload, train_params
name = sys.argv[1] if len(sys.argv) > 1 else "gdelt"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 40_000
k = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = make_workload(name, num_events=E)
cfg = w["cfg"]
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch,
                 cfg.staleness_k if k is None else k, train=dict(params=train_params(cfg.mem_dim, cfg.time_dim), lr=1e-4))
st = MemoryStage(sc, w["params"], g, dev)
t = {kk: torch.from_numpy(w[kk]).to(dev) for kk in ("src", "dst", "ts", "neg", "ef")}
st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
st.run()
torch.cuda.synchronize()
_C.check()
print(name, "batches", st.num_batches, "losses", st.trainer.losses[: st.num_batches].cpu().numpy())
