"""Debug / profiling: the stage with the row F4 training step (mode "train") or the
row F3 APAN updater at k = 0 (mode "apan"), eager (no graphs), on a workload prefix.
  python scripts/exp_train_stage.py <config> <events> [k] [train|apan]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2402_15113_b200 import MemoryStage, StageConfig, _C, build_tcsr
from synth import make_workload, train_params
name = sys.argv[1] if len(sys.argv) > 1 else "gdelt"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 40_000
k = int(sys.argv[3]) if len(sys.argv) > 3 else None
mode = sys.argv[4] if len(sys.argv) > 4 else "train"
w = make_workload(name, num_events=E)
cfg = w["cfg"]
dev = torch.device("cuda:0")
g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
kw = {}
if mode == "train":
    kw["train"] = dict(params=train_params(cfg.mem_dim, cfg.time_dim), lr=1e-4)
else:
    rng = np.random.default_rng(77)
    M, Dm = cfg.mem_dim, cfg.mail_dim
    kw.update(mailbox="apan", apan=dict(w_q=(rng.uniform(-1, 1, (M, M)) / np.sqrt(M)).astype(np.float32),
                                        w_k=(rng.uniform(-1, 1, (M, Dm)) / np.sqrt(Dm)).astype(np.float32)))
    k = 0
sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch,
                 cfg.staleness_k if k is None else k, **kw)
st = MemoryStage(sc, w["params"], g, dev)
t = {kk: torch.from_numpy(w[kk]).to(dev) for kk in ("src", "dst", "ts", "neg", "ef")}
st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
st.run()
torch.cuda.synchronize()
_C.check()
if mode == "train":
    print(name, "batches", st.num_batches, "losses", st.trainer.losses[: st.num_batches].cpu().numpy())
else:
    print(name, "batches", st.num_batches, "mean filled slots", float(st.apan.mb_cnt.float().mean().item()))
