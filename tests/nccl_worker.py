"""Worker of tests/test_gpu_nccl.py: one process per GPU (torchrun), node
memory sharded over the ranks with the library's window transport (CUDA IPC +
NCCL barriers), the whole stream through ShardRank (two streams when k >= 1),
then rank 0 assembles the global tables and compares them with the oracle at
the global batch G·B (pin P10)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    name, k, out_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2402_15113_b200 import ShardRank, StageConfig, _C, build_tcsr
    from paper_2402_15113_b200.dist import share_nccl_id
    from synth import make_workload
    w = make_workload(name, seed=21, num_events=12_000 if name != "tiny" else None)
    cfg = w["cfg"]
    sc = StageConfig(cfg.num_nodes, cfg.mem_dim, cfg.edge_dim, cfg.time_dim, cfg.fanout, cfg.batch, k)
    g = build_tcsr(cfg.num_nodes, w["src"], w["dst"], w["ts"], dev)
    st = ShardRank(sc, w["params"], g, dev, rank, world, share_nccl_id(rank))
    t = {kk: torch.from_numpy(w[kk]).to(dev) for kk in ("src", "dst", "ts", "neg", "ef")}
    st.bind_resident(t["src"], t["dst"], t["ts"], t["neg"], t["ef"])
    st.run()
    torch.cuda.synchronize()
    _C.check()
    sent = st.exchange_bytes()
    parts = {kk: getattr(st.memory, kk).cpu().numpy() for kk in ("mem", "mem_ts")}
    allp = [None] * world
    dist.all_gather_object(allp, parts)
    if rank == 0:
        import oracle
        N = cfg.num_nodes
        mem = np.zeros((N, cfg.mem_dim), np.float32)
        mts = np.zeros(N)
        for r, p in enumerate(allp):
            mem[r::world] = p["mem"]
            mts[r::world] = p["mem_ts"]
        ref, _ = oracle.run_stream(N, w["src"], w["dst"], w["ts"], w["ef"], w["params"], world * cfg.batch, k)
        rel = np.linalg.norm(mem - ref["mem"], axis=1) / np.maximum(np.linalg.norm(ref["mem"], axis=1), 1e-3)
        with open(out_path, "w") as f:
            json.dump({"mem_ts_equal": bool(np.array_equal(mts, ref["mem_ts"])), "rel_max": float(rel.max()),
                       "sent_bytes": sent, "batches": int(st.num_batches)}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
