"""Row E on real NCCL + NVLink: runs whenever >= 2 GPUs are visible (the
driver's one-GPU boxes skip it).  torchrun starts one process per GPU
(tests/nccl_worker.py); the sharded stream must equal the oracle at the
global batch G·B (pin P10): mem_ts bit-exact, memory within 1e-4."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,k", [("tiny", 0), ("wiki", 1), ("lastfm", 2)])
def test_nccl_sharded_stream_equals_oracle(tmp_path, name, k):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip(f"needs >= 2 GPUs ({n} visible)")
    world = min(n, 8)
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "nccl_worker.py"), name, str(k), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    print(f"{name} k={k} G={world}: row-rel max {res['rel_max']:.3g}, bytes stored per rank {res['sent_bytes']}")
    assert res["mem_ts_equal"]
    assert res["rel_max"] <= 1e-4
