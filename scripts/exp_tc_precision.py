"""Experiment: 3xTF32 error vs K-split count on the GDELT-shaped teacher-forced batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
sys.path.insert(0, "tests")
import test_gpu_parity as T
dev = torch.device("cuda:0")
for name, i, E in [("gdelt", 3, 20000), ("wiki", 137, None)]:
    st, sl, upd, ref, ev, _ = T._teacher_forced(dev, name, i, E=E, precision=1)
    U = int(upd["num"].item())
    g = upd["mem"][:U].cpu().numpy().astype(np.float64); o = ref["mem"].astype(np.float64)
    err = np.abs(g - o); rel = err / (np.abs(o) + 1e-2)
    bad = err > 1e-4 * np.abs(o) + 1e-6
    print(os.environ.get("MSPIPE_TC_SPLITS"), name, "max abs", err.max(), "mean abs", err.mean(), "bad", bad.sum(), "of", bad.size)
