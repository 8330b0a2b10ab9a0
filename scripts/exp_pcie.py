"""Raw pinned H2D / D2H copy throughput at the e2e record sizes (one B200)."""
import torch
dev = torch.device("cuda:0")
for nbytes in (12_000, 424_800, 4 << 20, 64 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            for _ in range(5):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 50
            e0.record(s)
            for _ in range(n):
                fn()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        print(f"{name} {nbytes:>10d} B: {us:8.2f} us/copy  {nbytes / us / 1e3:6.2f} GB/s")
