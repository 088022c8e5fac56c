"""Pinned host->device copy bandwidth on this box (the e2e ingestion bound): 31.36 MB like one epoch."""
import json

import torch

x = torch.empty(10000 * 784, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
res = {}
for label, chunk in (("whole", x.numel()), ("chunk_1group", 100 * 784)):
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(x, non_blocking=True)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            for lo in range(0, x.numel(), chunk):
                d[lo:lo + chunk].copy_(x[lo:lo + chunk], non_blocking=True)
        e1.record(s)
        s.synchronize()
    res[label + "_GBps"] = 5 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps(res))
