"""Pinned host->device bandwidth with 1, 2 and 4 concurrent copy streams (is the VM link or one copy
engine the limit?).  Measured on a 43-48 GB/s box: 2 streams +5-9%, 4 streams +5-18%."""
import json, torch
x = torch.empty(10000 * 784, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
res = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = x.numel() // ns
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in streams: st.wait_stream(torch.cuda.current_stream())
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                for _ in range(5):
                    d[i*part:(i+1)*part].copy_(x[i*part:(i+1)*part], non_blocking=True)
        for st in streams: torch.cuda.current_stream().wait_stream(st)
        e1.record(); torch.cuda.synchronize()
    res[f"{ns}_streams_GBps"] = 5 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps(res))
