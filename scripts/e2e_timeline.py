"""Where the end-to-end tlb_train call spends its time: pinned H2D bandwidth, then one traced call on
host buffers (CTA 0's per-step clock64 stamps) -- per-step image waits show whether the overlapped
ingestion kept ahead of the kernel.

    python scripts/e2e_timeline.py [--batch 100] [--n 10000] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import init_params, synth_make_digits, synth_make_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=100)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--u8", action="store_true", help="byte ingestion (tlb_train_u8) instead of fp32 images")
args = ap.parse_args()
mhz = 1965.0
x, y = synth_make_set(args.n, 1)
px = torch.from_numpy(x).pin_memory()
py = torch.from_numpy(y).pin_memory()
pu8 = torch.from_numpy(synth_make_digits(args.n, 1)[0]).pin_memory()
d = torch.empty_like(px, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
d.copy_(px, non_blocking=True)
e0.record()
for _ in range(5):
    d.copy_(px, non_blocking=True)
e1.record()
torch.cuda.synchronize()
h2d = 5 * px.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9
p0 = init_params(42)
ctx = Context(0, mode="fast")
steps = (args.n + args.batch - 1) // args.batch
tr = torch.zeros(steps * 16, dtype=torch.int64, device="cuda")
calls = []
for r in range(args.reps + 1):
    if r == args.reps:
        ctx.set_trace(tr.data_ptr())
    t0 = time.perf_counter()
    if args.u8:
        ctx.train_u8(p0, pu8.numpy(), py.numpy(), rate=0.05, epochs=1, batch=args.batch)
    else:
        ctx.train(p0, px.numpy(), py.numpy(), rate=0.05, epochs=1, batch=args.batch)
    calls.append(time.perf_counter() - t0)
t = tr.view(steps, 16).cpu().numpy().astype(np.int64)
wait = (t[:, 2] - t[:, 1]) / mhz
step = (t[1:, 0] - t[:-1, 0]) / mhz
out = {"u8": args.u8, "h2d_GBps": h2d, "call_ms": [round(c * 1e3, 3) for c in calls],
       "traced_kernel_ms": float((t[-1, 13] - t[0, 0]) / mhz / 1e3),
       "img_wait_us_total": float(wait.sum()), "img_wait_us_first": float(wait[0]),
       "steps_waiting_gt_1us": int((wait > 1.0).sum()), "step_us_median": float(np.median(step)),
       "img_wait_us_by_decile": [round(float(w.sum()), 1) for w in np.array_split(wait, 10)]}
print(json.dumps(out))
