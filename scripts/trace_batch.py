"""Per-CTA phase timing of the batched train kernel (batch_train.cu) from its globaltimer stamps: how long
the CTAs' rounds take, how far apart they finish, and what the grid barriers and the reduction cost.

    python scripts/trace_batch.py [--batch 16384] [--n 32768]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import init_params, synth_make_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16384)
ap.add_argument("--n", type=int, default=32768)
args = ap.parse_args()
dev = torch.device("cuda:0")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
x, y = synth_make_set(args.n, 1)
ctx = Context(0, mode="fast")
ctx.set_stream(s.cuda_stream)
ctx.set_batched(1)
d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
d_p = torch.zeros(3904, device=dev)
d_p[:3898] = torch.from_numpy(init_params(42)).to(dev)
loss = torch.zeros(4, dtype=torch.float64, device=dev)
steps = (args.n + args.batch - 1) // args.batch
ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 0, 1, args.batch, loss.data_ptr())
grid = 148 * 2 + 8  # upper bound on the batched grid; rows beyond the launch stay zero
tr = torch.zeros(steps * grid * 8, dtype=torch.int64, device=dev)
ctx.set_trace(tr.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 1, 1, args.batch, loss.data_ptr())
e1.record(s)
torch.cuda.synchronize()
ctx.set_trace(0)
info = ctx.info()
t = tr.view(-1, 8).cpu().numpy().astype(np.int64)
nb = int(np.count_nonzero(t[:, 0])) // steps
t = t[: steps * nb].reshape(steps, nb, 8)
us = lambda v: round(float(v) / 1000.0, 3)  # noqa: E731
per_step = []
for k in range(steps):
    z = t[k]
    start = z[:, 0].min()
    busy = z[:, 1] - z[:, 0]
    per_step.append({
        "step_us": us(z[:, 4].max() - (t[k - 1][:, 4].max() if k else start)),
        "rounds_us_min_med_max": [us(busy.min()), us(np.median(busy)), us(busy.max())],
        "rounds_per_cta_min_max": [int(z[:, 5].min()), int(z[:, 5].max())],
        "start_spread_us": us(z[:, 0].max() - z[:, 0].min()),
        "finish_spread_us": us(z[:, 1].max() - z[:, 1].min()),
        "barrier1_us": us(z[:, 2].max() - z[:, 1].max()),
        "reduce_us_max": us((z[:, 3] - z[:, 2]).max()),
        "barrier2_us": us(z[:, 4].max() - z[:, 3].max()),
        "idle_frac_before_barrier1": round(float(np.mean(z[:, 1].max() - z[:, 1]) / (z[:, 1].max() - start)), 4),
    })
    if os.environ.get("TRACE_DUMP"):
        np.save(os.environ["TRACE_DUMP"], t)
# co-resident CTAs: does the CTA that entered the kernel first (on its SM) finish its rounds first?
z0 = t[0]
pairs = {}
for b in range(nb):
    pairs.setdefault(int(z0[b, 6]), []).append(b)
first_faster, ratios = 0, []
for sm, bs in pairs.items():
    if len(bs) != 2:
        continue
    b0, b1 = sorted(bs, key=lambda b: z0[b, 7])
    busy = [float(np.sum(t[:, b, 1] - t[:, b, 0])) for b in (b0, b1)]
    first_faster += busy[0] < busy[1]
    ratios.append(max(busy) / max(min(busy), 1.0))
coresidency = {"sms_with_2_ctas": len(ratios), "first_entered_is_faster": int(first_faster),
               "slow_over_fast_busy_median": round(float(np.median(ratios)), 4) if ratios else None}
print(json.dumps({"coresidency": coresidency, "batch": args.batch, "n": args.n, "grid": nb, "epoch_ms": e0.elapsed_time(e1), "steps": per_step,
                  "info": info}))
