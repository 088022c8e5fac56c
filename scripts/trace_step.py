"""Per-stage timing of the persistent train kernel from CTA 0's clock64 stamps (one traced epoch).

    python scripts/trace_step.py [--mode fast|exact] [--grid G] [--batch B]
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

NAMES = ["params", "img_wait", "conv1", "conv2", "pool2", "fc", "fc_back", "conv2_back", "conv1_back",
         "partial_out", "barrier1", "reduce_sgd", "barrier2"]

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fast")
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--batch", type=int, default=100)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--flat", action="store_true", help="fast mode: force the flat (non-clustered) kernel")
args = ap.parse_args()
dev = torch.device("cuda:0")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
x, y = synth_make_set(args.n, 1)
ctx = Context(0, mode=args.mode)
ctx.set_stream(s.cuda_stream)
if args.grid:
    ctx.set_grid(args.grid)
if args.flat:
    ctx.set_cluster(False)
clustered = args.mode == "fast" and not args.flat and not args.grid and args.batch <= 128
if clustered:  # train_cluster_kernel stamps: 9 loss stash, 10 cluster barrier, 14 DSMEM pre-reduction,
    # 11 grid barrier, 12 slice reduce + sgd, 15 cluster barrier, 13 DSMEM gather + k2 copy
    NAMES = NAMES[:9] + ["cluster_barrier1", "dsmem_reduce+grid_barrier", "slice_reduce_sgd", "gather"]
d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
d_p = torch.zeros(3904, device=dev)
d_p[:3898] = torch.from_numpy(init_params(42)).to(dev)
loss = torch.zeros(4, dtype=torch.float64, device=dev)
steps = (args.n + args.batch - 1) // args.batch
ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 0, 1, args.batch, loss.data_ptr())
tr = torch.zeros(steps * 16, dtype=torch.int64, device=dev)
ctx.set_trace(tr.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 1, 1, args.batch, loss.data_ptr())
e1.record(s)
torch.cuda.synchronize()
t = tr.view(steps, 16).cpu().numpy().astype(np.int64)
if os.environ.get("TRACE_DUMP"):
    np.save(os.environ["TRACE_DUMP"], t)
d = np.diff(t[:, :14], axis=1)  # stage durations (cycles)
med = np.median(d[1:], axis=0)
mhz = 1965.0
sub = np.median(t[1:, 14] - t[1:, 11]) / 1965.0, np.median(t[1:, 15] - t[1:, 14]) / 1965.0, np.median(t[1:, 12] - t[1:, 15]) / 1965.0
if clustered:
    sub = (np.median(t[1:, 14] - t[1:, 10]) / mhz, np.median(t[1:, 11] - t[1:, 14]) / mhz,
           np.median(t[1:, 15] - t[1:, 12]) / mhz)
keys = ("dsmem_reduce", "grid_barrier", "cluster_barrier2") if clustered else ("stage_loads", "accumulate", "finish")
out = {"reduce_split_us": {k: round(float(v), 3) for k, v in zip(keys, sub)},
       "mode": args.mode, "kernel": "cluster" if clustered else "flat", "batch": args.batch, "epoch_ms": e0.elapsed_time(e1),
       "step_us_median": float(np.median(t[1:, 13] - t[1:, 0]) / mhz),
       "stage_us_median": {n: round(float(v) / mhz, 3) for n, v in zip(NAMES, med)},
       "info": ctx.info()}
print(json.dumps(out))
