"""Widened CNN (BASELINE.json configs[4]) on one B200: training images/s per GEMM engine, the three conv2
contractions timed alone per engine (the tensor-core question of configs[4]), and forward-only images/s.

    python scripts/wide_bench.py [--batch 100] [--n 1000] [--steps 3] [--out file.jsonl]

Each line is one JSON record.  FLOP counts are algorithmic (109,918,080 MAC per
training image; 34,611,200 MAC per conv2 contraction per image).  Device time by CUDA events on the
launching stream; L2 is flushed (256 MiB write) before every timed repetition.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import wide_init_params, wide_make_set  # noqa: E402

FLOP_TRAIN = 2 * 109_918_080
FLOP_GEMM = 2 * 34_611_200
FLOP_FWD = 2 * (2_880_000 + 34_611_200 + 108_160)
PEAK_FP32 = 148 * 128 * 2 * 1965e6 / 1e12       # TFLOP/s, CUDA cores at sm_max_mhz
PEAK_TF32 = 1612.4 / 2                           # dense TF32 = half the measured bf16 (MEASURED_PEAKS.json)

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=100)
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--out", default="")
args = ap.parse_args()

dev = torch.device("cuda:0")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
x, y = wide_make_set(args.n, 1)
p0 = wide_init_params(42)
d_x, d_y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
ctx = Context(0)
ctx.set_stream(s.cuda_stream)
out = open(args.out, "a") if args.out else None


def emit(rec):
    line = json.dumps(rec)
    print(line, flush=True)
    if out:
        out.write(line + "\n")


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for engine in ("tc", "fp32"):
    d_p = torch.from_numpy(p0.copy()).to(dev)
    loss = torch.zeros(4, dtype=torch.float64, device=dev)
    ctx.wide_train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 0, 1, args.batch,
                          loss.data_ptr(), engine)  # warm-up epoch
    ms = timed(lambda: ctx.wide_train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 0, 1,
                                             args.batch, loss.data_ptr(), engine), args.steps)
    ips = args.n / (ms / 1e3)
    emit({"config": "widened_train", "engine": engine, "batch": args.batch, "n": args.n, "ms_per_epoch": ms,
          "images_per_s": ips, "tflops": ips * FLOP_TRAIN / 1e12, "fp32_core_roofline_frac": ips * FLOP_TRAIN / 1e12 / PEAK_FP32,
          "loss": float(loss[0].item())})
    for which, name in ((0, "conv2_forward"), (1, "conv2_weight_grad"), (2, "conv2_backin")):
        for eng in ("tc", "fp32"):
            ms = timed(lambda: ctx.wide_gemm_device(which, eng), max(args.steps, 5))
            tf = args.batch * FLOP_GEMM / (ms / 1e3) / 1e12
            emit({"config": "widened_gemm", "gemm": name, "engine": eng, "batch": args.batch, "ms": ms, "tflops": tf,
                  "frac_of_engine_peak": tf / (PEAK_TF32 / 3 if eng == "tc" else PEAK_FP32),
                  "peak_note": "tc: 3xTF32 => 1/3 of dense TF32 (half of measured bf16); fp32: 148x128x2x1965 MHz"})
    break  # the GEMM comparison needs one trained group only
for engine in ("tc", "fp32"):
    ms = timed(lambda: ctx.wide_train_device(d_x.data_ptr(), d_y.data_ptr(), args.n, d_p.data_ptr(), 0.05, 0, 1,
                                             args.batch, loss.data_ptr(), engine), args.steps)
    ips = args.n / (ms / 1e3)
    emit({"config": "widened_train", "engine": engine, "batch": args.batch, "n": args.n, "ms_per_epoch": ms,
          "images_per_s": ips, "tflops": ips * FLOP_TRAIN / 1e12,
          "fp32_core_roofline_frac": ips * FLOP_TRAIN / 1e12 / PEAK_FP32})
