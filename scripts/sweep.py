"""BASELINE.json configs[2] and configs[3] on one B200 (the bench line itself is configs[1]).

  python scripts/sweep.py [--modes fast,exact] [--out gpurun_out/sweep.json]

* configs[3] -- training throughput vs per-step batch B in {1k .. 256k}: a corpus of max(2B, 10k) distinct
  synthetic images (synth::make_set(n, 1) generated on the device, byte-identical to the reference), one
  persistent-kernel launch per timed step = n/B SGD groups; CUDA events on the launching stream.
* configs[2] -- forward-only inference (net::evaluate: forward + argmax + correct count) for N in
  {100, 1k, 10k, 100k, 1M} distinct images (synth::make_set(N, 2) on the device); predictions on the first
  10k checked against the reference's golden predictions (trained params).
Each result is one JSON line with the roofline fraction against the FP32 CUDA-core peak
(148 SMs x 128 lanes x 2 FLOP x sm_max_mhz).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import init_params  # noqa: E402

TRAIN_FLOP, FWD_FLOP = 1_048_320, 407_040


def peak_tflops(sm_count: int) -> float:
    try:
        mhz = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"]
    except Exception:
        mhz = 1965.0
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def timed(stream, fn, reps: int, flush) -> float:
    times = []
    for r in range(reps):
        flush.fill_(float(r))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    return float(np.median(times))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="fast,exact")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--max-batch", type=int, default=262144)
    ap.add_argument("--threads", type=int, default=0, help="fast mode CTA size (256 = two CTAs per SM; 0 = library default)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    out = open(args.out, "w")

    def emit(rec):
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")

    for mode in args.modes.split(","):
        ctx = Context(0, mode=mode)
        ctx.set_stream(stream.cuda_stream)
        if args.threads:
            ctx.set_threads(args.threads)
        thr = args.threads or "auto"
        peak = peak_tflops(ctx.info()["sm_count"])
        # ---- configs[3]: batch sweep -------------------------------------------------------------
        B = 1024
        while B <= args.max_batch:
            n = max(2 * B, 10000)
            d_x = torch.empty(n, 784, device=dev)
            d_y = torch.empty(n, dtype=torch.int32, device=dev)
            ctx.synth_make_set_device(n, 1, d_x.data_ptr(), d_y.data_ptr())
            d_p = torch.zeros(3904, device=dev)
            d_p[:3898] = torch.from_numpy(init_params(42)).to(dev)
            loss = torch.zeros(16, dtype=torch.float64, device=dev)
            run = lambda: ctx.train_device(d_x.data_ptr(), d_y.data_ptr(), n, d_p.data_ptr(), 0.05, 0, 1, B,  # noqa
                                           loss.data_ptr())
            for _ in range(2):
                run()
            ms = timed(stream, run, 5, flush)
            ips = n / (ms / 1e3)
            emit({"config": "batch_sweep", "mode": mode, "threads": thr, "batch": B, "images_per_launch": n, "ms": ms,
                  "images_per_s": ips, "tflops": ips * TRAIN_FLOP / 1e12,
                  "fp32_roofline_frac": ips * TRAIN_FLOP / 1e12 / peak, "loss": float(loss[0])})
            del d_x, d_y
            B *= 2
        # ---- configs[2]: forward-only inference -----------------------------------------------------
        golden_p = np.fromfile(os.path.join(ROOT, "tests", "golden", "final_params.f32"), np.float32)
        golden_pred = np.fromfile(os.path.join(ROOT, "tests", "golden", "test_pred.u8"), np.uint8)
        d_p = torch.zeros(3904, device=dev)
        d_p[:3898] = torch.from_numpy(golden_p).to(dev)
        for N in (100, 1000, 10000, 100000, 1000000):
            d_x = torch.empty(N, 784, device=dev)
            d_y = torch.empty(N, dtype=torch.int32, device=dev)
            ctx.synth_make_set_device(N, 2, d_x.data_ptr(), d_y.data_ptr())
            pred = torch.zeros(N, dtype=torch.int32, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            run = lambda: (cnt.zero_(), ctx.evaluate_device(d_x.data_ptr(), d_y.data_ptr(), N, d_p.data_ptr(),  # noqa
                                                            pred.data_ptr(), cnt.data_ptr()))
            for _ in range(2):
                run()
            ms = timed(stream, run, 5, flush)
            ips = N / (ms / 1e3)
            p = pred[: min(N, 10000)].cpu().numpy()
            exact_pred = bool(np.array_equal(p, golden_pred[: len(p)].astype(np.int32)))
            emit({"config": "inference", "mode": mode, "threads": thr, "images": N, "ms": ms, "images_per_s": ips,
                  "tflops": ips * FWD_FLOP / 1e12, "fp32_roofline_frac": ips * FWD_FLOP / 1e12 / peak,
                  "accuracy": int(cnt.item()) / N, "pred_equal_reference": exact_pred})
            del d_x, d_y
        ctx.close()
    out.close()


if __name__ == "__main__":
    main()
