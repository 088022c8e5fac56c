"""Batched train kernel (batch_train.cu) vs the oracle and vs the flat kernel: parity at a few large groups,
then device timings at batch 1k / 16k / 256k (device-generated corpus).  Prints JSON lines.

  python scripts/batch_check.py [--parity] [--time] [--cfg 2x384x2]
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
from paper_1912_05234_b200.runtime import init_params, synth_make_set  # noqa: E402


def rel(got, want, floor=0.0):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)))


def parity():
    from oracle import Oracle
    orc = Oracle()
    x, y = synth_make_set(4100, 1)
    p0 = init_params(42)
    for n, batch, epochs in ((2048, 1024, 2), (4100, 2048, 1), (1500, 700, 1)):
        want_p, want_l = orc.train(x[:n], y[:n], p0, epochs=epochs, batch=batch)
        for mode in ((1,) if os.environ.get("TLB_BT_ONLY") else (1, 0)):
            with Context(0, mode="fast") as c:
                c.set_batched(mode)
                gp, gl = c.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
                gp2, gl2 = c.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
            big = np.abs(want_p) >= 1e-3
            print(json.dumps({"n": n, "batch": batch, "epochs": epochs, "kernel": "batched" if mode else "flat",
                              "params_max_rel": rel(gp, want_p), "params_max_rel_w_ge_1e-3": rel(gp[big], want_p[big]),
                              "params_max_abs_over_max_w": float(np.max(np.abs(gp - want_p)) / np.max(np.abs(want_p))),
                              "loss_max_rel": rel(gl, want_l), "deterministic": bool(np.array_equal(gp, gp2)),
                              "cfg": os.environ.get("TLB_BATCH_CFG", "default")}),
                  flush=True)


def timing(batches):
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for B in batches:
        n = max(2 * B, 32768)
        x = torch.empty(n, 784, device=dev)
        y = torch.empty(n, dtype=torch.int32, device=dev)
        for mode in ((1,) if os.environ.get("TLB_BT_ONLY") else (1, 0)):
            ctx = Context(0, mode="fast")
            ctx.set_stream(st.cuda_stream)
            ctx.set_batched(mode)
            ctx.synth_make_set_device(n, 1, x.data_ptr(), y.data_ptr())
            p = torch.zeros(3904, device=dev)
            p[:3898] = torch.from_numpy(init_params(42)).to(dev)
            loss = torch.zeros(4, dtype=torch.float64, device=dev)
            run = lambda: ctx.train_device(x.data_ptr(), y.data_ptr(), n, p.data_ptr(), 0.05, 0, 1, B,  # noqa
                                           loss.data_ptr())
            run()
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                run()
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[len(ts) // 2]
            print(json.dumps({"what": "train", "kernel": "batched" if mode else "flat", "batch": B, "n": n,
                              "ms": ms, "images_per_s": n / (ms / 1e3), "tflops": n * 1_048_320 / (ms / 1e3) / 1e12,
                              "cfg": os.environ.get("TLB_BATCH_CFG", "default")}), flush=True)
            ctx.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--parity", action="store_true")
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--batches", default="1024,4096,16384,262144")
    args = ap.parse_args()
    if args.parity:
        parity()
    if args.time:
        timing([int(b) for b in args.batches.split(",")])
