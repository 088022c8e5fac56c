"""Tiny invocation of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python scripts/sanitize.py [--only train_fast,...]

Each case runs a few images through the C ABI; the sanitizer reports hazards per kernel.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import (init_params, synth_make_set, wide_init_params,  # noqa: E402
                                           wide_make_set)

CASES = ["train_exact", "train_fast_cluster", "train_fast_flat", "train_batched", "train_batched_big", "forward",
         "cells", "eval", "wide_tc", "wide_fp32", "synth"]
ap = argparse.ArgumentParser()
ap.add_argument("--only", default=",".join(CASES))
args = ap.parse_args()
x, y = synth_make_set(24, 1)
p0 = init_params(42)
for case in args.only.split(","):
    if case == "train_exact":
        with Context(0, mode="exact") as c:
            c.train(p0, x[:12], y[:12], epochs=1, batch=6)
    elif case == "train_fast_cluster":
        with Context(0, mode="fast") as c:
            c.train(p0, x[:20], y[:20], epochs=1, batch=10)
    elif case == "train_fast_flat":
        with Context(0, mode="fast") as c:
            c.set_cluster(False)
            c.train(p0, x[:12], y[:12], epochs=1, batch=6)
    elif case == "train_batched":  # batch_train.cu (TLB_BATCH_CFG picks the configuration)
        with Context(0, mode="fast") as c:
            c.set_batched(1)
            c.train(p0, x[:12], y[:12], epochs=1, batch=6)
    elif case == "train_batched_big":  # a full grid: with 2 CTAs per SM the SM-pair work mapping is live
        bx, by = synth_make_set(600, 2)
        with Context(0, mode="fast") as c:
            c.set_batched(1)
            c.train(p0, bx, by, epochs=1, batch=600)
    elif case == "forward":
        with Context(0, mode="exact") as c:
            c.forward(x[:4], p0, acts=True)
    elif case == "cells":
        with Context(0, mode="fast") as c:
            c.forward_backward(x[:4], p0, labels=y[:4])
    elif case == "eval":
        with Context(0, mode="fast") as c:
            c.evaluate(p0, x[:24], y[:24])
    elif case in ("wide_tc", "wide_fp32"):
        wx, wy = wide_make_set(4, 1)
        with Context(0) as c:
            c.wide_train(wide_init_params(42), wx, wy, epochs=1, batch=4, engine=case[5:])
    elif case == "synth":
        with Context(0) as c:
            d = torch.zeros(9 * 784, dtype=torch.uint8, device="cuda:0")
            c.synth_make_digits_device(9, 3, d.data_ptr(), 0)
            torch.cuda.synchronize()
    print("case", case, "ok", flush=True)
