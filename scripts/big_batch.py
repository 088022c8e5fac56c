"""One large-batch launch family for profiling (configs[2]/[3] kernels): train at batch B over n images, or
evaluate n images; device-generated synthetic corpus.  Prints median ms and img/s.

  python scripts/big_batch.py --what train --batch 16384 --n 32768 [--reps 3]
  python scripts/big_batch.py --what eval --n 1000000
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1912_05234_b200 import Context  # noqa: E402
from paper_1912_05234_b200.runtime import init_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", choices=["train", "eval"], default="train")
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--check", action="store_true", help="eval: trained golden params, predictions of the first "
                                                         "10k images vs the reference's golden predictions")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = Context(0, mode=args.mode)
    ctx.set_stream(st.cuda_stream)
    if args.threads:
        ctx.set_threads(args.threads)
    n = args.n
    x = torch.empty(n, 784, device=dev)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    ctx.synth_make_set_device(n, 1 if args.what == "train" else 2, x.data_ptr(), y.data_ptr())
    p = torch.zeros(3904, device=dev)
    p[:3898] = torch.from_numpy(init_params(42)).to(dev)
    if args.check:
        import numpy as np
        gp = np.fromfile(os.path.join(ROOT, "tests", "golden", "final_params.f32"), np.float32)
        p[:3898] = torch.from_numpy(gp).to(dev)
    loss = torch.zeros(4, dtype=torch.float64, device=dev)
    pred = torch.zeros(n, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    if args.what == "train":
        run = lambda: ctx.train_device(x.data_ptr(), y.data_ptr(), n, p.data_ptr(), 0.05, 0, 1, args.batch,  # noqa
                                       loss.data_ptr())
        flop = 1_048_320
    else:
        run = lambda: ctx.evaluate_device(x.data_ptr(), y.data_ptr(), n, p.data_ptr(), pred.data_ptr(),  # noqa
                                          cnt.data_ptr())
        flop = 407_040
    run()
    ts = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    extra = {}
    if args.check and args.what == "eval":
        import numpy as np
        gpred = np.fromfile(os.path.join(ROOT, "tests", "golden", "test_pred.u8"), np.uint8).astype(np.int32)
        m = min(n, 10000)
        got = pred[:m].cpu().numpy()
        extra = {"pred_equal_reference_first_10k": bool(np.array_equal(got, gpred[:m])),
                 "mismatches": int((got != gpred[:m]).sum()), "correct": int(cnt.item())}
    print(json.dumps({**extra, "what": args.what, "batch": args.batch, "n": n, "mode": args.mode, "ms": ms,
                      "images_per_s": n / ms * 1e3, "tflops": n * flop / ms / 1e9}))


if __name__ == "__main__":
    main()
