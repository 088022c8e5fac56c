"""Generate the golden parity fixtures from the UNMODIFIED reference library.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

It loads oracle/_ref/libtloom_ref.so (the reference's own sources compiled in place by
oracle/Makefile) and records, for the paper protocol of BASELINE.json configs[0]:

* protocol.json  -- init_params(42) / synth hashes, the 10 epoch mean losses (%.17g), final-param and
                    prediction hashes, test accuracy;
* final_params.f32 -- the 3,898 trained fp32 weights (order k1,b1,k2,b2,fc,b = network.cpp:186-193);
* test_pred.u8     -- the reference's argmax predictions for the 10k test images;
* cells.f32        -- per-example train cells (3,898 grads + loss) of the first 8 training examples at
                      init_params(42) (network.cpp:228-234);
* ops.json         -- small random instances of the generic nn ops (conv, mconv, avgpool, backavgpool,
                      backin, backweights, sigmoid, backsigmoid, backbias) with the reference outputs.

Nothing on the GPU box reads /root/reference: the tests consume only these committed files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference, fp, lp  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ops_fixture(R: Reference, rng: np.random.Generator) -> list:
    out = []

    def rnd(shape):
        return rng.uniform(-1, 1, size=shape).astype(np.float32)

    def rshape(rmin, rmax, emin, emax):
        r = int(rng.integers(rmin, rmax + 1))
        return [int(rng.integers(emin, emax + 1)) for _ in range(r)]

    for _ in range(24):
        ins = rshape(1, 4, 1, 6)
        ks = [int(rng.integers(1, e + 1)) for e in ins]
        x, k = rnd(ins), rnd(ks)
        os_ = [a - b + 1 for a, b in zip(ins, ks)]
        o = np.zeros(int(np.prod(os_)), np.float32)
        R.L.ref_conv(fp(x), lp(np.array(ins, np.int64)), len(ins), fp(k), lp(np.array(ks, np.int64)),
                     len(ks), fp(o))
        out.append({"op": "conv", "in_shape": ins, "k_shape": ks, "in": x.ravel().tolist(),
                    "k": k.ravel().tolist(), "out": o.tolist()})
    for _ in range(16):
        ins = rshape(1, 3, 1, 6)
        cell = [int(rng.integers(1, e + 1)) for e in ins]
        nk = int(rng.integers(1, 5))
        ks = [nk] + cell
        x, k, b = rnd(ins), rnd(ks), rnd([nk])
        os_ = [nk] + [a - c + 1 for a, c in zip(ins, cell)]
        o = np.zeros(int(np.prod(os_)), np.float32)
        R.L.ref_mconv(fp(x), lp(np.array(ins, np.int64)), len(ins), fp(k), lp(np.array(ks, np.int64)),
                      len(ks), fp(b), lp(np.array([nk], np.int64)), 1, fp(o))
        out.append({"op": "mconv", "in_shape": ins, "k_shape": ks, "in": x.ravel().tolist(),
                    "k": k.ravel().tolist(), "b": b.tolist(), "out": o.tolist()})
    for _ in range(16):
        s = rshape(2, 4, 1, 3)
        s[-2] *= 2
        s[-1] *= 2
        x = rnd(s)
        o = np.zeros(x.size // 4, np.float32)
        R.L.ref_avgpool(fp(x), lp(np.array(s, np.int64)), len(s), fp(o))
        out.append({"op": "avgpool", "shape": s, "in": x.ravel().tolist(), "out": o.tolist()})
    for _ in range(16):
        s = rshape(2, 4, 1, 3)
        d = rnd(s)
        o = np.zeros(d.size * 4, np.float32)
        R.L.ref_backavgpool(fp(d), lp(np.array(s, np.int64)), len(s), fp(o))
        out.append({"op": "backavgpool", "shape": s, "in": d.ravel().tolist(), "out": o.tolist()})
    for _ in range(24):
        ins = rshape(1, 4, 1, 6)
        ks = [int(rng.integers(1, e + 1)) for e in ins]
        ds = [a - b + 1 for a, b in zip(ins, ks)]
        d, k = rnd(ds), rnd(ks)
        o = np.zeros(int(np.prod(ins)), np.float32)
        R.L.ref_backin(fp(d), lp(np.array(ds, np.int64)), fp(k), lp(np.array(ks, np.int64)),
                       lp(np.array(ins, np.int64)), len(ins), fp(o))
        out.append({"op": "backin", "d_shape": ds, "k_shape": ks, "in_shape": ins,
                    "d": d.ravel().tolist(), "k": k.ravel().tolist(), "out": o.tolist()})
    for _ in range(12):
        ins = rshape(1, 4, 1, 6)
        ks = [int(rng.integers(1, e + 1)) for e in ins]
        ds = [a - b + 1 for a, b in zip(ins, ks)]
        d, x = rnd(ds), rnd(ins)
        o = np.zeros(int(np.prod(ks)), np.float32)
        R.L.ref_backweights(fp(d), lp(np.array(ds, np.int64)), fp(x), lp(np.array(ins, np.int64)),
                            len(ins), fp(o))
        out.append({"op": "backweights", "d_shape": ds, "in_shape": ins, "d": d.ravel().tolist(),
                    "in": x.ravel().tolist(), "out": o.tolist()})
    for _ in range(8):
        s = rshape(1, 3, 1, 7)
        x = (rnd(s) * 30).astype(np.float32)
        o = np.zeros(x.size, np.float32)
        R.L.ref_sigmoid(fp(x), lp(np.array(s, np.int64)), len(s), fp(o))
        d = rnd(s)
        ob = np.zeros(x.size, np.float32)
        R.L.ref_backsigmoid(fp(d), fp(o), lp(np.array(s, np.int64)), len(s), fp(ob))
        bb = R.L.ref_backbias(fp(d), lp(np.array(s, np.int64)), len(s))
        out.append({"op": "sigmoid", "shape": s, "in": x.ravel().tolist(), "out": o.tolist(),
                    "d": d.ravel().tolist(), "backsigmoid": ob.tolist(), "backbias": float(bb)})
    return out


def main() -> None:
    R = Reference()
    R.set_workers(os.cpu_count() or 1)  # bitwise identical for any worker count (network.cpp:236-243)
    rec: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj @ oracle/_ref"}

    p0 = R.init_params(42)
    rec["init_params_42_sha256"] = sha(p0)
    rec["init_params_42_head"] = [float(v) for v in p0[:4]]
    tr_x, tr_y = R.make_set(10000, 1)
    te_x, te_y = R.make_set(10000, 2)
    px, _ = R.make_digits(10000, 1)
    rec["synth_10000_1_pixels_sha256"] = sha(px)
    rec["synth_10000_1_images_sha256"] = sha(tr_x)
    rec["synth_10000_2_images_sha256"] = sha(te_x)
    rec["synth_10000_1_labels_sha256"] = sha(tr_y)

    cells = np.stack([R.cell(tr_x[i], p0, np.eye(10, dtype=np.float32)[tr_y[i]]) for i in range(8)])
    cells.astype(np.float32).tofile(os.path.join(HERE, "cells.f32"))

    t0 = time.time()
    p, losses = R.train(tr_x, tr_y, p0, rate=0.05, epochs=10, batch=100)
    rec["train_seconds_here"] = time.time() - t0
    rec["epoch_mean_loss"] = ["%.17g" % v for v in losses]
    rec["final_params_sha256"] = sha(p)
    p.astype(np.float32).tofile(os.path.join(HERE, "final_params.f32"))
    acc, pred = R.evaluate(p, te_x, te_y)
    rec["test_accuracy"] = acc
    rec["test_pred_sha256"] = sha(pred.astype(np.uint8))
    pred.astype(np.uint8).tofile(os.path.join(HERE, "test_pred.u8"))

    # A3-style small protocol used by the fast CPU tests: 1 epoch of 300 images at batch 100.
    p_small, l_small = R.train(tr_x[:300], tr_y[:300], p0, rate=0.05, epochs=2, batch=100)
    rec["small_300x2_epoch_loss"] = ["%.17g" % v for v in l_small]
    rec["small_300x2_params_sha256"] = sha(p_small)

    with open(os.path.join(HERE, "protocol.json"), "w") as f:
        json.dump(rec, f, indent=1)
    with open(os.path.join(HERE, "ops.json"), "w") as f:
        json.dump(ops_fixture(R, np.random.default_rng(1912)), f)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
