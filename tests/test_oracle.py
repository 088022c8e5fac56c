"""CPU tests: the C restatement (oracle/) pinned against the reference's golden vectors.

The golden fixtures were produced by the UNMODIFIED reference (tests/golden/make_golden.py).  When the
reference build (oracle/_ref) is present, the oracle is also compared with it directly.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import REF_SO, fp, lp


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_init_params_matches_reference(orc, golden):
    p = orc.init_params(42)
    assert sha(p) == golden["init_params_42_sha256"]
    assert [float(v) for v in p[:4]] == golden["init_params_42_head"]
    # Glorot bounds and zero biases (test_network.cpp:61-81)
    assert np.all(np.abs(p[:150]) <= np.sqrt(np.float32(6.0) / np.float32(601.0)))
    assert np.all(p[150:156] == 0) and np.all(p[1956:1968] == 0) and np.all(p[3888:] == 0)
    assert not np.array_equal(p, orc.init_params(43))


def test_synth_corpus_matches_reference(orc, golden, zhang_sets):
    (tr_x, tr_y), (te_x, _) = zhang_sets
    px, _ = orc.make_digits(10000, 1)
    assert sha(px) == golden["synth_10000_1_pixels_sha256"]
    assert sha(tr_x) == golden["synth_10000_1_images_sha256"]
    assert sha(te_x) == golden["synth_10000_2_images_sha256"]
    assert sha(tr_y) == golden["synth_10000_1_labels_sha256"]
    assert list(tr_y[:12]) == [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 0, 1]


def test_example_cells_match_reference(orc, golden, zhang_sets):
    (tr_x, tr_y), _ = zhang_sets
    p = orc.init_params(42)
    for i in range(8):
        c = orc.cell(tr_x[i], p, int(tr_y[i]))
        assert np.array_equal(c.view(np.uint32), golden["cells"][i].view(np.uint32)), i


def test_small_protocol_bitwise(orc, golden, zhang_sets):
    (tr_x, tr_y), _ = zhang_sets
    p, losses = orc.train(tr_x[:300], tr_y[:300], orc.init_params(42), epochs=2, batch=100)
    assert ["%.17g" % v for v in losses] == golden["small_300x2_epoch_loss"]
    assert sha(p) == golden["small_300x2_params_sha256"]


@pytest.mark.slow
def test_full_protocol_bitwise(orc, golden, zhang_sets):
    """BASELINE configs[0]: 10 epochs x 10k, batch 100, lr 0.05 -- bitwise vs the reference."""
    (tr_x, tr_y), (te_x, te_y) = zhang_sets
    p, losses = orc.train(tr_x, tr_y, orc.init_params(42), epochs=10, batch=100)
    assert ["%.17g" % v for v in losses] == golden["epoch_mean_loss"]
    assert np.array_equal(p.view(np.uint32), golden["final_params"].view(np.uint32))
    correct, pred = orc.evaluate(p, te_x, te_y)
    assert correct / 10000 == golden["test_accuracy"] == 0.4025
    assert np.array_equal(pred, golden["test_pred"])


def test_generic_ops_match_reference_fixtures(orc, golden):
    L = orc.L
    for case in golden["ops"]:
        op = case["op"]
        f32 = lambda k: np.asarray(case[k], np.float32)  # noqa: E731
        i64 = lambda k: np.asarray(case[k], np.int64)  # noqa: E731
        want = f32("out") if "out" in case else None
        if op == "conv":
            out = np.zeros_like(want)
            L.orc_conv(fp(f32("in")), lp(i64("in_shape")), len(case["in_shape"]), fp(f32("k")),
                       lp(i64("k_shape")), fp(out))
        elif op == "mconv":
            out = np.zeros_like(want)
            L.orc_mconv(fp(f32("in")), lp(i64("in_shape")), len(case["in_shape"]), fp(f32("k")),
                        lp(i64("k_shape")), fp(f32("b")), fp(out))
        elif op == "avgpool":
            out = np.zeros_like(want)
            L.orc_avgpool(fp(f32("in")), lp(i64("shape")), len(case["shape"]), fp(out))
        elif op == "backavgpool":
            out = np.zeros_like(want)
            L.orc_backavgpool(fp(f32("in")), lp(i64("shape")), len(case["shape"]), fp(out))
        elif op == "backin":
            out = np.zeros_like(want)
            L.orc_backin(fp(f32("d")), lp(i64("d_shape")), fp(f32("k")), lp(i64("k_shape")),
                         len(case["d_shape"]), fp(out))
        elif op == "backweights":  # backweights(d, in) = conv(in, d) (nn.cpp:160)
            out = np.zeros_like(want)
            L.orc_conv(fp(f32("in")), lp(i64("in_shape")), len(case["in_shape"]), fp(f32("d")),
                       lp(i64("d_shape")), fp(out))
        elif op == "sigmoid":
            x = f32("in")
            out = np.array([L.orc_sigmoid(float(v)) for v in x], np.float32)
            d = f32("d")
            bs = (d * want) * (np.float32(1) - want)
            assert np.array_equal(bs, f32("backsigmoid"))
            assert L.orc_sum_all(fp(d), d.size) == np.float32(case["backbias"])
        else:
            raise AssertionError(op)
        assert np.array_equal(out.view(np.uint32), want.view(np.uint32)), op


def test_expf_port_matches_host_libm_sampled(orc):
    """glibc 2.39 expf restatement vs host libm on a dense sample of the sigmoid domain."""
    bad = orc.L.orc_expf_port_mismatches(0x3F000000, 0x3F400000, os.cpu_count() or 1)  # [0.5, 0.75]
    assert bad == 0
    bad = orc.L.orc_expf_port_mismatches(0xC2000000, 0xC2100000, os.cpu_count() or 1)  # [-32,-36)
    assert bad == 0
    for x in [0.0, -0.0, 1.0, -1.0, 88.7, 88.8, -103.9, -104.0, float("inf"), float("-inf")]:
        a, b = orc.L.orc_expf_port(x), orc.L.orc_expf(x)
        assert a == b or (a != a and b != b)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build (oracle/_ref) absent")
def test_oracle_vs_reference_library_direct(orc):
    from oracle import Reference
    R = Reference()
    x, y = orc.make_set(64, 5)
    assert np.array_equal(x, R.make_set(64, 5)[0])
    p = orc.init_params(9)
    for i in range(16):
        a = orc.forward(x[i], p)
        b = R.forward(x[i], p)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    p1, l1 = orc.train(x, y, p, epochs=2, batch=7)
    p2, l2 = R.train(x, y, p, epochs=2, batch=7)
    assert np.array_equal(p1.view(np.uint32), p2.view(np.uint32))
    assert list(l1) == list(l2)
