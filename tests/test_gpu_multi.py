"""In-process multi-GPU training (tlb_ctx_create_multi): every SGD group split over the
context's devices with static_chunk (runtime.cpp:138-145), the gradient reduced over all devices at every
step through peer memory.  The reference is bit-identical for any worker count; EXACT mode here is
bit-identical for any device count.  On a one-GPU box the same device is listed several times (the
kernels share it) -- the cross-device protocol (shard layout, peer rows, the grid barrier over every
device's CTAs, the update of every parameter copy) is the same.

Run on a B200:  python -m pytest tests/test_gpu_multi.py -m gpu -q
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def small(orc):
    return orc.make_set(256, 3)


@pytest.mark.parametrize("ndev", [2, 3, 4])
def test_exact_multi_device_bitwise_equals_single_device_and_reference(golden, zhang_sets, ndev):
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params
    (tr_x, tr_y), _ = zhang_sets
    p0 = init_params(42)
    with Context(mode="exact", devices=[0] * ndev) as c:
        assert c.device_count() == ndev
        p, l = c.train(p0, tr_x[:300], tr_y[:300], epochs=2, batch=100)
    assert ["%.17g" % v for v in l] == golden["small_300x2_epoch_loss"]
    import hashlib
    assert hashlib.sha256(p.tobytes()).hexdigest() == golden["small_300x2_params_sha256"]


@pytest.mark.parametrize("n,batch,epochs", [(250, 100, 2), (97, 9, 1), (64, 64, 1), (10, 3, 2)])
def test_exact_multi_device_ragged_groups(orc, small, n, batch, epochs):
    """Ragged last groups, groups smaller than the device count, shards of unequal size."""
    from paper_1912_05234_b200 import Context
    x, y = small
    p0 = orc.init_params(42)
    want_p, want_l = orc.train(x[:n], y[:n], p0, epochs=epochs, batch=batch)
    with Context(mode="exact", devices=[0, 0, 0]) as c:
        got_p, got_l = c.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
        seen = []
        cb_p, cb_l = c.train(p0, x[:n], y[:n], epochs=epochs, batch=batch, on_epoch=lambda e, v: seen.append((e, v)))
    assert np.array_equal(bits(got_p), bits(want_p)) and list(got_l) == list(want_l)
    assert np.array_equal(bits(cb_p), bits(want_p)) and [v for _, v in seen] == list(want_l)


def test_fast_multi_device_within_tolerance_and_deterministic(orc, zhang_sets):
    from paper_1912_05234_b200 import Context
    (tr_x, tr_y), _ = zhang_sets
    x, y = tr_x[:2000], tr_y[:2000]
    p0 = orc.init_params(42)
    want_p, want_l = orc.train(x, y, p0, epochs=2, batch=200)
    with Context(mode="fast", devices=[0, 0]) as c:
        p1, l1 = c.train(p0, x, y, epochs=2, batch=200)
        p2, l2 = c.train(p0, x, y, epochs=2, batch=200)
    d = np.abs(p1.astype(np.float64) - want_p)
    assert np.all(d <= 1e-4 * np.maximum(np.abs(want_p), 1e-3))
    assert np.max(np.abs(l1 - want_l) / want_l) <= 1e-4
    assert np.array_equal(bits(p1), bits(p2)) and list(l1) == list(l2)


def test_multi_device_bytes_path(zhang_sets):
    """Byte ingestion through a multi-device context: bit-identical to the fp32 images (EXACT)."""
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params, synth_make_digits
    px, lab = synth_make_digits(500, 1)
    images = px.astype(np.float32) / np.float32(255.0)
    p0 = init_params(42)
    with Context(mode="exact", devices=[0, 0]) as c:
        a_p, a_l = c.train(p0, images, lab, epochs=1, batch=100)
        b_p, b_l = c.train_u8(p0, px, lab, epochs=1, batch=100)
    with Context(0, mode="exact") as c1:
        s_p, s_l = c1.train(p0, images, lab, epochs=1, batch=100)
    assert np.array_equal(bits(a_p), bits(s_p)) and np.array_equal(bits(b_p), bits(s_p))
    assert list(a_l) == list(s_l) == list(b_l)
