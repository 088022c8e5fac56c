"""GPU parity tests: the sm_100a path (through the C ABI) against the CPU oracle and the reference's
golden vectors.  EXACT mode must be bitwise identical to the reference; FAST mode must stay within the
north-star tolerance (per-element relative 1e-4 on weights and losses, integer argmax exact).

Run on a B200:  python -m pytest tests -m gpu -x -q
"""
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4  # BASELINE.json north_star: per-epoch loss and final weights within 1e-4 relative


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def f2u(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


@pytest.fixture(scope="module")
def ctx():
    from paper_1912_05234_b200 import Context
    c = Context(0, mode="exact")
    yield c
    c.close()


@pytest.fixture(scope="module")
def small(orc):
    x, y = orc.make_set(256, 3)
    return x, y


def rel_err(got, want, floor=0.0):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)) if got.size else 0.0


# ---- scalar math ---------------------------------------------------------------------------------
def test_device_expf_matches_host_libm_exhaustive(ctx, orc):
    """glibc expf restatement on device == host libm expf on every float in [-104, 89] (sigmoid domain)."""
    threads = os.cpu_count() or 1
    ranges = [(0, f2u(89.0)), (0x80000000, f2u(-104.0))]
    chunk = 1 << 27
    total_bad = 0
    for lo, hi in ranges:
        start = lo
        while start <= hi:
            n = min(chunk, hi - start + 1)
            got = ctx.expf_range(start, n)
            first = np.zeros(1, np.uint32)
            import ctypes as C
            bad = orc.L.orc_expf_compare(start, n, got.ctypes.data_as(C.POINTER(C.c_float)), threads,
                                         first.ctypes.data_as(C.POINTER(C.c_uint32)))
            assert bad == 0, f"{bad} mismatches near bits {first[0]:#x}"
            total_bad += bad
            start += n
    assert total_bad == 0


def test_sigmoid_known_values(ctx):
    # test_nn.cpp:140-147: sigma(0) = 0.5 exactly, sigma(2) ~ 0.880797, symmetry
    s = ctx.sigmoid(np.array([0.0, 2.0, -2.0, 100.0, -100.0], np.float32))
    assert s[0] == 0.5
    assert abs(s[1] - 0.880797) < 1e-5
    assert abs(s[1] + s[2] - 1.0) < 1e-6
    assert s[3] == 1.0 and s[4] >= 0.0


# ---- generic nn ops vs the reference's own outputs ------------------------------------------------
def test_nn_ops_bitwise_vs_reference_fixtures(ctx, golden):
    for case in golden["ops"]:
        op = case["op"]
        f = lambda k, sh: np.asarray(case[k], np.float32).reshape(sh)  # noqa: E731
        if op == "conv":
            got = ctx.conv(f("in", case["in_shape"]), f("k", case["k_shape"]))
        elif op == "mconv":
            got = ctx.mconv(f("in", case["in_shape"]), f("k", case["k_shape"]), np.asarray(case["b"], np.float32))
        elif op == "avgpool":
            got = ctx.avgpool(f("in", case["shape"]))
        elif op == "backavgpool":
            got = ctx.backavgpool(f("in", case["shape"]))
        elif op == "backin":
            got = ctx.backin(f("d", case["d_shape"]), f("k", case["k_shape"]), case["in_shape"])
        elif op == "backweights":
            got = ctx.backweights(f("d", case["d_shape"]), f("in", case["in_shape"]))
        elif op == "sigmoid":
            x = f("in", case["shape"])
            got = ctx.sigmoid(x)
            o = np.asarray(case["out"], np.float32).reshape(case["shape"])
            d = f("d", case["shape"])
            assert np.array_equal(bits(ctx.backsigmoid(d, o)).ravel(), bits(case["backsigmoid"]))
            assert ctx.backbias(d) == np.float32(case["backbias"])
        assert np.array_equal(bits(got).ravel(), bits(case["out"])), op


def test_nn_worked_examples(ctx):
    # test_nn.cpp worked examples: avgpool 2x2 mean, backavgpool spread, backin zero-padded correlation
    assert ctx.avgpool(np.array([[1, 2], [3, 4]], np.float32))[0, 0] == 2.5
    np.testing.assert_array_equal(ctx.backavgpool(np.array([[4.0]], np.float32)), np.full((2, 2), 1.0, np.float32))
    d = np.arange(1, 5, dtype=np.float32).reshape(2, 2)
    k = np.array([[1, 2], [3, 4]], np.float32)
    got = ctx.backin(d, k, (3, 3))
    want = np.zeros((3, 3), np.float32)
    for i in range(2):
        for j in range(2):
            want[i:i + 2, j:j + 2] += d[i, j] * k
    np.testing.assert_allclose(got, want, rtol=0, atol=0)


# ---- network: forward / backward cells -------------------------------------------------------------
def test_forward_activations_bitwise(ctx, orc, small):
    x, _ = small
    p = orc.init_params(42)
    yhat, acts = ctx.forward(x[:64], p, acts=True)
    for i in range(64):
        want = orc.forward(x[i], p)
        assert np.array_equal(bits(acts[i]), bits(want)), i
        assert np.array_equal(bits(yhat[i]), bits(want[5280:5290]))


def test_example_cells_bitwise_vs_reference_golden(ctx, golden, zhang_sets):
    (tr_x, tr_y), _ = zhang_sets
    from paper_1912_05234_b200.runtime import init_params
    cells = ctx.forward_backward(tr_x[:8], init_params(42), labels=tr_y[:8])
    assert np.array_equal(bits(cells), bits(golden["cells"]))


def test_example_cells_bitwise_random_params(ctx, orc, small):
    x, y = small
    for seed in (5, 9):
        p = orc.init_params(seed)
        p[150:156] = np.float32(0.3)  # nonzero biases exercise the bias paths
        cells = ctx.forward_backward(x[:96], p, labels=y[:96])
        for i in range(96):
            assert np.array_equal(bits(cells[i]), bits(orc.cell(x[i], p, int(y[i])))), (seed, i)


def test_backward_zero_when_target_equals_output(ctx, orc, small):
    # test_network.cpp:129-144
    x, _ = small
    p = orc.init_params(5)
    yhat = ctx.forward(x[:4], p)
    cells = ctx.forward_backward(x[:4], p, targets=yhat)
    assert np.all(cells[:, :3898] == 0.0)
    assert np.all(cells[:, 3898] == 0.0)


def test_all_zero_params_give_one_half(ctx):
    # test_network.cpp:104-107
    yhat = ctx.forward(np.zeros((2, 784), np.float32), np.zeros(3898, np.float32))
    assert np.all(yhat == 0.5)


def test_sgd_step_arithmetic(ctx):
    # test_network.cpp:180-194
    g = np.zeros(3898, np.float32)
    g[:150] = 2.0
    q = ctx.sgd_step(np.zeros(3898, np.float32), g, 0.5, 4)
    assert np.all(q[:150] == -0.25) and np.all(q[150:] == 0.0)
    from paper_1912_05234_b200 import Error
    with pytest.raises(Error):
        ctx.sgd_step(q, g, 0.5, 0)


# ---- network: training -------------------------------------------------------------------------------
def test_train_argument_errors(ctx, small):
    from paper_1912_05234_b200 import Error
    x, y = small
    p = np.zeros(3898, np.float32)
    with pytest.raises(Error, match="train: empty dataset"):
        ctx.train(p, x[:0], y[:0])
    with pytest.raises(Error, match="negative epoch count"):
        ctx.train(p, x, y, epochs=-1)
    with pytest.raises(Error, match="rate must be > 0"):
        ctx.train(p, x, y, rate=0.0)
    with pytest.raises(Error, match="batches: size must be >= 1, got 0"):
        ctx.train(p, x, y, batch=0)


def test_train_zero_epochs_identity(ctx, orc, small):
    x, y = small
    p0 = orc.init_params(42)
    p, losses = ctx.train(p0, x[:4], y[:4], epochs=0)
    assert np.array_equal(bits(p), bits(p0)) and len(losses) == 0


@pytest.mark.parametrize("n,batch,epochs", [(3, 100, 1), (64, 7, 2), (30, 30, 1), (10, 1, 1), (256, 100, 2),
                                            (201, 50, 1)])
def test_train_exact_bitwise_vs_oracle(ctx, orc, small, n, batch, epochs):
    """Batch > n, ragged last group, batch 1, multi-epoch: bitwise vs the reference restatement."""
    x, y = small
    p0 = orc.init_params(42)
    want_p, want_l = orc.train(x[:n], y[:n], p0, epochs=epochs, batch=batch)
    got_p, got_l = ctx.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
    assert np.array_equal(bits(got_p), bits(want_p))
    assert list(got_l) == list(want_l)


@pytest.mark.parametrize("threads", [256, 512])
def test_train_exact_bitwise_cta_sizes(orc, small, threads):
    """EXACT mode is bitwise at both CTA sizes of the flat kernel (256 = two CTAs per SM, stages looping
    over their lanes), including a group larger than the SM count (the automatic 256-thread choice)."""
    from paper_1912_05234_b200 import Context
    x, y = small
    p0 = orc.init_params(42)
    want_p, want_l = orc.train(x[:256], y[:256], p0, epochs=1, batch=200)
    with Context(0, mode="exact") as c:
        c.set_threads(threads)
        got_p, got_l = c.train(p0, x[:256], y[:256], epochs=1, batch=200)
        yhat = c.forward(x[:8], got_p)
    assert np.array_equal(bits(got_p), bits(want_p)) and list(got_l) == list(want_l)
    for i in range(8):
        assert np.array_equal(bits(yhat[i]), bits(orc.forward(x[i], got_p)[5280:5290]))


def test_train_on_epoch_callback(ctx, orc, small):
    x, y = small
    seen = []
    p, l = ctx.train(orc.init_params(42), x[:10], y[:10], epochs=2, batch=5,
                     on_epoch=lambda e, loss: seen.append((e, loss)))
    assert [e for e, _ in seen] == [1, 2] and [v for _, v in seen] == list(l)


def test_small_protocol_bitwise_vs_reference_golden(ctx, golden, zhang_sets):
    (tr_x, tr_y), _ = zhang_sets
    from paper_1912_05234_b200.runtime import init_params
    p, l = ctx.train(init_params(42), tr_x[:300], tr_y[:300], epochs=2, batch=100)
    assert ["%.17g" % v for v in l] == golden["small_300x2_epoch_loss"]
    import hashlib
    assert hashlib.sha256(p.tobytes()).hexdigest() == golden["small_300x2_params_sha256"]


def test_full_protocol_exact_bitwise(ctx, golden, zhang_sets):
    """BASELINE configs[1] in EXACT mode: the 10-epoch x 10k run is bit-identical to the reference."""
    (tr_x, tr_y), (te_x, te_y) = zhang_sets
    from paper_1912_05234_b200.runtime import init_params
    p, l = ctx.train(init_params(42), tr_x, tr_y, epochs=10, batch=100)
    assert ["%.17g" % v for v in l] == golden["epoch_mean_loss"]
    assert np.array_equal(bits(p), bits(golden["final_params"]))
    acc, pred = ctx.evaluate(p, te_x, te_y, return_pred=True)
    assert acc == golden["test_accuracy"] == 0.4025
    assert np.array_equal(pred, golden["test_pred"])


def test_full_protocol_fast_within_tolerance(golden, zhang_sets):
    """BASELINE configs[1] in FAST mode (FFMA, per-CTA partials): within 1e-4 relative, argmax exact."""
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params
    (tr_x, tr_y), (te_x, te_y) = zhang_sets
    with Context(0, mode="fast") as fctx:
        p, l = fctx.train(init_params(42), tr_x, tr_y, epochs=10, batch=100)
        want_l = np.array([float(v) for v in golden["epoch_mean_loss"]])
        assert rel_err(l, want_l) <= REL_TOL
        w = golden["final_params"]
        assert rel_err(p, w) <= REL_TOL, rel_err(p, w)
        acc, pred = fctx.evaluate(p, te_x, te_y, return_pred=True)
        assert np.array_equal(pred, golden["test_pred"])
        assert acc == 0.4025
        # deterministic run to run
        p2, l2 = fctx.train(init_params(42), tr_x, tr_y, epochs=2, batch=100)
        p3, l3 = fctx.train(init_params(42), tr_x, tr_y, epochs=2, batch=100)
        assert np.array_equal(bits(p2), bits(p3)) and list(l2) == list(l3)


@pytest.mark.parametrize("n,batch,epochs", [(3, 100, 1), (64, 8, 2), (250, 100, 2), (256, 64, 1), (97, 9, 1),
                                            (1040, 1040, 1)])
@pytest.mark.parametrize("cluster", [True, False])
def test_train_fast_vs_oracle(orc, small, zhang_sets, n, batch, epochs, cluster):  # flat: auto CTA size
    """FAST mode, clustered (DSMEM pre-reduction, one grid barrier) and flat kernels: ragged last groups,
    batch > n, group sizes that fill 1..13 clusters partially, and a group larger than the clustered
    kernel's capacity (falls back to the flat kernel).  Within 1e-4 relative of the reference order;
    deterministic run to run."""
    from paper_1912_05234_b200 import Context
    (tr_x, tr_y), _ = zhang_sets
    x, y = (tr_x, tr_y) if n > len(small[1]) else small
    p0 = orc.init_params(42)
    want_p, want_l = orc.train(x[:n], y[:n], p0, epochs=epochs, batch=batch)
    with Context(0, mode="fast") as fctx:
        fctx.set_cluster(cluster)
        got_p, got_l = fctx.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
        again_p, again_l = fctx.train(p0, x[:n], y[:n], epochs=epochs, batch=batch)
    assert rel_err(got_l, want_l) <= REL_TOL
    # floored at |w| = 1e-3 (near-zero weights: absolute 1e-7); the unfloored maximum is reported beside it
    assert rel_err(got_p, want_p, floor=1e-3) <= REL_TOL, (rel_err(got_p, want_p, floor=1e-3), rel_err(got_p, want_p))
    assert np.array_equal(bits(got_p), bits(again_p)) and list(got_l) == list(again_l)


def test_evaluate_golden_params(ctx, golden, zhang_sets):
    _, (te_x, te_y) = zhang_sets
    acc, pred = ctx.evaluate(golden["final_params"], te_x, te_y, return_pred=True)
    assert acc == 0.4025
    assert np.array_equal(pred, golden["test_pred"])


def test_evaluate_ties_and_label_zero(ctx):
    # test_network.cpp:291-294: constant outputs -> argmax 0 -> counts label-0 examples
    acc = ctx.evaluate(np.zeros(3898, np.float32), np.zeros((4, 784), np.float32), np.array([0, 1, 0, 9]))
    assert acc == 0.5


# ---- data-parallel shard path ---------------------------------------------------------------------
def test_dp_shards_sum_to_the_full_group(orc, small):
    """Shard gradient sums (the NCCL allreduce operands) recombine to the full-group sum, which is the
    reference's example-order sum (bitwise in EXACT mode); groups 0 and 1 (shard offsets into the group);
    then the post-allreduce sgd_step equals one reference step."""
    import ctypes as C

    import torch
    from paper_1912_05234_b200 import Context
    x, y = small
    n, batch = 200, 100
    p0 = orc.init_params(42)
    dev = torch.device("cuda:0")
    d_x = torch.from_numpy(x[:n]).to(dev)
    d_y = torch.from_numpy(y[:n]).to(dev)
    for mode in ("exact", "fast"):
        for group, cuts in ((0, [(0, 50), (50, 100)]), (1, [(0, 30), (30, 100)])):
            with Context(0, mode=mode) as c:
                c.set_stream(torch.cuda.current_stream().cuda_stream)
                d_p = torch.zeros(3904, device=dev)
                d_p[:3898] = torch.from_numpy(p0).to(dev)
                gs = []
                for lo, hi in cuts:
                    g = torch.zeros(3904, device=dev)
                    ls = torch.zeros(1, dtype=torch.float64, device=dev)
                    c.train_shard_device(d_x.data_ptr(), d_y.data_ptr(), n, batch, group, lo, hi, d_p.data_ptr(),
                                         g.data_ptr(), ls.data_ptr())
                    gs.append((g, ls))
                full = torch.zeros(3904, device=dev)
                fl = torch.zeros(1, dtype=torch.float64, device=dev)
                c.train_shard_device(d_x.data_ptr(), d_y.data_ptr(), n, batch, group, 0, 100, d_p.data_ptr(),
                                     full.data_ptr(), fl.data_ptr())
                torch.cuda.synchronize()
                s = (gs[0][0] + gs[1][0]).cpu().numpy()[:3898]
                f = full.cpu().numpy()[:3898]
                np.testing.assert_allclose(s, f, rtol=1e-4, atol=1e-6)
                assert abs(float(gs[0][1] + gs[1][1]) - float(fl)) <= 1e-9 * abs(float(fl))
                rows = np.stack([orc.cell(x[group * batch + e], p0, int(y[group * batch + e])) for e in range(batch)])
                acc = np.zeros(3898, np.float32)
                for r in rows:
                    acc = (acc + r[:3898]).astype(np.float32)
                want_l = float(np.sum(rows[:, 3898].astype(np.float64)))
                if mode == "exact":
                    assert np.array_equal(bits(f), bits(acc))
                else:
                    np.testing.assert_allclose(f, acc, rtol=1e-4, atol=1e-6)
                assert abs(float(fl) - want_l) <= 1e-6 * abs(want_l)
                # apply the update and compare with one reference step of that group
                c.apply_sgd_device(d_p.data_ptr(), full.data_ptr(), 0.05, 100)
                torch.cuda.synchronize()
                want_p = p0.copy()
                loss = np.zeros(1)
                orc.L.orc_train_group(x.ctypes.data_as(C.POINTER(C.c_float)), y.ctypes.data_as(C.POINTER(C.c_int32)),
                                      group * batch, 100, want_p.ctypes.data_as(C.POINTER(C.c_float)), 0.05,
                                      loss.ctypes.data_as(C.POINTER(C.c_double)), 4)
                got_p = d_p.cpu().numpy()[:3898]
                if mode == "exact":
                    assert np.array_equal(bits(got_p), bits(want_p))
                else:
                    assert rel_err(got_p, want_p, floor=1e-3) <= REL_TOL


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_overlapped_ingestion_equals_resident_data(orc, zhang_sets, mode):
    """tlb_train streams the dataset in a ramp of whole-group chunks (1, 1, 2, 4, then 4 groups) on a copy stream while the
    kernel trains (device ready flags): for group counts on and around the chunk boundaries, pageable and
    pinned sources, and repeated calls with growing and shrinking sizes, the result equals training on
    device-resident data (tests/_ingest_check.py)."""
    from _ingest_check import check  # tests/ is on sys.path (pytest rootdir insertion)
    (tr_x, tr_y), _ = zhang_sets
    check(orc, tr_x, tr_y, mode)


@pytest.mark.parametrize("policy", ["0", "37", "200", "streams2", "threads1", "threads3", "pageable_first"])
def test_overlapped_ingestion_chunk_policies(policy):
    """The same check under the other chunk policies (TLB_INGEST_CHUNK: 0 = geometric group chunks,
    N = fixed chunks of N images, not group-aligned; 200 = the former 2-group default; streams2 = the ramp
    over two copy streams), the pageable bounce-slot path with 1 and 3 host copy threads (every slot reused
    several times), and the former copies-first policy for pageable sources, both modes, in a fresh process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    extra = {"streams2": {"TLB_INGEST_STREAMS": "2"}, "threads1": {"TLB_INGEST_THREADS": "1"},
             "threads3": {"TLB_INGEST_THREADS": "3", "TLB_INGEST_CHUNK": "150"},
             "pageable_first": {"TLB_PAGEABLE_COPIES_FIRST": "1"}}.get(policy, {"TLB_INGEST_CHUNK": policy})
    env = dict(os.environ, **extra)
    out = subprocess.run([sys.executable, os.path.join(root, "tests", "_ingest_check.py")], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "ingestion ok" in out.stdout


def test_host_registered_dataset_trains_identically(orc, zhang_sets):
    """tlb_host_register on a pageable numpy dataset (what the C++ mirror does for a set it trains twice):
    the call then takes the direct-DMA path and trains the same weights, bit for bit, as the pageable
    bounce path; unregistering restores the pageable path."""
    from paper_1912_05234_b200 import Context
    (tr_x, tr_y), _ = zhang_sets
    x = np.ascontiguousarray(tr_x[:3000])
    y = np.ascontiguousarray(tr_y[:3000], np.int32)
    p0 = orc.init_params(42)
    with Context(0, mode="fast") as c:
        want_p, want_l = c.train(p0, x, y, epochs=2, batch=100)
        c.host_register(x)
        try:
            got_p, got_l = c.train(p0, x, y, epochs=2, batch=100)
        finally:
            c.host_unregister(x)
        again_p, again_l = c.train(p0, x, y, epochs=2, batch=100)
    assert np.array_equal(bits(got_p), bits(want_p)) and list(got_l) == list(want_l)
    assert np.array_equal(bits(again_p), bits(want_p)) and list(again_l) == list(want_l)
