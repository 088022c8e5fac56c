"""CPU tests of the multi-GPU host logic (paper_1912_05234_b200.parallel) with world_size 2 over gloo.

The per-rank compute is the CPU oracle here (test infrastructure); on the B200 the same
``train_epoch`` drives tlb_train_shard_device + NCCL allreduce + tlb_apply_sgd_device (bench.py N>1).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_05234_b200.parallel import groups, static_chunk, train_epoch


class OracleBackend:
    def __init__(self, orc, images, labels, batch, params):
        self.orc, self.x, self.y, self.batch, self.p = orc, images, labels, batch, params

    def shard_grad(self, group, lo, hi, grad, loss):
        start = group * self.batch
        acc = np.zeros(3898, np.float32)
        l = 0.0
        for i in range(start + lo, start + hi):
            c = self.orc.cell(self.x[i], self.p, int(self.y[i]))
            acc = (acc + c[:3898]).astype(np.float32)
            l += float(c[3898])
        grad.zero_()
        grad[:3898] = torch.from_numpy(acc)
        loss[0] = l

    def apply(self, grad, rate, m):
        g = grad[:3898].numpy()
        self.p[:] = self.p - np.float32(rate) * (g / np.float32(m))


def test_static_chunk_matches_reference():
    # test_runtime.cpp:31-42
    assert [static_chunk(10, 4, w) for w in range(4)] == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert static_chunk(3, 8, 7) == (3, 3)
    rng = np.random.default_rng(0)
    for _ in range(200):  # exactly-once ownership (test_runtime.cpp:44-56)
        n, w = int(rng.integers(0, 300)), int(rng.integers(1, 65))
        seen = []
        for r in range(w):
            lo, hi = static_chunk(n, w, r)
            seen += list(range(lo, hi))
        assert seen == list(range(n))
    with pytest.raises(ValueError):
        static_chunk(5, 0, 0)


def test_groups_match_mnist_batches():
    assert groups(10, 4) == [(0, 4), (4, 4), (8, 2)]
    assert groups(3, 100) == [(0, 3)]
    with pytest.raises(ValueError, match="batches: size must be >= 1, got 0"):
        groups(5, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, batch, epochs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    orc = Oracle()
    x, y = orc.make_set(n, 4)
    p = orc.init_params(42)
    be = OracleBackend(orc, x, y, batch, p)
    grad = torch.zeros(3904)
    loss = torch.zeros(1, dtype=torch.float64)
    losses = []
    for _ in range(epochs):
        acc = torch.zeros(1, dtype=torch.float64)
        train_epoch(be, n, batch, 0.05, grad, loss, acc, world, rank,
                    lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)
        losses.append(float(acc) / n)
    q.put((rank, p.copy(), losses))
    dist.destroy_process_group()


def _run(world, n, batch, epochs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, batch, epochs, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_dp_world2_gloo_matches_single_process(orc):
    n, batch, epochs = 60, 20, 2
    res = _run(2, n, batch, epochs)
    # every rank applies the identical update -> bitwise identical replicas
    assert np.array_equal(res[0][1].view(np.uint32), res[1][1].view(np.uint32))
    assert res[0][2] == res[1][2]
    x, y = orc.make_set(n, 4)
    want_p, want_l = orc.train(x, y, orc.init_params(42), epochs=epochs, batch=batch)
    got = res[0][1]
    np.testing.assert_allclose(res[0][2], want_l, rtol=1e-6)
    assert np.max(np.abs(got - want_p) / np.maximum(np.abs(want_p), 1e-3)) <= 1e-4


def test_dp_world1_is_bitwise_reference(orc):
    n, batch = 30, 10
    (rank, p, l), = _run(1, n, batch, 1)
    x, y = orc.make_set(n, 4)
    want_p, want_l = orc.train(x, y, orc.init_params(42), epochs=1, batch=batch)
    assert np.array_equal(p.view(np.uint32), want_p.view(np.uint32))
    assert abs(l[0] - want_l[0]) <= 1e-15
