"""Host restatement of the batched train kernel's round mapping (paper_1912_05234_b200/csrc/batch_train.cu:
work_chunk, pair_slot, seek_round / step_round) and its invariant: for every group size, grid, images per
round and SM-pair share, the CTAs' rounds cover each example of the group exactly once -- contiguous chunks
and interleaved rounds alike, with and without the SM-pair split.  (The GPU tests check the kernel's results
against the oracle; this pins the index arithmetic over many more shapes than a GPU run can.)"""
import itertools

import pytest


def static_chunk(n, workers, w):
    """runtime.cpp:138-145 ceil-block split (tlb_common.cuh static_chunk)."""
    if n <= workers:
        lo = min(w, n)
        return lo, min(w + 1, n) if w < n else n
    block = (n + workers - 1) // workers
    lo = min(w * block, n)
    return lo, min(lo + block, n)


def f32_mul_trunc(share, length):
    import numpy as np
    return int(np.float32(share) * np.float32(length))


def work_chunk(m, grid, wid, paired, share, ni):
    if not paired:
        return static_chunk(m, grid, wid)
    plo, phi = static_chunk(m, grid // 2, wid >> 1)
    length = phi - plo
    s0 = f32_mul_trunc(share, length)
    s0 = min(length, (s0 + ni // 2) // ni * ni)
    return (plo + s0, phi) if wid & 1 else (plo, plo + s0)


def pair_slot(j, q):
    return 0 if ((j + 1) * q >> 10) != (j * q >> 10) else 1


def rounds_of(m, grid, wid, paired, share, ni, ilv):
    """The (first example, count) of every round CTA `wid` trains, in its order."""
    out = []
    if not ilv:
        lo, hi = work_chunk(m, grid, wid, paired, share, ni)
        e = lo
        while e < hi:
            out.append((e, min(ni, hi - e)))
            e += ni
        return out
    big_r = (m + ni - 1) // ni
    q = int(round(share * 1024))
    if not paired:
        j = 0
        while wid + j * grid < big_r:
            r = wid + j * grid
            out.append((r * ni, min(ni, m - r * ni)))
            j += 1
        return out
    pairs, p, sl = grid >> 1, wid >> 1, wid & 1
    j = 0
    while p + j * pairs < big_r:
        if pair_slot(j, q) == sl:
            r = p + j * pairs
            out.append((r * ni, min(ni, m - r * ni)))
        j += 1
    return out


CASES = list(itertools.product(
    [1, 7, 100, 591, 592, 700, 1024, 2048, 2367, 2368, 4099, 16384, 65537],  # group sizes
    [(4, 148, False), (2, 296, True), (2, 296, False), (4, 150, False), (2, 8, True)],  # (NI, grid, paired)
    [0.5, 0.54, 0.62],
    [False, True]))


@pytest.mark.parametrize("m,cfg,share,ilv", CASES)
def test_every_example_exactly_once(m, cfg, share, ilv):
    ni, grid, paired = cfg
    seen = [0] * m
    for wid in range(grid):
        for e, cnt in rounds_of(m, grid, wid, paired, share, ni, ilv):
            assert 0 < cnt <= ni
            for x in range(e, e + cnt):
                seen[x] += 1
    assert seen == [1] * m


def test_pair_slot_share():
    """Slot 0 takes floor((j + 1) share) - floor(j share) of the positions: ~share of them, spread evenly."""
    q = int(round(0.54 * 1024))
    slots = [pair_slot(j, q) for j in range(1000)]
    assert abs(slots.count(0) / 1000 - 0.54) < 0.002
    run = max(len(list(g)) for k, g in itertools.groupby(slots) if k == 1)
    assert run <= 2  # never three slot-1 positions in a row at 54%
