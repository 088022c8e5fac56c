"""CPU model of the clustered kernel's packed accumulator words (zhang_kernels.cu, kPackBias): each
cluster adds llrint(sum * 2^32) + 2^51 to a never-zeroed u64 word; a reader that remembers the word's
value at its last read decodes the number K of contributions since then and their exact integer sum S
from the difference modulo 2^64.  This checks the arithmetic the kernel relies on -- including wrap-around
of the word after many steps and partial arrivals (K < ncl keeps the reader polling)."""
import numpy as np

MASK = (1 << 64) - 1
BIAS = 1 << 51
FIX = float(1 << 32)


def encode(x: float) -> int:
    return (int(np.rint(x * FIX)) + BIAS) & MASK


def decode(v: int, prev: int):
    diff = (v - prev) & MASK
    k = ((diff + (1 << 50)) & MASK) >> 51
    s = diff - k * BIAS
    if s >= 1 << 63:
        s -= 1 << 64
    return k, s


def test_packed_words_decode_counts_and_sums_across_wraparound():
    rng = np.random.default_rng(7)
    ncl = 13
    word, prev = 0, 0
    for step in range(5000):  # ~5000 x 13 x 2^51 wraps the 64-bit word several thousand times
        sums = rng.uniform(-2.0e3, 2.0e3, ncl) * rng.choice([1e-6, 1e-2, 1.0], ncl)
        order = rng.permutation(ncl)
        want = 0
        for n, q in enumerate(order):
            word = (word + encode(sums[q])) & MASK
            want += int(np.rint(sums[q] * FIX))
            k, s = decode(word, prev)
            assert k == n + 1  # partial arrivals are seen as partial: the reader keeps polling
            if k == ncl:
                assert s == want
        prev = word


def test_packed_word_bounds():
    # the decode needs |S| < 2^50: a step's gradient sum |g| < 2^18 (kernel comment) in 2^-32 units,
    # and the count field must not overflow 64 bits for up to 13 clusters x 8 GPUs of contributions
    assert int(np.rint(0.999 * 2.0 ** 18 * FIX)) < 1 << 50
    assert 104 * BIAS < 1 << 64
    k, s = decode((13 * BIAS - int(0.999 * 2.0 ** 50)) & MASK, 0)  # most negative representable sum
    assert k == 13 and s == -int(0.999 * 2.0 ** 50)
