"""Device-side synthetic corpus (§8(f) rank 2): synth::make_digits / make_set generated on the B200 are
byte-identical to the host generator (itself pinned against the reference's golden hashes) for every
(n, seed), including segment boundaries that fall inside a 312-word state array."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,seed", [(1, 1), (7, 2), (312, 3), (313, 1), (1000, 12345), (10000, 1), (10000, 2),
                                    (20483, 9)])
def test_device_make_digits_equals_host(n, seed):
    import torch
    from paper_1912_05234_b200 import Context, _lib
    from paper_1912_05234_b200.runtime import synth_make_set
    L = _lib.lib()
    want_px = np.zeros(n * 784, np.uint8)
    want_lab = np.zeros(n, np.int32)
    assert L.tlb_synth_make_digits(n, seed, want_px.ctypes.data_as(_lib.u8p), want_lab.ctypes.data_as(_lib.i32p)) == 0
    dev = torch.device("cuda:0")
    px = torch.zeros(n * 784, dtype=torch.uint8, device=dev)
    lab = torch.zeros(n, dtype=torch.int32, device=dev)
    im = torch.zeros(n, 784, dtype=torch.float32, device=dev)
    with Context(0) as c:
        c.set_stream(torch.cuda.current_stream().cuda_stream)
        c.synth_make_digits_device(n, seed, px.data_ptr(), lab.data_ptr())
        c.synth_make_set_device(n, seed, im.data_ptr(), 0)
        torch.cuda.synchronize()
    assert np.array_equal(px.cpu().numpy(), want_px)
    assert np.array_equal(lab.cpu().numpy(), want_lab)
    if n <= 10000:
        x, _ = synth_make_set(n, seed)
        assert np.array_equal(im.cpu().numpy().view(np.uint32), x.view(np.uint32))


def test_device_make_digits_zero_and_reuse():
    import torch
    from paper_1912_05234_b200 import Context
    with Context(0) as c:
        c.synth_make_digits_device(0, 1, 0, 0)  # n = 0 is a no-op
        a = torch.zeros(50 * 784, dtype=torch.uint8, device="cuda:0")
        b = torch.zeros(50 * 784, dtype=torch.uint8, device="cuda:0")
        c.set_stream(torch.cuda.current_stream().cuda_stream)
        c.synth_make_digits_device(50, 4, a.data_ptr(), 0)
        c.synth_make_digits_device(50, 4, b.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
