"""Byte ingestion (tlb_train_u8 / tlb_train_idx / tlb_idx_parse): the pixel bytes an
MnistSet is made from cross the host link (1/4 of the fp32 volume) and become pixel / 255.0f on the device.

CPU: the IDX header check returns the reference's FormatError messages (proj/src/mnist.cpp:14-61).
GPU: training on the bytes is bit-identical to training on the converted images (EXACT and FAST), from raw
bytes and from encoded IDX files, with the reference's errors for bad labels / geometry / counts."""
import struct

import numpy as np
import pytest


def idx_images(px: np.ndarray, rows=28, cols=28) -> bytes:
    return struct.pack(">IIII", 2051, px.size // (rows * cols), rows, cols) + px.astype(np.uint8).tobytes()


def idx_labels(lab) -> bytes:
    lab = np.asarray(lab, np.uint8)
    return struct.pack(">II", 2049, lab.size) + lab.tobytes()


@pytest.mark.parametrize("data,kind,msg", [
    (b"\x00\x00\x08", "images", "idx: truncated header reading image magic: need 4 bytes, got 3"),
    (struct.pack(">IIII", 2049, 1, 28, 28) + bytes(784), "images", "idx: bad image magic 2049, expected 2051"),
    (struct.pack(">III", 2051, 1, 28), "images", "idx: truncated header reading column count: need 16 bytes, got 12"),
    (struct.pack(">IIII", 2051, 2, 28, 28) + bytes(784), "images",
     "idx: truncated image payload: expected 1584 bytes, got 800"),
    (struct.pack(">IIII", 2051, 1, 28, 28) + bytes(790), "images", "idx: 6 trailing bytes after image payload"),
    (struct.pack(">II", 2051, 1) + b"\x01", "labels", "idx: bad label magic 2051, expected 2049"),
    (struct.pack(">II", 2049, 3) + b"\x01", "labels", "idx: truncated label payload: expected 11 bytes, got 9"),
    (struct.pack(">II", 2049, 1) + b"\x01\x02", "labels", "idx: 1 trailing bytes after label payload"),
])
def test_idx_parse_reference_messages(data, kind, msg):
    from paper_1912_05234_b200.errors import FormatError
    from paper_1912_05234_b200.runtime import idx_parse
    with pytest.raises(FormatError) as ei:
        idx_parse(data, kind)
    assert str(ei.value) == msg


def test_idx_parse_ok():
    from paper_1912_05234_b200.runtime import idx_parse
    assert idx_parse(idx_images(np.zeros(3 * 784)), "images") == (3, 28, 28, 16)
    assert idx_parse(idx_labels([1, 2]), "labels") == (2, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_train_bytes_bitwise_equal_to_train_on_images(mode):
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.runtime import init_params, synth_make_digits
    px, lab = synth_make_digits(1000, 1)
    images = px.astype(np.float32) / np.float32(255.0)  # synth::make_set (synth.cpp:155-161)
    p0 = init_params(42)
    with Context(0, mode=mode) as c:
        want_p, want_l = c.train(p0, images, lab, epochs=2, batch=100)
        got_p, got_l = c.train_u8(p0, px, lab, epochs=2, batch=100)
        idx_p, idx_l = c.train_idx(p0, idx_images(px), idx_labels(lab), epochs=2, batch=100)
        # large groups (batched kernel in fast mode) and a ragged tail
        want_b, _ = c.train(p0, images, lab, epochs=1, batch=640)
        got_b, _ = c.train_u8(p0, px, lab, epochs=1, batch=640)
        # groups > 2 MiB of bytes on the link: fixed ~1 MiB chunks (not group-aligned), resident reference
        px5, lab5 = synth_make_digits(6000, 2)
        im5 = px5.astype(np.float32) / np.float32(255.0)
        want_c, want_cl = c.train(p0, im5, lab5, epochs=2, batch=2900)
        got_c, got_cl = c.train_u8(p0, px5, lab5, epochs=2, batch=2900)
    for got in (got_p, idx_p):
        assert np.array_equal(got.view(np.uint32), want_p.view(np.uint32))
    assert list(got_l) == list(want_l) == list(idx_l)
    assert np.array_equal(got_b.view(np.uint32), want_b.view(np.uint32))
    assert np.array_equal(got_c.view(np.uint32), want_c.view(np.uint32)) and list(got_cl) == list(want_cl)


@pytest.mark.gpu
def test_train_idx_errors():
    from paper_1912_05234_b200 import Context
    from paper_1912_05234_b200.errors import FormatError, ValueError_
    from paper_1912_05234_b200.runtime import init_params
    p0 = init_params(42)
    px = np.zeros(4 * 784, np.uint8)
    with Context(0, mode="fast") as c:
        with pytest.raises(ValueError_, match=r"idx: label 12 at offset 9 out of range 0\.\.9"):
            c.train_idx(p0, idx_images(px), idx_labels([0, 12, 1, 2]), epochs=1, batch=2)
        with pytest.raises(FormatError, match=r"dataset: 4 images but 3 labels"):
            c.train_idx(p0, idx_images(px), idx_labels([0, 1, 2]), epochs=1, batch=2)
        with pytest.raises(FormatError, match=r"expected \[n,28,28\]"):
            c.train_idx(p0, idx_images(np.zeros(4 * 16 * 49), 16, 49), idx_labels([0, 1, 2, 3]), epochs=1, batch=2)
