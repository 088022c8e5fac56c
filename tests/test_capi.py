"""CPU tests of the boundary: the C-ABI library loads, exports every declared entry point, and its
host-side pieces (init_params, synth corpus, shape functions, argument errors) match the reference.
No kernel is launched here (no GPU in this container)."""
import ctypes as C
import hashlib
import os
import subprocess

import numpy as np
import pytest

from paper_1912_05234_b200 import _lib, errors, runtime


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 38
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # and nothing the binding declares is absent from the header
    assert set(_lib._SIGS) <= set(declared)


def test_library_is_sm100a_cuda():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_init_params_matches_reference_golden(golden):
    p = runtime.init_params(42)
    assert sha(p) == golden["init_params_42_sha256"]


def test_synth_matches_reference_golden(golden):
    px, lab = runtime.synth_make_digits(10000, 1)
    assert sha(px) == golden["synth_10000_1_pixels_sha256"]
    im, lab2 = runtime.synth_make_set(10000, 1)
    assert sha(im) == golden["synth_10000_1_images_sha256"]
    assert sha(lab2) == golden["synth_10000_1_labels_sha256"]


def test_validate_set_errors():
    im, lab = runtime.synth_make_set(4, 3)
    runtime.validate_set(im, lab)
    bad = lab.copy()
    bad[2] = 10
    with pytest.raises(errors.ValueError_, match="label 10 at index 2 out of range 0..9"):
        runtime.validate_set(im, bad)
    imb = im.copy()
    imb[1, 5] = 1.5
    with pytest.raises(errors.ValueError_, match="out of range \\[0,1\\]"):
        runtime.validate_set(imb, lab)


def _shape_call(fn, *shapes):
    L = _lib.lib()
    out = np.zeros(8, np.int64)
    r = C.c_int()
    args = []
    for s in shapes:
        a = np.asarray(s, np.int64)
        args += [a.ctypes.data_as(_lib.i64p), len(s)]
    rc = getattr(L, fn)(*args, out.ctypes.data_as(_lib.i64p), C.byref(r))
    return rc, list(out[: r.value]), L.tlb_last_error().decode()


def test_shape_functions_match_reference_messages():
    # conv_result_shape (nn.cpp:37-49)
    assert _shape_call("tlb_nn_conv_shape", [5, 5], [3, 3])[:2] == (0, [3, 3])
    rc, _, msg = _shape_call("tlb_nn_conv_shape", [5, 5], [3, 3, 1])
    assert rc == _lib.TLB_ERR_SHAPE and msg == "conv: input rank 2 and kernel rank 3 differ"
    rc, _, msg = _shape_call("tlb_nn_conv_shape", [5, 2], [3, 3])
    assert msg == "conv: kernel shape [3,3] exceeds input shape [5,2] on axis 1"
    # mconv_result_shape (nn.cpp:51-60): the Zhang layers
    assert _shape_call("tlb_nn_mconv_shape", [28, 28], [6, 5, 5], [6])[:2] == (0, [6, 24, 24])
    assert _shape_call("tlb_nn_mconv_shape", [6, 12, 12], [12, 6, 5, 5], [12])[:2] == (0, [12, 1, 8, 8])
    assert _shape_call("tlb_nn_mconv_shape", [12, 1, 4, 4], [10, 12, 1, 4, 4], [10])[:2] == (0, [10, 1, 1, 1, 1])
    assert _shape_call("tlb_nn_mconv_shape", [28, 28], [6, 5, 5], [7])[2] == "mconv: 6 kernels but 7 biases"
    assert _shape_call("tlb_nn_mconv_shape", [28, 28], [6, 5], [6])[2] == \
        "mconv: kernel stack rank 2 must be input rank + 1 = 3"
    assert _shape_call("tlb_nn_mconv_shape", [28, 28], [6, 5, 5], [6, 1])[2] == "mconv: bias shape [6,1] is not rank 1"
    # avgpool / backavgpool / backin shapes
    assert _shape_call("tlb_nn_avgpool_shape", [6, 24, 24])[:2] == (0, [6, 12, 12])
    assert _shape_call("tlb_nn_avgpool_shape", [5, 4, 3])[2] == "avgpool: axis 2 extent 3 is not even"
    assert _shape_call("tlb_nn_avgpool_shape", [4])[2] == "avgpool: rank 1 input, need rank >= 2"
    assert _shape_call("tlb_nn_backavgpool_shape", [12, 1, 4, 4])[:2] == (0, [12, 1, 8, 8])
    assert _shape_call("tlb_nn_backin_shape", [1, 8, 8], [6, 5, 5], [6, 12, 12])[:2] == (0, [6, 12, 12])
    assert _shape_call("tlb_nn_backin_shape", [1, 8, 7], [6, 5, 5], [6, 12, 12])[2] == \
        "backin: error shape [1,8,7] does not match shape(in) - shape(k) + 1 = [1,8,8]"


def test_context_requires_a_b200_and_fails_loudly():
    if os.environ.get("CUDA_VISIBLE_DEVICES", None) == "" or not _has_gpu():
        with pytest.raises(errors.Error):
            runtime.Context(0)


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
