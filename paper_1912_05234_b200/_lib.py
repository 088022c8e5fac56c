"""ctypes binding of libtloom_b200.so (the C ABI in include/tloom_b200.h).

The product path is the CUDA library; there is no CPU fallback.  Loading fails loudly if the
in-tree library is missing (build it with ``python -m paper_1912_05234_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
# TLB_LIB: developer A/B builds (paper_1912_05234_b200.build.build_variant); default = the in-tree library
LIB_PATH = os.environ.get("TLB_LIB") or os.path.join(PKG, "lib", "libtloom_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "tloom_b200.h")

TLB_OK = 0
TLB_ERR_ERROR, TLB_ERR_SHAPE, TLB_ERR_BOUNDS, TLB_ERR_FORMAT, TLB_ERR_VALUE = 1, 2, 3, 4, 5
TLB_ERR_CUDA, TLB_ERR_NCCL, TLB_ERR_ARG = 10, 11, 12
TLB_MODE_EXACT, TLB_MODE_FAST = 0, 1
NPARAM, PSTRIDE, NACT, CELL = 3898, 3904, 5290, 3899

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_ulonglong)
vp = C.c_void_p
EPOCH_CB = C.CFUNCTYPE(None, C.c_int, C.c_double, C.c_void_p)

_SIGS = {
    "tlb_last_error": (C.c_char_p, []),
    "tlb_version": (C.c_char_p, []),
    "tlb_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "tlb_ctx_create_multi": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
    "tlb_ctx_device_count": (C.c_int, [vp, vp]),
    "tlb_ctx_destroy": (C.c_int, [vp]),
    "tlb_ctx_set_stream": (C.c_int, [vp, vp]),
    "tlb_ctx_set_mode": (C.c_int, [vp, C.c_int]),
    "tlb_ctx_get_mode": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "tlb_ctx_set_grid": (C.c_int, [vp, C.c_int]),
    "tlb_ctx_set_trace": (C.c_int, [vp, vp]),
    "tlb_ctx_set_cluster": (C.c_int, [vp, C.c_int]),
    "tlb_ctx_set_batched": (C.c_int, [vp, C.c_int]),
    "tlb_ctx_set_shard_layout": (C.c_int, [vp, C.c_int64]),
    "tlb_ctx_set_threads": (C.c_int, [vp, C.c_int]),
    "tlb_dp_workspace_bytes": (C.c_size_t, []),
    "tlb_train_dp_device": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_float, C.c_int32, C.c_int32, C.c_int64, vp,
                                      C.c_int, C.c_int, C.POINTER(vp), C.c_uint64, C.c_double]),
    "tlb_synth_make_digits_device": (C.c_int, [vp, C.c_int64, C.c_uint64, vp, vp]),
    "tlb_synth_make_set_device": (C.c_int, [vp, C.c_int64, C.c_uint64, vp, vp]),
    "tlb_wide_init_params": (C.c_int, [C.c_uint64, f32p]),
    "tlb_wide_make_set": (C.c_int, [C.c_int64, C.c_uint64, f32p, i32p]),
    "tlb_wide_train": (C.c_int, [vp, f32p, i32p, C.c_int64, f32p, C.c_float, C.c_int32, C.c_int64, f64p, C.c_int]),
    "tlb_wide_train_device": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_float, C.c_int32, C.c_int32, C.c_int64, vp,
                                        C.c_int]),
    "tlb_wide_forward": (C.c_int, [vp, f32p, C.c_int64, f32p, f32p, C.c_int]),
    "tlb_wide_gemm_device": (C.c_int, [vp, C.c_int, C.c_int]),
    "tlb_ctx_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), i64p]),
    "tlb_synchronize": (C.c_int, [vp]),
    "tlb_init_params": (C.c_int, [C.c_uint64, f32p]),
    "tlb_synth_make_digits": (C.c_int, [C.c_int64, C.c_uint64, u8p, i32p]),
    "tlb_synth_make_set": (C.c_int, [C.c_int64, C.c_uint64, f32p, i32p]),
    "tlb_validate_set": (C.c_int, [f32p, i32p, C.c_int64]),
    # raw addresses (c_void_p) on the e2e path: ~4 us per ctypes pointer conversion avoided per call
    "tlb_host_register": (C.c_int, [vp, vp, C.c_size_t]),
    "tlb_host_unregister": (C.c_int, [vp, vp]),
    "tlb_train": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_float, C.c_int32, C.c_int64, vp, EPOCH_CB, vp]),
    "tlb_train_u8": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_float, C.c_int32, C.c_int64, vp, EPOCH_CB, vp]),
    "tlb_train_idx": (C.c_int, [vp, vp, C.c_size_t, vp, C.c_size_t, vp, C.c_float, C.c_int32, C.c_int64, vp,
                                EPOCH_CB, vp]),
    "tlb_idx_parse": (C.c_int, [vp, C.c_size_t, C.c_int, vp, vp]),
    "tlb_pixels_to_images_device": (C.c_int, [vp, vp, C.c_int64, vp]),
    "tlb_forward": (C.c_int, [vp, f32p, C.c_int64, f32p, f32p, f32p]),
    "tlb_forward_backward": (C.c_int, [vp, f32p, i32p, f32p, C.c_int64, f32p, f32p, f32p]),
    "tlb_backward": (C.c_int, [vp, f32p, f32p, f32p, C.c_int64, f32p, f32p]),
    "tlb_loss": (C.c_int, [vp, f32p, f32p, C.c_int64, f32p]),
    "tlb_evaluate": (C.c_int, [vp, f32p, i32p, C.c_int64, f32p, i32p, i64p]),
    "tlb_sgd_step": (C.c_int, [vp, f32p, f32p, C.c_float, C.c_int64, f32p]),
    "tlb_train_device": (C.c_int, [vp, vp, vp, C.c_int64, vp, C.c_float, C.c_int32, C.c_int32, C.c_int64, vp]),
    "tlb_train_shard_device": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                         vp, vp, vp]),
    "tlb_apply_sgd_device": (C.c_int, [vp, vp, vp, C.c_float, C.c_int64]),
    "tlb_evaluate_device": (C.c_int, [vp, vp, vp, C.c_int64, vp, vp, vp]),
    "tlb_nn_conv": (C.c_int, [vp, f32p, i64p, C.c_int, f32p, i64p, C.c_int, f32p]),
    "tlb_nn_mconv": (C.c_int, [vp, f32p, i64p, C.c_int, f32p, i64p, C.c_int, f32p, i64p, C.c_int, f32p]),
    "tlb_nn_sigmoid": (C.c_int, [vp, f32p, C.c_int64, f32p]),
    "tlb_nn_backsigmoid": (C.c_int, [vp, f32p, f32p, C.c_int64, f32p]),
    "tlb_nn_avgpool": (C.c_int, [vp, f32p, i64p, C.c_int, f32p]),
    "tlb_nn_backavgpool": (C.c_int, [vp, f32p, i64p, C.c_int, f32p]),
    "tlb_nn_backweights": (C.c_int, [vp, f32p, i64p, C.c_int, f32p, i64p, C.c_int, f32p]),
    "tlb_nn_backbias": (C.c_int, [vp, f32p, C.c_int64, f32p]),
    "tlb_nn_backin": (C.c_int, [vp, f32p, i64p, C.c_int, f32p, i64p, C.c_int, i64p, C.c_int, f32p]),
    "tlb_nn_conv_shape": (C.c_int, [i64p, C.c_int, i64p, C.c_int, i64p, C.POINTER(C.c_int)]),
    "tlb_nn_mconv_shape": (C.c_int, [i64p, C.c_int, i64p, C.c_int, i64p, C.c_int, i64p, C.POINTER(C.c_int)]),
    "tlb_nn_avgpool_shape": (C.c_int, [i64p, C.c_int, i64p, C.POINTER(C.c_int)]),
    "tlb_nn_backavgpool_shape": (C.c_int, [i64p, C.c_int, i64p, C.POINTER(C.c_int)]),
    "tlb_nn_backin_shape": (C.c_int, [i64p, C.c_int, i64p, C.c_int, i64p, C.c_int, i64p, C.POINTER(C.c_int)]),
    "tlb_expf_range": (C.c_int, [vp, C.c_uint32, C.c_int64, f32p]),
}


def declared_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|size_t)\s+(tlb_\w+)\s*\(", text, re.M)))


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA library was not built "
                              "(python -m paper_1912_05234_b200.build); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB
