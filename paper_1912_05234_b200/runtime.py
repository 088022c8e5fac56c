"""Host-side mirror of the reference API over the C ABI (numpy in, numpy out).

``Context`` owns one ``tlb_ctx`` (device, stream, workspaces).  Method names follow the reference:
``train`` = tloom::net::train (network.cpp:209-251), ``forward`` = net::forward, ``evaluate`` =
net::evaluate, ``conv``/``mconv``/``avgpool``/``backin``/... = tloom::nn (nn.hpp:12-58).
Errors surface as the reference's exception types (errors.py).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import CELL, NACT, NPARAM, PSTRIDE, TLB_MODE_EXACT, TLB_MODE_FAST, f32p, i32p, i64p, u8p
from .errors import raise_for

MODES = {"exact": TLB_MODE_EXACT, "fast": TLB_MODE_FAST}


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a: Optional[np.ndarray]):
    return a.ctypes.data_as(f32p) if a is not None else None


def _ip(a: Optional[np.ndarray]):
    return a.ctypes.data_as(i32p) if a is not None else None


_NO_EPOCH_CB = _lib.EPOCH_CB()  # null callback


def _shape(s) -> np.ndarray:
    return np.ascontiguousarray(list(s), dtype=np.int64)


def _check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, _lib.lib().tlb_last_error().decode())


# ---- argument checks: the C ABI takes raw pointers, so sizes are verified here (the reference's typed
# tensors and Params::validate, network.cpp:42-49, make the same mistakes impossible in C++) ----------
def _check_params(p, who: str) -> None:
    if np.asarray(p).size != NPARAM:
        raise_for(2, f"{who}: params hold {np.asarray(p).size} floats, expected {NPARAM} "
                     "(k1,b1,k2,b2,fc,b in write_flat order)")


def _check_images(images: np.ndarray, n: int, who: str) -> None:
    if images.size != n * 784:
        raise_for(2, f"{who}: images hold {images.size} floats, expected {n} x 784 for {n} labels")


def _images_2d(images, who: str) -> np.ndarray:
    a = _f32(images)
    if a.size % 784:
        raise_for(2, f"{who}: {a.size} image floats is not a whole number of 28x28 images")
    return a.reshape(-1, 784)


# ---- host helpers that need no device ------------------------------------------------------------
def init_params(seed: int) -> np.ndarray:
    """net::init_params (network.cpp:56-79)."""
    p = np.zeros(NPARAM, np.float32)
    _check(_lib.lib().tlb_init_params(seed, _fp(p)))
    return p


def idx_parse(data: bytes, kind: str):
    """IDX header check (mnist.cpp:14-61 messages; no device): kind 'images' -> (count, rows, cols, payload
    offset), 'labels' -> (count, payload offset)."""
    buf = np.frombuffer(data, np.uint8)
    dims = np.zeros(3, np.int64)
    off = C.c_size_t()
    _check(_lib.lib().tlb_idx_parse(buf.ctypes.data if buf.size else None, buf.size, 0 if kind == "images" else 1,
                                    dims.ctypes.data, C.byref(off)))
    return (int(dims[0]), int(dims[1]), int(dims[2]), off.value) if kind == "images" else (int(dims[0]), off.value)


def synth_make_digits(n: int, seed: int):
    """synth::make_digits (synth.cpp:117-153): uint8 pixels [n,784], labels [n]."""
    px = np.zeros((max(n, 1), 784), np.uint8)
    lab = np.zeros(max(n, 1), np.int32)
    _check(_lib.lib().tlb_synth_make_digits(n, seed, px.ctypes.data_as(u8p), _ip(lab)))
    return px[:n], lab[:n]


def synth_make_set(n: int, seed: int):
    """synth::make_set (synth.cpp:155-161): fp32 images [n,784] in [0,1], labels [n]."""
    im = np.zeros((max(n, 1), 784), np.float32)
    lab = np.zeros(max(n, 1), np.int32)
    _check(_lib.lib().tlb_synth_make_set(n, seed, _fp(im), _ip(lab)))
    return im[:n], lab[:n]


def validate_set(images: np.ndarray, labels: np.ndarray) -> None:
    """mnist::make_set invariants (mnist.cpp:126-154)."""
    images, labels = _f32(images), np.ascontiguousarray(labels, np.int32)
    _check(_lib.lib().tlb_validate_set(_fp(images), _ip(labels), len(labels)))


WIDE_NPARAM, WIDE_IMG = 160266, 4096
WIDE_ENGINES = {"fp32": 0, "tc": 1}


def wide_init_params(seed: int = 42) -> np.ndarray:
    """Widened CNN (BASELINE configs[4]) parameters: network.cpp:56-79's rule with the widened fans."""
    p = np.zeros(WIDE_NPARAM, np.float32)
    _check(_lib.lib().tlb_wide_init_params(seed, _fp(p)))
    return p


def wide_make_set(n: int, seed: int):
    """n 64x64 inputs (synth::make_digits glyphs centred on a zero canvas, /255) and labels."""
    im = np.zeros((max(n, 1), WIDE_IMG), np.float32)
    lab = np.zeros(max(n, 1), np.int32)
    _check(_lib.lib().tlb_wide_make_set(n, seed, _fp(im), _ip(lab)))
    return im[:n], lab[:n]


class Context:
    """One device context of the CUDA library (tlb_ctx)."""

    def __init__(self, device: int = 0, mode: str = "exact", devices=None):
        """devices: several local GPUs in one context (tlb_ctx_create_multi) -- train() then splits every SGD
        group over them (EXACT: bit-identical to one device); `device` is ignored when given."""
        self._L = _lib.lib()
        h = C.c_void_p()
        if devices is not None:
            devs = np.ascontiguousarray(list(devices), np.int32)
            _check(self._L.tlb_ctx_create_multi(devs.ctypes.data, len(devs), C.byref(h)))
            device = int(devs[0])
        else:
            _check(self._L.tlb_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self.mode = mode

    def device_count(self) -> int:
        n = C.c_int()
        _check(self._L.tlb_ctx_device_count(self._h, C.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.tlb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- configuration ---------------------------------------------------------------------------
    @property
    def mode(self) -> str:
        m = C.c_int()
        _check(self._L.tlb_ctx_get_mode(self._h, C.byref(m)))
        return "exact" if m.value == TLB_MODE_EXACT else "fast"

    @mode.setter
    def mode(self, name: str) -> None:
        _check(self._L.tlb_ctx_set_mode(self._h, MODES[name]))

    def set_stream(self, cuda_stream_ptr: int) -> None:
        _check(self._L.tlb_ctx_set_stream(self._h, C.c_void_p(cuda_stream_ptr)))

    def set_grid(self, ctas: int) -> None:
        _check(self._L.tlb_ctx_set_grid(self._h, ctas))

    def set_threads(self, threads: int) -> None:
        """CTA size of the flat train / forward kernels: 0 automatic (default), 256 (two CTAs per SM) or 512."""
        _check(self._L.tlb_ctx_set_threads(self._h, threads))

    def set_cluster(self, enable: bool) -> None:
        """Fast mode: clustered train kernel (DSMEM pre-reduction) when the group fits (default on)."""
        _check(self._L.tlb_ctx_set_cluster(self._h, 1 if enable else 0))

    def set_batched(self, mode: int) -> None:
        """Fast mode, large groups: -1 automatic (batched kernel from 4 x SM-count examples per group), 0 the
        one-image-per-CTA flat kernel, 1 the batched kernel (NI images per CTA round) for every such group."""
        _check(self._L.tlb_ctx_set_batched(self._h, int(mode)))

    def set_shard_layout(self, local_stride: int) -> None:
        """Data-parallel entry points (train_shard_device / train_dp_device): 0 = the image/label buffers hold
        the whole dataset; > 0 = only this rank's shards, the shard of group g at example g * local_stride."""
        _check(self._L.tlb_ctx_set_shard_layout(self._h, int(local_stride)))

    def host_register(self, array) -> None:
        """Page-lock a host array (numpy, C-contiguous) so tlb_train / tlb_evaluate DMA straight from it
        (tlb_host_register); the caller keeps the array alive until host_unregister."""
        _check(self._L.tlb_host_register(self._h, array.ctypes.data, array.nbytes))

    def host_unregister(self, array) -> None:
        _check(self._L.tlb_host_unregister(self._h, array.ctypes.data))

    def set_trace(self, d_trace_ptr: int) -> None:
        """Per-stage clock64 stamps of CTA 0 into a device buffer of [steps][16] uint64 (0 disables)."""
        _check(self._L.tlb_ctx_set_trace(self._h, C.c_void_p(d_trace_ptr or None)))

    def info(self) -> dict:
        sm, ot, oe, sb = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        _check(self._L.tlb_ctx_info(self._h, C.byref(sm), C.byref(ot), C.byref(oe), C.byref(sb)))
        return {"sm_count": sm.value, "train_ctas_per_sm": ot.value, "eval_ctas_per_sm": oe.value,
                "smem_bytes_per_cta": sb.value}

    def synchronize(self) -> None:
        _check(self._L.tlb_synchronize(self._h))

    # ---- tloom::net --------------------------------------------------------------------------------
    def train(self, params, images, labels, rate: float = 0.05, epochs: int = 10, batch: int = 100,
              on_epoch: Optional[Callable[[int, float], None]] = None):
        """net::train -> (trained params [3898], epoch mean losses [epochs])."""
        p = np.array(params, np.float32, copy=True).reshape(-1)
        images, labels = _f32(images), np.ascontiguousarray(labels, np.int32).reshape(-1)
        _check_params(p, "train")
        _check_images(images, len(labels), "train")
        losses = np.zeros(max(epochs, 1), np.float64)
        cb = _lib.EPOCH_CB(lambda e, l, _u: on_epoch(e, l)) if on_epoch else _NO_EPOCH_CB
        _check(self._L.tlb_train(self._h, images.ctypes.data, labels.ctypes.data, len(labels), p.ctypes.data, rate,
                                 epochs, batch, losses.ctypes.data, cb, None))
        return p, losses[: max(epochs, 0)]

    def train_u8(self, params, pixels, labels, rate: float = 0.05, epochs: int = 10, batch: int = 100,
                 on_epoch: Optional[Callable[[int, float], None]] = None):
        """net::train on the pixel BYTES the images are made from (IDX payload / synth::make_digits): the
        bytes cross the host link and become pixel / 255.0f on the device -- bit-identical to train() on
        the converted images (tlb_train_u8)."""
        p = np.array(params, np.float32, copy=True).reshape(-1)
        px = np.ascontiguousarray(pixels, np.uint8).reshape(-1)
        labels = np.ascontiguousarray(labels, np.int32).reshape(-1)
        _check_params(p, "train_u8")
        if px.size != len(labels) * 784:
            raise_for(2, f"train_u8: pixels hold {px.size} bytes, expected {len(labels)} x 784")
        losses = np.zeros(max(epochs, 1), np.float64)
        cb = _lib.EPOCH_CB(lambda e, l, _u: on_epoch(e, l)) if on_epoch else _NO_EPOCH_CB
        _check(self._L.tlb_train_u8(self._h, px.ctypes.data, labels.ctypes.data, len(labels), p.ctypes.data, rate,
                                    epochs, batch, losses.ctypes.data, cb, None))
        return p, losses[: max(epochs, 0)]

    def train_idx(self, params, image_file: bytes, label_file: bytes, rate: float = 0.05, epochs: int = 10,
                  batch: int = 100, on_epoch: Optional[Callable[[int, float], None]] = None):
        """net::train straight from the bytes of an IDX image file and an IDX label file (tlb_train_idx)."""
        p = np.array(params, np.float32, copy=True).reshape(-1)
        _check_params(p, "train_idx")
        img = np.frombuffer(image_file, np.uint8)
        lab = np.frombuffer(label_file, np.uint8)
        losses = np.zeros(max(epochs, 1), np.float64)
        cb = _lib.EPOCH_CB(lambda e, l, _u: on_epoch(e, l)) if on_epoch else _NO_EPOCH_CB
        _check(self._L.tlb_train_idx(self._h, img.ctypes.data, img.size, lab.ctypes.data, lab.size, p.ctypes.data,
                                     rate, epochs, batch, losses.ctypes.data, cb, None))
        return p, losses[: max(epochs, 0)]

    def forward(self, images, params, acts: bool = False):
        """net::forward for n images -> yhat [n,10] (and activations [n,5290])."""
        images = _images_2d(images, "forward")
        _check_params(params, "forward")
        n = images.shape[0]
        yhat = np.zeros((max(n, 1), 10), np.float32)
        a = np.zeros((max(n, 1), NACT), np.float32) if acts else None
        _check(self._L.tlb_forward(self._h, _fp(images), n, _fp(_f32(params)), _fp(yhat), _fp(a)))
        return (yhat[:n], a[:n]) if acts else yhat[:n]

    def forward_backward(self, images, params, labels=None, targets=None, acts: bool = False):
        """forward + net::backward + net::loss -> cells [n,3899] (3898 grads + loss)."""
        images = _images_2d(images, "forward_backward")
        _check_params(params, "forward_backward")
        n = images.shape[0]
        if labels is not None and np.asarray(labels).size != n:
            raise_for(2, f"forward_backward: {np.asarray(labels).size} labels for {n} images")
        if targets is not None and np.asarray(targets).size != 10 * n:
            raise_for(2, f"forward_backward: targets hold {np.asarray(targets).size} floats, expected {10 * n}")
        cells = np.zeros((max(n, 1), CELL), np.float32)
        a = np.zeros((max(n, 1), NACT), np.float32) if acts else None
        lab = np.ascontiguousarray(labels, np.int32) if labels is not None else None
        tg = _f32(targets).reshape(-1, 10) if targets is not None else None
        _check(self._L.tlb_forward_backward(self._h, _fp(images), _ip(lab), _fp(tg), n, _fp(_f32(params)),
                                            _fp(cells), _fp(a)))
        return (cells[:n], a[:n]) if acts else cells[:n]

    def evaluate(self, params, images, labels, return_pred: bool = False):
        """net::evaluate -> accuracy (fraction correct); optionally the predictions."""
        images, labels = _images_2d(images, "evaluate"), np.ascontiguousarray(labels, np.int32).reshape(-1)
        _check_params(params, "evaluate")
        n = len(labels)
        _check_images(images, n, "evaluate")
        pred = np.zeros(max(n, 1), np.int32)
        correct = C.c_int64()
        _check(self._L.tlb_evaluate(self._h, _fp(images), _ip(labels), n, _fp(_f32(params)), _ip(pred),
                                    C.byref(correct)))
        acc = correct.value / n
        return (acc, pred[:n]) if return_pred else acc

    def sgd_step(self, params, grads, rate: float, batch: int) -> np.ndarray:
        _check_params(params, "sgd_step")
        _check_params(grads, "sgd_step")
        out = np.zeros(NPARAM, np.float32)
        _check(self._L.tlb_sgd_step(self._h, _fp(_f32(params)), _fp(_f32(grads)), rate, batch, _fp(out)))
        return out

    # ---- device-resident entry points (raw device pointers) ---------------------------------------
    def train_device(self, d_images: int, d_labels: int, n: int, d_params: int, rate: float, epoch_begin: int,
                     epochs: int, batch: int, d_epoch_loss: int) -> None:
        _check(self._L.tlb_train_device(self._h, d_images, d_labels, n, d_params, rate, epoch_begin, epochs,
                                        batch, d_epoch_loss))

    # ---- device synthetic corpus ------------------------------------------------------------------------
    def pixels_to_images_device(self, d_pixels: int, count: int, d_images: int) -> None:
        """d_images[i] = d_pixels[i] / 255.0f on the context stream (the device half of the byte ingestion)."""
        _check(self._L.tlb_pixels_to_images_device(self._h, d_pixels, count, d_images))

    def synth_make_set_device(self, n: int, seed: int, d_images: int, d_labels: int) -> None:
        """synth::make_set(n, seed) generated on the device into [n][784] fp32 / [n] int32 buffers."""
        _check(self._L.tlb_synth_make_set_device(self._h, n, seed, C.c_void_p(d_images or None),
                                                 C.c_void_p(d_labels or None)))

    def synth_make_digits_device(self, n: int, seed: int, d_pixels: int, d_labels: int) -> None:
        """synth::make_digits(n, seed) bytes generated on the device."""
        _check(self._L.tlb_synth_make_digits_device(self._h, n, seed, C.c_void_p(d_pixels or None),
                                                    C.c_void_p(d_labels or None)))

    # ---- widened CNN (BASELINE configs[4]) ------------------------------------------------------------
    def wide_train(self, params, images, labels, rate: float = 0.05, epochs: int = 1, batch: int = 100,
                   engine: str = "tc"):
        p = np.array(params, np.float32, copy=True)
        images, labels = _f32(images), np.ascontiguousarray(labels, np.int32)
        losses = np.zeros(max(epochs, 1), np.float64)
        _check(self._L.tlb_wide_train(self._h, _fp(images), _ip(labels), len(labels), _fp(p), rate, epochs, batch,
                                      losses.ctypes.data_as(_lib.f64p), WIDE_ENGINES[engine]))
        return p, losses[: max(epochs, 0)]

    def wide_train_device(self, d_images: int, d_labels: int, n: int, d_params: int, rate: float, epoch_begin: int,
                          epochs: int, batch: int, d_epoch_loss: int, engine: str = "tc") -> None:
        _check(self._L.tlb_wide_train_device(self._h, d_images, d_labels, n, d_params, rate, epoch_begin, epochs,
                                             batch, d_epoch_loss, WIDE_ENGINES[engine]))

    def wide_forward(self, images, params, engine: str = "tc") -> np.ndarray:
        images = _f32(images).reshape(-1, WIDE_IMG)
        n = images.shape[0]
        yhat = np.zeros((max(n, 1), 10), np.float32)
        _check(self._L.tlb_wide_forward(self._h, _fp(images), n, _fp(_f32(params)), _fp(yhat), WIDE_ENGINES[engine]))
        return yhat[:n]

    def wide_gemm_device(self, which: int, engine: str) -> None:
        _check(self._L.tlb_wide_gemm_device(self._h, which, WIDE_ENGINES[engine]))

    def train_dp_device(self, d_images: int, d_labels: int, n: int, d_params: int, rate: float, epoch_begin: int,
                        epochs: int, batch: int, d_epoch_loss: int, world: int, rank: int, peer_ws: list,
                        seq_base: int, timeout_s: float = 2.0) -> None:
        """Fused data parallelism over NVLink peer memory (tlb_train_dp_device)."""
        arr = (C.c_void_p * len(peer_ws))(*[C.c_void_p(p) for p in peer_ws])
        _check(self._L.tlb_train_dp_device(self._h, d_images, d_labels, n, d_params, rate, epoch_begin, epochs, batch,
                                           d_epoch_loss, world, rank, arr, seq_base, timeout_s))

    def train_shard_device(self, d_images: int, d_labels: int, n: int, batch: int, group: int, shard_lo: int,
                           shard_hi: int, d_params: int, d_grad_sum: int, d_loss_sum: int) -> None:
        _check(self._L.tlb_train_shard_device(self._h, d_images, d_labels, n, batch, group, shard_lo, shard_hi,
                                              d_params, d_grad_sum, d_loss_sum))

    def apply_sgd_device(self, d_params: int, d_grad_sum: int, rate: float, m: int) -> None:
        _check(self._L.tlb_apply_sgd_device(self._h, d_params, d_grad_sum, rate, m))

    def evaluate_device(self, d_images: int, d_labels: int, n: int, d_params: int, d_pred: int,
                        d_correct: int) -> None:
        _check(self._L.tlb_evaluate_device(self._h, d_images, d_labels or None, n, d_params, d_pred or None,
                                           d_correct or None))

    # ---- tloom::nn ---------------------------------------------------------------------------------
    def conv(self, x, k):
        x, k = _f32(x), _f32(k)
        os_ = np.zeros(8, np.int64)
        r = C.c_int()
        xs, ks = _shape(x.shape), _shape(k.shape)
        _check(self._L.tlb_nn_conv_shape(xs.ctypes.data_as(i64p), x.ndim, ks.ctypes.data_as(i64p), k.ndim,
                                         os_.ctypes.data_as(i64p), C.byref(r)))
        out = np.zeros(tuple(os_[: r.value]), np.float32)
        _check(self._L.tlb_nn_conv(self._h, _fp(x), xs.ctypes.data_as(i64p), x.ndim, _fp(k),
                                   ks.ctypes.data_as(i64p), k.ndim, _fp(out)))
        return out

    def mconv(self, x, k, b):
        x, k, b = _f32(x), _f32(k), _f32(b)
        os_ = np.zeros(8, np.int64)
        r = C.c_int()
        xs, ks, bs = _shape(x.shape), _shape(k.shape), _shape(b.shape)
        _check(self._L.tlb_nn_mconv_shape(xs.ctypes.data_as(i64p), x.ndim, ks.ctypes.data_as(i64p), k.ndim,
                                          bs.ctypes.data_as(i64p), b.ndim, os_.ctypes.data_as(i64p), C.byref(r)))
        out = np.zeros(tuple(os_[: r.value]), np.float32)
        _check(self._L.tlb_nn_mconv(self._h, _fp(x), xs.ctypes.data_as(i64p), x.ndim, _fp(k),
                                    ks.ctypes.data_as(i64p), k.ndim, _fp(b), bs.ctypes.data_as(i64p), b.ndim,
                                    _fp(out)))
        return out

    def sigmoid(self, x):
        x = _f32(x)
        out = np.zeros_like(x)
        _check(self._L.tlb_nn_sigmoid(self._h, _fp(x), x.size, _fp(out)))
        return out

    def backsigmoid(self, d, o):
        d, o = _f32(d), _f32(o)
        if d.shape != o.shape:
            raise_for(2, f"map_binary: shapes {list(d.shape)} and {list(o.shape)} differ")
        out = np.zeros_like(d)
        _check(self._L.tlb_nn_backsigmoid(self._h, _fp(d), _fp(o), d.size, _fp(out)))
        return out

    def avgpool(self, x):
        x = _f32(x)
        os_ = np.zeros(8, np.int64)
        r = C.c_int()
        xs = _shape(x.shape)
        _check(self._L.tlb_nn_avgpool_shape(xs.ctypes.data_as(i64p), x.ndim, os_.ctypes.data_as(i64p), C.byref(r)))
        out = np.zeros(tuple(os_[: r.value]), np.float32)
        _check(self._L.tlb_nn_avgpool(self._h, _fp(x), xs.ctypes.data_as(i64p), x.ndim, _fp(out)))
        return out

    def backavgpool(self, d):
        d = _f32(d)
        os_ = np.zeros(8, np.int64)
        r = C.c_int()
        ds = _shape(d.shape)
        _check(self._L.tlb_nn_backavgpool_shape(ds.ctypes.data_as(i64p), d.ndim, os_.ctypes.data_as(i64p),
                                                C.byref(r)))
        out = np.zeros(tuple(os_[: r.value]), np.float32)
        _check(self._L.tlb_nn_backavgpool(self._h, _fp(d), ds.ctypes.data_as(i64p), d.ndim, _fp(out)))
        return out

    def backweights(self, d, x):
        """nn::backweights(d_out, in) = conv(in, d_out) (nn.cpp:160)."""
        return self.conv(x, d)

    def backbias(self, d) -> float:
        d = _f32(d)
        out = np.zeros(1, np.float32)
        _check(self._L.tlb_nn_backbias(self._h, _fp(d), d.size, _fp(out)))
        return float(out[0])

    def backin(self, d, k, in_shape):
        d, k = _f32(d), _f32(k)
        ds, ks, is_ = _shape(d.shape), _shape(k.shape), _shape(in_shape)
        os_ = np.zeros(8, np.int64)
        r = C.c_int()
        _check(self._L.tlb_nn_backin_shape(ds.ctypes.data_as(i64p), d.ndim, ks.ctypes.data_as(i64p), k.ndim,
                                           is_.ctypes.data_as(i64p), len(is_), os_.ctypes.data_as(i64p), C.byref(r)))
        out = np.zeros(tuple(os_[: r.value]), np.float32)
        _check(self._L.tlb_nn_backin(self._h, _fp(d), ds.ctypes.data_as(i64p), d.ndim, _fp(k),
                                     ks.ctypes.data_as(i64p), k.ndim, is_.ctypes.data_as(i64p), len(is_), _fp(out)))
        return out

    def expf_range(self, start_bits: int, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.float32)
        _check(self._L.tlb_expf_range(self._h, start_bits, n, _fp(out)))
        return out[:n]


__all__ = ["Context", "init_params", "synth_make_set", "synth_make_digits", "validate_set", "NPARAM", "PSTRIDE",
           "NACT", "CELL"]
