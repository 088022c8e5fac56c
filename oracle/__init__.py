"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``Oracle``    -- oracle/_build/libtloom_oracle.so, the C restatement of the reference's hot path
                   (oracle/tloom_oracle.c).  Always available once ``make -C oracle`` ran.
* ``Reference`` -- oracle/_ref/libtloom_ref.so, the UNMODIFIED reference library
                   (/root/reference/proj/src/*.cpp compiled in place by oracle/Makefile) behind a
                   small extern "C" shim (oracle/ref_shim.cpp).  Built only where /root/reference
                   exists; the built .so travels to the GPU box with the repo snapshot.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference legs may import
this package, and only as the checker -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libtloom_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtloom_ref.so")
REF_SRC = "/root/reference/proj"

NPARAM = 3898
NACT = 5290

_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; the reference only when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def fp(a):
    return a.ctypes.data_as(_f32p)


def ip(a):
    return a.ctypes.data_as(_i32p)


def lp(a):
    return a.ctypes.data_as(_i64p)


class Oracle:
    """C restatement (oracle/tloom_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_init_params.argtypes = [C.c_uint64, _f32p]
        L.orc_make_digits.argtypes = [C.c_int64, C.c_uint64, _u8p, _i32p]
        L.orc_make_set.argtypes = [C.c_int64, C.c_uint64, _f32p, _i32p]
        L.orc_expf.argtypes = [C.c_float]
        L.orc_expf.restype = C.c_float
        L.orc_expf_port.argtypes = [C.c_float]
        L.orc_expf_port.restype = C.c_float
        L.orc_sigmoid.argtypes = [C.c_float]
        L.orc_sigmoid.restype = C.c_float
        L.orc_expf_port_mismatches.argtypes = [C.c_uint32, C.c_uint32, C.c_int]
        L.orc_expf_port_mismatches.restype = C.c_int64
        L.orc_expf_compare.argtypes = [C.c_uint32, C.c_int64, _f32p, C.c_int, C.POINTER(C.c_uint32)]
        L.orc_expf_compare.restype = C.c_int64
        L.orc_forward.argtypes = [_f32p, _f32p, _f32p]
        L.orc_loss.argtypes = [_f32p, _f32p]
        L.orc_loss.restype = C.c_float
        L.orc_backward.argtypes = [_f32p, _f32p, _f32p, _f32p, _f32p]
        L.orc_example_cell.argtypes = [_f32p, _f32p, C.c_int32, _f32p]
        L.orc_train.argtypes = [_f32p, _i32p, C.c_int64, _f32p, C.c_float, C.c_int, C.c_int64, _f64p, C.c_int]
        L.orc_train.restype = C.c_int
        L.orc_train_group.argtypes = [_f32p, _i32p, C.c_int64, C.c_int64, _f32p, C.c_float, _f64p, C.c_int]
        L.orc_predict.argtypes = [_f32p]
        L.orc_predict.restype = C.c_int
        L.orc_evaluate.argtypes = [_f32p, _f32p, _i32p, C.c_int64, _i32p, C.c_int]
        L.orc_evaluate.restype = C.c_int64
        L.orc_conv.argtypes = [_f32p, _i64p, C.c_int, _f32p, _i64p, _f32p]
        L.orc_mconv.argtypes = [_f32p, _i64p, C.c_int, _f32p, _i64p, _f32p, _f32p]
        L.orc_avgpool.argtypes = [_f32p, _i64p, C.c_int, _f32p]
        L.orc_backavgpool.argtypes = [_f32p, _i64p, C.c_int, _f32p]
        L.orc_backin.argtypes = [_f32p, _i64p, _f32p, _i64p, C.c_int, _f32p]
        L.orc_sum_all.argtypes = [_f32p, C.c_int64]
        L.orc_sum_all.restype = C.c_float

    def init_params(self, seed: int) -> np.ndarray:
        p = np.zeros(NPARAM, np.float32)
        self.L.orc_init_params(seed, fp(p))
        return p

    def make_digits(self, n: int, seed: int):
        px = np.zeros(max(n, 1) * 784, np.uint8)
        lab = np.zeros(max(n, 1), np.int32)
        self.L.orc_make_digits(n, seed, px.ctypes.data_as(_u8p), ip(lab))
        return px[: n * 784].reshape(n, 784), lab[:n]

    def make_set(self, n: int, seed: int):
        im = np.zeros((max(n, 1), 784), np.float32)
        lab = np.zeros(max(n, 1), np.int32)
        self.L.orc_make_set(n, seed, fp(im), ip(lab))
        return im[:n], lab[:n]

    def forward(self, image, params) -> np.ndarray:
        act = np.zeros(NACT, np.float32)
        self.L.orc_forward(fp(np.ascontiguousarray(image, np.float32)), fp(params), fp(act))
        return act

    def cell(self, image, params, label: int) -> np.ndarray:
        c = np.zeros(NPARAM + 1, np.float32)
        self.L.orc_example_cell(fp(np.ascontiguousarray(image, np.float32)), fp(params), label, fp(c))
        return c

    def backward(self, image, act, params, y) -> np.ndarray:
        g = np.zeros(NPARAM, np.float32)
        self.L.orc_backward(fp(image), fp(act), fp(params), fp(np.asarray(y, np.float32)), fp(g))
        return g

    def train(self, images, labels, params, rate=0.05, epochs=10, batch=100, threads=None):
        p = np.array(params, np.float32, copy=True)
        losses = np.zeros(max(epochs, 1), np.float64)
        threads = threads or os.cpu_count() or 1
        rc = self.L.orc_train(fp(images), ip(labels), len(labels), fp(p), rate, epochs, batch,
                              losses.ctypes.data_as(_f64p), threads)
        if rc != 0:
            raise ValueError(f"orc_train rc={rc}")
        return p, losses[:epochs]

    def evaluate(self, params, images, labels, threads=None):
        pred = np.zeros(max(len(labels), 1), np.int32)
        c = self.L.orc_evaluate(fp(params), fp(images), ip(labels), len(labels), ip(pred),
                                threads or os.cpu_count() or 1)
        return c, pred[: len(labels)]


class Reference:
    """The unmodified reference library behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_SRC):
                build()
            if not os.path.exists(path):
                raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_workers.argtypes = [C.c_int]
        L.ref_init_params.argtypes = [C.c_uint64, _f32p]
        L.ref_save_params.argtypes = [C.c_char_p, _f32p]
        L.ref_load_params.argtypes = [C.c_char_p, _f32p]
        L.ref_load_set.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_load_set.restype = C.c_int64
        L.ref_make_digits.argtypes = [C.c_int64, C.c_uint64, _u8p, _i32p]
        L.ref_make_set.argtypes = [C.c_int64, C.c_uint64, _f32p, _i32p]
        L.ref_forward.argtypes = [_f32p, _f32p, _f32p]
        L.ref_forward_backward.argtypes = [_f32p, _f32p, _f32p, _f32p]
        L.ref_train.argtypes = [_f32p, _i32p, C.c_int64, _f32p, C.c_float, C.c_int, C.c_int64, _f64p]
        L.ref_evaluate.argtypes = [_f32p, _f32p, _i32p, C.c_int64, _i32p, _f64p]
        L.ref_conv.argtypes = [_f32p, _i64p, C.c_int, _f32p, _i64p, C.c_int, _f32p]
        L.ref_mconv.argtypes = [_f32p, _i64p, C.c_int, _f32p, _i64p, C.c_int, _f32p, _i64p, C.c_int, _f32p]
        L.ref_sigmoid.argtypes = [_f32p, _i64p, C.c_int, _f32p]
        L.ref_avgpool.argtypes = [_f32p, _i64p, C.c_int, _f32p]
        L.ref_backavgpool.argtypes = [_f32p, _i64p, C.c_int, _f32p]
        L.ref_backin.argtypes = [_f32p, _i64p, _f32p, _i64p, _i64p, C.c_int, _f32p]
        L.ref_backweights.argtypes = [_f32p, _i64p, _f32p, _i64p, C.c_int, _f32p]
        L.ref_backsigmoid.argtypes = [_f32p, _f32p, _i64p, C.c_int, _f32p]
        L.ref_backbias.argtypes = [_f32p, _i64p, C.c_int]
        L.ref_backbias.restype = C.c_float

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def set_workers(self, w: int):
        self._check(self.L.ref_set_workers(w))

    def save_params(self, path: str, params) -> None:
        self._check(self.L.ref_save_params(path.encode(), fp(np.ascontiguousarray(params, np.float32))))

    def load_params(self, path: str) -> np.ndarray:
        p = np.zeros(NPARAM, np.float32)
        self._check(self.L.ref_load_params(path.encode(), fp(p)))
        return p

    def load_set(self, images_path: str, labels_path: str, limit: int = -1):
        n = self.L.ref_load_set(images_path.encode(), labels_path.encode(), limit, None, None)
        if n < 0:
            self._check(-n)
        x = np.zeros((max(n, 1), 784), np.float32)
        y = np.zeros(max(n, 1), np.int32)
        self.L.ref_load_set(images_path.encode(), labels_path.encode(), limit, x.ctypes.data, y.ctypes.data)
        return x[:n], y[:n]

    def init_params(self, seed: int) -> np.ndarray:
        p = np.zeros(NPARAM, np.float32)
        self.L.ref_init_params(seed, fp(p))
        return p

    def make_digits(self, n: int, seed: int):
        px = np.zeros(max(n, 1) * 784, np.uint8)
        lab = np.zeros(max(n, 1), np.int32)
        self.L.ref_make_digits(n, seed, px.ctypes.data_as(_u8p), ip(lab))
        return px[: n * 784].reshape(n, 784), lab[:n]

    def make_set(self, n: int, seed: int):
        im = np.zeros((max(n, 1), 784), np.float32)
        lab = np.zeros(max(n, 1), np.int32)
        self.L.ref_make_set(n, seed, fp(im), ip(lab))
        return im[:n], lab[:n]

    def forward(self, image, params) -> np.ndarray:
        act = np.zeros(NACT, np.float32)
        self._check(self.L.ref_forward(fp(np.ascontiguousarray(image, np.float32)), fp(params), fp(act)))
        return act

    def cell(self, image, params, y) -> np.ndarray:
        c = np.zeros(NPARAM + 1, np.float32)
        self._check(self.L.ref_forward_backward(fp(np.ascontiguousarray(image, np.float32)), fp(params),
                                                fp(np.asarray(y, np.float32)), fp(c)))
        return c

    def train(self, images, labels, params, rate=0.05, epochs=10, batch=100):
        p = np.array(params, np.float32, copy=True)
        losses = np.zeros(max(epochs, 1), np.float64)
        self._check(self.L.ref_train(fp(images), ip(labels), len(labels), fp(p), rate, epochs, batch,
                                     losses.ctypes.data_as(_f64p)))
        return p, losses[:epochs]

    def evaluate(self, params, images, labels):
        pred = np.zeros(max(len(labels), 1), np.int32)
        acc = C.c_double()
        self._check(self.L.ref_evaluate(fp(params), fp(images), ip(labels), len(labels), ip(pred),
                                        C.byref(acc)))
        return acc.value, pred[: len(labels)]
