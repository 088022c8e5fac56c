"""TEST INFRASTRUCTURE ONLY -- the widened CNN of BASELINE.json configs[4] composed from the UNMODIFIED
reference library's shape-polymorphic ``tloom::nn`` operators (oracle/_ref/libtloom_ref.so through
oracle/ref_shim.cpp).  ``net::*`` hardcodes the Zhang shapes (network.cpp:17-23), so the widened network
is the same composition with other extents:

    c1 = sigmoid(mconv(I[64,64], k1[32,5,5], b1[32]))      -> [32,60,60]   (network.cpp:89)
    s1 = avgpool(c1)                                       -> [32,30,30]   (network.cpp:90)
    c2 = sigmoid(mconv(s1, k2[64,32,5,5], b2[64]))         -> [64,1,26,26] (network.cpp:91)
    s2 = avgpool(c2)                                       -> [64,1,13,13] (network.cpp:92)
    out = sigmoid(mconv(s2, fc[10,64,1,13,13], b[10]))     -> [10,1,1,1,1] (network.cpp:93)

backward = mconv_layer_backward per layer (network.cpp:116-141, 145-169): d_z = backsigmoid(d_act, act);
grad_k[i] = backweights(d_z[i], in); grad_b[i] = backbias(d_z[i]); d_in = sum_i backin(d_z[i], k[i], in)
accumulated in kernel order; batch reduction in example order and sgd_step as network.cpp:171-180,
236-244.  Parameter init: network.cpp:56-79's Glorot rule and mt19937_64 stream with the widened fans
(k1: 25/3600, k2: 800/676, fc: 10816/1).  Inputs: synth::make_digits (28x28 bytes) centred on a 64x64
zero canvas, /255.

Slow by design (the reference's generic comprehension path, ~0.2 s per image): tests use a few images.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

K1 = (32, 5, 5)
B1 = (32,)
K2 = (64, 32, 5, 5)
B2 = (64,)
FC = (10, 64, 1, 13, 13)
BF = (10,)
SHAPES = (K1, B1, K2, B2, FC, BF)
SIZES = tuple(int(np.prod(s)) for s in SHAPES)
NPARAM = sum(SIZES)  # 160,266
IMG = 64
FANS = {0: (25, 60 * 60), 2: (32 * 25, 26 * 26), 4: (64 * 13 * 13, 1)}


def init_params(seed: int) -> np.ndarray:
    """network.cpp:56-79 with the widened fans: mt19937_64(seed), u = (rng()>>40)*2^-24,
    (2u-1)*limit, limit = sqrtf(6/(fan_in+fan_out)); fill order k1, k2, fc; biases zero."""
    rng = _MT64(seed)
    out = []
    for idx, n in enumerate(SIZES):
        if idx in FANS:
            fi, fo = FANS[idx]
            limit = np.float32(np.sqrt(np.float32(6.0) / np.float32(fi + fo)))
            u = np.array([rng.next() >> 40 for _ in range(n)], np.float64).astype(np.float32) * np.float32(2.0 ** -24)
            out.append(((u * np.float32(2.0) - np.float32(1.0)) * limit).astype(np.float32))
        else:
            out.append(np.zeros(n, np.float32))
    return np.concatenate(out)


class _MT64:
    """std::mt19937_64 (the reference's engine), restated for the parameter stream."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def next(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def zhang_init_params(seed: int) -> np.ndarray:
    """The same restatement with the Zhang fans (25/576, 150/64, 192/1): pinned against the reference's
    own init_params(42) in tests/test_widened.py."""
    rng = _MT64(seed)
    out = []
    for n, fans in ((150, (25, 576)), (6, None), (1800, (150, 64)), (12, None), (1920, (192, 1)), (10, None)):
        if fans:
            limit = np.float32(np.sqrt(np.float32(6.0) / np.float32(sum(fans))))
            u = np.array([rng.next() >> 40 for _ in range(n)], np.float64).astype(np.float32) * np.float32(2.0 ** -24)
            out.append(((u * np.float32(2.0) - np.float32(1.0)) * limit).astype(np.float32))
        else:
            out.append(np.zeros(n, np.float32))
    return np.concatenate(out)


def make_set(orc, n: int, seed: int):
    """64x64 inputs: synth::make_digits bytes centred (offset 18) on a zero canvas, /255.0f."""
    px, lab = orc.make_digits(n, seed)
    x = np.zeros((n, IMG, IMG), np.float32)
    x[:, 18:46, 18:46] = px.reshape(n, 28, 28).astype(np.float32) / np.float32(255.0)
    return x.reshape(n, IMG * IMG), lab


def split(p):
    out, o = [], 0
    for s, n in zip(SHAPES, SIZES):
        out.append(np.ascontiguousarray(p[o:o + n]).reshape(s))
        o += n
    return out


class WideReference:
    """Forward / backward / train step of the widened CNN through the reference's nn:: operators."""

    def __init__(self, ref):
        self.L = ref.L
        self.ref = ref

    # -- thin wrappers over oracle/ref_shim.cpp (shapes as int64 arrays) --
    @staticmethod
    def _s(shape):
        a = np.array(shape, np.int64)
        return a, a.ctypes.data_as(C.POINTER(C.c_int64)), len(shape)

    @staticmethod
    def _f(a):
        return np.ascontiguousarray(a, np.float32).ctypes.data_as(C.POINTER(C.c_float))

    def _rc(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.ref_last_error().decode()}")

    def mconv(self, x, k, b, out_shape):
        x, k, b = (np.ascontiguousarray(v, np.float32) for v in (x, k, b))
        out = np.zeros(out_shape, np.float32)
        xs, kss, bs = self._s(x.shape), self._s(k.shape), self._s(b.shape)
        self._rc(self.L.ref_mconv(self._f(x), xs[1], xs[2], self._f(k), kss[1], kss[2], self._f(b), bs[1], bs[2],
                                  self._f(out)))
        return out

    def unary(self, fn, x, out_shape):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(out_shape, np.float32)
        s = self._s(x.shape)
        self._rc(fn(self._f(x), s[1], s[2], self._f(out)))
        return out

    def sigmoid(self, x):
        return self.unary(self.L.ref_sigmoid, x, x.shape)

    def avgpool(self, x):
        return self.unary(self.L.ref_avgpool, x, x.shape[:-2] + (x.shape[-2] // 2, x.shape[-1] // 2))

    def backavgpool(self, d):
        return self.unary(self.L.ref_backavgpool, d, d.shape[:-2] + (d.shape[-2] * 2, d.shape[-1] * 2))

    def backsigmoid(self, d, o):
        d, o = np.ascontiguousarray(d, np.float32), np.ascontiguousarray(o, np.float32)
        out = np.zeros(d.shape, np.float32)
        s = self._s(d.shape)
        self._rc(self.L.ref_backsigmoid(self._f(d), self._f(o), s[1], s[2], self._f(out)))
        return out

    def backweights(self, d, x):
        d, x = np.ascontiguousarray(d, np.float32), np.ascontiguousarray(x, np.float32)
        out = np.zeros(tuple(a - b + 1 for a, b in zip(x.shape, d.shape)), np.float32)
        ds, xs = self._s(d.shape), self._s(x.shape)
        self._rc(self.L.ref_backweights(self._f(d), ds[1], self._f(x), xs[1], ds[2], self._f(out)))
        return out

    def backbias(self, d):
        d = np.ascontiguousarray(d, np.float32)
        s = self._s(d.shape)
        return np.float32(self.L.ref_backbias(self._f(d), s[1], s[2]))

    def backin(self, d, k, in_shape):
        d, k = np.ascontiguousarray(d, np.float32), np.ascontiguousarray(k, np.float32)
        out = np.zeros(in_shape, np.float32)
        ds, ks, ins = self._s(d.shape), self._s(k.shape), self._s(in_shape)
        self._rc(self.L.ref_backin(self._f(d), ds[1], self._f(k), ks[1], ins[1], ds[2], self._f(out)))
        return out

    # -- network (network.cpp:81-169 pattern) --
    def forward(self, image, p):
        k1, b1, k2, b2, fc, b = split(p)
        x = np.ascontiguousarray(image, np.float32).reshape(IMG, IMG)
        c1 = self.sigmoid(self.mconv(x, k1, b1, (32, 60, 60)))
        s1 = self.avgpool(c1)
        c2 = self.sigmoid(self.mconv(s1, k2, b2, (64, 1, 26, 26)))
        s2 = self.avgpool(c2)
        out = self.sigmoid(self.mconv(s2, fc, b, (10, 1, 1, 1, 1)))
        return dict(input=x, c1=c1, s1=s1, c2=c2, s2=s2, out=out)

    def layer_backward(self, d_act, act_out, x, k, need_d_in):
        dz = self.backsigmoid(d_act, act_out)
        nk = k.shape[0]
        gk = np.stack([self.backweights(dz[i], x) for i in range(nk)])
        gb = np.array([self.backbias(dz[i]) for i in range(nk)], np.float32)
        d_in = None
        if need_d_in:
            acc = np.zeros(x.shape, np.float32)
            for i in range(nk):
                acc = (acc + self.backin(dz[i], k[i], x.shape)).astype(np.float32)
            d_in = acc
        return gk, gb, d_in

    def backward(self, cache, p, y):
        k1, b1, k2, b2, fc, b = split(p)
        yhat = cache["out"].reshape(10)
        d = (yhat - np.asarray(y, np.float32)).astype(np.float32).reshape(10, 1, 1, 1, 1)
        gfc, gb, d_s2 = self.layer_backward(d, cache["out"], cache["s2"], fc, True)
        gk2, gb2, d_s1 = self.layer_backward(self.backavgpool(d_s2), cache["c2"], cache["s1"], k2, True)
        gk1, gb1, _ = self.layer_backward(self.backavgpool(d_s1), cache["c1"], cache["input"], k1, False)
        return np.concatenate([g.reshape(-1) for g in (gk1, gb1, gk2, gb2, gfc, gb)]).astype(np.float32)

    @staticmethod
    def loss(yhat, y):
        acc = np.float32(0.0)
        for i in range(10):
            dd = np.float32(y[i]) - np.float32(yhat[i])
            acc = np.float32(acc + np.float32(dd * dd))
        return np.float32(np.float32(0.5) * acc)

    def train_step(self, images, labels, p, rate):
        """One group (network.cpp:228-244): per-example forward/backward, example-order sum, sgd_step."""
        acc = np.zeros(NPARAM, np.float32)
        lsum = 0.0
        for img, lab in zip(images, labels):
            y = np.zeros(10, np.float32)
            y[int(lab)] = 1.0
            cache = self.forward(img, p)
            g = self.backward(cache, p, y)
            acc = (acc + g).astype(np.float32)
            lsum += float(self.loss(cache["out"].reshape(10), y))
        m = np.float32(len(labels))
        newp = (p - np.float32(rate) * (acc / m)).astype(np.float32)
        return newp, lsum, acc
