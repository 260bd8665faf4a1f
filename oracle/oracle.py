"""CPU oracle for the binary forward pass — TEST INFRASTRUCTURE ONLY.

This module restates the reference `bitnn` packed backend on the CPU so
the CUDA product can be checked bit for bit, and doubles as the CPU
baseline ("port") that bench.py times.  It must only be imported by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs; the product package never imports it.

Kernels live in oracle.c (one C function per reference Numba kernel,
``/root/reference/pkg/src/bitnn/_kernels.py``); this file holds the
ctypes bindings, the layer-level wrappers of ``layers.py`` and the
network compile/forward of ``network.py`` (packed backend only).

Pinned against the reference by tests/test_oracle_golden.py, using the
vectors tests/golden/make_golden.py produced by running the reference.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

ALWAYS = -(1 << 62)
NEVER = 1 << 62

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def wpl(bits: int) -> int:
    return -(-bits // 64)


I64 = ctypes.c_int64
I32 = ctypes.c_int32
XKIND = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.uint8): 2}


# ---------------------------------------------------------------- kernels

def pack_lines(lines: np.ndarray) -> np.ndarray:
    """_kernels.py:43-54."""
    lines = np.ascontiguousarray(lines, dtype=np.float32)
    n, bits = lines.shape
    out = np.zeros((n, wpl(bits)), dtype=np.uint64)
    lib().o_pack_lines(_p(lines), I64(n), I64(bits), _p(out))
    return out


def unpack_lines(words: np.ndarray, bits: int) -> np.ndarray:
    """_kernels.py:57-64."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    out = np.empty((words.shape[0], bits), dtype=np.float32)
    lib().o_unpack_lines(_p(words), I64(words.shape[0]), I64(bits), _p(out))
    return out


def pack_byte_planes(lines: np.ndarray) -> np.ndarray:
    """_kernels.py:67-82: (n_lines, bits) uint8 -> (8, n_lines, wpl)."""
    lines = np.ascontiguousarray(lines, dtype=np.uint8)
    n, bits = lines.shape
    out = np.zeros((8, n, wpl(bits)), dtype=np.uint64)
    lib().o_pack_byte_planes(_p(lines), I64(n), I64(bits), _p(out))
    return out


def bgemm(a_words: np.ndarray, b_words: np.ndarray, k: int, out=None) -> np.ndarray:
    """_kernels.py:85-106."""
    a_words = np.ascontiguousarray(a_words, dtype=np.uint64)
    b_words = np.ascontiguousarray(b_words, dtype=np.uint64)
    m, w = a_words.shape
    n = b_words.shape[0]
    assert b_words.shape[1] == w
    if out is None:
        out = np.empty((m, n), dtype=np.int32)
    lib().o_bgemm(_p(a_words), I64(m), _p(b_words), I64(n), I64(w), I32(k), _p(out))
    return out


def bgemv(a_words: np.ndarray, x_words: np.ndarray, k: int) -> np.ndarray:
    """_kernels.py:109-117."""
    a_words = np.ascontiguousarray(a_words, dtype=np.uint64)
    x_words = np.ascontiguousarray(x_words, dtype=np.uint64)
    out = np.empty(a_words.shape[0], dtype=np.int32)
    lib().o_bgemv(_p(a_words), I64(a_words.shape[0]), I64(a_words.shape[1]), _p(x_words), I32(k), _p(out))
    return out


def bitplane_matvec(planes: np.ndarray, w_words: np.ndarray) -> np.ndarray:
    """_kernels.py:120-147 (count_plane_bits + bitplane_matvec)."""
    planes = np.ascontiguousarray(planes, dtype=np.uint64)
    w_words = np.ascontiguousarray(w_words, dtype=np.uint64)
    pops = np.empty(8, dtype=np.int64)
    lib().o_count_plane_bits(_p(planes), I64(planes.shape[1]), _p(pops))
    out = np.empty(w_words.shape[0], dtype=np.int64)
    lib().o_bitplane_matvec(_p(planes), _p(pops), _p(w_words), I64(w_words.shape[0]), I64(w_words.shape[1]),
                            _p(out))
    return out


def unroll_packed(lines: np.ndarray, h, w, c, kh, kw, stride, pad) -> np.ndarray:
    """_kernels.py:170-199 (axis rule of tensor.py:165-166: channel axis iff c > 1)."""
    lines = np.ascontiguousarray(lines, dtype=np.uint64)
    h_out = (h + 2 * pad - kh) // stride + 1
    w_out = (w + 2 * pad - kw) // stride + 1
    out = np.zeros((h_out * w_out, wpl(kh * kw * c)), dtype=np.uint64)
    lib().o_unroll_packed(_p(lines), h, w, c, int(c > 1), kh, kw, stride, pad, _p(out))
    return out


def maxpool(x: np.ndarray, ph, pw, stride) -> np.ndarray:
    """_kernels.py:224-240 on int32 (H, W, C)."""
    x = np.ascontiguousarray(x, dtype=np.int32)
    h, w, c = x.shape
    out = np.empty(((h - ph) // stride + 1, (w - pw) // stride + 1, c), dtype=np.int32)
    lib().o_maxpool_i32(_p(x), h, w, c, ph, pw, stride, _p(out))
    return out


def threshold_sign_pack(x: np.ndarray, thresh: np.ndarray, ge_dir: np.ndarray, flat: bool) -> np.ndarray:
    """_kernels.py:243-267; x is (sites, C) int32/int64/uint8."""
    x = np.ascontiguousarray(x)
    sites, c = x.shape
    thresh = np.ascontiguousarray(thresh, dtype=np.int64)
    ge = np.ascontiguousarray(ge_dir, dtype=np.uint8)
    out = np.zeros((1, wpl(sites * c)) if flat else (sites, wpl(c)), dtype=np.uint64)
    lib().o_threshold_sign_pack(_p(x), XKIND[x.dtype], I64(sites), I64(c), _p(thresh), _p(ge), int(flat), _p(out))
    return out


def bn_affine(x: np.ndarray, mean64, scale64, beta64) -> np.ndarray:
    """_kernels.py:285-295 (float64, separately rounded)."""
    x = np.ascontiguousarray(x).reshape(-1)
    out = np.empty(x.shape[0], dtype=np.float64)
    m, s, b = (np.ascontiguousarray(v, dtype=np.float64) for v in (mean64, scale64, beta64))
    lib().o_bn_affine(_p(x), XKIND[x.dtype], I64(x.shape[0]), _p(m), _p(s), _p(b), I64(m.shape[0]), _p(out))
    return out


def bn_calibrate(mean, var, gamma, beta, eps):
    """layers.py:137-191: float64 scale and integer thresholds."""
    mean, var, gamma, beta = (np.ascontiguousarray(np.atleast_1d(v), dtype=np.float32) for v in (mean, var, gamma, beta))
    c = mean.shape[0]
    scale = np.empty(c, dtype=np.float64)
    thresh = np.empty(c, dtype=np.int64)
    ge = np.empty(c, dtype=np.uint8)
    lib().o_bn_calibrate(_p(mean), _p(var), _p(gamma), _p(beta), ctypes.c_double(float(eps)), I64(c),
                         _p(scale), _p(thresh), _p(ge))
    return scale, thresh, ge.astype(bool)


def compute_correction(w_words: np.ndarray, in_shape, kernel, stride, pad) -> np.ndarray:
    """layers.py:224-252 from packed filter lines (F, wpl(K))."""
    w_words = np.ascontiguousarray(w_words, dtype=np.uint64)
    h, w, c = in_shape
    kh, kw = kernel
    h_out = (h + 2 * pad - kh) // stride + 1
    w_out = (w + 2 * pad - kw) // stride + 1
    out = np.empty((h_out * w_out, w_words.shape[0]), dtype=np.int32)
    lib().o_compute_correction(_p(w_words), I64(w_words.shape[0]), h, w, c, kh, kw, stride, pad, _p(out))
    return out


def num_threads() -> int:
    return int(lib().o_num_threads())


# ---------------------------------------------------------------- network

class OracleNetwork:
    """network.py:331-486 _compile + :506-522 forward, packed backend only.

    `spec` is any object with `input_dims` and `records` whose records
    carry the ESPBDNN1 fields (the product's ModelSpec qualifies).
    """

    def __init__(self, spec):
        self.input_dims = tuple(spec.input_dims)
        self.stages = []
        recs = spec.records
        kinds = [type(r).__name__ for r in recs]
        shape = self.input_dims
        rep = "bytes"

        def nxt(i):
            return kinds[i + 1] if i + 1 < len(recs) else None

        for i, r in enumerate(recs):
            kind = kinds[i]
            last = i == len(recs) - 1
            if kind == "Input8Record":
                self.stages.append(("input8", r.words, r.input_len))
                shape, rep = (1, 1, r.units), "acc"
            elif kind == "DenseRecord":
                self.stages.append(("dense", r.words, r.input_len))
                shape, rep = (1, 1, r.units), "acc"
            elif kind == "ConvRecord":
                h, w, c = shape
                corr = compute_correction(r.words, shape, (r.kh, r.kw), r.stride, r.pad)
                self.stages.append(("conv", r, shape, corr))
                h_out = (h + 2 * r.pad - r.kh) // r.stride + 1
                w_out = (w + 2 * r.pad - r.kw) // r.stride + 1
                shape, rep = (h_out, w_out, r.filters), "acc"
            elif kind == "MaxPoolRecord":
                h, w, c = shape
                self.stages.append(("pool", r.ph, r.pw, r.stride))
                shape = ((h - r.ph) // r.stride + 1, (w - r.pw) // r.stride + 1, c)
            elif kind == "BatchNormRecord":
                scale, thresh, ge = bn_calibrate(r.mean, r.var, r.gamma, r.beta, r.eps)
                if last:
                    self.stages.append(("final", r.mean.astype(np.float64), scale, r.beta.astype(np.float64)))
                    continue
                h, w, c = shape
                flat = nxt(i) in ("DenseRecord", "Input8Record")
                sites = h * w
                # network.py:108-125 _bn_line_plan
                if flat or sites == 1:
                    plan = ((sites, c), thresh, ge, True)
                elif c == 1:
                    plan = ((h, w), np.full(w, thresh[0]), np.full(w, ge[0]), False)
                else:
                    plan = ((sites, c), thresh, ge, False)
                self.stages.append(("bn", plan))
                if flat:
                    shape = (1, 1, sites * c)
                rep = "packed"
        self.classes = shape[2]

    def forward(self, image: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(image, dtype=np.uint8)
        h0, w0, c0 = self.input_dims
        shape = (h0, w0, c0)
        for st in self.stages:
            kind = st[0]
            if kind == "input8":
                _, words, k = st
                planes = pack_byte_planes(x.reshape(1, -1))[:, 0, :]
                x = bitplane_matvec(planes, words)
                shape = (1, 1, x.shape[0])
            elif kind == "dense":
                _, words, k = st
                x = bgemv(words, x.reshape(-1), k)
                shape = (1, 1, x.shape[0])
            elif kind == "conv":
                _, r, in_shape, corr = st
                h, w, c = in_shape
                u = unroll_packed(x, h, w, c, r.kh, r.kw, r.stride, r.pad)
                acc = bgemm(u, r.words, r.k)
                acc += corr
                h_out = (h + 2 * r.pad - r.kh) // r.stride + 1
                w_out = (w + 2 * r.pad - r.kw) // r.stride + 1
                shape = (h_out, w_out, r.filters)
                x = acc.reshape(shape)
            elif kind == "pool":
                _, ph, pw, s = st
                x = maxpool(x.reshape(shape), ph, pw, s)
                shape = x.shape
            elif kind == "bn":
                view, thresh, ge, flat = st[1]
                x = threshold_sign_pack(np.ascontiguousarray(x).reshape(view), thresh, ge, flat)
            elif kind == "final":
                _, m, s, b = st
                x = bn_affine(x, m, s, b)
        return x

    def forward_batch(self, images: np.ndarray) -> np.ndarray:
        images = np.asarray(images)
        return np.stack([self.forward(images[i]) for i in range(images.shape[0])])
