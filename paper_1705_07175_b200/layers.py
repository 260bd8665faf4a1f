"""Layer types and layer-level forward ops (mirror of bitnn/layers.py:1-351).

Same semantics as the reference: convolution is bit-im2col + binary GEMM
with a padding-correction map, max-pool runs on integer accumulators
before batchnorm, and batchnorm + sign collapse to per-channel integer
thresholds calibrated in float64.  All arithmetic runs on the GPU
(calibration and correction maps included); arguments and results are
numpy arrays as in the reference.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .gemm import PackedMatrixA, PackedMatrixB, bgemv, bitplane_gemv
from .tensor import Axis, FloatTensor, PackedTensor, pack, pack_lines, words_per_line

ALWAYS = -(1 << 62)
NEVER = 1 << 62
DEFAULT_EPS = 1e-5
XKIND = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.uint8): 2, np.dtype(np.float64): 3}


def _thresh_struct(t32=None, t64=None, ge=None) -> _lib.Thresh:
    return _lib.Thresh(_dev.P(t32).value if t32 is not None else None,
                       _dev.P(t64).value if t64 is not None else None,
                       _dev.P(ge).value if ge is not None else None)


class Input8Layer:
    def __init__(self, weights: PackedMatrixA):
        self.weights = weights
        self.units = weights.rows
        self.input_len = weights.k


class DenseLayer:
    def __init__(self, weights: PackedMatrixA):
        self.weights = weights
        self.units = weights.rows
        self.input_len = weights.k


class ConvLayer:
    """2-D binary convolution, filters column-packed over kh*kw*C_in."""

    def __init__(self, weights: PackedMatrixB, kernel, stride: int, pad: int, in_shape):
        kh, kw = kernel
        h, w, c = in_shape
        if weights.k != kh * kw * c:
            raise ValueError(f"filter matrix has K={weights.k}, expected kh*kw*C = {kh * kw * c}")
        if stride < 1 or pad < 0:
            raise ValueError(f"bad stride/pad: {stride}, {pad}")
        if h + 2 * pad < kh or w + 2 * pad < kw:
            raise ValueError(f"kernel {kernel} larger than padded input {in_shape} + pad {pad}")
        self.weights = weights
        self.kernel = (kh, kw)
        self.stride = stride
        self.pad = pad
        self.in_shape = tuple(in_shape)
        self.filters = weights.cols
        h_out = (h + 2 * pad - kh) // stride + 1
        w_out = (w + 2 * pad - kw) // stride + 1
        self.out_shape = (h_out, w_out, self.filters)
        self.correction = compute_correction_packed(weights.words, in_shape, self.kernel, stride, pad)

    def weights_float(self) -> np.ndarray:
        out = _dev.empty((self.weights.cols, self.weights.k), np.float32)
        _lib.call("b2_unpack_lines_f32", _dev.P(_dev.upload(self.weights.words)), self.weights.cols, self.weights.k,
                  _dev.P(out), _dev.stream())
        return _dev.download(out, np.float32).T.copy()

    @classmethod
    def from_float(cls, w, kernel, stride, pad, in_shape) -> "ConvLayer":
        return cls(PackedMatrixB.from_float(w), kernel, stride, pad, in_shape)


class MaxPoolLayer:
    def __init__(self, window, stride: int):
        if stride < 1 or min(window) < 1:
            raise ValueError(f"bad pooling window/stride: {window}, {stride}")
        self.window = tuple(window)
        self.stride = stride

    def out_shape(self, in_shape):
        h, w, c = in_shape
        ph, pw = self.window
        if h < ph or w < pw:
            raise ValueError(f"pooling window {self.window} larger than input {in_shape}")
        return ((h - ph) // self.stride + 1, (w - pw) // self.stride + 1, c)


class BatchNormLayer:
    """Inference batchnorm; float64 working form and integer thresholds
    (layers.py:111-191 of the reference), calibrated by the device kernel
    b2_bn_calibrate."""

    def __init__(self, mean, var, gamma, beta, eps: float = DEFAULT_EPS):
        mean, var, gamma, beta = (np.atleast_1d(np.asarray(v, dtype=np.float32)) for v in (mean, var, gamma, beta))
        if not (mean.shape == var.shape == gamma.shape == beta.shape) or mean.ndim != 1:
            raise ValueError("batchnorm parameter vectors must share one length")
        if np.any(var < 0):
            raise ValueError("negative variance")
        if eps < 0:
            raise ValueError("negative epsilon")
        if np.any(var.astype(np.float64) + eps <= 0):
            raise ValueError("variance + epsilon must be positive")
        if not all(np.all(np.isfinite(v)) for v in (mean, var, gamma, beta)):
            raise ValueError("non-finite batchnorm parameter")
        self.mean, self.var, self.gamma, self.beta = mean, var, gamma, beta
        self.eps = float(eps)
        self.channels = mean.shape[0]
        self.mean64 = mean.astype(np.float64)
        self.beta64 = beta.astype(np.float64)
        dev = calibrate_device(mean, var, gamma, beta, self.eps, bound=0)
        self.scale64 = _dev.download(dev["scale64"], np.float64)
        self.thresh = _dev.download(dev["thresh64"], np.int64)
        self.ge_dir = _dev.download(dev["ge"], np.uint8).astype(np.bool_)


def calibrate_device(mean, var, gamma, beta, eps: float, bound: int) -> dict:
    """Upload float32 batchnorm params and calibrate on the GPU.

    Returns device tensors scale64, thresh64, ge (uint8), thresh32
    (clamped to [-(bound+1), bound+1]) plus mean64 / beta64."""
    c = int(np.asarray(mean).shape[0])
    f = [_dev.upload(np.ascontiguousarray(v, dtype=np.float32)) for v in (mean, var, gamma, beta)]
    out = {"scale64": _dev.empty((c,), np.float64), "thresh64": _dev.empty((c,), np.int64),
           "ge": _dev.empty((c,), np.uint8), "thresh32": _dev.empty((c,), np.int32)}
    _lib.call("b2_bn_calibrate", *[_dev.P(t) for t in f], float(eps), c, int(min(bound, (1 << 31) - 2)),
              _dev.P(out["scale64"]), _dev.P(out["thresh64"]), _dev.P(out["ge"]), _dev.P(out["thresh32"]),
              _dev.stream())
    out["mean64"] = _dev.upload(np.asarray(mean, dtype=np.float32).astype(np.float64))
    out["beta64"] = _dev.upload(np.asarray(beta, dtype=np.float32).astype(np.float64))
    return out


def input8_forward(layer: Input8Layer, data: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
    if data.shape[0] != layer.input_len:
        raise ValueError(f"expected {layer.input_len} input bytes, got {data.shape[0]}")
    planes = _dev.empty((8, 1, words_per_line(layer.input_len)), np.uint64)
    _lib.call("b2_pack_byte_planes", _dev.P(_dev.upload(data.reshape(1, -1))), 1, layer.input_len, _dev.P(planes),
              _dev.stream())
    return bitplane_gemv(_dev.download(planes, np.uint64)[:, 0, :], layer.weights, out=out)


def dense_forward(layer: DenseLayer, a: PackedTensor, out: np.ndarray | None = None) -> np.ndarray:
    if a.n_lines != 1 or a.bits_per_line != layer.input_len:
        raise ValueError(f"dense layer wants one {layer.input_len}-bit line, got {a.n_lines} x {a.bits_per_line}")
    return bgemv(layer.weights, a.words[0], out=out)


def unroll(a: PackedTensor, kernel, stride: int, pad: int) -> PackedMatrixA:
    h, w, c = a.dims
    kh, kw = kernel
    if h + 2 * pad < kh or w + 2 * pad < kw:
        raise ValueError(f"kernel {kernel} larger than padded input {a.dims} + pad {pad}")
    h_out = (h + 2 * pad - kh) // stride + 1
    w_out = (w + 2 * pad - kw) // stride + 1
    k = kh * kw * c
    out = _dev.empty((h_out * w_out, words_per_line(k)), np.uint64)
    _lib.call("b2_unroll_packed", _dev.P(_dev.upload(a.words)), 1, h, w, c, kh, kw, stride, pad, _dev.P(out),
              _dev.stream())
    return PackedMatrixA(h_out * w_out, k, _dev.download(out, np.uint64))


def correction_device(words_dev, filters: int, in_shape, kernel, stride: int, pad: int):
    h, w, c = in_shape
    kh, kw = kernel
    h_out = (h + 2 * pad - kh) // stride + 1
    w_out = (w + 2 * pad - kw) // stride + 1
    out = _dev.empty((h_out * w_out, filters), np.int32)
    _lib.call("b2_conv_correction", _dev.P(words_dev), filters, h, w, c, kh, kw, stride, pad, _dev.P(out),
              _dev.stream())
    return out


def compute_correction_packed(words: np.ndarray, in_shape, kernel, stride: int, pad: int) -> np.ndarray:
    return _dev.download(correction_device(_dev.upload(words), words.shape[0], in_shape, kernel, stride, pad),
                         np.int32)


def compute_correction(weights: np.ndarray, in_shape, kernel, stride: int, pad: int) -> np.ndarray:
    """Padding repair map from a (kh*kw*C, F) +/-1 weight matrix (layers.py:224-252)."""
    h, w, c = in_shape
    kh, kw = kernel
    wf = np.asarray(weights, dtype=np.float32)
    if wf.shape[0] != kh * kw * c:
        raise ValueError(f"weights rows {wf.shape[0]} != kh*kw*C {kh * kw * c}")
    words = pack_lines(np.ascontiguousarray(np.rint(wf).T))
    return compute_correction_packed(words, in_shape, kernel, stride, pad)


def conv_forward(layer: ConvLayer, a: PackedTensor) -> np.ndarray:
    """Zero-padded binary convolution, exact int32 (H_out, W_out, F) view
    of the (positions, F) GEMM buffer."""
    if a.dims != layer.in_shape:
        raise ValueError(f"expected input dims {layer.in_shape}, got {a.dims}")
    h, w, c = a.dims
    kh, kw = layer.kernel
    acc = _dev.empty((layer.out_shape[0] * layer.out_shape[1], layer.filters), np.int32)
    scratch_words = int(_lib.raw("b2_conv_scratch_words")(1, h, w, c, kh, kw, layer.stride, layer.pad))
    scratch = _dev.empty((max(scratch_words, 1),), np.uint64) if scratch_words else None
    corr = _dev.upload(layer.correction)
    _lib.call("b2_conv_forward", _dev.P(_dev.upload(a.words)), 1, h, w, c, _dev.P(_dev.upload(layer.weights.words)),
              layer.filters, kh, kw, layer.stride, layer.pad, _dev.P(corr), _dev.P(scratch), _dev.P(acc),
              _dev.stream())
    return _dev.download(acc, np.int32).reshape(layer.out_shape)


def maxpool_forward(x: np.ndarray, window, stride: int, out: np.ndarray | None = None) -> np.ndarray:
    if x.ndim != 3:
        raise ValueError(f"expected (H, W, C) input, got shape {x.shape}")
    h, w, c = x.shape
    ph, pw = window
    if h < ph or w < pw or stride < 1:
        raise ValueError(f"pooling window {window} stride {stride} does not fit input {x.shape}")
    h_out = (h - ph) // stride + 1
    w_out = (w - pw) // stride + 1
    if x.dtype != np.int32:
        raise ValueError(f"the device max-pool works on int32 accumulators, got {x.dtype}")
    res = _dev.empty((h_out, w_out, c), np.int32)
    _lib.call("b2_maxpool_i32", _dev.P(_dev.upload(x)), 1, h, w, c, ph, pw, stride, _dev.P(res), _dev.stream())
    host = _dev.download(res, np.int32)
    if out is None:
        return host
    out[...] = host
    return out


def batchnorm_forward(layer: BatchNormLayer, x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    x = np.asarray(x)
    if x.shape[-1] != layer.channels:
        raise ValueError(f"channel mismatch: input {x.shape[-1]}, layer {layer.channels}")
    xs = np.ascontiguousarray(x if x.dtype in (np.int32, np.int64, np.float64) else x.astype(np.float64))
    res = _dev.empty(x.shape, np.float64)
    if xs.size:
        _lib.call("b2_bn_affine_f64", _dev.P(_dev.upload(xs)), XKIND[xs.dtype], xs.size,
                  _dev.P(_dev.upload(layer.mean64)), _dev.P(_dev.upload(layer.scale64)),
                  _dev.P(_dev.upload(layer.beta64)), layer.channels, _dev.P(res), _dev.stream())
    host = _dev.download(res, np.float64)
    if out is None:
        return host
    out[...] = host
    return out


def sign_pack(x: np.ndarray) -> PackedTensor:
    x = np.asarray(x)
    if x.ndim == 1:
        x = x.reshape(1, 1, -1)
    return pack(FloatTensor(np.where(x < 0, np.float32(-1.0), np.float32(1.0))))


def threshold_pack_device(x_dev, xkind: int, batch: int, sites: int, c: int, t64_dev, ge_dev, flat: bool, out_dev):
    _lib.call("b2_threshold_pack", _dev.P(x_dev), xkind, batch, sites, c, _thresh_struct(t64=t64_dev, ge=ge_dev),
              int(flat), _dev.P(out_dev), _dev.stream())
    return out_dev


def fused_bn_sign(layer: BatchNormLayer, x: np.ndarray, flat: bool = False,
                  out: np.ndarray | None = None) -> PackedTensor:
    x = np.asarray(x)
    if x.ndim == 1:
        x = x.reshape(1, 1, -1)
    if x.ndim != 3 or x.shape[-1] != layer.channels:
        raise ValueError(f"expected (.., .., {layer.channels}) integer activations, got {x.shape}")
    if x.dtype.kind not in "iu":
        raise ValueError(f"fused path wants integer activations, got {x.dtype}")
    if x.dtype not in (np.int32, np.int64, np.uint8):
        x = x.astype(np.int64)
    h, w, c = x.shape
    sites = h * w
    t64, ge = layer.thresh, layer.ge_dir.astype(np.uint8)
    if c == 1 and not flat and sites > 1:
        # single-channel spatial tensor: column-axis lines, channel-0 rule per row
        view, dims, axis, bits, flat_k = (h, w), (h, w, 1), Axis.COLUMN, w, False
        t64, ge = np.full(w, t64[0], dtype=np.int64), np.full(w, ge[0], dtype=np.uint8)
    elif flat or sites == 1:
        view, dims, axis, bits, flat_k = (sites, c), (1, 1, sites * c), None, sites * c, True
    else:
        view, dims, axis, bits, flat_k = (sites, c), (h, w, c), Axis.CHANNEL, c, False
    axis = axis or (Axis.CHANNEL if dims[2] > 1 else Axis.COLUMN)
    n_lines = 1 if flat_k else view[0]
    res = _dev.empty((n_lines, words_per_line(bits)), np.uint64)
    xv = np.ascontiguousarray(x).reshape(view)
    threshold_pack_device(_dev.upload(xv), XKIND[xv.dtype], 1, view[0], view[1], _dev.upload(t64), _dev.upload(ge),
                          flat_k, res)
    words = _dev.download(res, np.uint64)
    if out is not None:
        out[...] = words
        words = out
    return PackedTensor(dims, axis, words, bits)
