"""Network runtime on the GPU (mirror of bitnn/network.py:1-588, packed backend).

A model spec is validated exactly like the reference (`_compile`,
network.py:331-486: same checks, same order, same "layer i: ..." messages),
then planned into a short list of device stages.  Adjacent reference
stages are fused where the layout allows it:

    _PackedInput8 + _PackedBN            -> b2_input8_bn_pack
    _PackedByteBN + _PackedConv + _PackedBN (window <= 32 bits)
                                         -> b2_byte_conv_bn_pack
    _PackedConv [+ _Pool 2x2/2] + _PackedBN (C % 32 == 0)
                                         -> b2_conv_bn_pack
    _PackedDense + _PackedBN             -> b2_dense_bn_pack
    _FinalBN                             -> b2_bn_affine_f64

and every other combination runs through the general kernels (unroll +
bgemm + correction, maxpool, threshold-pack), all on the device.

Every buffer is allocated at construction for `max_batch` images (the
reference's Workspace, network.py:50-66); a forward pass performs no
allocation and replays a CUDA graph captured per batch size.  `forward`
keeps the reference's batch-1 contract and returns a reused host buffer;
`forward_batch` runs any number of images.
"""

from __future__ import annotations

import ctypes
import enum

import numpy as np
import torch

from . import _dev, _lib
from .layers import XKIND, _thresh_struct, calibrate_device, correction_device
from .modelfile import (BatchNormRecord, ConvRecord, DenseRecord, Input8Record, MaxPoolRecord, ModelSpec,
                        ModelValidationError, load_model, write_model)
from .tensor import words_per_line

MAX_K = 1 << 24


class Backend(enum.Enum):
    PACKED = "packed"
    REFERENCE = "reference"


def _wpl(bits):
    return words_per_line(bits)


# --------------------------------------------------------------------------- stages
# Each stage owns its device output buffer for `cap` images; `src` is the
# producing stage (None = network input bytes).  launch(batch) enqueues the
# kernels for the first `batch` images on the current stream.


class _Stage:
    name = "stage"
    out_dtype = np.uint64

    is_last = False  # writes the scores (the batch-1 graph may point it at pinned host memory)
    # as the first stage, reads the image straight from pinned host memory in
    # the batch-1 graph: only kernels that read their input once, in parallel
    # (each dependent host read is a PCIe round trip)
    zero_copy_in = False

    def __init__(self, src):
        self.src = src
        self.out = None

    def per_image(self):
        raise NotImplementedError

    def alloc(self, cap: int):
        self.out = _dev.empty((cap, *self.per_image()), self.out_dtype)

    def src_ptr(self, net):
        if self.src is None:
            return net._io_ptrs[0] if net._io_ptrs else _dev.P(net._in)
        return _dev.P(self.src.out)

    def out_ptr(self, net):
        if net._io_ptrs and self.is_last and net._io_ptrs[1] is not None:
            return net._io_ptrs[1]
        return _dev.P(self.out)

    def launches(self) -> int:
        return 1


class _Input8Fused(_Stage):
    name = "input8+bn"

    def __init__(self, src, rec, bn_dev):
        super().__init__(src)
        self.k, self.units = rec.input_len, rec.units
        self.w = _dev.upload(rec.words)
        self.bn = bn_dev
        self.tc = _lib.ENGINE == "tc" and self.k % 4 == 0
        # bytes x +/-1 weights in natural K order (the u8 operand is not widened)
        self.w8 = _dev.widen_i8(self.w, self.units, self.k, permute=False) if self.tc else None

    def per_image(self):
        return (_wpl(self.units),)

    def launch(self, net, batch, st):
        if self.tc and batch >= TC_MIN_ROWS:
            _lib.call("b2_tc_input8_bn_pack", self.src_ptr(net), batch, self.k, _dev.P(self.w8), self.units,
                      _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]), _dev.P(self.out), st)
            return
        _lib.call("b2_input8_bn_pack", self.src_ptr(net), batch, self.k, _dev.P(self.w), self.units,
                  _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]), _dev.P(self.out), st)


class _Input8Raw(_Stage):
    name = "input8"
    out_dtype = np.int64

    def __init__(self, src, rec):
        super().__init__(src)
        self.k, self.units = rec.input_len, rec.units
        self.w = _dev.upload(rec.words)

    def per_image(self):
        return (self.units,)

    def alloc(self, cap):
        super().alloc(cap)
        self.planes = _dev.empty((8, cap, _wpl(self.k)), np.uint64)

    def launch(self, net, batch, st):
        _lib.call("b2_pack_byte_planes", self.src_ptr(net), batch, self.k, _dev.P(self.planes), st)
        _lib.call("b2_bitplane_gemv", _dev.P(self.planes), batch, _dev.P(self.w), self.units, _wpl(self.k),
                  _dev.P(self.out), st)

    def launches(self):
        return 2


class _ByteConvFused(_Stage):
    name = "bytebn+conv+bn"
    zero_copy_in = True  # k_byte_unroll / k_byte_conv_bn_pack stage the image bands once

    def __init__(self, src, in_shape, bn0, rec, bn1):
        super().__init__(src)
        self.in_shape = in_shape
        self.rec = rec
        h, w, c = in_shape
        self.h_out = (h + 2 * rec.pad - rec.kh) // rec.stride + 1
        self.w_out = (w + 2 * rec.pad - rec.kw) // rec.stride + 1
        self.w = _dev.upload(rec.words)
        self.bn0, self.bn1 = bn0, bn1
        self.tc = _lib.ENGINE == "tc" and rec.k <= 128 and c <= 8
        if not self.tc and (rec.k > 32 or rec.filters > 1024):
            raise AssertionError("planner chose the fused byte conv for an ineligible shape")
        # one K=32/64 MMA per tile: the kernel is producer/epilogue-bound and
        # the int8 form (TMEM operand, 8-column stores) measured faster than fp4
        self.fmt = "i8"
        self.wt = _dev.tc_weights(self.w, rec.filters, rec.k, self.fmt) if self.tc else None

    def per_image(self):
        return (self.h_out * self.w_out, _wpl(self.rec.filters))

    def alloc(self, cap):
        super().alloc(cap)
        h, w, c = self.in_shape
        r = self.rec
        # the fused kernel (b2_tc_byte_conv_path == 1) needs no unrolled scratch
        self.fused = self.tc and int(_lib.raw("b2_tc_byte_conv_path")(cap, h, w, c, r.filters, r.kh, r.kw, r.stride,
                                                                         r.pad, 0)) == 1
        n = 8 if self.fused else int(_lib.raw("b2_tc_byte_conv_scratch_bytes")(cap, h, w, c, r.kh, r.kw, r.stride,
                                                                                 r.pad))
        self.codes = _dev.empty((n,), np.uint8) if self.tc else None

    def launches(self):
        return (1 if self.fused else 2) if self.tc else 1

    def launch(self, net, batch, st):
        h, w, c = self.in_shape
        r = self.rec
        if self.tc:
            _lib.call(_lib.tc_entry("byte_conv_bn_pack", self.fmt), self.src_ptr(net), batch, h, w, c,
                      _thresh_struct(self.bn0["thresh32"], self.bn0["thresh64"], self.bn0["ge"]), _dev.P(self.wt),
                      r.filters, r.kh, r.kw, r.stride, r.pad, 0,
                      _thresh_struct(self.bn1["thresh32"], self.bn1["thresh64"], self.bn1["ge"]), _dev.P(self.codes),
                      _dev.P(self.out), st)
            return
        _lib.call("b2_byte_conv_bn_pack", self.src_ptr(net), batch, h, w, c,
                  _thresh_struct(self.bn0["thresh32"], self.bn0["thresh64"], self.bn0["ge"]), _dev.P(self.w),
                  r.filters, r.kh, r.kw, r.stride, r.pad,
                  _thresh_struct(self.bn1["thresh32"], self.bn1["thresh64"], self.bn1["ge"]), _dev.P(self.out), st)


class _ConvFused(_Stage):
    name = "conv+bn"

    def __init__(self, src, in_shape, rec, pool: bool, bn_dev):
        super().__init__(src)
        self.in_shape, self.rec, self.pool, self.bn = in_shape, rec, pool, bn_dev
        h, w, c = in_shape
        self.h_out = (h + 2 * rec.pad - rec.kh) // rec.stride + 1
        self.w_out = (w + 2 * rec.pad - rec.kw) // rec.stride + 1
        self.w = _dev.upload(rec.words)
        self.tc = _lib.ENGINE == "tc" and c % 64 == 0
        if self.tc:  # zero padding on the tensor cores: no correction map needed
            self.fmt = _lib.TC_FORMAT
            self.wt, self.corr = _dev.tc_weights(self.w, rec.filters, rec.k, self.fmt), None
        else:
            self.corr = correction_device(self.w, rec.filters, in_shape, (rec.kh, rec.kw), rec.stride, rec.pad)
        if pool:
            self.name = "conv+pool+bn"

    def per_image(self):
        sites = self.h_out * self.w_out // (4 if self.pool else 1)
        return (sites, _wpl(self.rec.filters))

    def launch(self, net, batch, st):
        h, w, c = self.in_shape
        r = self.rec
        if self.tc:
            _lib.call(_lib.tc_entry("conv_bn_pack", self.fmt), self.src_ptr(net), batch, h, w, c, _dev.P(self.wt), r.filters, r.kh,
                      r.kw, r.stride, r.pad, int(self.pool),
                      _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]), _dev.P(self.out), st)
            return
        _lib.call("b2_conv_bn_pack", self.src_ptr(net), batch, h, w, c, _dev.P(self.w), r.filters, r.kh, r.kw,
                  r.stride, r.pad, _dev.P(self.corr), int(self.pool),
                  _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]), _dev.P(self.out), st)


class _Conv(_Stage):
    name = "conv"
    out_dtype = np.int32

    def __init__(self, src, in_shape, rec):
        super().__init__(src)
        self.in_shape, self.rec = in_shape, rec
        h, w, c = in_shape
        self.h_out = (h + 2 * rec.pad - rec.kh) // rec.stride + 1
        self.w_out = (w + 2 * rec.pad - rec.kw) // rec.stride + 1
        self.w = _dev.upload(rec.words)
        self.tc = _lib.ENGINE == "tc" and c % 64 == 0
        if self.tc:
            self.fmt = _lib.TC_FORMAT
            self.wt, self.corr = _dev.tc_weights(self.w, rec.filters, rec.k, self.fmt), None
        else:
            self.corr = correction_device(self.w, rec.filters, in_shape, (rec.kh, rec.kw), rec.stride, rec.pad)

    def per_image(self):
        return (self.h_out, self.w_out, self.rec.filters)

    def alloc(self, cap):
        super().alloc(cap)
        h, w, c = self.in_shape
        r = self.rec
        n = 0 if self.tc else int(_lib.raw("b2_conv_scratch_words")(cap, h, w, c, r.kh, r.kw, r.stride, r.pad))
        self.scratch = _dev.empty((n,), np.uint64) if n else None

    def launch(self, net, batch, st):
        h, w, c = self.in_shape
        r = self.rec
        if self.tc:
            _lib.call(_lib.tc_entry("conv_forward", self.fmt), self.src_ptr(net), batch, h, w, c, _dev.P(self.wt), r.filters, r.kh,
                      r.kw, r.stride, r.pad, _dev.P(self.out), st)
            return
        _lib.call("b2_conv_forward", self.src_ptr(net), batch, h, w, c, _dev.P(self.w), r.filters, r.kh, r.kw,
                  r.stride, r.pad, _dev.P(self.corr), _dev.P(self.scratch), _dev.P(self.out), st)

    def launches(self):
        return 3 if self.scratch is not None else 1


class _Pool(_Stage):
    name = "maxpool"
    out_dtype = np.int32

    def __init__(self, src, in_shape, rec):
        super().__init__(src)
        self.in_shape, self.rec = in_shape, rec
        h, w, c = in_shape
        self.out_shape = ((h - rec.ph) // rec.stride + 1, (w - rec.pw) // rec.stride + 1, c)

    def per_image(self):
        return self.out_shape

    def launch(self, net, batch, st):
        h, w, c = self.in_shape
        _lib.call("b2_maxpool_i32", self.src_ptr(net), batch, h, w, c, self.rec.ph, self.rec.pw, self.rec.stride,
                  _dev.P(self.out), st)


class _BN(_Stage):
    """Generic batchnorm + sign + pack (network.py:108-125 line plans)."""

    name = "bn"

    def __init__(self, src, dims, bn_dev, flat: bool, xkind: int):
        super().__init__(src)
        h, w, c = dims
        sites = h * w
        self.xkind = xkind
        t64, ge = bn_dev["thresh64"], bn_dev["ge"]
        if flat or sites == 1:
            self.view, self.flat, self.lines, self.bits = (sites, c), True, 1, sites * c
        elif c == 1:
            self.view, self.flat, self.lines, self.bits = (h, w), False, h, w
            t64, ge = t64[:1].expand(w).contiguous(), ge[:1].expand(w).contiguous()
        else:
            self.view, self.flat, self.lines, self.bits = (sites, c), False, sites, c
        self.t64, self.ge = t64, ge

    def per_image(self):
        return (self.lines, _wpl(self.bits))

    def launch(self, net, batch, st):
        _lib.call("b2_threshold_pack", self.src_ptr(net), self.xkind, batch, self.view[0], self.view[1],
                  _thresh_struct(None, self.t64, self.ge), int(self.flat), _dev.P(self.out), st)


# Dense / Input8 stages use the tensor cores from this many activation rows
# up (measured: even at batch 1 the tcgen05 kernels beat the packed-weight
# GEMV and the bit-plane POPC kernel, BMLP batch-1 latency 115 -> 69 us);
# B2_TC_MIN_ROWS overrides it for comparisons.
TC_MIN_ROWS = int(__import__("os").environ.get("B2_TC_MIN_ROWS", "1"))
# Dense stages below this many rows stream the packed weights on the CUDA
# cores (k_dense_small: all of a unit's K words in flight, 8x fewer bytes
# than the int8 tiles) instead of the tensor cores.
TC_MIN_ROWS_DENSE = int(__import__("os").environ.get("B2_TC_MIN_ROWS_DENSE", "9"))


class _DenseFused(_Stage):
    name = "dense+bn"

    def __init__(self, src, rec, bn_dev):
        super().__init__(src)
        self.rec, self.bn = rec, bn_dev
        self.w = _dev.upload(rec.words)
        self.fmt = _lib.TC_FORMAT
        self.wt = _dev.tc_weights(self.w, rec.units, rec.input_len, self.fmt) if _lib.ENGINE == "tc" else None

    def per_image(self):
        return (_wpl(self.rec.units),)

    def launch(self, net, batch, st):
        r = self.rec
        if self.wt is not None and batch >= max(TC_MIN_ROWS, TC_MIN_ROWS_DENSE):
            _lib.call(_lib.tc_entry("dense_bn_pack", self.fmt), self.src_ptr(net), batch, _dev.P(self.wt), r.units, _wpl(r.input_len),
                      r.input_len, _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]),
                      _dev.P(self.out), st)
            return
        _lib.call("b2_dense_bn_pack", self.src_ptr(net), batch, _dev.P(self.w), r.units, _wpl(r.input_len),
                  r.input_len, _thresh_struct(self.bn["thresh32"], self.bn["thresh64"], self.bn["ge"]),
                  _dev.P(self.out), st)


class _Dense(_Stage):
    name = "dense"
    out_dtype = np.int32

    def __init__(self, src, rec):
        super().__init__(src)
        self.rec = rec
        self.w = _dev.upload(rec.words)
        self.fmt = _lib.TC_FORMAT
        self.wt = _dev.tc_weights(self.w, rec.units, rec.input_len, self.fmt) if _lib.ENGINE == "tc" else None

    def per_image(self):
        return (self.rec.units,)

    def launch(self, net, batch, st):
        r = self.rec
        if self.wt is not None and batch >= max(TC_MIN_ROWS, TC_MIN_ROWS_DENSE):
            _lib.call(_lib.tc_entry("bgemm", self.fmt), self.src_ptr(net), batch, _dev.P(self.wt), r.units, _wpl(r.input_len),
                      r.input_len, _dev.P(self.out), st)
            return
        _lib.call("b2_bgemv", _dev.P(self.w), r.units, _wpl(r.input_len), self.src_ptr(net), batch, r.input_len,
                  _dev.P(self.out), st)


class _DenseFinal(_Stage):
    """_PackedDense -> _FinalBN in one tensor-core launch (network.py:153-162,
    259-270): int32 dot products, then float64 scores in the epilogue."""

    name = "dense+final-bn"
    out_dtype = np.float64

    def __init__(self, src, rec, bn_dev, dense: "_Dense"):
        super().__init__(src)
        self.rec, self.bn = rec, bn_dev
        self.dense = dense  # the unfused pair, for batches below TC_MIN_ROWS
        self.final = _FinalBN(dense, bn_dev, rec.units, XKIND[np.dtype(np.int32)])

    def per_image(self):
        return (self.rec.units,)

    def alloc(self, cap):
        super().alloc(cap)
        self.dense.alloc(cap)
        self.final.out = self.out

    def launches(self):
        return 1

    def launch(self, net, batch, st):
        r = self.rec
        if batch < max(TC_MIN_ROWS, TC_MIN_ROWS_DENSE):
            self.dense.launch(net, batch, st)
            self.final.launch(net, batch, st)
            return
        _lib.call(_lib.tc_entry("dense_affine_f64", self.dense.fmt), self.src_ptr(net), batch, _dev.P(self.dense.wt), r.units,
                  _wpl(r.input_len), r.input_len, _dev.P(self.bn["mean64"]), _dev.P(self.bn["scale64"]),
                  _dev.P(self.bn["beta64"]), self.out_ptr(net), st)


class _FinalBN(_Stage):
    name = "final-bn"
    out_dtype = np.float64

    def __init__(self, src, bn_dev, classes: int, xkind: int):
        super().__init__(src)
        self.bn, self.classes, self.xkind = bn_dev, classes, xkind

    def per_image(self):
        return (self.classes,)

    def launch(self, net, batch, st):
        _lib.call("b2_bn_affine_f64", self.src_ptr(net), self.xkind, batch * self.classes, _dev.P(self.bn["mean64"]),
                  _dev.P(self.bn["scale64"]), _dev.P(self.bn["beta64"]), self.classes, self.out_ptr(net), st)


# --------------------------------------------------------------------------- network


class Network:
    """A model compiled for the GPU.  One instance per thread / stream."""

    def __init__(self, spec: ModelSpec, backend=Backend.PACKED, layer_backends=None, max_batch: int = 1,
                 use_graphs: bool = True):
        if isinstance(backend, str):
            backend = Backend(backend)
        n_compute = sum(1 for r in spec.records if isinstance(r, (Input8Record, DenseRecord, ConvRecord)))
        if layer_backends is None:
            assigned = [backend] * n_compute
        else:
            assigned = [Backend(b) if isinstance(b, str) else b for b in layer_backends]
            if len(assigned) != n_compute:
                raise ModelValidationError(
                    f"layer_backends needs one entry per weight layer ({n_compute}), got {len(assigned)}")
        if any(b != Backend.PACKED for b in assigned):
            raise NotImplementedError("only the packed backend exists on the GPU; the float reference backend "
                                      "and hybrid mixes are out of scope (see DESIGN.md)")
        self.spec = spec
        self.input_dims = tuple(spec.input_dims)
        self.backend = Backend.PACKED
        self.layer_backends = assigned
        self.use_graphs = use_graphs
        ops, self.classes = self._validate(spec)
        _dev.require_cuda()
        self.device = _dev.device()
        self.stages = self._plan(ops)
        # the batch-1 graph reads the image from, and writes the scores to,
        # pinned host memory directly (mapped, UVA) when the last stage is a
        # float64 score stage: no H2D / D2H nodes on the latency path
        self._io_ptrs = None
        self._pipe_split = None  # H2D share of the per-image host->scores time (measured on first use)
        last = self.stages[-1]
        self._zero_copy_out = isinstance(last, (_FinalBN, _DenseFinal))
        if self._zero_copy_out:
            last.is_last = True
            if isinstance(last, _DenseFinal):
                last.final.is_last = True
        self.cap = 0
        self._graphs = {}
        self._copy_stream = None
        self._reserve(max(1, int(max_batch)))
        self._scores1 = None

    # -- validation: network.py:331-486, same checks in the same order --------

    def _validate(self, spec):
        recs = spec.records
        if not recs:
            raise ModelValidationError("model has no layers")
        if not isinstance(recs[-1], BatchNormRecord):
            raise ModelValidationError(f"layer {len(recs) - 1}: model must end with a batchnorm score layer")
        for i, r in enumerate(recs):
            if isinstance(r, BatchNormRecord):
                _check_bn_params(r, i)
        ops = []
        rep, shape = "bytes", self.input_dims
        acc_kind = None

        def consumer(i):
            return recs[i + 1] if i + 1 < len(recs) else None

        def want_flat(i):
            return isinstance(consumer(i), (DenseRecord, Input8Record))

        for i, rec in enumerate(recs):
            last = i == len(recs) - 1
            if isinstance(rec, Input8Record):
                if i != 0:
                    raise ModelValidationError(f"layer {i}: input8 is only valid as the first layer")
                h, w, c = shape
                if rec.input_len != h * w * c:
                    raise ModelValidationError(
                        f"layer {i}: input8 expects {rec.input_len} bytes but input dims give {h * w * c}")
                ops.append(dict(kind="input8", rec=rec, i=i))
                rep, shape, acc_kind = "acc", (1, 1, rec.units), ("input8", rec.input_len)
            elif isinstance(rec, DenseRecord):
                if rep not in ("packed", "float"):
                    raise ModelValidationError(f"layer {i}: dense layer needs a signed activation input")
                h, w, c = shape
                if rec.input_len != h * w * c:
                    raise ModelValidationError(
                        f"layer {i}: dense expects {rec.input_len} inputs, previous layer gives {h * w * c}")
                if h * w != 1:
                    raise ModelValidationError(f"layer {i}: dense needs a flat activation line")
                ops.append(dict(kind="dense", rec=rec, i=i))
                rep, shape, acc_kind = "acc", (1, 1, rec.units), ("binary", rec.input_len)
            elif isinstance(rec, ConvRecord):
                if rep not in ("packed", "float") or shape[0] * shape[1] == 1:
                    raise ModelValidationError(f"layer {i}: conv needs a spatial signed activation input")
                h, w, c = shape
                if c != rec.in_channels:
                    raise ModelValidationError(
                        f"layer {i}: conv expects {rec.in_channels} channels, previous layer gives {c}")
                if h + 2 * rec.pad < rec.kh or w + 2 * rec.pad < rec.kw:
                    raise ModelValidationError(f"layer {i}: kernel {rec.kh}x{rec.kw} larger than padded input")
                if rec.k > MAX_K:
                    raise ModelValidationError(f"layer {i}: dot length {rec.k} over limit {MAX_K}")
                h_out = (h + 2 * rec.pad - rec.kh) // rec.stride + 1
                w_out = (w + 2 * rec.pad - rec.kw) // rec.stride + 1
                ops.append(dict(kind="conv", rec=rec, i=i, in_shape=shape, out_shape=(h_out, w_out, rec.filters)))
                rep, shape, acc_kind = "acc", (h_out, w_out, rec.filters), ("binary", rec.k)
            elif isinstance(rec, MaxPoolRecord):
                if rep != "acc" or shape[0] * shape[1] == 1:
                    raise ModelValidationError(f"layer {i}: maxpool needs spatial integer accumulators")
                h, w, c = shape
                if h < rec.ph or w < rec.pw:
                    raise ModelValidationError(f"layer {i}: pooling window {rec.ph}x{rec.pw} larger than {h}x{w}")
                out = ((h - rec.ph) // rec.stride + 1, (w - rec.pw) // rec.stride + 1, c)
                ops.append(dict(kind="pool", rec=rec, i=i, in_shape=shape, out_shape=out))
                shape = out
            elif isinstance(rec, BatchNormRecord):
                if i == 0:
                    h, w, c = shape
                    if rec.channels != c:
                        raise ModelValidationError(f"layer {i}: batchnorm has {rec.channels} channels, input has {c}")
                    if last:
                        raise ModelValidationError("layer 0: model cannot be a lone batchnorm")
                    flat = want_flat(i)
                    ops.append(dict(kind="bytebn", rec=rec, i=i, dims=shape, flat=flat))
                    rep = "packed"
                    if flat:
                        shape = (1, 1, h * w * c)
                    continue
                if rep != "acc":
                    raise ModelValidationError(f"layer {i}: batchnorm needs accumulator input")
                if rec.channels != shape[2]:
                    raise ModelValidationError(
                        f"layer {i}: batchnorm has {rec.channels} channels, previous layer gives {shape[2]}")
                if last:
                    if shape[0] * shape[1] != 1:
                        raise ModelValidationError(f"layer {i}: final batchnorm must see a flat score vector")
                    ops.append(dict(kind="final", rec=rec, i=i, acc=acc_kind))
                    rep = "scores"
                    continue
                if not isinstance(consumer(i), (DenseRecord, ConvRecord)):
                    raise ModelValidationError(f"layer {i}: batchnorm output has no consumer layer")
                flat = want_flat(i)
                ops.append(dict(kind="bn", rec=rec, i=i, dims=shape, flat=flat, acc=acc_kind))
                rep = "packed"
                if flat:
                    shape = (1, 1, shape[0] * shape[1] * shape[2])
            else:
                raise ModelValidationError(f"layer {i}: unknown record {rec!r}")
        if rep != "scores":
            raise ModelValidationError("model does not end in a score-emitting batchnorm")
        return ops, shape[2]

    # -- planning: fuse adjacent reference stages into device kernels ---------

    @staticmethod
    def _bound(acc_kind) -> int:
        kind, k = acc_kind
        return 255 * k if kind == "input8" else k

    def _plan(self, ops):
        stages = []
        src = None
        j = 0
        n = len(ops)

        def cal(op, bound):
            r = op["rec"]
            return calibrate_device(r.mean, r.var, r.gamma, r.beta, r.eps, bound)

        while j < n:
            op = ops[j]
            kind = op["kind"]
            nxt = ops[j + 1] if j + 1 < n else None
            nxt2 = ops[j + 2] if j + 2 < n else None
            if kind == "input8":
                r = op["rec"]
                if nxt["kind"] == "bn" and 2 * _wpl(r.input_len) <= 128:
                    st = _Input8Fused(src, r, cal(nxt, 255 * r.input_len))
                    j += 2
                else:
                    st = _Input8Raw(src, r)
                    j += 1
            elif kind == "bytebn":
                h, w, c = op["dims"]
                conv = nxt if nxt is not None and nxt["kind"] == "conv" else None
                crec = conv["rec"] if conv is not None else None
                tc_ok = _lib.ENGINE == "tc" and crec is not None and crec.k <= 128 and c <= 8
                kmax, fmax = (128, 1 << 30) if tc_ok else (32, 1024)
                if (conv is not None and not op["flat"] and conv["rec"].k <= kmax and 1 < conv["rec"].filters <= fmax
                        and nxt2 is not None and nxt2["kind"] == "bn"
                        and (not nxt2["flat"] or conv["rec"].filters % 64 == 0)):
                    st = _ByteConvFused(src, op["dims"], cal(op, 255), conv["rec"], cal(nxt2, conv["rec"].k))
                    j += 3
                else:
                    st = _BN(src, op["dims"], cal(op, 255), op["flat"], XKIND[np.dtype(np.uint8)])
                    j += 1
            elif kind == "conv":
                r = op["rec"]
                h, w, c = op["in_shape"]
                ho, wo, f = op["out_shape"]
                fusable_in = c % 32 == 0 and f > 1
                pool_ok = (nxt is not None and nxt["kind"] == "pool" and (nxt["rec"].ph, nxt["rec"].pw,
                                                                          nxt["rec"].stride) == (2, 2, 2)
                           and ho % 2 == 0 and wo % 2 == 0 and nxt2 is not None and nxt2["kind"] == "bn")
                if fusable_in and nxt is not None and nxt["kind"] == "bn" and (not nxt["flat"] or f % 64 == 0):
                    st = _ConvFused(src, op["in_shape"], r, False, cal(nxt, r.k))
                    j += 2
                elif fusable_in and pool_ok and (not nxt2["flat"] or f % 64 == 0):
                    st = _ConvFused(src, op["in_shape"], r, True, cal(nxt2, r.k))
                    j += 3
                else:
                    st = _Conv(src, op["in_shape"], r)
                    j += 1
            elif kind == "pool":
                st = _Pool(src, op["in_shape"], op["rec"])
                j += 1
            elif kind == "bn":
                xk = XKIND[np.dtype(np.int64 if op["acc"][0] == "input8" else np.int32)]
                st = _BN(src, op["dims"], cal(op, self._bound(op["acc"])), op["flat"], xk)
                j += 1
            elif kind == "dense":
                r = op["rec"]
                if nxt["kind"] == "bn":
                    st = _DenseFused(src, r, cal(nxt, r.input_len))
                    j += 2
                elif nxt["kind"] == "final" and _lib.ENGINE == "tc":
                    dense = _Dense(src, r)
                    st = _DenseFinal(src, r, cal(nxt, 0), dense)
                    dense.src = src
                    j += 2
                else:
                    st = _Dense(src, r)
                    j += 1
            elif kind == "final":
                xk = XKIND[np.dtype(np.int64 if op["acc"][0] == "input8" else np.int32)]
                st = _FinalBN(src, cal(op, 0), op["rec"].channels, xk)
                j += 1
            else:  # pragma: no cover
                raise AssertionError(kind)
            stages.append(st)
            src = st
        return stages

    # -- workspace / execution ---------------------------------------------------

    @property
    def input_len(self) -> int:
        h, w, c = self.input_dims
        return h * w * c

    GROW_LIMIT = 8192  # forward_batch grows a smaller workspace to at most this many images

    def _reserve(self, cap: int):
        if cap <= self.cap:
            return
        self._graphs.clear()
        self._in = _dev.empty((cap, self.input_len), np.uint8)
        for st in self.stages:
            st.alloc(cap)
        self._in_host = torch.empty((cap, self.input_len), dtype=torch.uint8, pin_memory=True)
        self._out_host = torch.empty((cap, self.classes), dtype=torch.float64, pin_memory=True)
        self._in_host_np = self._in_host.numpy()
        self._out_host_np = self._out_host.numpy()
        # H2D staging for the pipelined host path (forward_host), allocated
        # with the workspace so a forward pass allocates nothing
        self._copy_stream = torch.cuda.Stream()
        self._staged = [torch.empty_like(self._in), torch.empty_like(self._in)]
        self.cap = cap
        self._scores1 = None

    @property
    def scores_device(self):
        return self.stages[-1].out

    @property
    def input_device(self):
        return self._in

    @property
    def workspace_bytes(self) -> int:
        tot = self._in.numel()
        for st in self.stages:
            for t in (st.out, getattr(st, "planes", None), getattr(st, "scratch", None)):
                if t is not None:
                    tot += t.numel() * t.element_size()
        return tot

    def launches_per_forward(self) -> int:
        return sum(st.launches() for st in self.stages)

    def _launch_all(self, batch: int):
        st = _dev.stream()
        for s in self.stages:
            s.launch(self, batch, st)

    def run(self, batch: int):
        """Enqueue the forward pass of the first `batch` images already in
        `input_device` on the current stream (scores land in `scores_device`)."""
        if batch > self.cap:
            raise ValueError(f"batch {batch} exceeds workspace capacity {self.cap}")
        if batch <= 0:
            return
        if not self.use_graphs:
            self._launch_all(batch)
            return
        g = self._graphs.get(batch)
        if g is None:
            self._launch_all(batch)  # eager warm-up (module load, attributes)
            torch.cuda.current_stream().synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch_all(batch)
            self._graphs[batch] = g
        g.replay()

    def forward_host(self, images: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """(N, input_len) uint8 host images -> (N, classes) float64 scores.

        Pipelined in chunks: the host copy of chunk i+1 into pinned staging
        (multi-threaded) and its H2D copy (side stream) overlap the forward
        pass of chunk i; each chunk's scores come back with one D2H."""
        n = images.shape[0]
        if out is None:
            out = np.empty((n, self.classes), dtype=np.float64)
        if n > self.cap and self.cap < self.GROW_LIMIT:
            # a workspace built for fewer images (load() defaults to one) would
            # run the batch block by block like the reference's per-image loop:
            # grow it once, up to GROW_LIMIT images
            self._reserve(min(n, self.GROW_LIMIT))
        for s0 in range(0, n, self.cap):
            self._forward_host_block(images[s0:s0 + self.cap], out[s0:s0 + self.cap])
        return out

    def pinned_images(self, n: int) -> np.ndarray:
        """A page-locked (n, input_len) uint8 host array: forward_batch copies
        from it straight to the device (no staging copy on the host)."""
        # the array's base keeps the pinned tensor (and its allocation) alive
        return torch.empty((int(n), self.input_len), dtype=torch.uint8, pin_memory=True).numpy()

    def pinned_scores(self, n: int) -> np.ndarray:
        """A page-locked (n, classes) float64 host array: passed as
        forward_batch's `out`, the scores are copied straight into it."""
        return torch.empty((int(n), self.classes), dtype=torch.float64, pin_memory=True).numpy()

    def _chunk_plan(self, n: int, pinned: bool) -> list:
        """Chunks of the pipelined host path.

        Pinned input (one graph per call): two chunks.  The first chunk's H2D
        cannot overlap anything, and the second chunk's H2D must hide under
        the first chunk's forward pass, so the first chunk is the smallest
        multiple of 512 with c0 >= n * h / (h + t) (h, t = H2D and compute
        time per image, measured once per network; n/8 until then).  More,
        smaller chunks lose more to per-pass inefficiency than they gain.
        Staged input: equal chunks that fit half the pinned workspace."""
        if pinned:
            f = self._pipe_split if self._pipe_split is not None else 0.125
            # chunk i+1's H2D hides under chunk i's pass when c_{i+1} <= r c_i
            # (r = compute / H2D time per image), so the sizes grow
            # geometrically and only the first, smallest chunk's H2D is
            # exposed; three chunks when the first stays >= 2048 images
            # (two chunks exposed ~5 % of a 65536-image BCNN call)
            r = (1.0 - f) / max(f, 1e-3)
            if r > 1.0 and n * 1.0 / (1.0 + r + r * r) >= 2048:
                c0 = max(512, -(-int(n / (1.0 + r + r * r)) // 512) * 512)
                c1 = max(512, int(c0 * r) // 512 * 512)
                if c0 + c1 + 512 <= n:
                    return [(0, c0), (c0, c1), (c0 + c1, n - c0 - c1)]
            c0 = max(512, -(-int(n * f) // 512) * 512)
            return [(0, c0), (c0, n - c0)] if n - c0 >= 512 else [(0, n)]
        ck = self.cap if self.cap < 2048 else max(1024, self.cap // 4)
        return [(b0, min(ck, n - b0)) for b0 in range(0, n, ck)]

    def _measure_pipe_split(self, n: int, src: torch.Tensor):
        """h / (h + t) from one timed H2D of the call's input and one timed
        forward pass over it (CUDA events, after a warm-up pass)."""
        cur = torch.cuda.current_stream()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        self._launch_all(n)
        e[0].record(cur)
        self._in[:n].copy_(src[:n], non_blocking=True)
        e[1].record(cur)
        self._launch_all(n)
        e[2].record(cur)
        cur.synchronize()
        h, t = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
        self._pipe_split = min(0.5, max(0.0, h / max(h + t, 1e-9)))

    _PIPE_GRAPHS = 2  # pointer-keyed whole-call graphs kept per network

    def _pipe_graph(self, n: int, src: torch.Tensor, dst: torch.Tensor | None):
        """One CUDA graph for a whole pipelined call on pinned input: the
        copy stream forks and copies every chunk straight into its rows of
        the workspace; the compute stream waits per chunk, runs the stages on
        row-offset input pointers and copies the chunk's scores into the
        pinned output (`dst`, else the pinned workspace).  No host work
        between chunks.  None when the plan has a single chunk."""
        key = ("pipe", n, src.data_ptr(), 0 if dst is None else dst.data_ptr())
        g = self._graphs.get(key)
        if g is not None:
            return g
        if self._pipe_split is None:
            self._measure_pipe_split(n, src)
        chunks = self._chunk_plan(n, True)
        if len(chunks) < 2:
            return None
        for _, b in chunks:  # eager warm-up of every chunk size (lazy module / attribute work)
            self._launch_all(b)
        torch.cuda.current_stream().synchronize()
        old = [k for k in self._graphs if isinstance(k, tuple) and k[0] == "pipe"]
        for k in old[:max(0, len(old) - self._PIPE_GRAPHS + 1)]:
            del self._graphs[k]
        L = self.input_len
        sink = dst if dst is not None else self._out_host
        ready = [torch.cuda.Event() for _ in chunks]
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g):
                cap = torch.cuda.current_stream()
                self._copy_stream.wait_stream(cap)
                with torch.cuda.stream(self._copy_stream):
                    for i, (b0, b) in enumerate(chunks):
                        self._in[b0:b0 + b].copy_(src[b0:b0 + b], non_blocking=True)
                        ready[i].record(self._copy_stream)
                for i, (b0, b) in enumerate(chunks):
                    cap.wait_event(ready[i])
                    self._io_ptrs = (ctypes.c_void_p(self._in.data_ptr() + b0 * L), None)
                    self._launch_all(b)
                    # a D2H node per chunk: at large batch, score kernels
                    # writing host memory directly are slower (measured)
                    sink[b0:b0 + b].copy_(self.scores_device[:b], non_blocking=True)
                cap.wait_stream(self._copy_stream)
        finally:
            self._io_ptrs = None
        self._graphs[key] = g
        return g

    def _forward_host_block(self, images: np.ndarray, out: np.ndarray):
        n = images.shape[0]
        if n == 0:
            return
        compute = torch.cuda.current_stream()
        src = torch.from_numpy(images) if images.flags.c_contiguous else None
        pinned = src is not None and src.is_pinned()  # caller's page-locked memory: no host staging copy
        dst = torch.from_numpy(out) if out.flags.c_contiguous else None
        direct_out = dst is not None and dst.is_pinned()  # D2H straight into the caller's buffer
        if pinned and self.use_graphs and n >= 1024:
            g = self._pipe_graph(n, src, dst if direct_out else None)
            if g is not None:
                g.replay()
                compute.synchronize()
                if not direct_out:
                    _parallel_copy(out[:n], self._out_host_np[:n])
                return
        chunks = self._chunk_plan(n, pinned)
        half = self.cap // 2 if len(chunks) > 1 else 0  # pinned rows of slot 1
        h2d_done = [torch.cuda.Event() for _ in chunks]   # staging buffer filled
        consumed = [torch.cuda.Event() for _ in chunks]   # staging buffer copied into the workspace
        d2h_done = [torch.cuda.Event() for _ in chunks]   # chunk scores in pinned memory

        def stage(i):
            b0, b = chunks[i]
            sl = i % 2
            if pinned:
                host = src[b0:b0 + b]
            else:
                if i >= 2:
                    h2d_done[i - 2].synchronize()  # the H2D that read this pinned slot has finished
                pin = slice(sl * half, sl * half + b)
                _parallel_copy(self._in_host_np[pin], images[b0:b0 + b])
                host = self._in_host[pin]
            with torch.cuda.stream(self._copy_stream):
                if i >= 2:
                    self._copy_stream.wait_event(consumed[i - 2])
                self._staged[sl][:b].copy_(host, non_blocking=True)
                h2d_done[i].record(self._copy_stream)

        def collect(i):  # host copy of chunk i's scores (not for a pinned `out`)
            b0, b = chunks[i]
            d2h_done[i].synchronize()
            out[b0:b0 + b] = self._out_host_np[b0:b0 + b]

        stage(0)
        for i, (b0, b) in enumerate(chunks):
            compute.wait_event(h2d_done[i])
            self._in[:b].copy_(self._staged[i % 2][:b], non_blocking=True)
            consumed[i].record(compute)
            self.run(b)
            (dst if direct_out else self._out_host)[b0:b0 + b].copy_(self.scores_device[:b], non_blocking=True)
            d2h_done[i].record(compute)
            if i + 1 < len(chunks):
                stage(i + 1)  # host work overlaps the forward pass just enqueued
            if not direct_out and i >= 1:
                collect(i - 1)  # overlaps the forward pass of chunk i
        compute.synchronize()
        if not direct_out:
            collect(len(chunks) - 1)


_COPY_POOL = None


def _parallel_copy(dst: np.ndarray, src: np.ndarray, min_bytes: int = 1 << 22):
    """dst[...] = src with several host threads for large copies (numpy
    releases the GIL while copying)."""
    global _COPY_POOL
    if dst.nbytes < min_bytes:
        np.copyto(dst, src)
        return
    import concurrent.futures
    import os
    if _COPY_POOL is None:
        _COPY_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    parts = _COPY_POOL._max_workers
    step = -(-dst.shape[0] // parts)
    futs = [_COPY_POOL.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, dst.shape[0], step)]
    for f in futs:
        f.result()


def _check_bn_params(r: BatchNormRecord, i: int):
    """BatchNormLayer.__init__ checks (layers.py:119-130), raised as the reference's ValueError."""
    mean, var, gamma, beta = (np.atleast_1d(np.asarray(v, dtype=np.float32)) for v in (r.mean, r.var, r.gamma,
                                                                                      r.beta))
    if not (mean.shape == var.shape == gamma.shape == beta.shape) or mean.ndim != 1:
        raise ValueError("batchnorm parameter vectors must share one length")
    if np.any(var < 0):
        raise ValueError("negative variance")
    if r.eps < 0:
        raise ValueError("negative epsilon")
    if np.any(var.astype(np.float64) + r.eps <= 0):
        raise ValueError("variance + epsilon must be positive")
    if not all(np.all(np.isfinite(v)) for v in (mean, var, gamma, beta)):
        raise ValueError("non-finite batchnorm parameter")


def load(path, backend=Backend.PACKED, layer_backends=None, max_batch: int = 1) -> Network:
    return Network(load_model(path), backend, layer_backends, max_batch=max_batch)


def _check_image(net: Network, image) -> np.ndarray:
    x = np.asarray(image)
    if x.dtype != np.uint8:
        raise ValueError(f"expected uint8 input, got {x.dtype}")
    h, w, c = net.input_dims
    if x.shape != (h, w, c) and x.shape != (h * w * c,):
        raise ValueError(f"expected input shape {(h, w, c)} or ({h * w * c},), got {x.shape}")
    if not x.flags.c_contiguous:
        raise ValueError("input must be C-contiguous")
    return x


def forward(net: Network, image: np.ndarray) -> np.ndarray:
    """One image -> its float64 score vector.  Like the reference the result
    lives in the network's (pinned host) workspace and is overwritten by the
    next call; the same array object is returned every time."""
    x = _check_image(net, image)
    net._in_host_np[0] = x.reshape(-1)
    if net.use_graphs:
        # one graph per image: the forward pass reading the pinned image and
        # writing the pinned scores (zero-copy), a single launch
        g = net._graphs.get("io1")
        if g is None:
            net.run(1)  # eager warm-up + the batch-1 compute graph
            torch.cuda.current_stream().synchronize()
            g = torch.cuda.CUDAGraph()
            # zero-copy: the first kernel reads the pinned image, the last
            # writes the pinned scores (a memcpy node each costs ~4-6 us)
            zc_in = net.stages[0].zero_copy_in
            net._io_ptrs = (_dev.P(net._in_host) if zc_in else _dev.P(net._in), _dev.P(net._out_host))
            try:
                with torch.cuda.graph(g):
                    if not zc_in:
                        net._in[:1].copy_(net._in_host[:1], non_blocking=True)
                    net._launch_all(1)
                    if not net._zero_copy_out:
                        net._out_host[:1].copy_(net.scores_device[:1], non_blocking=True)
            finally:
                net._io_ptrs = None
            net._graphs["io1"] = g
        g.replay()
    else:
        net._in[:1].copy_(net._in_host[:1], non_blocking=True)
        net.run(1)
        net._out_host[:1].copy_(net.scores_device[:1], non_blocking=True)
    torch.cuda.current_stream().synchronize()
    if net._scores1 is None:
        net._scores1 = net._out_host_np[0]
    return net._scores1


def forward_batch(net: Network, images: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """N images (N, H, W, C) or (N, H*W*C) uint8 -> (N, classes) float64 scores."""
    x = np.asarray(images)
    if x.dtype != np.uint8:
        raise ValueError(f"expected uint8 input, got {x.dtype}")
    h, w, c = net.input_dims
    if x.ndim < 1 or (x.shape[1:] != (h, w, c) and x.shape[1:] != (h * w * c,)):
        raise ValueError(f"expected input shape (N, {h}, {w}, {c}) or (N, {h * w * c}), got {x.shape}")
    x = np.ascontiguousarray(x).reshape(x.shape[0], -1)
    return net.forward_host(x, out)


def classify(net: Network, image: np.ndarray) -> int:
    return int(np.argmax(forward(net, image)))


def classify_batch(net: Network, images: np.ndarray) -> np.ndarray:
    return np.argmax(forward_batch(net, images), axis=1)


def convert(net: Network, target) -> Network:
    if isinstance(target, str):
        target = Backend(target)
    if target != Backend.PACKED:
        raise NotImplementedError("the float reference backend is out of scope on the GPU (see DESIGN.md)")
    return Network(net.spec, Backend.PACKED, max_batch=net.cap)


def serialize(net: Network) -> bytes:
    return write_model(net.spec)


def model_size(obj) -> dict:
    """Serialized parameter bytes per representation (network.py:562-588)."""
    spec = obj.spec if isinstance(obj, Network) else obj
    packed_w = ref_w = bn = 0
    for rec in spec.records:
        if isinstance(rec, (Input8Record, DenseRecord)):
            packed_w += rec.words.nbytes
            ref_w += 4 * rec.units * rec.input_len
        elif isinstance(rec, ConvRecord):
            packed_w += rec.words.nbytes
            ref_w += 4 * rec.filters * rec.k
        elif isinstance(rec, BatchNormRecord):
            bn += 4 * (4 * rec.channels + 1)
    return {"reference": ref_w + bn, "packed": packed_w + bn, "reference_weights": ref_w,
            "packed_weights": packed_w, "batchnorm_bytes": bn}
