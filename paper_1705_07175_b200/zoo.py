"""Seeded synthetic models for the BASELINE.json configs.

The recipes follow the reference's fixture conventions
(/root/reference/pkg/tests/fixtures/generate.py:29-41): +/-1 weights from
``rng.random(shape) < 0.5 -> -1``, batchnorm parameters mean = N(0,1)*spread,
var = U[1, 51), gamma, beta = N(0,1), eps = 1e-5, drawn in record order.
tests/golden/make_golden.py builds the same specs with the reference's
own classes; the serialized bytes hash identically (test_zoo_hashes).
Weights are packed on the host with numpy (LSB-first words), so specs can
be built without a GPU.
"""

from __future__ import annotations

import numpy as np

from .modelfile import BatchNormRecord, ConvRecord, DenseRecord, Input8Record, MaxPoolRecord, ModelSpec


def pack_bits_host(bits: np.ndarray) -> np.ndarray:
    """(rows, k) bool -> (rows, ceil(k/64)) uint64, LSB-first, zero padding."""
    rows, k = bits.shape
    wpl = -(-k // 64)
    by = np.packbits(bits.astype(np.uint8), axis=1, bitorder="little")
    buf = np.zeros((rows, wpl * 8), dtype=np.uint8)
    buf[:, :by.shape[1]] = by
    return buf.view("<u8").astype(np.uint64)


def rand_rows(rng, rows: int, k: int) -> np.ndarray:
    # +1 (bit 1) iff rng.random() >= 0.5, exactly as np.where(r < 0.5, -1, 1)
    return pack_bits_host(rng.random((rows, k)) >= 0.5)


def rand_bn(rng, c: int, spread: float) -> BatchNormRecord:
    return BatchNormRecord(
        (rng.standard_normal(c) * spread).astype(np.float32),
        (rng.random(c) * 50 + 1).astype(np.float32),
        rng.standard_normal(c).astype(np.float32),
        rng.standard_normal(c).astype(np.float32),
        1e-5,
    )


def bmlp_spec(seed: int = 0x784) -> ModelSpec:
    """BinaryNet MLP 784-4096-4096-4096-10 on MNIST-shaped bytes (BASELINE config 1)."""
    rng = np.random.default_rng(seed)
    return ModelSpec((1, 1, 784), [
        Input8Record(4096, 784, rand_rows(rng, 4096, 784)), rand_bn(rng, 4096, 5000.0),
        DenseRecord(4096, 4096, rand_rows(rng, 4096, 4096)), rand_bn(rng, 4096, 60.0),
        DenseRecord(4096, 4096, rand_rows(rng, 4096, 4096)), rand_bn(rng, 4096, 60.0),
        DenseRecord(10, 4096, rand_rows(rng, 10, 4096)), rand_bn(rng, 10, 4.0),
    ])


def bcnn_spec(seed: int = 0x1705) -> ModelSpec:
    """VGG-style BCNN 2x128C3-MP2-2x256C3-MP2-2x512C3-MP2-1024FC-1024FC-10
    on 32x32x3 bytes (BASELINE config 2)."""
    rng = np.random.default_rng(seed)
    return ModelSpec((32, 32, 3), [
        rand_bn(rng, 3, 100.0),
        ConvRecord(128, 3, 3, 1, 1, 3, rand_rows(rng, 128, 27)), rand_bn(rng, 128, 8.0),
        ConvRecord(128, 3, 3, 1, 1, 128, rand_rows(rng, 128, 1152)), MaxPoolRecord(2, 2, 2), rand_bn(rng, 128, 40.0),
        ConvRecord(256, 3, 3, 1, 1, 128, rand_rows(rng, 256, 1152)), rand_bn(rng, 256, 30.0),
        ConvRecord(256, 3, 3, 1, 1, 256, rand_rows(rng, 256, 2304)), MaxPoolRecord(2, 2, 2), rand_bn(rng, 256, 60.0),
        ConvRecord(512, 3, 3, 1, 1, 256, rand_rows(rng, 512, 2304)), rand_bn(rng, 512, 45.0),
        ConvRecord(512, 3, 3, 1, 1, 512, rand_rows(rng, 512, 4608)), MaxPoolRecord(2, 2, 2), rand_bn(rng, 512, 80.0),
        DenseRecord(1024, 8192, rand_rows(rng, 1024, 8192)), rand_bn(rng, 1024, 80.0),
        DenseRecord(1024, 1024, rand_rows(rng, 1024, 1024)), rand_bn(rng, 1024, 30.0),
        DenseRecord(10, 1024, rand_rows(rng, 10, 1024)), rand_bn(rng, 10, 4.0),
    ])


# Algorithmic work per image (binary MACs; 1 MAC = 2 bit-ops), SURVEY.md §8(d)
def macs_per_image(spec: ModelSpec) -> int:
    h, w, c = spec.input_dims
    shape = (h, w, c)
    macs = 0
    for r in spec.records:
        if isinstance(r, Input8Record):
            macs += r.units * r.input_len * 8  # counted as 8 bit-planes
            shape = (1, 1, r.units)
        elif isinstance(r, DenseRecord):
            macs += r.units * r.input_len
            shape = (1, 1, r.units)
        elif isinstance(r, ConvRecord):
            hh, ww, _ = shape
            ho = (hh + 2 * r.pad - r.kh) // r.stride + 1
            wo = (ww + 2 * r.pad - r.kw) // r.stride + 1
            macs += ho * wo * r.filters * r.k
            shape = (ho, wo, r.filters)
        elif isinstance(r, MaxPoolRecord):
            hh, ww, cc = shape
            shape = ((hh - r.ph) // r.stride + 1, (ww - r.pw) // r.stride + 1, cc)
    return macs
