"""Regenerate the inputs of tests/golden/acceptance.npz (written by
make_golden.py from the REFERENCE): the reference acceptance CNN
(/root/reference/pkg/tests/test_acceptance.py:80-98) rebuilt with this
package's record classes from the same rng stream — its bytes must equal the
committed vgg.bdnn — and the seeded image sets, which are not stored."""

import os

import numpy as np

from paper_1705_07175_b200 import zoo
from paper_1705_07175_b200.modelfile import ConvRecord, DenseRecord, MaxPoolRecord, ModelSpec, write_model

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def vgg_like_cnn(rng):
    r, b = zoo.rand_rows, zoo.rand_bn
    return ModelSpec((32, 32, 3), [
        b(rng, 3, 100.0),
        ConvRecord(32, 3, 3, 1, 1, 3, r(rng, 32, 27)), b(rng, 32, 8.0),
        ConvRecord(32, 3, 3, 1, 1, 32, r(rng, 32, 288)), MaxPoolRecord(2, 2, 2), b(rng, 32, 30.0),
        ConvRecord(64, 3, 3, 1, 1, 32, r(rng, 64, 288)), b(rng, 64, 30.0),
        ConvRecord(64, 3, 3, 1, 1, 64, r(rng, 64, 576)), MaxPoolRecord(2, 2, 2), b(rng, 64, 60.0),
        DenseRecord(256, 4096, r(rng, 256, 4096)), b(rng, 256, 20.0),
        DenseRecord(10, 256, r(rng, 10, 256)), b(rng, 10, 4.0),
    ])


def vgg_set():
    """(spec, 1000 images) exactly as test_acceptance.py:166-172 draws them."""
    rng = np.random.default_rng(2028)
    spec = vgg_like_cnn(rng)
    with open(os.path.join(GOLDEN, "vgg.bdnn"), "rb") as fh:
        assert write_model(spec) == fh.read(), "rebuilt acceptance CNN differs from the reference's bytes"
    imgs = np.stack([rng.integers(0, 256, (32, 32, 3), dtype=np.uint8) for _ in range(1000)])
    return spec, imgs


def images1024(name):
    shape = (32, 32, 3) if name == "bcnn" else (784,)
    return np.random.default_rng(4242).integers(0, 256, (1024,) + shape, dtype=np.uint8)
