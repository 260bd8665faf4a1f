"""Synthetic MNIST-format data for the trainer-export round trip (SURVEY
§8(f)-3).  MNIST itself is not in this image; this is a learnable 10-class
set of 28x28 u8 images (class prototypes of random strokes + noise), written
as IDX files exactly as MNIST ships.  Deterministic from the seed: the golden
generator (tests/golden/make_trainer_golden.py) and the tests build the same
bytes."""

import os
import struct

import numpy as np

N_TRAIN, N_TEST, SEED = 6000, 1000, 1234


def _prototypes(rng):
    protos = np.zeros((10, 28, 28), dtype=np.float64)
    for c in range(10):
        for _ in range(6):  # a few thick random strokes per class
            y0, x0, y1, x1 = rng.integers(4, 24, 4)
            for t in np.linspace(0.0, 1.0, 40):
                y, x = int(round(y0 + t * (y1 - y0))), int(round(x0 + t * (x1 - x0)))
                protos[c, max(0, y - 1):y + 2, max(0, x - 1):x + 2] = 1.0
    return protos


def make_set():
    """(train_x, train_y, test_x, test_y): u8 (n, 28, 28) images, u8 labels."""
    rng = np.random.default_rng(SEED)
    protos = _prototypes(rng)

    def draw(n):
        y = rng.integers(0, 10, n).astype(np.uint8)
        shift = rng.integers(-2, 3, (n, 2))
        x = np.empty((n, 28, 28), dtype=np.uint8)
        for i in range(n):
            img = np.roll(protos[y[i]], tuple(shift[i]), axis=(0, 1)) * rng.uniform(60, 200)
            img = img + rng.normal(0.0, 110.0, (28, 28))
            x[i] = np.clip(img, 0, 255).astype(np.uint8)
        return x, y

    tx, ty = draw(N_TRAIN)
    vx, vy = draw(N_TEST)
    return tx, ty, vx, vy


def write_idx(data_dir, tx, ty, vx, vy):
    os.makedirs(data_dir, exist_ok=True)
    for stem, x, y in (("train", tx, ty), ("t10k", vx, vy)):
        with open(os.path.join(data_dir, f"{stem}-images-idx3-ubyte"), "wb") as fh:
            fh.write(struct.pack(">IIII", 2051, x.shape[0], 28, 28) + x.tobytes())
        with open(os.path.join(data_dir, f"{stem}-labels-idx1-ubyte"), "wb") as fh:
            fh.write(struct.pack(">II", 2049, y.shape[0]) + y.tobytes())
