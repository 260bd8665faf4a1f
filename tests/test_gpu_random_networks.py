"""Randomized whole-network parity: seeded random binarized CNN / MLP
architectures go through the planner and every device path it picks
(tensor-core convs with 64-256 filters, 128- and 256-column tiles, fused
2x2 pools, unfused pools with other windows, byte-BN first convs with
3x3 / 5x5 windows, dense heads with and without the fused final
batch-norm, gamma = 0 and gamma < 0 channels) and must reproduce the CPU
oracle's float64 scores bit for bit, at batch 1 and in a batch."""

import numpy as np
import pytest

from paper_1705_07175_b200 import forward, forward_batch, zoo
from paper_1705_07175_b200.modelfile import (BatchNormRecord, ConvRecord, DenseRecord, Input8Record, MaxPoolRecord,
                                             ModelSpec)
from paper_1705_07175_b200.network import Network

pytestmark = pytest.mark.gpu


def rows(rng, n, k):
    return zoo.pack_bits_host(rng.random((n, k)) >= 0.5)


def bn(rng, c, spread):
    r = zoo.rand_bn(rng, c, spread)
    g = r.gamma.copy()
    g[rng.random(c) < 0.1] = 0.0          # ALWAYS / NEVER sentinels
    flip = rng.random(c) < 0.2
    g[flip] = -np.abs(g[flip])             # reversed comparison direction
    return BatchNormRecord(r.mean, r.var, g, r.beta, r.eps)


def random_cnn(rng):
    h = int(rng.choice([8, 12, 16]))
    c0 = int(rng.choice([1, 3, 4]))
    k0 = int(rng.choice([3, 5])) if c0 <= 3 else 3
    recs = [bn(rng, c0, 100.0)]
    c = int(rng.choice([32, 64, 128]))  # 32: CUDA-core conv kernels even on the tensor-core engine
    recs.append(ConvRecord(c, k0, k0, 1, k0 // 2, c0, rows(rng, c, k0 * k0 * c0)))
    size = h
    for _ in range(int(rng.integers(1, 4))):
        if rng.random() < 0.6 and size % 2 == 0 and size >= 4:
            recs.append(MaxPoolRecord(2, 2, 2))
            size //= 2
        elif rng.random() < 0.2 and size >= 3:
            recs.append(MaxPoolRecord(3, 3, 1))  # unfused pool path
            size -= 2
        recs.append(bn(rng, c, 8.0 * np.sqrt(9 * c) / 10))
        f = int(rng.choice([64, 96, 128, 192, 256]))
        recs.append(ConvRecord(f, 3, 3, 1, 1, c, rows(rng, f, 9 * c)))
        c = f
    if size % 2 == 0 and rng.random() < 0.5:
        recs.append(MaxPoolRecord(2, 2, 2))
        size //= 2
    recs.append(bn(rng, c, 20.0))
    units = int(rng.choice([32, 64, 200]))
    recs += [DenseRecord(units, size * size * c, rows(rng, units, size * size * c)), bn(rng, units, 8.0),
             DenseRecord(10, units, rows(rng, 10, units)), bn(rng, 10, 4.0)]
    return ModelSpec((h, h, c0), recs)


def random_mlp(rng):
    k = int(rng.choice([64, 784, 100]))
    u1 = int(rng.choice([64, 256, 1000]))
    u2 = int(rng.choice([10, 64, 300]))
    recs = [Input8Record(u1, k, rows(rng, u1, k)), bn(rng, u1, 2000.0), DenseRecord(u2, u1, rows(rng, u2, u1)),
            bn(rng, u2, 8.0), DenseRecord(10, u2, rows(rng, 10, u2)), bn(rng, 10, 4.0)]
    return ModelSpec((1, 1, k), recs)


@pytest.mark.parametrize("engine", ["tc", "tc8", "popc"])  # tc: fp4 tensor-core operands, tc8: int8
@pytest.mark.parametrize("seed", range(16))
def test_random_networks_vs_oracle(oracle, seed, engine, monkeypatch):
    from paper_1705_07175_b200 import _lib
    monkeypatch.setattr(_lib, "ENGINE", "tc" if engine == "tc8" else engine)
    monkeypatch.setattr(_lib, "TC_FORMAT", "i8" if engine == "tc8" else "f4")
    rng = np.random.default_rng(9000 + seed)
    spec = random_cnn(rng) if seed % 3 else random_mlp(rng)
    h, w, c = spec.input_dims
    imgs = rng.integers(0, 256, (70, h, w, c), dtype=np.uint8)
    ref = oracle.OracleNetwork(spec)
    want = np.stack([ref.forward(imgs[i]) for i in range(imgs.shape[0])])
    net = Network(spec, max_batch=imgs.shape[0])
    assert np.array_equal(forward_batch(net, imgs), want), [type(r).__name__ for r in spec.records]
    one = Network(spec)
    for i in range(2):
        assert np.array_equal(forward(one, imgs[i]), want[i])
