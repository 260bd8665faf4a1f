"""End-to-end GPU parity: whole networks against the reference's own
scores (golden, bit-exact float64) and against the CPU oracle, plus the
reference's network-level contracts (frozen classes, buffer reuse,
input checks, gamma 0 / negative, single-channel, flat vs shaped)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1705_07175_b200 import classify, forward, forward_batch, load, zoo
from paper_1705_07175_b200.modelfile import (BatchNormRecord, ConvRecord, DenseRecord, Input8Record, MaxPoolRecord,
                                             ModelSpec)
from paper_1705_07175_b200.network import Network

pytestmark = pytest.mark.gpu


def rand_rows(rng, rows, k):
    return zoo.pack_bits_host(rng.random((rows, k)) >= 0.5)


def bn_rec(rng, c, spread=20.0):
    return zoo.rand_bn(rng, c, spread)


def mlp_spec(rng, hidden=32):
    return ModelSpec((1, 1, 784), [Input8Record(hidden, 784, rand_rows(rng, hidden, 784)), bn_rec(rng, hidden, 5000.0),
                                   DenseRecord(10, hidden, rand_rows(rng, 10, hidden)), bn_rec(rng, 10, 4.0)])


def cnn_spec(rng):
    return ModelSpec((16, 16, 3), [
        bn_rec(rng, 3, 100.0), ConvRecord(16, 3, 3, 1, 1, 3, rand_rows(rng, 16, 27)), MaxPoolRecord(2, 2, 2),
        bn_rec(rng, 16, 10.0), ConvRecord(32, 3, 3, 1, 1, 16, rand_rows(rng, 32, 144)), MaxPoolRecord(2, 2, 2),
        bn_rec(rng, 32, 10.0), DenseRecord(64, 512, rand_rows(rng, 64, 512)), bn_rec(rng, 64, 8.0),
        DenseRecord(10, 64, rand_rows(rng, 10, 64)), bn_rec(rng, 10, 4.0)])


def test_fixture_scores_match_reference(networks_golden):
    for name in ("mlp", "cnn"):
        net = load(os.path.join(GOLDEN, f"{name}.bdnn"))
        imgs, want = networks_golden[f"{name}_images"], networks_golden[f"{name}_scores"]
        for i in range(imgs.shape[0]):
            assert np.array_equal(forward(net, imgs[i]), want[i]), (name, i)
        big = load(os.path.join(GOLDEN, f"{name}.bdnn"), max_batch=7)
        assert np.array_equal(forward_batch(big, imgs), want), name


def test_fixture_frozen_classifications(networks_golden):
    mlp = load(os.path.join(GOLDEN, "mlp.bdnn"))
    rng = np.random.default_rng(7)
    assert [classify(mlp, rng.integers(0, 256, 784, dtype=np.uint8)) for _ in range(5)] == [0, 0, 0, 0, 7]
    assert classify(mlp, np.zeros(784, dtype=np.uint8)) == 7
    cnn = load(os.path.join(GOLDEN, "cnn.bdnn"))
    rng = np.random.default_rng(7)
    assert [classify(cnn, rng.integers(0, 256, (32, 32, 3), dtype=np.uint8)) for _ in range(5)] == [5] * 5
    assert classify(cnn, np.zeros((32, 32, 3), dtype=np.uint8)) == 5


@pytest.mark.parametrize("name", ["bmlp", "bcnn"])
def test_baseline_models_match_reference(networks_golden, name):
    spec = getattr(zoo, f"{name}_spec")()
    imgs, want = networks_golden[f"{name}_images"], networks_golden[f"{name}_scores"]
    net = Network(spec, max_batch=imgs.shape[0])
    assert np.array_equal(forward_batch(net, imgs), want)
    one = Network(spec)
    for i in range(3):
        assert np.array_equal(forward(one, imgs[i]), want[i])


@pytest.mark.parametrize("name", ["bmlp", "bcnn"])
def test_baseline_models_large_batch_vs_oracle(oracle, name):
    """Full-size batch through the device path, every 97th image checked
    against the oracle (size-independent sampling of a 2048 batch)."""
    spec = getattr(zoo, f"{name}_spec")()
    onet = oracle.OracleNetwork(spec)
    rng = np.random.default_rng(99)
    shape = (784,) if name == "bmlp" else (32, 32, 3)
    imgs = rng.integers(0, 256, (2048,) + shape, dtype=np.uint8)
    net = Network(spec, max_batch=1024)
    got = forward_batch(net, imgs)
    for i in range(0, 2048, 97):
        assert np.array_equal(got[i], onet.forward(imgs[i])), i
    # chunking-invariance: batch 1024 vs 2 x 512 vs 1
    small = Network(spec, max_batch=512)
    assert np.array_equal(forward_batch(small, imgs[:1024]), got[:1024])


def test_small_models_vs_oracle(oracle):
    rng = np.random.default_rng(30)
    for spec, shape in ((mlp_spec(rng), (784,)), (cnn_spec(rng), (16, 16, 3))):
        onet = oracle.OracleNetwork(spec)
        net = Network(spec, max_batch=50)
        imgs = rng.integers(0, 256, (50,) + shape, dtype=np.uint8)
        got = forward_batch(net, imgs)
        for i in range(50):
            assert np.array_equal(got[i], onet.forward(imgs[i])), i


def test_single_channel_input(oracle):
    # test_network.py:255-268
    rng = np.random.default_rng(32)
    spec = ModelSpec((12, 12, 1), [
        bn_rec(rng, 1, 100.0), ConvRecord(8, 3, 3, 1, 1, 1, rand_rows(rng, 8, 9)), MaxPoolRecord(2, 2, 2),
        bn_rec(rng, 8, 4.0), DenseRecord(10, 288, rand_rows(rng, 10, 288)), bn_rec(rng, 10, 4.0)])
    onet, net = oracle.OracleNetwork(spec), Network(spec, max_batch=30)
    imgs = rng.integers(0, 256, (30, 12, 12, 1), dtype=np.uint8)
    got = forward_batch(net, imgs)
    for i in range(30):
        assert np.array_equal(got[i], onet.forward(imgs[i]))


def test_gamma_zero_and_negative(oracle):
    # test_network.py:300-317
    rng = np.random.default_rng(36)
    spec = mlp_spec(rng)
    bn1 = spec.records[1]
    gamma, beta = bn1.gamma.copy(), bn1.beta.copy()
    gamma[0] = 0.0
    gamma[1] = -abs(gamma[1])
    gamma[2] = 0.0
    beta[2] = -0.25
    spec = ModelSpec(spec.input_dims, [spec.records[0], BatchNormRecord(bn1.mean, bn1.var, gamma, beta, bn1.eps),
                                       spec.records[2], spec.records[3]])
    onet, net = oracle.OracleNetwork(spec), Network(spec, max_batch=30)
    imgs = rng.integers(0, 256, (30, 784), dtype=np.uint8)
    got = forward_batch(net, imgs)
    for i in range(30):
        assert np.array_equal(got[i], onet.forward(imgs[i]))


def test_unfused_general_paths(oracle):
    """Shapes that take the general kernels: C % 32 != 0 convs, stride 2,
    3x2 pooling, flat BN with C % 64 != 0, conv -> pool -> bn -> conv."""
    rng = np.random.default_rng(77)
    spec = ModelSpec((11, 9, 5), [
        bn_rec(rng, 5, 100.0), ConvRecord(20, 3, 3, 2, 2, 5, rand_rows(rng, 20, 45)), bn_rec(rng, 20, 6.0),
        ConvRecord(33, 2, 3, 1, 0, 20, rand_rows(rng, 33, 120)), MaxPoolRecord(3, 2, 2), bn_rec(rng, 33, 10.0),
        DenseRecord(70, 132, rand_rows(rng, 70, 132)), bn_rec(rng, 70, 6.0), DenseRecord(7, 70, rand_rows(rng, 7, 70)),
        bn_rec(rng, 7, 3.0)])
    onet, net = oracle.OracleNetwork(spec), Network(spec, max_batch=16)
    imgs = rng.integers(0, 256, (16, 11, 9, 5), dtype=np.uint8)
    got = forward_batch(net, imgs)
    for i in range(16):
        assert np.array_equal(got[i], onet.forward(imgs[i])), i


def test_input8_to_final_bn(oracle):
    # beta_only_spec of test_network.py:354-373 (input8 straight into the score layer)
    n = 3
    z = np.zeros(n, np.float32)
    for beta, want in (([0.1, 0.9, 0.3], 1), ([0.5, 0.5, 0.1], 0)):
        spec = ModelSpec((1, 1, 64), [Input8Record(n, 64, zoo.pack_bits_host(np.ones((n, 64), bool))),
                                      BatchNormRecord(z, z + 1, z + 1, np.asarray(beta, np.float32), 0.0)])
        assert classify(Network(spec), np.zeros(64, dtype=np.uint8)) == want


def test_forward_contracts():
    rng = np.random.default_rng(38)
    net = Network(mlp_spec(rng))
    with pytest.raises(ValueError, match="uint8"):
        forward(net, np.zeros(784, dtype=np.float32))
    with pytest.raises(ValueError, match="shape"):
        forward(net, np.zeros(783, dtype=np.uint8))
    with pytest.raises(ValueError, match="contiguous"):
        forward(net, np.zeros(1568, dtype=np.uint8)[::2])
    a, b = (rng.integers(0, 256, 784, dtype=np.uint8) for _ in range(2))
    s = forward(net, a)
    kept = s.copy()
    assert forward(net, b) is s
    assert not np.array_equal(kept, s)
    cs = cnn_spec(rng)
    cnet = Network(cs)
    img = rng.integers(0, 256, (16, 16, 3), dtype=np.uint8)
    assert np.array_equal(forward(cnet, img).copy(), forward(cnet, img.reshape(-1)))


def test_no_allocation_in_forward():
    import torch
    rng = np.random.default_rng(48)
    net = Network(cnn_spec(rng), max_batch=8)
    imgs = rng.integers(0, 256, (8, 16, 16, 3), dtype=np.uint8)
    forward_batch(net, imgs)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    for _ in range(5):
        forward_batch(net, imgs)
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == before


def test_no_allocation_in_forward_bcnn_timed_kernels():
    """The bench's kernels (fused first layer, row-aligned padded-row conv
    with the pool fused, im2col convs, dense) allocate nothing per call: the
    torch allocator, the device's free memory and the device's default CUDA
    memory pool (what cudaMallocAsync would draw from) all stay put."""
    import torch
    from cuda.bindings import runtime as rt
    from paper_1705_07175_b200 import _lib
    assert _lib._so.b2_tc4_conv_path(64, 32, 32, 128, 128, 3, 3, 1, 1, 1) == 3
    assert _lib._so.b2_tc_byte_conv_path(64, 32, 32, 3, 128, 3, 3, 1, 1, 0) == 1
    net = Network(zoo.bcnn_spec(), max_batch=64)
    imgs = np.random.default_rng(3).integers(0, 256, (64, 32, 32, 3), dtype=np.uint8)
    err, dev = rt.cudaGetDevice()
    err, pool = rt.cudaDeviceGetDefaultMemPool(dev)

    def pool_reserved():
        err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh)
        return int(v)

    # the high watermark is reset first, so earlier tests in the process that
    # used the stream-ordered pool do not count (order independence)
    torch.cuda.synchronize()
    from cuda.bindings import driver as cu_driver
    rt.cudaMemPoolSetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh, cu_driver.cuuint64_t(0))
    base = pool_reserved()
    forward_batch(net, imgs)
    torch.cuda.synchronize()
    before = (torch.cuda.memory_allocated(), torch.cuda.mem_get_info()[0], pool_reserved())
    for _ in range(5):
        forward_batch(net, imgs)
        net.run(64)
    torch.cuda.synchronize()
    assert (torch.cuda.memory_allocated(), torch.cuda.mem_get_info()[0], pool_reserved()) == before
    assert before[2] == base  # the network path never grew the stream-ordered pool


def test_forward_batch_grows_small_workspace(networks_golden):
    # load() defaults to max_batch=1; a large forward_batch grows
    # the workspace once instead of running image by image
    net = load(os.path.join(GOLDEN, "cnn.bdnn"))
    assert net.cap == 1
    g = networks_golden
    got = forward_batch(net, g["cnn_images"])
    assert net.cap == min(g["cnn_images"].shape[0], net.GROW_LIMIT)
    assert np.array_equal(got, g["cnn_scores"])
