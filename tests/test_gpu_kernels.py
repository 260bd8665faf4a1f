"""GPU parity of every kernel behind the C ABI against the reference's
golden vectors (bit-exact) and against the CPU oracle on seeded random
inputs, including ragged K, padding edge cases and batched layouts."""

import numpy as np
import pytest

from paper_1705_07175_b200 import _dev, _lib, gemm, layers, tensor
from paper_1705_07175_b200.layers import BatchNormLayer, ConvLayer
from paper_1705_07175_b200.tensor import FloatTensor, PackedTensor, Axis

pytestmark = pytest.mark.gpu


def rand_pm1(rng, *shape):
    return np.where(rng.random(shape) < 0.5, -1.0, 1.0).astype(np.float32)


def test_pack_lines_golden(kernels_golden):
    g = kernels_golden
    assert np.array_equal(tensor.pack_lines(g["pack_in"]), g["pack_out"])


def test_pack_random_vs_oracle(oracle):
    rng = np.random.default_rng(1)
    for bits in (1, 31, 32, 33, 63, 64, 65, 200, 1000):
        x = rng.standard_normal((13, bits)).astype(np.float32)
        x[0, 0] = 0.0
        assert np.array_equal(tensor.pack_lines(x), oracle.pack_lines(x)), bits


def test_unpack_roundtrip():
    rng = np.random.default_rng(7)
    for dims in [(5, 9, 3), (2, 70, 1), (1, 1, 200), (4, 4, 8)]:
        arr = rand_pm1(rng, *dims)
        assert np.array_equal(tensor.unpack(tensor.pack(FloatTensor(arr))).array, arr)


def test_byte_planes_golden(kernels_golden):
    g = kernels_golden
    bp = tensor.bitplanes(g["planes_in"].reshape(5, 70, 1))
    got = np.stack([p.words for p in bp.planes])
    assert np.array_equal(got, g["planes_out"])


def test_bgemm_golden(kernels_golden):
    g = kernels_golden
    for t in range(24):
        a, b, k = g[f"bgemm{t}_a"], g[f"bgemm{t}_b"], int(g[f"bgemm{t}_k"])
        got = gemm.bgemm(gemm.PackedMatrixA(a.shape[0], k, a), gemm.PackedMatrixB(k, b.shape[0], b))
        assert np.array_equal(got, g[f"bgemm{t}_c"]), t


def test_bgemm_acceptance_shapes(oracle):
    # test_acceptance.py:101-115 — 200 random shapes, forced K list
    rng = np.random.default_rng(2024)
    forced = [1, 63, 64, 65, 128, 129, 192, 255, 256, 300]
    for trial in range(200):
        m, n = int(rng.integers(1, 257)), int(rng.integers(1, 257))
        k = forced[trial] if trial < len(forced) else int(rng.integers(1, 301))
        af, bf = rand_pm1(rng, m, k), rand_pm1(rng, k, n)
        got = gemm.bgemm(gemm.PackedMatrixA.from_float(af), gemm.PackedMatrixB.from_float(bf))
        assert np.array_equal(got, (af.astype(np.int64) @ bf.astype(np.int64)).astype(np.int32)), (m, k, n)


def test_bgemm_large_vs_oracle(oracle):
    rng = np.random.default_rng(3)
    for m, n, k in ((1000, 333, 4096), (257, 1024, 1152), (64, 64, 16384)):
        a = oracle.pack_lines(rand_pm1(rng, m, k))
        b = oracle.pack_lines(rand_pm1(rng, n, k))
        got = gemm.bgemm(gemm.PackedMatrixA(m, k, a), gemm.PackedMatrixB(k, n, b))
        assert np.array_equal(got, oracle.bgemm(a, b, k)), (m, n, k)


def test_bdot_and_bgemv():
    rng = np.random.default_rng(2025)
    for k in list(range(1, 66)) + [127, 128, 129, 300]:
        a = rand_pm1(rng, k)
        wa = gemm.PackedMatrixA.from_float(a.reshape(1, -1)).words[0]
        assert gemm.bdot(wa, wa, k) == k
    fa, fx = rand_pm1(rng, 50, 300), rand_pm1(rng, 300)
    x = gemm.PackedMatrixA.from_float(fx.reshape(1, -1)).words[0]
    assert np.array_equal(gemm.bgemv(gemm.PackedMatrixA.from_float(fa), x),
                          (fa.astype(np.int64) @ fx.astype(np.int64)).astype(np.int32))


def test_bitplane_golden(kernels_golden):
    g = kernels_golden
    layer = layers.Input8Layer(gemm.PackedMatrixA(16, 784, g["i8_w"]))
    assert np.array_equal(layers.input8_forward(layer, g["i8_u"]), g["i8_y"])


def test_byte_input_first_layer():
    # test_acceptance.py:133-142 (subset) incl. the 255*64 saturation KAT
    rng = np.random.default_rng(2026)
    for _ in range(50):
        u = rng.integers(0, 256, size=784, dtype=np.uint8)
        w = rand_pm1(rng, 4, 784)
        layer = layers.Input8Layer(gemm.PackedMatrixA.from_float(w))
        assert np.array_equal(layers.input8_forward(layer, u), w.astype(np.int64) @ u.astype(np.int64))
    planes = np.stack([p.words[0] for p in tensor.bitplanes(np.full((1, 1, 64), 255, np.uint8)).planes])
    neg = gemm.PackedMatrixA.from_float(-np.ones((1, 64), np.float32)).words[0]
    assert gemm.bitplane_dot(planes, neg, 64) == -255 * 64


def test_unroll_correction_conv_golden(kernels_golden):
    g = kernels_golden
    for t in range(8):
        h, w, c, kh, kw, s, pad, f = (int(v) for v in g[f"conv{t}_params"])
        x = PackedTensor((h, w, c), Axis.CHANNEL if c > 1 else Axis.COLUMN, g[f"conv{t}_x"], c if c > 1 else w)
        assert np.array_equal(layers.unroll(x, (kh, kw), s, pad).words, g[f"conv{t}_unroll"]), t
        layer = ConvLayer(gemm.PackedMatrixB(kh * kw * c, f, g[f"conv{t}_w"]), (kh, kw), s, pad, (h, w, c))
        assert np.array_equal(layer.correction, g[f"conv{t}_corr"]), t
        assert np.array_equal(layers.conv_forward(layer, x), g[f"conv{t}_out"]), t


def test_padding_correction_acceptance():
    # test_acceptance.py:145-163 — 200 random convs, direct zero-padded oracle
    rng = np.random.default_rng(2027)
    for trial in range(200):
        pad = trial % 3
        stride = int(rng.integers(1, 3))
        kh, kw = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        c = int(rng.choice([1, 2, 3, 4, 8, 16, 32, 64]))
        f = int(rng.integers(1, 9))
        h = int(rng.integers(max(1, kh - 2 * pad), 13))
        w = int(rng.integers(max(1, kw - 2 * pad), 13))
        if h + 2 * pad < kh or w + 2 * pad < kw:
            continue
        x = rand_pm1(rng, h, w, c)
        wf = rand_pm1(rng, kh * kw * c, f)
        layer = ConvLayer.from_float(wf, (kh, kw), stride, pad, (h, w, c))
        got = layers.conv_forward(layer, tensor.pack(FloatTensor(x)))
        xp = np.zeros((h + 2 * pad, w + 2 * pad, c))
        xp[pad:pad + h, pad:pad + w] = x
        ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
        w4 = wf.reshape(kh, kw, c, f).astype(np.float64)
        want = np.zeros((ho, wo, f))
        for i in range(ho):
            for j in range(wo):
                win = xp[i * stride:i * stride + kh, j * stride:j * stride + kw, :]
                want[i, j] = np.tensordot(win, w4, axes=3)
        assert np.array_equal(got.astype(np.float64), want), (h, w, c, kh, kw, stride, pad)


def test_maxpool_golden(kernels_golden):
    g = kernels_golden
    for t in range(4):
        ph, pw, s = (int(v) for v in g[f"pool{t}_params"])
        assert np.array_equal(layers.maxpool_forward(g[f"pool{t}_x"], (ph, pw), s), g[f"pool{t}_out"]), t


def test_calibration_golden(kernels_golden):
    g = kernels_golden
    bn = BatchNormLayer(g["bn_mean"], g["bn_var"], g["bn_gamma"], g["bn_beta"], float(g["bn_eps"]))
    assert np.array_equal(bn.scale64, g["bn_scale"])
    assert np.array_equal(bn.thresh, g["bn_thresh"])
    assert np.array_equal(bn.ge_dir, g["bn_ge"])


def test_threshold_kats():
    # test_layers.py:337-363
    layer = BatchNormLayer([3.0], [4.0], [2.0], [-1.5], eps=0.0)
    assert layer.ge_dir[0] and layer.thresh[0] == 5
    layer = BatchNormLayer([0.0], [1.0], [-1.0], [0.5], eps=0.0)
    assert not layer.ge_dir[0] and layer.thresh[0] == 0
    got = layers.fused_bn_sign(layer, np.array([-2, -1, 0, 1, 2], dtype=np.int32).reshape(1, 5, 1))
    assert [got.bit(0, n, 0) for n in range(5)] == [1, 1, 1, 0, 0]


def test_threshold_pack_golden(kernels_golden):
    g = kernels_golden
    for t in range(5):
        x = g[f"thr{t}_x"]
        c = x.shape[-1]
        bn = BatchNormLayer(np.zeros(c), np.ones(c), np.ones(c), np.zeros(c))
        bn.thresh, bn.ge_dir = g[f"thr{t}_thresh"], g[f"thr{t}_ge"]
        got = layers.fused_bn_sign(bn, x, flat=bool(g[f"thr{t}_flat"]))
        assert np.array_equal(got.words, g[f"thr{t}_out"]), t


def test_bn_affine_golden(kernels_golden):
    g = kernels_golden
    x = _dev.upload(g["aff_x"])
    out = _dev.empty((x.shape[0],), np.float64)
    _lib.call("b2_bn_affine_f64", _dev.P(x), 0, x.shape[0], _dev.P(_dev.upload(g["aff_mean"])),
              _dev.P(_dev.upload(g["aff_scale"])), _dev.P(_dev.upload(g["aff_beta"])), g["aff_mean"].shape[0],
              _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.float64), g["aff_out"])


def test_fused_conv_kernel_vs_oracle(oracle):
    """b2_conv_bn_pack (implicit im2col + correction + [pool] + threshold)
    against oracle unroll -> bgemm -> +corr -> maxpool -> threshold pack."""
    rng = np.random.default_rng(5)
    for (h, w, c, f, pool, batch) in ((8, 8, 128, 128, True, 3), (6, 10, 64, 96, False, 2), (4, 4, 32, 40, True, 5),
                                      (16, 16, 256, 256, True, 2), (8, 8, 512, 64, False, 2)):
        xs = [oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)]
        wt = oracle.pack_lines(rand_pm1(rng, f, 9 * c))
        mean = rng.standard_normal(f) * 20
        bn = BatchNormLayer(mean, rng.random(f) * 5 + 1, rng.standard_normal(f), rng.standard_normal(f))
        corr = oracle.compute_correction(wt, (h, w, c), (3, 3), 1, 1)
        want = []
        for x in xs:
            acc = (oracle.bgemm(oracle.unroll_packed(x, h, w, c, 3, 3, 1, 1), wt, 9 * c) + corr).reshape(h, w, f)
            if pool:
                acc = oracle.maxpool(acc, 2, 2, 2)
            want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn.thresh, bn.ge_dir, False))
        cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
        xd = _dev.upload(np.stack(xs))
        sites = h * w // (4 if pool else 1)
        out = _dev.empty((batch, sites, -(-f // 64)), np.uint64)
        _lib.call("b2_conv_bn_pack", _dev.P(xd), batch, h, w, c, _dev.P(_dev.upload(wt)), f, 3, 3, 1, 1,
                  _dev.P(_dev.upload(corr)), int(pool), layers._thresh_struct(cal["thresh32"], cal["thresh64"],
                                                                              cal["ge"]), _dev.P(out), _dev.stream())
        assert np.array_equal(_dev.download(out, np.uint64), np.stack(want)), (h, w, c, f, pool)


def test_dense_bn_pack_batched_vs_oracle(oracle):
    rng = np.random.default_rng(6)
    for batch, units, k in ((1, 300, 4096), (5, 64, 1000), (37, 1024, 8192), (200, 4096, 4096)):
        x = oracle.pack_lines(rand_pm1(rng, batch, k))
        wt = oracle.pack_lines(rand_pm1(rng, units, k))
        bn = BatchNormLayer(rng.standard_normal(units) * 30, rng.random(units) * 5 + 1, rng.standard_normal(units),
                            rng.standard_normal(units))
        acc = oracle.bgemm(x, wt, k)
        want = np.stack([oracle.threshold_sign_pack(acc[i].reshape(1, -1), bn.thresh, bn.ge_dir, True)[0]
                         for i in range(batch)])
        cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, k)
        out = _dev.empty((batch, -(-units // 64)), np.uint64)
        _lib.call("b2_dense_bn_pack", _dev.P(_dev.upload(x)), batch, _dev.P(_dev.upload(wt)), units, -(-k // 64), k,
                  layers._thresh_struct(cal["thresh32"], cal["thresh64"], cal["ge"]), _dev.P(out), _dev.stream())
        assert np.array_equal(_dev.download(out, np.uint64), want), (batch, units, k)


# the TMA-fed packing kernels (bits % 4 == 0 floats, bits % 16 == 0 bytes):
# whole and partial 1024-float / 512-byte chunks, more chunks than warps in
# flight, NaN / -0.0 / +-inf, against the oracle
@pytest.mark.parametrize("lines,bits", [(1, 4), (3, 1028), (7, 4096), (5, 12), (600, 1024), (2, 8192), (9000, 64)])
def test_pack_lines_tma_vs_oracle(oracle, lines, bits):
    rng = np.random.default_rng(lines * 7 + bits)
    x = rng.standard_normal((lines, bits)).astype(np.float32)
    x.flat[::97] = 0.0
    x.flat[5::101] = -0.0
    x.flat[7::103] = np.nan
    x.flat[9::107] = -np.inf
    assert np.array_equal(tensor.pack_lines(x), oracle.pack_lines(x))


@pytest.mark.parametrize("lines,bits", [(5, 16), (3, 784), (4, 512), (2, 528), (3000, 784), (7, 1024)])
def test_byte_planes_tma_vs_oracle(oracle, lines, bits):
    rng = np.random.default_rng(lines + bits)
    u = rng.integers(0, 256, (lines, bits), dtype=np.uint8)
    wpl = -(-bits // 64)
    out = _dev.empty((8, lines, wpl), np.uint64)
    out.fill_(-1)
    _lib.call("b2_pack_byte_planes", _dev.P(_dev.upload(u)), lines, bits, _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), oracle.pack_byte_planes(u))
