"""GPU parity of the tensor-core (tcgen05 kind::i8) entry points against the
CPU oracle: plain GEMM (ragged K, tails in M and N, both tile widths),
implicit-im2col convolutions (padding 0-2, stride 1-2, 1x1..5x5, channel
counts 64..512, int32 and fused threshold/pool/pack epilogues), dense,
byte-input first layers, and whole networks with both engines."""

import numpy as np
import pytest

from paper_1705_07175_b200 import _dev, _lib, forward_batch, gemm, layers, zoo
from paper_1705_07175_b200.layers import BatchNormLayer
from paper_1705_07175_b200.network import Network

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["f4", "i8"])
def fmt(request):
    """Tensor-core weight format: kind::mxf4 e2m1 or kind::i8."""
    return request.param


def rand_pm1(rng, *shape):
    return np.where(rng.random(shape) < 0.5, -1.0, 1.0).astype(np.float32)


def rand_bn(rng, c, spread):
    return BatchNormLayer(rng.standard_normal(c) * spread, rng.random(c) * 5 + 1, rng.standard_normal(c),
                          rng.standard_normal(c))


def th(cal):
    return layers._thresh_struct(cal["thresh32"], cal["thresh64"], cal["ge"])


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (5, 3, 63), (128, 128, 128), (129, 127, 129), (300, 200, 300),
                                   (64, 257, 1000), (1000, 333, 4096), (257, 1024, 1152), (100, 64, 16384),
                                   (513, 300, 2304)])
def test_tc_bgemm_vs_oracle(oracle, m, n, k, fmt):
    rng = np.random.default_rng(m * 7 + n * 13 + k)
    a = oracle.pack_lines(rand_pm1(rng, m, k))
    b = oracle.pack_lines(rand_pm1(rng, n, k))
    got = gemm.bgemm_device(_dev.upload(a), m, _dev.upload(b), n, a.shape[1], k, engine="tc", fmt=fmt)
    assert np.array_equal(_dev.download(got, np.int32), oracle.bgemm(a, b, k))


def test_tc_and_popc_engines_agree(fmt):
    rng = np.random.default_rng(11)
    for m, n, k in ((2048, 512, 4608), (777, 129, 65)):
        a = _dev.upload(zoo.pack_bits_host(rng.random((m, k)) >= 0.5))
        b = _dev.upload(zoo.pack_bits_host(rng.random((n, k)) >= 0.5))
        wpl = -(-k // 64)
        tc = _dev.download(gemm.bgemm_device(a, m, b, n, wpl, k, engine="tc", fmt=fmt), np.int32)
        pc = _dev.download(gemm.bgemm_device(a, m, b, n, wpl, k, engine="popc"), np.int32)
        assert np.array_equal(tc, pc), (m, n, k)


CONV_CASES = [  # h, w, c, f, kh, kw, stride, pad, batch
    (8, 8, 128, 128, 3, 3, 1, 1, 3), (6, 10, 64, 96, 3, 3, 1, 1, 2), (16, 16, 256, 256, 3, 3, 1, 1, 2),
    (8, 8, 512, 64, 3, 3, 1, 1, 2), (7, 9, 64, 10, 5, 5, 2, 2, 2), (5, 5, 128, 300, 1, 1, 1, 0, 3),
    (9, 7, 192, 40, 3, 2, 2, 0, 2), (4, 4, 512, 512, 3, 3, 1, 1, 4), (3, 3, 64, 17, 3, 3, 1, 2, 1)]


@pytest.mark.parametrize("h,w,c,f,kh,kw,stride,pad,batch", CONV_CASES)
def test_tc_conv_forward_vs_oracle(oracle, h, w, c, f, kh, kw, stride, pad, batch, fmt):
    rng = np.random.default_rng(h * 31 + c + f)
    xs = np.stack([oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)])
    wt = oracle.pack_lines(rand_pm1(rng, f, kh * kw * c))
    corr = oracle.compute_correction(wt, (h, w, c), (kh, kw), stride, pad)
    ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    want = np.stack([oracle.bgemm(oracle.unroll_packed(x, h, w, c, kh, kw, stride, pad), wt, kh * kw * c) + corr
                     for x in xs]).reshape(batch, ho, wo, f)
    wd = _dev.upload(wt)
    w8 = _dev.tc_weights(wd, f, kh * kw * c, fmt)
    out = _dev.empty((batch, ho, wo, f), np.int32)
    _lib.call(_lib.tc_entry("conv_forward", fmt), _dev.P(_dev.upload(xs)), batch, h, w, c, _dev.P(w8), f, kh, kw, stride, pad,
              _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.int32), want)


# the last five take the cluster split-K path (>= 8 K stages of 512, few
# tiles): ragged N, a 2048-column output, pooled and unpooled
@pytest.mark.parametrize("h,w,c,f,pool,batch", [(8, 8, 128, 128, True, 3), (6, 10, 64, 96, False, 2),
                                                (16, 16, 256, 256, True, 2), (8, 8, 512, 64, False, 2),
                                                (4, 4, 512, 512, True, 5), (32, 32, 128, 128, True, 2),
                                                (6, 6, 64, 200, True, 3),
                                                (4, 4, 512, 512, True, 1), (8, 8, 512, 200, False, 3),
                                                (6, 6, 512, 130, True, 2), (8, 8, 1024, 64, False, 1),
                                                (2, 2, 512, 2048, True, 1),
                                                # fp4 padded-row implicit GEMM (>= 128 x 148 virtual rows,
                                                # <= 128 filters): pooled, unpooled, ragged filter count
                                                (32, 32, 128, 128, True, 20), (16, 16, 128, 64, False, 80),
                                                (8, 8, 128, 100, True, 240),
                                                # ... its 256-column variant (one accumulator, 129-256 filters)
                                                (16, 16, 128, 256, False, 80), (16, 16, 128, 200, True, 80),
                                                # band slots wider than the 16 KB minimum (W > 62): 128- and
                                                # 256-column variants; the widest image whose band the producer
                                                # warps cover (W = 190) and the first one past it (im2col kernel)
                                                (62, 62, 128, 128, False, 6), (64, 64, 128, 128, True, 6),
                                                (16, 64, 128, 200, True, 20), (8, 190, 128, 64, False, 20),
                                                (8, 191, 128, 64, False, 20),
                                                # row-aligned padded-row tiles (pool fused): one image per tile
                                                # at 8x16, four rows at 4x32
                                                (8, 16, 128, 96, True, 160), (4, 32, 128, 128, False, 160),
                                                # >= 148 tiles, even M-tile count: the bias-folded kernel with
                                                # weight stages multicast to CTA pairs (conv4-conv6 shapes)
                                                (16, 16, 256, 256, True, 80), (8, 8, 512, 512, True, 160),
                                                (8, 8, 256, 512, False, 160),
                                                # 129-256 filters as two 128-filter row-aligned launches:
                                                # ragged, pooled, the 129-filter edge
                                                (16, 16, 128, 200, False, 80), (16, 16, 128, 256, True, 80),
                                                (16, 16, 128, 160, True, 80), (16, 16, 128, 129, False, 80)])
def test_tc_conv_bn_pack_vs_oracle(oracle, h, w, c, f, pool, batch, fmt):
    rng = np.random.default_rng(5 + h + c + f)
    xs = [oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)]
    wt = oracle.pack_lines(rand_pm1(rng, f, 9 * c))
    bn = rand_bn(rng, f, 20.0)
    bn.gamma[::7] = 0.0  # ALWAYS / NEVER sentinels
    bn.gamma[3::11] *= -1
    bn = BatchNormLayer(bn.mean, bn.var, bn.gamma, bn.beta)
    corr = oracle.compute_correction(wt, (h, w, c), (3, 3), 1, 1)
    want = []
    for x in xs:
        acc = (oracle.bgemm(oracle.unroll_packed(x, h, w, c, 3, 3, 1, 1), wt, 9 * c) + corr).reshape(h, w, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn.thresh, bn.ge_dir, False))
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
    wd = _dev.upload(wt)
    w8 = _dev.tc_weights(wd, f, 9 * c, fmt)
    sites = h * w // (4 if pool else 1)
    out = _dev.empty((batch, sites, -(-f // 64)), np.uint64)
    _lib.call(_lib.tc_entry("conv_bn_pack", fmt), _dev.P(_dev.upload(np.stack(xs))), batch, h, w, c, _dev.P(w8), f, 3, 3, 1, 1,
              int(pool), th(cal), _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want))


# split-K cases: (1, 300, 4096), (37, 1024, 8192) and the last four (a
# partial last K stage, M over one tile, 2048 columns)
@pytest.mark.parametrize("batch,units,k", [(1, 300, 4096), (5, 64, 1000), (37, 1024, 8192), (200, 4096, 4096),
                                           (129, 10, 1024), (300, 130, 300), (64, 1000, 784),
                                           (17, 64, 3600), (130, 200, 4096), (5, 2048, 16384), (3, 100, 5000)])
def test_tc_dense_bn_pack_vs_oracle(oracle, batch, units, k, fmt):
    rng = np.random.default_rng(batch + units + k)
    x = oracle.pack_lines(rand_pm1(rng, batch, k))
    wt = oracle.pack_lines(rand_pm1(rng, units, k))
    bn = rand_bn(rng, units, 30.0)
    acc = oracle.bgemm(x, wt, k)
    want = np.stack([oracle.threshold_sign_pack(acc[i].reshape(1, -1), bn.thresh, bn.ge_dir, True)[0]
                     for i in range(batch)])
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, k)
    w8 = _dev.tc_weights(_dev.upload(wt), units, k, fmt)
    out = _dev.empty((batch, -(-units // 64)), np.uint64)
    _lib.call(_lib.tc_entry("dense_bn_pack", fmt), _dev.P(_dev.upload(x)), batch, _dev.P(w8), units, -(-k // 64), k, th(cal),
              _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), want)


@pytest.mark.parametrize("batch,units,k", [(64, 4096, 784), (300, 100, 784), (129, 256, 12), (70, 64, 1024)])
def test_tc_input8_bn_pack_vs_oracle(oracle, batch, units, k):
    rng = np.random.default_rng(batch * units + k)
    u = rng.integers(0, 256, (batch, k), dtype=np.uint8)
    u[0] = 255
    wt = oracle.pack_lines(rand_pm1(rng, units, k))
    bn = rand_bn(rng, units, 5000.0)
    want = []
    for i in range(batch):
        y = oracle.bitplane_matvec(oracle.pack_byte_planes(u[i].reshape(1, -1))[:, 0, :], wt)
        want.append(oracle.threshold_sign_pack(y.reshape(1, -1), bn.thresh, bn.ge_dir, True)[0])
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 255 * k)
    w8 = _dev.widen_i8(_dev.upload(wt), units, k, permute=False)
    out = _dev.empty((batch, -(-units // 64)), np.uint64)
    _lib.call("b2_tc_input8_bn_pack", _dev.P(_dev.upload(u)), batch, k, _dev.P(w8), units, th(cal), _dev.P(out),
              _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want))


@pytest.mark.parametrize("h,w,c,f,kh,pad,stride,pool", [(32, 32, 3, 128, 3, 1, 1, False), (16, 12, 3, 64, 3, 1, 1, True),
                                                        (9, 9, 4, 200, 5, 2, 2, False), (8, 8, 8, 32, 3, 1, 1, True), (10, 6, 5, 64, 5, 2, 1, True),
                                                        (5, 7, 1, 10, 3, 0, 1, False)])
def test_tc_byte_conv_bn_pack_vs_oracle(oracle, h, w, c, f, kh, pad, stride, pool, fmt):
    rng = np.random.default_rng(h * w + c + f)
    batch = 3
    imgs = rng.integers(0, 256, (batch, h, w, c), dtype=np.uint8)
    bn0 = rand_bn(rng, c, 100.0)
    k = kh * kh * c
    wt = oracle.pack_lines(rand_pm1(rng, f, k))
    bn1 = rand_bn(rng, f, 8.0)
    corr = oracle.compute_correction(wt, (h, w, c), (kh, kh), stride, pad)
    ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kh) // stride + 1
    want = []
    for i in range(batch):
        if c == 1:  # single-channel maps are per-row lines (tensor.py:165-173, network.py:121-124)
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h, w).astype(np.int64), np.repeat(bn0.thresh, w),
                                               np.repeat(bn0.ge_dir, w), False)
        else:
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h * w, c).astype(np.int64), bn0.thresh, bn0.ge_dir,
                                               False)
        acc = (oracle.bgemm(oracle.unroll_packed(lines, h, w, c, kh, kh, stride, pad), wt, k) + corr)
        acc = acc.reshape(ho, wo, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn1.thresh, bn1.ge_dir, False))
    cal0 = layers.calibrate_device(bn0.mean, bn0.var, bn0.gamma, bn0.beta, bn0.eps, 255)
    cal1 = layers.calibrate_device(bn1.mean, bn1.var, bn1.gamma, bn1.beta, bn1.eps, k)
    w8 = _dev.tc_weights(_dev.upload(wt), f, k, fmt)
    sites = ho * wo // (4 if pool else 1)
    out = _dev.empty((batch, sites, -(-f // 64)), np.uint64)
    codes = _dev.empty((_lib.raw("b2_tc_byte_conv_scratch_bytes")(batch, h, w, c, kh, kh, stride, pad),), np.uint8)
    _lib.call(_lib.tc_entry("byte_conv_bn_pack", fmt), _dev.P(_dev.upload(imgs)), batch, h, w, c, th(cal0), _dev.P(w8), f, kh, kh,
              stride, pad, int(pool), th(cal1), _dev.P(codes), _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want))


@pytest.mark.parametrize("h,w,c,f,kh,pool,batch", [(32, 32, 3, 128, 3, False, 3), (16, 12, 3, 64, 3, True, 2),
                                                  (8, 8, 8, 32, 3, True, 5), (10, 6, 5, 64, 5, True, 2),
                                                  (5, 7, 1, 10, 3, False, 4), (32, 32, 3, 100, 3, True, 20)])
def test_tc4_byte_conv_padrow_vs_oracle(oracle, h, w, c, f, kh, pool, batch):
    """Byte-BN first layer on the padded-row fp4 kernel (stride 1, same
    padding): the image is thresholded per channel while the band is built."""
    rng = np.random.default_rng(7 * h * w + c + f)
    pad = kh // 2
    imgs = rng.integers(0, 256, (batch, h, w, c), dtype=np.uint8)
    bn0 = rand_bn(rng, c, 100.0)
    k = kh * kh * c
    wt = oracle.pack_lines(rand_pm1(rng, f, k))
    bn1 = rand_bn(rng, f, 8.0)
    corr = oracle.compute_correction(wt, (h, w, c), (kh, kh), 1, pad)
    want = []
    for i in range(batch):
        if c == 1:  # single-channel maps are per-row lines (tensor.py:165-173, network.py:121-124)
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h, w).astype(np.int64), np.repeat(bn0.thresh, w),
                                               np.repeat(bn0.ge_dir, w), False)
        else:
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h * w, c).astype(np.int64), bn0.thresh, bn0.ge_dir,
                                               False)
        acc = (oracle.bgemm(oracle.unroll_packed(lines, h, w, c, kh, kh, 1, pad), wt, k) + corr).reshape(h, w, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn1.thresh, bn1.ge_dir, False))
    cal0 = layers.calibrate_device(bn0.mean, bn0.var, bn0.gamma, bn0.beta, bn0.eps, 255)
    cal1 = layers.calibrate_device(bn1.mean, bn1.var, bn1.gamma, bn1.beta, bn1.eps, k)
    row = int(_lib.raw("b2_f4_cells_row_bytes")(kh * kh))
    wc = _dev.empty((f, row), np.uint8)
    _lib.call("b2_expand_f4_cells", _dev.P(_dev.upload(wt)), f, -(-k // 64), kh * kh, c, _dev.P(wc), _dev.stream())
    sites = h * w // (4 if pool else 1)
    out = _dev.empty((batch, sites, -(-f // 64)), np.uint64)
    _lib.call("b2_tc4_byte_conv_padrow", _dev.P(_dev.upload(imgs)), batch, h, w, c, th(cal0), _dev.P(wc), f, kh, kh,
              pad, int(pool), th(cal1), _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want))


@pytest.mark.parametrize("name", ["bcnn", "bmlp"])
def test_network_engines_agree(networks_golden, name, monkeypatch):
    spec = zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()
    imgs = networks_golden[f"{name}_images"]
    want = networks_golden[f"{name}_scores"]
    reps = 300 // imgs.shape[0] + 1  # > TC_MIN_ROWS so the dense layers take the tensor-core path
    batch = np.concatenate([imgs] * reps)
    for engine in ("tc", "popc"):
        monkeypatch.setattr(_lib, "ENGINE", engine)
        net = Network(spec, max_batch=batch.shape[0])
        got = forward_batch(net, batch)
        assert np.array_equal(got, np.concatenate([want] * reps)), engine


def test_forward_batch_pipelined_chunks(networks_golden):
    """forward_host pipelines chunks of cap/4 through pinned staging and two
    device staging buffers; with N > cap it also runs several blocks.  Every
    image must still get its own reference scores."""
    imgs = networks_golden["bcnn_images"]
    want = networks_golden["bcnn_scores"]
    n = 5000
    idx = np.arange(n) % imgs.shape[0]
    net = Network(zoo.bcnn_spec(), max_batch=4096)
    got = forward_batch(net, imgs[idx])
    assert np.array_equal(got, want[idx])
    got2 = forward_batch(net, imgs[idx[:3000]])  # one block, 3 chunks (last ragged)
    assert np.array_equal(got2, want[idx[:3000]])


def test_forward_batch_from_pinned_images(networks_golden):
    imgs = networks_golden["bcnn_images"]
    want = networks_golden["bcnn_scores"]
    idx = np.arange(3000) % imgs.shape[0]
    net = Network(zoo.bcnn_spec(), max_batch=2048)
    pin = net.pinned_images(3000)
    pin[...] = imgs[idx].reshape(3000, -1)
    assert np.array_equal(forward_batch(net, pin), want[idx])


@pytest.mark.parametrize("n,cap", [(5000, 8192), (4096, 4096), (9000, 4096)])
def test_forward_batch_pinned_geometric_chunks(networks_golden, n, cap):
    """Pinned input runs as one pipeline graph of two chunks (several blocks
    when n > cap); a pinned `out` takes the scores by direct D2H, a plain
    `out` through the pinned workspace."""
    imgs = networks_golden["bcnn_images"]
    want = networks_golden["bcnn_scores"]
    idx = (np.arange(n) * 7) % imgs.shape[0]
    net = Network(zoo.bcnn_spec(), max_batch=cap)
    plan = net._chunk_plan(min(n, cap), True)
    assert sum(b for _, b in plan) == min(n, cap) and len(plan) > 1
    pin = net.pinned_images(n)
    pin[...] = imgs[idx].reshape(n, -1)
    out = net.pinned_scores(n)
    out[...] = np.nan
    assert forward_batch(net, pin, out) is out
    assert np.array_equal(out, want[idx])
    plain = np.full((n, net.classes), np.nan)
    forward_batch(net, pin, plain)
    assert np.array_equal(plain, want[idx])


def test_small_batch_cuda_core_kernels(networks_golden, monkeypatch):
    """With the tensor-core threshold raised, dense and Input8 stages at small
    batch run the packed-weight GEMV / bit-plane POPC kernels; they must give
    the reference's scores too."""
    from paper_1705_07175_b200 import forward, network
    monkeypatch.setattr(network, "TC_MIN_ROWS", 64)
    for name, spec in (("bmlp", zoo.bmlp_spec()), ("bcnn", zoo.bcnn_spec())):
        imgs, want = networks_golden[f"{name}_images"][:5], networks_golden[f"{name}_scores"][:5]
        net = Network(spec, max_batch=5)
        assert np.array_equal(forward_batch(net, imgs), want), name
        net1 = Network(spec, max_batch=1)
        for i in range(2):
            assert np.array_equal(forward(net1, imgs[i]), want[i]), (name, i)


# our fused device stage -> the reference stage whose output it reproduces
# (tests/golden/make_golden.py records every reference stage of image 0)
# (the last dense layer and the final batch-norm run as one stage: its
# output is the reference's float64 scores)
STAGE_REF = {"bcnn": {0: 2, 1: 5, 2: 7, 3: 10, 4: 12, 5: 15, 6: 17, 7: 19, 8: 21},
             "bmlp": {0: 1, 1: 3, 2: 5, 3: 7}}


@pytest.mark.parametrize("name", ["bcnn", "bmlp"])
@pytest.mark.parametrize("batch", [1, 24, 300])
def test_stage_intermediates_match_reference(networks_golden, name, batch):
    """Every fused device stage's output for image 0 equals the reference's
    intermediate (packed words, int32 accumulators, float64 scores)."""
    spec = zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()
    imgs = networks_golden[f"{name}_images"]
    net = Network(spec, max_batch=batch, use_graphs=False)
    forward_batch(net, imgs[np.arange(batch) % imgs.shape[0]])
    for i, st in enumerate(net.stages):
        got = st.out[0].detach().cpu().numpy()
        want = networks_golden[f"{name}_stage{STAGE_REF[name][i]}"]
        if got.dtype == np.int64 and want.dtype == np.uint64:
            got = got.view(np.uint64)
        assert np.array_equal(got.reshape(-1), want.reshape(-1).astype(got.dtype)), (name, batch, i, st.name)


def test_bcnn_batch_65536(networks_golden):
    """BASELINE configs[4]'s whole batch on one GPU (the 8-GPU run gives each
    rank 8192 of these): every one of the 65536 images gets its reference scores."""
    imgs, want = networks_golden["bcnn_images"], networks_golden["bcnn_scores"]
    n = 65536
    idx = np.arange(n) % imgs.shape[0]
    net = Network(zoo.bcnn_spec(), max_batch=n)
    pin = net.pinned_images(n)
    pin[...] = imgs[idx].reshape(n, -1)
    assert np.array_equal(forward_batch(net, pin), want[idx])


@pytest.mark.parametrize("batch", [1, 3, 100])
@pytest.mark.parametrize("units,k", [(10, 64), (200, 4608), (32, 32), (65, 100), (130, 1000)])
def test_packed_outputs_fully_written(oracle, batch, units, k, fmt):
    """Every kernel writes its whole `out` (include/bitnn_b200.h): packed
    lines are padded to whole uint64 words and the padding bits must come out
    0 even when the buffer held garbage (the next layer XORs them)."""
    rng = np.random.default_rng(units * 7 + k + batch)
    x = oracle.pack_lines(rand_pm1(rng, batch, k))
    wt = oracle.pack_lines(rand_pm1(rng, units, k))
    bn = rand_bn(rng, units, 3.0)
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, k)
    want = oracle.threshold_sign_pack(oracle.bgemm(x, wt, k), bn.thresh, bn.ge_dir, True) if batch == 1 else \
        np.stack([oracle.threshold_sign_pack(r.reshape(1, -1), bn.thresh, bn.ge_dir, True)[0]
                  for r in oracle.bgemm(x, wt, k)])
    want = want.reshape(batch, -1)
    for name in ("b2_dense_bn_pack", _lib.tc_entry("dense_bn_pack", fmt)):
        out = _dev.upload(np.full((batch, -(-units // 64)), 0xFFFFFFFFFFFFFFFF, np.uint64))
        wd = _dev.upload(wt) if name == "b2_dense_bn_pack" else _dev.tc_weights(_dev.upload(wt), units, k, fmt)
        _lib.call(name, _dev.P(_dev.upload(x)), batch, _dev.P(wd), units, -(-k // 64), k, th(cal), _dev.P(out),
                  _dev.stream())
        assert np.array_equal(_dev.download(out, np.uint64), want), name


@pytest.mark.parametrize("seed", range(30))
def test_tc_conv_forward_random_geometry(oracle, seed, fmt):
    rng = np.random.default_rng(4000 + seed)
    c = int(rng.choice([64, 128, 192, 256, 320]))
    kh, kw = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    stride, pad = int(rng.integers(1, 4)), int(rng.integers(0, 3))
    h = int(rng.integers(max(1, kh - 2 * pad), 21))
    w = int(rng.integers(max(1, kw - 2 * pad), 21))
    f, batch = int(rng.integers(1, 301)), int(rng.integers(1, 5))
    xs = np.stack([oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)])
    wt = oracle.pack_lines(rand_pm1(rng, f, kh * kw * c))
    corr = oracle.compute_correction(wt, (h, w, c), (kh, kw), stride, pad)
    ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    want = np.stack([oracle.bgemm(oracle.unroll_packed(x, h, w, c, kh, kw, stride, pad), wt, kh * kw * c) + corr
                     for x in xs]).reshape(batch, ho, wo, f)
    w8 = _dev.tc_weights(_dev.upload(wt), f, kh * kw * c, fmt)
    out = _dev.upload(np.full((batch, ho, wo, f), -7, np.int32))
    _lib.call(_lib.tc_entry("conv_forward", fmt), _dev.P(_dev.upload(xs)), batch, h, w, c, _dev.P(w8), f, kh, kw, stride, pad,
              _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.int32), want), (h, w, c, f, kh, kw, stride, pad, batch)


# random row-aligned padded-row launches (>= one 128-pixel tile per SM): 16x16
# or 32x32, C = 128, 1-256 filters (the 129-256 split included), pooled or
# not, BN thresholds with ALWAYS / NEVER sentinels and le filters; checked
# bit-exact against the oracle and asserted to take the row-aligned path
@pytest.mark.parametrize("seed", range(12))
def test_tc_conv_bn_pack_random_aligned(oracle, seed):
    rng = np.random.default_rng(9000 + seed)
    h = w = int(rng.choice([16, 32]))
    c = 128
    f = int(rng.integers(1, 257))
    pool = bool(rng.integers(0, 2))
    batch = 80 if h == 16 else 20
    if _lib._so.b2_tc4_conv_path(batch, h, w, c, f, 3, 3, 1, 1, int(pool)) != 3:
        pytest.skip("shape not on the row-aligned path")
    xs = [oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)]
    wt = oracle.pack_lines(rand_pm1(rng, f, 9 * c))
    bn = rand_bn(rng, f, 20.0)
    bn.gamma[::7] = 0.0
    bn.gamma[3::11] *= -1
    bn = BatchNormLayer(bn.mean, bn.var, bn.gamma, bn.beta)
    corr = oracle.compute_correction(wt, (h, w, c), (3, 3), 1, 1)
    want = []
    for x in xs:
        acc = (oracle.bgemm(oracle.unroll_packed(x, h, w, c, 3, 3, 1, 1), wt, 9 * c) + corr).reshape(h, w, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn.thresh, bn.ge_dir, False))
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
    w8 = _dev.tc_weights(_dev.upload(wt), f, 9 * c, "f4")
    sites = h * w // (4 if pool else 1)
    out = _dev.upload(np.full((batch, sites, -(-f // 64)), 0xFFFFFFFFFFFFFFFF, np.uint64))
    _lib.call(_lib.tc_entry("conv_bn_pack", "f4"), _dev.P(_dev.upload(np.stack(xs))), batch, h, w, c, _dev.P(w8), f,
              3, 3, 1, 1, int(pool), th(cal), _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want)), (h, w, f, pool)


@pytest.mark.parametrize("seed", range(20))
def test_tc_conv_bn_pack_random_geometry(oracle, seed, fmt):
    rng = np.random.default_rng(5000 + seed)
    c = int(rng.choice([64, 128, 256]))
    pool = bool(rng.integers(0, 2))
    h, w = 2 * int(rng.integers(1, 9)), 2 * int(rng.integers(1, 9))
    f, batch = int(rng.integers(1, 300)), int(rng.integers(1, 4))
    xs = [oracle.pack_lines(rand_pm1(rng, h * w, c)) for _ in range(batch)]
    wt = oracle.pack_lines(rand_pm1(rng, f, 9 * c))
    bn = rand_bn(rng, f, 10.0)
    corr = oracle.compute_correction(wt, (h, w, c), (3, 3), 1, 1)
    want = []
    for x in xs:
        acc = (oracle.bgemm(oracle.unroll_packed(x, h, w, c, 3, 3, 1, 1), wt, 9 * c) + corr).reshape(h, w, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn.thresh, bn.ge_dir, False))
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
    w8 = _dev.tc_weights(_dev.upload(wt), f, 9 * c, fmt)
    sites = h * w // (4 if pool else 1)
    out = _dev.upload(np.full((batch, sites, -(-f // 64)), 0xFFFFFFFFFFFFFFFF, np.uint64))
    _lib.call(_lib.tc_entry("conv_bn_pack", fmt), _dev.P(_dev.upload(np.stack(xs))), batch, h, w, c, _dev.P(w8), f, 3, 3, 1, 1,
              int(pool), th(cal), _dev.P(out), _dev.stream())
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want)), (h, w, c, f, pool, batch)


# the fused first-layer kernel (tc_byteconv.cuh, b2_tc_byte_conv_path == 1):
# row-aligned tiles, window + folded threshold in one int8 MMA; gamma = 0
# (ALWAYS / NEVER sentinels) and gamma < 0 (le filters, negated weights) in
# both batch norms; 128- and 256-column tiles
@pytest.mark.parametrize("h,w,c,f,kh,batch", [(32, 32, 3, 128, 3, 3), (16, 16, 3, 64, 3, 5), (8, 16, 2, 200, 3, 4),
                                              (32, 32, 1, 128, 5, 2), (64, 64, 3, 96, 3, 1), (16, 16, 1, 10, 3, 7),
                                              (32, 32, 3, 256, 3, 2), (4, 32, 3, 128, 1, 3)])
def test_fused_byte_conv_vs_oracle(oracle, h, w, c, f, kh, batch):
    pad = (kh - 1) // 2
    assert _lib._so.b2_tc_byte_conv_path(batch, h, w, c, f, kh, kh, 1, pad, 0) == 1
    rng = np.random.default_rng(h * w * 7 + c + f + kh)
    imgs = rng.integers(0, 256, (batch, h, w, c), dtype=np.uint8)
    imgs[0, :2] = 0
    imgs[-1, -2:] = 255
    bn0 = rand_bn(rng, c, 100.0)
    if c > 1:
        bn0.gamma[1] *= -1
    bn0 = BatchNormLayer(bn0.mean, bn0.var, bn0.gamma, bn0.beta)
    k = kh * kh * c
    wt = oracle.pack_lines(rand_pm1(rng, f, k))
    bn1 = rand_bn(rng, f, 4.0)
    bn1.gamma[::7] = 0.0
    bn1.gamma[3::5] *= -1
    bn1 = BatchNormLayer(bn1.mean, bn1.var, bn1.gamma, bn1.beta)
    corr = oracle.compute_correction(wt, (h, w, c), (kh, kh), 1, pad)
    want = []
    for i in range(batch):
        if c == 1:
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h, w).astype(np.int64), np.repeat(bn0.thresh, w),
                                               np.repeat(bn0.ge_dir, w), False)
        else:
            lines = oracle.threshold_sign_pack(imgs[i].reshape(h * w, c).astype(np.int64), bn0.thresh, bn0.ge_dir,
                                               False)
        acc = oracle.bgemm(oracle.unroll_packed(lines, h, w, c, kh, kh, 1, pad), wt, k) + corr
        want.append(oracle.threshold_sign_pack(acc.reshape(-1, f), bn1.thresh, bn1.ge_dir, False))
    cal0 = layers.calibrate_device(bn0.mean, bn0.var, bn0.gamma, bn0.beta, bn0.eps, 255)
    cal1 = layers.calibrate_device(bn1.mean, bn1.var, bn1.gamma, bn1.beta, bn1.eps, k)
    w8 = _dev.tc_weights(_dev.upload(wt), f, k, "i8")
    out = _dev.empty((batch, h * w, -(-f // 64)), np.uint64)
    out.fill_(-1)  # every word must be written
    codes = _dev.empty((8,), np.uint8)  # the fused kernel takes no scratch
    c0 = _lib.launch_count()
    _lib.call("b2_tc_byte_conv_bn_pack", _dev.P(_dev.upload(imgs)), batch, h, w, c, th(cal0), _dev.P(w8), f, kh, kh,
              1, pad, 0, th(cal1), _dev.P(codes), _dev.P(out), _dev.stream())
    assert _lib.launch_count() - c0 == 1
    assert np.array_equal(_dev.download(out, np.uint64), np.stack(want))


@pytest.mark.parametrize("h,w,c,f,kh,pad,stride,pool", [(16, 12, 3, 64, 3, 1, 1, True), (9, 9, 4, 200, 5, 2, 2, False),
                                                        (8, 8, 8, 32, 3, 1, 1, True), (5, 7, 1, 10, 3, 0, 1, False)])
def test_byte_conv_unfused_path_kept(h, w, c, f, kh, pad, stride, pool):
    assert _lib._so.b2_tc_byte_conv_path(3, h, w, c, f, kh, kh, stride, pad, int(pool)) == 0


# ---- CTA-pair kernel (tc_pair.cuh): launches with >= 74 256x256 tiles.
# Ragged M / N / K, int32 / packed / pooled / float64 epilogues; the oracle
# checks a sample of rows (every row of the GPU output is computed).
def _sample_rows(m, n=48):
    return np.unique(np.concatenate([np.arange(min(m, 8)), np.linspace(0, m - 1, n).astype(np.int64),
                                     np.arange(max(0, m - 8), m)]))


@pytest.mark.parametrize("m,n,k", [(4096, 1280, 1000), (19000, 300, 777), (9100, 2048, 4608), (38000, 257, 64)])
def test_pair_bgemm_vs_oracle(oracle, m, n, k):
    rng = np.random.default_rng(m + n + k)
    a = zoo.pack_bits_host(rng.random((m, k)) >= 0.5)
    b = zoo.pack_bits_host(rng.random((n, k)) >= 0.5)
    got = _dev.download(gemm.bgemm_device(_dev.upload(a), m, _dev.upload(b), n, a.shape[1], k, engine="tc", fmt="f4"),
                        np.int32)
    rows = _sample_rows(m)
    assert np.array_equal(got[rows], oracle.bgemm(np.ascontiguousarray(a[rows]), b, k))


@pytest.mark.parametrize("batch,units,k", [(20000, 512, 2048), (40000, 300, 1000), (19000, 1024, 8192)])
def test_pair_dense_bn_pack_vs_oracle(oracle, batch, units, k):
    rng = np.random.default_rng(batch + units + k)
    x = zoo.pack_bits_host(rng.random((batch, k)) >= 0.5)
    wt = zoo.pack_bits_host(rng.random((units, k)) >= 0.5)
    bn = rand_bn(rng, units, 30.0)
    bn.gamma[::9] = 0.0
    bn.gamma[4::7] *= -1
    bn = BatchNormLayer(bn.mean, bn.var, bn.gamma, bn.beta)
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, k)
    w8 = _dev.tc_weights(_dev.upload(wt), units, k, "f4")
    out = _dev.empty((batch, -(-units // 64)), np.uint64)
    _lib.call("b2_tc4_dense_bn_pack", _dev.P(_dev.upload(x)), batch, _dev.P(w8), units, -(-k // 64), k, th(cal),
              _dev.P(out), _dev.stream())
    got = _dev.download(out, np.uint64)
    rows = _sample_rows(batch)
    acc = oracle.bgemm(np.ascontiguousarray(x[rows]), wt, k)
    want = np.stack([oracle.threshold_sign_pack(acc[i].reshape(1, -1), bn.thresh, bn.ge_dir, True)[0]
                     for i in range(len(rows))])
    assert np.array_equal(got[rows], want)


@pytest.mark.parametrize("h,w,c,f,pool,batch", [(16, 16, 256, 256, True, 300), (8, 8, 512, 320, False, 1200),
                                                (8, 8, 256, 512, True, 1200), (4, 4, 512, 512, False, 5000)])
def test_pair_conv_bn_pack_vs_oracle(oracle, h, w, c, f, pool, batch):
    rng = np.random.default_rng(h + c + f + batch)
    xs = zoo.pack_bits_host(rng.random((batch * h * w, c)) >= 0.5).reshape(batch, h * w, -1)
    wt = zoo.pack_bits_host(rng.random((f, 9 * c)) >= 0.5)
    bn = rand_bn(rng, f, 20.0)
    bn.gamma[::7] = 0.0
    bn.gamma[3::11] *= -1
    bn = BatchNormLayer(bn.mean, bn.var, bn.gamma, bn.beta)
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
    w8 = _dev.tc_weights(_dev.upload(wt), f, 9 * c, "f4")
    sites = h * w // (4 if pool else 1)
    out = _dev.empty((batch, sites, -(-f // 64)), np.uint64)
    _lib.call("b2_tc4_conv_bn_pack", _dev.P(_dev.upload(xs)), batch, h, w, c, _dev.P(w8), f, 3, 3, 1, 1, int(pool),
              th(cal), _dev.P(out), _dev.stream())
    got = _dev.download(out, np.uint64)
    corr = oracle.compute_correction(wt, (h, w, c), (3, 3), 1, 1)
    for i in (0, 1, batch // 2, batch - 1):
        acc = (oracle.bgemm(oracle.unroll_packed(xs[i], h, w, c, 3, 3, 1, 1), wt, 9 * c) + corr).reshape(h, w, f)
        if pool:
            acc = oracle.maxpool(acc, 2, 2, 2)
        want = oracle.threshold_sign_pack(acc.reshape(-1, f), bn.thresh, bn.ge_dir, False)
        assert np.array_equal(got[i], want), i


def test_pair_dense_affine_vs_oracle(oracle):
    batch, units, k = 20000, 300, 1000
    rng = np.random.default_rng(3)
    x = zoo.pack_bits_host(rng.random((batch, k)) >= 0.5)
    wt = zoo.pack_bits_host(rng.random((units, k)) >= 0.5)
    bn = rand_bn(rng, units, 10.0)
    w8 = _dev.tc_weights(_dev.upload(wt), units, k, "f4")
    out = _dev.empty((batch, units), np.float64)
    mean, scale, beta = (_dev.upload(np.asarray(v, dtype=np.float64)) for v in (bn.mean64, bn.scale64, bn.beta64))
    _lib.call("b2_tc4_dense_affine_f64", _dev.P(_dev.upload(x)), batch, _dev.P(w8), units, -(-k // 64), k,
              _dev.P(mean), _dev.P(scale), _dev.P(beta), _dev.P(out), _dev.stream())
    got = _dev.download(out, np.float64)
    rows = _sample_rows(batch)
    acc = oracle.bgemm(np.ascontiguousarray(x[rows]), wt, k)
    want = np.stack([oracle.bn_affine(acc[i], bn.mean64, bn.scale64, bn.beta64) for i in range(len(rows))])
    assert np.array_equal(got[rows], want)
