"""Pin the CPU oracle to the reference: every golden vector that
tests/golden/make_golden.py produced by running the reference `bitnn`
must be reproduced bit for bit (float64 scores included)."""

import os

import numpy as np

from conftest import GOLDEN
from paper_1705_07175_b200 import modelfile, zoo


def test_pack_lines(kernels_golden, oracle):
    g = kernels_golden
    assert np.array_equal(oracle.pack_lines(g["pack_in"]), g["pack_out"])


def test_pack_byte_planes(kernels_golden, oracle):
    g = kernels_golden
    assert np.array_equal(oracle.pack_byte_planes(g["planes_in"]), g["planes_out"])


def test_bgemm_shapes(kernels_golden, oracle):
    g = kernels_golden
    for t in range(24):
        got = oracle.bgemm(g[f"bgemm{t}_a"], g[f"bgemm{t}_b"], int(g[f"bgemm{t}_k"]))
        assert np.array_equal(got, g[f"bgemm{t}_c"]), t


def test_bitplane_matvec(kernels_golden, oracle):
    g = kernels_golden
    planes = oracle.pack_byte_planes(g["i8_u"].reshape(1, -1))[:, 0, :]
    assert np.array_equal(oracle.bitplane_matvec(planes, g["i8_w"]), g["i8_y"])


def test_unroll_correction_conv(kernels_golden, oracle):
    g = kernels_golden
    for t in range(8):
        h, w, c, kh, kw, s, pad, f = (int(v) for v in g[f"conv{t}_params"])
        u = oracle.unroll_packed(g[f"conv{t}_x"], h, w, c, kh, kw, s, pad)
        assert np.array_equal(u, g[f"conv{t}_unroll"]), t
        corr = oracle.compute_correction(g[f"conv{t}_w"], (h, w, c), (kh, kw), s, pad)
        assert np.array_equal(corr, g[f"conv{t}_corr"]), t
        acc = oracle.bgemm(u, g[f"conv{t}_w"], kh * kw * c) + corr
        assert np.array_equal(acc.reshape(g[f"conv{t}_out"].shape), g[f"conv{t}_out"]), t


def test_maxpool(kernels_golden, oracle):
    g = kernels_golden
    for t in range(4):
        ph, pw, s = (int(v) for v in g[f"pool{t}_params"])
        assert np.array_equal(oracle.maxpool(g[f"pool{t}_x"], ph, pw, s), g[f"pool{t}_out"]), t


def test_calibration(kernels_golden, oracle):
    g = kernels_golden
    scale, thresh, ge = oracle.bn_calibrate(g["bn_mean"], g["bn_var"], g["bn_gamma"], g["bn_beta"],
                                            float(g["bn_eps"]))
    assert np.array_equal(scale, g["bn_scale"])
    assert np.array_equal(thresh, g["bn_thresh"])
    assert np.array_equal(ge, g["bn_ge"])


def test_threshold_pack(kernels_golden, oracle):
    g = kernels_golden
    for t in range(5):
        x = g[f"thr{t}_x"]
        h, w, c = x.shape
        flat = bool(g[f"thr{t}_flat"])
        th, ge = g[f"thr{t}_thresh"], g[f"thr{t}_ge"]
        if c == 1 and not flat and h * w > 1:
            got = oracle.threshold_sign_pack(x.reshape(h, w), np.full(w, th[0]), np.full(w, ge[0]), False)
        else:
            got = oracle.threshold_sign_pack(x.reshape(h * w, c), th, ge, flat or h * w == 1)
        assert np.array_equal(got, g[f"thr{t}_out"]), t


def test_bn_affine_bit_exact(kernels_golden, oracle):
    g = kernels_golden
    got = oracle.bn_affine(g["aff_x"], g["aff_mean"], g["aff_scale"], g["aff_beta"])
    assert np.array_equal(got, g["aff_out"])


def test_fixture_models_bytes_and_scores(networks_golden, oracle):
    for name in ("mlp", "cnn"):
        spec = modelfile.load_model(os.path.join(GOLDEN, f"{name}.bdnn"))
        net = oracle.OracleNetwork(spec)
        imgs = networks_golden[f"{name}_images"]
        want = networks_golden[f"{name}_scores"]
        for i in range(imgs.shape[0]):
            assert np.array_equal(net.forward(imgs[i]), want[i]), (name, i)


def test_fixture_frozen_classes(networks_golden, oracle):
    # test_fixtures.py:110-124 of the reference
    mlp = oracle.OracleNetwork(modelfile.load_model(os.path.join(GOLDEN, "mlp.bdnn")))
    cnn = oracle.OracleNetwork(modelfile.load_model(os.path.join(GOLDEN, "cnn.bdnn")))
    m = [int(np.argmax(mlp.forward(im))) for im in networks_golden["mlp_images"][:6]]
    c = [int(np.argmax(cnn.forward(im))) for im in networks_golden["cnn_images"][:6]]
    assert m == [0, 0, 0, 0, 7, 7]
    assert c == [5, 5, 5, 5, 5, 5]


def test_baseline_models_scores(networks_golden, oracle):
    for name, n in (("bmlp", 8), ("bcnn", 4)):
        spec = getattr(zoo, f"{name}_spec")()
        net = oracle.OracleNetwork(spec)
        imgs = networks_golden[f"{name}_images"][:n]
        want = networks_golden[f"{name}_scores"][:n]
        for i in range(n):
            assert np.array_equal(net.forward(imgs[i]), want[i]), (name, i)


def test_acceptance_set_oracle(oracle):
    """The oracle against the reference's acceptance CNN (1000 images, both
    backends agree: argmax identical, gap < 1e-4) and 1024 distinct images
    through the BASELINE BMLP / a 96-image sample through BCNN."""
    from acceptance_set import images1024, vgg_set
    acc = np.load(os.path.join(GOLDEN, "acceptance.npz"))
    spec, imgs = vgg_set()
    net = oracle.OracleNetwork(spec)
    got = np.stack([net.forward(im) for im in imgs])
    assert np.array_equal(got, acc["vgg_packed_scores"])
    assert np.array_equal(np.argmax(got, 1), np.argmax(acc["vgg_reference_scores"], 1))
    assert float(np.max(np.abs(got - acc["vgg_reference_scores"]))) < 1e-4
    bm = oracle.OracleNetwork(zoo.bmlp_spec())
    x = images1024("bmlp")
    assert np.array_equal(np.stack([bm.forward(im) for im in x]), acc["bmlp1024_scores"])
    bc = oracle.OracleNetwork(zoo.bcnn_spec())
    x = images1024("bcnn")
    idx = np.arange(0, 1024, 11)
    assert np.array_equal(np.stack([bc.forward(x[i]) for i in idx]), acc["bcnn1024_scores"][idx])
