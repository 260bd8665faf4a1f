"""Generate golden vectors by running the REFERENCE `bitnn` package.

Run once in the build container (the reference is importable there from
/root/reference/pkg/src; it does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes into tests/golden/:
  * mlp.bdnn, cnn.bdnn      — the reference fixture models, produced by the
                              reference's own tests/fixtures/generate.py builders
  * kernels.npz             — per-kernel input/output vectors
  * networks.npz            — scores of the fixture models and of the
                              BASELINE-sized BMLP / BCNN on seeded images,
                              plus the SHA-256 of each model's serialized bytes
  * vgg.bdnn, acceptance.npz — the reference's acceptance CNN and its
                              1000-image scores (both backends), and 1024
                              seeded images each through BCNN / BMLP

The BASELINE-sized models are built here with the reference's record
classes using the recipe documented in paper_1705_07175_b200/zoo.py
(same rng call order); tests rebuild them with zoo.py and compare hashes.
"""

import hashlib
import os
import runpy
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_FIXTURES = "/root/reference/pkg/tests/fixtures/generate.py"
HERE = os.path.dirname(os.path.abspath(__file__))

sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from bitnn import _kernels  # noqa: E402
from bitnn.gemm import PackedMatrixA, PackedMatrixB, bgemm  # noqa: E402
from bitnn.layers import BatchNormLayer, ConvLayer, conv_forward, fused_bn_sign, unroll  # noqa: E402
from bitnn.modelfile import (BatchNormRecord, ConvRecord, DenseRecord, Input8Record,  # noqa: E402
                             MaxPoolRecord, ModelSpec, write_model)
from bitnn.network import Network, forward  # noqa: E402
from bitnn.tensor import FloatTensor, pack  # noqa: E402


def rand_pm1(rng, *shape):
    return np.where(rng.random(shape) < 0.5, -1.0, 1.0).astype(np.float32)


def pack_rows(rng, rows, k):
    return PackedMatrixA.from_float(rand_pm1(rng, rows, k)).words


def bn(rng, c, spread):
    return BatchNormRecord(
        (rng.standard_normal(c) * spread).astype(np.float32),
        (rng.random(c) * 50 + 1).astype(np.float32),
        rng.standard_normal(c).astype(np.float32),
        rng.standard_normal(c).astype(np.float32),
        1e-5,
    )


# Recipes mirrored by paper_1705_07175_b200/zoo.py (keep in sync).
def bmlp_spec(seed=0x784):
    rng = np.random.default_rng(seed)
    return ModelSpec((1, 1, 784), [
        Input8Record(4096, 784, pack_rows(rng, 4096, 784)), bn(rng, 4096, 5000.0),
        DenseRecord(4096, 4096, pack_rows(rng, 4096, 4096)), bn(rng, 4096, 60.0),
        DenseRecord(4096, 4096, pack_rows(rng, 4096, 4096)), bn(rng, 4096, 60.0),
        DenseRecord(10, 4096, pack_rows(rng, 10, 4096)), bn(rng, 10, 4.0),
    ])


def bcnn_spec(seed=0x1705):
    rng = np.random.default_rng(seed)
    return ModelSpec((32, 32, 3), [
        bn(rng, 3, 100.0),
        ConvRecord(128, 3, 3, 1, 1, 3, pack_rows(rng, 128, 27)), bn(rng, 128, 8.0),
        ConvRecord(128, 3, 3, 1, 1, 128, pack_rows(rng, 128, 1152)), MaxPoolRecord(2, 2, 2), bn(rng, 128, 40.0),
        ConvRecord(256, 3, 3, 1, 1, 128, pack_rows(rng, 256, 1152)), bn(rng, 256, 30.0),
        ConvRecord(256, 3, 3, 1, 1, 256, pack_rows(rng, 256, 2304)), MaxPoolRecord(2, 2, 2), bn(rng, 256, 60.0),
        ConvRecord(512, 3, 3, 1, 1, 256, pack_rows(rng, 512, 2304)), bn(rng, 512, 45.0),
        ConvRecord(512, 3, 3, 1, 1, 512, pack_rows(rng, 512, 4608)), MaxPoolRecord(2, 2, 2), bn(rng, 512, 80.0),
        DenseRecord(1024, 8192, pack_rows(rng, 1024, 8192)), bn(rng, 1024, 80.0),
        DenseRecord(1024, 1024, pack_rows(rng, 1024, 1024)), bn(rng, 1024, 30.0),
        DenseRecord(10, 1024, pack_rows(rng, 10, 1024)), bn(rng, 10, 4.0),
    ])


def kernel_vectors():
    rng = np.random.default_rng(20251017)
    out = {}
    # K2 pack_lines incl. 0.0, -0.0, NaN, inf
    x = rng.standard_normal((7, 203)).astype(np.float32)
    x[0, :5] = [0.0, -0.0, np.nan, -np.inf, np.inf]
    x[3, 64] = 0.0
    w = np.zeros((7, 4), dtype=np.uint64)
    _kernels.pack_lines(x, w)
    out["pack_in"], out["pack_out"] = x, w
    # K4 pack_byte_planes
    u = rng.integers(0, 256, (5, 70), dtype=np.uint8)
    p = np.zeros((8, 5, 2), dtype=np.uint64)
    _kernels.pack_byte_planes(u, p)
    out["planes_in"], out["planes_out"] = u, p
    # K5 bgemm: forced K list of test_acceptance.py:104 plus random shapes
    forced = [1, 63, 64, 65, 128, 129, 192, 255, 256, 300, 1152, 4608]
    for t in range(24):
        m = int(rng.integers(1, 97))
        n = int(rng.integers(1, 97))
        k = forced[t] if t < len(forced) else int(rng.integers(1, 700))
        a = PackedMatrixA.from_float(rand_pm1(rng, m, k))
        b = PackedMatrixB.from_float(rand_pm1(rng, k, n))
        out[f"bgemm{t}_a"], out[f"bgemm{t}_b"], out[f"bgemm{t}_k"] = a.words, b.words, np.int64(k)
        out[f"bgemm{t}_c"] = bgemm(a, b)
    # K8 bitplane matvec (BMLP first layer shape, 16 units)
    u = rng.integers(0, 256, 784, dtype=np.uint8)
    planes = np.zeros((8, 1, 13), dtype=np.uint64)
    _kernels.pack_byte_planes(u.reshape(1, -1), planes)
    pops = np.zeros(8, dtype=np.int64)
    _kernels.count_plane_bits(planes[:, 0, :], pops)
    wt = pack_rows(rng, 16, 784)
    y = np.zeros(16, dtype=np.int64)
    _kernels.bitplane_matvec(planes[:, 0, :], pops, wt, y)
    out["i8_u"], out["i8_w"], out["i8_y"] = u, wt, y
    # K9 unroll + a-9 correction + a-10 conv_forward
    cases = [(8, 8, 16, 3, 3, 1, 1), (5, 7, 3, 3, 3, 2, 2), (6, 6, 1, 2, 2, 2, 0), (4, 4, 70, 3, 3, 1, 1),
             (6, 5, 32, 3, 3, 1, 1), (4, 4, 128, 3, 3, 1, 1), (7, 7, 2, 5, 5, 2, 2), (9, 9, 1, 3, 3, 1, 1)]
    for t, (h, ww, c, kh, kw, s, pad) in enumerate(cases):
        xf = rand_pm1(rng, h, ww, c)
        xp = pack(FloatTensor(xf))
        f = int(rng.integers(1, 40))
        wf = rand_pm1(rng, kh * kw * c, f)
        layer = ConvLayer.from_float(wf, (kh, kw), s, pad, (h, ww, c))
        out[f"conv{t}_params"] = np.array([h, ww, c, kh, kw, s, pad, f], dtype=np.int64)
        out[f"conv{t}_x"] = xp.words
        out[f"conv{t}_w"] = layer.weights.words
        out[f"conv{t}_unroll"] = unroll(xp, (kh, kw), s, pad).words
        out[f"conv{t}_corr"] = layer.correction
        out[f"conv{t}_out"] = conv_forward(layer, xp)
    # a-11 maxpool
    for t, (h, ww, c, ph, pw, s) in enumerate([(6, 6, 4, 2, 2, 2), (7, 5, 3, 3, 2, 2), (5, 5, 1, 2, 2, 1),
                                               (32, 32, 128, 2, 2, 2)]):
        xi = rng.integers(-3000, 3000, size=(h, ww, c)).astype(np.int32)
        o = np.zeros(((h - ph) // s + 1, (ww - pw) // s + 1, c), dtype=np.int32)
        _kernels.maxpool(xi, ph, pw, s, o)
        out[f"pool{t}_params"] = np.array([ph, pw, s], dtype=np.int64)
        out[f"pool{t}_x"], out[f"pool{t}_out"] = xi, o
    # a-12 calibration incl. gamma 0 / negative / tiny variance / huge spread
    c = 300
    mean = (rng.standard_normal(c) * np.geomspace(1, 1e6, c)).astype(np.float32)
    var = (rng.random(c) * 50).astype(np.float32)
    var[:10] = 0.0
    gamma = rng.standard_normal(c).astype(np.float32)
    gamma[10:20] = 0.0
    gamma[20:40] = -np.abs(gamma[20:40])
    beta = rng.standard_normal(c).astype(np.float32)
    beta[10:15] = -beta[10:15] ** 2 - 0.1
    layer = BatchNormLayer(mean, var, gamma, beta, eps=float(np.float32(1e-5)))
    out["bn_mean"], out["bn_var"], out["bn_gamma"], out["bn_beta"] = mean, var, gamma, beta
    out["bn_eps"] = np.float64(np.float32(1e-5))
    out["bn_thresh"], out["bn_ge"], out["bn_scale"] = layer.thresh, layer.ge_dir, layer.scale64
    # a-13 fused threshold pack: per-site, flat, single channel; boundary values
    for t, (h, ww, cc, flat) in enumerate([(4, 4, 40, False), (3, 5, 40, True), (6, 7, 1, False),
                                           (2, 2, 130, False), (1, 1, 300, False)]):
        sub = BatchNormLayer(mean[:cc] / 1000, var[:cc] + 1, rng.standard_normal(cc).astype(np.float32), beta[:cc], eps=1e-5)
        xi = rng.integers(-2000, 2000, size=(h, ww, cc)).astype(np.int32)
        for ch in range(min(cc, h * ww)):
            tt = int(sub.thresh[ch])
            if abs(tt) < 2 ** 31 - 2:
                xi[ch // ww % h, ch % ww, ch] = tt + int(rng.integers(-1, 2))
        pk = fused_bn_sign(sub, xi, flat=flat)
        out[f"thr{t}_x"], out[f"thr{t}_flat"] = xi, np.int64(flat)
        out[f"thr{t}_thresh"], out[f"thr{t}_ge"] = sub.thresh, sub.ge_dir
        out[f"thr{t}_out"] = pk.words
    # a-14 final bn affine (float64, no FMA)
    xi = rng.integers(-5000, 5000, size=4000).astype(np.int32)
    sub = BatchNormLayer(mean[:10] / 1e5, var[:10] + 1, gamma[40:50], beta[:10])
    o = np.zeros(4000, dtype=np.float64)
    _kernels.bn_affine(xi, sub.mean64, sub.scale64, sub.beta64, o)
    out["aff_x"], out["aff_mean"], out["aff_scale"], out["aff_beta"], out["aff_out"] = (
        xi, sub.mean64, sub.scale64, sub.beta64, o)
    return out


def network_vectors():
    out = {}
    gen = runpy.run_path(REF_FIXTURES)
    for name in ("mlp", "cnn"):
        spec = gen[f"build_{name}"]()
        data = write_model(spec)
        with open(os.path.join(HERE, f"{name}.bdnn"), "wb") as fh:
            fh.write(data)
        net = Network(spec)
        shape = (784,) if name == "mlp" else (32, 32, 3)
        rng = np.random.default_rng(7)
        imgs = np.stack([rng.integers(0, 256, shape, dtype=np.uint8) for _ in range(5)]
                        + [np.zeros(shape, dtype=np.uint8)])
        rng = np.random.default_rng(8)
        imgs = np.concatenate([imgs, np.stack([rng.integers(0, 256, shape, dtype=np.uint8) for _ in range(26)])])
        out[f"{name}_images"] = imgs
        out[f"{name}_scores"] = np.stack([forward(net, im).copy() for im in imgs])
    for name, spec, shape, n in (("bmlp", bmlp_spec(), (784,), 64), ("bcnn", bcnn_spec(), (32, 32, 3), 24)):
        data = write_model(spec)
        out[f"{name}_sha256"] = np.array(hashlib.sha256(data).hexdigest())
        net = Network(spec)
        rng = np.random.default_rng(11)
        imgs = rng.integers(0, 256, (n,) + shape, dtype=np.uint8)
        out[f"{name}_images"] = imgs
        out[f"{name}_scores"] = np.stack([forward(net, im).copy() for im in imgs])
        # intermediate packed activations of image 0, for layer-by-layer debugging
        x = imgs[0]
        for si, st in enumerate(net.stages):
            x = st.run(x)
            out[f"{name}_stage{si}"] = np.array(x, copy=True)
    return out


def vgg_like_cnn(rng):
    """The reference acceptance network (pkg/tests/test_acceptance.py:80-98):
    32x32x3 input, 2x(32C3) - MP2 - 2x(64C3) - MP2 - FC256 - FC10, drawn from
    `rng` in the same call order."""
    return ModelSpec((32, 32, 3), [
        bn(rng, 3, 100.0),
        ConvRecord(32, 3, 3, 1, 1, 3, pack_rows(rng, 32, 27)), bn(rng, 32, 8.0),
        ConvRecord(32, 3, 3, 1, 1, 32, pack_rows(rng, 32, 288)), MaxPoolRecord(2, 2, 2), bn(rng, 32, 30.0),
        ConvRecord(64, 3, 3, 1, 1, 32, pack_rows(rng, 64, 288)), bn(rng, 64, 30.0),
        ConvRecord(64, 3, 3, 1, 1, 64, pack_rows(rng, 64, 576)), MaxPoolRecord(2, 2, 2), bn(rng, 64, 60.0),
        DenseRecord(256, 4096, pack_rows(rng, 256, 4096)), bn(rng, 256, 20.0),
        DenseRecord(10, 256, pack_rows(rng, 10, 256)), bn(rng, 10, 4.0),
    ])


def acceptance_vectors():
    """Wider parity set (round 2): the reference's own acceptance network with
    its 1000-image cross-backend check (test_acceptance.py:166-179), both
    backends' scores, and 1024 distinct images each for the BASELINE-sized
    BCNN and BMLP.  Images are NOT stored: tests regenerate them from the
    seeds below (same rng recipe), so the fixture stays small."""
    from bitnn.network import Backend
    out = {}
    rng = np.random.default_rng(2028)
    spec = vgg_like_cnn(rng)
    with open(os.path.join(HERE, "vgg.bdnn"), "wb") as fh:
        fh.write(write_model(spec))
    packed, ref = Network(spec, Backend.PACKED), Network(spec, Backend.REFERENCE)
    sp, sr = [], []
    for _ in range(1000):
        img = rng.integers(0, 256, (32, 32, 3), dtype=np.uint8)
        sp.append(forward(packed, img).copy())
        sr.append(forward(ref, img).copy())
    out["vgg_packed_scores"], out["vgg_reference_scores"] = np.stack(sp), np.stack(sr)
    for name, spec, shape in (("bcnn", bcnn_spec(), (32, 32, 3)), ("bmlp", bmlp_spec(), (784,))):
        net = Network(spec)
        imgs = np.random.default_rng(4242).integers(0, 256, (1024,) + shape, dtype=np.uint8)
        out[f"{name}1024_scores"] = np.stack([forward(net, im).copy() for im in imgs])
    out["seeds"] = np.array([2028, 4242])
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernel_vectors())
    np.savez_compressed(os.path.join(HERE, "networks.npz"), **network_vectors())
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **acceptance_vectors())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
