"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, the ESPBDNN1 reader/writer is byte-compatible with the reference
fixtures and raises the reference's errors, and network validation
(host logic) matches network.py:331-486."""

import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_1705_07175_b200 import _lib, modelfile, zoo
from paper_1705_07175_b200.modelfile import (BatchNormRecord, ConvRecord, DenseRecord, Input8Record, MaxPoolRecord,
                                             ModelFormatError, ModelSpec, ModelValidationError, read_model,
                                             write_model)
from paper_1705_07175_b200.network import Network, model_size


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bitnn_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(b2_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib._so, s), s
    assert sorted(_lib.exported_symbols()) == syms
    assert "sm_100a" in _lib.version()


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def rand_rows(rng, rows, k):
    return zoo.pack_bits_host(rng.random((rows, k)) >= 0.5)


def bn_rec(rng, c, spread=20.0):
    return zoo.rand_bn(rng, c, spread)


def mlp_spec(rng, hidden=32, n_in=784, n_out=10):
    return ModelSpec((1, 1, n_in), [Input8Record(hidden, n_in, rand_rows(rng, hidden, n_in)),
                                    bn_rec(rng, hidden, 5000.0),
                                    DenseRecord(n_out, hidden, rand_rows(rng, n_out, hidden)), bn_rec(rng, n_out, 4.0)])


def cnn_spec(rng):
    return ModelSpec((16, 16, 3), [
        bn_rec(rng, 3, 100.0), ConvRecord(16, 3, 3, 1, 1, 3, rand_rows(rng, 16, 27)), MaxPoolRecord(2, 2, 2),
        bn_rec(rng, 16, 10.0), ConvRecord(32, 3, 3, 1, 1, 16, rand_rows(rng, 32, 144)), MaxPoolRecord(2, 2, 2),
        bn_rec(rng, 32, 10.0), DenseRecord(64, 512, rand_rows(rng, 64, 512)), bn_rec(rng, 64, 8.0),
        DenseRecord(10, 64, rand_rows(rng, 10, 64)), bn_rec(rng, 10, 4.0)])


# ---- model file (ports of the reference's test_network.py:98-162) ----

def test_fixture_bytes_round_trip():
    for name in ("mlp", "cnn"):
        data = open(os.path.join(GOLDEN, f"{name}.bdnn"), "rb").read()
        assert write_model(read_model(data)) == data


def test_zoo_specs_hash_like_reference(networks_golden):
    import hashlib
    for name in ("bmlp", "bcnn"):
        data = write_model(getattr(zoo, f"{name}_spec")())
        assert hashlib.sha256(data).hexdigest() == str(networks_golden[f"{name}_sha256"])


def test_format_errors():
    rng = np.random.default_rng(10)
    data = write_model(mlp_spec(rng))
    with pytest.raises(ModelFormatError, match="magic"):
        read_model(b"XXXXXXXX" + data[8:])
    bad = bytearray(data)
    bad[8:12] = (2).to_bytes(4, "little")
    with pytest.raises(ModelFormatError, match="version"):
        read_model(bytes(bad))
    with pytest.raises(ModelFormatError, match="truncated"):
        read_model(data[:-5])
    with pytest.raises(ModelFormatError, match="trailing"):
        read_model(data + b"\x00")
    bad = bytearray(data)
    assert bad[28] == 0
    bad[28] = 9
    with pytest.raises(ModelFormatError, match="unknown tag"):
        read_model(bytes(bad))
    assert issubclass(ModelFormatError, ValueError) and issubclass(ModelValidationError, ValueError)


def test_dirty_padding_rejected():
    rng = np.random.default_rng(15)
    spec = mlp_spec(rng)
    words = spec.records[0].words.copy()
    words[0, -1] |= np.uint64(1) << np.uint64(40)
    dirty = ModelSpec(spec.input_dims, [Input8Record(32, 784, words)] + spec.records[1:])
    with pytest.raises(ModelValidationError, match="layer 0.*padding"):
        read_model(write_model(dirty))


def test_eps_quantised_to_float32():
    r = BatchNormRecord(np.zeros(1, np.float32), np.ones(1, np.float32), np.ones(1, np.float32),
                        np.zeros(1, np.float32), 1e-5)
    assert r.eps == float(np.float32(1e-5))


# ---- validation (test_network.py:167-228) ----

def test_validation_messages():
    rng = np.random.default_rng(20)
    spec = mlp_spec(rng)
    with pytest.raises(ModelValidationError, match="layer 1"):
        Network(ModelSpec(spec.input_dims, [spec.records[0], bn_rec(rng, 16)] + spec.records[2:]))
    with pytest.raises(ModelValidationError, match="layer 2"):
        Network(ModelSpec(spec.input_dims, spec.records[:2] + [DenseRecord(10, 64, rand_rows(rng, 10, 64)),
                                                               spec.records[3]]))
    cs = cnn_spec(rng)
    with pytest.raises(ModelValidationError, match="layer 1"):
        Network(ModelSpec(cs.input_dims, [cs.records[0], ConvRecord(16, 3, 3, 1, 1, 4, rand_rows(rng, 16, 36))]
                          + cs.records[2:]))
    with pytest.raises(ModelValidationError, match="first layer"):
        Network(ModelSpec(cs.input_dims, cs.records[:3] + [Input8Record(8, 64, rand_rows(rng, 8, 64))]
                          + cs.records[3:]))
    with pytest.raises(ModelValidationError, match="batchnorm"):
        Network(ModelSpec(spec.input_dims, spec.records[:3]))
    with pytest.raises(ModelValidationError):
        Network(ModelSpec((4, 4, 2), [bn_rec(rng, 2), bn_rec(rng, 2)]))
    with pytest.raises(ModelValidationError):
        Network(ModelSpec(spec.input_dims, spec.records[:2] + [MaxPoolRecord(2, 2, 2)] + spec.records[2:]))
    with pytest.raises(ModelValidationError, match="layer_backends"):
        Network(spec, layer_backends=["packed"])


# ---- model_size (test_network.py:446-495) ----

def test_model_size_paper_mlp():
    def dense(units, k):
        return DenseRecord(units, k, np.zeros((units, -(-k // 64)), dtype=np.uint64))

    def bn(c):
        z = np.zeros(c, dtype=np.float32)
        return BatchNormRecord(z, np.ones(c, dtype=np.float32), z + 1, z, 1e-5)

    spec = ModelSpec((1, 1, 784), [Input8Record(4096, 784, np.zeros((4096, 13), dtype=np.uint64)), bn(4096),
                                   dense(4096, 4096), bn(4096), dense(4096, 4096), bn(4096), dense(10, 4096), bn(10)])
    size = model_size(spec)
    assert size["reference_weights"] == 4 * (4096 * 784 + 4096 * 4096 * 2 + 10 * 4096)
    assert size["packed_weights"] == 8 * (4096 * 13 + 4096 * 64 * 2 + 10 * 64)
    mib = 1024 * 1024
    assert abs(size["reference"] / mib - 140.6) / 140.6 < 0.05
    assert abs(size["packed"] / mib - 4.6) / 4.6 < 0.05
    bc = model_size(zoo.bcnn_spec())
    assert bc["reference"] == 56149752 and bc["packed"] == 1815032  # SURVEY.md §6 (reference-measured)


def test_work_per_image():
    assert 2 * zoo.macs_per_image(zoo.bcnn_spec()) == 1233932288
    assert 2 * zoo.macs_per_image(zoo.bmlp_spec()) == 118571008


# (h, w, c, filters, pool, batch) -> fp4 conv kernel (b2_tc4_conv_path: 0 im2col,
# 1 split-K, 2 padded-row, 3 row-aligned padded-row).  Pins which kernel each
# GPU parity case of tests/test_gpu_tc.py exercises, and BCNN's layers at the
# bench batch.  Path choice is host logic: it runs without a GPU.
CONV_PATHS = [
    # 129-256 filters at K = 1152: 160 KB of resident weights leave no room for the
    # row-aligned kernel's input staging ring -> its register-prefetch producers
    ((32, 32, 128, 128, 1, 20), 3), ((16, 16, 128, 64, 0, 80), 3), ((16, 16, 128, 256, 0, 80), 3),
    ((64, 64, 128, 128, 1, 6), 3), ((8, 16, 128, 96, 1, 160), 3), ((4, 32, 128, 128, 0, 160), 3),
    ((8, 8, 128, 100, 1, 240), 0), ((62, 62, 128, 128, 0, 6), 2),
    ((16, 16, 128, 200, 1, 80), 3), ((16, 64, 128, 200, 1, 20), 3),
    ((8, 190, 128, 64, 0, 20), 2), ((8, 191, 128, 64, 0, 20), 0), ((32, 32, 128, 128, 1, 2), 0),
    ((4, 4, 512, 512, 1, 1), 1), ((8, 8, 512, 200, 0, 3), 1),
    # BCNN conv2..conv6 at 8192 images
    ((32, 32, 128, 128, 1, 8192), 3), ((16, 16, 128, 256, 0, 8192), 3), ((16, 16, 256, 256, 1, 8192), 0),
    ((8, 8, 256, 512, 0, 8192), 0), ((8, 8, 512, 512, 1, 8192), 0),
]


@pytest.mark.parametrize("shape,path", CONV_PATHS)
def test_conv_kernel_choice(shape, path):
    h, w, c, f, pool, batch = shape
    assert _lib._so.b2_tc4_conv_path(batch, h, w, c, f, 3, 3, 1, 1, pool) == path


def test_padrow_rejects_inexact_index_split():
    # a 4000 x 4000 1x1 conv would split virtual rows inexactly
    assert _lib._so.b2_tc4_conv_path(1, 4000, 4000, 128, 128, 1, 1, 1, 0, 0) == 0
