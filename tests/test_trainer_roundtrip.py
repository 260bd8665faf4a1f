"""Trainer export round trip (the reference's
pkg/trainer/tests/test_train.py:62-78 on a synthetic MNIST-format set, MNIST
itself not being in this image): a 784-256-256-10 binary MLP trained by the
REFERENCE trainer and exported by its own writer (tests/golden/
make_trainer_golden.py) loads here, and this package's GPU classify agrees
with the trainer's float64 evaluation on every test image (the reference
requires >= 99.9 %) and reproduces the reference engine's scores bit for bit,
read through the MNIST IDX ingest path."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1705_07175_b200 import load, modelfile
from trainer_set import make_set, write_idx

MODEL = os.path.join(GOLDEN, "trained_mlp.bdnn")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "trainer.npz"))


def test_trained_model_parses_and_oracle_matches_engine(golden, oracle):
    spec = modelfile.load_model(MODEL)
    assert spec.input_dims == (28, 28, 1) and [getattr(r, "units", None) for r in spec.records][::2] == [256, 256, 10]
    _, _, vx, vy = make_set()
    net = oracle.OracleNetwork(spec)
    got = np.stack([net.forward(im.reshape(-1)) for im in vx[:200]])
    assert np.array_equal(got, golden["engine_scores"][:200])
    assert np.array_equal(np.argmax(got, 1), golden["trainer_preds"][:200])


@pytest.mark.gpu
def test_gpu_classify_agrees_with_trainer(golden, tmp_path):
    from paper_1705_07175_b200.datasets import classify_images, discover
    from paper_1705_07175_b200 import forward_batch
    tx, ty, vx, vy = make_set()
    write_idx(str(tmp_path), tx[:10], ty[:10], vx, vy)
    ds = discover(str(tmp_path))  # t10k split first, as the reference CLI
    assert ds.count == vx.shape[0] and np.array_equal(ds.labels, vy)
    net = load(MODEL)
    res = classify_images(net, ds.images, ds.labels)
    agreement = float(np.mean(res["predictions"] == golden["trainer_preds"]))
    assert agreement >= 0.999  # test_train.py:76
    assert abs(res["accuracy"] - float(golden["trainer_accuracy"])) <= 0.001  # test_train.py:77
    assert np.array_equal(forward_batch(net, ds.images.reshape(ds.count, -1)), golden["engine_scores"])
