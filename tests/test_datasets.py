"""Dataset ingest (bitnn/datasets.py formats) on CPU, and the batched
classify front end on the GPU against the reference's golden scores."""

import os

import numpy as np
import pytest

from paper_1705_07175_b200.datasets import (DatasetError, classify_images, discover, read_cifar10, read_idx_images,
                                            read_idx_labels, read_mnist)


def write_idx(path, magic, dims, payload):
    with open(path, "wb") as f:
        f.write(magic.to_bytes(4, "big"))
        for d in dims:
            f.write(int(d).to_bytes(4, "big"))
        f.write(payload)


def test_mnist_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    imgs = rng.integers(0, 256, (7, 28, 28), dtype=np.uint8)
    labels = rng.integers(0, 10, 7, dtype=np.uint8)
    write_idx(tmp_path / "t10k-images-idx3-ubyte", 0x803, imgs.shape, imgs.tobytes())
    write_idx(tmp_path / "t10k-labels-idx1-ubyte", 0x801, (7,), labels.tobytes())
    ds = discover(tmp_path)
    assert ds.kind == "mnist-idx" and ds.count == 7
    assert np.array_equal(ds.images[..., 0], imgs) and ds.images.shape == (7, 28, 28, 1)
    assert np.array_equal(ds.labels, labels)


def test_mnist_errors(tmp_path):
    p = tmp_path / "x"
    write_idx(p, 0x804, (1, 2, 2), b"\0" * 4)
    with pytest.raises(DatasetError, match="magic"):
        read_idx_images(p)
    write_idx(p, 0x803, (2, 2, 2), b"\0" * 4)
    with pytest.raises(DatasetError, match="promises"):
        read_idx_images(p)
    p.write_bytes(b"\0\0\x08")
    with pytest.raises(DatasetError, match="truncated"):
        read_idx_images(p)
    write_idx(p, 0x801, (3,), b"\0" * 2)
    with pytest.raises(DatasetError, match="promises"):
        read_idx_labels(p)
    write_idx(tmp_path / "i", 0x803, (2, 1, 1), b"\0" * 2)
    write_idx(tmp_path / "l", 0x801, (3,), b"\0" * 3)
    with pytest.raises(DatasetError, match="does not match"):
        read_mnist(tmp_path / "i", tmp_path / "l")
    with pytest.raises(DatasetError, match="cannot read"):
        read_idx_images(tmp_path / "missing")


def test_cifar_planar_to_interleaved(tmp_path):
    rng = np.random.default_rng(2)
    planar = rng.integers(0, 256, (5, 3, 32, 32), dtype=np.uint8)
    labels = rng.integers(0, 10, 5, dtype=np.uint8)
    rows = np.concatenate([labels[:, None], planar.reshape(5, -1)], axis=1)
    (tmp_path / "data_batch_1.bin").write_bytes(rows[:3].tobytes())
    (tmp_path / "data_batch_2.bin").write_bytes(rows[3:].tobytes())
    ds = discover(tmp_path)
    assert ds.kind == "cifar10-binary" and ds.count == 5
    assert np.array_equal(ds.images, planar.transpose(0, 2, 3, 1))
    assert np.array_equal(ds.labels, labels)
    (tmp_path / "bad.bin").write_bytes(b"\0" * 100)
    with pytest.raises(DatasetError, match="whole number"):
        read_cifar10(tmp_path / "bad.bin")
    with pytest.raises(DatasetError, match="no CIFAR"):
        read_cifar10([])


def test_discover_nothing(tmp_path):
    with pytest.raises(DatasetError, match="no MNIST"):
        discover(tmp_path)


@pytest.mark.gpu
def test_classify_cifar_file_matches_reference(tmp_path, networks_golden):
    """CIFAR-10 binary file -> batched classify == argmax of the reference's scores."""
    from paper_1705_07175_b200 import zoo
    from paper_1705_07175_b200.network import Network
    imgs = networks_golden["bcnn_images"]
    want = networks_golden["bcnn_scores"]
    labels = np.argmax(want, axis=1).astype(np.uint8)
    rows = np.concatenate([labels[:, None], imgs.transpose(0, 3, 1, 2).reshape(len(imgs), -1)], axis=1)
    (tmp_path / "test_batch.bin").write_bytes(rows.tobytes())
    ds = discover(tmp_path)
    net = Network(zoo.bcnn_spec(), max_batch=len(imgs))
    res = classify_images(net, ds.images, ds.labels)
    assert np.array_equal(res["predictions"], np.argmax(want, axis=1))
    assert res["accuracy"] == 1.0
