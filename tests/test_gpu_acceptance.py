"""GPU parity against the REFERENCE on the wider round-2 fixture set
(tests/golden/acceptance.npz, written by make_golden.py from the reference):

* the reference's acceptance CNN (pkg/tests/test_acceptance.py:80-98) on its
  1000-image cross-backend check (:166-179) — our scores equal the packed
  backend's float64 scores bit for bit, argmax equals the float reference
  backend's and the gap stays below 1e-4; its 32-channel convs take the
  CUDA-core POPC kernels (c % 64 != 0), pinned here to the reference directly;
* 1024 distinct images through the BASELINE BCNN and BMLP at batch 1024 —
  large enough for the fused first layer and the row-aligned padded-row conv
  (the kernels the bench times) — plus the same images split over two
  processes sharing cuda:0 (forward_sharded / classify_images(sharded=True),
  gloo for the gather), i.e. the multi-GPU path on one device.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from acceptance_set import GOLDEN, images1024, vgg_set
from paper_1705_07175_b200 import _lib, forward_batch, zoo
from paper_1705_07175_b200.network import Network

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acc():
    return np.load(os.path.join(GOLDEN, "acceptance.npz"))


def test_reference_acceptance_cnn_1000_images(acc):
    spec, imgs = vgg_set()
    net = Network(spec, max_batch=1000)
    got = forward_batch(net, imgs)
    assert np.array_equal(got, acc["vgg_packed_scores"])
    assert np.array_equal(np.argmax(got, 1), np.argmax(acc["vgg_reference_scores"], 1))
    assert float(np.max(np.abs(got - acc["vgg_reference_scores"]))) < 1e-4  # test_acceptance.py:179


@pytest.mark.parametrize("name", ["bcnn", "bmlp"])
def test_baseline_models_1024_distinct_images(acc, name):
    spec = zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()
    x = images1024(name)
    net = Network(spec, max_batch=1024)
    assert np.array_equal(forward_batch(net, x), acc[f"{name}1024_scores"])
    if name == "bcnn":  # the timed kernels engage at this batch
        assert _lib._so.b2_tc_byte_conv_path(1024, 32, 32, 3, 128, 3, 3, 1, 1, 0) == 1
        assert _lib._so.b2_tc4_conv_path(1024, 32, 32, 128, 128, 3, 3, 1, 1, 1) == 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)  # two ranks share one GPU: no NCCL
    try:
        import torch

        from paper_1705_07175_b200.datasets import classify_images
        from paper_1705_07175_b200.shard import forward_sharded
        torch.cuda.set_device(0)
        spec = zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()
        x = images1024(name)
        net = Network(spec, max_batch=512)
        scores = forward_sharded(net, x.reshape(x.shape[0], -1), rank, world)
        res = classify_images(net, x, sharded=True)
        if rank == 0:
            np.save(result_path, scores)
            np.save(str(result_path) + ".pred.npy", res["predictions"])
        else:
            assert scores is None and res == {}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["bcnn", "bmlp"])
def test_sharded_two_processes_one_gpu(tmp_path, acc, name):
    result = tmp_path / "scores.npy"
    mp.start_processes(_worker, args=(2, _free_port(), name, str(result)), nprocs=2, join=True,
                       start_method="spawn")
    want = acc[f"{name}1024_scores"]
    assert np.array_equal(np.load(result), want)
    assert np.array_equal(np.load(str(result) + ".pred.npy"), np.argmax(want, 1))
