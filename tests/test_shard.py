"""Batch-slice sharding on CPU with the gloo backend,
world_size 2: the partition covers every image exactly once, and a
sharded forward + gather equals the single-process result bit for bit.
The per-rank compute is the CPU oracle (test infrastructure), so these
tests run without a GPU; on the B200 box the same code runs over NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_07175_b200.shard import forward_sharded, shard_bounds


@pytest.mark.parametrize("n", [0, 1, 7, 64, 65536, 65537])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_partition(n, world):
    spans = [shard_bounds(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (lo, hi), (lo2, _) in zip(spans, spans[1:]):
        assert hi == lo2
    sizes = [hi - lo for lo, hi in spans]
    assert max(sizes) - min(sizes) <= 1


def test_shard_bounds_rejects_bad_args():
    with pytest.raises(ValueError):
        shard_bounds(10, 0, 0)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, spec_path, images, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        from paper_1705_07175_b200.modelfile import load_model
        ref = o.OracleNetwork(load_model(spec_path))
        out = forward_sharded(None, images, rank, world, compute=ref.forward_batch)
        if rank == 0:
            np.save(result_path, out)
        else:
            assert out is None
        local = forward_sharded(None, images, rank, world, gather=False, compute=ref.forward_batch)
        lo, hi = shard_bounds(images.shape[0], world, rank)
        assert local.shape[0] == hi - lo
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [5, 24])
def test_sharded_forward_gloo_world2(tmp_path, n):
    from conftest import GOLDEN
    from oracle import oracle as o
    from paper_1705_07175_b200.modelfile import load_model
    spec_path = os.path.join(GOLDEN, "cnn.bdnn")
    g = np.load(os.path.join(GOLDEN, "networks.npz"))
    images = np.ascontiguousarray(g["cnn_images"][:n])
    result = tmp_path / "scores.npy"
    mp.start_processes(_worker, args=(2, _free_port(), spec_path, images, str(result)), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(result)
    want = o.OracleNetwork(load_model(spec_path)).forward_batch(images)
    assert np.array_equal(got, want)
    assert np.array_equal(got, g["cnn_scores"][:n])
