"""Multi-GPU inference by batch slices.

Images are independent (no reference layer mixes images: network.py:506-522
runs one image at a time), so a batch shards into contiguous slices, one
per GPU, with NO collective on the data path.  One process per GPU
(torchrun), each holding its own Network replica, stream and pinned input
slice; the only cross-rank traffic is the optional gather of the
(N, classes) float64 scores to one rank for output, after compute.

    rank r of W owns images [lo_r, hi_r) with the first N % W ranks taking
    one extra image (shard_bounds).

The partition and gather logic is device-agnostic and is exercised with
the gloo backend on CPU (tests/test_shard.py); on the GPU box the same
code runs over NCCL.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of n images owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} world={world} rank={rank}")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def dist_info() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def gather_scores(local: np.ndarray, n: int, rank: int, world: int, dst: int = 0) -> np.ndarray | None:
    """Collect every rank's (slice, classes) float64 scores on `dst`
    (output collection after compute; not part of the timed data path).
    Returns the full (n, classes) array on `dst`, None elsewhere."""
    if world == 1:
        return local
    classes = local.shape[1]
    cap = -(-n // world)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    buf = torch.zeros((cap, classes), dtype=torch.float64, device=dev)
    buf[:local.shape[0]] = torch.from_numpy(local).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    if rank != dst:
        return None
    out = np.empty((n, classes), dtype=np.float64)
    for r, t in enumerate(parts):
        lo, hi = shard_bounds(n, world, r)
        out[lo:hi] = t[:hi - lo].cpu().numpy()
    return out


def forward_sharded(net, images: np.ndarray, rank: int | None = None, world: int | None = None,
                    gather: bool = True, compute=None):
    """Run this rank's slice of `images` through `net` (forward_batch) and,
    with `gather`, return the full score matrix on rank 0 (None on other
    ranks); without `gather`, return this rank's slice scores.  `compute`
    replaces forward_batch (tests drive the partition logic on CPU)."""
    if rank is None or world is None:
        rank, world = dist_info()
    from .network import forward_batch
    fn = compute or (lambda x: forward_batch(net, x))
    n = images.shape[0]
    lo, hi = shard_bounds(n, world, rank)
    local = fn(images[lo:hi]) if hi > lo else np.empty((0, _classes(net)), dtype=np.float64)
    if not gather:
        return local
    return gather_scores(np.ascontiguousarray(local, dtype=np.float64), n, rank, world)


def _classes(net) -> int:
    return int(getattr(net, "classes", 0))
