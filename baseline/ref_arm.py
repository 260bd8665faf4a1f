"""Reference arm: the UNMODIFIED reference package `bitnn` timed on host cores.

The driver installs the reference once into ``baseline/_ref``
(``pip install --no-index --no-build-isolation --find-links /opt/wheelhouse
--target baseline/_ref --no-deps <copy of /root/reference/pkg>``); this
module imports it from there and times its own public API and stock code
path (the packed Numba backend), with ``NUMBA_NUM_THREADS`` = every host core
this process may run on:

* networks: ``bitnn.network.forward`` image by image, exactly the loop of
  ``/root/reference/pkg/src/bitnn/cli.py:101-104`` (the reference is batch-1
  only, ``network.py:506-522``);
* the bit-packed GEMM sweep (BASELINE configs[2]): ``bitnn.gemm.bgemm`` on
  ``PackedMatrixA/B.from_float`` operands built as
  ``bitnn/bench.py:79-90`` builds them (``_kernels.bgemm_packed``,
  ``_kernels.py:85-106``);
* the conv sweep (configs[3]): ``bitnn.layers.conv_forward``
  (``layers.py:255-266``) on ``ConvLayer.from_float`` layers.

Nothing from the product package (paper_1705_07175_b200) or its CUDA
library is imported here: this process maps no product code.  The models
are built with the reference's own record classes from the seeded recipe
documented in paper_1705_07175_b200/zoo.py, and their serialized bytes are
checked against the SHA-256 committed in tests/golden/networks.npz, so both
arms run the same model on the same kind of input.

    python baseline/ref_arm.py --what all --seconds 8     # JSON on stdout
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_DIR = os.path.join(HERE, "_ref")


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "bitnn"))


def import_bitnn():
    """Import the driver-installed reference with all host threads."""
    if not available():
        raise ImportError(f"reference not installed in {REF_DIR}")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(host_cores()))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/b2_ref_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import bitnn  # noqa: F401
    return bitnn


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# --------------------------------------------------------------------------- models (reference classes)

def _pm1(rng, *shape):
    return np.where(rng.random(shape) < 0.5, -1.0, 1.0).astype(np.float32)


def _rows(rng, rows, k):
    from bitnn.gemm import PackedMatrixA
    return PackedMatrixA.from_float(_pm1(rng, rows, k)).words


def _bn(rng, c, spread):
    from bitnn.modelfile import BatchNormRecord
    return BatchNormRecord((rng.standard_normal(c) * spread).astype(np.float32),
                           (rng.random(c) * 50 + 1).astype(np.float32),
                           rng.standard_normal(c).astype(np.float32),
                           rng.standard_normal(c).astype(np.float32), 1e-5)


def bmlp_spec(seed=0x784):
    """BASELINE configs[0] model, recipe of paper_1705_07175_b200/zoo.py:bmlp_spec."""
    from bitnn.modelfile import DenseRecord, Input8Record, ModelSpec
    rng = np.random.default_rng(seed)
    return ModelSpec((1, 1, 784), [
        Input8Record(4096, 784, _rows(rng, 4096, 784)), _bn(rng, 4096, 5000.0),
        DenseRecord(4096, 4096, _rows(rng, 4096, 4096)), _bn(rng, 4096, 60.0),
        DenseRecord(4096, 4096, _rows(rng, 4096, 4096)), _bn(rng, 4096, 60.0),
        DenseRecord(10, 4096, _rows(rng, 10, 4096)), _bn(rng, 10, 4.0),
    ])


def bcnn_spec(seed=0x1705):
    """BASELINE configs[1]/[4] model, recipe of paper_1705_07175_b200/zoo.py:bcnn_spec."""
    from bitnn.modelfile import ConvRecord, DenseRecord, MaxPoolRecord, ModelSpec
    rng = np.random.default_rng(seed)
    return ModelSpec((32, 32, 3), [
        _bn(rng, 3, 100.0),
        ConvRecord(128, 3, 3, 1, 1, 3, _rows(rng, 128, 27)), _bn(rng, 128, 8.0),
        ConvRecord(128, 3, 3, 1, 1, 128, _rows(rng, 128, 1152)), MaxPoolRecord(2, 2, 2), _bn(rng, 128, 40.0),
        ConvRecord(256, 3, 3, 1, 1, 128, _rows(rng, 256, 1152)), _bn(rng, 256, 30.0),
        ConvRecord(256, 3, 3, 1, 1, 256, _rows(rng, 256, 2304)), MaxPoolRecord(2, 2, 2), _bn(rng, 256, 60.0),
        ConvRecord(512, 3, 3, 1, 1, 256, _rows(rng, 512, 2304)), _bn(rng, 512, 45.0),
        ConvRecord(512, 3, 3, 1, 1, 512, _rows(rng, 512, 4608)), MaxPoolRecord(2, 2, 2), _bn(rng, 512, 80.0),
        DenseRecord(1024, 8192, _rows(rng, 1024, 8192)), _bn(rng, 1024, 80.0),
        DenseRecord(1024, 1024, _rows(rng, 1024, 1024)), _bn(rng, 1024, 30.0),
        DenseRecord(10, 1024, _rows(rng, 10, 1024)), _bn(rng, 10, 4.0),
    ])


SHAPES = {"bcnn": (32, 32, 3), "bmlp": (784,)}


def model(name):
    """(reference Network, input shape); the model bytes must hash to the golden SHA."""
    from bitnn.modelfile import write_model
    from bitnn.network import Network
    spec = bcnn_spec() if name == "bcnn" else bmlp_spec()
    sha = hashlib.sha256(write_model(spec)).hexdigest()
    golden = np.load(os.path.join(ROOT, "tests", "golden", "networks.npz"))
    if sha != str(golden[f"{name}_sha256"]):
        raise RuntimeError(f"{name}: reference-built model hash {sha} != golden {golden[name + '_sha256']}")
    return Network(spec), SHAPES[name]


# --------------------------------------------------------------------------- timers

def time_network(name, images_per_step, steps, warmup, seed=1000):
    """Per-step seconds of the reference forward loop (cli.py:101-104) over
    `images_per_step` seeded images (the same rng recipe as the product
    arm's bench input)."""
    from bitnn.network import forward
    net, shape = model(name)
    rng = np.random.default_rng(seed)
    imgs = rng.integers(0, 256, (images_per_step,) + shape, dtype=np.uint8)
    preds = np.empty(images_per_step, dtype=np.int64)
    for _ in range(warmup):
        for i in range(images_per_step):
            preds[i] = int(np.argmax(forward(net, imgs[i])))
    per_step = []
    for _ in range(steps):
        t0 = time.perf_counter()
        for i in range(images_per_step):
            preds[i] = int(np.argmax(forward(net, imgs[i])))
        per_step.append(time.perf_counter() - t0)
    return per_step


def rate_network(name, seconds, min_images=8, seed=1000):
    """images/s of the reference forward loop over about `seconds`."""
    from bitnn.network import forward
    net, shape = model(name)
    rng = np.random.default_rng(seed)
    imgs = rng.integers(0, 256, (64,) + shape, dtype=np.uint8)
    for i in range(3):
        forward(net, imgs[i])
    n, t0 = 0, time.perf_counter()
    while True:
        int(np.argmax(forward(net, imgs[n % 64])))
        n += 1
        dt = time.perf_counter() - t0
        if n >= min_images and dt >= seconds:
            return {"images_per_s": n / dt, "images": n, "seconds": round(dt, 3)}


def rate_bgemm(n, budget_s, seed=0):
    """`bitnn.gemm.bgemm` on n^3 +/-1 operands built as bitnn/bench.py:83-87."""
    from bitnn.gemm import PackedMatrixA, PackedMatrixB, bgemm
    rng = np.random.default_rng(seed)
    pa = PackedMatrixA.from_float(_pm1(rng, n, n))
    pb = PackedMatrixB.from_float(_pm1(rng, n, n))
    out = np.zeros((n, n), dtype=np.int32)
    bgemm(pa, pb, out=out)  # compile / warm
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        bgemm(pa, pb, out=out)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() >= t_end or len(times) >= 20:
            break
    t = float(np.median(times))
    return {"gops": 2.0 * n ** 3 / t / 1e9, "ms": t * 1e3, "iters": len(times),
            "checksum": int(np.sum(out, dtype=np.int64))}


def rate_conv(c, hw, budget_s=0.4, max_images=32, seed=0):
    """`bitnn.layers.conv_forward` (3x3, stride 1, pad 1, C_in = C_out = c)
    on hw x hw images (the reference convolves one image per call), at least
    2 images and about `budget_s`; returns per-image ms."""
    from bitnn.layers import ConvLayer, conv_forward
    from bitnn.tensor import FloatTensor, pack
    rng = np.random.default_rng(seed)
    layer = ConvLayer.from_float(_pm1(rng, 9 * c, c), (3, 3), 1, 1, (hw, hw, c))
    x = pack(FloatTensor(_pm1(rng, hw, hw, c)))
    conv_forward(layer, x)  # compile / warm
    n, t0 = 0, time.perf_counter()
    while True:
        conv_forward(layer, x)
        n += 1
        dt = time.perf_counter() - t0
        if n >= max_images or (n >= 2 and dt >= budget_s):
            break
    dt /= n
    return {"ms_per_image": dt * 1e3, "gops": 2.0 * hw * hw * c * 9 * c / dt / 1e9, "sample_images": n}


def check_parity(path):
    """Scores of the product's timed batch (a sample saved by bench.py)
    against the reference's own `forward` on the same images: bit-exact
    float64 (tolerance 0) and identical argmax (lowest index on ties)."""
    from bitnn.network import forward
    d = np.load(path)
    name = str(d["workload"])
    net, shape = model(name)
    imgs, theirs = d["images"], d["scores"]
    ref = np.stack([forward(net, imgs[i].reshape(shape)).copy() for i in range(imgs.shape[0])])
    return {"images": int(imgs.shape[0]), "of_batch_indices": [int(d["global_index"][0]), int(d["global_index"][-1])],
            "bit_exact": bool(np.array_equal(ref, theirs)), "max_abs_diff": float(np.max(np.abs(ref - theirs))),
            "argmax_agree": int(np.sum(np.argmax(ref, 1) == np.argmax(theirs, 1))),
            "vs": "reference bitnn.network.forward (baseline/_ref), float64 scores, tolerance 0"}


def describe():
    import numba
    try:
        layer = numba.threading_layer()
    except ValueError:  # no parallel region run yet
        layer = "not initialised"
    return {"cores": numba.get_num_threads(), "host_cores": host_cores(), "cpu_model": cpu_model(),
            "numba": numba.__version__, "threading_layer": layer, "kind": "reference",
            "source": "baseline/_ref (unmodified reference bitnn, packed Numba backend)"}


# conv sweep points (configs[3]): C x spatial, batch 256 -> sampled images per point
CONV_POINTS = [(c, hw) for c in (128, 256, 512, 1024) for hw in (8, 16, 32, 64)]
GEMM_SIZES = (1024, 2048, 4096, 8192, 16384)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="all", help="comma list of bcnn,bmlp,bgemm,conv or all")
    ap.add_argument("--seconds", type=float, default=8.0, help="per network")
    ap.add_argument("--gemm-seconds", type=float, default=2.0, help="per GEMM size")
    ap.add_argument("--parity", default=None, help="npz of product scores to check against the reference")
    args = ap.parse_args(argv)
    import_bitnn()
    what = {"bcnn", "bmlp", "bgemm", "conv"} if args.what == "all" else set(args.what.split(","))
    out = {}
    for name in ("bcnn", "bmlp"):
        if name in what:
            out[name] = rate_network(name, args.seconds)
    if "bgemm" in what:
        out["bgemm"] = {str(n): rate_bgemm(n, args.gemm_seconds) for n in GEMM_SIZES}
    if "conv" in what:
        out["conv"] = {f"C{c}_{hw}px": rate_conv(c, hw) for c, hw in CONV_POINTS}
    if args.parity:
        out["parity"] = check_parity(args.parity)
    out["host"] = describe()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
