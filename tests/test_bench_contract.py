"""bench.py contract pieces that run without a GPU.

* The reference arm (`bench.py --impl reference`) runs the unmodified
  reference package from baseline/_ref and must not import or map this
  package's code or CUDA library (the arm's process once mapped
  libbitnn_b200.so through an import side effect).
* Both arms emit the same `config` dict.
* baseline/ref_arm.py builds the BASELINE models with the reference's own
  classes; their bytes hash to the golden SHA-256 that zoo.py's specs hash to.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from baseline import ref_arm  # noqa: E402

needs_ref = pytest.mark.skipif(not ref_arm.available(), reason="reference not installed in baseline/_ref")

PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample", "1"] + sys.argv[1:]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
mods = [m for m in sys.modules if m.startswith("paper_1705_07175_b200") or m == "torch"]
print(json.dumps({"libbitnn_mapped": "libbitnn" in maps, "product_modules": mods}))
"""


@needs_ref
@pytest.mark.parametrize("workload", ["bcnn", "bmlp"])
def test_reference_arm_maps_no_product_code(workload):
    res = subprocess.run([sys.executable, "-c", PROBE, "--workload", workload], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(x) for x in res.stdout.strip().splitlines()]
    line, probe = lines[0], lines[1]
    assert line["impl"] == "reference" and line["unit"] == "images/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "images/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert not probe["libbitnn_mapped"], "reference arm mapped the product library"
    assert probe["product_modules"] == [], probe["product_modules"]


def test_config_identical_across_arms():
    import argparse

    import bench
    for wl in ("bcnn", "bmlp"):
        for world in (1, 2, 8):
            a = argparse.Namespace(workload=wl, batch=bench.DEFAULT_BATCH[wl])
            assert bench.config_dict(a, world) == bench.config_dict(argparse.Namespace(**vars(a)), world)
            assert bench.config_dict(a, world)["images_per_gpu_per_step"] * world >= a.batch
    assert bench.DEFAULT_BATCH["bcnn"] == 65536  # BASELINE configs[4]


@needs_ref
@pytest.mark.parametrize("name", ["bcnn", "bmlp"])
def test_ref_arm_models_hash_to_golden(name, networks_golden):
    ref_arm.import_bitnn()
    net, shape = ref_arm.model(name)  # raises on a hash mismatch
    assert shape == ref_arm.SHAPES[name]


def test_bench_images_match_ref_arm_images():
    """The product arm's seeded batch and the reference arm's sample are the
    same images (same rng stream), so both arms time the same input."""
    import numpy as np

    import bench
    for name in ("bcnn", "bmlp"):
        full = bench.bench_images(name, 64, 1000)
        rng = np.random.default_rng(1000)
        sample = rng.integers(0, 256, (8,) + ref_arm.SHAPES[name], dtype=np.uint8)
        assert np.array_equal(full[:8].reshape(sample.shape), sample)
