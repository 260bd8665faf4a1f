"""Opt-in kernel variants stay bit-exact: each environment switch is read
once per process, so the relevant parity cases re-run in a child pytest
with the switch set.

* B2_MCAST=1 — conv weight stages shared by CTA pairs through TMA multicast
  (tc_i8.cuh MC; off by default);
* B2_PADROW_TW=1 — the row-aligned padded-row conv with the filters on the
  MMA's M side and the weights in TMEM (tc_padrow.cuh TW);
* B2_ALIGN_SPLIT=0 — 129-256 filters in one 256-column row-aligned launch;
* B2_ALIGN_NOBIAS=1 — the row-aligned kernels with the threshold table
  instead of the folded threshold MMA.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    ("B2_MCAST", "1", "conv_bn_pack_vs_oracle and (16-16-256-256 or 8-8-512-512 or 8-8-256-512)"),
    ("B2_PADROW_TW", "1", "conv_bn_pack_vs_oracle and (32-32-128-128 or 8-16-128-96 or 4-32-128-128)"),
    ("B2_ALIGN_SPLIT", "0", "conv_bn_pack_vs_oracle and (16-16-128-256 or 16-16-128-200)"),
    ("B2_ALIGN_NOBIAS", "1", "conv_bn_pack_vs_oracle and (32-32-128-128 or 16-16-128-256)"),
]


@pytest.mark.parametrize("var,value,select", CASES)
def test_optin_variant_parity(var, value, select):
    env = dict(os.environ, **{var: value})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", select,
                        os.path.join(ROOT, "tests", "test_gpu_tc.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "deselected" in r.stdout, tail
