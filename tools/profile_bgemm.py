"""One bit-packed GEMM launch (for ncu captures): python tools/profile_bgemm.py [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_07175_b200 import _dev, gemm, zoo  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(n)
a = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
b = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
c = _dev.empty((n, n), np.int32)
b8 = _dev.tc_weights(b, n, n)
gemm.bgemm_device(a, n, b, n, n // 64, n, c, b_i8=b8)
torch.cuda.synchronize()
