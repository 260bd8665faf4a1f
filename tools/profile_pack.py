"""Launch the packing kernels once each on large inputs (for ncu captures).

    python tools/profile_pack.py [--reps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_07175_b200 import _dev, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    lines, bits = 262144, 4096
    x = torch.randn((lines, bits), dtype=torch.float32, device="cuda")
    o = _dev.empty((lines, bits // 64), np.uint64)
    u = torch.randint(0, 256, (1048576, 784), dtype=torch.uint8, device="cuda")
    p = _dev.empty((8, 1048576, 13), np.uint64)
    for _ in range(a.reps):
        _lib.call("b2_pack_lines_f32", _dev.P(x), lines, bits, _dev.P(o), _dev.stream())
        _lib.call("b2_pack_byte_planes", _dev.P(u), 1048576, 784, _dev.P(p), _dev.stream())
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
