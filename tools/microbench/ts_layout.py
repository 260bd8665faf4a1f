"""Decode tools/microbench/ts_layout.cu's dump: which TMEM nibble -> K mapping
of a kind::mxf4 A operand reproduces the MMA's D (B's smem order taken as
k = 32 plane + 2 byte + nibble)."""

import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
aw = np.frombuffer(raw[:128 * 16 * 4], np.uint32).reshape(128, 16)
bb = np.frombuffer(raw[128 * 16 * 4:128 * 16 * 4 + 4096], np.uint8).reshape(2, 2048)
d = np.frombuffer(raw[128 * 16 * 4 + 4096:], np.float32).reshape(128, 128)
val = {0x0: 0, 0x2: 1, 0xA: -1}


def nib(x, j):
    return (x >> (4 * j)) & 0xF


def b_matrix(swap):
    B = np.zeros((128, 64), np.int64)
    for p in range(2):
        for n in range(128):
            for b in range(16):
                byte = int(bb[p, n * 16 + b])
                lo, hi = (byte >> 4, byte & 0xF) if swap else (byte & 0xF, byte >> 4)
                B[n, 32 * p + 2 * b] = val[lo]
                B[n, 32 * p + 2 * b + 1] = val[hi]
    return B


def a_matrix(mapping):
    A = np.zeros((128, 64), np.int64)
    for m in range(128):
        for c in range(16):
            for j in range(8):
                k = mapping(c, j)
                if k is not None:
                    A[m, k] = val[int(nib(int(aw[m, c]), j))]
    return A


hyps = {
    "packed: k = 8 col + nibble": lambda c, j: 8 * c + j if c < 8 else None,
    "bytes: k = 4 col + byte (low nibble)": lambda c, j: 4 * c + j // 2 if j % 2 == 0 else None,
    "bytes: k = 4 col + byte (high nibble)": lambda c, j: 4 * c + j // 2 if j % 2 == 1 else None,
}
for swap in (False, True):
    B = b_matrix(swap)
    for name, h in hyps.items():
        D = a_matrix(h) @ B.T
        print(f"B nibbles swapped={swap} | {name}: match={np.array_equal(D, d.astype(np.int64))} "
              f"mism={int((D != d).sum())}")
print("d[0,:8] =", d[0, :8])
