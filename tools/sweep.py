"""BASELINE configs[2] and [3]: standalone sweeps on one B200.

    python tools/sweep.py [--quick] > profiles/r01_sweeps.jsonl

* bgemm M=N=K in {1024, 2048, 4096, 8192, 16384}: int32 output
  (_kernels.py:85-106 bgemm_packed semantics) through gemm.bgemm_device on
  device-resident packed operands (B widened once, outside the timing, like
  a layer's weights); both engines.
* sign-pack (_kernels.py:43-54, float32 -> bits) and byte bit-planes
  (_kernels.py:67-82): HBM-bound, reported in GB/s of algorithmic bytes
  (input + output) against MEASURED_PEAKS.json's copy bandwidth.
* binary conv 3x3 / stride 1 / pad 1, C_in = C_out in {128, 256, 512, 1024},
  H = W in {8, 16, 32, 64}, batch 256, fused batchnorm-threshold + repack
  output (b2_tc_conv_bn_pack), i.e. a network conv stage.

Times are CUDA events over `reps` launches after 3 warm-ups, inputs larger
than or flushed from L2 between timed blocks; ops = 2 per binary MAC.  One
JSON line per case.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_07175_b200 import _dev, _lib, gemm, layers, zoo  # noqa: E402


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def bgemm_case(n, engine, flush, reps):
    rng = np.random.default_rng(n)
    wpl = n // 64
    a = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
    b = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
    out = _dev.empty((n, n), np.int32)
    fmt = _lib.TC_FORMAT
    b8 = _dev.tc_weights(b, n, n, fmt) if engine == "tc" else None
    ms = timed(lambda: gemm.bgemm_device(a, n, b, n, wpl, n, out, engine=engine, b_i8=b8, fmt=fmt), reps, flush)
    # spot-check 64 entries against the packed definition on the host
    ah, bh = _dev.download(a, np.uint64), _dev.download(b, np.uint64)
    got = _dev.download(out, np.int32)
    for i, j in zip(rng.integers(0, n, 64), rng.integers(0, n, 64)):
        ref = n - 2 * int(np.bitwise_count(ah[i] ^ bh[j]).sum())
        assert got[i, j] == ref, (n, i, j)
    ops = 2.0 * n ** 3
    return {"case": "bgemm", "engine": engine if engine != "tc" else "tc-" + fmt, "M": n, "N": n, "K": n, "ms": round(ms, 4),
            "Tops": round(ops / (ms / 1e3) / 1e12, 1), "Gops": round(ops / (ms / 1e3) / 1e9)}


def conv_case(c, hw, batch, flush, reps):
    rng = np.random.default_rng(c * 100 + hw)
    x = _dev.upload(zoo.pack_bits_host(rng.random((batch * hw * hw, c)) >= 0.5))
    w = _dev.upload(zoo.pack_bits_host(rng.random((c, 9 * c)) >= 0.5))
    w8 = _dev.tc_weights(w, c, 9 * c)
    bn = zoo.rand_bn(rng, c, 20.0)
    cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
    th = layers._thresh_struct(cal["thresh32"], cal["thresh64"], cal["ge"])
    out = _dev.empty((batch, hw * hw, -(-c // 64)), np.uint64)

    def run():
        _lib.call(_lib.tc_entry("conv_bn_pack"), _dev.P(x), batch, hw, hw, c, _dev.P(w8), c, 3, 3, 1, 1, 0,
                  layers._thresh_struct(cal["thresh32"], cal["thresh64"], cal["ge"]), _dev.P(out), _dev.stream())

    del th
    ms = timed(run, reps, flush)
    ops = 2.0 * batch * hw * hw * c * 9 * c
    return {"case": "conv3x3", "engine": "tc-" + _lib.TC_FORMAT, "C": c, "HW": hw, "batch": batch, "ms": round(ms, 4),
            "Tops": round(ops / (ms / 1e3) / 1e12, 1), "images_per_s": round(batch / (ms / 1e3))}


def pack_case(kind, flush, reps):
    rng = np.random.default_rng(3)
    if kind == "sign_pack_f32":
        lines, bits = 262144, 4096  # 4 GiB of float32 in, 128 MiB of words out
        x = torch.randn((lines, bits), dtype=torch.float32, device="cuda")
        out = _dev.empty((lines, bits // 64), np.uint64)
        fn = lambda: _lib.call("b2_pack_lines_f32", _dev.P(x), lines, bits, _dev.P(out), _dev.stream())  # noqa: E731
        nbytes = lines * bits * 4 + lines * bits // 8
        ref_in = x[:4].cpu().numpy()
        fn()
        got = _dev.download(out[:4], np.uint64)
        want = zoo.pack_bits_host(~(ref_in < 0))
        assert np.array_equal(got, want)
    else:
        lines, bits = 1048576, 784  # MNIST-shaped bytes -> 8 bit-planes
        x = torch.from_numpy(rng.integers(0, 256, (lines, bits), dtype=np.uint8)).cuda()
        out = _dev.empty((8, lines, -(-bits // 64)), np.uint64)
        fn = lambda: _lib.call("b2_pack_byte_planes", _dev.P(x), lines, bits, _dev.P(out), _dev.stream())  # noqa: E731
        nbytes = lines * bits + 8 * lines * (-(-bits // 64)) * 8
    ms = timed(fn, reps, flush)
    import json as _j
    peak = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    gbs = nbytes / (ms / 1e3) / 1e9
    return {"case": kind, "lines": lines, "bits": bits, "ms": round(ms, 4), "GBps": round(gbs, 1),
            "frac_of_hbm": round(gbs / peak, 3), "hbm_peak_GBps": peak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sizes = [1024, 2048, 4096, 8192] if a.quick else [1024, 2048, 4096, 8192, 16384]
    for n in sizes:
        for engine in ("tc", "popc"):
            if engine == "popc" and n > 8192:
                continue
            print(json.dumps(bgemm_case(n, engine, flush, 3 if n >= 8192 else 10)), flush=True)
    for kind in ("sign_pack_f32", "byte_planes"):
        print(json.dumps(pack_case(kind, flush, 5)), flush=True)
    for c in (128, 256, 512, 1024):
        for hw in (8, 16, 32, 64):
            if a.quick and (c, hw) not in ((128, 32), (512, 8)):
                continue
            print(json.dumps(conv_case(c, hw, 256, flush, 5)), flush=True)


if __name__ == "__main__":
    main()
