#!/usr/bin/env python
"""Benchmark: binary forward pass on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload bcnn|bmlp]
                    [--batch GLOBAL] [--impl ours|reference] [--no-cpu] [--no-extra]

Workload (config.workload): BASELINE configs[4], the BCNN CIFAR-10 network
on a FIXED global batch of 65536 synthetic 32x32x3 u8 images, sliced into
contiguous per-GPU slices (65536 / 32768 / 16384 / 8192 images at N = 1 / 2 /
4 / 8: strong scaling).  Images are independent, so there is no collective
on the data path — the only NCCL calls are the barrier and the max-over-ranks
reduction of the timings.  Multi-GPU runs are launched with torchrun, one
rank per GPU.  `--workload bmlp` runs configs[0]'s model instead.

`value`  — device throughput: inputs resident in HBM, K steps timed with CUDA
           events on the launching stream (each step is one CUDA-graph replay
           of the whole network), L2 flushed (256 MB write) between steps.
`e2e`    — the same metric through the public API `forward_batch` with host
           u8 images in page-locked memory: H2D of every step's inputs +
           forward + D2H of the float64 scores inside the timed region.
`roofline` — per-stage device times; the dominant stage's achieved ops/s (2
           per binary MAC) against the dense tensor peak of its operand format
           derived from MEASURED_PEAKS.json (fp4 = 4 x bf16, int8 = 2 x bf16);
           the same-run cuBLASLt NVFP4 / int8 GEMMs are reported beside it.
`parity_checked` — a sample of the timed batch's scores compared bit for bit
           with the REFERENCE package's own `forward` on the same images.
`cpu_baseline` / `--impl reference` — the unmodified reference `bitnn`
           (installed by the driver in baseline/_ref) timed through its own
           API on all host cores (baseline/ref_arm.py, run as a separate
           process that maps none of this package's code); the oracle port
           only if the reference is not installed.
`sweeps` — BASELINE configs[0]/[1] batch sizes (device and e2e), configs[2]
           (bgemm 1024-16384, with cuBLASLt NVFP4 at the same size) and
           configs[3] (3x3 conv, C 128-1024, 8-64 px, batch 256), each with
           the reference's CPU figure from the same run.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "images/sec (BMLP MNIST, BCNN CIFAR-10) at 1/2/4/8 B200; binary GEMM Gop/s"
# Measured POPC pipe rate (tools/microbench/pipes.cu on this pool's B200:
# 15.66 POPC/clk/SM -> 4.555e12 popc/s x 32 bit-MAC x 2 = 291.5 T bit-op/s).
POPC_PEAK_TBITOPS = 4.555e12 * 64 / 1e12
POPC_PEAK_SOURCE = "tools/microbench/pipes.cu popc_xor on B200 (profiles/pipes_r01.jsonl): 15.66 POPC/clk/SM"
DEFAULT_BATCH = {"bcnn": 65536, "bmlp": 16384}
SHAPES = {"bcnn": (32, 32, 3), "bmlp": (784,)}
WORKLOADS = {
    "bcnn": "BCNN VGG-style CIFAR-10 2x128C3-MP2-2x256C3-MP2-2x512C3-MP2-1024FC-1024FC-10, 32x32x3 u8 "
            "(BASELINE configs[4]: fixed global batch sliced across GPUs)",
    "bmlp": "BinaryNet MLP 784-4096-4096-4096-10 on MNIST-shaped u8 (BASELINE configs[0] model)",
}
DTYPE = ("u1 packed (+/-1) activations; tensor-core operands e2m1 (fp4, unit block scales) or s8 (u8-input "
         "layer), exact fp32 / s32 accumulators; f64 scores")


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def config_dict(args, world):
    """Identical in both arms (the reference arm describes its sample in
    cpu_baseline.sample, not here)."""
    return {"workload": WORKLOADS[args.workload], "global_batch": args.batch,
            "images_per_gpu_per_step": -(-args.batch // world),
            "parallelism": f"dp{world} (contiguous batch slices, no collective)",
            "l2": "flushed between timed steps (256 MB write)",
            "weights": "seeded random +/-1 (paper_1705_07175_b200/zoo.py recipe; model SHA-256 in "
                       "tests/golden/networks.npz)"}


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line).

    Started before the warm-up so the first sample exists when timing
    begins; `mark()` brackets the timed region and `summary()` keeps the
    samples taken inside it (each line is timestamped on arrival)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 20):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            deadline = time.time() + 5.0
            while not self.lines and time.time() < deadline:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(2 * self.period_ms / 1e3)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = self.t1 if self.t1 is not None else time.time()
        inside = [ln for ts, ln in self.lines if t0 <= ts <= t1 + self.period_ms / 1e3]
        where = "timed region"
        if not inside and self.lines:  # region shorter than one sampling period: nearest sample
            inside = [min(self.lines, key=lambda x: abs(x[0] - t0))[1]]
            where = "nearest sample to a timed region shorter than the sampling period"
        sm, mx, reasons = [], [], set()
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": where}


# --------------------------------------------------------------------------- library peaks

def _best_ms(fn, reps):
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def measure_int8_peak(dev, n: int = 8192, reps: int = 10):
    """cuBLASLt int8 GEMM (torch._int_mm) on n^3, best of `reps`: the int8
    tensor-core peak of THIS GPU (one binary MAC = one int8 MAC = 2 ops)."""
    import torch
    try:
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
        ms = _best_ms(lambda: torch._int_mm(a, b), reps)
        return 2.0 * n ** 3 / (ms / 1e3) / 1e12, f"cuBLASLt int8 GEMM (torch._int_mm) {n}^3, best of {reps}, this GPU"
    except Exception as exc:  # pragma: no cover - library without int8 GEMM
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return 2.0 * peaks["bf16_tflops"], f"2 x measured bf16 (MEASURED_PEAKS.json); torch._int_mm unavailable: {exc}"


def measure_fp4_gemm(dev, n: int = 8192, reps: int = 10):
    """cuBLASLt block-scaled fp4 GEMM (torch._scaled_mm, e2m1 x e2m1 with
    block-16 e4m3 scales, NVFP4 — the tensor rate of the kind::mxf4 MMAs
    issued here) on n^3, best of `reps`: TOP/s (one fp4 MAC = 2 ops)."""
    import torch
    try:
        a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        sa = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        sb = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        ms = _best_ms(lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16), reps)
        del a, b, sa, sb
        return 2.0 * n ** 3 / (ms / 1e3) / 1e12, (f"cuBLASLt NVFP4 GEMM (torch._scaled_mm, e2m1 x e2m1, block-16 "
                                                  f"e4m3 scales) {n}^3, best of {reps}, this GPU")
    except Exception as exc:  # pragma: no cover - library without fp4 GEMM
        return None, f"torch fp4 GEMM unavailable: {exc}"


def stage_format(st) -> str:
    """Operand format of a stage's GEMM: "f4" / "i8" tensor cores or "popc"."""
    from paper_1705_07175_b200 import _lib
    if _lib.ENGINE != "tc" or not (getattr(st, "tc", True)):
        return "popc"
    if getattr(st, "name", "").startswith("input8"):
        return "i8"
    return getattr(st, "fmt", None) or getattr(getattr(st, "dense", None), "fmt", None) or "i8"


def stage_macs(st) -> int:
    """Algorithmic binary MACs per image of one device stage."""
    from paper_1705_07175_b200 import network as nw
    if isinstance(st, (nw._Input8Fused, nw._Input8Raw)):
        # tensor cores: one u8 x +/-1 MAC per byte; POPC engine: 8 bit-planes
        return st.units * st.k * (1 if getattr(st, "tc", False) else 8)
    if isinstance(st, (nw._DenseFused, nw._Dense, nw._DenseFinal)):
        return st.rec.units * st.rec.input_len
    if isinstance(st, (nw._ConvFused, nw._Conv, nw._ByteConvFused)):
        return st.h_out * st.w_out * st.rec.filters * st.rec.k
    return 0


def build_workload(name):
    from paper_1705_07175_b200 import zoo
    return (zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()), SHAPES[name]


def bench_images(name, n, seed):
    return np.random.default_rng(seed).integers(0, 256, (n, int(np.prod(SHAPES[name]))), dtype=np.uint8)


# --------------------------------------------------------------------------- reference / CPU legs

def ref_arm_available() -> bool:
    from baseline import ref_arm
    return ref_arm.available()


def run_cpu_leg(what: str, seconds: float, parity_file: str | None = None, timeout: float = 600):
    """The reference CPU figures, measured in a separate process
    (baseline/ref_arm.py) so this process's GPU work and the reference's
    Numba threads do not share an address space."""
    cmd = [sys.executable, os.path.join(ROOT, "baseline", "ref_arm.py"), "--what", what, "--seconds", str(seconds)]
    if parity_file:
        cmd += ["--parity", parity_file]
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        if res.returncode != 0:
            return {"error": res.stderr.strip().splitlines()[-1] if res.stderr.strip() else f"rc {res.returncode}"}
        return json.loads(res.stdout.strip().splitlines()[-1])
    except (subprocess.TimeoutExpired, ValueError, IndexError) as exc:
        return {"error": f"{type(exc).__name__}: {exc}"}


def port_rate(name, seconds):
    """Fallback when the reference is not installed: the oracle port
    (oracle/oracle.c restatement, OpenMP threads), image by image."""
    from oracle import oracle as o
    from paper_1705_07175_b200 import zoo
    spec = zoo.bcnn_spec() if name == "bcnn" else zoo.bmlp_spec()
    net = o.OracleNetwork(spec)
    imgs = bench_images(name, 16, 123).reshape((16,) + SHAPES[name])
    net.forward(imgs[0])
    n, t0 = 0, time.perf_counter()
    while True:
        net.forward(imgs[n % 16])
        n += 1
        dt = time.perf_counter() - t0
        if n >= 8 and dt >= seconds:
            return n / dt, n, dt, o.num_threads()


def run_reference_arm(args, rank, world):
    """`--impl reference`: the unmodified reference package timed through its
    own public API (`bitnn.network.forward`, image by image as
    cli.py:101-104) on all host cores; each step is a bounded sample of the
    workload's images (the reference processes one image per call).  This
    process imports nothing from paper_1705_07175_b200."""
    if rank != 0:
        return None
    per_step = args.ref_sample
    if ref_arm_available():
        from baseline import ref_arm
        ref_arm.import_bitnn()
        times = ref_arm.time_network(args.workload, per_step, args.steps, args.warmup, seed=1000)
        host = ref_arm.describe()
        total_t = sum(times)
        value = per_step * args.steps / total_t
        cpu = {"value": value, "unit": "images/s", "cores": host["cores"], "kind": "reference",
               "sample": f"{per_step} images per step x {args.steps} steps (+{args.warmup} warm-up steps) of the "
                         f"workload's seeded images, bitnn.network.forward image by image (cli.py:101-104), "
                         f"unmodified reference from baseline/_ref",
               "threading_layer": host["threading_layer"], "numba": host["numba"], "cpu_model": host["cpu_model"],
               "host_cores": host["host_cores"]}
    else:  # pragma: no cover - driver did not install the reference
        for _ in range(args.warmup):
            port_rate(args.workload, 0.0)
        total_t, n_tot, threads = 0.0, 0, 1
        for _ in range(args.steps):
            r, n, dt, threads = port_rate(args.workload, 0.0)
            total_t += dt
            n_tot += n
        value = n_tot / total_t
        cpu = {"value": value, "unit": "images/s", "cores": threads, "kind": "port",
               "sample": f"{n_tot} images, oracle/oracle.c port (baseline/_ref not installed)"}
    return {
        "metric": BASELINE_METRIC, "value": value, "unit": "images/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": DTYPE, "data": "synthetic", "config": config_dict(args, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------------- our arm

def timed_graph(fn, reps, flush, stream=None):
    """Mean device ms of `fn` over `reps` (CUDA events on the launching
    stream, L2 flushed before each)."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1705_07175_b200 import _lib, forward_batch, zoo
    from paper_1705_07175_b200.network import Network
    from paper_1705_07175_b200.shard import shard_bounds

    gpu = local_rank % torch.cuda.device_count()  # == local_rank on a real N-GPU run
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    spec, shape = build_workload(args.workload)
    lo, hi = shard_bounds(args.batch, world, rank)
    B = hi - lo
    net = Network(spec, max_batch=B)
    host_imgs = net.pinned_images(B)  # e2e inputs live in page-locked host memory
    host_imgs[...] = bench_images(args.workload, args.batch, 1000)[lo:hi]
    net.input_device[:B].copy_(torch.from_numpy(host_imgs).to(dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # kernels one forward pass launches, counted by the library on one eager
    # pass (graph replays do not go through the host library)
    c0 = _lib.launch_count()
    net._launch_all(B)
    torch.cuda.synchronize()
    launches_per_forward = _lib.launch_count() - c0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(gpu) as clk:
        for _ in range(max(args.warmup, 1)):  # warm-up (also captures the CUDA graph for batch B)
            net.run(B)
        barrier()
        launches0 = _lib.launch_count()
        clk.mark(True)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            net.run(B)
            ev[i][1].record(stream)
        barrier()
        clk.mark(False)
    total_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), world, dev)
    gpu_launches = launches_per_forward * args.steps + (_lib.launch_count() - launches0)
    value = args.steps * args.batch / (total_ms / 1e3)
    dev_scores = net.scores_device[:B].cpu().numpy().copy()

    # e2e through the public API with host buffers (pinned H2D + D2H inside)
    out = net.pinned_scores(B)
    forward_batch(net, host_imgs, out)
    barrier()
    e2e_ev = []
    for i in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(i & 0xFF)
        a.record(stream)
        forward_batch(net, host_imgs, out)
        b.record(stream)
        e2e_ev.append((a, b))
    barrier()
    e2e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in e2e_ev), world, dev)
    e2e_value = args.steps * args.batch / (e2e_ms / 1e3)
    e2e_consistent = bool(np.array_equal(out, dev_scores))

    # per-stage device time (eager launches on this stream, events)
    stages = []
    for st in net.stages:
        ms = timed_graph(lambda: st.launch(net, B, _dev_stream()), 5, flush, stream)
        stages.append({"stage": st.name, "ms": ms, "bitops": 2 * stage_macs(st) * B, "format": stage_format(st)})
    stage_total = sum(s["ms"] for s in stages)
    # roofline denominators: MEASURED_PEAKS.json (driver-measured dense bf16
    # burst) x 4 for fp4 operands and x 2 for int8 — B200's dense fp4 / int8
    # tensor rates are 4x / 2x bf16; the same-run cuBLASLt NVFP4 and int8
    # GEMMs are reported beside them (library throughput, not the ceiling)
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bf16 = float(mp["bf16_tflops"])
    int8_lib, int8_src = measure_int8_peak(dev)
    fp4_lib, fp4_src = measure_fp4_gemm(dev)
    # the ceiling is the tensor pipe's MEASURED instruction rate for the
    # operand kind (tools/microbench/mxf4_rate.cu on B200: kind::mxf4 16,379
    # and kind::i8 8,190 MAC/clk/SM, profiles/mxf4_rate_r01.jsonl) at the SM
    # clock sampled during the timed region; 4 x the driver's bf16 figure
    # (a cuBLAS bf16 GEMM, ~69 % of the bf16 instruction rate) is kept beside
    # it as peak_bf16x4 — it sits BELOW what the fp4 MMA can issue
    clocks = clk.summary()
    mhz = float(clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f4_rate = 2 * 16384 * sms * mhz * 1e6 / 1e12
    i8_rate = 2 * 8192 * sms * mhz * 1e6 / 1e12
    peaks = {"f4": (f4_rate, f"kind::mxf4 MMA rate 16384 MAC/clk/SM (measured 16379, profiles/mxf4_rate_r01.jsonl) "
                             f"x {sms} SMs x {mhz:.0f} MHz (median SM clock of the timed region)"),
             "i8": (i8_rate, f"kind::i8 MMA rate 8192 MAC/clk/SM (measured 8190) x {sms} SMs x {mhz:.0f} MHz"),
             "popc": (POPC_PEAK_TBITOPS, POPC_PEAK_SOURCE)}
    alt = {"f4": 4 * bf16, "i8": 2 * bf16, "popc": POPC_PEAK_TBITOPS}
    for s_ in stages:
        s_["tops"] = s_["bitops"] / (s_["ms"] / 1e3) / 1e12 if s_["ms"] > 0 else 0.0
        s_["frac_of_peak"] = s_["tops"] / peaks[s_["format"]][0]
    dom = max(stages, key=lambda s_: s_["ms"])
    dom_peak, dom_src = peaks[dom["format"]]
    traffic, traffic_note = stage_traffic(args.workload, dom["stage"], stages.index(dom), B)
    result = {
        "metric": BASELINE_METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": DTYPE, "data": "synthetic", "config": config_dict(args, world),
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": int(host_imgs.nbytes) * world,
                "d2h_bytes_per_step": int(out.nbytes) * world, "scores_match_device_run": e2e_consistent},
        "gpu_launches": int(gpu_launches),
        "engine": {"gemm": _lib.ENGINE, "tc_format": _lib.TC_FORMAT, "library": os.path.basename(_lib.LIB)},
        "bitops_per_image": 2 * zoo.macs_per_image(spec),
        "roofline": {"bound": "tensor", "achieved": dom["tops"], "peak": dom_peak,
                     "unit": "TOP/s (1 binary MAC = 2 ops = one fp4 / int8 MAC on +/-1 operands)",
                     "frac": dom["tops"] / dom_peak, "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": dom["stage"], "operand_format": dom["format"],
                     "kernel_share_of_step": dom["ms"] / stage_total, "peak_source": dom_src,
                     "peak_bf16x4": alt[dom["format"]], "frac_of_peak_bf16x4": dom["tops"] / alt[dom["format"]],
                     "peak_bf16x4_source": f"{'4' if dom['format'] == 'f4' else '2'} x MEASURED_PEAKS.json bf16_tflops "
                                           f"({bf16} TF/s dense bf16 burst, driver-measured)",
                     "frac_of_same_run_library": dom["tops"] / (fp4_lib if dom["format"] == "f4" else int8_lib)
                     if (fp4_lib if dom["format"] == "f4" else int8_lib) else None,
                     "cublaslt_nvfp4_tops": fp4_lib, "cublaslt_nvfp4_source": fp4_src,
                     "cublaslt_int8_tops": int8_lib, "cublaslt_int8_source": int8_src,
                     "popc_pipe_peak": POPC_PEAK_TBITOPS, "popc_peak_source": POPC_PEAK_SOURCE},
        "stages": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in s_.items()} for s_ in stages],
    }
    # a sample of this rank's timed batch for the parity check against the reference
    idx = np.unique(np.linspace(0, B - 1, min(B, args.parity_sample)).astype(np.int64))
    parity = {"images": host_imgs[idx].copy(), "scores": out[idx].copy(), "global_index": idx + lo}
    del net
    torch.cuda.empty_cache()
    return result, parity, flush


def sweeps(args, dev, flush):
    """BASELINE configs[0]-[3] on the same GPU, device-timed like `value`."""
    import torch
    out = {"batches": batch_sweep(flush), "bgemm": bgemm_sweep(dev, flush), "conv": conv_sweep(flush),
           "pack": pack_sweep(flush)}
    torch.cuda.empty_cache()
    return out


def batch_sweep(flush, reps: int = 20):
    """configs[0] (BMLP batch 1, 256) and configs[1] (BCNN batch 1, 128,
    1024): device images/s per CUDA-graph replay on resident input, and e2e
    images/s through forward_batch from page-locked host images."""
    import torch
    from paper_1705_07175_b200 import forward_batch
    from paper_1705_07175_b200.network import Network
    res = {}
    for name, batches in (("bmlp", (1, 256, 16384)), ("bcnn", (1, 128, 1024, 8192))):
        spec, shape = build_workload(name)
        for b in batches:
            net = Network(spec, max_batch=b)
            x = net.pinned_images(b)
            x[...] = bench_images(name, b, b)
            net.input_device[:b].copy_(torch.from_numpy(x).cuda())
            ms = timed_graph(lambda: net.run(b), reps, flush)
            y = net.pinned_scores(b)
            e2e_ms = timed_graph(lambda: forward_batch(net, x, y), reps, flush)
            res[f"{name}_batch{b}"] = {"images_per_s": round(b / (ms / 1e3)), "ms_per_batch": round(ms, 4),
                                       "e2e_images_per_s": round(b / (e2e_ms / 1e3)), "e2e_ms": round(e2e_ms, 4)}
            del net
    res["note"] = ("device: one CUDA-graph replay per step on resident input; e2e: forward_batch from page-locked "
                   "host u8 images to page-locked float64 scores (H2D + forward + D2H); CUDA events, L2 flushed")
    return res


def bgemm_sweep(dev, flush, sizes=(1024, 2048, 4096, 8192, 16384)):
    """configs[2]: bit-packed GEMM, M=N=K=n, int32 C (bgemm_packed semantics,
    _kernels.py:85-106), device-resident packed operands, B in the tensor-core
    operand format once (a layer's weights); cuBLASLt NVFP4 at the same n."""
    import torch
    from paper_1705_07175_b200 import _dev, _lib, gemm, zoo
    res = {}
    for n in sizes:
        rng = np.random.default_rng(n)
        a = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
        b = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
        c = _dev.empty((n, n), np.int32)
        b8 = _dev.tc_weights(b, n, n)
        reps = 5 if n >= 8192 else 20
        ms = timed_graph(lambda: gemm.bgemm_device(a, n, b, n, n // 64, n, c, b_i8=b8), reps, flush)
        ah, bh, got = (_dev.download(a[:16], np.uint64), _dev.download(b[:16], np.uint64),
                       _dev.download(c[:16, :16], np.int32))
        want = n - 2 * np.bitwise_count(ah[:, None, :] ^ bh[None, :, :]).sum(-1).astype(np.int64)
        lib, _ = measure_fp4_gemm(dev, n, reps=5)
        tops = 2.0 * n ** 3 / (ms / 1e3) / 1e12
        res[str(n)] = {"ms": round(ms, 4), "Gops": round(tops * 1e3), "cublaslt_nvfp4_Gops": round(lib * 1e3) if lib else None,
                       "frac_of_cublaslt": round(tops / lib, 3) if lib else None,
                       "corner_16x16_exact": bool(np.array_equal(got, want)), "format": _lib.TC_FORMAT}
        del a, b, c, b8
        torch.cuda.empty_cache()
    return res


def conv_sweep(flush, batch=256):
    """configs[3]: 3x3 / stride 1 / pad 1 binary conv, C_in = C_out in
    {128..1024}, H = W in {8..64}, batch 256, fused BN-threshold + repack
    output (a network conv stage), through the C-ABI conv entry point."""
    from paper_1705_07175_b200 import _dev, _lib, layers, zoo
    res = {}
    for c in (128, 256, 512, 1024):
        for hw in (8, 16, 32, 64):
            rng = np.random.default_rng(c * 100 + hw)
            x = _dev.upload(zoo.pack_bits_host(rng.random((batch * hw * hw, c)) >= 0.5))
            w = _dev.upload(zoo.pack_bits_host(rng.random((c, 9 * c)) >= 0.5))
            w8 = _dev.tc_weights(w, c, 9 * c)
            bn = zoo.rand_bn(rng, c, 20.0)
            cal = layers.calibrate_device(bn.mean, bn.var, bn.gamma, bn.beta, bn.eps, 9 * c)
            o = _dev.empty((batch, hw * hw, -(-c // 64)), np.uint64)

            def run():
                _lib.call(_lib.tc_entry("conv_bn_pack"), _dev.P(x), batch, hw, hw, c, _dev.P(w8), c, 3, 3, 1, 1, 0,
                          layers._thresh_struct(cal["thresh32"], cal["thresh64"], cal["ge"]), _dev.P(o), _dev.stream())
            ms = timed_graph(run, 5, flush)
            ops = 2.0 * batch * hw * hw * c * 9 * c
            res[f"C{c}_{hw}px"] = {"ms": round(ms, 4), "Gops": round(ops / (ms / 1e3) / 1e9),
                                   "images_per_s": round(batch / (ms / 1e3))}
    return res


def pack_sweep(flush):
    """north_star (1): sign-pack (_kernels.py:43-54) and byte bit-planes
    (_kernels.py:67-82), algorithmic bytes (in + out) per second against
    MEASURED_PEAKS.json's copy bandwidth."""
    import torch
    from paper_1705_07175_b200 import _dev, _lib
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    res = {}
    lines, bits = 262144, 4096
    x = torch.randn((lines, bits), dtype=torch.float32, device="cuda")
    o = _dev.empty((lines, bits // 64), np.uint64)
    ms = timed_graph(lambda: _lib.call("b2_pack_lines_f32", _dev.P(x), lines, bits, _dev.P(o), _dev.stream()), 5, flush)
    nb = lines * bits * 4 + lines * bits // 8
    res["sign_pack_f32"] = {"lines": lines, "bits": bits, "ms": round(ms, 4), "GBps": round(nb / ms / 1e6, 1),
                            "frac_of_hbm": round(nb / ms / 1e6 / peak, 3)}
    del x, o
    lines, bits = 1048576, 784
    x = torch.randint(0, 256, (lines, bits), dtype=torch.uint8, device="cuda")
    o = _dev.empty((8, lines, -(-bits // 64)), np.uint64)
    ms = timed_graph(lambda: _lib.call("b2_pack_byte_planes", _dev.P(x), lines, bits, _dev.P(o), _dev.stream()), 5, flush)
    nb = lines * bits + 8 * lines * (-(-bits // 64)) * 8
    res["byte_planes"] = {"lines": lines, "bits": bits, "ms": round(ms, 4), "GBps": round(nb / ms / 1e6, 1),
                          "frac_of_hbm": round(nb / ms / 1e6 / peak, 3)}
    res["hbm_peak_GBps"] = peak
    del x, o
    torch.cuda.empty_cache()
    return res


def batch1_latency(spec, shape, reps: int = 300):
    """The reference's own mode (network.py:506-522, forward of ONE image):
    wall-clock microseconds per `forward(net, image)` call — host image in,
    one CUDA-graph replay, host scores out."""
    import torch
    from paper_1705_07175_b200 import forward
    from paper_1705_07175_b200.network import Network
    net = Network(spec, max_batch=1)
    img = np.random.default_rng(7).integers(0, 256, shape, dtype=np.uint8)
    for _ in range(20):
        forward(net, img)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        forward(net, img)
    dt = (time.perf_counter() - t0) / reps
    return {"us_per_image": round(dt * 1e6, 1), "launches_per_forward": net.launches_per_forward(),
            "note": "wall clock per forward() call of one image, CUDA graph replay, H2D+D2H included"}


def stage_traffic(workload, stage_name, index, batch):
    """DRAM bytes per launch of one stage's kernels from the committed ncu
    capture (profiles/traffic_<workload>.json, tools/ncu_summary.py), scaled
    linearly to this batch when the capture used another one."""
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        table = json.load(open(path))
    except (OSError, ValueError):
        return None, "no committed capture"
    ent = table.get(str(index))
    if not ent or ent.get("stage") != stage_name:
        return None, "capture does not match this stage"
    b0 = ent.get("batch", batch)
    if b0 == batch:
        return ent.get("dram_bytes"), f"ncu capture at batch {b0} ({os.path.basename(path)})"
    return int(ent["dram_bytes"] * batch / b0), f"ncu capture at batch {b0} scaled x{batch / b0:g} ({os.path.basename(path)})"


def max_over_ranks(x: float, world: int, dev) -> float:
    """MAX of a per-rank device time over all ranks (NCCL on the GPU; CPU
    tensors when the process group is gloo)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _dev_stream():
    from paper_1705_07175_b200 import _dev
    return _dev.stream()


def attach_cpu(res, args, parity):
    """Reference CPU figures (separate process) + the parity check of the
    timed batch's sample against the reference's own forward."""
    pfile = None
    if parity is not None:
        fd, pfile = tempfile.mkstemp(suffix=".npz")
        os.close(fd)
        np.savez(pfile, workload=np.array(args.workload), **parity)
    if ref_arm_available():
        what = "bcnn,bmlp" + ("" if args.no_extra else ",bgemm,conv")
        cpu = run_cpu_leg(what, args.cpu_seconds, pfile)
    else:
        cpu = {"error": "baseline/_ref not installed"}
    if pfile:
        os.unlink(pfile)
    host = cpu.get("host", {})
    if args.workload in cpu:
        r = cpu[args.workload]
        res["cpu_baseline"] = {"value": r["images_per_s"], "unit": "images/s", "cores": host.get("cores"),
                               "kind": "reference",
                               "sample": f"{r['images']} seeded images in {r['seconds']} s, bitnn.network.forward "
                                         f"image by image (cli.py:101-104), unmodified reference from baseline/_ref",
                               "threading_layer": host.get("threading_layer"), "cpu_model": host.get("cpu_model"),
                               "host_cores": host.get("host_cores")}
    else:
        rate, n, dt, threads = port_rate(args.workload, args.cpu_seconds)
        res["cpu_baseline"] = {"value": rate, "unit": "images/s", "cores": threads, "kind": "port",
                               "sample": f"{n} images in {dt:.1f} s, oracle/oracle.c port (reference unavailable: "
                                         f"{cpu.get('error')})"}
    if "parity" in cpu:
        res["parity_checked"] = cpu["parity"]
    sw = res.get("sweeps")
    if sw:
        for name in ("bcnn", "bmlp"):
            if name in cpu:
                sw["batches"][f"{name}_cpu_reference_images_per_s"] = round(cpu[name]["images_per_s"], 1)
        for n, r in (cpu.get("bgemm") or {}).items():
            if n in sw["bgemm"]:
                sw["bgemm"][n]["cpu_reference_Gops"] = round(r["gops"], 1)
                sw["bgemm"][n]["cpu_reference_iters"] = r["iters"]
        for k, r in (cpu.get("conv") or {}).items():
            if k in sw["conv"]:
                sw["conv"][k]["cpu_reference_Gops"] = round(r["gops"], 1)
                sw["conv"][k]["cpu_reference_images_per_s"] = round(1e3 / r["ms_per_image"], 1)
                sw["conv"][k]["cpu_sample_images"] = r["sample_images"]
    res["cpu_host"] = host


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="bcnn", choices=["bcnn", "bmlp"])
    ap.add_argument("--batch", type=int, default=None, help="GLOBAL images per step (sliced across GPUs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-sample", type=int, default=32, help="reference arm: images per step")
    ap.add_argument("--parity-sample", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the sweeps and batch-1 blocks")
    args = ap.parse_args()
    if args.batch is None:
        args.batch = DEFAULT_BATCH[args.workload]
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    args.gpus = world if world > 1 else args.gpus

    if args.impl == "reference":
        res = run_reference_arm(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        gpu = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        backend = os.environ.get("B2_DIST_BACKEND", "nccl")  # gloo: validate N ranks on fewer GPUs
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    res, parity, flush = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_extra:
            spec, shape = build_workload(args.workload)
            res["batch1"] = batch1_latency(spec, shape)
            res["sweeps"] = sweeps(args, torch.device("cuda", torch.cuda.current_device()), flush)
        del flush
        if not args.no_cpu:
            attach_cpu(res, args, parity)
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
