#!/usr/bin/env python
"""Benchmark: binary forward pass on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload bcnn|bmlp|bgemm]
                    [--batch B] [--impl ours|reference]

One step = one forward pass of the workload over one batch of synthetic
input per GPU (weak scaling: each rank owns its own batch slice; images
are independent, so there is no collective on the data path — the only
NCCL calls are the barrier and the max-over-ranks reduction of the
timings).  Multi-GPU runs are launched with torchrun, one rank per GPU.

`value`  — device throughput: inputs resident in HBM, K steps timed with
           CUDA events on the launching stream (each step is one CUDA-graph
           replay of the whole network), L2 flushed between steps.
`e2e`    — the same metric through the public API `forward_batch` with host
           uint8 images in page-locked memory (Network.pinned_images): the
           H2D copy of every step's inputs + forward + D2H of the float64
           scores inside the timed region.
`roofline` — per-stage device times (CUDA events, eager launches on the
           same stream); the dominant stage's achieved ops/s (2 per binary
           MAC) against the int8 tensor-core peak measured on this GPU in the
           same run (cuBLASLt int8 GEMM); the measured POPC-pipe peak is
           reported beside it.
`cpu_baseline` — the CPU oracle port of the reference (oracle/, OpenMP
           threads where the reference uses numba prange) on a bounded
           sample, rank 0 only.
`--impl reference` — the reference arm: that same CPU path timed on the
           host for the same metric/config (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
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


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


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


def measure_int8_peak(dev, n: int = 8192, reps: int = 10):
    """Dense int8 tensor-core peak of THIS GPU, measured: cuBLASLt int8 GEMM
    (torch._int_mm, int32 accumulate) on n^3, best of `reps`, CUDA events.
    The binary GEMM counts 2 ops per binary MAC; on the tensor pipe one
    binary MAC is one int8 MAC, so the units match (TOP/s)."""
    import torch
    try:
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best / 1e3) / 1e12, f"cuBLASLt int8 GEMM (torch._int_mm) {n}^3, best of {reps}, this GPU"
    except Exception as exc:  # pragma: no cover - library without int8 GEMM
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return 2.0 * peaks["bf16_tflops"], f"2 x measured bf16 ({peaks['bf16_tflops']} TF/s, MEASURED_PEAKS.json); " \
                                           f"torch._int_mm unavailable: {exc}"


def measure_fp4_peak(dev, n: int = 8192, reps: int = 10):
    """Dense fp4 tensor-core peak of THIS GPU, measured: cuBLASLt block-scaled
    fp4 GEMM (torch._scaled_mm on float4_e2m1fn_x2 with block-16 e4m3 scales,
    NVFP4 — the same tensor rate as the MXFP4 kind::mxf4 MMAs this framework
    issues) on n^3, best of `reps`, CUDA events.  One binary MAC is one fp4
    MAC on +/-1 values (2 ops)."""
    import torch
    try:
        a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        sa = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        sb = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device=dev).view(torch.float8_e4m3fn)
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)  # noqa: E731
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, sa, sb
        return 2.0 * n ** 3 / (best / 1e3) / 1e12, (f"cuBLASLt NVFP4 GEMM (torch._scaled_mm, e2m1 x e2m1, block-16 "
                                                    f"e4m3 scales) {n}^3, best of {reps}, this GPU")
    except Exception as exc:  # pragma: no cover - library without fp4 GEMM
        return 9000.0, f"B200_PROFILING.md dense fp4 9 PFLOP/s (fallback: torch fp4 GEMM unavailable: {exc})"


def stage_format(st) -> str:
    """Operand format of a stage's GEMM: "f4" / "i8" tensor cores or "popc"."""
    from paper_1705_07175_b200 import _lib
    if _lib.ENGINE != "tc" or not (getattr(st, "tc", True)):
        return "popc"
    if getattr(st, "name", "").startswith("input8"):
        return "i8"
    return getattr(st, "fmt", None) or getattr(getattr(st, "dense", None), "fmt", None) or "i8"


# --------------------------------------------------------------------------- workloads

def build_workload(name):
    from paper_1705_07175_b200 import zoo
    if name == "bcnn":
        return zoo.bcnn_spec(), (32, 32, 3)
    if name == "bmlp":
        return zoo.bmlp_spec(), (784,)
    raise ValueError(name)


def cpu_sample(spec, shape, seconds: float, min_images: int, seed: int = 123):
    """Time the CPU oracle (reference restatement) image by image, like the
    reference's cli.py:101-104 loop, for about `seconds`."""
    from oracle import oracle as o
    net = o.OracleNetwork(spec)
    rng = np.random.default_rng(seed)
    imgs = rng.integers(0, 256, (max(min_images, 8),) + shape, dtype=np.uint8)
    net.forward(imgs[0])  # warm caches
    n = 0
    t0 = time.perf_counter()
    while True:
        net.forward(imgs[n % imgs.shape[0]])
        n += 1
        dt = time.perf_counter() - t0
        if n >= min_images and dt >= seconds:
            break
    return n / dt, n, dt, o.num_threads()


def run_reference_arm(args, rank):
    if rank != 0:
        return None
    spec, shape = build_workload(args.workload)
    per_step = args.ref_sample
    for _ in range(args.warmup):
        cpu_sample(spec, shape, 0.0, per_step)
    rates, total_n, total_t = [], 0, 0.0
    threads = 0
    for _ in range(args.steps):
        r, n, dt, threads = cpu_sample(spec, shape, 0.0, per_step)
        rates.append(r)
        total_n += n
        total_t += dt
    value = total_n / total_t
    return {
        "metric": BASELINE_METRIC, "value": value, "unit": "images/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64-packed bits / int32 acc / f64 scores", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step} images per step, {args.steps} steps, per-image forward "
                                   f"(oracle/oracle.c restatement of the reference packed kernels, OpenMP "
                                   f"where the reference uses numba prange)"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def config_dict(args):
    if args.workload == "bcnn":
        wl = "BCNN VGG-style CIFAR-10 2x128C3-MP2-2x256C3-MP2-2x512C3-MP2-1024FC-1024FC-10, 32x32x3 u8"
    else:
        wl = "BinaryNet MLP 784-4096-4096-4096-10 on MNIST-shaped u8"
    return {"workload": wl, "images_per_gpu_per_step": args.batch, "global_batch": args.batch * args.gpus,
            "parallelism": f"dp{args.gpus} (batch slices, no collective)", "l2": "flushed between timed steps",
            "weights": "seeded random +/-1 (paper_1705_07175_b200/zoo.py)"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1705_07175_b200 import _lib, forward_batch, zoo
    from paper_1705_07175_b200.network import Network

    gpu = local_rank % torch.cuda.device_count()  # == local_rank on a real N-GPU run
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    spec, shape = build_workload(args.workload)
    B = args.batch
    net = Network(spec, max_batch=B)
    rng = np.random.default_rng(1000 + rank)
    host_imgs = net.pinned_images(B)  # e2e inputs live in page-locked host memory
    host_imgs[...] = rng.integers(0, 256, (B, int(np.prod(shape))), dtype=np.uint8)
    net.input_device.copy_(torch.from_numpy(host_imgs).to(dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # kernels one forward pass launches, counted by the library on one eager
    # pass (the graph replays below do not go through the host library)
    c0 = _lib.launch_count()
    net._launch_all(B)
    torch.cuda.synchronize()
    launches_per_forward = _lib.launch_count() - c0
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(gpu) as clk:
        # warm-up (also captures the CUDA graph for batch B)
        for _ in range(max(args.warmup, 1)):
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
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    total_ms = max_over_ranks(total_ms, world, dev)
    launches_direct = _lib.launch_count() - launches0
    gpu_launches = launches_per_forward * args.steps + launches_direct
    value = args.steps * B * world / (total_ms / 1e3)

    # e2e through the public API with host buffers (pinned H2D + D2H inside)
    out = net.pinned_scores(B)  # page-locked score buffer: D2H lands in it directly
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
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    e2e_ms = max_over_ranks(e2e_ms, world, dev)
    e2e_value = args.steps * B * world / (e2e_ms / 1e3)

    # per-stage device time (eager launches on this stream, events)
    stages = []
    for st in net.stages:
        reps = 5
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.launch(net, B, _dev_stream())
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            st.launch(net, B, _dev_stream())
        b.record(stream)
        torch.cuda.synchronize()
        stages.append({"stage": st.name, "ms": a.elapsed_time(b) / reps, "bitops": 2 * stage_macs(st) * B,
                       "format": stage_format(st)})
    stage_total = sum(s["ms"] for s in stages)
    batch1 = batch1_latency(spec, shape) if rank == 0 else None
    others = other_metrics(args, dev, flush) if rank == 0 and not args.no_extra else None
    sweep = batch_sweep(flush) if rank == 0 and not args.no_extra else None
    int8_peak, int8_src = measure_int8_peak(dev)
    fp4_peak, fp4_src = measure_fp4_peak(dev)
    peaks = {"f4": (fp4_peak, fp4_src), "i8": (int8_peak, int8_src), "popc": (POPC_PEAK_TBITOPS, POPC_PEAK_SOURCE)}
    for s_ in stages:
        s_["tops"] = s_["bitops"] / (s_["ms"] / 1e3) / 1e12 if s_["ms"] > 0 else 0.0
        s_["frac_of_peak"] = s_["tops"] / peaks[s_["format"]][0]
    dom = max(stages, key=lambda s_: s_["ms"])
    achieved = dom["tops"]
    dom_peak, dom_src = peaks[dom["format"]]
    traffic = stage_traffic(args.workload, dom["stage"], stages.index(dom))
    result = {
        "metric": BASELINE_METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u1 packed (+/-1) activations; tensor-core operands e2m1 (fp4, unit block scales) "
                 "or s8 (u8-input layer), exact fp32 / s32 accumulators; f64 scores",
        "data": "synthetic",
        "config": config_dict(args) | {"global_batch": B * world, "engine": _lib.ENGINE},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": int(host_imgs.nbytes),
                "d2h_bytes_per_step": int(out.nbytes)},
        "gpu_launches": int(gpu_launches),
        "bitops_per_image": 2 * zoo.macs_per_image(spec),
        "achieved_tbitops_network": 2 * zoo.macs_per_image(spec) * value / world / 1e12,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": dom_peak,
                     "unit": "TOP/s (1 binary MAC = 2 ops = one fp4 / int8 MAC on +/-1 operands)",
                     "frac": achieved / dom_peak, "traffic": traffic, "kernel": dom["stage"],
                     "operand_format": dom["format"], "kernel_share_of_step": dom["ms"] / stage_total,
                     "peak_source": dom_src, "fp4_peak": fp4_peak, "int8_peak": int8_peak, "int8_peak_source": int8_src,
                     "popc_pipe_peak": POPC_PEAK_TBITOPS, "popc_peak_source": POPC_PEAK_SOURCE},
        "stages": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in s_.items()} for s_ in stages],
        "batch1": batch1,
        "other_metrics": others,
        "batch_sweep": sweep,
    }
    return result


def other_metrics(args, dev, flush, steps: int = 10):
    """The rest of BASELINE's metric on the same GPU, device-timed like
    `value`: the other network (BMLP for a BCNN run and vice versa) and the
    bit-packed GEMM at M=N=K=8192 (configs[2])."""
    import torch
    from paper_1705_07175_b200 import _dev, _lib, gemm, zoo
    from paper_1705_07175_b200.network import Network
    out = {}
    other = "bmlp" if args.workload == "bcnn" else "bcnn"
    spec, shape = build_workload(other)
    b = 16384 if other == "bmlp" else 8192
    net = Network(spec, max_batch=b)
    net.input_device.copy_(torch.from_numpy(
        np.random.default_rng(5).integers(0, 256, (b, int(np.prod(shape))), dtype=np.uint8)).to(dev))
    for _ in range(3):
        net.run(b)
    ms = 0.0
    for _ in range(steps):
        flush.fill_(7)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        net.run(b)
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    out[f"{other}_images_per_s"] = b * steps / (ms / 1e3)
    out[f"{other}_batch"] = b
    del net
    n = 8192
    rng = np.random.default_rng(6)
    a = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
    w = _dev.upload(zoo.pack_bits_host(rng.random((n, n)) >= 0.5))
    w8 = _dev.tc_weights(w, n, n)  # tensor-core weights in the default operand format
    c = _dev.empty((n, n), np.int32)
    for _ in range(3):
        gemm.bgemm_device(a, n, w, n, n // 64, n, c, b_i8=w8)
    ms = 0.0
    for _ in range(5):
        flush.fill_(9)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gemm.bgemm_device(a, n, w, n, n // 64, n, c, b_i8=w8)
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    out["bgemm_8192_Gops"] = 2.0 * n ** 3 * 5 / (ms / 1e3) / 1e9
    out["bgemm_operand_format"] = _lib.TC_FORMAT
    out["note"] = "device time, CUDA events, L2 flushed between steps; ops = 2 per binary MAC"
    return out


def batch_sweep(flush, reps: int = 20):
    """BASELINE configs[0] / configs[1] batch sizes (BMLP 1 and 256, BCNN 1,
    128 and 1024): device throughput of one CUDA-graph replay of the whole
    network per step on resident input, CUDA events, L2 flushed between
    steps.  Batch 1 here is device time; `batch1` below is the wall-clock
    latency of the public `forward` call."""
    import torch
    from paper_1705_07175_b200.network import Network
    out = {}
    for name, batches in (("bmlp", (1, 256)), ("bcnn", (1, 128, 1024))):
        spec, shape = build_workload(name)
        for b in batches:
            net = Network(spec, max_batch=b)
            x = np.random.default_rng(b).integers(0, 256, (b, int(np.prod(shape))), dtype=np.uint8)
            net.input_device[:b].copy_(torch.from_numpy(x).cuda())
            for _ in range(3):
                net.run(b)
            torch.cuda.synchronize()
            ms = 0.0
            for _ in range(reps):
                flush.fill_(3)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                net.run(b)
                e1.record()
                torch.cuda.synchronize()
                ms += e0.elapsed_time(e1)
            out[f"{name}_batch{b}"] = {"images_per_s": round(b * reps / (ms / 1e3)), "ms_per_batch": round(ms / reps, 4)}
    out["note"] = "device time per graph replay, CUDA events, L2 flushed between steps"
    return out


def batch1_latency(spec, shape, reps: int = 300):
    """The reference's own mode (network.py:506-522, forward of ONE image):
    wall-clock microseconds per `forward(net, image)` call — host image in,
    H2D, one CUDA-graph replay, D2H of the scores, host scores out."""
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


def stage_traffic(workload, stage_name, index):
    """DRAM bytes per launch of one stage's kernel from the committed ncu
    capture (profiles/traffic_<workload>.json, written by
    tools/ncu_summary.py from `ncu --set full`), or None."""
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        table = json.load(open(path))
    except (OSError, ValueError):
        return None
    ent = table.get(str(index))
    if ent and ent.get("stage") == stage_name:
        return ent.get("dram_bytes")
    return None


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="bcnn", choices=["bcnn", "bmlp"])
    ap.add_argument("--batch", type=int, default=None, help="images per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other_metrics block")
    args = ap.parse_args()
    if args.batch is None:
        args.batch = 8192 if args.workload == "bcnn" else 16384
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    args.gpus = world if world > 1 else args.gpus

    if args.impl == "reference":
        res = run_reference_arm(args, rank)
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
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu:
            spec, shape = build_workload(args.workload)
            rate, n, dt, threads = cpu_sample(spec, shape, args.cpu_seconds, 8)
            res["cpu_baseline"] = {"value": rate, "unit": "images/s", "cores": threads, "kind": "port",
                                   "sample": f"{n} images in {dt:.1f} s, per-image forward of the oracle port "
                                             f"(oracle/oracle.c, OpenMP where the reference uses prange)"}
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
