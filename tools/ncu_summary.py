"""Summarise ncu reports / launch lists into profiles/ (run in the build container).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/xxx_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/xxx_full.md
    python tools/ncu_summary.py traffic gpurun_out/traffic.csv gpurun_out/stage_map.json > profiles/traffic_bcnn.json
    python tools/ncu_summary.py stalls gpurun_out/prof.ncu-rep [top] >> profiles/xxx_full.md

`traffic` joins an ncu metrics list (dram__bytes_read/write.sum,
gpu__time_duration.sum over `tools/profile_stage.py --map`) with the stage
map that script wrote: our kernels are counted in launch order (namespace
b2::, every launch of the library increments b2_launch_count), so the
library launch index of each ncu row is its position among b2:: kernels.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

# Tensor-core activity of tcgen05 kernels: sm__pipe_tensor_cycles_active (=
# the hmma subpipe) counts cycles the 5th-gen tensor pipe is busy; for a
# kind::mxf4 kernel it equals (MACs / 16384 per SM-cycle) / elapsed cycles, so
# it reconciles with the bench's achieved TOP/s at the ncu clock.  The
# TriageCompute "*_realtime" metrics round 1 quoted (xu 73 % / 171 %, tensor
# 14 %) are sampled on another clock domain and are not utilisations: they
# are left out.
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        name = r.get("Kernel Name", "?")
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        if name not in agg:
            order.append(name)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for n in sorted(order, key=lambda n: -agg[n][1]):
        c, us = agg[n]
        print(f"| `{n[:110]}` | {c} | {us:.1f} | {100 * us / tot:.1f}% |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"### `{vals[hdr.index('Kernel Name')][:160]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h.endswith(k):
                    print(f"| {h} | {vals[i]} | {units[i]} |")
                    break
        print()


def stalls(path, top="25"):
    """Per-SASS-line warp-state samples (ncu --page source): the top lines,
    then every mbarrier wait (SYNCS.PHASECHK) and tcgen05 MMA / commit line
    with its execution count — a wait line executed far more often than its
    loop body is a role spinning on that barrier."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    samp = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)  # noqa: E731
    tot = sum(samp(r) for r in data)
    print(f"{rows[0][1][:150]}\n\ntotal warp samples {tot}\n")
    print("| samples | share | executed | SASS |\n|---|---|---|---|")
    for r in sorted(data, key=lambda r: -samp(r))[:int(top)]:
        print(f"| {samp(r)} | {100 * samp(r) / max(tot, 1):.1f}% | {r[ix['Instructions Executed']]} | "
              f"`{r[ix['Source']].strip()[:90]}` |")
    print("\n| samples | executed | barrier / tensor-core line |\n|---|---|---|")
    for r in data:
        src = r[ix["Source"]].strip()
        if any(k in src for k in ("PHASECHK", "UTCQMMA", "UTCOMMA", "UTCHMMA", "UTCIMMA", "UTCBAR")):
            print(f"| {samp(r)} | {r[ix['Instructions Executed']]} | `{src[:90]}` |")


def traffic(csv_path, map_path):
    import json
    lines = open(csv_path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    per = defaultdict(dict)  # ncu launch ID -> metrics
    names = {}
    for r in rows:
        lid = int(r["ID"])
        names[lid] = r.get("Kernel Name", "")
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
        unit = r.get("Metric Unit", "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
                "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        per[lid][r["Metric Name"]] = v * mult
    # ncu drops the outer b2:: namespace; everything that is not a torch /
    # library kernel is ours
    foreign = ("at::", "cutlass", "nccl", "cublas", "void at::")
    ours = [lid for lid in sorted(per) if not any(f in names[lid] for f in foreign)]
    smap = json.load(open(map_path))
    base = smap["spans"]["0"]["first"]
    # the map's launches are the LAST len(map) b2:: launches of the capture
    total = max(sp["last"] for sp in smap["spans"].values()) - base
    ours = ours[-total:]
    out = {}
    for k, sp in smap["spans"].items():
        ids = ours[sp["first"] - base:sp["last"] - base]
        out[k] = {"stage": sp["stage"], "batch": smap["batch"], "kernels": [names[i][:80] for i in ids],
                  "dram_bytes": int(sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
                                        for i in ids)),
                  "ncu_ns": int(sum(per[i].get("gpu__time_duration.sum", 0) for i in ids))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic, "stalls": stalls}[sys.argv[1]](*sys.argv[2:])
