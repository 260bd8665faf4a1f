"""Launch one stage of a baseline network eagerly (for ncu captures).

    python tools/profile_stage.py --workload bcnn --stage 0 --batch 8192 --reps 3

The network is built and warmed once; then stage `--stage` is launched
`--reps` times on the current stream.  Use with
`ncu -k regex:k_tc_gemm -s <skip> -c 1 ...`."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_07175_b200 import _dev, zoo  # noqa: E402
from paper_1705_07175_b200.network import Network  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bcnn", choices=["bcnn", "bmlp"])
    ap.add_argument("--stage", type=int, default=0, help="stage index, -1 = all")
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--graph", action="store_true", help="time the reps as one captured CUDA graph (no host "
                                                         "launch overhead; what a graph-replayed forward sees)")
    ap.add_argument("--map", default=None, help="write {stage: [first, last) library launch index} JSON here "
                                                 "(one untimed launch per stage, for tools/ncu_summary.py traffic)")
    a = ap.parse_args()
    spec = zoo.bcnn_spec() if a.workload == "bcnn" else zoo.bmlp_spec()
    net = Network(spec, max_batch=a.batch, use_graphs=False)
    rng = np.random.default_rng(0)
    n = net.input_len
    net.input_device.copy_(torch.from_numpy(rng.integers(0, 256, (a.batch, n), dtype=np.uint8)).cuda())
    net.run(a.batch)
    torch.cuda.synchronize()
    if a.map:
        import json
        from paper_1705_07175_b200 import _lib
        spans = {}
        for i, st in enumerate(net.stages):
            c0 = _lib.launch_count()
            st.launch(net, a.batch, _dev.stream())
            spans[str(i)] = {"stage": st.name, "first": c0, "last": _lib.launch_count()}
        torch.cuda.synchronize()
        json.dump({"workload": a.workload, "batch": a.batch, "spans": spans}, open(a.map, "w"), indent=1)
        return
    stages = range(len(net.stages)) if a.stage < 0 else [a.stage]
    for i in stages:
        st = net.stages[i]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.launch(net, a.batch, _dev.stream())
        if a.graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.Stream()):
                for _ in range(a.reps):
                    st.launch(net, a.batch, _dev.stream())
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
        else:
            e0.record()
            for _ in range(a.reps):
                st.launch(net, a.batch, _dev.stream())
            e1.record()
        torch.cuda.synchronize()
        print(f"stage {i} {st.name}: {e0.elapsed_time(e1) / a.reps:.4f} ms  launches/stage {st.launches()}")


if __name__ == "__main__":
    main()
