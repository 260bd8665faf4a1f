"""GPU time of the whole-call pipeline graph for several chunk plans."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_07175_b200 import zoo, forward_batch
from paper_1705_07175_b200.network import Network
PLANS = {"bmlp": [[2048, 4096, 10240], [1024, 2048, 4096, 9216], [4096, 12288], [2048, 14336], [1024, 15360],
                  [4096, 4096, 8192], [8192, 8192], [16384]],
         "bcnn": [[1536, 6656], [1024, 7168], [768, 7424], [512, 2048, 5632], [512, 1536, 6144], [256, 1280, 6656],
                  [1024, 3072, 4096]]}
for name, spec, B in (("bcnn", zoo.bcnn_spec(), 8192),):
    net = Network(spec, max_batch=B)
    imgs = net.pinned_images(B); imgs[:] = 3
    out = net.pinned_scores(B)
    for plan in PLANS[name]:
        chunks, b0 = [], 0
        for b in plan:
            chunks.append((b0, b)); b0 += b
        net._chunk_plan = lambda n, pinned, c=chunks: c
        net._graphs = {k: v for k, v in net._graphs.items() if not isinstance(k, tuple)}
        if len(chunks) == 1:
            from paper_1705_07175_b200 import network as nw
            g = None
        forward_batch(net, imgs, out)
        keys = [k for k in net._graphs if isinstance(k, tuple)]
        if not keys:
            print(name, plan, "single chunk: stream path"); continue
        g = net._graphs[keys[-1]]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): g.replay()
        e1.record(); torch.cuda.synchronize()
        print(name, plan, f"graph GPU {e0.elapsed_time(e1) / 10:.3f} ms  -> {B / (e0.elapsed_time(e1) / 10) / 1e3:.2f} M img/s")
