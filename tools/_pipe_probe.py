"""GPU time of the whole-call pipeline graph vs wall time of forward_batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_07175_b200 import zoo, forward_batch
from paper_1705_07175_b200.network import Network
for name, spec, B in (("bmlp", zoo.bmlp_spec(), 16384), ("bcnn", zoo.bcnn_spec(), 8192)):
    net = Network(spec, max_batch=B)
    imgs = net.pinned_images(B); imgs[:] = 3
    for label, out in (("pinned out", net.pinned_scores(B)), ("plain out", np.empty((B, net.classes)))):
        for _ in range(3): forward_batch(net, imgs, out)
        key = [k for k in net._graphs if isinstance(k, tuple)][-1]
        g = net._graphs[key]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): g.replay()
        e1.record(); torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter(); forward_batch(net, imgs, out); ts.append(time.perf_counter() - t0)
        print(name, label, f"graph GPU {e0.elapsed_time(e1) / 10:.3f} ms   forward_batch wall {np.median(ts) * 1e3:.3f} ms", net._chunk_plan(B, True))
