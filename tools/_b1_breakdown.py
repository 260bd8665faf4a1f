"""Batch-1 latency breakdown: device time of the io1 graph (events), host
replay+sync wall time, full forward() wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_07175_b200 import forward, zoo
from paper_1705_07175_b200.network import Network
for name, spec, shape in (("bcnn", zoo.bcnn_spec(), (32, 32, 3)), ("bmlp", zoo.bmlp_spec(), (784,))):
    net = Network(spec, max_batch=1)
    img = np.random.default_rng(7).integers(0, 256, shape, dtype=np.uint8)
    for _ in range(20): forward(net, img)
    g = net._graphs["io1"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(); [g.replay() for _ in range(200)]; e1.record(); torch.cuda.synchronize()
    dev_back2back = e0.elapsed_time(e1) / 200 * 1e3
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); g.replay(); torch.cuda.current_stream().synchronize(); ts.append(time.perf_counter() - t0)
    t_rs = np.median(ts) * 1e6
    ts = []
    for _ in range(200):
        t0 = time.perf_counter(); forward(net, img); ts.append(time.perf_counter() - t0)
    t_fw = np.median(ts) * 1e6
    gc = net._graphs[1]  # compute-only graph (no H2D / D2H)
    torch.cuda.synchronize()
    e0.record(); [gc.replay() for _ in range(200)]; e1.record(); torch.cuda.synchronize()
    dev_c = e0.elapsed_time(e1) / 200 * 1e3
    from paper_1705_07175_b200 import _lib
    for on in (0, 1):
        _lib.set_pdl(bool(on))
        n2 = Network(spec, max_batch=1)
        forward(n2, img)
        torch.cuda.synchronize()
        e0.record(); [n2._graphs[1].replay() for _ in range(200)]; e1.record(); torch.cuda.synchronize()
        print(name, "compute graph pdl", on, f"{e0.elapsed_time(e1) / 200 * 1e3:.1f} us")
    print(name, f"compute-only graph device {dev_c:.1f} us")
    print(name, f"io1 graph back-to-back device {dev_back2back:.1f} us | replay+sync wall {t_rs:.1f} us | forward() wall {t_fw:.1f} us", "graphs", list(net._graphs))
