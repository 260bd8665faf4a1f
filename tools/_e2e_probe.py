"""Where the BMLP / BCNN forward_batch time goes: device time per chunk size,
wall time with the final host copy removed, chunk-count sweep."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_07175_b200 import zoo, forward_batch
from paper_1705_07175_b200 import network as nw
from paper_1705_07175_b200.network import Network
def dev_time(net, b, reps=10):
    net.run(b); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): net.run(b)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for name, spec, B in (("bmlp", zoo.bmlp_spec(), 16384), ("bcnn", zoo.bcnn_spec(), 8192)):
    net = Network(spec, max_batch=B)
    imgs = net.pinned_images(B)
    imgs[:] = np.random.default_rng(0).integers(0, 256, imgs.shape, dtype=np.uint8)
    for b in (B // 8, B // 4, B // 2, B):
        print(name, f"device t({b}) = {dev_time(net, b):.3f} ms  x{B // b} = {dev_time(net, b) * B / b:.3f}")
    out = np.empty((B, net.classes))
    for _ in range(3): forward_batch(net, imgs, out)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); forward_batch(net, imgs, out); ts.append(time.perf_counter() - t0)
    print(name, f"forward_batch(out=) wall {np.median(ts) * 1e3:.3f} ms")
    t0 = time.perf_counter()
    for _ in range(10): out[:] = net._out_host_np[:B]
    print(name, f"final host copy {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
