"""H2D / D2H bandwidth of this box and the BMLP forward_batch timeline."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
for mb in (0.25, 1, 3.2, 12.8, 64):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    e0.record()
    for _ in range(20): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t2 = e0.elapsed_time(e1) / 20
    print(f"{mb:6.2f} MB  H2D {n / t / 1e6:.1f} GB/s  D2H {n / t2 / 1e6:.1f} GB/s")
# concurrent H2D on a side stream while the compute stream runs a kernel-heavy loop
from paper_1705_07175_b200 import zoo, forward_batch
from paper_1705_07175_b200.network import Network
for name, spec, B in (("bmlp", zoo.bmlp_spec(), 16384), ("bcnn", zoo.bcnn_spec(), 8192)):
    net = Network(spec, max_batch=B)
    imgs = net.pinned_images(B)
    imgs[:] = np.random.default_rng(0).integers(0, 256, imgs.shape, dtype=np.uint8)
    for _ in range(3): forward_batch(net, imgs)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); forward_batch(net, imgs); ts.append(time.perf_counter() - t0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    net.input_device[:B].copy_(torch.from_numpy(imgs).cuda())
    net.run(B); torch.cuda.synchronize(); e0.record()
    for _ in range(10): net.run(B)
    e1.record(); torch.cuda.synchronize()
    print(name, f"forward_batch wall {np.median(ts) * 1e3:.3f} ms  ({B / np.median(ts) / 1e6:.2f} M img/s)  device-only {e0.elapsed_time(e1) / 10:.3f} ms  in {imgs.nbytes / 1e6:.1f} MB")
