"""Event timeline of one pipelined forward_batch (BMLP 16384, pinned in/out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_07175_b200 import zoo, forward_batch
from paper_1705_07175_b200.network import Network
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
net = Network(zoo.bmlp_spec(), max_batch=B)
imgs = net.pinned_images(B); imgs[:] = 1
out = net.pinned_scores(B)
for _ in range(3): forward_batch(net, imgs, out)
torch.cuda.synchronize()
marks = []
orig_run = net.run
T0 = torch.cuda.Event(enable_timing=True)
def ev(tag, stream=None):
    e = torch.cuda.Event(enable_timing=True); e.record(stream or torch.cuda.current_stream()); marks.append((tag, e, time.perf_counter()))
def run(b):
    ev(f"run{b} start"); orig_run(b); ev(f"run{b} end")
net.run = run
T0.record(); h0 = time.perf_counter()
forward_batch(net, imgs, out)
ev("done")
torch.cuda.synchronize()
h1 = time.perf_counter()
for tag, e, h in marks:
    print(f"{tag:22s} gpu {T0.elapsed_time(e) * 1e3:8.1f} us   host {(h - h0) * 1e6:8.1f} us")
print("host total", (h1 - h0) * 1e6)
print("plan", net._chunk_plan(B, True))
