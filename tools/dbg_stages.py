"""Debug aid: compare every device stage of a BCNN forward (image 0) with the
reference's per-stage golden intermediates (tests/golden/networks.npz) at
several batch sizes.  python tools/dbg_stages.py (on a GPU box)."""
import numpy as np, torch, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1705_07175_b200 import zoo, _dev, forward_batch
from paper_1705_07175_b200.network import Network
g = np.load(__import__("os").path.join(sys.path[0], "tests", "golden", "networks.npz"))
imgs = g["bcnn_images"]
ref_of = {0: 2, 1: 5, 2: 7, 3: 10, 4: 12, 5: 15, 6: 17, 7: 19, 8: 21}  # 8 = dense + final batch-norm
for B in (1, 24, 300):
    net = Network(zoo.bcnn_spec(), max_batch=B, use_graphs=False)
    x = imgs[np.arange(B) % 24]
    forward_batch(net, x)
    bad = []
    for i, st in enumerate(net.stages):
        o = st.out[0].detach().cpu().numpy()
        r = g[f"bcnn_stage{ref_of[i]}"]
        o = o.view(np.uint64) if o.dtype == np.int64 and r.dtype == np.uint64 else o
        ok = np.array_equal(o.reshape(-1), r.reshape(-1).astype(o.dtype))
        bad.append((i, st.name, ok))
    print(B, bad)
