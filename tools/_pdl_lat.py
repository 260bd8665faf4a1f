import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1705_07175_b200 import zoo, _lib
for on in (0, 1, 0, 1):
    _lib.set_pdl(bool(on))
    print("pdl", on, bench.batch1_latency(zoo.bcnn_spec(), (32,32,3))["us_per_image"], bench.batch1_latency(zoo.bmlp_spec(), (784,))["us_per_image"], flush=True)
