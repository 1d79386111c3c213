import sys, os
sys.path.insert(0, "/root/repo")
os.environ["DPQ_HOST_TRACE"] = "1"
import numpy as np, torch
import bench
from paper_1905_06900_b200.flat import FlatIndex
sys.argv = [sys.argv[0]]
args = bench.parse()
cfg, _ = bench.resolve(args, 1)
w = bench.build_flat(cfg, args, torch.device("cuda", 0), 0, cfg["n"], 8 * 1024)
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
import time
for s in range(8):
    q = w["queries"][s * 1024:(s + 1) * 1024]
    t0 = time.perf_counter()
    d, i = idx.search(q, 100, mode="derived", r2=1000)
    print(f"search {1e6*(time.perf_counter()-t0):.1f} us", file=sys.stderr)
