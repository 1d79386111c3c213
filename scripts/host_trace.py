"""Host-side segments of FlatIndex.search on the bench workload: the C call's
own trace (DPQ_HOST_TRACE) next to the Python wrapper's steps.

    python scripts/host_trace.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["DPQ_HOST_TRACE"] = "1"
import numpy as np
import torch

import bench
from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import FlatIndex, rotated_queries
from sklearn.utils.validation import check_is_fitted

sys.argv = [sys.argv[0]]
args = bench.parse()
cfg, _ = bench.resolve(args, 1)
w = bench.build_flat(cfg, args, torch.device("cuda", 0), 0, cfg["n"], 12 * 1024)
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
for s in range(6):
    q = w["queries"][s * 1024:(s + 1) * 1024]
    t0 = time.perf_counter()
    d, i = idx.search(q, 100, mode="derived", r2=1000)
    print(f"search {1e6 * (time.perf_counter() - t0):.1f} us", file=sys.stderr)
L = _lib.lib()
h = idx._handle()
for s in range(6, 12):
    Y = w["queries"][s * 1024:(s + 1) * 1024]
    t = [time.perf_counter()]
    check_is_fitted(idx, "codes_"); t.append(time.perf_counter())
    Yq = _lib.query_array(Y); t.append(time.perf_counter())
    yr = rotated_queries(idx.quantizer, Yq); t.append(time.perf_counter())
    dists = np.empty((1024, 100)); ids = np.empty((1024, 100), dtype=np.int64); t.append(time.perf_counter())
    rc = L.dpq_flat_search_derived(h.raw, _lib.ptr(yr), 1024, 100, 1000, 1, _lib.ptr(dists), _lib.ptr(ids),
                                   _lib.ptr(None)); t.append(time.perf_counter())
    seg = [1e6 * (b - a) for a, b in zip(t, t[1:])]
    print("py segments us: fitted %.1f | query_array %.1f | rotate %.1f | alloc %.1f | C call %.1f" % tuple(seg),
          file=sys.stderr)
