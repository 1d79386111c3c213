"""Break down the host-API (e2e) cost of one 1024-query batch on the bench
workload: Python wrapper vs C call vs device batch."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import bench
from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import FlatIndex

sys.argv = [sys.argv[0], "--steps", "8", "--warmup", "0"]
args = bench.parse()
w = bench.build_workload(args, "cuda:0")
Y = np.ascontiguousarray(w["queries"][: 8 * 1024])
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
h = idx._handle()
L = _lib.lib()
dd = np.empty((1024, 100))
ii = np.empty((1024, 100), np.int64)
idx.search(Y[:1024], 100, mode="derived", r2=1000)
for rep in range(1, 8):
    q = Y[rep * 1024:(rep + 1) * 1024]
    t0 = time.perf_counter()
    d, i = idx.search(q, 100, mode="derived", r2=1000)
    t1 = time.perf_counter()
    rc = L.dpq_flat_search_derived(h.raw, _lib.ptr(q), 1024, 100, 1000, 1, _lib.ptr(dd), _lib.ptr(ii), None)
    t2 = time.perf_counter()
    h.set_timing(True)
    L.dpq_flat_search_derived(h.raw, _lib.ptr(q), 1024, 100, 1000, 1, _lib.ptr(dd), _lib.ptr(ii), None)
    h.set_timing(False)
    ph = h.phase_ms()
    print(f"python search {1e3 * (t1 - t0):.3f} ms | C call {1e3 * (t2 - t1):.3f} ms | device batch {ph[6]:.3f} ms",
          flush=True)
