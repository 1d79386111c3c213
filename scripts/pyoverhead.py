"""Python-side overhead of FlatIndex.search pieces, called the way the e2e
loop calls them (a ~1 ms GPU wait between calls)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from sklearn.utils.validation import check_is_fitted

from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import FlatIndex, rotated_queries

rng = np.random.default_rng(0)
cb = rng.normal(size=(4, 256, 32)).astype(np.float32)
codes = rng.integers(0, 256, (1000, 4)).astype(np.uint16)
idx = FlatIndex.from_arrays(cb, cb[:, :256].copy(), codes)
Y = rng.normal(size=(1024, 128)).astype(np.float32)


def t(f, n=300):
    out = []
    for _ in range(n):
        time.sleep(0.001)
        t0 = time.perf_counter()
        f()
        out.append(time.perf_counter() - t0)
    return round(float(np.median(out)) * 1e6, 1)


print("check_is_fitted", t(lambda: check_is_fitted(idx, "codes_")))
print("query_array", t(lambda: _lib.query_array(Y)))
print("rotated", t(lambda: rotated_queries(idx.quantizer, Y)))
print("empty x2", t(lambda: (np.empty((1024, 100)), np.empty((1024, 100), np.int64))))
h = idx._handle()
print("_handle", t(lambda: idx._handle()))
L = _lib.lib()
d = np.empty((1024, 100)); i = np.empty((1024, 100), np.int64)
print("ptr x4", t(lambda: (_lib.ptr(Y), _lib.ptr(d), _lib.ptr(i), _lib.ptr(None))))
