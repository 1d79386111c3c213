"""Break down the host-API (e2e) cost of one 1024-query batch."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import FlatIndex

rng = np.random.default_rng(0)
n, k, m, dsub = 10_000_000, 65536, 4, 32
cb = (rng.random((m, k, dsub), dtype=np.float32) * 100)
der = cb.reshape(m, 256, 256, dsub).mean(axis=1).astype(np.float32)
codes = rng.integers(0, k, size=(n, m)).astype(np.uint16)
Y = (rng.random((1024 * 4, m * dsub), dtype=np.float32) * 100)
idx = FlatIndex.from_arrays(cb, der, codes)
h = idx._handle()
L = _lib.lib()
for rep in range(4):
    q = Y[rep * 1024:(rep + 1) * 1024]
    t0 = time.perf_counter(); d, i = idx.search(q, 100, mode="derived", r2=1000); t1 = time.perf_counter()
    dd = np.empty((1024, 100)); ii = np.empty((1024, 100), np.int64)
    t2 = time.perf_counter()
    rc = L.dpq_flat_search_derived(h.raw, _lib.ptr(q), 1024, 100, 1000, 1, _lib.ptr(dd), _lib.ptr(ii), None)
    t3 = time.perf_counter()
    h.set_timing(True)
    rc = L.dpq_flat_search_derived(h.raw, _lib.ptr(q), 1024, 100, 1000, 1, _lib.ptr(dd), _lib.ptr(ii), None)
    t4 = time.perf_counter()
    ph = h.phase_ms()
    h.set_timing(False)
    print(f"search {1e3*(t1-t0):.2f} ms | C call {1e3*(t3-t2):.2f} ms | C call+timing {1e3*(t4-t3):.2f} ms | phases {np.round(ph,3)}", flush=True)
print(h.counters())

# bench conditions: torch stream + L2 flush before each step
stream = torch.cuda.Stream()
h.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in ("noflush", "flush", "flush+sleep"):
    ts = []
    for rep in range(4):
        q = Y[rep * 1024:(rep + 1) * 1024]
        if mode != "noflush":
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
        if mode == "flush+sleep":
            time.sleep(0.05)
        t0 = time.perf_counter(); d, i = idx.search(q, 100, mode="derived", r2=1000); ts.append(time.perf_counter() - t0)
    print(mode, [round(1e3 * t, 2) for t in ts], flush=True)
