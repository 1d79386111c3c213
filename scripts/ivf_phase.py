"""IVF (configs[3] shape) phase split: N rows per GPU, nq queries per
search call, batches of the driver's default size; prints queries/s and the
per-batch phase times (CUDA events), and with DPQ_HOST_TRACE=1 the host
segments of each batch.

    python scripts/ivf_phase.py [N] [nq] [reps]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import fullsize  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = dict(fullsize.CONFIGS["c4"])
cfg["n"] = n
w = fullsize.build(cfg, nq=nq)
idx = fullsize.make_index(w)
Y = w["queries"]
idx.search(Y, 100, ma=64, mode="derived", r2=1000)  # warm-up (buffers, plans)
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    d, i = idx.search(Y, 100, ma=64, mode="derived", r2=1000)
    ts.append(time.perf_counter() - t0)
d, i, t = idx.search(Y, 100, ma=64, mode="derived", r2=1000, return_timings=True)
h = idx._handle()
out = {"n": n, "nq": nq, "qps_host": round(nq / min(ts), 1), "search_s": [round(x, 4) for x in ts],
       "phase_us_per_query": {k: round(float(np.mean(v)), 3) for k, v in t.items()},
       "last_batch_ms": dict(zip(("tables", "guard", "scan", "threshold", "refine", "fallback(probe)", "total"),
                                 [round(float(x), 4) for x in h.phase_ms()])),
       "counters": h.counters_ex()}
print(json.dumps(out))
