"""Host-side cost of writing one batch of results (1.6 MB) into fresh numpy
arrays (first-touch page faults) vs into already-touched memory."""
import time

import numpy as np

src = np.random.rand(1024 * 100 * 2)
for label, fresh in (("fresh np.empty", True), ("reused", False)):
    dst = np.empty_like(src)
    ts = []
    for _ in range(30):
        if fresh:
            dst = np.empty_like(src)
        t0 = time.perf_counter()
        np.copyto(dst, src)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{label:16s} copy 1.6 MB: {ts[len(ts) // 2] * 1e6:7.1f} us")
import os
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), "cpus", os.cpu_count())
