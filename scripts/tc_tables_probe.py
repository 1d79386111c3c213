"""One derived search on a configs[4]-shaped flat index (PQ 8x65536, dsub =
120, derived 8x256) with random codes, so the only k_tct_gemm launches are
the search's tensor-core full tables (no encoder): for an ncu capture.

    ncu --set full -k regex:k_tct_gemm -s 1 -c 1 python scripts/tc_tables_probe.py [n] [nq]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_1905_06900_b200.flat import FlatIndex  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(5)
m, k, kbar, dsub = 8, 65536, 256, 120
centres = rng.uniform(0, 1, size=(64, m * dsub)).astype(np.float32)
cb = (centres[rng.integers(0, 64, size=k)].reshape(k, m, dsub).transpose(1, 0, 2)
      + rng.normal(0, 0.05, size=(m, k, dsub))).astype(np.float32)
der = cb.reshape(m, k // kbar, kbar, dsub).mean(axis=1).astype(np.float32)  # group means (low bits = group)
codes = rng.integers(0, k, size=(n, m), dtype=np.uint16)
Y = (centres[rng.integers(0, 64, size=nq)] + rng.normal(0, 0.05, size=(nq, m * dsub))).astype(np.float32)
idx = FlatIndex.from_arrays(cb, der, codes)
for _ in range(2):
    d, i = idx.search(Y, 100, mode="derived", r2=2000)
print("done", i[0, :3])
