"""Debug: IVF batch vs single-query results vs oracle on a c4-shaped index."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import fullsize

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
cfg = dict(fullsize.CONFIGS["c4"]); cfg["n"] = n
w = fullsize.build(cfg, nq=nq)
idx = fullsize.make_index(w)
Y = w["queries"]
d, i = idx.search(Y, 100, ma=64, mode="derived", r2=1000)
sel = np.linspace(0, nq - 1, 16).astype(int)
bad = []
for q in sel:
    d1, i1 = idx.search(Y[q:q + 1], 100, ma=64, mode="derived", r2=1000)
    if not (np.array_equal(d1[0], d[q]) and np.array_equal(i1[0], i[q])):
        bad.append((q, d1[0], i1[0]))
print("mismatching queries:", [b[0] for b in bad])
if bad:
    orc = fullsize.oracle_rows(w, [b[0] for b in bad], 100)
    for q, d1, i1 in bad:
        od, oi = orc[q]
        print(q, "batch==oracle", np.array_equal(oi, i[q]) and np.array_equal(od, d[q]),
              "single==oracle", np.array_equal(oi, i1) and np.array_equal(od, d1))
