"""One c4-shaped IVF batch for an ncu launch list (N rows, nq queries)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import fullsize

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = dict(fullsize.CONFIGS["c4"]); cfg["n"] = n
w = fullsize.build(cfg, nq=nq)
idx = fullsize.make_index(w)
for _ in range(2):
    idx.search(w["queries"], 100, ma=64, mode="derived", r2=1000)
print("done")
