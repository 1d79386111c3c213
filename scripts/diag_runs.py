"""Fraction of (g0, g1) runs a query tile could skip (no query with e0+e1 <= B)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1905_06900_b200.flat import FlatIndex

sys.argv = [sys.argv[0], "--n", "10000000", "--steps", "1", "--warmup", "0"]
args = bench.parse()
w = bench.build_workload(args, "cuda:0")
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
Y = w["queries"][:1024]
bstar, _ = idx.candidate_counts(Y, 1000)
_, q8, _, _ = idx.quantized_tables(Y, 1000)
codes = torch.as_tensor(w["codes"].astype(np.int32), device="cuda")
key = (codes[:, 0] & 255) * 256 + (codes[:, 1] & 255)
runw = torch.bincount(key, minlength=65536).double()  # rows per (g0, g1)
q = torch.as_tensor(q8.astype(np.int32), device="cuda")
B = torch.as_tensor(bstar, device="cuda")
P = q[:, 0, :, None] + q[:, 1, None, :]  # (1024, 256, 256) partial sums
pot = (P <= B[:, None, None]).reshape(1024, -1)  # query can still hit in run
print("per-query potential row fraction:", float((pot.double() @ runw).mean() / runw.sum()))
g0s = q[:, 0, :].argmin(1).cpu().numpy(); g1s = q[:, 1, :].argmin(1).cpu().numpy()
orders = {
    "identity": np.arange(1024),
    "by B": np.argsort(bstar, kind="stable"),
    "by (B>30, g0*, g1*)": np.lexsort((g1s, g0s, bstar > 30)),
    "by (g0*, g1*)": np.lexsort((g1s, g0s)),
}
for name, order in orders.items():
    for qt in (128, 64, 32):
        fr = []
        for t in range(0, 1024, qt):
            sl = torch.as_tensor(order[t:t + qt], device="cuda")
            anyp = pot[sl].any(0).double()
            fr.append(float(anyp @ runw / runw.sum()))
        print(f"{name:24s} QT={qt:3d}: rows with potential {np.mean(fr):.3f}")
