"""Per-query statistics of the (g0, g1) run filter on the bench workload:
how many rows share a key with e0[g0] + e1[g1] <= b* for ONE query (the
tile-level figure of the scan is the union over 128 clustered queries).

    python scripts/key_potential.py [--r2 1000] [--nq 1024]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1905_06900_b200.flat import FlatIndex

ap = argparse.ArgumentParser()
ap.add_argument("--r2", type=int, nargs="+", default=[1000])
ap.add_argument("--nq", type=int, default=1024)
a = ap.parse_args()
sys.argv = [sys.argv[0]]
args = bench.parse()
cfg, _ = bench.resolve(args, 1)
w = bench.build_flat(cfg, args, torch.device("cuda", 0), 0, cfg["n"], a.nq)
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
codes = torch.as_tensor(w["codes"].astype(np.int32), device="cuda")
low = codes & 0xFF
key = (low[:, 0] | (low[:, 1] << 8)).long()
runlen = torch.bincount(key, minlength=65536).double().view(256, 256)  # [g1][g0]
key3 = (key | (low[:, 2].long() << 16))
runlen3 = torch.bincount(key3, minlength=1 << 24).double().view(256, 256, 256)  # [g2][g1][g0]
out = {}
for r2 in a.r2:
    _, q8, _, _ = idx.quantized_tables(w["queries"][: a.nq], r2)
    bstar, ncand = idx.candidate_counts(w["queries"][: a.nq], r2)
    q = torch.as_tensor(q8.astype(np.int32), device="cuda")
    b = torch.as_tensor(bstar, device="cuda")
    rows2 = torch.empty(a.nq, dtype=torch.float64, device="cuda")
    keys2 = torch.empty(a.nq, dtype=torch.float64, device="cuda")
    rows3 = torch.empty(a.nq, dtype=torch.float64, device="cuda")
    keys3 = torch.empty(a.nq, dtype=torch.float64, device="cuda")
    for i in range(a.nq):
        s01 = q[i, 1][:, None] + q[i, 0][None, :]          # [g1][g0]
        ok = s01 <= b[i]
        rows2[i] = (runlen * ok).sum()
        keys2[i] = ok.sum()
        s012 = q[i, 2][:, None, None] + s01[None]
        ok3 = s012 <= b[i]
        rows3[i] = (runlen3 * ok3).sum()
        keys3[i] = (ok3 & (runlen3 > 0)).sum()
    st = lambda t: {"mean": float(t.mean()), "median": float(t.median()), "max": float(t.max())}
    out[str(r2)] = {"bstar": st(b.double()), "ncand": st(torch.as_tensor(ncand).double()),
                    "rows_key2": st(rows2), "keys2": st(keys2), "rows_key3": st(rows3), "keys3_nonempty": st(keys3)}
print(json.dumps(out, indent=1))
