"""Distribution of the bucket cut b* (and candidate counts) on the bench workload."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import bench
from paper_1905_06900_b200.flat import FlatIndex

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--r2", type=int, default=1000)
a = ap.parse_args()
sys.argv = [sys.argv[0], "--n", str(a.n), "--steps", "1", "--warmup", "0"]
args = bench.parse()
w = bench.build_workload(args, "cuda:0")
idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
bstar, ncand = idx.candidate_counts(w["queries"][:1024], a.r2)
print("b* percentiles (0,10,50,90,100):", np.percentile(bstar, [0, 10, 50, 90, 100]))
print("candidates percentiles:", np.percentile(ncand, [0, 10, 50, 90, 100]))
hist = np.bincount(bstar, minlength=256)
print("b* <= 30:", (bstar <= 30).mean(), " <= 62:", (bstar <= 62).mean(), " <= 126:", (bstar <= 126).mean())
small, q, qmin, qmax = idx.quantized_tables(w["queries"][:64], a.r2)
print("table entries <= 31 fraction:", (q <= 31).mean(), " <= 63:", (q <= 63).mean())

# score at the guard's target rank (sample 16384 of N: lambda + 3 sqrt(lambda) + 4 hits)
import torch
codes = torch.as_tensor(w["codes"].astype(np.int32), device="cuda")
lo = (codes & 0xFF).long()
qt = torch.as_tensor(q.astype(np.int32), device="cuda")  # (64, m, kbar)
lam = a.r2 * 16384 / a.n
rank_g = int((lam + 3 * lam ** 0.5 + 4) / 16384 * a.n)
gs, bs = [], []
for i in range(qt.shape[0]):
    s = sum(qt[i, j][lo[:, j]] for j in range(lo.shape[1]))
    h = torch.bincount(s.clamp(max=255), minlength=256).cumsum(0)
    bs.append(int((h >= a.r2).nonzero()[0]))
    gs.append(int((h >= rank_g).nonzero()[0]))
gs, bs = np.array(gs), np.array(bs)
print("rank_g", rank_g, "b* (torch)", np.percentile(bs, [0, 50, 90, 100]), "guard-rank score", np.percentile(gs, [0, 50, 90, 100]))
print("guard <= 30:", (gs <= 30).mean(), "<= 62:", (gs <= 62).mean())
