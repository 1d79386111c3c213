"""Tensor-core encoder throughput (dpq_encode_dev) vs the torch/cuBLAS
encoder (train.encode), on seeded SIFT-like rows (tf32-exact: 2 passes) and
on float rows (3 passes), PQ 4x16 (k = 65536, dsub = 32).

    python scripts/encode_bench.py [--n 10000000]

Prints one JSON line: rows/s, algorithmic TFLOP/s (2 n m k dsub per encode)
and MMA TFLOP/s actually issued, agreement with the torch encoder.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1905_06900_b200 import _lib, datagen, train

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--n-torch", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
m, k, dsub = 4, 65536, 32
st = datagen.seed_streams(42)
centres = datagen.sift_centres(st["centres"])
pts = datagen.sift_like(st["train"], centres, k)
rng = np.random.default_rng(1)
cb = np.stack([pts[rng.permutation(k), j * dsub:(j + 1) * dsub] + rng.normal(0, 0.5, (k, dsub))
               for j in range(m)]).astype(np.float32)
enc = _lib.Encoder(cb)
out = {"n": a.n, "m": m, "k": k, "dsub": dsub}
for kind in ("sift_int", "float"):
    x = datagen.sift_like_torch(a.n, 7, centres, device=dev)
    if kind == "float":
        x += torch.rand_like(x)
    codes = torch.empty((a.n, m), dtype=torch.int32, device=dev)
    enc.encode_dev(x[:1024], codes[:1024])
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        enc.encode_dev(x, codes)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = min(ts)
    passes = 2 if kind == "sift_int" else 3
    kp = 32 * passes + 8
    res = {"s": round(t, 4), "rows_per_s": a.n / t,
           "alg_tflops": 2.0 * a.n * m * k * dsub / t / 1e12,
           "mma_tflops": 2.0 * a.n * m * k * kp / t / 1e12, "passes": passes}
    nt = min(a.n, a.n_torch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ref = train.encode(x[:nt], cb)
    torch.cuda.synchronize()
    tt = time.perf_counter() - t0
    res["torch_rows_per_s"] = nt / tt
    res["agree_vs_torch_tf32"] = float((ref == codes[:nt]).float().mean())
    # exact f64 check on a sample
    xs = x[:2000].double()
    exact = torch.empty((2000, m), dtype=torch.int64, device=dev)
    for j in range(m):
        c = torch.as_tensor(cb[j], device=dev).double()
        sub = xs[:, j * dsub:(j + 1) * dsub]
        d2 = (c * c).sum(1)[None, :] - 2 * sub @ c.T
        exact[:, j] = d2.argmin(1)
    res["agree_vs_f64_sample"] = float((exact == codes[:2000].long()).float().mean())
    out[kind] = res
    del x, codes
    torch.cuda.empty_cache()
print(json.dumps(out))
