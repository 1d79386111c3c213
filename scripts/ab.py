"""A/B two libdpq builds on the same box and workload: device ms per
1024-query batch (L2 flushed between steps), interleaved A, B, A, B ...

    python scripts/ab.py OLD.so NEW.so [--reps 4] [--steps 10]
    python scripts/ab.py LIB.so:DPQ_REFINE_WARP=0 LIB.so:DPQ_REFINE_WARP=1

A spec PATH:VAR=VAL[,VAR=VAL] sets environment variables while that
variant's index is created.  Also checks that every variant returns the
same ids and distances as the first.
"""
import os
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_1905_06900_b200 import _lib
from paper_1905_06900_b200.flat import FlatIndex

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
sys.argv = [sys.argv[0], "--steps", str(a.steps), "--warmup", "3"]
args = bench.parse()
cfg, _ = bench.resolve(args, 1)
w = bench.build_flat(cfg, args, torch.device("cuda", 0), 0, cfg["n"], a.steps * 1024)
Q = torch.as_tensor(w["queries"][: a.steps * 1024], device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
results = {p: [] for p in a.libs}
ref_out = None
phases = {p: [] for p in a.libs}
for rep in range(a.reps):
    for path in a.libs:
        lib_path, _, env = path.partition(":")
        saved = {}
        for kv in filter(None, env.split(",")):
            kk, vv = kv.split("=", 1)
            saved[kk] = os.environ.get(kk)
            os.environ[kk] = vv
        _lib._PATH = Path(lib_path).resolve()
        _lib._lib = None
        idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"])
        h = idx._handle()
        stream = torch.cuda.Stream()
        h.set_stream(stream.cuda_stream)
        L = _lib.lib()
        out_d = torch.empty((1024, 100), dtype=torch.float64, device="cuda")
        out_i = torch.empty((1024, 100), dtype=torch.int64, device="cuda")
        ts = []
        with torch.cuda.stream(stream):
            for s in range(-3, a.steps):
                q = Q[(max(s, 0) % a.steps) * 1024:][:1024]
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _lib.check(L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(q), 1024, 100, 1000, _lib.ptr(out_d),
                                                         _lib.ptr(out_i)), "search")
                e1.record(stream)
                stream.synchronize()
                if s >= 0:
                    ts.append(e0.elapsed_time(e1))
        h.set_timing(True)
        with torch.cuda.stream(stream):
            _lib.check(L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(Q[:1024]), 1024, 100, 1000, _lib.ptr(out_d),
                                                     _lib.ptr(out_i)), "search")
        stream.synchronize()
        phases[path].append(h.phase_ms().copy())
        got = (out_d.cpu().numpy().copy(), out_i.cpu().numpy().copy())
        if ref_out is None:
            ref_out = got
        elif not (np.array_equal(got[0], ref_out[0]) and np.array_equal(got[1], ref_out[1])):
            print(f"RESULTS DIFFER: {path}", flush=True)
        h.set_stream(None)
        del idx, h
        for kk, vv in saved.items():  # the variant's environment held for its searches too
            if vv is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = vv
        torch.cuda.synchronize()
        results[path].append(float(np.median(ts)))
for path in a.libs:
    ph = np.median(np.array(phases[path]), axis=0)
    print(f"{Path(path).name:28s} median batch ms {np.median(results[path]):.4f}  runs {np.round(results[path], 4)}"
          f"  phases {np.round(ph, 3)}", flush=True)
