"""Container load throughput: the reference's
vecio.load_model (host read + zlib CRC-32 + validate) vs the device loader
(container.load_model: threaded reads into pinned buffers, H2D, CRC-32 and
validation on the GPU), on a flat PQ 4x16 index of N codes written in the
reference's format; plus the device CRC kernel alone (CUDA events).

    python scripts/container_bench.py [--n 100000000] > profiles/r2_container_bench.json

Both loaders read the same file from the page cache (it was just written).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--crc-mb", type=int, default=4096)
    args = ap.parse_args()
    import torch

    from paper_1905_06900_b200 import container as C
    from paper_1905_06900_b200.flat import FlatIndex

    rng = np.random.default_rng(0)
    m, k, kbar, dsub = 4, 65536, 256, 32
    cb = rng.normal(size=(m, k, dsub)).astype(np.float32)
    dcb = rng.normal(size=(m, kbar, dsub)).astype(np.float32)
    codes = rng.integers(0, 65536, size=(args.n, m), dtype=np.uint16)
    idx = FlatIndex.from_arrays(cb, dcb, codes)
    q = idx.quantizer
    q._kind, q._params, q.distortions_ = "pq", {"m": m, "b": 16, "bbar": 8, "seed": 42, "max_iters": 50}, np.zeros(m)
    out = {"n": args.n, "codes_bytes": int(codes.nbytes)}
    with tempfile.TemporaryDirectory(prefix="dpqc_") as tmp:
        path = Path(tmp) / "flat.dpq"
        t0 = time.perf_counter()
        C.save_model(idx, path)
        out["file_bytes"] = path.stat().st_size
        out["save_s"] = round(time.perf_counter() - t0, 3)
        del idx
        # device loader (twice: the first call pays CUDA/pinned setup)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev = C.load_model(path)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            st = dict(C.load_model.last_stats)
            del dev
        out["device_loader"] = {"total_s": round(dt, 3), "bulk_read_and_crc_s": round(st["total_s"], 3),
                                "host_read_s": round(st["read_s"], 3),
                                "bulk_gbs": round(st["bytes"] / st["total_s"] / 1e9, 2),
                                "note": "includes handle build (row sort, plane) and device validation"}
        # the reference's loader
        if REF.exists():
            sys.path.insert(0, str(REF))
            from derivedpq import load_model as ref_load

            t0 = time.perf_counter()
            r = ref_load(path)
            out["reference_loader"] = {"total_s": round(time.perf_counter() - t0, 3),
                                       "what": "derivedpq.vecio.load_model(path) (baseline/_ref, unmodified): "
                                               "read + zlib.crc32 + copy + validate, one host thread"}
            del r
    # CRC kernel alone
    nb = args.crc_mb << 20
    buf = torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda")
    C.crc32_device(buf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        c = C.crc32_device(buf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    h = buf[: 64 << 20].cpu().numpy()
    t0 = time.perf_counter()
    zlib.crc32(h)
    zs = time.perf_counter() - t0
    out["crc_kernel"] = {"bytes": nb, "ms": round(ms, 3), "gbs": round(nb / ms / 1e6, 1),
                         "zlib_host_gbs": round(h.nbytes / zs / 1e9, 2),
                         "note": "per call incl. scratch alloc + sync (dpq_crc32_dev)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
