"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over the hot kernels: the flat derived search on the golden
fixtures (generic, wide 5/6-bit and run-filtered scan loops, refine, group
tables), the IVF derived search, the device shard protocol + merge, and the
tensor-core encoder.

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py
"""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import c1_codebooks, load_golden  # noqa: E402
from oracle import derived_search as O  # noqa: E402
from paper_1905_06900_b200 import _lib  # noqa: E402
from paper_1905_06900_b200.flat import FlatIndex  # noqa: E402
from paper_1905_06900_b200.ivf import IVFIndex  # noqa: E402


def flat_golden():
    g = load_golden("pq_blobs")
    m = g["meta"]
    d, i = FlatIndex.from_arrays(g["codebooks"], g["derived"], g["codes"]).search(g["queries"], m["r"],
                                                                               mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])


def flat_c1(nq=16, n=30000):
    g = load_golden("c1_sampled")
    cb = c1_codebooks(g)
    codes = g["codes"][:n]
    Y = g["queries"][:nq]
    idx = FlatIndex.from_arrays(cb, g["derived"], codes)
    d, i = idx.search(Y, 100, mode="derived", r2=1000)
    d0, i0 = O.flat_search(cb, g["derived"], codes, Y[:2], 100, "derived", 1000)
    assert np.array_equal(i[:2], i0)
    idx.search(Y[:4], 10)  # conventional path


def ivf_golden():
    g = load_golden("ivf_blobs")
    m = g["meta"]
    idx = IVFIndex.from_arrays(g["codebooks"], g["derived"], g["centers"], g["offsets"], g["sorted_codes"],
                               g["sorted_ids"], cell_of=g.get("cell_of"))
    d, i = idx.search(g["queries"], m["r"], ma=m["ma"], mode="derived", r2=m["r2"])
    assert np.array_equal(i, g["exp_derived_i"])


def encoder_small():
    g = load_golden("c1_sampled")
    cb = c1_codebooks(g)
    enc = _lib.Encoder(cb, device=0)
    X = np.random.default_rng(0).uniform(0, 64, size=(700, 128)).astype(np.float32)
    enc.encode(X)


if __name__ == "__main__":
    which = sys.argv[1:] or ["flat_golden", "flat_c1", "ivf_golden", "encoder_small"]
    for w in which:
        globals()[w]()
        print(w, "ok", flush=True)
