"""Generate the model-container fixtures under tests/golden/containers/ with
the REFERENCE's own save_model (derivedpq.vecio.save_model, vecio.py:124-153).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_containers.py

Each case writes `<case>.dpq` (the reference's bytes) and `<case>.npz` with
queries and the reference's own search results on the model it saved, so the
GPU loader (paper_1905_06900_b200.container.load_model) is pinned to the
reference on both the file format and the search it feeds.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from derivedpq import FlatIndex, IVFIndex, OptimizedProductQuantizer, ProductQuantizer, save_model

OUT = Path(__file__).resolve().parent / "containers"


def blobs(rng, n, d, centres=16, scale=4.0):
    c = rng.uniform(0, 64, size=(centres, d))
    return (c[rng.integers(0, centres, n)] + rng.normal(0, scale, size=(n, d))).astype(np.float32)


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(1905)
    # quantizer only (test_vecio.py:120-123 shape)
    Xq = rng.normal(size=(600, 8)).astype(np.float32)
    pq = ProductQuantizer(m=2, b=4, bbar=2, seed=5).fit(Xq)
    save_model(pq, OUT / "pq_small.dpq")
    np.savez(OUT / "pq_small.npz", X=Xq, codes=pq.encode(Xq))
    # flat PQ 4x8 / derived 4x4 (u8 codes) and 2x10 / derived 2x6 (u16 codes)
    for name, m, b, bbar, d in (("flat_u8", 4, 8, 4, 16), ("flat_u16", 2, 10, 6, 8)):
        X = blobs(rng, 3000, d)
        Y = blobs(rng, 12, d)
        idx = FlatIndex(ProductQuantizer(m=m, b=b, bbar=bbar, seed=3, max_iters=8)).fit(X)
        save_model(idx, OUT / f"{name}.dpq")
        dc, ic = idx.search(Y, 10)
        dd, id_ = idx.search(Y, 10, mode="derived", r2=200)
        np.savez(OUT / f"{name}.npz", queries=Y, exp_conv_d=dc, exp_conv_i=ic, exp_der_d=dd, exp_der_i=id_,
                 meta=json.dumps({"r": 10, "r2": 200}))
    # OPQ flat (rotation array)
    X = blobs(rng, 3000, 8)
    Y = blobs(rng, 8, 8)
    idx = FlatIndex(OptimizedProductQuantizer(m=2, b=8, bbar=4, seed=4, max_iters=6, outer_iters=2,
                                              inner_iters=2)).fit(X)
    save_model(idx, OUT / "flat_opq.dpq")
    dd, id_ = idx.search(Y, 5, mode="derived", r2=100)
    np.savez(OUT / "flat_opq.npz", queries=Y, exp_der_d=dd, exp_der_i=id_, meta=json.dumps({"r": 5, "r2": 100}))
    # IVF (test_vecio.py:160-172 shape, larger)
    X = blobs(rng, 4000, 8)
    Y = blobs(rng, 10, 8)
    ivf = IVFIndex(ProductQuantizer(m=2, b=8, bbar=4, seed=0, max_iters=6), n_cells=16, seed=0,
                   coarse_iters=8).fit(X)
    save_model(ivf, OUT / "ivf_small.dpq")
    dc, ic = ivf.search(Y, 10, ma=4)
    dd, id_ = ivf.search(Y, 10, ma=4, mode="derived", r2=100)
    np.savez(OUT / "ivf_small.npz", queries=Y, exp_conv_d=dc, exp_conv_i=ic, exp_der_d=dd, exp_der_i=id_,
             meta=json.dumps({"r": 10, "r2": 100, "ma": 4}))
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
