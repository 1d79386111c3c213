"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports /root/reference/pkg/src):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [case ...]

Every expected value in the .npz files is produced by the unmodified
`derivedpq` package: its trainers (small cases), its compute_tables /
quantize_tables / scan_derived / CappedBuckets walk / nns_derived /
FlatIndex.search / IVFIndex.search.  The GPU box has no /root/reference, so
tests compare the oracle and the CUDA path against these files.

The config-1-shape case (`c1_sampled`, PQ 4x16 / derived 4x8 at N=100k,
Q=100, r2=1000, r=100) cannot use the reference k-means trainer (hours, and
it rejects BASELINE's 50k training set): its full
codebooks are 65,536 seeded training sub-vectors per subspace re-ordered by
a balanced partition (stored as `perm`), its derived codebooks the group
means — a valid model in the reference's own invariant (quantizer.py:
250-266), checked with the reference's validate().  Codes come from the
reference encoder.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from derivedpq import FlatIndex, IVFIndex, OptimizedProductQuantizer, ProductQuantizer  # noqa: E402
from derivedpq.clustering import kmeans  # noqa: E402
from derivedpq.quantizer import build_final_codebook  # noqa: E402
from derivedpq.search import compute_tables  # noqa: E402
from derivedpq.twopass import nns_derived, quantize_tables, scan_derived  # noqa: E402

from paper_1905_06900_b200 import datagen  # noqa: E402


def walk(buckets, r2):
    """refine's bucket walk (twopass.py:295-302) -> (last bucket, count)."""
    taken, last = 0, -1
    for b in range(buckets.bound):
        ids = buckets.bucket_ids(b)
        if ids.size == 0:
            continue
        taken += ids.size
        last = b
        if taken >= r2:
            break
    return last, taken


def flat_case(name, pq, X, queries, r, r2, store_codebooks=True, extra=None):
    t0 = time.time()
    index = FlatIndex(pq).fit(X)
    codes = index.codes_
    out = {
        "derived": pq.derived_codebooks_,
        "codes": codes,
        "queries": queries,
    }
    if store_codebooks:
        out["codebooks"] = pq.codebooks_
    if pq.rotation_ is not None:
        out["rotation"] = pq.rotation_
    nq = queries.shape[0]
    m, kbar = pq.m, pq.kbar_
    small_all = np.empty((nq, m, kbar), np.float32)
    q_all = np.empty((nq, m, kbar), np.uint8)
    qmin = np.empty(nq)
    qmax = np.empty(nq)
    bwalk = np.empty(nq, np.int32)
    ncand = np.empty(nq, np.int64)
    for qi in range(nq):
        yr = pq.rotate(queries[qi : qi + 1]).reshape(-1)
        small = compute_tables(yr, pq.derived_codebooks_)
        qt = quantize_tables(small, codes[: min(r2, codes.shape[0])], r2)
        buckets = scan_derived(codes, qt, r2)
        small_all[qi], q_all[qi] = small, qt.q
        qmin[qi], qmax[qi] = qt.qmin, qt.qmax
        bwalk[qi], ncand[qi] = walk(buckets, r2)
    out.update(exp_small=small_all, exp_q=q_all, exp_qmin=qmin, exp_qmax=qmax,
               exp_bwalk=bwalk, exp_ncand=ncand)
    d, i = index.search(queries, r, mode="derived", r2=r2)
    out.update(exp_derived_d=d, exp_derived_i=i)
    # uncapped, same budget: identical results (twopass.py:171-201)
    d2, i2 = index.search(queries, r, mode="derived", r2=r2, capped=False)
    assert np.array_equal(i, i2) and np.array_equal(d, d2)
    # full budget, uncapped: the exhaustive result (test_search_derived.py:339-357)
    if codes.shape[0] <= 20000:
        df, i_f = index.search(queries[:4], min(r, 10), mode="derived", r2=codes.shape[0], capped=False)
        out.update(exp_full_d=df, exp_full_i=i_f)
        dc, ic = index.search(queries, r)
        out.update(exp_conv_d=dc, exp_conv_i=ic)
    meta = {"kind": "flat", "m": m, "b": int(pq.b), "bbar": int(pq.bbar_), "r": r, "r2": r2,
            "n": int(codes.shape[0]), "seconds": round(time.time() - t0, 1)}
    meta.update(extra or {})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, meta, flush=True)


def ivf_case(name, pq, X, queries, n_cells, r, r2, ma):
    t0 = time.time()
    index = IVFIndex(pq, n_cells=n_cells, seed=0).fit(X)
    out = {
        "codebooks": pq.codebooks_, "derived": pq.derived_codebooks_,
        "centers": index.centers_, "offsets": index.offsets_,
        "sorted_codes": index.sorted_codes_, "sorted_ids": index.sorted_ids_,
        "cell_of": index.cell_of_, "queries": queries,
    }
    if pq.rotation_ is not None:
        out["rotation"] = pq.rotation_
    cells = np.stack([index.probe(y, ma)[0] for y in queries])
    out["exp_cells"] = cells
    d, i = index.search(queries, r, ma=ma, mode="derived", r2=r2)
    out.update(exp_derived_d=d, exp_derived_i=i)
    dc, ic = index.search(queries, r, ma=ma)
    out.update(exp_conv_d=dc, exp_conv_i=ic)
    df, i_f = index.search(queries[:4], 8, ma=n_cells, mode="derived", r2=index.n_, capped=False)
    out.update(exp_full_d=df, exp_full_i=i_f)
    meta = {"kind": "ivf", "m": pq.m, "b": int(pq.b), "bbar": int(pq.bbar_), "r": r, "r2": r2,
            "ma": ma, "n_cells": n_cells, "n": int(index.n_), "seconds": round(time.time() - t0, 1)}
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, meta, flush=True)


def case_pq_blobs():
    X = datagen.gaussian_blobs(6000, 16, 24, seed=911)
    Q = datagen.gaussian_blobs(24, 16, 24, seed=912)
    flat_case("pq_blobs", ProductQuantizer(m=4, b=8, bbar=4, seed=0), X, Q, r=10, r2=300)


def case_pq_m2():
    X = datagen.gaussian_blobs(3000, 8, 10, seed=913)
    Q = datagen.gaussian_blobs(16, 8, 10, seed=914)
    flat_case("pq_m2", ProductQuantizer(m=2, b=5, bbar=3, seed=2), X, Q, r=5, r2=100)


def case_pq_m8():
    X = datagen.gaussian_blobs(4000, 32, 16, seed=915)
    Q = datagen.gaussian_blobs(16, 32, 16, seed=916)
    flat_case("pq_m8", ProductQuantizer(m=8, b=8, seed=3), X, Q, r=10, r2=250)


def case_opq_blobs():
    X = datagen.gaussian_blobs(5000, 16, 24, seed=917)
    Q = datagen.gaussian_blobs(16, 16, 24, seed=918)
    flat_case("opq_blobs", OptimizedProductQuantizer(m=4, b=6, bbar=3, seed=0, outer_iters=3), X, Q,
              r=10, r2=200)


def case_ivf_blobs():
    X = datagen.gaussian_blobs(6000, 16, 24, seed=919)
    rng = np.random.default_rng(920)
    Q = X[rng.choice(6000, size=20, replace=False)] + rng.normal(0, 0.02, size=(20, 16)).astype(np.float32)
    ivf_case("ivf_blobs", ProductQuantizer(m=4, b=6, bbar=3, seed=0), X, Q.astype(np.float32),
             n_cells=16, r=10, r2=400, ma=4)


def case_ivf_opq():
    X = datagen.gaussian_blobs(4000, 16, 20, seed=921)
    Q = datagen.gaussian_blobs(12, 16, 20, seed=922)
    ivf_case("ivf_opq", OptimizedProductQuantizer(m=4, b=5, bbar=3, seed=1, outer_iters=2), X, Q,
             n_cells=8, r=8, r2=300, ma=3)


def c1_model(seed=datagen.SEED):
    """Config-1-shape 4x16/8 model: see module docstring.  Returns
    (codebooks, derived, perm, streams)."""
    st = datagen.seed_streams(seed)
    centres = datagen.sift_centres(st["centres"])
    train = datagen.sift_like(st["train"], centres, 100_000)
    m, k, kbar, dsub = 4, 65536, 256, 32
    pick = np.random.default_rng(seed + 7).choice(train.shape[0], size=k, replace=False)
    temp = np.ascontiguousarray(train[pick])
    cbs, ders, perms = [], [], []
    for j in range(m):
        sub = np.ascontiguousarray(temp[:, j * dsub:(j + 1) * dsub])
        groups = balanced_groups(sub, kbar, seed + j)
        perm = build_perm(groups, 8)
        cbs.append(sub[perm])
        ders.append(np.stack([sub[g].astype(np.float64).mean(axis=0) for g in groups]).astype(np.float32))
        perms.append(perm.astype(np.uint16))
    return np.stack(cbs), np.stack(ders), np.stack(perms), st, centres


def balanced_groups(points, kbar, seed):
    """kbar equal-size groups: reference k-means (few iterations) for
    centres, then greedy capacity assignment by margin (the idea of
    clustering.py:182-203, vectorised here)."""
    km = kmeans(points, kbar, seed=seed, max_iters=8)
    c = km.centroids.astype(np.float64)
    p = points.astype(np.float64)
    d2 = (p * p).sum(1)[:, None] - 2 * p @ c.T + (c * c).sum(1)[None, :]
    cap = points.shape[0] // kbar
    two = np.partition(d2, 1, axis=1)[:, :2]
    order = np.argsort(two[:, 0] - two[:, 1], kind="stable")
    ranked = np.argsort(d2, axis=1, kind="stable")
    room = np.full(kbar, cap)
    label = np.empty(points.shape[0], np.int64)
    for pt in order:
        for cc in ranked[pt]:
            if room[cc]:
                label[pt] = cc
                room[cc] -= 1
                break
    return [np.flatnonzero(label == g) for g in range(kbar)]


def build_perm(groups, bbar):
    perm = np.empty(sum(len(g) for g in groups), np.int64)
    for gid, members in enumerate(groups):
        for ibar, old in enumerate(members):
            perm[(ibar << bbar) | gid] = old
    return perm


def case_c1_sampled():
    t0 = time.time()
    cb, der, perm, st, centres = c1_model()
    pq = ProductQuantizer(m=4, b=16, bbar=8, seed=42)
    pq.codebooks_, pq.derived_codebooks_ = cb, der
    pq.derived_assignments_ = np.tile((np.arange(65536) & 255).astype(np.int32), (4, 1))
    pq.distortions_ = np.zeros(4)
    pq.rotation_ = None
    pq.d_, pq.dsub_, pq.bbar_, pq.k_, pq.kbar_ = 128, 32, 8, 65536, 256
    pq.code_dtype_ = np.uint16
    pq.validate()
    # re-check the temp partition -> build_final_codebook equivalence
    X = datagen.sift_like(st["database"], centres, 100_000)
    Q = datagen.sift_like(st["queries"], centres, 100)
    print("c1 model built", round(time.time() - t0, 1), flush=True)
    flat_case("c1_sampled", pq, X, Q, r=100, r2=1000, store_codebooks=False,
              extra={"perm_note": "codebooks = train[pick][:, j] reordered by perm[j]"})
    z = dict(np.load(HERE / "c1_sampled.npz"))
    z["perm"] = perm
    np.savez_compressed(HERE / "c1_sampled.npz", **z)
    _ = build_final_codebook  # reference helper, same mapping as build_perm


CASES = {
    "pq_blobs": case_pq_blobs, "pq_m2": case_pq_m2, "pq_m8": case_pq_m8,
    "opq_blobs": case_opq_blobs, "ivf_blobs": case_ivf_blobs, "ivf_opq": case_ivf_opq,
    "c1_sampled": case_c1_sampled,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
