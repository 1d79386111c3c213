"""Full-size parity runs at BASELINE.json's configs (GPU), checked through
size-independent properties plus a sampled bit-exact comparison with the
CPU oracle.

    python scripts/fullsize.py --config c3 [--n 100000000] [--queries 1024] [--check 4]

Configs (BASELINE.json configs[1..4], one GPU holds the whole database):
  c2  flat PQ 4x16 + derived 4x8, SIFT-like, N = 10M,  r2 = 1000
  c3  OPQ 4x16 + derived 4x8 (data rotated by a seeded orthogonal matrix,
      quantizer rotation undoes it), N = 100M, r2 = 2000
  c4  IVF K = 8192 + residual PQ 4x16/8, ma = 64, r2 = 1000; N = 125M
      (one of the eight 1B shards)
  c5  flat PQ 8x16 + derived 8x8, 960-d GIST-like, dsub = 120, N = 50M,
      r2 = 2000, Q = 4096

Properties checked on every query of the batch (any size):
  * distances ascending, ids unique, ids in [0, N), no padding (r <= N);
  * every returned distance equals the f64 subspace-order sum of exact
    full-table entries (dpq_debug_full_tables) of the returned code;
  * |candidate set| >= r2 and b* in [0, 254] (dpq_debug_candidates);
  * batch invariance: a sub-batch searched alone returns the same rows.
And bit-exact equality with oracle/derived_search.py (the checker) for
`--check` queries, run on forked CPU workers.

Data are seeded synthetic stand-ins (SIFT1B / GIST are not available);
codebooks are trained on the GPU (train.py) and codes encoded on the GPU
with the tensor-core encoder (dpq_encode) in chunks, so no 50-190 GB float
database is ever resident.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c2": dict(kind="flat", m=4, dsub=32, n=10_000_000, r2=1000, data="sift", opq=False),
    "c3": dict(kind="flat", m=4, dsub=32, n=100_000_000, r2=2000, data="sift", opq=True),
    "c4": dict(kind="ivf", m=4, dsub=32, n=125_000_000, r2=1000, data="sift", opq=False, cells=8192, ma=64),
    "c5": dict(kind="flat", m=8, dsub=120, n=50_000_000, r2=2000, data="gist", opq=False),
    # configs[3] at its full 1B rows on ONE GPU (~28 GB of index in HBM)
    "c4b": dict(kind="ivf", m=4, dsub=32, n=1_000_000_000, r2=1000, data="sift", opq=False, cells=8192, ma=64),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def _gen_chunk(cfg, centres, seed, start, count, device):
    """Rows [start, start+count) of the seeded database (chunked Philox)."""
    import torch

    from paper_1905_06900_b200 import datagen

    c = torch.as_tensor(np.asarray(centres), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + start // (1 << 20))
    pick = torch.randint(0, c.shape[0], (count,), generator=g, device=device)
    noise = torch.randn((count, c.shape[1]), generator=g, device=device)
    if cfg["data"] == "sift":
        return (c[pick] + noise.abs_().mul_(20.0)).round_().clamp_(0, 255)
    return (c[pick] + noise.mul_(0.05)).clamp_(0.0, 1.0)


def build(cfg, seed=42, device=None, chunk=1 << 20, nq=1024, encoder="tc"):
    """Train on 100k seeded vectors, encode N rows chunk by chunk."""
    import torch

    from paper_1905_06900_b200 import datagen, train

    device = device or torch.device("cuda", 0)
    st = datagen.seed_streams(seed)
    d = cfg["m"] * cfg["dsub"]
    if cfg["data"] == "sift":
        centres = datagen.sift_centres(st["centres"])
        tr = datagen.sift_like(st["train"], centres, 100_000)
        Y = datagen.sift_like(st["queries"], centres, nq)
    else:
        centres = datagen.gist_centres(st["centres"])
        tr = datagen.gist_like(st["train"], centres, 100_000)
        Y = datagen.gist_like(st["queries"], centres, nq)
    rot = None
    if cfg["opq"]:  # data live in a rotated frame; the quantizer's rotation undoes it
        R0 = datagen.random_orthogonal(d, seed + 3)
        tr = (tr @ R0).astype(np.float32)
        Y = (Y @ R0).astype(np.float32)
        rot = np.ascontiguousarray(R0.T)
        rot_t = torch.as_tensor(rot, device=device)
        R0_t = torch.as_tensor(R0, device=device)
    trt = torch.as_tensor(tr, device=device)
    if rot is not None:
        trt = trt @ rot_t
    t0 = time.time()
    coarse = None
    if cfg["kind"] == "ivf":
        coarse = train.kmeans_gpu(trt, cfg["cells"], 10, seed)
        trt = trt - coarse[train.coarse_assign(trt, coarse)]
    cb, der = train.train_pq(trt, cfg["m"], 16, 8, iters=10, seed=seed)
    t1 = time.time()
    n = cfg["n"]
    enc = train.make_encoder(cb, device=device, kind=encoder if cfg["dsub"] <= 128 else "torch")
    # IVF coarse assignment (ivf.py:83-101): the same tensor-core encoder with m = 1, dsub = d
    cenc = train.make_encoder(coarse.cpu().numpy()[None], device=device, kind=encoder) if coarse is not None \
        else None
    out = {"codebooks": cb, "derived": der, "queries": Y, "rotation": rot, "cfg": cfg}
    if coarse is None:
        codes = np.empty((n, cfg["m"]), np.uint16)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            x = _gen_chunk(cfg, centres, seed + 1, s, e - s, device)
            if rot is not None:
                x = (x @ R0_t) @ rot_t  # rotated data, back through the quantizer rotation
            codes[s:e] = enc(x).cpu().numpy().astype(np.uint16)
        out["codes"] = codes
    else:  # IVF: cells and codes stay on the GPU (u16 bit patterns in int16), lists sorted there
        cells_t = torch.empty(n, dtype=torch.int32, device=device)
        codes_t = torch.empty((n, cfg["m"]), dtype=torch.int16, device=device)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            x = _gen_chunk(cfg, centres, seed + 1, s, e - s, device)
            if rot is not None:
                x = (x @ R0_t) @ rot_t
            cl = cenc(x)[:, 0].long()
            cells_t[s:e] = cl.to(torch.int32)
            codes_t[s:e] = enc(x - coarse[cl]).to(torch.int16)
            del x, cl
        sorted_cells, order = torch.sort(cells_t, stable=True)
        counts = torch.bincount(cells_t, minlength=cfg["cells"])
        del sorted_cells
        offsets = np.zeros(cfg["cells"] + 1, np.int64)
        offsets[1:] = np.cumsum(counts.cpu().numpy())
        out.update(centers=coarse.cpu().numpy(), offsets=offsets,
                   sorted_codes=codes_t[order].cpu().numpy().view(np.uint16),
                   sorted_ids=order.cpu().numpy(), cell_of=cells_t.cpu().numpy().astype(np.int64))
        del cells_t, codes_t, order
        torch.cuda.empty_cache()
    t2 = time.time()
    log(f"[fullsize] train {t1 - t0:.1f}s, generate+encode {n} rows {t2 - t1:.1f}s")
    return out


def make_index(w, device=0):
    if w["cfg"]["kind"] == "flat":
        from paper_1905_06900_b200.flat import FlatIndex

        return FlatIndex.from_arrays(w["codebooks"], w["derived"], w["codes"], rotation=w["rotation"],
                                     device=device)
    from paper_1905_06900_b200.ivf import IVFIndex

    return IVFIndex.from_arrays(w["codebooks"], w["derived"], w["centers"], w["offsets"], w["sorted_codes"],
                                w["sorted_ids"], cell_of=w["cell_of"], rotation=w["rotation"], device=device)


# ----------------------------------------------------- CPU reference --

_W = {}
REF_PATH = ROOT / "baseline" / "_ref"


def _reference_index(w):
    """The unmodified reference (derivedpq, baseline/_ref) over the same
    arrays: fitted attributes set directly, codes / inverted lists injected
    (SURVEY 8c).  None when the reference is not installed."""
    if str(REF_PATH) not in sys.path:
        sys.path.insert(0, str(REF_PATH))
    try:
        from derivedpq import FlatIndex as RFlat, IVFIndex as RIVF, ProductQuantizer
    except ImportError:
        return None
    cb, der = w["codebooks"], w["derived"]
    m, k, dsub = cb.shape
    kbar = der.shape[1]
    pq = ProductQuantizer(m=m, b=int(k).bit_length() - 1, bbar=int(kbar).bit_length() - 1, seed=42)
    pq.codebooks_, pq.derived_codebooks_ = cb, der
    pq.derived_assignments_ = np.tile((np.arange(k) & (kbar - 1)).astype(np.int32), (m, 1))
    pq.distortions_ = np.zeros(m)
    pq.rotation_ = w["rotation"]
    pq.d_, pq.dsub_, pq.k_, pq.kbar_, pq.bbar_ = m * dsub, dsub, k, kbar, int(kbar).bit_length() - 1
    pq.code_dtype_ = np.uint16
    if w["cfg"]["kind"] == "flat":
        idx = RFlat(pq)
        idx.codes_ = w["codes"]
        idx.n_ = w["codes"].shape[0]
        return idx
    idx = RIVF(pq, n_cells=w["centers"].shape[0])
    idx.centers_ = w["centers"]
    idx.sorted_ids_ = w["sorted_ids"]
    idx.sorted_codes_ = w["sorted_codes"]
    idx.offsets_ = w["offsets"]
    idx.cell_of_ = w["cell_of"]
    n = w["sorted_ids"].shape[0]
    idx.row_of_ = np.empty(n, dtype=np.int64)
    idx.row_of_[w["sorted_ids"]] = np.arange(n)
    idx.n_ = n
    return idx


def _ref_worker(qi):
    w = _W
    cfg = w["cfg"]
    y = w["queries"][qi: qi + 1]
    if w["ref"] is not None:
        kw = {"ma": cfg["ma"]} if cfg["kind"] == "ivf" else {}
        d, i = w["ref"].search(y, w["r"], mode="derived", r2=cfg["r2"], **kw)
        return qi, d[0], i[0]
    from oracle import derived_search as O  # labelled fallback: the oracle port

    if cfg["kind"] == "flat":
        d, i = O.flat_search(w["codebooks"], w["derived"], w["codes"], y, w["r"], "derived", cfg["r2"],
                             rotation=w["rotation"])
    else:
        row_of = np.empty_like(w["sorted_ids"])
        row_of[w["sorted_ids"]] = np.arange(w["sorted_ids"].shape[0])
        iv = {"centers": w["centers"], "offsets": w["offsets"], "sorted_codes": w["sorted_codes"],
              "sorted_ids": w["sorted_ids"], "cell_of": w["cell_of"], "row_of": row_of,
              "codebooks": w["codebooks"], "derived": w["derived"], "bbar": 8,
              "rotate": O.make_rotate(w["rotation"])}
        d, i = O.ivf_search(iv, y, w["r"], ma=cfg["ma"], mode="derived", r2=cfg["r2"])
    return qi, d[0], i[0]


def reference_rows(w, qis, r):
    """Results of the given query rows from the unmodified reference (or,
    when it is not installed, the oracle port) on forked CPU workers."""
    import multiprocessing as mp

    from threadpoolctl import threadpool_limits

    _W.clear()
    _W.update(w)
    _W["r"] = r
    _W["ref"] = _reference_index(w)
    procs = max(1, min(len(qis), os.cpu_count() or 1))
    with threadpool_limits(1), mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_worker, list(qis))
    kind = "reference" if _W["ref"] is not None else "port"
    return {qi: (d, i) for qi, d, i in res}, kind


# -------------------------------------------------------------- checks --

def check(w, r=100, check_queries=4, sub=8, device=0):
    cfg = w["cfg"]
    idx = make_index(w, device=device)
    Y = w["queries"]
    kw = dict(mode="derived", r2=cfg["r2"])
    if cfg["kind"] == "ivf":
        kw["ma"] = cfg["ma"]
    t = time.time()
    d, i = idx.search(Y, r, **kw)  # first call: sizes buffers
    t_first = time.time() - t
    t = time.time()
    d, i = idx.search(Y, r, **kw)
    t_second = time.time() - t
    n = cfg["n"]
    rep = {"config": {k: v for k, v in cfg.items()}, "queries": int(Y.shape[0]), "r": r,
           "search_s_first": round(t_first, 4), "search_s": round(t_second, 4),
           "qps_host": round(Y.shape[0] / t_second, 1)}
    # ---- ordering / ids
    assert np.all(np.isfinite(d)) and np.all(i >= 0) and np.all(i < n), "padding or id out of range"
    assert np.all(np.diff(d, axis=1) >= 0), "distances not ascending"
    assert all(len(np.unique(row)) == r for row in i), "duplicate ids"
    ties = (np.diff(d, axis=1) == 0)
    assert np.all(np.diff(i, axis=1)[ties] > 0), "ties not in ascending id order"
    # ---- distances = f64 sums of exact full-table entries of the returned codes
    m = cfg["m"]
    nt = min(Y.shape[0], 64)
    if cfg["kind"] == "flat":
        tabs = idx.full_tables(Y[:nt])  # (nt, m, k) exact f32 entries (bitwise numpy, other tests)
        cods = w["codes"][i[:nt]]  # (nt, r, m)
        acc = np.zeros((nt, r))
        for j in range(m):
            acc += np.take_along_axis(tabs[:, j, :], cods[:, :, j].astype(np.int64), axis=1).astype(np.float64)
        assert np.array_equal(acc, d[:nt]), "distance != f64 sum of exact table entries"
        bstar, ncand = idx.candidate_counts(Y, cfg["r2"])
        assert np.all(ncand >= min(cfg["r2"], n)) and np.all((bstar >= 0) & (bstar <= 254))
        rep.update(bstar_median=float(np.median(bstar)), bstar_max=int(bstar.max()),
                   candidates_mean=float(ncand.mean()), candidates_max=int(ncand.max()))
        c = idx._handle().counters()

    elif w["rotation"] is None:  # ivf: each distance = f64 sum of exact entries in its own cell frame (ivf.py:253-268)
        from paper_1905_06900_b200.flat import FlatIndex

        tab_idx = FlatIndex.from_arrays(w["codebooks"], w["derived"], w["sorted_codes"][:1], rotation=w["rotation"],
                                        device=device)
        row_of = np.empty_like(w["sorted_ids"])
        row_of[w["sorted_ids"]] = np.arange(w["sorted_ids"].shape[0])
        nt = min(Y.shape[0], 16)
        ok = 0
        for q in range(nt):
            cells = w["cell_of"][i[q]]
            ucells, inv = np.unique(cells, return_inverse=True)
            res = (Y[q][None, :] - w["centers"][ucells]).astype(np.float32)  # ivf.py:120, f32
            tabs = tab_idx.full_tables(res)  # quantizer.rotate in the (ma, d) shape is applied inside
            cods = w["sorted_codes"][row_of[i[q]]].astype(np.int64)
            acc = np.zeros(r)
            for j in range(m):
                acc += tabs[inv, j, cods[:, j]].astype(np.float64)
            ok += int(np.array_equal(acc, d[q]))
        assert ok == nt, f"ivf distance recompute {ok}/{nt}"
        rep["ivf_distance_recompute_queries"] = nt
    # ---- batch invariance
    sel = np.linspace(0, Y.shape[0] - 1, sub).astype(int)
    d2, i2 = idx.search(Y[sel], r, **kw)
    assert np.array_equal(i2, i[sel]) and np.array_equal(d2, d[sel]), "batch invariance"
    rep["properties"] = "ok"
    # ---- phase split (CUDA events per batch, amortised per query)
    _, _, tm = idx.search(Y, r, return_timings=True, **kw)
    rep["phase_us_per_query"] = {k2: round(float(v.mean()), 3) for k2, v in tm.items()}
    rep["counters"] = idx._handle().counters_ex() if cfg["kind"] == "flat" else idx._handle().counters()
    if True:
        pm = idx._handle().phase_ms()
        rep["last_batch_ms"] = dict(zip(("tables", "guard", "scan", "threshold", "refine", "fallback", "total"),
                                        [round(float(v), 4) for v in pm]))
    # ---- the unmodified reference (CPU), sampled queries
    if check_queries:
        qis = np.linspace(0, Y.shape[0] - 1, check_queries).astype(int)
        t = time.time()
        orc, kind = reference_rows(w, qis, r)
        same_i = sum(bool(np.array_equal(orc[q][1], i[q])) for q in qis)
        same_d = sum(bool(np.array_equal(orc[q][0].view(np.uint64), d[q].view(np.uint64))) for q in qis)
        rep["oracle"] = {"queries": len(qis), "ids_identical": same_i, "dists_identical": same_d,
                         "against": kind, "cpu_s": round(time.time() - t, 1)}
        assert same_i == len(qis) and same_d == len(qis), f"reference mismatch {rep['oracle']}"
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--check", type=int, default=64, help="queries checked against the unmodified reference")
    ap.add_argument("--encoder", default="tc", choices=["tc", "torch"])
    ap.add_argument("--r2", type=int, default=None, help="override the config's r2 (the paper uses 9k-200k)")
    ap.add_argument("--r", type=int, default=100, help="results per query (k)")
    a = ap.parse_args()
    cfg = dict(CONFIGS[a.config])
    if a.n:
        cfg["n"] = a.n
    if a.r2:
        cfg["r2"] = a.r2
    nq = a.queries or (4096 if a.config == "c5" else 1024)
    t = time.time()
    w = build(cfg, nq=nq, encoder=a.encoder)
    setup = time.time() - t
    rep = check(w, r=a.r, check_queries=a.check)
    rep["setup_s"] = round(setup, 1)
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
